// kernel instances for registry ids [13, 18)
#define SLP_INST_PART 3
#define SLP_INST_LO 13
#define SLP_INST_HI 18
#include "slp_inst_common.cuh"
