// kernel instances for registry ids [9, 13)
#define SLP_INST_PART 2
#define SLP_INST_LO 9
#define SLP_INST_HI 13
#include "slp_inst_common.cuh"
