// kernel instances for registry ids [18, 25)
#define SLP_INST_PART 4
#define SLP_INST_LO 18
#define SLP_INST_HI 25
#include "slp_inst_common.cuh"
