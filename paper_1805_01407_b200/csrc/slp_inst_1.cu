// kernel instances for registry ids [5, 9)
#define SLP_INST_PART 1
#define SLP_INST_LO 5
#define SLP_INST_HI 9
#include "slp_inst_common.cuh"
