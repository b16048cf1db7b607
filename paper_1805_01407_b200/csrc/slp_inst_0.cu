// kernel instances for registry ids [0, 5)
#define SLP_INST_PART 0
#define SLP_INST_LO 0
#define SLP_INST_HI 5
#include "slp_inst_common.cuh"
