// kernel instances for registry ids [25, 27)
#define SLP_INST_PART 5
#define SLP_INST_LO 25
#define SLP_INST_HI 27
#include "slp_inst_common.cuh"
