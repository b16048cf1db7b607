// run-time parameter kernel instances (custom engines) for shapes [3, 6)
#define SLP_RT_PART 1
#define SLP_RT_LO 3
#define SLP_RT_HI 6
#include "slp_inst_rt_common.cuh"
