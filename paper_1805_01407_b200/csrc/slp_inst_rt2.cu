// run-time parameter kernel instances (custom engines) for shapes [6, 9)
#define SLP_RT_PART 2
#define SLP_RT_LO 6
#define SLP_RT_HI 9
#include "slp_inst_rt_common.cuh"
