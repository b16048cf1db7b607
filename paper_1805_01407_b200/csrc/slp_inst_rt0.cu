// run-time parameter kernel instances (custom engines) for shapes [0, 3)
#define SLP_RT_PART 0
#define SLP_RT_LO 0
#define SLP_RT_HI 3
#include "slp_inst_rt_common.cuh"
