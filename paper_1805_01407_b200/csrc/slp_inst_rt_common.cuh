// Instantiates the run-time parameter kernels (GenR<>, custom engines) of
// engine shapes [SLP_RT_LO, SLP_RT_HI) of SLP_RT_SHAPES into the dispatch
// table slp_ops_rt_<SLP_RT_PART>; split like slp_inst_common.cuh so nvcc
// compiles the shapes in parallel.
#include "slp_device.cuh"

namespace slp {
namespace dev {
template <bool On, class G>
struct MaybeOpsRt {
  static GenOps get() { return make_ops<G>(); }
};
template <class G>
struct MaybeOpsRt<false, G> {
  static GenOps get() { return GenOps{}; }
};
}  // namespace dev
}  // namespace slp

#define SLP_RT_CAT2(a, b) a##b
#define SLP_RT_CAT(a, b) SLP_RT_CAT2(a, b)
#define SLP_RT_INST_X(i, fam, k, w) \
  ::slp::dev::MaybeOpsRt<((i) >= SLP_RT_LO && (i) < SLP_RT_HI), ::slp::dev::GenR<fam, k, w>>::get(),

extern const ::slp::GenOps SLP_RT_CAT(slp_ops_rt_, SLP_RT_PART)[SLP_NUM_RT_SHAPES];
const ::slp::GenOps SLP_RT_CAT(slp_ops_rt_, SLP_RT_PART)[SLP_NUM_RT_SHAPES] = {SLP_RT_SHAPES(SLP_RT_INST_X)};
