// Instantiates the device kernels of registry entries [SLP_INST_LO, SLP_INST_HI)
// into the dispatch table slp_ops_part_<SLP_INST_PART>.  Split over several
// translation units so nvcc compiles the ~27 generator instances in parallel.
#include "slp_device.cuh"

namespace slp {
namespace dev {
template <bool On, class G>
struct MaybeOps {
  static GenOps get() { return make_ops<G>(); }
};
template <class G>
struct MaybeOps<false, G> {
  static GenOps get() { return GenOps{}; }
};
}  // namespace dev
}  // namespace slp

#define SLP_CAT2(a, b) a##b
#define SLP_CAT(a, b) SLP_CAT2(a, b)
#define SLP_INST_X(id, name, fam, k, w, a, b, c, sc, wi, wj, S, R, T)                      \
  ::slp::dev::MaybeOps<((id) >= SLP_INST_LO && (id) < SLP_INST_HI),                          \
                       SLP_GEN_TYPE(id, name, fam, k, w, a, b, c, sc, wi, wj, S, R, T)>::get(),

extern const ::slp::GenOps SLP_CAT(slp_ops_part_, SLP_INST_PART)[SLP_NUM_GENERATORS];
const ::slp::GenOps SLP_CAT(slp_ops_part_, SLP_INST_PART)[SLP_NUM_GENERATORS] = {SLP_REGISTRY(SLP_INST_X)};
