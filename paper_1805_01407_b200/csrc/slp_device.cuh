// Device templates for the scrambled linear generators on sm_100a.
//
// One template instance per registry generator (slp_registry.h): the whole
// state lives in registers in FLAT word order (engines.py:14-18).  The cyclic
// engines (xoroshiro, incl. the 16-word ring of xoroshiro1024, and xorshift)
// are stepped as a register ring whose offset is a compile-time constant
// inside fully unrolled chunks of a multiple of k steps, so the reference's
// ring pointer (generators.py:260-274) costs nothing at run time.
//
// Kernels (paths relative to /root/reference/pkg/src/slprng/):
//   K1    k_jump        state * p(M) as sum of state*M^d (generators.py:315-334, :493-505)  slp_jump.cuh
//   K1t   k_jump_table  the same by four-Russians tables of the jump matrix                  slp_jump.cuh
//   K2/K3 k_fill        scramble + step + convert + store (generators.py:244-311, :465-490) slp_fill.cuh
//   K4    k_fused       scramble + step + in-register reduction (new)                        slp_fused.cuh
//   K6    k_hwd         Hamming-weight-dependency counting (hwd.py:206-247)                  slp_hwd.cuh
// Word operations, Gen<>, conversions and PTX helpers: slp_gen.cuh.  This
// header adds the per-generator dispatch table (make_ops).
#pragma once

#include "slp_fill.cuh"
#include "slp_fused.cuh"
#include "slp_hwd.cuh"
#include "slp_jump.cuh"

namespace slp {
namespace dev {

template <class G>
GenOps make_ops() {
  GenOps o;
  o.fill = &fill_impl<G>;
  o.fill_csum = &fill_csum_impl<G>;
  o.fused = &fused_impl<G>;
  o.fused_grid_cap = &fused_grid_cap<G>;
  o.jump = &jump_impl<G>;
  o.hwd = &hwd_impl<G>;
  o.table_words = &table_words_impl<G>;
  o.build_table = &build_table_impl<G>;
  o.jump_table = &jump_table_impl<G>;
  return o;
}

}  // namespace dev
}  // namespace slp

// Gen<> type of registry entry `id`
#define SLP_GEN_TYPE(id, name, fam, k, w, a, b, c, sc, wi, wj, S, R, T) \
  ::slp::dev::Gen<id, fam, k, w, a, b, c, sc, wi, wj, S, R, T>
