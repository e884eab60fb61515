// Fused-level kernels, DIMS=3, R=2: heat (config 2's so4) F = 1, 2, 3; wave F = 1, 2.
#include "st_fused.cuh"

namespace st {

FusedFn fused_lookup_d3_r2(int F, int ty, int fast, int model) {
  if (model == kWave) {   // leapfrog wave: the u^{n-1} / m tiles ride in the ring
    if (F == 1) return fused_entry<2, 1, 16, 2, 4, kWave>(fast);
    if (F == 2) return fused_entry<2, 2, 16, 2, 2, kWave>(fast);
    return FusedFn{};
  }
  if (F == 1) return fused_entry<2, 1, 16, 2, 8>(fast);
  if (F == 2) return ty >= 24 ? fused_entry<2, 2, 24, 2, 6>(fast) : fused_entry<2, 2, 16, 2, 8>(fast);
  if (F == 3) return fused_entry<2, 3, 8, 2, 8>(fast);
  return FusedFn{};
}

}  // namespace st
