// Fused-level kernels, DIMS=3, R=1 (heat so2): F = 1 .. 4.
#include "st_fused.cuh"

namespace st {

FusedFn fused_lookup_d3_r1(int F, int ty, int fast) {
  (void)ty;
  if (F == 1) return fused_entry<1, 1, 16, 2, 8>(fast);
  if (F == 2) return fused_entry<1, 2, 16, 2, 6>(fast);
  if (F == 3) return fused_entry<1, 3, 16, 2, 4>(fast);
  if (F == 4) return fused_entry<1, 4, 8, 2, 6>(fast);
  return FusedFn{};
}

}  // namespace st
