// Fused-level kernels, DIMS=3, R=2 (config 2's heat so4): F = 1, 2, 3.
#include "st_fused.cuh"

namespace st {

template <int R, int F, int TY, int VY, int PD>
static FusedFn fused_entry(int fast) {
  constexpr FusedShape s = fused_shape(R, F, TY, VY, PD);
  FusedFn f{};
  f.fn = fast ? (void*)&fused_kernel<R, F, TY, VY, PD, true> : (void*)&fused_kernel<R, F, TY, VY, PD, false>;
  f.threads = fused_threads(R, F, TY, VY, PD);
  f.smem = fused_smem_bytes(R, F, TY, VY, PD);
  f.ty = TY;
  f.bw = s.BW;
  f.bh = s.BH;
  return f;
}

FusedFn fused_lookup_d3_r2(int F, int ty, int fast) {
  if (F == 1) return fused_entry<2, 1, 16, 2, 8>(fast);
  if (F == 2) return ty >= 24 ? fused_entry<2, 2, 24, 2, 6>(fast) : fused_entry<2, 2, 16, 2, 8>(fast);
  if (F == 3) return fused_entry<2, 3, 8, 2, 8>(fast);
  return FusedFn{};
}

}  // namespace st
