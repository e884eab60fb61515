// Fused-level kernels, DIMS=3, R=1: heat (so2) F = 1 .. 4; wave F = 1 .. 3.
#include "st_fused.cuh"

namespace st {

FusedFn fused_lookup_d3_r1(int F, int ty, int fast, int model) {
  if (model == kWave) {
    if (F == 1) return fused_entry<1, 1, 16, 2, 4, kWave>(fast);
    if (F == 2) return fused_entry<1, 2, 16, 2, 3, kWave>(fast);
    if (F == 3) return fused_entry<1, 3, 16, 2, 1, kWave>(fast);
    return FusedFn{};
  }
  if (F == 1) return fused_entry<1, 1, 16, 2, 8>(fast);
  if (F == 2) return fused_entry<1, 2, 16, 2, 6>(fast);
  // <= 12 warps per CTA: 3 per SMSP keeps ~168 registers (a 13th warp caps
  // them at 128 through the per-SMSP register file, and F = 4 spills)
  if (F == 3) return ty >= 24 ? fused_entry<1, 3, 24, 2, 3>(fast) : fused_entry<1, 3, 16, 2, 4>(fast);
  if (F == 4) return ty > 0 && ty <= 8 ? fused_entry<1, 4, 8, 2, 6>(fast) : fused_entry<1, 4, 14, 2, 4>(fast);
  return FusedFn{};
}

}  // namespace st
