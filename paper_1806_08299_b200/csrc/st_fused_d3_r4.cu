// Fused-level kernels, DIMS=3, R=4: the leapfrog wave at F = 2 (measurement of
// SURVEY 7's radius-4 temporal blocking).  Two 9-plane windows
// per point leave room for 8-row output tiles only: level 0 runs on 136 x 16
// points per 128 x 8 outputs.
#include "st_fused.cuh"

namespace st {

FusedFn fused_lookup_d3_r4(int F, int ty, int fast, int model) {
  if (model == kWave && F == 1) return fused_entry<4, 1, 16, 2, 2, kWave>(fast);   // remainder passes
  if (model == kWave && F == 2) {
    return ty == 4 ? fused_entry<4, 2, 8, 2, 1, kWave>(fast) : fused_entry<4, 2, 8, 1, 1, kWave>(fast);
  }
  return FusedFn{};
}

}  // namespace st
