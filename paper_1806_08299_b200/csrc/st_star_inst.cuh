// st_star_inst.cuh -- explicit instantiation helper: each st_star_*.cu TU
// instantiates the star kernels of one (R, DIMS) pair and exposes a lookup.
#pragma once
#include "st_kernels.cuh"

#define ST_STAR_LOOKUP(NAME, R, DIMS, VY)                                      \
  namespace st {                                                              \
  void* NAME(int model, int fast, int wf) {                                   \
    if (model == kTerms) {                                                    \
      if (!fast && !wf) return (void*)&star_kernel<R, DIMS, VY, kTerms, false, false>; \
      if (!fast && wf) return (void*)&star_kernel<R, DIMS, VY, kTerms, false, true>;   \
      if (fast && !wf) return (void*)&star_kernel<R, DIMS, VY, kTerms, true, false>;   \
      return (void*)&star_kernel<R, DIMS, VY, kTerms, true, true>;            \
    }                                                                         \
    if (!fast && !wf) return (void*)&star_kernel<R, DIMS, VY, kWave, false, false>;   \
    if (!fast && wf) return (void*)&star_kernel<R, DIMS, VY, kWave, false, true>;     \
    if (fast && !wf) return (void*)&star_kernel<R, DIMS, VY, kWave, true, false>;     \
    return (void*)&star_kernel<R, DIMS, VY, kWave, true, true>;               \
  }                                                                           \
  }
