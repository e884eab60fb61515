// st_star_inst.cuh -- explicit instantiation helper: each st_star_*.cu TU
// instantiates the star kernels of one (R, DIMS) pair and exposes a lookup.
#pragma once
#include "st_kernels.cuh"

#define ST_STAR_LOOKUP(NAME, R, DIMS)                                      \
  namespace st {                                                              \
  void* NAME(int model, int fast, int wf) {                                   \
    if (model == kTerms) {                                                    \
      if (!fast && !wf) return (void*)&star_kernel<R, DIMS, kTerms, false, false>; \
      if (!fast && wf) return (void*)&star_kernel<R, DIMS, kTerms, false, true>;   \
      if (fast && !wf) return (void*)&star_kernel<R, DIMS, kTerms, true, false>;   \
      return (void*)&star_kernel<R, DIMS, kTerms, true, true>;            \
    }                                                                         \
    if (!fast && !wf) return (void*)&star_kernel<R, DIMS, kWave, false, false>;   \
    if (!fast && wf) return (void*)&star_kernel<R, DIMS, kWave, false, true>;     \
    if (fast && !wf) return (void*)&star_kernel<R, DIMS, kWave, true, false>;     \
    return (void*)&star_kernel<R, DIMS, kWave, true, true>;               \
  }                                                                           \
  }
