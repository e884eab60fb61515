// st_star_inst.cuh -- explicit instantiation helper: each st_star_*.cu TU
// instantiates the star kernels of one (R, DIMS[, variant]) and exposes a
// lookup.
#pragma once
#include "st_kernels.cuh"

#define ST_STAR_LOOKUP_V(NAME, R, DIMS, V)                                                  \
  namespace st {                                                                           \
  void* NAME(int model, int fast, int wf) {                                                \
    if (model == kTerms) {                                                                 \
      if (!fast && !wf) return (void*)&star_kernel<R, DIMS, kTerms, false, false, V>;      \
      if (!fast && wf) return (void*)&star_kernel<R, DIMS, kTerms, false, true, V>;        \
      if (fast && !wf) return (void*)&star_kernel<R, DIMS, kTerms, true, false, V>;        \
      return (void*)&star_kernel<R, DIMS, kTerms, true, true, V>;                          \
    }                                                                                      \
    if (!fast && !wf) return (void*)&star_kernel<R, DIMS, kWave, false, false, V>;         \
    if (!fast && wf) return (void*)&star_kernel<R, DIMS, kWave, false, true, V>;           \
    if (fast && !wf) return (void*)&star_kernel<R, DIMS, kWave, true, false, V>;           \
    return (void*)&star_kernel<R, DIMS, kWave, true, true, V>;                             \
  }                                                                                        \
  }

#define ST_STAR_LOOKUP(NAME, R, DIMS) ST_STAR_LOOKUP_V(NAME, R, DIMS, 0)
