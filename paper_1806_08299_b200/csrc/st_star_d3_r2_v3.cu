// Star kernels, DIMS=3, R=2, shape variant 3 (tuning experiments).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r2_v3, 2, 3, 3)
