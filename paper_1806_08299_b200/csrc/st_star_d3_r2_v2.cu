// Star kernels, DIMS=3, R=2, shape variant 2 (tuning experiments).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r2_v2, 2, 3, 2)
