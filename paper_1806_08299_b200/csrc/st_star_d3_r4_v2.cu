// Star kernels, DIMS=3, R=4, shape variant 2 (tuning experiments).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r4_v2, 4, 3, 2)
