// Star kernels, DIMS=3, R=8, shape variant 7 (12 warps x 1 row).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r8_v7, 8, 3, 7)
