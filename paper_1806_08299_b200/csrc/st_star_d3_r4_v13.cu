// Star kernels, DIMS=3, R=4, shape variant 13 (12 warps x 2 rows, coded-m operand stage, 4-plane prefetch).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r4_v13, 4, 3, 13)
