// Star kernels, DIMS=3, R=4, shape variant 6 (16 warps x 1 row, unrolled window).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r4_v6, 4, 3, 6)
