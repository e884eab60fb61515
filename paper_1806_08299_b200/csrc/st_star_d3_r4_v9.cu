// Star kernels, DIMS=3, R=4, shape variant 9 (14 warps x 2 rows, 28-row tile).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r4_v9, 4, 3, 9)
