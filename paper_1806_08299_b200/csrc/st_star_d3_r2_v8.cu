// Star kernels, DIMS=3, R=2, shape variant 8 (12 warps x 2 rows, 24-row tile).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r2_v8, 2, 3, 8)
