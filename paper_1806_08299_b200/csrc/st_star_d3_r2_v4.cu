// Star kernels, DIMS=3, R=2, shape variant 4 (32 rows, 4 rows per thread).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r2_v4, 2, 3, 4)
