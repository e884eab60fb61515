// Star kernels, DIMS=3, R=2, shape variant 5 (16 rows, 4 rows per thread, 2 CTAs/SM).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r2_v5, 2, 3, 5)
