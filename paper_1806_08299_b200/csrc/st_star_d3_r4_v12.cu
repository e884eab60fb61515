// Star kernels, DIMS=3, R=4, shape variant 12 (14 warps x 2 rows, coded-m operand stage).
#include "st_star_inst.cuh"
ST_STAR_LOOKUP_V(star_lookup_d3_r4_v12, 4, 3, 12)
