// Star kernels, DIMS=3, R=8.
#include "st_star_inst.cuh"
ST_STAR_LOOKUP(star_lookup_d3_r8, 8, 3)
