// Star kernels, DIMS=3, R=2.
#include "st_star_inst.cuh"
ST_STAR_LOOKUP(star_lookup_d3_r2, 2, 3)
