// Star kernels, DIMS=3, R=4.
#include "st_star_inst.cuh"
ST_STAR_LOOKUP(star_lookup_d3_r4, 4, 3)
