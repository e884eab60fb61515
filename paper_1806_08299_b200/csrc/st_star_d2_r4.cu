// Star kernels, DIMS=2, R=4.
#include "st_star_inst.cuh"
ST_STAR_LOOKUP(star_lookup_d2_r4, 4, 2)
