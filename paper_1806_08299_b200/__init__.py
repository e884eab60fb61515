"""B200-native executor for repeated explicit stencil sweeps (the hot path of
arXiv 1806.08299's time-tiling: untiled, space-tiled and time-tiled sweeps).

The product is ``libstencil_tiler.so`` (hand-written sm_100a kernels behind
the C-ABI in ``include/stencil_tiler.h``); ``tiler`` mirrors the reference
operator API over it and ``configs`` fixes the five benchmark
configurations.  There is no CPU compute path: if the native library is
missing, using the executor raises.
"""
from . import configs  # noqa: F401
from . import _native  # noqa: F401
from .tiler import (  # noqa: F401
    Context, DeviceGrid, Error, ExecReport, Grid, GridLayout, IterationSpace, LegalityViolation, LoopNest,
    ParseError, StencilSpec, StencilTerm, TilePlan, build_canonical_nest, check_legality, default_context,
    execute, flops_per_point, init_gaussian, init_grid, init_unit, min_skew_factor, parse_spec, required_slots,
    tile_space_minmax, tile_time, time_buffer_slots, verify_bitwise, Dist, dist_partition, nccl_unique_id,
    CacheConfig, TrafficReport, simulate, measured_ai_elems,
    MODE_FAST, MODE_REFERENCE, MODEL_TERMS, MODEL_WAVE, SCHED_CANONICAL, SCHED_SPACE, SCHED_TIME,
)

__all__ = [n for n in dir() if not n.startswith("_")]
