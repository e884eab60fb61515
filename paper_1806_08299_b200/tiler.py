"""Python mirror of the reference operator API (namespace ``tiler``), executed
on the B200 through the C-ABI (include/stencil_tiler.h).

Reference -> here
  StencilTerm / StencilSpec::make      stencil.hpp:42-63    StencilTerm, StencilSpec.make
  IterationSpace, TilePlan             stencil.hpp:28-40,65 IterationSpace, TilePlan
  parse_spec                           stencil.hpp:87-97    parse_spec
  min_skew_factor / time_buffer_slots
  / flops_per_point                    stencil.hpp:99-108   same names
  build_canonical_nest                 loop_ir.hpp:111-114  build_canonical_nest
  tile_space_minmax / tile_time        transforms.hpp:29-59 same names
  check_legality                       transforms.hpp:43-51 check_legality
  GridLayout / Grid                    executor.hpp:17-56   GridLayout, Grid
  required_slots / init_grid           executor.hpp:83-90   same names
  execute                              executor.hpp:92-98   execute (on the GPU)
  verify_bitwise                       executor.hpp:107-110 verify_bitwise
  Error / ParseError                   stencil.hpp:11-26    Error / ParseError

A ``LoopNest`` here is a *schedule descriptor* (canonical / space-tiled /
time-tiled + TilePlan): the GPU realises the schedule directly instead of
interpreting an IR.  Results are bit-identical to the
reference interpreter for every legal plan in ``mode="reference"``.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N

SCHED_CANONICAL, SCHED_SPACE, SCHED_TIME = 0, 1, 2
MODEL_TERMS, MODEL_WAVE = 0, 1
MODE_REFERENCE, MODE_FAST = 0, 1

ST_OK, ST_ERR_INVALID, ST_ERR_ILLEGAL_PLAN, ST_ERR_SLOTS = 0, 1, 2, 3
ST_ERR_CUDA, ST_ERR_NCCL, ST_ERR_UNSUPPORTED, ST_ERR_PARSE, ST_ERR_STATE = 4, 5, 6, 7, 8


class Error(RuntimeError):
    """tiler::Error (stencil.hpp:12-15); carries the C-ABI status code."""

    def __init__(self, msg: str, code: int = ST_ERR_INVALID):
        super().__init__(msg)
        self.code = code


class ParseError(Error):
    """tiler::ParseError (stencil.hpp:18-26): 1-based source line."""

    def __init__(self, line: int, msg: str):
        super().__init__(msg, ST_ERR_PARSE)
        self._line = line

    def line(self) -> int:
        return self._line


def _lib():
    return N.load()


def _check(rc: int):
    if rc != ST_OK:
        msg = _lib().st_last_error().decode()
        raise Error(msg, rc)


@dataclasses.dataclass(frozen=True)
class StencilTerm:
    coeff: float
    dt: int = 1
    offsets: Tuple[int, ...] = ()


@dataclasses.dataclass(frozen=True)
class IterationSpace:
    time_steps: int
    extents: Tuple[int, ...]

    def ndims(self) -> int:
        return len(self.extents)

    def points_per_step(self) -> int:
        return int(np.prod(self.extents, dtype=np.int64))


@dataclasses.dataclass(frozen=True)
class TilePlan:
    skew: int = 0
    time_tile: int = 1
    space_tiles: Tuple[int, ...] = ()
    # executor extension (st_plan.fused_levels): levels advanced on-chip per
    # pass over memory; 0 = the wavefront realisation of tile_time
    fused_levels: int = 0
    # executor extension (st_plan.band_rows / band_skew): tile_time along d_2 too
    # -- bands of band_rows rows, skewed band_skew rows per level (0 = off)
    band_rows: int = 0
    band_skew: int = 0


@dataclasses.dataclass(frozen=True)
class LegalityViolation:
    skew: int
    required_minimum: int


class StencilSpec:
    """StencilSpec (stencil.hpp:52-63); owns an st_stencil handle."""

    def __init__(self, handle, name: str):
        self._h = C.c_void_p(handle)
        self.name = name

    @staticmethod
    def make(name: str, ndims: int, terms: Sequence[StencilTerm], model: int = MODEL_TERMS) -> "StencilSpec":
        arr = (N.st_term * max(1, len(terms)))()
        for k, t in enumerate(terms):
            arr[k].coeff = float(t.coeff)
            arr[k].dt = int(t.dt)
            for i, o in enumerate(t.offsets):
                arr[k].offsets[i] = int(o)
        h = C.c_void_p()
        _check(_lib().st_stencil_create(name.encode(), int(ndims), arr, len(terms), int(model), C.byref(h)))
        return StencilSpec(h.value, name)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and N._lib is not None:
            N._lib.st_stencil_destroy(self._h)
            self._h = C.c_void_p()

    @property
    def handle(self):
        return self._h

    @property
    def ndims(self) -> int:
        return _lib().st_stencil_ndims(self._h)

    @property
    def model(self) -> int:
        return _lib().st_stencil_model(self._h)

    @property
    def time_depth(self) -> int:
        return _lib().st_stencil_time_depth(self._h)

    @property
    def radii(self) -> List[int]:
        return [_lib().st_stencil_radius(self._h, i) for i in range(self.ndims)]

    @property
    def terms(self) -> List[StencilTerm]:
        out = []
        t = N.st_term()
        for k in range(_lib().st_stencil_nterms(self._h)):
            _check(_lib().st_stencil_term(self._h, k, C.byref(t)))
            out.append(StencilTerm(t.coeff, t.dt, tuple(t.offsets[i] for i in range(self.ndims))))
        return out


def parse_spec(text: str) -> Tuple[StencilSpec, IterationSpace]:
    """parse_spec (stencil.hpp:87-97): raises ParseError(line) on failure."""
    h = C.c_void_p()
    nd = C.c_int()
    ext = (C.c_int64 * 3)()
    steps = C.c_int64()
    line = C.c_int(0)
    rc = _lib().st_stencil_parse(text.encode(), C.byref(h), C.byref(nd), ext, C.byref(steps), C.byref(line))
    if rc == ST_ERR_PARSE:
        raise ParseError(line.value, _lib().st_last_error().decode())
    _check(rc)
    spec = StencilSpec(h.value, "")
    return spec, IterationSpace(int(steps.value), tuple(int(ext[i]) for i in range(nd.value)))


def min_skew_factor(spec: StencilSpec) -> int:
    return _lib().st_min_skew_factor(spec.handle)


def time_buffer_slots(spec: StencilSpec, time_tile: int) -> int:
    return int(_lib().st_time_buffer_slots(spec.handle, int(time_tile)))


def flops_per_point(spec: StencilSpec) -> int:
    return int(_lib().st_flops_per_point(spec.handle))


def _plan_struct(schedule: int, plan: Optional[TilePlan]) -> N.st_plan:
    p = N.st_plan()
    p.schedule = schedule
    if plan is not None:
        p.skew = int(plan.skew)
        p.time_tile = int(plan.time_tile)
        for i, t in enumerate(plan.space_tiles):
            p.space_tiles[i] = int(t)
        p.fused_levels = int(getattr(plan, "fused_levels", 0))
        p.band_rows = int(getattr(plan, "band_rows", 0))
        p.band_skew = int(getattr(plan, "band_skew", 0))
    else:
        p.time_tile = 1
    return p


def check_legality(spec: StencilSpec, plan: TilePlan) -> Optional[LegalityViolation]:
    """check_legality (transforms.hpp:43-51): None when legal."""
    req = C.c_int()
    p = _plan_struct(SCHED_TIME, plan)
    rc = _lib().st_check_legality(spec.handle, C.byref(p), C.byref(req))
    if rc == ST_OK:
        return None
    if rc == ST_ERR_ILLEGAL_PLAN:
        return LegalityViolation(plan.skew, req.value)
    _check(rc)
    return None


@dataclasses.dataclass(frozen=True)
class LoopNest:
    """Schedule descriptor standing in for the reference LoopNest."""

    schedule: int
    plan: Optional[TilePlan] = None


def build_canonical_nest(spec: StencilSpec, space: IterationSpace) -> LoopNest:
    return LoopNest(SCHED_CANONICAL, None)


def tile_space_minmax(nest: LoopNest, sizes: Sequence[int]) -> LoopNest:
    if nest.schedule != SCHED_CANONICAL:
        raise Error("tile_space_minmax: the nest must be canonical")
    if any(int(s) < 0 for s in sizes):
        raise Error("tile size < 1 (0 = executor's choice)")
    return LoopNest(SCHED_SPACE, TilePlan(0, 1, tuple(int(s) for s in sizes)))


def tile_time(nest: LoopNest, spec: StencilSpec, space: IterationSpace, plan: TilePlan) -> LoopNest:
    if nest.schedule != SCHED_CANONICAL:
        raise Error("tile_time: the nest must be canonical")
    v = check_legality(spec, plan)
    if v is not None:
        raise Error(f"illegal plan: skew {v.skew} < minimum skew factor {v.required_minimum}", ST_ERR_ILLEGAL_PLAN)
    if plan.time_tile < 1 or any(int(s) < 0 for s in plan.space_tiles):
        raise Error("tile sizes must be >= 1 (0 = executor's choice)")
    return LoopNest(SCHED_TIME, plan)


def required_slots(nest: LoopNest, spec: StencilSpec) -> int:
    p = _plan_struct(nest.schedule, nest.plan)
    return int(_lib().st_required_slots(spec.handle, C.byref(p)))


@dataclasses.dataclass
class GridLayout:
    slots: int
    time_depth: int
    interior: Tuple[int, ...]
    halo: Tuple[int, ...]

    @property
    def padded(self) -> Tuple[int, ...]:
        return tuple(d + 2 * h for d, h in zip(self.interior, self.halo))

    def plane(self) -> int:
        return int(np.prod(self.padded, dtype=np.int64))

    def total_elems(self) -> int:
        return self.slots * self.plane()

    @staticmethod
    def make(spec: StencilSpec, space: IterationSpace, slots: int) -> "GridLayout":
        return GridLayout(int(slots), spec.time_depth, tuple(int(e) for e in space.extents), tuple(spec.radii))


class Grid:
    """Time-buffered float32 state in the reference layout (host memory)."""

    def __init__(self, layout: GridLayout, data: Optional[np.ndarray] = None, last_level: int = 0):
        self.layout = layout
        self.data = data if data is not None else np.zeros(layout.total_elems(), dtype=np.float32)
        assert self.data.dtype == np.float32 and self.data.size == layout.total_elems()
        self.last_level = last_level

    def view(self) -> np.ndarray:
        return self.data.reshape((self.layout.slots,) + self.layout.padded)

    def level(self, level: int) -> np.ndarray:
        return self.view()[level % self.layout.slots]

    def interior(self, level: int) -> np.ndarray:
        v = self.level(level)
        return v[tuple(slice(h, h + d) for h, d in zip(self.layout.halo, self.layout.interior))]


def _host_f32(a, what: str):
    """Host buffers cross the C-ABI as float* + element count: anything but a
    C-contiguous float32 ndarray would be misread or overrun (checked
    explicitly, not with assert, so python -O keeps the check)."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags.c_contiguous:
        raise Error(f"{what}: host buffer must be a C-contiguous float32 ndarray "
                    f"(got {getattr(a, 'dtype', type(a).__name__)})", ST_ERR_INVALID)
    if what != "upload" and not a.flags.writeable:
        raise Error(f"{what}: host buffer is read-only", ST_ERR_INVALID)


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def init_grid(spec: StencilSpec, space: IterationSpace, seed: int, slots: int) -> Grid:
    """init_grid (executor.hpp:87-90): levels [0, delta_t) incl. halo from the
    frozen LCG, values in [0.001, 0.002); remaining slots zero."""
    lay = GridLayout.make(spec, space, slots)
    g = Grid(lay, last_level=spec.time_depth - 1)
    _check(_lib().st_init_reference(spec.handle, N.i64array(space.extents), _fptr(g.data), int(slots), int(seed) & (2**64 - 1)))
    return g


def init_unit(spec: StencilSpec, space: IterationSpace, seed: int, slots: int) -> Grid:
    lay = GridLayout.make(spec, space, slots)
    g = Grid(lay, last_level=spec.time_depth - 1)
    _check(_lib().st_init_unit(spec.handle, N.i64array(space.extents), _fptr(g.data), int(slots), int(seed) & (2**64 - 1)))
    return g


def init_gaussian(spec: StencilSpec, space: IterationSpace, slots: int, sigma: float,
                  centre: Sequence[int], z_begin: int = 0) -> Grid:
    lay = GridLayout.make(spec, space, slots)
    g = Grid(lay, last_level=spec.time_depth - 1)
    c = N.i64array(centre)
    _check(_lib().st_init_gaussian_slab(spec.handle, N.i64array(space.extents), _fptr(g.data), int(slots),
                                        float(sigma), c, int(z_begin)))
    return g


@dataclasses.dataclass
class ExecReport:
    points_updated: int
    flops: int
    wall_seconds: float
    device_seconds: float = 0.0
    time_tile_used: int = 1
    kernel_launches: int = 0
    tile: Tuple[int, int, int] = (0, 0, 0)
    mode_used: int = MODE_REFERENCE
    kernel_kind: int = 0


class Context:
    """One device + stream (st_context)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(_lib().st_context_create(int(device), C.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return _lib().st_context_stream(self._h) or 0

    @property
    def sm_count(self) -> int:
        return _lib().st_context_sm_count(self._h)

    def flush_l2(self):
        """Overwrite twice the L2 on the context's stream (between timed trials)."""
        _check(_lib().st_context_flush_l2(self._h))

    def close(self):
        if self._h and self._h.value:
            _lib().st_context_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class DeviceGrid:
    """A Grid resident on the device (st_grid): upload once, apply many."""

    def __init__(self, ctx: Context, spec: StencilSpec, extents: Sequence[int], slots: int):
        self.ctx, self.spec, self.extents, self.slots = ctx, spec, tuple(int(e) for e in extents), int(slots)
        h = C.c_void_p()
        _check(_lib().st_grid_create(ctx.handle, spec.handle, N.i64array(self.extents), self.slots, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def upload(self, data: np.ndarray, last_level: int, uniform_halo: bool = False):
        _host_f32(data, "upload")
        _check(_lib().st_grid_upload(self._h, _fptr(data), data.size, int(last_level), 1 if uniform_halo else 0))

    def upload_ptr(self, ptr: int, nelems: int, last_level: int, uniform_halo: bool = False):
        _check(_lib().st_grid_upload(self._h, C.cast(C.c_void_p(ptr), C.POINTER(C.c_float)), int(nelems),
                                     int(last_level), 1 if uniform_halo else 0))

    def set_field(self, m: np.ndarray):
        m = np.ascontiguousarray(m, dtype=np.float32)
        _check(_lib().st_grid_set_field(self._h, _fptr(m), m.size))

    def download(self, data: np.ndarray) -> int:
        _host_f32(data, "download")
        ll = C.c_int64()
        _check(_lib().st_grid_download(self._h, _fptr(data), data.size, C.byref(ll)))
        return ll.value

    def download_ptr(self, ptr: int, nelems: int) -> int:
        ll = C.c_int64()
        _check(_lib().st_grid_download(self._h, C.cast(C.c_void_p(ptr), C.POINTER(C.c_float)), int(nelems), C.byref(ll)))
        return ll.value

    def last_level(self) -> int:
        ll = C.c_int64()
        _check(_lib().st_grid_last_level(self._h, C.byref(ll)))
        return ll.value

    def device_bytes(self) -> int:
        return int(_lib().st_grid_device_bytes(self._h))

    def apply(self, t_begin: int, t_end: int, nest: LoopNest, mode: int = MODE_REFERENCE) -> ExecReport:
        p = _plan_struct(nest.schedule, nest.plan)
        r = N.st_report()
        _check(_lib().st_apply(self._h, int(t_begin), int(t_end), C.byref(p), int(mode), C.byref(r)))
        return ExecReport(r.points_updated, r.flops, r.wall_seconds, r.device_seconds, r.time_tile_used,
                          r.kernel_launches, tuple(r.tile), r.mode_used, r.kernel_kind)

    def execute_host(self, data: np.ndarray, t_begin: int, t_end: int, nest: LoopNest, mode: int = MODE_REFERENCE,
                     uniform_halo: bool = False) -> ExecReport:
        """execute on a host grid (st_execute_host): levels [t_begin, t_begin + delta_t)
        of ``data`` in, steps [t_begin, t_end), the interior of the newest delta_t
        levels back into their slots.  Page-locked ``data`` takes the copy-engine
        path; the call releases the GIL, so grids of different contexts driven from
        different threads overlap."""
        _host_f32(data, "execute_host")
        p = _plan_struct(nest.schedule, nest.plan)
        r = N.st_report()
        _check(_lib().st_execute_host(self._h, _fptr(data), data.size, int(t_begin), int(t_end), C.byref(p), int(mode),
                                      1 if uniform_halo else 0, C.byref(r)))
        return ExecReport(r.points_updated, r.flops, r.wall_seconds, r.device_seconds, r.time_tile_used,
                          r.kernel_launches, tuple(r.tile), r.mode_used, r.kernel_kind)

    def close(self):
        if self._h and self._h.value:
            _lib().st_grid_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def execute(nest: LoopNest, spec: StencilSpec, space: IterationSpace, grid: Grid,
            mode: int = MODE_REFERENCE, field: Optional[np.ndarray] = None,
            ctx: Optional[Context] = None) -> ExecReport:
    """execute (executor.hpp:92-98) on the B200: runs steps [0, D_t) of the
    nest's schedule over ``grid`` in place (upload, apply, download).
    Raises Error on an illegal plan or insufficient slots (executor.hpp:95-97)."""
    ctx = ctx or default_context()
    if grid.layout.slots < required_slots(nest, spec):
        raise Error(f"grid has {grid.layout.slots} slots, nest requires {required_slots(nest, spec)}", ST_ERR_SLOTS)
    dg = DeviceGrid(ctx, spec, space.extents, grid.layout.slots)
    try:
        dg.upload(grid.data, grid.last_level)
        if spec.model == MODEL_WAVE:
            if field is None:
                raise Error("wave model needs a coefficient field", ST_ERR_STATE)
            dg.set_field(field)
        t0 = grid.last_level - spec.time_depth + 1
        rep = dg.apply(t0, t0 + space.time_steps, nest, mode)
        grid.last_level = dg.download(grid.data)
    finally:
        dg.close()
    return rep


def verify_bitwise(a: Grid, b: Grid, compare_levels: int, spec: Optional[StencilSpec] = None) -> bool:
    """verify_bitwise (executor.hpp:107-110) over the interior of the last
    compare_levels levels; raises Error if a grid no longer retains them."""
    if a.layout.interior != b.layout.interior or a.layout.halo != b.layout.halo:
        raise Error("verify_bitwise: spatial shape mismatch")
    if a.last_level != b.last_level:
        return False
    eq = C.c_int()
    _check(_lib().st_verify_bitwise_layout(len(a.layout.interior), N.i64array(a.layout.interior),
                                           N.i64array(a.layout.halo), _fptr(a.data), a.layout.slots, _fptr(b.data),
                                           b.layout.slots, int(a.last_level), int(compare_levels), C.byref(eq)))
    return bool(eq.value)


# ------------------------------------------------------------ cache-sim ---
@dataclasses.dataclass
class CacheConfig:
    """cache_sim.hpp:13-17: fully associative LRU, write-allocate + write-back;
    capacity and line size in float32 elements."""
    capacity_elems: int = 1
    line_elems: int = 16


@dataclasses.dataclass
class TrafficReport:
    lines_loaded: int
    lines_written_back: int
    line_elems: int
    bytes: int
    flops: int
    measured_ai: float


def simulate(nest: LoopNest, spec: StencilSpec, space: IterationSpace, cache: CacheConfig,
             cap: int = 1_000_000_000) -> TrafficReport:
    """simulate (cache_sim.hpp:28-34): replay the nest's access stream against
    the LRU cache; raises Error past `cap` traced points (host-only)."""
    p = _plan_struct(nest.schedule, nest.plan)
    r = N.st_traffic()
    _check(_lib().st_simulate(spec.handle, N.i64array(space.extents), int(space.time_steps), C.byref(p),
                              int(cache.capacity_elems), int(cache.line_elems), int(cap), C.byref(r)))
    return TrafficReport(r.lines_loaded, r.lines_written_back, r.line_elems, r.bytes, r.flops, r.measured_ai)


def measured_ai_elems(report: TrafficReport) -> float:
    """cache_sim.hpp:45-47: flops per byte of a traffic report; error without traffic."""
    if report.bytes <= 0:
        raise Error("traffic report carries no traffic")
    return report.flops / report.bytes


# ------------------------------------------------------------- z-slabs ---
def dist_partition(global_nz: int, world: int, rank: int, ghost: int) -> Tuple[int, int, int, int]:
    """(z_begin, z_count, ghost_lo, ghost_hi) of `rank`'s slab along d_1."""
    out = [C.c_int64() for _ in range(4)]
    _check(_lib().st_dist_partition(int(global_nz), int(world), int(rank), int(ghost), *[C.byref(o) for o in out]))
    return tuple(int(o.value) for o in out)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib().st_nccl_unique_id(buf))
    return buf.raw


class Dist:
    """One rank's z-slab: a DeviceGrid holding slab + ghosts, exchanging
    ghost planes every time tile (NCCL id given) or in-process (loopback)."""

    def __init__(self, local: DeviceGrid, rank: int, world: int, ghost_lo: int, ghost_hi: int,
                 nccl_id: Optional[bytes] = None):
        h = C.c_void_p()
        _check(_lib().st_dist_create(local.handle, int(rank), int(world), nccl_id, int(ghost_lo), int(ghost_hi),
                                     C.byref(h)))
        self._h, self.local, self.rank, self.world = h, local, rank, world

    @staticmethod
    def link_loopback(members: Sequence["Dist"]):
        arr = (C.c_void_p * len(members))(*[m._h.value for m in members])
        _check(_lib().st_dist_link_loopback(arr, len(members)))
        for m in members:
            m._group = arr   # keep alive

    def apply(self, t_begin: int, t_end: int, nest: LoopNest, mode: int = MODE_REFERENCE) -> ExecReport:
        p = _plan_struct(nest.schedule, nest.plan)
        r = N.st_report()
        _check(_lib().st_dist_apply(self._h, int(t_begin), int(t_end), C.byref(p), int(mode), C.byref(r)))
        return ExecReport(r.points_updated, r.flops, r.wall_seconds, r.device_seconds, r.time_tile_used,
                          r.kernel_launches, tuple(r.tile), r.mode_used, r.kernel_kind)

    def close(self):
        if self._h and self._h.value:
            _lib().st_dist_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
