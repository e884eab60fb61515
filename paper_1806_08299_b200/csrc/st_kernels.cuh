// st_kernels.cuh -- sm_100a stencil kernels (templates; instantiated in the
// st_star*.cu / st_gen.cu translation units).
//
// One device routine processes one *item*: a column of cz planes along z of
// a (TY x TX) tile of the level being written, streamed plane by plane
// (2.5D): the z-neighbourhood of every output point lives in registers (a
// 2*RZ+2 deep window including a one-plane lookahead), the current plane with
// its x/y halo is staged in shared memory (double-buffered, one barrier per
// plane), y-neighbours inside a thread's VY-point strip come from registers.
//
// Two drivers:
//  * sweep (WF=false): one launch per level, blockIdx = item -- the
//    canonical / tile_space_minmax schedule (all points of step t before step
//    t+1), reads through the read-only path.
//  * wavefront (WF=true): a persistent kernel takes items in ticket order
//    (level-major) and streams level L+1 behind level L with a lag of `skew`
//    planes, synchronised by per-item progress counters (acquire/release at
//    gpu scope, reads via ld.global.cg).  At most T levels are in flight --
//    the tile_time schedule (transforms.hpp:53-59) realised as a skewed
//    wavefront whose working set stays in the 126 MB L2, so a level is read
//    from HBM once per T steps instead of once per step.  Level buffers are
//    ping-ponged (delta_t + 1 of them), so the intermediate levels overwrite
//    lines that are still L2-resident instead of streaming to HBM.
//
// Arithmetic: ST_MODE_REFERENCE evaluates acc = c1*r1; acc = acc + ck*rk in
// spec term order with __fmul_rn/__fadd_rn (never contracted), which is the
// reference FP contract (executor.hpp:92-95, CMakeLists.txt:12-13).
// ST_MODE_FAST pairs symmetric taps and uses FFMA.
#pragma once

#include <cuda_runtime.h>

#include <cuda/std/type_traits>

#ifndef ST_EXP
#define ST_EXP 0  // experiment switch (0 = product build)
#endif
#ifndef ST_NO_F32X2
#define ST_NO_F32X2 0  // 1 = scalar FP32 only (ablation)
#endif
#ifndef ST_UNROLL_MAX_R
#define ST_UNROLL_MAX_R 2  // unroll the phase loop by the window depth up to this radius
#endif
#ifndef ST_P2_MIN_R_EXACT
#define ST_P2_MIN_R_EXACT 1   // smallest radius whose bit-exact taps are paired (FFMA2 + FADD2)
#endif
#ifndef ST_P2_MIN_R_FAST
#define ST_P2_MIN_R_FAST 4    // ... and FAST taps (FFMA2)
#endif
#ifndef ST_WAVE_FAST_ORDERED
#define ST_WAVE_FAST_ORDERED 0   // 1: FAST wave taps as fma(c, u, acc) in the reference term order
#endif
#ifndef ST_WAVE_HYBRID_K0
#define ST_WAVE_HYBRID_K0 2   // radius-4 wave FAST: taps at distance >= this are fused in the reference order (0 = pairs + FMA)
#endif
#ifndef ST_P2_ODD_X
#define ST_P2_ODD_X 0   // 1: pair the odd-offset x taps too (register moves form the pairs)
#endif
#ifndef ST_ROLL_U
#define ST_ROLL_U 1        // phases per block of the rolled loop, r > ST_UNROLL_MAX_R (2: same speed, 2x code)
#endif
#ifndef ST_ROLL_U_R8
#define ST_ROLL_U_R8 ST_ROLL_U   // ... for radius 8 (1 row per thread: a short body, 16 window moves per update)
#endif
#ifndef ST_CHECKS
#define ST_CHECKS 0        // 1: device-side bounds checks (make EXP=13; compute-sanitizer is closed on the pool)
#endif

#include "st_internal.h"

namespace st {

template <bool WF>
__device__ __forceinline__ float ld_src(const float* p) {
  if constexpr (WF) return __ldcg(p);
  else return __ldg(p);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Release fence for the publication patterns (fence + st.relaxed.gpu):
// acq_rel is enough for a release pattern and is cumulative over the stores
// the publishing thread acquired at CTA scope.  ST_FENCE_SC=1 restores the
// sequentially consistent fence (__threadfence) for comparison.
#ifndef ST_FENCE_SC
#define ST_FENCE_SC 0
#endif
__device__ __forceinline__ void fence_release_gpu() {
#if ST_FENCE_SC
  __threadfence();
#else
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <bool FAST>
__device__ __forceinline__ float tap(float acc, float c, float v) {
  if constexpr (FAST) return __fmaf_rn(c, v, acc);
  else return __fadd_rn(acc, __fmul_rn(c, v));
}

// One unit of work: relative level, column (y-tile, x-tile), plane range
// [z0, z1), streaming direction (0 = increasing z) and, for the wavefront,
// its progress-counter index.
struct Work {
  int lrel, col, z0, z1, dir;
  int y0;   // first row of the tile (row-skewed y-bands shift it by -ysk per level; may be < 0)
  long long ctr;
};

// Wavefront ticket -> work (skewed chunk geometry, see Items).  Returns
// false past the last ticket; an item beyond the last level or with an
// empty (clipped) plane range comes back with z1 <= z0.
__device__ __forceinline__ bool wf_decode(const KParams& p, long long t, Work& w) {
  const Items& it = p.it;
  if (t >= it.ntickets) return false;
  const long long per_lv = (long long)it.cy * it.nxb;          // tickets per (chunk, y-chunk, level)
  const long long per_yc = per_lv * p.T;
  const long long per_zc = per_yc * it.nyc;
  const long long per_tile = per_zc * it.nch;
  const int tb = (int)(t / per_tile);
  long long r = t - tb * per_tile;
  const int c = (int)(r / per_zc);
  r -= (long long)c * per_zc;
  const int yc = (int)(r / per_yc);
  r -= (long long)yc * per_yc;
  const int lt = (int)(r / per_lv);
  r -= (long long)lt * per_lv;
  // x-fastest inside a (chunk, level) group: x-neighbour tiles on adjacent
  // tickets.  (y-fastest measured worse: config 5 FAST 1257 -> 1399 GB of DRAM
  // reads per run, 260 -> 289 ms.)
  const int jy = (int)(r / it.nxb);
  const int xb = (int)(r - (long long)jy * it.nxb);
  const int yb = yc * it.cy - (it.ysk == 0 && it.nyc > 1 ? lt : 0) + jy;
  w.lrel = tb * p.T + lt;
  w.y0 = yb * it.ty - it.ysk * lt;
  w.dir = 0;
  const int sh = p.skew * lt;
  w.z0 = max(0, c * it.cz - sh);
  w.z1 = min(p.g.nz, (c + 1) * it.cz - sh);
  if (p.zr_on && w.lrel < p.nsteps) {   // z-slab trapezoid: level range
    w.z0 = max(w.z0, p.zr_lo[w.lrel]);
    w.z1 = min(w.z1, p.zr_hi[w.lrel]);
  }
  const bool yin = yb >= 0 && yb < it.nyb && w.y0 + it.ty > 0 && w.y0 < p.g.ny;
  if (w.lrel >= p.nsteps || !yin) w.z1 = w.z0;   // past the last level / outside the grid: empty
  w.col = yin ? yb * it.nxb + xb : 0;
  w.ctr = ((long long)w.lrel * it.nch + c) * it.ncol + w.col;
  return true;
}

// Sweep (canonical / space-tiled schedules, one launch per level): CTA b
// owns the balanced column-plane range [W*b/G, W*(b+1)/G) of W = ncol * nz
// (no tail wave).  The cursor can also sweep downward (dir = 1); the kernels
// currently always sweep upward.
struct ZigZagCursor {
  long long lo, hi, cur;
  int lrel, dir;
  __device__ void init(const KParams& p, int level) {
    const long long W = (long long)p.it.ncol * (p.zhi - p.zlo);
    lo = W * blockIdx.x / gridDim.x;
    hi = W * (blockIdx.x + 1) / gridDim.x;
    lrel = level;
    dir = 0;   // always upward: a downward variant doubles the (I-cache bound) body
    cur = lo;
  }
  __device__ bool next(const KParams& p, Work& w) {
    const int nz = p.zhi - p.zlo;   // column-planes are counted within [zlo, zhi)
    if (dir == 0 && cur < hi) {
      w.col = (int)(cur / nz);
      w.z0 = (int)(cur - (long long)w.col * nz);
      w.z1 = (int)min((long long)nz, w.z0 + (hi - cur));
      cur += w.z1 - w.z0;
    } else if (dir == 1 && cur > lo) {
      w.col = (int)((cur - 1) / nz);
      const long long cb = (long long)w.col * nz;
      w.z1 = (int)(cur - cb);
      w.z0 = (int)(max(cb, lo) - cb);
      cur = cb + w.z0;
    } else {
      return false;
    }
    w.z0 += p.zlo;
    w.z1 += p.zlo;
    w.lrel = lrel;
    w.dir = dir;
    w.ctr = 0;
    w.y0 = (w.col / p.it.nxb) * p.it.ty;
    return true;
  }
};

// Generic kernel sweep: CTA b streams the column-planes [b*W/G, (b+1)*W/G)
// of one level (one launch per level).
struct SweepCursor {
  long long pos, end;
  __device__ void init(const KParams& p) {
    const long long W = (long long)p.it.ncol * (p.zhi - p.zlo);
    pos = W * blockIdx.x / gridDim.x;
    end = W * (blockIdx.x + 1) / gridDim.x;
  }
  __device__ bool next(const KParams& p, int lrel, Work& w) {
    if (pos >= end) return false;
    const int nz = p.zhi - p.zlo;
    w.col = (int)(pos / nz);
    w.z0 = (int)(pos - (long long)w.col * nz) + p.zlo;
    w.z1 = (int)min((long long)p.zhi, w.z0 + (end - pos));
    w.lrel = lrel;
    w.dir = 0;
    w.ctr = 0;
    w.y0 = (w.col / p.it.nxb) * p.it.ty;
    pos += w.z1 - w.z0;
    return true;
  }
};

// Per-lane cache: the counter last read (counters only grow) and the plane
// range it covers, so the owner lookup (a 64-bit division) runs only when a
// neighbour column's planes cross into another item / CTA range.
struct DepCache {
  long long idx;     // counter index (-1 = none)
  long long lo, hi;  // PIPE: [lo, hi) column-plane range of the cached owner; WF: chunk [lo, hi)
  unsigned have;
  int col, lrel;
};

// Watchdog: a dependency that never resolves is a bug; record what was
// awaited in zero-copy host memory and trap instead of hanging the GPU.
static __device__ __noinline__ void watchdog_trip(const KParams& p, int kind, long long a, long long b, long long c) {
  if (p.dbg) {
    volatile long long* d = p.dbg;
    d[1] = kind;
    d[2] = blockIdx.x;
    d[3] = threadIdx.x;
    d[4] = a;
    d[5] = b;
    d[6] = c;
    __threadfence_system();
    d[0] = 1;
    __threadfence_system();
  }
  __trap();
}

// The neighbour column a lane of the producer warp watches for one item
// (lanes 0..8: the 3 x 3 block of tiles around the item's column), fixed per
// item so the per-plane wait carries no index arithmetic.
struct DepLane {
  bool mine;
  int c2;   // watched column of level lrel - 1
};

__device__ __forceinline__ DepLane dep_lane(const KParams& p, int lrel, int col, bool box) {
  DepLane d{false, 0};
  if (lrel == 0) return d;
  const Items& it = p.it;
  const int lane = threadIdx.x & 31;
  if (lane < 9) {
    const int yb = col / it.nxb, xb = col - yb * it.nxb;
    const int dy = lane / 3 - 1, dx = lane % 3 - 1;
    int yy = yb + dy;
    const int xx = xb + dx;
    if (it.ysk > 0) {
      // row-skewed y-bands: level Lp's tile grid sits at rows yy*ty - ysk*(Lp % T).  The rows
      // this tile reads, [y0 - ry, y0 + ty + ry) clipped to the interior, span at most 3 of
      // its tiles (2 inside a time tile: yb - 1 and yb); the x-neighbour columns of the same
      // tile rows are needed too (the shifted grids make the "diagonal" tiles real
      // dependences), so every lane of the 3 x 3 block watches.
      const int y0 = yb * it.ty - it.ysk * (lrel % p.T);
      const int sp = it.ysk * ((lrel - 1) % p.T);
      const int rlo = max(y0 - p.g.ry, 0), rhi = min(y0 + it.ty + p.g.ry, p.g.ny) - 1;
      yy = (rlo + sp) / it.ty + (dy + 1);
      d.mine = rhi >= rlo && yy <= (rhi + sp) / it.ty && xx >= 0 && xx < it.nxb;
    } else {
      d.mine = (box || dy == 0 || dx == 0) && yy >= 0 && yy < it.nyb && xx >= 0 && xx < it.nxb;
    }
    d.c2 = yy * it.nxb + xx;
  }
  return d;
}

// Warp 0 (all 32 lanes): before loading plane pz of level lrel-1, wait
// until it is complete in every neighbour column of the item (5-point star or
// 9-point box neighbourhood of tiles; dep_lane).  Lane i < 9 watches one
// neighbour's counter; counts are in units of p.pipe.unit per plane.
__device__ __forceinline__ void wait_plane(const KParams& p, int lrel, const DepLane& dl, int pz, DepCache& dc) {
  if (lrel == 0) return;
  const Items& it = p.it;
  const int Lp = lrel - 1;
  unsigned need = 0;
  bool mine = dl.mine;
  // z-slab trapezoid: a plane level Lp does not compute is exchanged
  // ghost data, already in place
  if (mine && p.zr_on && (pz < p.zr_lo[Lp] || pz >= p.zr_hi[Lp])) mine = false;
  if (mine) {
    const int c2 = dl.c2;
    if (dc.idx < 0 || dc.col != c2 || dc.lrel != Lp || pz < dc.lo || pz >= dc.hi) {
      const int sh = p.skew * (Lp % p.T);
      const int cc = (pz + sh) / it.cz;
      dc.lo = max(p.zr_on ? p.zr_lo[Lp] : 0, cc * it.cz - sh);
      dc.hi = min(p.zr_on ? p.zr_hi[Lp] : p.g.nz, (cc + 1) * it.cz - sh);
      dc.idx = ((long long)Lp * it.nch + cc) * it.ncol + c2;
      dc.col = c2;
      dc.lrel = Lp;
      dc.have = 0;
    }
    need = (unsigned)(pz - dc.lo + 1) * (unsigned)p.pipe.unit;
  }
  if (__all_sync(0xffffffffu, !mine || dc.have >= need)) return;
  int ns = 32;
  for (long long spin = 0;; ++spin) {
    if (mine && dc.have < need) dc.have = ld_acquire(p.prog + (dc.idx << p.ctr_shift));
    if (__all_sync(0xffffffffu, !mine || dc.have >= need)) break;
    __nanosleep(ns);
    ns = ns < p.sleep_dep ? ns * 2 : p.sleep_dep;
    if (spin > (1LL << 24)) {
      if (mine && dc.have < need) watchdog_trip(p, 1, dc.idx, need, dc.have);
      __syncwarp();
    }
  }
  fence_proxy_async_global();
}


// Per-slot frozen halos (reference init_grid halos differ per slot): the
// item writing level L also writes the halo cells of the destination buffer
// adjacent to its region at plane z from the bank copy of slot L mod S.
template <int RZ, int RY, int RX>
__device__ void halo_refresh(const KParams& p, float* __restrict__ dst,
                             long long L, int z, int y0, int TY, int x0,
                             int TX, int tid, int NT) {
  const DevGeom& g = p.g;
  const bool by0 = RY > 0 && y0 == 0, by1 = RY > 0 && y0 + TY >= g.ny;
  const bool bx0 = x0 == 0, bx1 = x0 + TX >= g.nx;
  const bool zf0 = RZ > 0 && z == 0, zf1 = RZ > 0 && z == g.nz - 1;
  if (!(by0 || by1 || bx0 || bx1 || zf0 || zf1)) return;
  const float* __restrict__ bk = p.bank + (L % p.bank_slots) * g.buf_elems;
  const int eylo = by0 ? -RY : y0, eyhi = by1 ? g.ny + RY : min(g.ny, y0 + TY);
  const int exlo = bx0 ? -RX : x0, exhi = bx1 ? g.nx + RX : min(g.nx, x0 + TX);
  const int W = exhi - exlo, H = eyhi - eylo;
  auto copy_plane = [&](int zz, bool all) {
    for (int i = tid; i < W * H; i += NT) {
      const int yy = eylo + i / W, xx = exlo + i % W;
      const bool interior = yy >= 0 && yy < g.ny && xx >= 0 && xx < g.nx;
      if (all || !interior) {
        const long long idx = dev_index(g, zz, yy, xx);
        dst[idx] = bk[idx];
      }
    }
  };
  if (by0 || by1 || bx0 || bx1) copy_plane(z, false);
  if (zf0)
    for (int zz = -RZ; zz < 0; ++zz) copy_plane(zz, true);
  if (zf1)
    for (int zz = g.nz; zz < g.nz + RZ; ++zz) copy_plane(zz, true);
}

// ---------------------------------------------------------------------------
// TMA / mbarrier primitives (sm_90+; SASS: UTMALDG, SYNCS.*)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking phase test (never suspends the thread).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// ROLE only separates the call sites in profiles (0 consumer full, 1 producer
// empty, 2 ticket queue, 3 wave operand ring, 5/6 fused-level ring).  The
// fused kernel has no cross-CTA waits, so its rings trap after seconds.
// The slow path suspends in try_wait (up to ST_MBAR_SUSPEND_NS per call; the
// thread resumes as soon as the phase completes) instead of re-issuing it:
// a spinning warp steals issue slots from the consumers beside it.
#ifndef ST_MBAR_SUSPEND_NS
#define ST_MBAR_SUSPEND_NS 1000
#endif
__device__ __forceinline__ bool mbar_try_suspend(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ST_MBAR_SUSPEND_NS)
      : "memory");
  return ok != 0;
}
// Variants on precomputed 32-bit shared addresses (the consumer's plane loop:
// no generic->shared conversion per phase).
__device__ __forceinline__ void mbar_arrive_a(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// Lane-0 arrive as a predicated instruction: no divergent branch around it.
__device__ __forceinline__ void mbar_arrive_if(uint32_t a, unsigned p) {
  asm volatile(
      "{\n\t.reg .pred q;\n\t"
      "setp.ne.u32 q, %1, 0;\n\t"
      "@q mbarrier.arrive.shared::cta.b64 _, [%0];\n}" ::"r"(a), "r"(p)
      : "memory");
}
__device__ __forceinline__ void st_release_cta_if(uint32_t a, unsigned v, unsigned p) {
  asm volatile(
      "{\n\t.reg .pred q;\n\t"
      "setp.ne.u32 q, %2, 0;\n\t"
      "@q st.release.cta.shared.u32 [%0], %1;\n}" ::"r"(a), "r"(v), "r"(p)
      : "memory");
}
__device__ __forceinline__ bool mbar_try_a(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_a(uint32_t a, uint32_t parity) {
  if (!mbar_try_a(a, parity)) {
    for (int spin = 0;; ++spin) {
      uint32_t ok;
      asm volatile(
          "{\n\t.reg .pred P1;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
          "selp.u32 %0, 1, 0, P1;\n}"
          : "=r"(ok)
          : "r"(a), "r"(parity), "r"(ST_MBAR_SUSPEND_NS)
          : "memory");
      if (ok) break;
      if (spin > (1 << 26)) __trap();   // ring protocol bug: never hang the GPU
    }
  }
}

// The slow path is inline (a call would make every live register of the
// unrolled plane loop caller-saved across it: ptxas then spills them).
template <int ROLE = 0>
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  constexpr int kLimit = ROLE >= 5 ? (1 << 21) : (1 << 26);   // tries of <= 1 us each
  if (!mbar_try(bar, parity)) {
    for (int spin = 0; !mbar_try_suspend(bar, parity); ++spin)
      if (spin > kLimit) __trap();   // ring protocol bug: never hang the GPU
  }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                            int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// Star kernel: stencils whose terms are the canonical star (centre, then per
// reference axis d_1..d_n: -1, +1, -2, +2, ..., -R, +R), all reading level
// L-1 (heat) or the wave model.
//
// Warp-specialised: warp 0 is the producer -- it resolves wavefront
// dependencies and issues one TMA box load per plane (the tile plus its x/y
// halo, and for the wave the u^{n-1} / m tiles) into an NS-deep shared ring
// guarded by full/empty mbarriers; warps 1..NC consume.  A consumer thread
// owns VX = 4 consecutive x of VY rows: it keeps the z-window (2RZ+1 planes)
// of its points in registers (float4), reads x/y neighbours of the centre
// plane from the ring with LDS.128, accumulates term-major over its strip
// (independent FP chains) and writes the output with STG.128.
// ---------------------------------------------------------------------------
// Paired FP32 (sm_100 FADD2 / FMUL2 / FFMA2: two lanes of a 64-bit register
// pair per instruction, each lane IEEE round-to-nearest exactly like the
// scalar op).  ptxas contracts an f32x2 multiply feeding an f32x2 add into
// FFMA2 even with --fmad=false (and folds fma(c, u, -0.0) to a multiply
// first), which would change the reference rounding.  So the bit-exact
// product is fma.rn.f32x2(c, u, nz) with nz = -0.0 read from the kernel
// parameters (KParams::nzero, opaque to the compiler): round(c*u + -0) is
// round(c*u) for every input, sign of zero included, and ptxas does not
// contract an FFMA2 into the FADD2 that follows -- 2 instructions per pair
// of taps (FFMA2 + FADD2) instead of 3 (FMUL2 + 2 scalar FADD).  FAST taps
// are whole FFMA2s.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 ffma2(float c, float a, float b, float acc0, float acc1) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a, b)), "l"(pk2(c, c)), "l"(pk2(acc0, acc1)));
  return upk2(d);
}
__device__ __forceinline__ float2 ffma2v(float a0, float a1, float b0, float b1, float c0, float c1) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a0, a1)), "l"(pk2(b0, b1)), "l"(pk2(c0, c1)));
  return upk2(d);
}
// bit-exact products (see above): nz must be a runtime -0.0
__device__ __forceinline__ float2 fmul2(float c, float a, float b, float nz) { return ffma2(c, a, b, nz, nz); }
__device__ __forceinline__ float2 fmul2v(float a0, float a1, float b0, float b1, float nz) {
  return ffma2v(a0, a1, b0, b1, nz, nz);
}
__device__ __forceinline__ float2 fsub2(float a0, float a1, float b0, float b1) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a0, a1)), "l"(pk2(b0, b1)));
  return upk2(d);
}
__device__ __forceinline__ float2 fadd2(float a0, float a1, float b0, float b1) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a0, a1)), "l"(pk2(b0, b1)));
  return upk2(d);
}

template <bool FAST, bool P2>
__device__ __forceinline__ float4 tap4(float4 a, float c, float4 v, float nz = 0.f) {
  if constexpr (!P2) {
    return make_float4(tap<FAST>(a.x, c, v.x), tap<FAST>(a.y, c, v.y), tap<FAST>(a.z, c, v.z),
                       tap<FAST>(a.w, c, v.w));
  } else if constexpr (FAST) {
    const float2 lo = ffma2(c, v.x, v.y, a.x, a.y), hi = ffma2(c, v.z, v.w, a.z, a.w);
    return make_float4(lo.x, lo.y, hi.x, hi.y);
  } else {
    const float2 lo = fmul2(c, v.x, v.y, nz), hi = fmul2(c, v.z, v.w, nz);
    const float2 s0 = fadd2(a.x, a.y, lo.x, lo.y), s1 = fadd2(a.z, a.w, hi.x, hi.y);
    return make_float4(s0.x, s0.y, s1.x, s1.y);
  }
}
template <bool P2>
__device__ __forceinline__ float4 mul4(float c, float4 v, float nz = 0.f) {
  if constexpr (!P2) {
    return make_float4(__fmul_rn(c, v.x), __fmul_rn(c, v.y), __fmul_rn(c, v.z), __fmul_rn(c, v.w));
  } else {
    const float2 lo = fmul2(c, v.x, v.y, nz), hi = fmul2(c, v.z, v.w, nz);
    return make_float4(lo.x, lo.y, hi.x, hi.y);
  }
}
template <bool P2>
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  if constexpr (!P2) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
  } else {
    const float2 lo = fadd2(a.x, a.y, b.x, b.y), hi = fadd2(a.z, a.w, b.z, b.w);
    return make_float4(lo.x, lo.y, hi.x, hi.y);
  }
}
__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float f4get(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// Window slot of the plane `x` phases after the current one: with the
// fully unrolled phase loop the window rotates (slot (jj + x) mod NQ);
// otherwise the loop is unrolled ST_ROLL_U phases deep over a window of
// NQ + ST_ROLL_U - 1 slots (slot jj + x) that shifts by ST_ROLL_U per block.
#define WI(jj, x) (UNROLLW ? ((jj) + (x)) % NQ : (jj) + (x))

// Register budget: all of the register file split over MINB resident CTAs
// (allocation granularity 8 per thread).
ST_HD constexpr int star_threads(int R, int DIMS, int MODEL, int V, bool WF) {
  return 32 * (1 + star_shape(R, DIMS, MODEL, V).NC + (WF ? 1 : 0));
}
ST_HD constexpr int star_maxreg(int R, int DIMS, int MODEL, int V, bool WF) {
  const int r = 65536 / (star_shape(R, DIMS, MODEL, V).MINB * star_threads(R, DIMS, MODEL, V, WF)) / 8 * 8;
  return r > 255 ? 255 : r;
}

template <int R, int DIMS, int MODEL, bool FAST, bool WF, int V = 0>
__global__ void __launch_bounds__(star_threads(R, DIMS, MODEL, V, WF), 1)
__maxnreg__(star_maxreg(R, DIMS, MODEL, V, WF))
star_kernel(const __grid_constant__ KParams p, int level) {
  constexpr StarShape S = star_shape(R, DIMS, MODEL, V);
  constexpr int RZ = DIMS >= 2 ? R : 0;
  constexpr int RY = DIMS == 3 ? R : 0;
  constexpr int RX = R;
  constexpr int NQ = 2 * RZ + 1;
  constexpr bool UNROLLW = RZ <= ST_UNROLL_MAX_R || V == 6;   // see the phase loop
  // r >= 4 phases take the leaner bookkeeping (precomputed shared addresses,
  // one STG per row when every x tile is full):
  // +2.6% on configs 3 / 5; the fully unrolled r <= 2 bodies measured slower
  // with it (register allocation at the per-SMSP cap), so they keep the plain one
  constexpr bool LEAN = RZ >= 4;
  // paired FP32: bit-exact taps at every radius since the FFMA2(-0) + FADD2
  // form (config 2 bit-exact: wavefront 546 -> 584, sweep 448 -> 508;
  // configs 3-5 +4% over FMUL2 + scalar FADD); FAST taps for r >= 4 only
  // (for r <= 2 the pair constraints cost more register moves than FFMA2
  // saves: measured -4% on config 2)
  constexpr bool P2 = !ST_NO_F32X2 && R >= (FAST ? ST_P2_MIN_R_FAST : ST_P2_MIN_R_EXACT);
  // FAST wave: every tap fused in the reference order (no symmetric pairing),
  // which stays closer to the reference over a non-dissipative run
  constexpr bool OFMA = FAST && MODEL == kWave && ST_WAVE_FAST_ORDERED;
  // FAST for the radius-4 leapfrog (configs 3 / 5): pairing symmetric taps
  // drifts 1.29e-5 from the reference over config 3's 200 non-dissipative
  // steps -- past the 1e-5 contract.  The ordered hybrid keeps the reference's
  // summation order and every rounded sum, and fuses only the products of the
  // taps at distance >= HK0 (|c| <= 0.2) into their sums: those products'
  // roundings are a small fraction of the sums' own, and the full run stays
  // 4.5e-6 from the reference (profiles/tools/hybrid_drift.cpp; distance >= 1
  // fused: 1.9e-5).  35 FP32 operations per update instead of 53.
  constexpr int HK0 = (FAST && MODEL == kWave && R == 4 && !ST_WAVE_FAST_ORDERED) ? ST_WAVE_HYBRID_K0 : 0;
  constexpr bool HYB = HK0 > 0;
  constexpr int VY = S.VY, NC = S.NC, TX = S.TX, TY = S.TY, XH = S.XH, SW = S.SW;
  constexpr int NS = S.NS, NSA = S.NSA, STAGE = S.STAGE, AUXF = S.AUX;
  constexpr int NT = NC * 32;
  constexpr int QD = 2;                     // work queue depth (wavefront)
  constexpr unsigned MAIN_BYTES = SW * S.SH * 4;
  constexpr unsigned AUX_BYTES = MODEL == kWave ? 2 * TX * TY * 4 : 0;
  constexpr unsigned AUX_BYTES_CODED = MODEL == kWave ? TX * TY * 4 + TX * TY : 0;
  constexpr int CZ0 = 1;                    // coef offset of the z taps
  constexpr int CY0 = 1 + 2 * RZ;           // y taps
  constexpr int CX0 = 1 + 2 * RZ + 2 * RY;  // x taps
  constexpr int XL = XH / 4;                // float4 loads per side for x taps
  constexpr int QW = NC + (WF ? 1 : 0);     // warps reading the work queue

  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ long long s_q[QD];
  __shared__ unsigned s_wdone[NC];          // per consumer warp: planes stored (wavefront)
  __shared__ float s_pal[MODEL == kWave ? 256 : 1];   // palette of the coded m field

  const DevGeom& g = p.g;
  const Items& it = p.it;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + NS;
  uint64_t* emptya = empty + NS;
  uint64_t* qfull = emptya + NSA;
  uint64_t* qempty = qfull + QD;
  float* ring = reinterpret_cast<float*>(smem_raw + 1024);
  float* aux = ring + NS * STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NC);
    }
    for (int s = 0; s < NSA; ++s) mbar_init(emptya + s, NC);
    for (int s = 0; s < QD; ++s) {
      mbar_init(qfull + s, 1);
      mbar_init(qempty + s, QW);
    }
    for (int w = 0; w < NC; ++w) s_wdone[w] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (MODEL == kWave) {
    if (p.mcode_on)
      for (int i = threadIdx.x; i < p.npal; i += blockDim.x) s_pal[i] = p.mpal[i];
  }
  __syncthreads();

  unsigned mseq = 0, aseq = 0;  // CTA-lifetime ring sequence numbers (both roles)

  if (warp == 0) {
    // =================== producer ==========================================
    int slot = 0, aslot = 0;
    unsigned use = 0, ause = 0;   // completed passes over the ring
    DepCache dc{-1, 0, 0, 0, -1, -1};
    auto produce = [&](const Work& w) {
      const int yb = w.col / it.nxb, xb = w.col - yb * it.nxb;
      const int y0 = w.y0, x0 = xb * TX;
      const int nph = w.z1 - w.z0, NP = nph + 2 * RZ;
      const int zfirst = w.dir ? w.z1 - 1 : w.z0;   // first output plane
      const int zs = w.dir ? -1 : 1;
      const long long L = p.level0 + w.lrel;
      const int bsrc = (int)((L - 1) % p.nbuf);
      const int bu2 = MODEL == kWave ? (int)((L - 2) % p.nbuf) : 0;
      DepLane dl{false, 0};
      if constexpr (WF) dl = dep_lane(p, w.lrel, w.col, false);
      for (int j = 0; j < NP; ++j) {
        if (use > 0) mbar_wait<1>(empty + slot, (use - 1) & 1);
        const int pz = zfirst + zs * (j - RZ);   // plane (interior coords)
        if constexpr (WF) {
          // planes below 0 are the z halo: with per-slot halos (bank) the
          // level writes it when it stores plane 0, so wait for that plane
          if (pz < g.nz && (pz >= 0 || p.bank)) wait_plane(p, w.lrel, dl, max(pz, 0), dc);
        }
        const bool with_aux = MODEL == kWave && j >= 2 * RZ;
        if (with_aux && ause > 0) mbar_wait<3>(emptya + aslot, (ause - 1) & 1);
        if (lane == 0) {
          mbar_expect_tx(full + slot, MAIN_BYTES + (with_aux ? (p.mcode_on ? AUX_BYTES_CODED : AUX_BYTES) : 0u));
          tma_load_3d(ring + slot * STAGE, &p.tm.main[bsrc], full + slot, g.xo + x0 - XH, y0, pz + g.rz);
          if (with_aux) {
            const int zc = pz - zs * RZ;          // centre plane of this phase
            float* a = aux + aslot * AUXF;
            tma_load_3d(a, &p.tm.aux[bu2], full + slot, g.xo + x0, y0 + g.ry, zc + g.rz);
            // m as 1-byte palette codes (TX x TY bytes) or as floats
            tma_load_3d(a + TX * TY, p.mcode_on ? &p.tm.mcodes : &p.tm.mfield, full + slot, g.xo + x0, y0 + g.ry,
                        zc + g.rz);
          }
        }
        __syncwarp();
        if (++slot == NS) { slot = 0; ++use; }
        if (with_aux && ++aslot == NSA) { aslot = 0; ++ause; }
      }
    };
    if constexpr (WF) {
      for (unsigned i = 0;; ++i) {
        Work w;
        bool have;
        long long t;
        do {
          unsigned tt = 0;
          if (lane == 0) tt = atomicAdd(p.ticket, 1u);
          t = (long long)__shfl_sync(0xffffffffu, tt, 0);
          have = wf_decode(p, t, w);
        } while (have && w.z1 <= w.z0);
        const int e = (int)(i % QD);
        if (i >= QD) mbar_wait<2>(qempty + e, ((i / QD) - 1) & 1);
        if (lane == 0) {
          s_q[e] = have ? t : -1;
          mbar_arrive(qfull + e);
        }
        __syncwarp();
        if (!have) break;
        produce(w);
      }
    } else {
      ZigZagCursor cur;
      cur.init(p, level);
      Work w;
      while (cur.next(p, w)) produce(w);
    }
  } else if (WF && warp == NC + 1) {
    // =================== publisher (wavefront) =============================
    // Turns the consumer warps' CTA-scope plane counts (min over warps) into
    // GPU-scope progress counters, so only this warp ever waits on a
    // device-wide fence.
    unsigned base = 0;
    for (unsigned i = 0;; ++i) {
      const int e = (int)(i % QD);
      mbar_wait<4>(qfull + e, (i / QD) & 1);
      const long long t = s_q[e];
      __syncwarp();
      if (lane == 0) mbar_arrive(qempty + e);
      if (t < 0) break;
      Work w;
      wf_decode(p, t, w);
      const unsigned nph = (unsigned)(w.z1 - w.z0);
      unsigned done = 0;
      int ns = 32;
      for (long long spin = 0; done < nph; ++spin) {
        // planes stored by EVERY consumer warp (warps are not in lockstep)
        unsigned v = 0xffffffffu;
        if (lane < NC) {
          asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&s_wdone[lane])) : "memory");
        }
        v = __reduce_min_sync(0xffffffffu, v);
        const unsigned k = min(nph, v - base);
        if (k > done) {
          done = k;
          // release pattern: fence + strong store.  The fence is cumulative,
          // so it also orders the consumer warps' stores this warp acquired at
          // CTA scope.  (fence + st.relaxed measured 5% faster than a bare
          // st.release.gpu, which in turn beat ld.relaxed polling + fence.)
          if (lane == 0) {
            fence_release_gpu();
            st_relaxed(p.prog + (w.ctr << p.ctr_shift), done);
          }
          __syncwarp();
          ns = 32;
        } else {
          __nanosleep(ns);
          ns = ns < p.sleep_pub ? ns * 2 : p.sleep_pub;
          if (spin > (1LL << 26)) watchdog_trip(p, 2, w.ctr, nph, done);
        }
      }
      base += nph;
    }
  } else {
    // =================== consumers =========================================
    const int ct = threadIdx.x - 32;
    const int cw = warp - 1;
    const float nz = p.nzero;   // -0.0, opaque to ptxas (bit-exact paired products)
    const int cx4 = lane * 4;
    const int so = (RY + cw * VY) * SW + XH + cx4;   // own point, stage-relative
    const int ao = cw * VY * TX + cx4;                // own point, aux-relative
    const long long pitch = g.pitch, pstride = g.pstride;
    unsigned wdone = 0;   // planes this warp has stored (wavefront publication)
    const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty), emptya_a = smem_u32(emptya);
    const uint32_t wdone_a = smem_u32(&s_wdone[cw]);
    const unsigned is0 = lane == 0;
    // BANK (per-slot halo banks) and MC (palettized m) are hoisted out of the
    // plane loop: each unrolled phase then carries no code for them
    auto consume = [&](auto down_tag, auto bank_tag, auto mc_tag, auto xf_tag, const Work& w) {
      constexpr bool DOWN = decltype(down_tag)::value;
      constexpr bool BANK = decltype(bank_tag)::value;
      constexpr bool MC = MODEL == kWave && decltype(mc_tag)::value;
      constexpr bool XF = decltype(xf_tag)::value;   // every x tile full: one STG.128 per row
      const int yb = w.col / it.nxb, xb = w.col - yb * it.nxb;
      const int y0 = w.y0, x0 = xb * TX;
      const int nph = w.z1 - w.z0, NP = nph + 2 * RZ;
      const int zfirst = DOWN ? w.z1 - 1 : w.z0;
      const long long L = p.level0 + w.lrel;
      const int gx = x0 + cx4;
      const bool xfull = gx + 4 <= g.nx, xany = gx < g.nx;
      float* __restrict__ dst = p.buf[(int)(L % p.nbuf)];
      float* op = dst + dev_index(g, zfirst, y0 + cw * VY, gx);
      const long long zstep = DOWN ? -pstride : pstride;
      bool yok[VY];
#pragma unroll
      for (int v = 0; v < VY; ++v) yok[v] = (unsigned)(y0 + cw * VY + v) < (unsigned)g.ny;   // y0 < 0: skewed bands
      // every shared-memory read of a stage stays inside it (rows 0 .. SH-1,
      // columns 0 .. SW-1 of the TMA box)
      static_assert((RY + NC * VY + RY) * SW <= STAGE, "stage reads stay inside the stage");
#if ST_CHECKS
      {   // the item and every store it makes lie inside the level buffer
        const bool zok = 0 <= w.z0 && w.z0 <= w.z1 && w.z1 <= g.nz && w.col >= 0 && w.col < it.ncol;
        const long long i0 = dev_index(g, zfirst, y0 + cw * VY, gx);
        const long long i1 = dev_index(g, DOWN ? w.z0 : w.z1 - 1, y0 + cw * VY + VY - 1, gx + 3);
        const bool store = xany && yok[0] && nph > 0;
        if (!zok || (store && (min(i0, i1) < 0 || max(i0, i1) >= g.buf_elems))) watchdog_trip(p, 10, i0, i1, w.col);
      }
#endif

      const int ms = (int)(mseq % NS);
      const unsigned mp = (mseq / NS) & 1;
      constexpr int ROLLU = RZ >= 8 ? ST_ROLL_U_R8 : ST_ROLL_U;
      float4 q[UNROLLW ? NQ : NQ + ROLLU - 1][VY];
      // prologue: planes 0 .. 2RZ-1 of the item into the register window
#pragma unroll
      for (int j = 0; j < 2 * RZ; ++j) {
        int sl = ms + j;
        unsigned par = mp;
        while (sl >= NS) { sl -= NS; par ^= 1; }   // 2RZ may exceed NS (r = 8)
        mbar_wait(full + sl, par);
        const float* st = ring + sl * STAGE + so;
#pragma unroll
        for (int v = 0; v < VY; ++v) q[j][v] = lds4(st + v * SW);
        if (j < RZ || j >= NP - RZ) {     // never a centre plane: last use
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + sl);
        }
      }
      int sn = ms + 2 * RZ, sc = ms + RZ;
      unsigned pn = mp;
      while (sn >= NS) { sn -= NS; pn ^= 1; }
      while (sc >= NS) sc -= NS;
      int sa = MODEL == kWave ? (int)(aseq % NSA) : 0;

      // r <= 2: unroll the phase loop by the window depth so the window
      // rotates by register renaming; r >= 4: blocks of ST_ROLL_U phases
      // that shift the window once per block (the NQ-times unrolled body
      // would overflow the instruction cache -- ncu showed 60%
      // "no_instructions" stalls).  The window moves are 12% of the so16
      // kernel's instructions, but halving them (ST_ROLL_U = 2) measured
      // no faster: that kernel is bound by the FP pipe and smem.
      constexpr int UNR = UNROLLW ? NQ : ROLLU;
      for (int kb = 0; kb < nph; kb += UNR) {
#pragma unroll
        for (int jj = 0; jj < UNR; ++jj) {
          const int k = kb + jj;
          if (k >= nph) break;
          // newest plane (index k + 2RZ) into the window
#if ST_EXP != 1
          if constexpr (LEAN) mbar_wait_a(full_a + 8 * sn, pn);
          else mbar_wait(full + sn, pn);
#endif
          {
            const float* st = ring + sn * STAGE + so;
#pragma unroll
            for (int v = 0; v < VY; ++v) q[WI(jj, 2 * RZ)][v] = lds4(st + v * SW);
          }
          if constexpr (LEAN) {   // beyond-chunk z halo: last use
            if (k + 2 * RZ >= NP - RZ) {
              __syncwarp();
              mbar_arrive_if(empty_a + 8 * sn, is0);
            }
          } else if (RZ > 0 && k + 2 * RZ >= NP - RZ) {
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + sn);
          }
          if (++sn == NS) { sn = 0; pn ^= 1; }
          const float* cs = ring + sc * STAGE + so;

          float4 acc[VY];
#pragma unroll
          for (int v = 0; v < VY; ++v) {
            const float4 cc = q[WI(jj, RZ)][v];
            acc[v] = mul4<P2>(p.coef[0], cc, nz);
          }
#pragma unroll
          for (int kk = 1; kk <= RZ; ++kk) {
#pragma unroll
            for (int v = 0; v < VY; ++v) {
              // window index i holds the i-th plane in streaming order
              const float4 zm = q[WI(jj, RZ + (DOWN ? kk : -kk))][v];
              const float4 zp = q[WI(jj, RZ + (DOWN ? -kk : kk))][v];
              if constexpr (HYB) {
                if (kk >= HK0) {
                  acc[v] = tap4<true, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1)], zm);
                  acc[v] = tap4<true, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1) + 1], zp);
                } else {
                  acc[v] = tap4<false, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1)], zm, nz);
                  acc[v] = tap4<false, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1) + 1], zp, nz);
                }
              } else if constexpr (OFMA) {
                acc[v] = tap4<true, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1)], zm);
                acc[v] = tap4<true, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1) + 1], zp);
              } else if constexpr (FAST) {
                acc[v] = tap4<true, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1)], add4<P2>(zm, zp));
              } else {
                acc[v] = tap4<false, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1)], zm, nz);
                acc[v] = tap4<false, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1) + 1], zp, nz);
              }
            }
          }
#pragma unroll
          for (int kk = 1; kk <= RY; ++kk) {
#pragma unroll
            for (int v = 0; v < VY; ++v) {
              const float4 ym = (v - kk >= 0) ? q[WI(jj, RZ)][(v - kk >= 0) ? v - kk : 0]
                                              : lds4(cs + (v - kk) * SW);
              const float4 yp = (v + kk < VY) ? q[WI(jj, RZ)][(v + kk < VY) ? v + kk : 0]
                                              : lds4(cs + (v + kk) * SW);
              if constexpr (HYB) {
                if (kk >= HK0) {
                  acc[v] = tap4<true, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1)], ym);
                  acc[v] = tap4<true, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1) + 1], yp);
                } else {
                  acc[v] = tap4<false, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1)], ym, nz);
                  acc[v] = tap4<false, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1) + 1], yp, nz);
                }
              } else if constexpr (OFMA) {
                acc[v] = tap4<true, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1)], ym);
                acc[v] = tap4<true, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1) + 1], yp);
              } else if constexpr (FAST) {
                acc[v] = tap4<true, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1)], add4<P2>(ym, yp));
              } else {
                acc[v] = tap4<false, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1)], ym, nz);
                acc[v] = tap4<false, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1) + 1], yp, nz);
              }
            }
          }
#pragma unroll
          for (int v = 0; v < VY; ++v) {
            // row segment x-XH .. x+3+XH of the centre plane
            float xs[2 * XH + 4];
#pragma unroll
            for (int l = 0; l < XL; ++l) {
              const float4 a = lds4(cs + v * SW - XH + 4 * l);
              xs[4 * l] = a.x; xs[4 * l + 1] = a.y; xs[4 * l + 2] = a.z; xs[4 * l + 3] = a.w;
              const float4 b = lds4(cs + v * SW + 4 + 4 * l);
              xs[XH + 4 + 4 * l] = b.x; xs[XH + 5 + 4 * l] = b.y; xs[XH + 6 + 4 * l] = b.z;
              xs[XH + 7 + 4 * l] = b.w;
            }
            const float4 cc = q[WI(jj, RZ)][v];
            xs[XH] = cc.x; xs[XH + 1] = cc.y; xs[XH + 2] = cc.z; xs[XH + 3] = cc.w;
            float a4[4] = {acc[v].x, acc[v].y, acc[v].z, acc[v].w};
#pragma unroll
            for (int kk = 1; kk <= RX; ++kk) {
              const float cm = p.coef[CX0 + 2 * (kk - 1)], cp = p.coef[CX0 + 2 * (kk - 1) + 1];
              if (P2 && (kk % 2 == 0 || ST_P2_ODD_X)) {
                // even offsets: x-neighbour pairs are aligned register pairs;
                // odd ones need two moves to form each pair (ST_P2_ODD_X)
#pragma unroll
                for (int i = 0; i < 4; i += 2) {
                  if constexpr (OFMA || HYB) {   // (HYB: paired x taps are the even distances, all >= HK0 = 2)
                    static_assert(!HYB || HK0 <= 2, "paired (even-distance) x taps are fused");
                    const float2 r0 = ffma2(cm, xs[XH + i - kk], xs[XH + i + 1 - kk], a4[i], a4[i + 1]);
                    const float2 r = ffma2(cp, xs[XH + i + kk], xs[XH + i + 1 + kk], r0.x, r0.y);
                    a4[i] = r.x; a4[i + 1] = r.y;
                  } else if constexpr (FAST) {
                    const float2 s2 = fadd2(xs[XH + i - kk], xs[XH + i + 1 - kk], xs[XH + i + kk], xs[XH + i + 1 + kk]);
                    const float2 r = ffma2(cm, s2.x, s2.y, a4[i], a4[i + 1]);
                    a4[i] = r.x; a4[i + 1] = r.y;
                  } else {
                    const float2 mm = fmul2(cm, xs[XH + i - kk], xs[XH + i + 1 - kk], nz);
                    const float2 s0 = fadd2(a4[i], a4[i + 1], mm.x, mm.y);
                    const float2 mp = fmul2(cp, xs[XH + i + kk], xs[XH + i + 1 + kk], nz);
                    const float2 s1 = fadd2(s0.x, s0.y, mp.x, mp.y);
                    a4[i] = s1.x; a4[i + 1] = s1.y;
                  }
                }
              } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float xm = xs[XH + i - kk], xp = xs[XH + i + kk];
                  if constexpr (OFMA || HYB) {
                    if (!HYB || kk >= HK0) {
                      a4[i] = __fmaf_rn(cp, xp, __fmaf_rn(cm, xm, a4[i]));
                    } else {
                      a4[i] = tap<false>(a4[i], cm, xm);
                      a4[i] = tap<false>(a4[i], cp, xp);
                    }
                  } else if constexpr (FAST) {
                    a4[i] = __fmaf_rn(cm, __fadd_rn(xm, xp), a4[i]);
                  } else {
                    a4[i] = tap<false>(a4[i], cm, xm);
                    a4[i] = tap<false>(a4[i], cp, xp);
                  }
                }
              }
            }
            acc[v] = make_float4(a4[0], a4[1], a4[2], a4[3]);
          }
          if constexpr (MODEL == kWave) {
            const float* aw = aux + sa * AUXF + ao;
#pragma unroll
            for (int v = 0; v < VY; ++v) {
              const float4 cc = q[WI(jj, RZ)][v];
              const float4 w2 = lds4(aw + v * TX);
              float4 mm;
              if constexpr (MC) {   // 4 one-byte codes -> the exact palette floats
                const unsigned c4 =
                    *reinterpret_cast<const unsigned*>(reinterpret_cast<const unsigned char*>(aw - ao + TX * TY) +
                                                       (cw * VY + v) * TX + cx4);
                mm = make_float4(s_pal[c4 & 255u], s_pal[(c4 >> 8) & 255u], s_pal[(c4 >> 16) & 255u], s_pal[c4 >> 24]);
              } else {
                mm = lds4(aw + TX * TY + v * TX);
              }
              if constexpr (!P2) {
              const float4 b = make_float4(__fsub_rn(__fadd_rn(cc.x, cc.x), w2.x), __fsub_rn(__fadd_rn(cc.y, cc.y), w2.y),
                                           __fsub_rn(__fadd_rn(cc.z, cc.z), w2.z), __fsub_rn(__fadd_rn(cc.w, cc.w), w2.w));
              if constexpr (FAST && !HYB) {
                acc[v] = make_float4(__fmaf_rn(mm.x, acc[v].x, b.x), __fmaf_rn(mm.y, acc[v].y, b.y),
                                     __fmaf_rn(mm.z, acc[v].z, b.z), __fmaf_rn(mm.w, acc[v].w, b.w));
              } else {
                acc[v] = make_float4(__fadd_rn(b.x, __fmul_rn(mm.x, acc[v].x)), __fadd_rn(b.y, __fmul_rn(mm.y, acc[v].y)),
                                     __fadd_rn(b.z, __fmul_rn(mm.z, acc[v].z)), __fadd_rn(b.w, __fmul_rn(mm.w, acc[v].w)));
              }
              } else {
              // 2u - u_prev (an FADD2 feeding an FSUB2: nothing to contract)
              const float2 b01 = fadd2(cc.x, cc.y, cc.x, cc.y), b23 = fadd2(cc.z, cc.w, cc.z, cc.w);
              const float2 c01 = fsub2(b01.x, b01.y, w2.x, w2.y), c23 = fsub2(b23.x, b23.y, w2.z, w2.w);
              if constexpr (FAST && !HYB) {
                const float2 r01 = ffma2v(mm.x, mm.y, acc[v].x, acc[v].y, c01.x, c01.y);
                const float2 r23 = ffma2v(mm.z, mm.w, acc[v].z, acc[v].w, c23.x, c23.y);
                acc[v] = make_float4(r01.x, r01.y, r23.x, r23.y);
              } else {
                const float2 m01 = fmul2v(mm.x, mm.y, acc[v].x, acc[v].y, nz);
                const float2 m23 = fmul2v(mm.z, mm.w, acc[v].z, acc[v].w, nz);
                const float2 r01 = fadd2(c01.x, c01.y, m01.x, m01.y), r23 = fadd2(c23.x, c23.y, m23.x, m23.y);
                acc[v] = make_float4(r01.x, r01.y, r23.x, r23.y);
              }
              }
            }
          }
#if ST_EXP == 2
#pragma unroll
          for (int v = 0; v < VY; ++v) acc[v] = q[WI(jj, RZ)][v];
#endif
          // release the centre stage (and the wave operands) of this phase
          __syncwarp();
          if constexpr (LEAN) {
            mbar_arrive_if(empty_a + 8 * sc, is0);
            if constexpr (MODEL == kWave) mbar_arrive_if(emptya_a + 8 * sa, is0);
          } else if (lane == 0) {
            mbar_arrive(empty + sc);
            if constexpr (MODEL == kWave) mbar_arrive(emptya + sa);
          }
          if (++sc == NS) sc = 0;
          if constexpr (MODEL == kWave) {
            if (++sa == NSA) sa = 0;
          }
#pragma unroll
          for (int v = 0; v < VY; ++v) {
            float* o = op + v * pitch;
            if (yok[v]) {
              if (XF || xfull) {
                *reinterpret_cast<float4*>(o) = acc[v];
              } else if (xany) {
                o[0] = acc[v].x;
                if (gx + 1 < g.nx) o[1] = acc[v].y;
                if (gx + 2 < g.nx) o[2] = acc[v].z;
              }
            }
          }
          op += zstep;
          if constexpr (BANK) halo_refresh<RZ, RY, RX>(p, dst, L, zfirst + (DOWN ? -k : k), y0, TY, x0, TX, ct, NT);
          if constexpr (WF) {
            // this warp's stores of plane k -> CTA-scope count for the
            // publisher.  Published at once: deferring it by a phase (so the
            // release fence finds the stores complete) measured 8% slower --
            // the wavefront is bound by the level-to-level lag.
            // (Posting only every 2nd / 4th plane measured slower: 350 vs 371
            // GPts/s on config 3 -- followers wait longer -- and its modulo cost
            // 15 instructions per phase.)
            ++wdone;
            if constexpr (LEAN) {
              __syncwarp();
              st_release_cta_if(wdone_a, wdone, is0);
            } else {
              __syncwarp();
              if (lane == 0)
                asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(&s_wdone[cw])), "r"(wdone) : "memory");
            }
          }
        }
        if constexpr (!UNROLLW) {   // next block: the window moves UNR planes
#pragma unroll
          for (int i = 0; i < 2 * RZ; ++i)
#pragma unroll
            for (int v = 0; v < VY; ++v) q[i][v] = q[i + UNR][v];
        }
      }
      mseq += NP;
      aseq += (unsigned)nph;
    };
    auto run = [&](const Work& w) {
      using F = cuda::std::false_type;
      using T = cuda::std::true_type;
      if (p.bank) {   // per-slot halo banks: rare (literal reference init), general stores
        if (MODEL == kWave && p.mcode_on) consume(F{}, T{}, T{}, F{}, w);
        else consume(F{}, T{}, F{}, F{}, w);
      } else if (R >= 4 && g.nx % TX == 0) {   // every x tile full (r >= 4: smaller phases stay one copy)
        if (MODEL == kWave && p.mcode_on) consume(F{}, F{}, T{}, T{}, w);
        else consume(F{}, F{}, F{}, T{}, w);
      } else {
        if (MODEL == kWave && p.mcode_on) consume(F{}, F{}, T{}, F{}, w);
        else consume(F{}, F{}, F{}, F{}, w);
      }
    };
    if constexpr (WF) {
      for (unsigned i = 0;; ++i) {
        const int e = (int)(i % QD);
        mbar_wait<2>(qfull + e, (i / QD) & 1);
        const long long t = s_q[e];
        __syncwarp();
        if (lane == 0) mbar_arrive(qempty + e);
        if (t < 0) break;
        Work w;
        wf_decode(p, t, w);
        run(w);
      }
    } else {
      ZigZagCursor cur;
      cur.init(p, level);
      Work w;
      while (cur.next(p, w)) run(w);
    }
  }
}

// ---------------------------------------------------------------------------
// Generic kernel: any term set (any offsets within the radii, any dt), read
// straight from global memory per term.  blockDim = (TX, BYT); each thread
// owns column x and rows ty, ty+BYT, ... of the tile.
// ---------------------------------------------------------------------------
template <int MODEL, bool WF>
__global__ void __launch_bounds__(256)
gen_kernel(const __grid_constant__ KParams p, int lrel_sweep) {
  __shared__ long long s_ticket;
  const int TX = blockDim.x, BYT = blockDim.y;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TX + tx, NT = TX * BYT;
  const DevGeom& g = p.g;
  const Items& it = p.it;
  const int TY = it.ty;
  SweepCursor cur;
  if constexpr (!WF) cur.init(p);
  for (;;) {
    Work w;
    if constexpr (WF) {
      __syncthreads();
      if (tid == 0) {
        long long t;
        Work tw;
        bool have;
        do {
          t = (long long)atomicAdd(p.ticket, 1u);
          have = wf_decode(p, t, tw);
        } while (have && tw.z1 <= tw.z0);
        s_ticket = have ? t : -1;
      }
      __syncthreads();
      const long long t = s_ticket;
      if (t < 0) break;
      wf_decode(p, t, w);
    } else {
      if (!cur.next(p, lrel_sweep, w)) break;
    }
    const int yb = w.col / it.nxb, xb = w.col - (w.col / it.nxb) * it.nxb;
    const int z0 = w.z0, z1 = w.z1;
    const int y0 = yb * TY, x0 = xb * TX;
    const long long L = p.level0 + w.lrel;
    float* __restrict__ dst = p.buf[L % p.nbuf];
    const float* __restrict__ u1 = p.buf[(L - 1) % p.nbuf];
    const float* __restrict__ u2 = MODEL == kWave ? p.buf[(L - 2) % p.nbuf] : nullptr;
    const int x = x0 + tx;
    DepCache dc{-1, 0, 0, 0, -1, -1};
    DepLane dl{false, 0};
    if constexpr (WF) {
      if (tid < 32) {
        dl = dep_lane(p, w.lrel, w.col, true);
        for (int pz = max(0, z0 - g.rz); pz < min(z0 + g.rz, g.nz); ++pz) wait_plane(p, w.lrel, dl, pz, dc);
      }
    }
    for (int z = z0; z < z1; ++z) {
      if constexpr (WF) {
        if (tid < 32 && z + g.rz < g.nz) wait_plane(p, w.lrel, dl, z + g.rz, dc);
        __syncthreads();
        if (tid == 0 && z > z0) st_release(p.prog + (w.ctr << p.ctr_shift), (unsigned)(z - z0));
      }
      for (int yy = ty; yy < TY; yy += BYT) {
        const int y = y0 + yy;
        if (x >= g.nx || y >= g.ny) continue;
        const long long idx = dev_index(g, z, y, x);
        float out;
        if constexpr (MODEL == kWave) {
          float acc = __fmul_rn(p.terms[0].c, ld_src<WF>(u1 + idx + p.terms[0].off));
          for (int k = 1; k < p.nterms; ++k)
            acc = tap<false>(acc, p.terms[k].c, ld_src<WF>(u1 + idx + p.terms[k].off));
          const float cc = ld_src<WF>(u1 + idx);
          const float b = __fsub_rn(__fadd_rn(cc, cc), ld_src<WF>(u2 + idx));
          out = __fadd_rn(b, __fmul_rn(__ldg(p.mfield + idx), acc));
        } else {
          const float* s0 = p.buf[(L - p.terms[0].dt) % p.nbuf];
          float acc = __fmul_rn(p.terms[0].c, ld_src<WF>(s0 + idx + p.terms[0].off));
          for (int k = 1; k < p.nterms; ++k) {
            const float* sk = p.buf[(L - p.terms[k].dt) % p.nbuf];
            acc = tap<false>(acc, p.terms[k].c, ld_src<WF>(sk + idx + p.terms[k].off));
          }
          out = acc;
        }
        dst[idx] = out;
      }
      if (p.bank) {
        const int Rz = g.rz, Ry = g.ry, Rx = g.rx;
        const bool by0 = Ry > 0 && y0 == 0, by1 = Ry > 0 && y0 + TY >= g.ny;
        const bool bx0 = Rx > 0 && x0 == 0, bx1 = Rx > 0 && x0 + TX >= g.nx;
        const bool zf0 = Rz > 0 && z == 0, zf1 = Rz > 0 && z == g.nz - 1;
        if (by0 || by1 || bx0 || bx1 || zf0 || zf1) {
          const float* __restrict__ bk = p.bank + (L % p.bank_slots) * g.buf_elems;
          const int eylo = by0 ? -Ry : y0, eyhi = by1 ? g.ny + Ry : min(g.ny, y0 + TY);
          const int exlo = bx0 ? -Rx : x0, exhi = bx1 ? g.nx + Rx : min(g.nx, x0 + TX);
          const int W = exhi - exlo, H = eyhi - eylo;
          auto copy_plane = [&](int zz, bool all) {
            for (int i = tid; i < W * H; i += NT) {
              const int yy = eylo + i / W, xx = exlo + i % W;
              const bool interior = yy >= 0 && yy < g.ny && xx >= 0 && xx < g.nx;
              if (all || !interior) {
                const long long idx = dev_index(g, zz, yy, xx);
                dst[idx] = bk[idx];
              }
            }
          };
          if (by0 || by1 || bx0 || bx1) copy_plane(z, false);
          if (zf0)
            for (int zz = -Rz; zz < 0; ++zz) copy_plane(zz, true);
          if (zf1)
            for (int zz = g.nz; zz < g.nz + Rz; ++zz) copy_plane(zz, true);
        }
      }
    }
    if constexpr (WF) {
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_release(p.prog + (w.ctr << p.ctr_shift), (unsigned)(z1 - z0));
      }
    }
  }
}

}  // namespace st
