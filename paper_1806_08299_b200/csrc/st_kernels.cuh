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

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool FAST>
__device__ __forceinline__ float tap(float acc, float c, float v) {
  if constexpr (FAST) return __fmaf_rn(c, v, acc);
  else return __fadd_rn(acc, __fmul_rn(c, v));
}

// Warp 0 (all 32 lanes): wait until level lrel-1 has completed planes
// [zlo, zneed] of every neighbour column of (yb, xb) -- 5-point (star) or
// 9-point (box) neighbourhood of tiles.  `ready` (lane-uniform) caches the
// highest plane known complete; a successful poll advances it as far as
// the counters allow so later planes rarely poll.
__device__ __forceinline__ void wf_wait_planes(const KParams& p, int lrel,
                                               int yb, int xb, int zlo,
                                               int zneed, bool box,
                                               int& ready) {
  if (lrel == 0 || zneed <= ready) return;
  const Items& it = p.it;
  const int lane = threadIdx.x & 31;
  const unsigned* prog = p.prog + (long long)(lrel - 1) * it.nitems;
  const int dy = lane / 3 - 1, dx = lane % 3 - 1;
  const int yy = yb + dy, xx = xb + dx;
  const bool mine = lane < 9 && (box || dy == 0 || dx == 0) && yy >= 0 &&
                    yy < it.nyb && xx >= 0 && xx < it.nxb;
  int zs = zlo > ready + 1 ? zlo : ready + 1;
  const int c0 = zs / it.cz, c1 = zneed / it.cz;
  int new_ready = zneed;
  for (int cc = c0; cc <= c1; ++cc) {
    const int start = cc * it.cz;
    const int end = min(p.g.nz, start + it.cz);
    const int need_hi = min(zneed, end - 1);
    const unsigned need = (unsigned)(need_hi - start + 1);
    const unsigned* f = prog + ((long long)cc * it.nyb + yy) * it.nxb + xx;
    unsigned have = mine ? ld_acquire(f) : 0xffffffffu;
    int ns = 32;
    while (true) {
      const unsigned mn = __reduce_min_sync(0xffffffffu, have);
      if (mn >= need) {
        if (cc == c1) new_ready = max(zneed, start + (int)min(mn, (unsigned)(end - start)) - 1);
        break;
      }
      __nanosleep(ns);
      ns = ns < 512 ? ns * 2 : 512;
      if (mine) have = ld_acquire(f);
    }
  }
  ready = new_ready;
}

__device__ __forceinline__ void wf_wait_level(const KParams& p, int lrel) {
  // time-tile window: level lrel may start once level lrel - T is complete
  if (lrel < p.T) return;
  const unsigned* d = p.done + (lrel - p.T);
  const unsigned need = (unsigned)p.it.nitems;
  int ns = 64;
  while (ld_acquire(d) < need) {
    __nanosleep(ns);
    ns = ns < 1024 ? ns * 2 : 1024;
  }
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

// Item fetch shared by both kernels.  Returns false when no work is left.
template <bool WF>
__device__ __forceinline__ bool next_item(const KParams& p, int lrel_sweep,
                                          int* s_ticket, int& lrel,
                                          int& item) {
  if constexpr (WF) {
    __syncthreads();  // previous item fully done with smem / s_ticket
    if (threadIdx.x == 0 && threadIdx.y == 0) *s_ticket = atomicAdd(p.ticket, 1u);
    __syncthreads();
    const int t = *s_ticket;
    if (t >= p.nsteps * p.it.nitems) return false;
    lrel = t / p.it.nitems;
    item = t - lrel * p.it.nitems;
    return true;
  } else {
    lrel = lrel_sweep;
    item = blockIdx.x;
    return true;
  }
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                            int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
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
// owns one x column and VY consecutive rows; it keeps the z-window
// (2RZ+1 planes) of its points in registers, takes x/y neighbours of the
// centre plane from the ring, and writes the output plane straight to HBM.
// blockDim.x = 32 * (1 + NC), NC = TX * BYT / 32, TY = BYT * VY.
// ---------------------------------------------------------------------------
template <int R, int DIMS, int VY, int MODEL, bool FAST, bool WF>
__global__ void __launch_bounds__(32 * 9, 1)
star_kernel(const __grid_constant__ KParams p, int lrel_sweep) {
  constexpr int RZ = DIMS >= 2 ? R : 0;
  constexpr int RY = DIMS == 3 ? R : 0;
  constexpr int RX = R;
  constexpr int NQ = 2 * RZ + 1;
  constexpr int XH = (RX + 3) / 4 * 4;      // x halo in a stage (TMA boxes start 16-B aligned)
  constexpr int CZ0 = 1;                    // coef offset of the z taps
  constexpr int CY0 = 1 + 2 * RZ;           // y taps
  constexpr int CX0 = 1 + 2 * RZ + 2 * RY;  // x taps

  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ int s_item[2];

  const DevGeom& g = p.g;
  const Items& it = p.it;
  const Pipe& pp = p.pipe;
  const int TX = it.tx, TY = it.ty;
  const int NC = (blockDim.x >> 5) - 1;     // consumer warps
  const int NT = NC * 32;                   // consumer threads
  const int NS = pp.ns, NSA = pp.nsa, SW = pp.sw;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + NS;
  uint64_t* emptya = empty + NS;
  float* ring = reinterpret_cast<float*>(smem_raw + 1024);
  float* aux = ring + (size_t)NS * pp.stage_floats;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NC);
    }
    for (int s = 0; s < NSA; ++s) mbar_init(emptya + s, NC);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  unsigned mseq = 0, aseq = 0;  // CTA-lifetime ring sequence numbers
  int next_static = blockIdx.x;
  for (;;) {
    // ---- item fetch (all threads) ----------------------------------------
    if (threadIdx.x == 0) {
      int t;
      if constexpr (WF) t = (int)atomicAdd(p.ticket, 1u);
      else t = next_static;
      s_item[0] = t;
    }
    __syncthreads();
    const int t = s_item[0];
    __syncthreads();
    int lrel, item;
    if constexpr (WF) {
      if (t >= p.nsteps * it.nitems) break;
      lrel = t / it.nitems;
      item = t - lrel * it.nitems;
    } else {
      if (t >= it.nitems) break;
      lrel = lrel_sweep;
      item = t;
      next_static += gridDim.x;
    }
    const int xb = item % it.nxb;
    const int yb = (item / it.nxb) % it.nyb;
    const int c = item / (it.nxb * it.nyb);
    const int z0 = c * it.cz, z1 = min(g.nz, z0 + it.cz);
    const int y0 = yb * TY, x0 = xb * TX;
    const int NP = z1 - z0 + 2 * RZ;        // planes loaded (incl. z halo)
    const long long L = p.level0 + lrel;
    const int bsrc = (int)((L - 1) % p.nbuf);
    const int bdst = (int)(L % p.nbuf);
    const int bu2 = MODEL == kWave ? (int)((L - 2) % p.nbuf) : 0;

    if (warp == 0) {
      // ================= producer ============================================
      int ready = z0 - RZ - 1;
      if (WF && lane == 0) wf_wait_level(p, lrel);
      __syncwarp();
      for (int j = 0; j < NP; ++j) {
        const unsigned gs = mseq + j;
        const int slot = (int)(gs % NS);
        if (gs >= (unsigned)NS) mbar_wait(empty + slot, ((gs / NS) - 1) & 1);
        const int pz = z0 - RZ + j;           // plane (interior coords)
        if constexpr (WF) {
          if (pz >= 0 && pz < g.nz) {
            const int before = ready;
            wf_wait_planes(p, lrel, yb, xb, max(0, z0 - RZ),
                           min(pz + (p.skew - RZ), g.nz - 1), false, ready);
            if (ready != before) fence_proxy_async_global();
          }
        }
        const bool with_aux = MODEL == kWave && j >= 2 * RZ;
        unsigned ga = 0;
        int aslot = 0;
        if (with_aux) {
          ga = aseq + (j - 2 * RZ);
          aslot = (int)(ga % NSA);
          if (ga >= (unsigned)NSA) mbar_wait(emptya + aslot, ((ga / NSA) - 1) & 1);
        }
        if (lane == 0) {
          mbar_expect_tx(full + slot, pp.main_bytes + (with_aux ? pp.aux_bytes : 0));
          tma_load_3d(ring + (size_t)slot * pp.stage_floats, &p.tm.main[bsrc], full + slot,
                      g.xo + x0 - XH, y0, pz + g.rz);
          if (with_aux) {
            const int zc = pz - RZ;           // centre plane of this phase
            float* a = aux + (size_t)aslot * pp.aux_floats;
            tma_load_3d(a, &p.tm.aux[bu2], full + slot, g.xo + x0, y0 + g.ry, zc + g.rz);
            tma_load_3d(a + TX * TY, &p.tm.mfield, full + slot, g.xo + x0, y0 + g.ry, zc + g.rz);
          }
        }
        __syncwarp();
      }
    } else {
      // ================= consumers ===========================================
      const int ct = threadIdx.x - 32;
      const int cx = ct % TX, cy = ct / TX;
      const int row0 = RY + cy * VY;          // first own row in a stage
      const bool xin = x0 + cx < g.nx;
      float* __restrict__ dst = p.buf[bdst];
      const long long col = dev_index(g, 0, y0 + cy * VY, x0 + cx);
      float q[NQ][VY];
      // prologue: planes 0 .. 2RZ-1 of the item into the register window
#pragma unroll
      for (int j = 0; j < 2 * RZ; ++j) {
        const unsigned gs = mseq + j;
        const int slot = (int)(gs % NS);
        mbar_wait(full + slot, (gs / NS) & 1);
        const float* st = ring + (size_t)slot * pp.stage_floats;
#pragma unroll
        for (int v = 0; v < VY; ++v) q[j][v] = st[(row0 + v) * SW + XH + cx];
        if (j < RZ || j >= NP - RZ) {         // never a centre plane: last use
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + slot);
        }
      }
      const int nph = z1 - z0;
      for (int kb = 0; kb < nph; kb += NQ) {
#pragma unroll
        for (int jj = 0; jj < NQ; ++jj) {
          const int k = kb + jj;
          if (k >= nph) break;
          const int z = z0 + k;
          // newest plane (index k + 2RZ) into the window
          {
            const unsigned gs = mseq + k + 2 * RZ;
            const int slot = (int)(gs % NS);
            mbar_wait(full + slot, (gs / NS) & 1);
            const float* st = ring + (size_t)slot * pp.stage_floats;
#pragma unroll
            for (int v = 0; v < VY; ++v) q[(jj + 2 * RZ) % NQ][v] = st[(row0 + v) * SW + XH + cx];
            if (k + 2 * RZ >= NP - RZ && RZ > 0) {  // above-chunk z halo: last use
              __syncwarp();
              if (lane == 0) mbar_arrive(empty + slot);
            }
          }
          const unsigned gc = mseq + k + RZ;        // centre plane stage
          const int cslot = (int)(gc % NS);
          const float* cs = ring + (size_t)cslot * pp.stage_floats;
          const float* aw = MODEL == kWave ? aux + (size_t)((aseq + k) % NSA) * pp.aux_floats : aux;
#pragma unroll
          for (int v = 0; v < VY; ++v) {
            const float cc = q[(jj + RZ) % NQ][v];
            float acc = __fmul_rn(p.coef[0], cc);
#pragma unroll
            for (int kk = 1; kk <= RZ; ++kk) {
              const float zm = q[(jj + RZ - kk) % NQ][v];
              const float zp = q[(jj + RZ + kk) % NQ][v];
              if constexpr (FAST) {
                acc = __fmaf_rn(p.coef[CZ0 + 2 * (kk - 1)], __fadd_rn(zm, zp), acc);
              } else {
                acc = tap<false>(acc, p.coef[CZ0 + 2 * (kk - 1)], zm);
                acc = tap<false>(acc, p.coef[CZ0 + 2 * (kk - 1) + 1], zp);
              }
            }
#pragma unroll
            for (int kk = 1; kk <= RY; ++kk) {
              const float ym = (v - kk >= 0) ? q[(jj + RZ) % NQ][(v - kk >= 0) ? v - kk : 0]
                                             : cs[(row0 + v - kk) * SW + XH + cx];
              const float yp = (v + kk < VY) ? q[(jj + RZ) % NQ][(v + kk < VY) ? v + kk : 0]
                                             : cs[(row0 + v + kk) * SW + XH + cx];
              if constexpr (FAST) {
                acc = __fmaf_rn(p.coef[CY0 + 2 * (kk - 1)], __fadd_rn(ym, yp), acc);
              } else {
                acc = tap<false>(acc, p.coef[CY0 + 2 * (kk - 1)], ym);
                acc = tap<false>(acc, p.coef[CY0 + 2 * (kk - 1) + 1], yp);
              }
            }
            const float* rp = cs + (row0 + v) * SW + XH + cx;
#pragma unroll
            for (int kk = 1; kk <= RX; ++kk) {
              const float xm = rp[-kk];
              const float xp = rp[kk];
              if constexpr (FAST) {
                acc = __fmaf_rn(p.coef[CX0 + 2 * (kk - 1)], __fadd_rn(xm, xp), acc);
              } else {
                acc = tap<false>(acc, p.coef[CX0 + 2 * (kk - 1)], xm);
                acc = tap<false>(acc, p.coef[CX0 + 2 * (kk - 1) + 1], xp);
              }
            }
            float out;
            if constexpr (MODEL == kWave) {
              const int ai = (cy * VY + v) * TX + cx;
              const float b = __fsub_rn(__fadd_rn(cc, cc), aw[ai]);
              const float mm = aw[TX * TY + ai];
              if constexpr (FAST) out = __fmaf_rn(mm, acc, b);
              else out = __fadd_rn(b, __fmul_rn(mm, acc));
            } else {
              out = acc;
            }
            if (xin && y0 + cy * VY + v < g.ny) dst[col + (long long)z * g.pstride + v * g.pitch] = out;
          }
          // release the centre stage (and the wave operands) of this phase
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(empty + cslot);
            if constexpr (MODEL == kWave) mbar_arrive(emptya + (int)((aseq + k) % NSA));
          }
          if (p.bank) halo_refresh<RZ, RY, RX>(p, dst, L, z, y0, TY, x0, TX, ct, NT);
          if constexpr (WF) {
            if ((k + 1) % pp.pub == 0 && k + 1 < nph) {
              named_bar_sync(1, NT);
              if (ct == 0) {
                __threadfence();
                st_release(p.prog + (long long)lrel * it.nitems + item, (unsigned)(k + 1));
              }
            }
          }
        }
      }
      if constexpr (WF) {
        named_bar_sync(1, NT);
        if (ct == 0) {
          __threadfence();
          st_release(p.prog + (long long)lrel * it.nitems + item, (unsigned)nph);
          atomicAdd(p.done + lrel, 1u);
        }
      }
    }
    mseq += NP;
    aseq += (unsigned)(z1 - z0);
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
  __shared__ int s_ticket;
  const int TX = blockDim.x, BYT = blockDim.y;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TX + tx, NT = TX * BYT;
  const DevGeom& g = p.g;
  const Items& it = p.it;
  const int TY = it.ty;
  int lrel, item;
  while (next_item<WF>(p, lrel_sweep, &s_ticket, lrel, item)) {
    const int xb = item % it.nxb;
    const int yb = (item / it.nxb) % it.nyb;
    const int c = item / (it.nxb * it.nyb);
    const int z0 = c * it.cz, z1 = min(g.nz, z0 + it.cz);
    const int y0 = yb * TY, x0 = xb * TX;
    const long long L = p.level0 + lrel;
    float* __restrict__ dst = p.buf[L % p.nbuf];
    const float* __restrict__ u1 = p.buf[(L - 1) % p.nbuf];
    const float* __restrict__ u2 = MODEL == kWave ? p.buf[(L - 2) % p.nbuf] : nullptr;
    const int zlast_need = min(z1 - 1 + g.rz, g.nz - 1);
    int ready = z0 - g.rz - 1;
    if constexpr (WF) {
      if (tid < 32 && tid == 0) wf_wait_level(p, lrel);
    }
    const int x = x0 + tx;
    for (int z = z0; z < z1; ++z) {
      if constexpr (WF) {
        if (tid < 32)
          wf_wait_planes(p, lrel, yb, xb, max(0, z0 - g.rz),
                         min(z + p.skew, zlast_need), true, ready);
      }
      __syncthreads();
      if constexpr (WF) {
        if (tid == 0 && z > z0)
          st_release(p.prog + (long long)lrel * it.nitems + item, (unsigned)(z - z0));
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
        // generic radii are runtime: reuse the star refresh with a runtime
        // shape by dispatching on the (small) radius set seen in practice
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
        st_release(p.prog + (long long)lrel * it.nitems + item, (unsigned)(z1 - z0));
        atomicAdd(p.done + lrel, 1u);
      }
    } else {
      break;
    }
  }
}

}  // namespace st
