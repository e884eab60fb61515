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
// Star kernel: stencils whose terms are the canonical star (centre, then per
// reference axis d_1..d_n: -1, +1, -2, +2, ..., -R, +R), all reading level
// L-1 (heat) or the wave model.  blockDim = (TX, BYT); TY = BYT * VY.
// ---------------------------------------------------------------------------
template <int R, int DIMS, int VY, int MODEL, bool FAST, bool WF>
__global__ void __launch_bounds__(256)
star_kernel(const __grid_constant__ KParams p, int lrel_sweep) {
  constexpr int RZ = DIMS >= 2 ? R : 0;
  constexpr int RY = DIMS == 3 ? R : 0;
  constexpr int RX = R;
  constexpr int NQ = 2 * RZ + 2;
  constexpr int HPT = 4;
  constexpr int CZ0 = 1;                 // coef offset of the z taps
  constexpr int CY0 = 1 + 2 * RZ;        // y taps
  constexpr int CX0 = 1 + 2 * RZ + 2 * RY;  // x taps

  extern __shared__ float smem[];
  __shared__ int s_ticket;

  const int TX = blockDim.x, BYT = blockDim.y;
  const int TY = BYT * VY;
  const int SW = TX + 2 * RX, SH = TY + 2 * RY;
  float* const sm0 = smem;
  float* const sm1 = smem + SW * SH;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TX + tx, NT = TX * BYT;
  const DevGeom& g = p.g;
  const Items& it = p.it;

  // Fixed assignment of the tile's plane halo cells to threads.
  const int NHY = 2 * RY * TX, NH = NHY + 2 * RX * TY;
  int h_sm[HPT], h_rel[HPT];
#pragma unroll
  for (int k = 0; k < HPT; ++k) {
    const int h = tid + k * NT;
    h_sm[k] = -1;
    h_rel[k] = 0;
    if (h < NH) {
      int row, col, gy, gx;
      if (h < NHY) {
        const int i = h / TX;
        col = RX + h % TX;
        row = i < RY ? i : TY + i;
        gy = row - RY;
        gx = col - RX;
      } else {
        const int h2 = h - NHY;
        const int r = h2 / (2 * RX), j = h2 % (2 * RX);
        col = j < RX ? j : TX + j;
        row = RY + r;
        gy = r;
        gx = col - RX;
      }
      h_sm[k] = row * SW + col;
      h_rel[k] = (int)(gy * g.pitch + gx);
    }
  }

  int lrel, item;
  while (next_item<WF>(p, lrel_sweep, &s_ticket, lrel, item)) {
    const int xb = item % it.nxb;
    const int yb = (item / it.nxb) % it.nyb;
    const int c = item / (it.nxb * it.nyb);
    const int z0 = c * it.cz, z1 = min(g.nz, z0 + it.cz);
    const int y0 = yb * TY, x0 = xb * TX;
    const long long L = p.level0 + lrel;
    const float* __restrict__ src = p.buf[(L - 1) % p.nbuf];
    float* __restrict__ dst = p.buf[L % p.nbuf];
    const float* __restrict__ u2 = MODEL == kWave ? p.buf[(L - 2) % p.nbuf] : nullptr;
    const int zlast_need = min(z1 - 1 + RZ, g.nz - 1);  // last interior plane read

    int ready = z0 - RZ - 1;
    if constexpr (WF) {
      if (tid < 32) {
        if (tid == 0) wf_wait_level(p, lrel);
        wf_wait_planes(p, lrel, yb, xb, max(0, z0 - RZ),
                       min(z0 + p.skew + 1, zlast_need), false, ready);
      }
      __syncthreads();
    }

    const long long col = dev_index(g, 0, y0 + ty * VY, x0 + tx);
    const long long hb = dev_index(g, 0, y0, x0);
    const bool xin = x0 + tx < g.nx;

    float q[NQ][VY];
#pragma unroll
    for (int d = 0; d < 2 * RZ + 1; ++d) {
      const float* pz = src + col + (long long)(z0 - RZ + d) * g.pstride;
#pragma unroll
      for (int v = 0; v < VY; ++v) q[d][v] = ld_src<WF>(pz + v * g.pitch);
    }
    float hv[HPT];
#pragma unroll
    for (int k = 0; k < HPT; ++k)
      hv[k] = h_sm[k] >= 0 ? ld_src<WF>(src + hb + (long long)z0 * g.pstride + h_rel[k]) : 0.f;
    float w2[2][VY], wm[2][VY];
    if constexpr (MODEL == kWave) {
#pragma unroll
      for (int v = 0; v < VY; ++v) {
        w2[0][v] = ld_src<WF>(u2 + col + (long long)z0 * g.pstride + v * g.pitch);
        wm[0][v] = __ldg(p.mfield + col + (long long)z0 * g.pstride + v * g.pitch);
      }
    }

    for (int zb = z0; zb < z1; zb += NQ) {
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const int z = zb + j;
        if (z >= z1) break;
        // (a) lookahead: plane z+RZ+1 of the source level
        if (z + 1 < z1) {
          const float* pz = src + col + (long long)(z + RZ + 1) * g.pstride;
#pragma unroll
          for (int v = 0; v < VY; ++v)
            q[(j + 2 * RZ + 1) % NQ][v] = ld_src<WF>(pz + v * g.pitch);
        }
        // (b) stage plane z (centre + halo) in shared memory
        float* const sm = (j & 1) ? sm1 : sm0;
#pragma unroll
        for (int v = 0; v < VY; ++v)
          sm[(RY + ty * VY + v) * SW + RX + tx] = q[(j + RZ) % NQ][v];
#pragma unroll
        for (int k = 0; k < HPT; ++k)
          if (h_sm[k] >= 0) sm[h_sm[k]] = hv[k];
        // (c) prefetch halo / wave operands of plane z+1
        if (z + 1 < z1) {
#pragma unroll
          for (int k = 0; k < HPT; ++k)
            if (h_sm[k] >= 0)
              hv[k] = ld_src<WF>(src + hb + (long long)(z + 1) * g.pstride + h_rel[k]);
          if constexpr (MODEL == kWave) {
#pragma unroll
            for (int v = 0; v < VY; ++v) {
              w2[(j + 1) & 1][v] = ld_src<WF>(u2 + col + (long long)(z + 1) * g.pstride + v * g.pitch);
              wm[(j + 1) & 1][v] = __ldg(p.mfield + col + (long long)(z + 1) * g.pstride + v * g.pitch);
            }
          }
        }
        // (d) wavefront: make the planes the next step loads visible
        if constexpr (WF) {
          if (tid < 32)
            wf_wait_planes(p, lrel, yb, xb, 0,
                           min(z + p.skew + 2, zlast_need), false, ready);
        }
        __syncthreads();
        if constexpr (WF) {
          // every thread finished plane z-1 (stores included)
          if (tid == 0 && z > z0)
            st_release(p.prog + (long long)lrel * it.nitems + item, (unsigned)(z - z0));
        }
        // (f) the update, canonical term order
        const int srow = RY + ty * VY;
#pragma unroll
        for (int v = 0; v < VY; ++v) {
          const float cc = q[(j + RZ) % NQ][v];
          float acc = __fmul_rn(p.coef[0], cc);
#pragma unroll
          for (int k = 1; k <= RZ; ++k) {
            const float zm = q[(j + RZ - k) % NQ][v];
            const float zp = q[(j + RZ + k) % NQ][v];
            if constexpr (FAST) {
              acc = __fmaf_rn(p.coef[CZ0 + 2 * (k - 1)], __fadd_rn(zm, zp), acc);
            } else {
              acc = tap<false>(acc, p.coef[CZ0 + 2 * (k - 1)], zm);
              acc = tap<false>(acc, p.coef[CZ0 + 2 * (k - 1) + 1], zp);
            }
          }
#pragma unroll
          for (int k = 1; k <= RY; ++k) {
            const float ym = (v - k >= 0) ? q[(j + RZ) % NQ][(v - k >= 0) ? v - k : 0]
                                          : sm[(srow + v - k) * SW + RX + tx];
            const float yp = (v + k < VY) ? q[(j + RZ) % NQ][(v + k < VY) ? v + k : 0]
                                          : sm[(srow + v + k) * SW + RX + tx];
            if constexpr (FAST) {
              acc = __fmaf_rn(p.coef[CY0 + 2 * (k - 1)], __fadd_rn(ym, yp), acc);
            } else {
              acc = tap<false>(acc, p.coef[CY0 + 2 * (k - 1)], ym);
              acc = tap<false>(acc, p.coef[CY0 + 2 * (k - 1) + 1], yp);
            }
          }
          const float* srowp = sm + (srow + v) * SW + RX + tx;
#pragma unroll
          for (int k = 1; k <= RX; ++k) {
            const float xm = srowp[-k];
            const float xp = srowp[k];
            if constexpr (FAST) {
              acc = __fmaf_rn(p.coef[CX0 + 2 * (k - 1)], __fadd_rn(xm, xp), acc);
            } else {
              acc = tap<false>(acc, p.coef[CX0 + 2 * (k - 1)], xm);
              acc = tap<false>(acc, p.coef[CX0 + 2 * (k - 1) + 1], xp);
            }
          }
          float out;
          if constexpr (MODEL == kWave) {
            const float b = __fsub_rn(__fadd_rn(cc, cc), w2[j & 1][v]);
            if constexpr (FAST) out = __fmaf_rn(wm[j & 1][v], acc, b);
            else out = __fadd_rn(b, __fmul_rn(wm[j & 1][v], acc));
          } else {
            out = acc;
          }
          if (xin && y0 + ty * VY + v < g.ny)
            dst[col + (long long)z * g.pstride + v * g.pitch] = out;
        }
        if (p.bank) halo_refresh<RZ, RY, RX>(p, dst, L, z, y0, TY, x0, TX, tid, NT);
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
