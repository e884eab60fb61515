// st_resident.cuh -- SM-resident time tiling for 2-D grids that fit in the
// GPU's aggregate shared memory (config 1: 1024^2 fp32 = 4 MiB over 148 SMs).
//
// One persistent (cooperative) launch runs every step.  The grid is cut
// into GX x GY tiles (p.rgx = GX; GX = 1: row strips); CTA b owns rows
// [r0, r1) of d_1 and float4-aligned columns [c0, c1) of d_2, and keeps the
// tile plus an H-wide ring (H = R * F; HC = H rounded up to a float4 along
// d_2) of the current level in shared memory (two buffers, ping-pong per
// level).  An *epoch* advances F levels on-chip: level j of the epoch is
// valid on the tile grown by H - jR on each side (overlapped / trapezoidal
// tiles; sides at the grid boundary never shrink, the frozen halo is always
// valid).  After F levels the owned tile goes to an L2-resident level buffer
// (ping-pong per epoch) and a per-CTA epoch counter is released; the CTA
// then waits for the counters of the CTAs owning its halo ring and reads it
// back.  Memory traffic: the ring + the owned tile per F levels, all in L2;
// HBM sees the input level once and the output once.  2-D tiles keep the
// ring small for large F (fewer exchanges) where strips would recompute
// 2H rows per strip of nz / 148.
//
// Arithmetic per point is the star kernel's (reference order, or FAST
// symmetric pairs with FFMA), so results are bitwise those of the sweep.
// Halo columns and the halo rows beyond the grid are loaded once into both
// buffers and never written (frozen, uniform halos only).
#pragma once

#include "st_kernels.cuh"

namespace st {

constexpr int kResThreads = 512;

template <int R, bool FAST>
__global__ void __launch_bounds__(kResThreads, 1)
resident2d_kernel(const __grid_constant__ KParams p) {
  constexpr int XH = round_up_c(R, 4);   // frozen halo columns held at the grid's sides
  static_assert(R <= 4, "x neighbours come from one float4 per side");
  constexpr bool P2 = !ST_NO_F32X2 && !FAST && R >= ST_P2_MIN_R_EXACT;
  const float nzero = p.nzero;
  const DevGeom& g = p.g;
  const int nz = g.nz, nx = g.nx;
  const int F = p.T;                      // levels per epoch
  const int H = R * F, HC = round_up_c(H, 4);
  const int GX = p.rgx > 0 ? p.rgx : 1;
  const int G = gridDim.x / GX, b = blockIdx.x / GX, bc = blockIdx.x - b * GX, tid = threadIdx.x;
  const int NX4 = (nx + 3) / 4;
  const int r0 = (int)((long long)nz * b / G), r1 = (int)((long long)nz * (b + 1) / G);
  const int c0 = 4 * (int)((long long)NX4 * bc / GX), c1 = min(4 * (int)((long long)NX4 * (bc + 1) / GX), nx);
  // local rows [lr0, lr1) (padded rows: -R .. nz + R - 1) and columns
  // [lcs, lce) (float4 aligned); a side that reaches the grid edge takes the
  // whole frozen halo and never shrinks there
  const bool top = r0 - H <= 0, bot = r1 + H >= nz;
  const bool lft = c0 - HC <= 0, rgt = c1 + HC >= nx;
  const int lr0 = top ? -R : r0 - H, lr1 = bot ? nz + R : r1 + H;
  const int lcs = lft ? -XH : c0 - HC, lce = rgt ? 4 * NX4 + XH : c1 + HC;
  const int LR = lr1 - lr0;
  const int SW = lce - lcs + 8;           // + one float4 of slack per side (edge lanes' neighbours)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* const sbase = reinterpret_cast<float*>(smem_raw);
  const int bstride = LR * SW;
  {   // the planner sized the launch for the largest tile (resident_tile_bytes)
    unsigned dsm;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsm));
    if ((unsigned long long)2 * bstride * 4 > dsm) __trap();
  }
  auto sbuf = [&](int c) { return sbase + c * bstride; };
  // smem element of (row z, column x) in buffer c
  auto sat = [&](int c, int z, int x) { return sbuf(c) + (z - lr0) * SW + 4 + (x - lcs); };
  // device row z of a level buffer, column x = 0 at index g.xo (2-D: z = d_1)
  auto grow = [&](auto* buf, int z) { return buf + g.base + (long long)z * g.pstride; };

  // ---- load the input level into both buffers (halo columns / rows too;
  // the slack columns are zeroed: they only feed outputs outside the tile)
  {
    const int W4 = SW / 4;
    for (int i = tid; i < LR * W4; i += kResThreads) {
      const int lr = i / W4, x = lcs - 4 + (i - lr * W4) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (x >= lcs && x < lce) v = __ldcg(reinterpret_cast<const float4*>(grow(p.fin, lr0 + lr) + x));
      *reinterpret_cast<float4*>(sbase + lr * SW + (x - lcs + 4)) = v;
      *reinterpret_cast<float4*>(sbase + bstride + lr * SW + (x - lcs + 4)) = v;
    }
  }
  __syncthreads();

  // 2-D thread mapping (no divisions in the level loop): TXT float4 columns
  // x TYT rows per pass, sized for the widest (first) level of an epoch
  const int n4max = ((rgt ? 4 * NX4 : c1 + HC) - (lft ? 0 : c0 - HC)) / 4;
  const int TXT = n4max >= kResThreads ? kResThreads : (n4max + 31) / 32 * 32;
  const int TYT = kResThreads / TXT;
  const int tx = tid % TXT, ty = tid / TXT;
  // TXT need not divide the block: threads with ty >= TYT (whole warps, as
  // TXT is a multiple of 32) sit the row loops out
  const bool tya = ty < TYT;
  const unsigned rcp_tyt = 0xffffffffu / (unsigned)TYT + 1u;   // ceil(2^32 / TYT); TYT = 1 wraps to 0 and takes the whole range
  const int nepoch = (p.nsteps + F - 1) / F;
  int cur = 0;
  for (int e = 0; e < nepoch; ++e) {
    const int f = min(F, p.nsteps - e * F);
    for (int j = 1; j <= f; ++j) {
      const int lo = top ? 0 : r0 - H + j * R, hi = bot ? nz : r1 + H - j * R;
      // float4 columns of level j: [xlo, xhi) (the valid range rounded out)
      const int xlo = lft ? 0 : ((c0 - HC + j * R) & ~3);
      const int xhi = rgt ? 4 * NX4 : ((c1 + HC - j * R + 3) & ~3);
      const int n4 = (xhi - xlo) >> 2, n4r = (n4 + 31) & ~31;
      const float* __restrict__ src = sbuf(cur);
      float* __restrict__ dst = sbuf(cur ^ 1);
      // thread (ty, tx): float4 column tx (+ TXT ...) over a contiguous chunk
      // of rows, the z-window (2R+1 rows) of its column in registers: one
      // LDS.128 per row; x neighbours from the adjacent lanes (SHFL), from
      // shared memory only at warp / range edges.  Lanes past the last
      // column run along (shuffles need the whole warp) and store nothing.
      const int n = hi - lo;
      // chunk bounds n*ty / TYT by a reciprocal multiply (exact while n*TYT < 2^16,
      // which the shared-memory bound on LR guarantees)
      const int ra = !tya ? hi : TYT == 1 ? lo : lo + (int)__umulhi((unsigned)(n * ty), rcp_tyt);
      const int rb = !tya ? hi : TYT == 1 ? hi : lo + (int)__umulhi((unsigned)(n * (ty + 1)), rcp_tyt);
      const int lane = tid & 31;
      for (int x4i = tx; x4i < n4r; x4i += TXT) {
        const bool act = x4i < n4;
        const int x4 = xlo + (act ? x4i * 4 : 0);
        const bool needL = lane == 0, needR = lane == 31 || x4i + 1 >= n4;
        const float* col = src + 4 + (x4 - lcs) - lr0 * SW;   // + z * SW = row z of this column
        float* ocol = dst + 4 + (x4 - lcs) - lr0 * SW;
        float4 w[2 * R + 1];
#pragma unroll
        for (int k = 0; k < 2 * R; ++k) w[k] = lds4(col + (ra - R + k) * SW);
        // running row pointers (row r of this column in src / dst).  The row
        // loop keeps the compiler's unrolling: unroll 2, or 2R+1 (window
        // rotation by renaming, 7% fewer instructions), measured 2-4% slower
        const float* cr = col + ra * SW;
        float* orow = ocol + ra * SW;
        for (int r = ra; r < rb; ++r, cr += SW, orow += SW) {
          w[2 * R] = lds4(cr + R * SW);
          const float4 cc = w[R];
          // centre and z taps on paired FP32 (bit-exact FFMA2(-0) + FADD2, see
          // st_kernels.cuh); the x taps straddle register pairs, so scalar
          float4 acc = mul4<P2>(p.coef[0], cc, nzero);
#pragma unroll
          for (int k = 1; k <= R; ++k) {
            if constexpr (FAST) {
              acc = tap4<true, false>(acc, p.coef[1 + 2 * (k - 1)], add4<false>(w[R - k], w[R + k]));
            } else {
              acc = tap4<false, P2>(acc, p.coef[1 + 2 * (k - 1)], w[R - k], nzero);
              acc = tap4<false, P2>(acc, p.coef[2 + 2 * (k - 1)], w[R + k], nzero);
            }
          }
          // columns x4-4 .. x4-1 (left lane) and x4+4 .. x4+7 (right lane)
          float4 lf, rt;
          lf.w = __shfl_up_sync(0xffffffffu, cc.w, 1);
          rt.x = __shfl_down_sync(0xffffffffu, cc.x, 1);
          if constexpr (R >= 2) {
            lf.z = __shfl_up_sync(0xffffffffu, cc.z, 1);
            rt.y = __shfl_down_sync(0xffffffffu, cc.y, 1);
          }
          if constexpr (R >= 3) {
            lf.y = __shfl_up_sync(0xffffffffu, cc.y, 1);
            rt.z = __shfl_down_sync(0xffffffffu, cc.z, 1);
            lf.x = __shfl_up_sync(0xffffffffu, cc.x, 1);
            rt.w = __shfl_down_sync(0xffffffffu, cc.w, 1);
          }
          if (needL) lf = lds4(cr - 4);
          if (needR) rt = lds4(cr + 4);
          const float xs[12] = {lf.x, lf.y, lf.z, lf.w, cc.x, cc.y, cc.z, cc.w, rt.x, rt.y, rt.z, rt.w};
          float a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
          for (int k = 1; k <= R; ++k) {
            const float cm = p.coef[1 + 2 * R + 2 * (k - 1)], cp = p.coef[2 + 2 * R + 2 * (k - 1)];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if constexpr (FAST) {
                a4[q] = __fmaf_rn(cm, __fadd_rn(xs[4 + q - k], xs[4 + q + k]), a4[q]);
              } else {
                a4[q] = tap<false>(a4[q], cm, xs[4 + q - k]);
                a4[q] = tap<false>(a4[q], cp, xs[4 + q + k]);
              }
            }
          }
          if (act) {
            float* o = orow;
            if (x4 + 4 <= nx) {
              *reinterpret_cast<float4*>(o) = make_float4(a4[0], a4[1], a4[2], a4[3]);
            } else {
              o[0] = a4[0];
              if (x4 + 1 < nx) o[1] = a4[1];
              if (x4 + 2 < nx) o[2] = a4[2];
            }
          }
#pragma unroll
          for (int k = 0; k < 2 * R; ++k) w[k] = w[k + 1];
        }
      }
      cur ^= 1;
      __syncthreads();
    }
    if (e + 1 == nepoch) break;
    // ---- exchange: owned tile out, halo ring in
    float* gx = (e & 1) ? p.xch1 : p.xch0;
    // (thread (ty, tx): rows r0 + ty, + TYT ..., float4 columns c0 + 4 tx, + 4 TXT ...)
    const int oc4 = (c1 - c0 + 3) / 4;
    for (int z = r0 + ty; tya && z < r1; z += TYT)
      for (int k = tx; k < oc4; k += TXT) {
        const int x4 = c0 + 4 * k;
        const float* s = sat(cur, z, x4);
        float* d = grow(gx, z) + x4;
        if (x4 + 4 <= nx) __stcg(reinterpret_cast<float4*>(d), lds4(s));
        else for (int q = 0; q < nx - x4; ++q) d[q] = s[q];
      }
    __syncthreads();
    if (tid == 0) {
      fence_release_gpu();
      st_relaxed(p.prog + ((long long)blockIdx.x << p.ctr_shift), (unsigned)(e + 1));
    }
    // wait for the owners of the interior part of the ring: rows [hz0, hz1)
    // x columns [hx0, hx1) minus the own tile
    const int hz0 = max(lr0, 0), hz1 = min(lr1, nz);
    const int hx0 = max(lcs, 0), hx1 = min(lce, nx);
    if (tid < 32) {
      // owner of row z: the largest o with nz*o/G <= z (columns: of float4 column x4)
      auto owner = [](long long z, int G_, int n_) { return (int)(((z + 1) * G_ + n_ - 1) / n_) - 1; };
      const int ob0 = owner(hz0, G, nz), ob1 = owner(hz1 - 1, G, nz);
      const int oc0 = owner(hx0 / 4, GX, NX4), oc1 = owner((hx1 - 1) / 4, GX, NX4);
      const int ncx = oc1 - oc0 + 1, nown = (ob1 - ob0 + 1) * ncx;
      for (int k = tid; k < nown; k += 32) {
        const int o = (ob0 + k / ncx) * GX + oc0 + k % ncx;
        if (o == (int)blockIdx.x) continue;
        long long spin = 0;
        int ns = 32;
        while (ld_acquire(p.prog + ((long long)o << p.ctr_shift)) < (unsigned)(e + 1)) {
          __nanosleep(ns);
          ns = ns < 256 ? ns * 2 : 256;
          if (++spin > (1LL << 24)) watchdog_trip(p, 3, o, e + 1, 0);
        }
      }
    }
    __syncthreads();
    {
      // rows outside the tile: every column of [hx0, hx1); rows of the tile:
      // the side columns [hx0, c0) and [c1, hx1) only
      const int hc4 = (hx1 - hx0 + 3) / 4, nl = (c0 - hx0) / 4, nr = (hx1 - c1 + 3) / 4;
      for (int z = hz0 + ty; tya && z < hz1; z += TYT) {
        const bool own = z >= r0 && z < r1;
        const int nk = own ? nl + nr : hc4;
        for (int k = tx; k < nk; k += TXT) {
          const int x4 = own && k >= nl ? c1 + 4 * (k - nl) : hx0 + 4 * k;
          const float* s = grow(gx, z) + x4;
          float* d = sat(cur, z, x4);
          if (x4 + 4 <= nx) *reinterpret_cast<float4*>(d) = __ldcg(reinterpret_cast<const float4*>(s));
          else for (int q = 0; q < nx - x4; ++q) d[q] = __ldcg(s + q);
        }
      }
    }
    __syncthreads();
  }
  // ---- the newest level's owned tile to the output buffer
  {
    const int oc4 = (c1 - c0 + 3) / 4;
    for (int z = r0 + ty; tya && z < r1; z += TYT)
      for (int k = tx; k < oc4; k += TXT) {
        const int x4 = c0 + 4 * k;
        const float* s = sat(cur, z, x4);
        float* d = grow(p.fout, z) + x4;
        if (x4 + 4 <= nx) *reinterpret_cast<float4*>(d) = lds4(s);
        else for (int q = 0; q < nx - x4; ++q) d[q] = s[q];
      }
  }
}

}  // namespace st
