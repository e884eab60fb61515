// st_resident.cuh -- SM-resident time tiling for 2-D grids that fit in the
// GPU's aggregate shared memory (config 1: 1024^2 fp32 = 4 MiB over 148 SMs).
//
// One persistent (cooperative) launch runs every step.  CTA b owns the row
// range [r0, r1) of d_1 (balanced) and keeps rows [r0 - H, r1 + H) of the
// current level in shared memory (two buffers, ping-pong per level), H =
// R * F.  An *epoch* advances F levels on-chip: level j of the epoch is valid
// on rows [r0 - H + jR, r1 + H - jR) (overlapped / trapezoidal tiles along
// d_1; rows at the grid boundary never shrink, the frozen halo rows are
// always valid).  After F levels the owned rows go to an L2-resident level
// buffer (ping-pong per epoch) and a per-CTA epoch counter is released; the
// CTA then waits for the counters of the CTAs owning its 2H halo rows and
// reads them back.  Memory traffic: 2H halo rows + the owned rows per F
// levels, all in L2; HBM sees the input level once and the output once.
//
// Arithmetic per point is the star kernel's (reference order, or FAST
// symmetric pairs with FFMA), so results are bitwise those of the sweep.
// Halo columns and the halo rows beyond the grid are loaded once into both
// buffers and never written (frozen, uniform halos only).
#pragma once

#include "st_kernels.cuh"

namespace st {

constexpr int kResThreads = 512;

template <int R>
ST_HD constexpr int resident_row_floats(int nx) {
  return round_up_c(nx + 2 * round_up_c(R, 4), 4);
}

template <int R, bool FAST>
__global__ void __launch_bounds__(kResThreads, 1)
resident2d_kernel(const __grid_constant__ KParams p) {
  constexpr int XH = round_up_c(R, 4);   // column of x = 0 inside a smem row
  static_assert(R <= 4, "x neighbours come from one float4 per side");
  constexpr bool P2 = !ST_NO_F32X2 && !FAST && R >= ST_P2_MIN_R_EXACT;
  const float nzero = p.nzero;
  const DevGeom& g = p.g;
  const int nz = g.nz, nx = g.nx;
  const int F = p.T;                      // levels per epoch
  const int H = R * F;
  const int SW = round_up_c(nx + 2 * XH, 4);
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int r0 = (int)((long long)nz * b / G), r1 = (int)((long long)nz * (b + 1) / G);
  // local rows [lr0, lr1) (padded rows: -R .. nz + R - 1); a range that
  // reaches the grid edge takes the whole frozen halo and never shrinks there
  const bool top = r0 - H <= 0, bot = r1 + H >= nz;
  const int lr0 = top ? -R : r0 - H, lr1 = bot ? nz + R : r1 + H;
  const int LR = lr1 - lr0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* const sbase = reinterpret_cast<float*>(smem_raw);
  const int bstride = LR * SW;
  auto sbuf = [&](int c) { return sbase + c * bstride; };
  const long long pitch = g.pitch;
  // device row z of a level buffer, column x = 0 at index g.xo (2-D: z = d_1)
  auto grow = [&](auto* buf, int z) { return buf + g.base + (long long)z * g.pstride; };
  (void)pitch;

  // ---- load the input level into both buffers (halo columns / rows too)
  {
    // float4 columns [-XH, nx + XH): the halo columns plus aligned slack
    // (g.xo >= XH, pitch covers nx + XH)
    const int W4 = (nx + 2 * XH + 3) / 4;
    for (int i = tid; i < LR * W4; i += kResThreads) {
      const int lr = i / W4, x = (i - lr * W4) * 4 - XH;
      const float4 v = __ldcg(reinterpret_cast<const float4*>(grow(p.fin, lr0 + lr) + x));
      *reinterpret_cast<float4*>(sbase + lr * SW + XH + x) = v;
      *reinterpret_cast<float4*>(sbase + bstride + lr * SW + XH + x) = v;
    }
  }
  __syncthreads();

  const int NX4 = (nx + 3) / 4;
  // 2-D thread mapping (no divisions in the level loop): TXT float4 columns
  // x TYT rows per pass
  const int TXT = NX4 >= kResThreads ? kResThreads : (NX4 + 31) / 32 * 32;
  const int TYT = kResThreads / TXT;
  const int NX4r = (NX4 + 31) / 32 * 32;   // columns incl. the idle lanes of the last warp
  const int tx = tid % TXT, ty = tid / TXT;
  // TXT need not divide the block: threads with ty >= TYT (whole warps, as
  // TXT is a multiple of 32) sit the row loops out
  const bool tya = ty < TYT;
  const int nepoch = (p.nsteps + F - 1) / F;
  int cur = 0;
  for (int e = 0; e < nepoch; ++e) {
    const int f = min(F, p.nsteps - e * F);
    for (int j = 1; j <= f; ++j) {
      const int lo = top ? 0 : r0 - H + j * R, hi = bot ? nz : r1 + H - j * R;
      const float* __restrict__ src = sbuf(cur);
      float* __restrict__ dst = sbuf(cur ^ 1);
      // thread (ty, tx): float4 column tx (+ TXT ...) over a contiguous chunk
      // of rows, the z-window (2R+1 rows) of its column in registers: one
      // LDS.128 per row; x neighbours from the adjacent lanes (SHFL), from
      // shared memory only at warp / grid edges.  Lanes past the last column
      // run along (shuffles need the whole warp) and store nothing.
      const int n = hi - lo;
      const int ra = tya ? lo + (n * ty) / TYT : hi, rb = tya ? lo + (n * (ty + 1)) / TYT : hi;
      const int lane = tid & 31;
      for (int x4i = tx; x4i < NX4r; x4i += TXT) {
        const bool act = x4i < NX4;
        const int x4 = act ? x4i * 4 : 0;
        const bool needL = lane == 0, needR = lane == 31 || x4i + 1 >= NX4;
        const float* col = src + XH + x4 - lr0 * SW;   // + z * SW = row z of this column
        float* ocol = dst + XH + x4 - lr0 * SW;
        float4 w[2 * R + 1];
#pragma unroll
        for (int k = 0; k < 2 * R; ++k) w[k] = lds4(col + (ra - R + k) * SW);
#pragma unroll 2
        for (int r = ra; r < rb; ++r) {
          w[2 * R] = lds4(col + (r + R) * SW);
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
          if (needL) lf = lds4(col + r * SW - 4);
          if (needR) rt = lds4(col + r * SW + 4);
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
            float* o = ocol + r * SW;
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
    // ---- exchange: owned rows out, halo rows in
    float* gx = (e & 1) ? p.xch1 : p.xch0;
    for (int x4i = tx; tya && x4i < NX4; x4i += TXT)
      for (int z = r0 + ty; z < r1; z += TYT) {
        const int x4 = x4i * 4;
        const float* s = sbuf(cur) + (z - lr0) * SW + XH + x4;
        float* d = grow(gx, z) + x4;
        if (x4 + 4 <= nx) __stcg(reinterpret_cast<float4*>(d), lds4(s));
        else for (int q = 0; q < nx - x4; ++q) d[q] = s[q];
      }
    __syncthreads();
    if (tid == 0) {
      fence_release_gpu();
      st_relaxed(p.prog + ((long long)b << p.ctr_shift), (unsigned)(e + 1));
    }
    // wait for the owners of the halo rows [lr0, r0) and [r1, lr1) (interior rows only)
    const int hz0 = max(lr0, 0), hz1 = min(lr1, nz);
    if (tid < 32) {
      // owner of row z: the largest o with nz*o/G <= z
      auto owner = [&](int z) { return (int)((((long long)z + 1) * G + nz - 1) / nz) - 1; };
      const int ob0 = hz0 < r0 ? owner(hz0) : b;
      const int ob1 = hz1 > r1 ? owner(hz1 - 1) : b;
      for (int o = ob0 + tid; o <= ob1; o += 32) {
        if (o == b) continue;
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
      const int nh = (r0 - hz0) + (hz1 - r1);   // halo rows: [hz0, r0) then [r1, hz1)
      for (int x4i = tx; tya && x4i < NX4; x4i += TXT)
        for (int rr = ty; rr < nh; rr += TYT) {
          const int x4 = x4i * 4;
          const int z = rr < r0 - hz0 ? hz0 + rr : r1 + (rr - (r0 - hz0));
          const float* s = grow(gx, z) + x4;
          float* d = sbuf(cur) + (z - lr0) * SW + XH + x4;
          if (x4 + 4 <= nx) *reinterpret_cast<float4*>(d) = __ldcg(reinterpret_cast<const float4*>(s));
          else for (int q = 0; q < nx - x4; ++q) d[q] = __ldcg(s + q);
        }
    }
    __syncthreads();
  }
  // ---- the newest level's owned rows to the output buffer
  for (int x4i = tx; tya && x4i < NX4; x4i += TXT)
    for (int z = r0 + ty; z < r1; z += TYT) {
      const int x4 = x4i * 4;
      const float* s = sbuf(cur) + (z - lr0) * SW + XH + x4;
      float* d = grow(p.fout, z) + x4;
      if (x4 + 4 <= nx) *reinterpret_cast<float4*>(d) = lds4(s);
      else for (int q = 0; q < nx - x4; ++q) d[q] = s[q];
    }
}

}  // namespace st
