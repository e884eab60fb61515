// st_fused.cuh -- on-chip temporal blocking: F levels per HBM round trip
// (heat and leapfrog-wave star stencils, radius 1 and 2; the radius-4 wave at
// F = 2 as a measurement).
//
// The wavefront kernel (st_kernels.cuh) writes every level to memory and
// relies on L2 for reuse.  This kernel realises the time tile the way the
// paper's overlapped tile_time does on a CPU cache, but on-chip: one pass
// reads level L-1 once, advances it F levels in registers + shared memory
// and writes only level L+F-1.  The x/y tile is *overlapped*: the thread
// grid covers the output tile plus a halo of R*(F-1) points on each side,
// whose values are recomputed redundantly by neighbouring tiles (no
// inter-CTA communication).  Along z each CTA streams a balanced range of
// column-planes; a range starts R*F planes early and ends R*F planes late
// (the trapezoid of the time tile).
//
// Per CTA: warp 0 = TMA producer (one box per level-0 plane: the compute
// grid plus an R halo, into an NS-deep ring guarded by full/empty
// mbarriers); main warps own 128 x of VY rows each (lane = 4 consecutive x,
// LDS.128/STG.128); edge warps own the 4-wide x-halo columns.  Every level
// j < F keeps the (2R+1)-plane z-window of its own points in registers;
// levels j >= 1 publish their centre plane to a double-buffered shared
// plane (one named barrier per plane for all F levels) from which level
// j+1 reads x/y neighbours.  Level j at plane iteration k computes plane
// z_s + k - j*R (z_s = first level-0 plane of the range).
//
// Frozen halos: a point outside the interior keeps its
// (uniform) halo value at every level -- the value it had one level down,
// never recomputed.  Only uniform-halo grids take this path.
//
// The leapfrog wave (MODEL 1) reads two levels and writes two: each ring
// stage also carries the u^{n-1} and m tiles of the compute grid (level 1's
// operands); level j >= 2 takes u_{j-2} from the oldest slot of window j-2
// and m from the stage loaded (j-1)R planes earlier.
//
// Arithmetic per point is the star kernel's exactly (same term order, same
// rounding; FAST pairs symmetric taps with FFMA), so every F gives results
// bitwise equal to the one-level-per-pass sweep.
#pragma once

#include "st_kernels.cuh"

namespace st {

// Compile-time shape: R radius, F fused levels, TY output rows, VY rows per
// thread, PD prefetch planes.
struct FusedShape {
  int TX, HX, HY, XH, CX, CY, NRG, EC, NW, NE, NCW, BW, BH, MAINF, MOFF, AUX, STAGE, LAG, NS;
};

// MODEL 1 (wave): each ring stage also carries the u^{n-1} and m tiles of the
// compute grid (level 1's operands; m is reused by level j  (j-1)R planes
// later, so a stage lives LAG = R*max(1, F-1) iterations).
ST_HD constexpr FusedShape fused_shape(int R, int F, int TY, int VY, int PD, int MODEL = 0) {
  FusedShape s{};
  s.TX = 128;
  s.HX = round_up_c(R * (F - 1), 4);   // x compute halo (float4 granules)
  s.HY = R * (F - 1);                  // y compute halo
  s.XH = round_up_c(R, 4);             // box x halo beyond the compute grid (16-B aligned TMA)
  s.CX = s.TX + 2 * s.HX;
  s.CY = TY + 2 * s.HY;
  s.NRG = s.CY / VY;                   // row groups = main warps
  s.EC = s.HX / 4;                     // edge float4 columns per side
  s.NW = s.NRG;
  s.NE = (2 * s.EC * s.NRG + 31) / 32;
  s.NCW = s.NW + s.NE;                 // consumer warps
  s.BW = s.CX + 2 * s.XH;              // TMA box / smem plane row (floats)
  s.BH = s.CY + 2 * R;
  s.MAINF = round_up_c(s.BW * s.BH, 32);
  s.MOFF = round_up_c(s.CX * s.CY, 32);   // m tile offset inside the aux area (128-B aligned)
  s.AUX = MODEL == 1 ? 2 * s.MOFF : 0;
  s.STAGE = s.MAINF + s.AUX;
  s.LAG = MODEL == 1 ? R * (F > 2 ? F - 1 : 1) : R;
  s.NS = s.LAG + 1 + PD;
  return s;
}

ST_HD constexpr int fused_smem_bytes(int R, int F, int TY, int VY, int PD, int MODEL = 0) {
  return 1024 + (fused_shape(R, F, TY, VY, PD, MODEL).NS * fused_shape(R, F, TY, VY, PD, MODEL).STAGE +
                 2 * (F - 1) * fused_shape(R, F, TY, VY, PD, MODEL).MAINF) * 4;
}
ST_HD constexpr int fused_threads(int R, int F, int TY, int VY, int PD, int MODEL = 0) {
  return 32 * (1 + fused_shape(R, F, TY, VY, PD, MODEL).NCW);
}

// One level at the thread's VY x 4 points: acc = star(window w, centre plane
// smem at cs).  Window slot (jj + i) % NQ holds plane (centre - R + i).
template <int R, int VY, int BW, bool FAST>
__device__ __forceinline__ void fused_point(const KParams& p, const float4 (&w)[2 * R + 1][VY], int jj,
                                            const float* cs, float4 (&acc)[VY]) {
  constexpr int NQ = 2 * R + 1;
  constexpr bool P2 = !ST_NO_F32X2 && R >= (FAST ? ST_P2_MIN_R_FAST : ST_P2_MIN_R_EXACT);   // as the star kernel
  constexpr int XH = round_up_c(R, 4), XL = XH / 4;
  constexpr int CZ0 = 1, CY0 = 1 + 2 * R, CX0 = 1 + 4 * R;
#pragma unroll
  for (int v = 0; v < VY; ++v) acc[v] = mul4<P2>(p.coef[0], w[(jj + R) % NQ][v], p.nzero);
#pragma unroll
  for (int kk = 1; kk <= R; ++kk) {
#pragma unroll
    for (int v = 0; v < VY; ++v) {
      const float4 zm = w[(jj + R - kk) % NQ][v];
      const float4 zp = w[(jj + R + kk) % NQ][v];
      if constexpr (FAST) {
        acc[v] = tap4<true, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1)], add4<P2>(zm, zp));
      } else {
        acc[v] = tap4<false, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1)], zm, p.nzero);
        acc[v] = tap4<false, P2>(acc[v], p.coef[CZ0 + 2 * (kk - 1) + 1], zp, p.nzero);
      }
    }
  }
#pragma unroll
  for (int kk = 1; kk <= R; ++kk) {
#pragma unroll
    for (int v = 0; v < VY; ++v) {
      const float4 ym = (v - kk >= 0) ? w[(jj + R) % NQ][(v - kk >= 0) ? v - kk : 0] : lds4(cs + (v - kk) * BW);
      const float4 yp = (v + kk < VY) ? w[(jj + R) % NQ][(v + kk < VY) ? v + kk : 0] : lds4(cs + (v + kk) * BW);
      if constexpr (FAST) {
        acc[v] = tap4<true, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1)], add4<P2>(ym, yp));
      } else {
        acc[v] = tap4<false, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1)], ym, p.nzero);
        acc[v] = tap4<false, P2>(acc[v], p.coef[CY0 + 2 * (kk - 1) + 1], yp, p.nzero);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < VY; ++v) {
    float xs[2 * XH + 4];
#pragma unroll
    for (int l = 0; l < XL; ++l) {
      const float4 a = lds4(cs + v * BW - XH + 4 * l);
      xs[4 * l] = a.x; xs[4 * l + 1] = a.y; xs[4 * l + 2] = a.z; xs[4 * l + 3] = a.w;
      const float4 b = lds4(cs + v * BW + 4 + 4 * l);
      xs[XH + 4 + 4 * l] = b.x; xs[XH + 5 + 4 * l] = b.y; xs[XH + 6 + 4 * l] = b.z; xs[XH + 7 + 4 * l] = b.w;
    }
    const float4 cc = w[(jj + R) % NQ][v];
    xs[XH] = cc.x; xs[XH + 1] = cc.y; xs[XH + 2] = cc.z; xs[XH + 3] = cc.w;
    float a4[4] = {acc[v].x, acc[v].y, acc[v].z, acc[v].w};
#pragma unroll
    for (int kk = 1; kk <= R; ++kk) {
      const float cm = p.coef[CX0 + 2 * (kk - 1)], cp = p.coef[CX0 + 2 * (kk - 1) + 1];
      if (P2 && kk % 2 == 0) {
#pragma unroll
        for (int i = 0; i < 4; i += 2) {
          if constexpr (FAST) {
            const float2 s2 = fadd2(xs[XH + i - kk], xs[XH + i + 1 - kk], xs[XH + i + kk], xs[XH + i + 1 + kk]);
            const float2 r = ffma2(cm, s2.x, s2.y, a4[i], a4[i + 1]);
            a4[i] = r.x; a4[i + 1] = r.y;
          } else {
            const float2 mm = fmul2(cm, xs[XH + i - kk], xs[XH + i + 1 - kk], p.nzero);
            const float2 s0 = fadd2(a4[i], a4[i + 1], mm.x, mm.y);
            const float2 mp = fmul2(cp, xs[XH + i + kk], xs[XH + i + 1 + kk], p.nzero);
            const float2 s1 = fadd2(s0.x, s0.y, mp.x, mp.y);
            a4[i] = s1.x; a4[i + 1] = s1.y;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float xm = xs[XH + i - kk], xp = xs[XH + i + kk];
          if constexpr (FAST) {
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
}

// Frozen halo: a point outside the interior keeps its value at every level
// (SPEC.md:337), so its level-j value is its level-(j-1) value -- the centre
// of the source window (by induction down to level 0, which the TMA box read
// from the buffer's uniform halo).  Points beyond the padded grid carry
// whatever level 0 had there (TMA zero fill); no valid point reads them.
template <int VY>
__device__ __forceinline__ void fused_halo(const DevGeom& g, float4 (&val)[VY], const float4 (&centre)[VY], int P,
                                           int gy, int gx, bool allin) {
  const bool zin = P >= 0 && P < g.nz;
  if (zin && allin) return;
#pragma unroll
  for (int v = 0; v < VY; ++v) {
    const int y = gy + v;
    const bool yin = zin && y >= 0 && y < g.ny;
    val[v].x = (yin && gx >= 0 && gx < g.nx) ? val[v].x : centre[v].x;
    val[v].y = (yin && gx + 1 >= 0 && gx + 1 < g.nx) ? val[v].y : centre[v].y;
    val[v].z = (yin && gx + 2 >= 0 && gx + 2 < g.nx) ? val[v].z : centre[v].z;
    val[v].w = (yin && gx + 3 >= 0 && gx + 3 < g.nx) ? val[v].w : centre[v].w;
  }
}

template <int R, int F, int TY, int VY, int PD, bool FAST, int MODEL = 0>
__global__ void __launch_bounds__(fused_threads(R, F, TY, VY, PD, MODEL), 1)
fused_kernel(const __grid_constant__ KParams p) {
  constexpr FusedShape S = fused_shape(R, F, TY, VY, PD, MODEL);
  constexpr int NQ = 2 * R + 1, NS = S.NS, BW = S.BW, STAGE = S.STAGE, MAINF = S.MAINF, TX = S.TX;
  constexpr int HX = S.HX, HY = S.HY, XH = S.XH, NW = S.NW, EC = S.EC, NRG = S.NRG;
  constexpr int CX = S.CX, CY = S.CY, LAG = S.LAG, MOFF = S.MOFF;
  constexpr int NCT = S.NCW * 32;
  constexpr bool WAVE = MODEL == kWave;
  constexpr bool P2 = !ST_NO_F32X2 && R >= (FAST ? ST_P2_MIN_R_FAST : ST_P2_MIN_R_EXACT);
  constexpr unsigned BOX_BYTES = S.BW * S.BH * 4 + (WAVE ? 2 * CX * CY * 4 : 0);
  static_assert(S.CY % VY == 0, "compute rows must split into row groups");
  static_assert(S.BW <= 256 && S.BH <= 256, "TMA box dims <= 256");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const DevGeom& g = p.g;
  const Items& it = p.it;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + NS;
  float* ring = reinterpret_cast<float*>(smem_raw + 1024);
  float* ibuf = ring + NS * STAGE;   // [F-1][2] planes of levels 1..F-1 (MAINF floats each)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, S.NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // =================== producer: level-0 boxes ==========================
    int slot = 0;
    unsigned use = 0;
    ZigZagCursor cur;
    cur.init(p, 0);
    Work w;
    while (cur.next(p, w)) {
      const int yb = w.col / it.nxb, xb = w.col - yb * it.nxb;
      const int x0 = xb * TX, y0 = yb * TY;
      const int zs = w.z0 - R * F, NP = (w.z1 - w.z0) + 2 * R * F;
      for (int j = 0; j < NP; ++j) {
        if (use > 0) mbar_wait<6>(empty + slot, (use - 1) & 1);
        if (lane == 0) {
          mbar_expect_tx(full + slot, BOX_BYTES);
          tma_load_3d(ring + slot * STAGE, &p.tm.fused, full + slot, g.xo + x0 - HX - XH, g.ry + y0 - HY - R,
                      g.rz + zs + j);
          if constexpr (WAVE) {   // u^{n-1} and m of plane zs + j - R (level 1 of this iteration)
            float* a = ring + slot * STAGE + MAINF;
            tma_load_3d(a, &p.tm.fused_u2, full + slot, g.xo + x0 - HX, g.ry + y0 - HY, g.rz + zs + j - R);
            tma_load_3d(a + MOFF, &p.tm.fused_m, full + slot, g.xo + x0 - HX, g.ry + y0 - HY, g.rz + zs + j - R);
          }
        }
        __syncwarp();
        if (++slot == NS) { slot = 0; ++use; }
      }
    }
    return;
  }

  // =================== consumers ===========================================
  const int cw = warp - 1;
  const bool edge = cw >= NW;
  bool active = true;
  int rg, sx;
  if (!edge) {
    rg = cw;
    sx = XH + HX + 4 * lane;
  } else {
    int e = (cw - NW) * 32 + lane;
    if (e >= 2 * EC * NRG) { active = false; e = 0; }
    const int side = e / (EC > 0 ? EC * NRG : 1);
    const int rem = e - side * EC * NRG;
    rg = rem / (EC > 0 ? EC : 1);
    const int c = rem - rg * EC;
    sx = side == 0 ? XH + 4 * c : XH + HX + TX + 4 * c;
  }
  const int sy = R + rg * VY;
  const int so = sy * BW + sx;   // own first point inside a plane stage
  const int ao = rg * VY * CX + (sx - XH);   // own first point inside a CX x CY aux tile (wave)
  // level j is needed on rows [y0 - R(F-j), y0 + TY + R(F-j)) (row offset
  // within the compute grid: [HY - R(F-j), HY + TY + R(F-j))); the last level
  // only by main warps
  auto need = [&](int j) {
    if (j == F && edge) return false;
    const int lo = HY - R * (F - j), hi = HY + TY + R * (F - j);
    return rg * VY + VY > lo && rg * VY < hi;
  };
  const long long pitch = g.pitch, pstride = g.pstride;

  int ls = 0;          // ring slot of the next level-0 plane (CTA lifetime) ...
  unsigned lp = 0;     // ... and its phase parity
  int ib = 0;          // intermediate plane buffer parity
  float4 win[F][NQ][VY];
#pragma unroll
  for (int j = 0; j < F; ++j)
#pragma unroll
    for (int i = 0; i < NQ; ++i)
#pragma unroll
      for (int v = 0; v < VY; ++v) win[j][i][v] = make_float4(0.f, 0.f, 0.f, 0.f);

  ZigZagCursor cur;
  cur.init(p, 0);
  Work w;
  while (cur.next(p, w)) {
    const int yb = w.col / it.nxb, xb = w.col - yb * it.nxb;
    const int x0 = xb * TX, y0 = yb * TY;
    const int gx = x0 - HX - XH + sx, gy = y0 - HY - R + sy;   // interior coords of own first point
    const int zs = w.z0 - R * F, NP = (w.z1 - w.z0) + 2 * R * F;
    bool allin = gx >= 0 && gx + 4 <= g.nx && gy >= 0 && gy + VY <= g.ny;
    // output: main-warp rows inside [y0, y0 + TY) and the grid, x inside the grid
    const bool xfull = gx + 4 <= g.nx, xany = gx < g.nx;
    bool yok[VY];
#pragma unroll
    for (int v = 0; v < VY; ++v) {
      const int r = rg * VY + v - HY;
      yok[v] = !edge && active && r >= 0 && r < TY && gy + v < g.ny;
    }
    float* op = p.fout + dev_index(g, zs - R * F, gy, gx);   // plane of level F at k = 0
#if ST_CHECKS
    {   // the stores of this item (planes [w.z0, w.z1) of the output rows) stay inside the buffer
      const long long i0 = dev_index(g, w.z0, gy, gx), i1 = dev_index(g, w.z1 - 1, gy + VY - 1, gx + 3);
      const bool store = !edge && active && xany && w.z1 > w.z0 && gy >= 0 && gy < g.ny;
      if (w.z0 < 0 || w.z1 > g.nz || (store && (i0 < 0 || i1 >= g.buf_elems))) watchdog_trip(p, 11, i0, i1, w.col);
    }
#endif
    // wave: level F-1 (the second newest) is an output too, plane zs + k - (F-1)R
    float* op2 = WAVE && F > 1 ? p.fout2 + dev_index(g, zs - R * (F - 1), gy, gx) : nullptr;
    const bool need1 = need(1);
    bool needj[F + 1];
#pragma unroll
    for (int j = 1; j <= F; ++j) needj[j] = need(j);
    (void)need1;

    // One plane iteration (k = plane index within the item, jj = k mod NQ).
    bool ready = false;   // full barrier of plane k already seen complete (early test)
    auto iter = [&](const int k, const int jj) {
      // ring slots advance incrementally (no modulo by the non-power-of-2 NS)
      const bool wrap = ls + 1 == NS;
      const int nls = wrap ? 0 : ls + 1;
      const unsigned nlp = wrap ? lp ^ 1u : lp;
      // 1. newest level-0 plane (zs + k) into the window
      if (!ready) mbar_wait<5>(full + ls, lp);
      {
        const float* st = ring + ls * STAGE + so;
#pragma unroll
        for (int v = 0; v < VY; ++v) win[0][(jj + 2 * R) % NQ][v] = lds4(st + v * BW);
      }
      // peek at the next plane's barrier now; its latency hides behind this plane
      ready = k + 1 < NP && mbar_test(full + nls, nlp);
      if (!WAVE && (k < R || k >= NP - R)) {   // never a centre plane: last use
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + ls);
      }
      // 2. publish the centre planes of levels 1..F-1 (computed R planes ago)
#pragma unroll
      for (int j = 1; j < F; ++j) {
        if (active) {
          float* d = ibuf + ((j - 1) * 2 + ib) * MAINF + so;
#pragma unroll
          for (int v = 0; v < VY; ++v) *reinterpret_cast<float4*>(d + v * BW) = win[j][(jj + R) % NQ][v];
        }
      }
      if constexpr (F > 1) named_bar_sync(1, NCT);
      // 3. levels 1..F
      const int cslot = ls >= R ? ls - R : ls - R + NS;   // plane zs + k - R (level-1 centre)
#pragma unroll
      for (int j = 1; j <= F; ++j) {
        const int P = zs + k - j * R;
        float4 val[VY];
        const bool run = k >= 2 * j * R && needj[j];
        if (run) {
          const float* cs = (j == 1 ? ring + cslot * STAGE : ibuf + ((j - 2) * 2 + ib) * MAINF) + so;
          fused_point<R, VY, BW, FAST>(p, win[j - 1], jj, cs, val);
          if constexpr (WAVE) {
            // u_j = (2 u_{j-1} - u_{j-2}) + m * lap, the reference order
            // (executor wave model): u_{j-2} from the aux tile (j = 1) or the
            // oldest slot of window j-2; m from the aux tile loaded with the
            // plane, (j-1)R iterations ago
            const int d = (j - 1) * R;
            const int mslot = ls >= d ? ls - d : ls - d + NS;
            const float* aw = ring + mslot * STAGE + MAINF + MOFF + ao;
            const float* uw = ring + ls * STAGE + MAINF + ao;
#pragma unroll
            for (int v = 0; v < VY; ++v) {
              const float4 cc = win[j - 1][(jj + R) % NQ][v];
              const float4 w2 = j == 1 ? lds4(uw + v * CX) : win[j >= 2 ? j - 2 : 0][jj % NQ][v];
              const float4 mm = lds4(aw + v * CX);
              const float4 lap = val[v];
              if constexpr (!P2) {
                const float4 b = make_float4(__fsub_rn(__fadd_rn(cc.x, cc.x), w2.x), __fsub_rn(__fadd_rn(cc.y, cc.y), w2.y),
                                             __fsub_rn(__fadd_rn(cc.z, cc.z), w2.z), __fsub_rn(__fadd_rn(cc.w, cc.w), w2.w));
                if constexpr (FAST) {
                  val[v] = make_float4(__fmaf_rn(mm.x, lap.x, b.x), __fmaf_rn(mm.y, lap.y, b.y),
                                       __fmaf_rn(mm.z, lap.z, b.z), __fmaf_rn(mm.w, lap.w, b.w));
                } else {
                  val[v] = make_float4(__fadd_rn(b.x, __fmul_rn(mm.x, lap.x)), __fadd_rn(b.y, __fmul_rn(mm.y, lap.y)),
                                       __fadd_rn(b.z, __fmul_rn(mm.z, lap.z)), __fadd_rn(b.w, __fmul_rn(mm.w, lap.w)));
                }
              } else {
                const float2 b01 = fadd2(cc.x, cc.y, cc.x, cc.y), b23 = fadd2(cc.z, cc.w, cc.z, cc.w);
                const float2 c01 = fsub2(b01.x, b01.y, w2.x, w2.y), c23 = fsub2(b23.x, b23.y, w2.z, w2.w);
                if constexpr (FAST) {
                  const float2 r01 = ffma2v(mm.x, mm.y, lap.x, lap.y, c01.x, c01.y);
                  const float2 r23 = ffma2v(mm.z, mm.w, lap.z, lap.w, c23.x, c23.y);
                  val[v] = make_float4(r01.x, r01.y, r23.x, r23.y);
                } else {
                  const float2 m01 = fmul2v(mm.x, mm.y, lap.x, lap.y, p.nzero);
                  const float2 m23 = fmul2v(mm.z, mm.w, lap.z, lap.w, p.nzero);
                  const float2 r01 = fadd2(c01.x, c01.y, m01.x, m01.y), r23 = fadd2(c23.x, c23.y, m23.x, m23.y);
                  val[v] = make_float4(r01.x, r01.y, r23.x, r23.y);
                }
              }
            }
          }
          fused_halo<VY>(g, val, win[j - 1][(jj + R) % NQ], P, gy, gx, allin);
        }
        if (!WAVE && j == 1 && k >= 2 * R) {   // level-1 centre plane released (planes < R went at load)
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + cslot);
        }
        if constexpr (WAVE && F > 1) {   // level F-1 is the second newest output
          if (j == F - 1 && run && k >= (2 * F - 1) * R && k < NP - R) {
            float* o = op2 + (long long)k * pstride;
#pragma unroll
            for (int v = 0; v < VY; ++v) {
              if (yok[v]) {
                float* ov = o + v * pitch;
                if (xfull) {
                  *reinterpret_cast<float4*>(ov) = val[v];
                } else if (xany) {
                  ov[0] = val[v].x;
                  if (gx + 1 < g.nx) ov[1] = val[v].y;
                  if (gx + 2 < g.nx) ov[2] = val[v].z;
                }
              }
            }
          }
        }
        if (j < F) {
          if (run) {
#pragma unroll
            for (int v = 0; v < VY; ++v) win[j][(jj + 2 * R) % NQ][v] = val[v];
          }
        } else if (run && k >= 2 * R * F) {
          float* o = op + (long long)k * pstride;
#pragma unroll
          for (int v = 0; v < VY; ++v) {
            if (yok[v]) {
              float* ov = o + v * pitch;
              if (xfull) {
                *reinterpret_cast<float4*>(ov) = val[v];
              } else if (xany) {
                ov[0] = val[v].x;
                if (gx + 1 < g.nx) ov[1] = val[v].y;
                if (gx + 2 < g.nx) ov[2] = val[v].z;
              }
            }
          }
        }
      }
      if constexpr (WAVE) {
        // stage of iteration q: main box (centre at q + R) and aux tiles (m of
        // level F at q + (F-1)R) -- released LAG iterations later, the tail of
        // the item at its last iteration
        __syncwarp();
        if (lane == 0) {
          if (k >= LAG) mbar_arrive(empty + (ls >= LAG ? ls - LAG : ls - LAG + NS));
          if (k == NP - 1)
            for (int q = (NP > LAG ? NP - LAG : 0); q < NP; ++q) {
              const int d = k - q;
              mbar_arrive(empty + (ls >= d ? ls - d : ls - d + NS));
            }
        }
      }
      ib ^= 1;
      ls = nls;
      lp = nlp;
    };
    // one unrolled body for every phase: a second, check-free steady-state
    // copy measured slower (instruction-cache misses outweigh the tests)
    for (int kb = 0; kb < NP; kb += NQ) {
#pragma unroll
      for (int jj = 0; jj < NQ; ++jj)
        if (kb + jj < NP) iter(kb + jj, jj);
    }
    ready = false;
  }
}

// Host-side table entry of one compiled shape.
template <int R, int F, int TY, int VY, int PD, int MODEL = 0>
static FusedFn fused_entry(int fast) {
  constexpr FusedShape s = fused_shape(R, F, TY, VY, PD, MODEL);
  static_assert(fused_smem_bytes(R, F, TY, VY, PD, MODEL) <= 227 * 1024, "shared memory budget");
  FusedFn f{};
  f.fn = fast ? (void*)&fused_kernel<R, F, TY, VY, PD, true, MODEL>
              : (void*)&fused_kernel<R, F, TY, VY, PD, false, MODEL>;
  f.threads = fused_threads(R, F, TY, VY, PD, MODEL);
  f.smem = fused_smem_bytes(R, F, TY, VY, PD, MODEL);
  f.ty = TY;
  f.bw = s.BW;
  f.bh = s.BH;
  f.cx = s.CX;
  f.cy = s.CY;
  return f;
}

}  // namespace st
