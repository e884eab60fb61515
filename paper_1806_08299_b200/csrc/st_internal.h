// st_internal.h -- structures shared by the host layer (st_host.cpp) and the
// sm_100a kernels (st_kernels_*.cu).  Not part of the public ABI.
#pragma once

#include <cuda.h>  // CUtensorMap

#include <cstdint>

#ifdef __CUDACC__
#define ST_HD __host__ __device__
#else
#define ST_HD
#endif

namespace st {

// Device axes: z = streaming axis (reference d_1 for n >= 2), y, x
// (contiguous).  n = 3: (d1, d2, d3) -> (z, y, x); n = 2: d1 -> z,
// d2 -> x, y dummy; n = 1: d1 -> x, z and y dummy.
struct DevGeom {
  int nz, ny, nx;        // interior extents
  int rz, ry, rx;        // halo widths (= radii)
  int xo;                // column of interior x = 0 inside a row (>= rx, %4==0)
  int pad_;
  long long pitch;       // floats per row (multiple of 32 -> 128 B rows)
  long long pstride;     // floats per plane = (ny + 2 ry) * pitch
  long long base;        // element offset of interior (0, 0, 0)
  long long buf_elems;   // allocation per level buffer (incl. slack)
};

ST_HD inline long long dev_index(const DevGeom& g, long long z,
                                               long long y, long long x) {
  return g.base + z * g.pstride + y * g.pitch + x;
}

constexpr int kMaxBuffers = 8;
constexpr int kMaxGenTerms = 128;
constexpr int kMaxStarCoef = 1 + 6 * 8;
constexpr int kMaxZrLevels = 64;   // levels per wavefront launch with z-slab ranges

struct GenTerm {
  float c;
  int dt;
  long long off;  // device element offset (same for every level buffer)
};

// Item decomposition of one level: (chunk, y-tile, x-tile) columns, chunk-
// major.  A chunk is a run of cz planes along z streamed by one CTA.
// Work decomposition.  A column is one (TY x TX) tile of the x/y plane; an
// item is a run of planes of one column.
//  * sweep (one launch per level): CTA b streams the column-planes
//    [b*W/G, (b+1)*W/G) of W = ncol * nz (balanced, no tail wave);
//  * wavefront: skewed chunks -- chunk c of a level with index lt inside its
//    time tile covers planes [c*cz - s*lt, (c+1)*cz - s*lt) (tile_time,
//    transforms.hpp:53-59) -- and, as tile_time tiles every
//    spatial dimension, y-chunks of cy tiles skewed by one tile per level
//    (tiles are >= the radius tall) or, with ysk > 0, y-bands whose tile grid
//    shifts by ysk rows per level (the L2 time tile: a band's T levels chase
//    one another along z a few planes apart, so level L+1 reads what level L
//    just wrote from L2, and only ~4r rows per band and level come back from
//    HBM instead of a tile's worth).  Tickets are ordered (time tile,
//    z-chunk, y-chunk, level-in-tile, column-in-chunk): a topological order
//    of the dependences because the skews are >= the radii.
struct Items {
  int cz, ty, tx;        // chunk planes (wavefront), tile rows, tile columns
  int nyb, nxb, ncol;    // column grid
  int nch;               // z-chunks per level (wavefront)
  int cy;                // y-tiles per y-chunk (wavefront; skewed 1 tile/level)
  int nyc;               // y-chunks per level
  int ysk;               // > 0: y-bands skewed by ysk ROWS per level (the tile grid of the level with
                         // index lt in its time tile is shifted to rows yb*ty - ysk*lt; r <= ysk,
                         // 2*ysk + r <= ty); 0: y-chunks skewed by one tile per level
  long long ntickets;    // wavefront tickets
};

// TMA tensor maps (cp.async.bulk.tensor) of the level buffers and the m
// field: `main` boxes are one plane of a tile with its x/y halo, `aux`
// boxes one plane of a tile without halo (wave u^{n-1} and m operands).
struct alignas(64) TmaMaps {
  CUtensorMap main[kMaxBuffers > 4 ? 4 : kMaxBuffers];
  CUtensorMap aux[4];
  CUtensorMap mfield;
  CUtensorMap fused;   // fused-level kernel: level-0 box of the input buffer
  CUtensorMap fused_u2;  // ... wave: u^{n-1} compute-grid tile of the second input level
  CUtensorMap fused_m;   // ... wave: m compute-grid tile
  CUtensorMap mcodes;  // palettized m field: 1-byte codes, box TX x TY
};

// Shared-memory pipeline shape of the star kernel.
struct Pipe {
  int ns;            // main ring depth (planes with halo)
  int nsa;           // aux ring depth (wave operands)
  int sw;            // smem row stride of a main stage (floats, %4 == 0)
  int stage_floats;  // floats per main stage (128-B multiple)
  int aux_floats;    // floats per aux stage (u^{n-1} tile + m tile)
  int unit;          // progress-counter units per completed plane
  int main_bytes;    // TMA bytes per main stage
  int aux_bytes;     // TMA bytes per aux stage
};

// Compile-time shape of the star kernel for (R, DIMS, MODEL): a consumer
// thread owns VX = 4 consecutive x (one LDS.128 / STG.128) of VY rows; NC
// consumer warps stack in y (3D) -- tile TX x TY = 128 x NC*VY.  The plane
// ring holds RZ + 1 + PD stages of (TY + 2RY) x SW floats (TMA boxes with an
// x halo of XH = round_up(R, 4) so box starts stay 16-B aligned); the wave
// operand ring PD + 2 stages of 2 x TX x TY floats.  MINB CTAs per SM.
struct StarShape {
  int VX, VY, NC, TX, TY, XH, SW, SH, PD, NS, NSA, STAGE, AUX, MINB;
  int MCO;   // wave operand stage sized for 1-byte m codes only (needs a palettized m field)
};

ST_HD constexpr int round_up_c(int a, int b) { return (a + b - 1) / b * b; }

ST_HD constexpr StarShape star_shape(int R, int DIMS, int MODEL, int V = 0) {
  const int RZ = DIMS >= 2 ? R : 0, RY = DIMS == 3 ? R : 0;
  StarShape s{};
  s.VX = 4;
  s.VY = DIMS == 3 ? (R >= 8 ? 1 : 2) : 1;
  s.NC = DIMS == 3 ? 8 : 1;
  if (DIMS != 3) {
    s.PD = 8;
    s.MINB = 8;
  } else if (MODEL == 0) {
    s.PD = R <= 1 ? 8 : (R == 2 ? 6 : (R == 4 ? 3 : 4));
    s.MINB = R <= 2 ? 2 : 1;
  } else {
    s.PD = R <= 1 ? 2 : 3;
    s.MINB = R <= 1 ? 2 : 1;
  }
  // experimental variants (V > 0) for shape tuning
  // tile-height variants (selected by the plan's d_2 space tile)
  if (DIMS == 3 && V == 1) { s.NC = 16; s.VY = 2; s.MINB = 1; s.PD = MODEL == 0 ? 8 : 1; }
  if (DIMS == 3 && V == 2) { s.NC = 8; s.VY = 1; s.MINB = 2; s.PD = MODEL == 0 ? 12 : 3; }
  if (DIMS == 3 && V == 3) { s.NC = 8; s.VY = 2; s.MINB = 1; s.PD = MODEL == 0 ? 14 : 4; }
  if (DIMS == 3 && V == 4) { s.NC = 8; s.VY = 4; s.MINB = 1; s.PD = MODEL == 0 ? 8 : 1; }   // 32 rows, 10 warps
  if (DIMS == 3 && V == 5) { s.NC = 4; s.VY = 4; s.MINB = 2; s.PD = MODEL == 0 ? 6 : 1; }   // 16 rows, 2 CTAs/SM
  // 16 rows as 16 warps x 1 row, 1 CTA/SM: the phase loop unrolled by the
  // window depth (register renaming instead of window moves, st_kernels.cuh)
  if (DIMS == 3 && V == 6) { s.NC = 16; s.VY = 1; s.MINB = 1; s.PD = 4; }
  // 12 rows as 12 warps x 1 row, 1 CTA/SM (radius 8: 50% more warps than the
  // 8-row shape within the shared memory of an 11-stage ring; config 4:
  // 203 -> 250 GPts/s FAST, 195 -> 223 bit-exact.  14 rows (PD 1): 214;
  // 10 rows: 231)
  if (DIMS == 3 && V == 7) { s.NC = 12; s.VY = 1; s.MINB = 1; s.PD = 2; }
  // 24 rows as 12 warps x 2 rows, 1 CTA/SM (radius 4): three consumer warps per
  // scheduler instead of two, at the 128 registers the per-scheduler file allows
  if (DIMS == 3 && V == 8) { s.NC = 12; s.VY = 2; s.MINB = 1; s.PD = MODEL == 0 ? 4 : 2; }
  // ... with the wave operand stage sized for m as 1-byte codes: a 3-plane prefetch in the same
  // shared memory (config 3: 397 -> 407 GPts/s, config 5: 405 -> 423; the prefetch depth matters:
  // 1 plane 330 / 335; 14 warps x 2 rows (28 rows) only fits 2 planes: 387 / 403)
  if (DIMS == 3 && V == 11) { s.NC = 12; s.VY = 2; s.MINB = 1; s.PD = MODEL == 0 ? 4 : 3; s.MCO = 1; }
  s.TX = 32 * s.VX;
  s.TY = s.NC * s.VY;
  s.XH = round_up_c(R, 4);
  s.SW = s.TX + 2 * s.XH;
  s.SH = s.TY + 2 * RY;
  s.STAGE = round_up_c(s.SW * s.SH, 32);
  s.AUX = MODEL == 1 ? round_up_c(s.MCO ? s.TX * s.TY + s.TX * s.TY / 4 : 2 * s.TX * s.TY, 32) : 0;
  s.NS = RZ + 1 + s.PD;
  s.NSA = MODEL == 1 ? s.PD + 2 : 0;
  // keep every shape inside the opt-in shared memory (227 KB, minus ~4 KB of
  // static queues / palette): shallower prefetch for the big-halo shapes
  // (e.g. r = 4 heat on the 32-row tile)
  while (s.PD > 1 && 1024 + (s.NS * s.STAGE + s.NSA * s.AUX) * 4 > 223 * 1024) {
    --s.PD;
    s.NS = RZ + 1 + s.PD;
    s.NSA = MODEL == 1 ? s.PD + 2 : 0;
  }
  return s;
}

ST_HD constexpr int star_smem_bytes(const StarShape& s) { return 1024 + (s.NS * s.STAGE + s.NSA * s.AUX) * 4; }

struct KParams {
  TmaMaps tm;
  DevGeom g;
  Items it;
  float* buf[kMaxBuffers];   // level L lives in buf[L % nbuf]
  const float* fin;          // fused-level pass: input level buffer
  float* fout;               // fused-level pass: output (last level) buffer
  float* fout2;              // fused-level pass, wave: output of the second newest level
  float* xch0;               // SM-resident 2-D kernel: epoch exchange buffers
  float* xch1;
  int nbuf;
  int dtd;                   // delta_t
  const float* mfield;       // wave coefficient field (device layout) or null
  const float* mpal;         // palette of the m field (<= 256 floats) when mcode_on
  int mcode_on;              // 1: the star kernel reads m as 1-byte codes (tm.mcodes)
  int npal;
  const float* bank;         // per-slot halo bank (device layout) or null
  long long bank_slots;      // reference slot count S (bank has S buffers)
  long long level0;          // absolute level written by relative level 0
  int nsteps;                // relative levels [0, nsteps)
  int T;                     // wavefront: levels in flight (time tile)
  int skew;                  // wavefront lag along z (>= rz)
  int zlo, zhi;              // sweep: interior planes [zlo, zhi) computed (z-slab ghosts)
  int sleep_pub;             // wavefront back-off caps (ns): publisher,
  int ctr_shift;             // progress counter i lives at prog[i << ctr_shift] (own L2 line)
  int rgx;                   // SM-resident 2-D kernel: column tiles (CTA = (b % rgx, b / rgx))
  unsigned* prog;            // [nsteps][nch][ncol] planes completed per item
  unsigned* ticket;          // work counter
  long long* dbg;            // zero-copy host diagnostics (watchdog), may be null
  int zr_on;                 // wavefront over z-slab ranges: level l computes [zr_lo[l], zr_hi[l])
  int zr_lo[kMaxZrLevels], zr_hi[kMaxZrLevels];
  float coef[kMaxStarCoef];  // star coefficients, canonical order
  float nzero;               // -0.0f: addend of the bit-exact paired products (st_kernels.cuh)
  int nterms;
  int sleep_dep;             // ... and producer dependency polls
  int pad3_;
  Pipe pipe;
  GenTerm terms[kMaxGenTerms];
};

enum Model { kTerms = 0, kWave = 1 };

// Launch interface implemented in the .cu files.
struct LaunchCfg {
  int star;      // 1 = star kernel, 0 = generic
  int R;         // star radius
  int dims;      // 1..3
  int model;     // Model
  int fast;      // 0/1
  int wf;        // 1 = persistent wavefront kernel
  int bx, byt;   // block shape (star: consumer tile TX x BYT; +1 producer warp)
  int grid;      // persistent CTAs
  int smem;      // dynamic shared memory bytes
  int variant;   // star shape variant (0 = default)
};

// Returns 0 on success, else a CUDA error code; `launches` incremented.
int launch_sweep(const LaunchCfg& lc, const KParams& p, int rel_level,
                 void* stream);
int launch_wavefront(const LaunchCfg& lc, const KParams& p, void* stream);
// Persistent level-pipelined sweep (cooperative launch: all CTAs resident).
int launch_pipe(const LaunchCfg& lc, const KParams& p, void* stream);
// Occupancy-derived persistent grid size, or <0 on error.
int wavefront_grid(const LaunchCfg& lc, int sm_count);
// Compile-time variant lookup: is (star, R, dims) built?
bool star_supported(int R, int dims);
// Layout conversion kernels.
int launch_ref_to_dev(const float* ref, float* dev, const DevGeom& g, int n,
                      const long long* ref_padded, void* stream);
int launch_dev_to_ref(const float* dev, float* ref, const DevGeom& g, int n,
                      const long long* ref_padded, void* stream);
// padded planes [z0, z1) between the reference layout (in/out at offset 0 =
// padded plane 0) and a device level buffer, with a small grid of `ctas`;
// halo_only (to_dev): only the halo cells of those planes
int launch_rows(bool to_dev, const float* in, float* out, const DevGeom& g, long long z0, long long z1, int ctas,
                void* stream, bool halo_only = false);
// Fused-level (on-chip time tile) kernels: F levels per pass, TY output
// rows.  Fills threads / smem / compile-time box (bw, bh) of the variant;
// returns the kernel or null when (R, F, TY) is not built.
struct FusedFn {
  void* fn;
  int threads, smem, ty, bw, bh, cx, cy;
};
FusedFn fused_lookup(int R, int F, int ty, int fast, int model = 0);
int launch_fused(const FusedFn& f, const KParams& p, int grid, void* stream);
// SM-resident 2-D time tiling (st_resident.cuh): one cooperative launch of
// `grid` CTAs (one per SM) with `smem` bytes each; null/err if R not built.
int launch_resident2d(int R, int fast, const KParams& p, int grid, int smem, void* stream);
bool resident2d_supported(int R);
int fused_grid(const FusedFn& f, int sm_count);
// Palettize a device interior m field: on success *npal in [1, 256] and the
// codes (device layout) / palette are written; *npal = 0 when the field has
// more than 256 distinct values.  Returns a CUDA error code.
int build_palette(const float* m_interior, const DevGeom& g, unsigned char* codes, float* pal_dev, float* pal_host,
                  int* npal, void* stream);
int launch_interior_to_dev(const float* interior, float* dev, const DevGeom& g,
                           void* stream);

}  // namespace st
