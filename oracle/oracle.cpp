// oracle.cpp -- CPU restatement of the reference executor (TEST
// INFRASTRUCTURE ONLY: the checker and the CPU baseline, never the product).
// See oracle.h for the reference file:line map.
//
// Build contract (proj/CMakeLists.txt:6-13): -O3 -ffp-contract=off, no
// fast-math, no FTZ/DAZ.  Accumulation is `acc = c1*r1; acc = acc + ck*rk`
// in spec term order in float32 (executor.hpp:92-95).
//
// Loops are explicit compiled loop nests (not an IR interpreter), with the
// integer MIN/MAX bounds of tile_space_minmax / tile_time
// and OpenMP on the loop mark_parallel selects.  The inner
// accumulation runs over a contiguous row segment so it vectorises; the
// per-point operation order is unchanged by that (each point is independent
// within a step), so results are bit-identical to a point-at-a-time loop.

#include "oracle.h"

#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

struct Geo {
  int n = 0;           // reference ndims
  int64_t E[3];        // interior extents, 3D-embedded (leading 1s)
  int R[3];            // radii, 3D-embedded (leading 0s)
  int64_t P[3];        // padded extents
  int64_t plane = 0;   // elements per slot
  int dtd = 1;         // delta_t
};

// Map reference dimension i (0-based) of an n-dim spec to the 3D axis.
inline int axis_of(int n, int i) { return 3 - n + i; }

bool make_geo(const or_spec* s, const int64_t* ext, Geo& g) {
  if (!s || s->ndims < 1 || s->ndims > 3 || s->nterms < 1 || !s->terms)
    return false;
  g.n = s->ndims;
  for (int a = 0; a < 3; ++a) { g.E[a] = 1; g.R[a] = 0; }
  for (int i = 0; i < g.n; ++i) {
    if (ext[i] < 1) return false;
    g.E[axis_of(g.n, i)] = ext[i];
  }
  g.dtd = 0;
  for (int k = 0; k < s->nterms; ++k) {
    const or_term& t = s->terms[k];
    if (t.dt < 1) return false;                      // stencil.hpp:43
    if (s->model == OR_MODEL_WAVE && t.dt != 1) return false;
    g.dtd = std::max(g.dtd, t.dt);
    for (int i = 0; i < g.n; ++i) {
      int a = axis_of(g.n, i);
      g.R[a] = std::max(g.R[a], std::abs(t.off[i]));
    }
  }
  if (s->model == OR_MODEL_WAVE) g.dtd = 2;  // u^{n-1} is read (ledger A.3)
  g.plane = 1;
  for (int a = 0; a < 3; ++a) {
    g.P[a] = g.E[a] + 2 * g.R[a];
    g.plane *= g.P[a];
  }
  return true;
}

inline int64_t row_off(const Geo& g, int64_t z, int64_t y) {
  return ((z + g.R[0]) * g.P[1] + (y + g.R[1])) * g.P[2] + g.R[2];
}

struct Lcg {  // executor.hpp:73-81 recurrence (frozen)
  uint64_t state;
  explicit Lcg(uint64_t s) : state(s) {}
  uint64_t step() {
    state = state * 6364136223846793005ULL + 1442695040888963407ULL;
    return state;
  }
  float next_reference() {
    uint64_t s = step();
    return static_cast<float>(0.001 + 0.001 * (static_cast<double>(s >> 40) /
                                               16777216.0));
  }
  double next_unit_double() {
    uint64_t s = step();
    return static_cast<double>(s >> 40) / 16777216.0;
  }
};

struct Exec {
  Geo g;
  const or_spec* s;
  float* grid;
  int64_t slots;
  const float* m;
  std::vector<float> c;
  std::vector<int> dt;
  std::vector<int64_t> off;  // element offset within a slot

  void setup() {
    for (int k = 0; k < s->nterms; ++k) {
      const or_term& t = s->terms[k];
      int64_t o[3] = {0, 0, 0};
      for (int i = 0; i < g.n; ++i) o[axis_of(g.n, i)] = t.off[i];
      c.push_back(t.coeff);
      dt.push_back(t.dt);
      off.push_back((o[0] * g.P[1] + o[1]) * g.P[2] + o[2]);
    }
  }

  // Update logical points (z, y, x0..x1) of step t.  Step t writes level
  // t + delta_t (executor.hpp:14-16); term k reads level t + delta_t - dt_k.
  inline void row(int64_t t, int64_t z, int64_t y, int64_t x0, int64_t x1) const {
    const int64_t lw = t + g.dtd;
    const int64_t ro = row_off(g, z, y) + x0;
    float* __restrict dst = grid + (lw % slots) * g.plane + ro;
    const int64_t n = x1 - x0;
    const int K = static_cast<int>(c.size());
    if (s->model == OR_MODEL_TERMS) {
      {
        const float* __restrict src =
            grid + ((lw - dt[0]) % slots) * g.plane + ro + off[0];
        const float c0 = c[0];
        for (int64_t i = 0; i < n; ++i) dst[i] = c0 * src[i];
      }
      for (int k = 1; k < K; ++k) {
        const float* __restrict src =
            grid + ((lw - dt[k]) % slots) * g.plane + ro + off[k];
        const float ck = c[k];
        for (int64_t i = 0; i < n; ++i) dst[i] = dst[i] + ck * src[i];
      }
    } else {
      // Wave ledger: lap = sum_k w_k u^n[x+off_k] in
      // spec order; u^{n+1} = (2 u^n - u^{n-1}) + m * lap.
      const float* __restrict u1 = grid + ((lw - 1) % slots) * g.plane + ro;
      const float* __restrict u2 = grid + ((lw - 2) % slots) * g.plane + ro;
      {
        const float c0 = c[0];
        const float* __restrict src = u1 + off[0];
        for (int64_t i = 0; i < n; ++i) dst[i] = c0 * src[i];
      }
      for (int k = 1; k < K; ++k) {
        const float ck = c[k];
        const float* __restrict src = u1 + off[k];
        for (int64_t i = 0; i < n; ++i) dst[i] = dst[i] + ck * src[i];
      }
      const float* __restrict mm = m + (z * g.E[1] + y) * g.E[2] + x0;
      for (int64_t i = 0; i < n; ++i)
        dst[i] = (2.0f * u1[i] - u2[i]) + mm[i] * dst[i];
    }
  }

  // Execute the box lo..hi (skewed coordinates; logical = skewed - sh) of
  // step t.  The loop over axis pa (the mark_parallel loop) is distributed
  // over the OpenMP team (orphaned `omp for`, implicit barrier) or, with
  // rev, iterated in reverse.  Must be called by every team thread.
  void box(int64_t t, const int64_t lo[3], const int64_t hi[3],
           const int64_t sh[3], int pa, bool rev, bool par) const {
    for (int a = 0; a < 3; ++a)
      if (lo[a] >= hi[a]) return;
    auto body = [&](int64_t z, int64_t y, int64_t xa, int64_t xb) {
      row(t, z - sh[0], y - sh[1], xa - sh[2], xb - sh[2]);
    };
    if (pa == 0) {
      if (rev) {
        for (int64_t z = hi[0] - 1; z >= lo[0]; --z)
          for (int64_t y = lo[1]; y < hi[1]; ++y) body(z, y, lo[2], hi[2]);
      } else if (par) {
#pragma omp for schedule(static)
        for (int64_t z = lo[0]; z < hi[0]; ++z)
          for (int64_t y = lo[1]; y < hi[1]; ++y) body(z, y, lo[2], hi[2]);
      } else {
        for (int64_t z = lo[0]; z < hi[0]; ++z)
          for (int64_t y = lo[1]; y < hi[1]; ++y) body(z, y, lo[2], hi[2]);
      }
    } else if (pa == 1) {  // 2D: rows are the outermost real loop
      for (int64_t z = lo[0]; z < hi[0]; ++z) {
        if (rev) {
          for (int64_t y = hi[1] - 1; y >= lo[1]; --y) body(z, y, lo[2], hi[2]);
        } else if (par) {
#pragma omp for schedule(static)
          for (int64_t y = lo[1]; y < hi[1]; ++y) body(z, y, lo[2], hi[2]);
        } else {
          for (int64_t y = lo[1]; y < hi[1]; ++y) body(z, y, lo[2], hi[2]);
        }
      }
    } else {  // 1D: the x loop itself is parallel
      for (int64_t z = lo[0]; z < hi[0]; ++z)
        for (int64_t y = lo[1]; y < hi[1]; ++y) {
          if (rev) {
            for (int64_t x = hi[2] - 1; x >= lo[2]; --x) body(z, y, x, x + 1);
          } else if (par) {
            const int64_t CH = 256;
            const int64_t nch = (hi[2] - lo[2] + CH - 1) / CH;
#pragma omp for schedule(static)
            for (int64_t j = 0; j < nch; ++j) {
              int64_t xa = lo[2] + j * CH;
              body(z, y, xa, std::min(hi[2], xa + CH));
            }
          } else {
            body(z, y, lo[2], hi[2]);
          }
        }
    }
  }
};

}  // namespace

extern "C" {

int or_validate(const or_spec* s) {
  Geo g;
  int64_t ext[3] = {1, 1, 1};
  return make_geo(s, ext, g) ? OR_OK : OR_EINVAL;
}

int or_time_depth(const or_spec* s) {
  Geo g;
  int64_t ext[3] = {1, 1, 1};
  return make_geo(s, ext, g) ? g.dtd : -1;
}

int or_radius(const or_spec* s, int dim) {
  Geo g;
  int64_t ext[3] = {1, 1, 1};
  if (!make_geo(s, ext, g) || dim < 0 || dim >= s->ndims) return -1;
  return g.R[axis_of(g.n, dim)];
}

int64_t or_flops_per_point(const or_spec* s) {
  // stencil.hpp:107-108: k multiplies + (k-1) adds.  Wave ledger adds
  // 2u (1), -u^{n-1} (1), m*lap (1), + (1).
  if (!s || s->nterms < 1) return -1;
  int64_t f = 2LL * s->nterms - 1;
  if (s->model == OR_MODEL_WAVE) f += 4;
  return f;
}

int64_t or_plane(const or_spec* s, const int64_t* extents) {
  Geo g;
  if (!make_geo(s, extents, g)) return -1;
  return g.plane;
}

void or_lcg_reference(uint64_t seed, int64_t n, float* out) {
  Lcg l(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = l.next_reference();
}

void or_init_reference(const or_spec* s, const int64_t* extents, float* grid,
                       int64_t slots, uint64_t seed) {
  // executor.hpp:87-90: levels [0, delta_t) filled, halo included, from the
  // LCG stream in level-major, row-major order; remaining slots zero.
  Geo g;
  if (!make_geo(s, extents, g)) return;
  std::memset(grid, 0, sizeof(float) * slots * g.plane);
  Lcg l(seed);
  for (int lv = 0; lv < g.dtd; ++lv) {
    float* p = grid + (lv % slots) * g.plane;
    for (int64_t i = 0; i < g.plane; ++i) p[i] = l.next_reference();
  }
}

void or_init_unit(const or_spec* s, const int64_t* extents, float* grid,
                  int64_t slots, uint64_t seed) {
  // Ledger A.4: zero halo; interior of levels [0, delta_t) from the same
  // LCG recurrence with value (s>>40)/2^24 in [0,1), level-major, row-major.
  Geo g;
  if (!make_geo(s, extents, g)) return;
  std::memset(grid, 0, sizeof(float) * slots * g.plane);
  Lcg l(seed);
  for (int lv = 0; lv < g.dtd; ++lv) {
    float* p = grid + (lv % slots) * g.plane;
    for (int64_t z = 0; z < g.E[0]; ++z)
      for (int64_t y = 0; y < g.E[1]; ++y) {
        float* r = p + row_off(g, z, y);
        for (int64_t x = 0; x < g.E[2]; ++x)
          r[x] = static_cast<float>(l.next_unit_double());
      }
  }
}

void or_init_gaussian(const or_spec* s, const int64_t* extents, float* grid,
                      int64_t slots, double sigma, const int64_t* centre) {
  // Ledger A.5: u = exp(-|x-c|^2 / (2 sigma^2)) in double, cast once;
  // identical levels [0, delta_t); zero halo.
  Geo g;
  if (!make_geo(s, extents, g)) return;
  std::memset(grid, 0, sizeof(float) * slots * g.plane);
  int64_t c3[3] = {0, 0, 0};
  for (int i = 0; i < g.n; ++i) c3[axis_of(g.n, i)] = centre[i];
  const double inv = 1.0 / (2.0 * sigma * sigma);
  for (int lv = 0; lv < g.dtd; ++lv) {
    float* p = grid + (lv % slots) * g.plane;
    for (int64_t z = 0; z < g.E[0]; ++z)
      for (int64_t y = 0; y < g.E[1]; ++y) {
        float* r = p + row_off(g, z, y);
        for (int64_t x = 0; x < g.E[2]; ++x) {
          double dz = double(z - c3[0]), dy = double(y - c3[1]),
                 dx = double(x - c3[2]);
          r[x] = static_cast<float>(std::exp(-(dz * dz + dy * dy + dx * dx) * inv));
        }
      }
  }
}

void or_mfield_layered(int ndims, const int64_t* extents, float* m,
                       double v_top, double v_bottom, int64_t split, double dt,
                       double h) {
  // m = (c dt / h)^2 in double, cast once (ledger A.3); c = v_top for
  // d_1 < split, else v_bottom.
  int64_t inner = 1;
  for (int i = 1; i < ndims; ++i) inner *= extents[i];
  for (int64_t z = 0; z < extents[0]; ++z) {
    double v = z < split ? v_top : v_bottom;
    double q = v * dt / h;
    float mv = static_cast<float>(q * q);
    for (int64_t i = 0; i < inner; ++i) m[z * inner + i] = mv;
  }
}

void or_mfield_random_smoothed(int ndims, const int64_t* extents, float* m,
                               uint64_t seed, double vmin, double vmax,
                               double dt, double h) {
  // Config 4: v = LCG U[vmin, vmax] (row-major interior), then a 3^n box
  // filter clamped to the edge, all in double; m = (v dt / h)^2 cast once.
  int64_t E[3] = {1, 1, 1};
  for (int i = 0; i < ndims; ++i) E[3 - ndims + i] = extents[i];
  const int64_t N = E[0] * E[1] * E[2];
  std::vector<double> v(N);
  Lcg l(seed);
  for (int64_t i = 0; i < N; ++i) v[i] = vmin + (vmax - vmin) * l.next_unit_double();
  const int rz = E[0] > 1 ? 1 : 0, ry = E[1] > 1 ? 1 : 0, rx = E[2] > 1 ? 1 : 0;
  const double cnt = double((2 * rz + 1) * (2 * ry + 1) * (2 * rx + 1));
  for (int64_t z = 0; z < E[0]; ++z)
    for (int64_t y = 0; y < E[1]; ++y)
      for (int64_t x = 0; x < E[2]; ++x) {
        double acc = 0.0;
        for (int dz = -rz; dz <= rz; ++dz)
          for (int dy = -ry; dy <= ry; ++dy)
            for (int dx = -rx; dx <= rx; ++dx) {
              int64_t zz = std::clamp<int64_t>(z + dz, 0, E[0] - 1);
              int64_t yy = std::clamp<int64_t>(y + dy, 0, E[1] - 1);
              int64_t xx = std::clamp<int64_t>(x + dx, 0, E[2] - 1);
              acc += v[(zz * E[1] + yy) * E[2] + xx];
            }
        double vs = acc / cnt;
        double q = vs * dt / h;
        m[(z * E[1] + y) * E[2] + x] = static_cast<float>(q * q);
      }
}

int or_check_legality(const or_spec* s, int skew, int* required_min) {
  // transforms.hpp:43-51: legal iff skew >= max_i delta_i.
  int rmin = 0;
  for (int i = 0; i < s->ndims; ++i) rmin = std::max(rmin, or_radius(s, i));
  if (required_min) *required_min = rmin;
  return skew >= rmin ? 0 : rmin;
}

int or_execute(const or_spec* s, const int64_t* extents, float* grid,
               int64_t slots, int64_t t_begin, int64_t t_end,
               const float* mfield, int schedule, int skew, int64_t time_tile,
               const int64_t* tiles, int reverse_parallel, int nthreads,
               double* wall_seconds, int64_t* points_updated) {
  Exec ex;
  ex.s = s;
  if (!make_geo(s, extents, ex.g)) return OR_EINVAL;
  if (t_begin < 0 || t_end < t_begin) return OR_EINVAL;
  if (s->model == OR_MODEL_WAVE && !mfield) return OR_EINVAL;
  ex.grid = grid;
  ex.slots = slots;
  ex.m = mfield;
  ex.setup();
  const Geo& g = ex.g;
  const int n = g.n;
  const int pa = axis_of(n, 0);  // outermost real spatial axis
  const int64_t Dt = t_end - t_begin;

  int64_t tl[3] = {1, 1, 1};
  if (schedule != OR_SCHED_CANONICAL) {
    if (!tiles) return OR_EINVAL;
    for (int i = 0; i < n; ++i) {
      if (tiles[i] < 1) return OR_EINVAL;
      tl[axis_of(n, i)] = tiles[i];
    }
  }
  // required_slots (executor.hpp:83-85)
  int64_t need = g.dtd + 1;
  if (schedule == OR_SCHED_TIME) {
    if (time_tile < 1) return OR_EINVAL;
    int rmin = 0;
    if (or_check_legality(s, skew, &rmin) != 0) return OR_EILLEGAL;
    need = g.dtd + time_tile;
  }
  if (slots < need) return OR_ESLOTS;

  const bool rev = reverse_parallel != 0;
  int nt = rev ? 1 : std::max(1, nthreads);
  auto t0 = std::chrono::steady_clock::now();

#pragma omp parallel num_threads(nt) if (nt > 1)
  {
    const bool par = nt > 1;
    const int64_t zero[3] = {0, 0, 0};
    if (schedule == OR_SCHED_CANONICAL) {
      // loop_ir.hpp:111-114: t outer, spatial loops in declaration order;
      // mark_parallel: the outermost spatial loop is parallel.
      const int64_t lo[3] = {0, 0, 0};
      const int64_t hi[3] = {g.E[0], g.E[1], g.E[2]};
      for (int64_t t = t_begin; t < t_end; ++t)
        ex.box(t, lo, hi, zero, pa, rev, par);
    } else if (schedule == OR_SCHED_SPACE) {
      // tile_space_minmax: t, x1_blk..xn_blk (parallel),
      // x_i in [max(0, blk), min(D_i, blk + t_i)).
      int64_t nb[3];
      for (int a = 0; a < 3; ++a) nb[a] = (g.E[a] + tl[a] - 1) / tl[a];
      const int64_t ntile = nb[0] * nb[1] * nb[2];
      for (int64_t t = t_begin; t < t_end; ++t) {
        auto tile_body = [&](int64_t f) {
          int64_t b[3] = {f / (nb[1] * nb[2]), (f / nb[2]) % nb[1], f % nb[2]};
          int64_t lo[3], hi[3];
          for (int a = 0; a < 3; ++a) {
            int64_t blk = b[a] * tl[a];
            lo[a] = std::max<int64_t>(0, blk);
            hi[a] = std::min<int64_t>(g.E[a], blk + tl[a]);
          }
          ex.box(t, lo, hi, zero, -1, false, false);
        };
        if (rev) {
          for (int64_t f = ntile - 1; f >= 0; --f) tile_body(f);
        } else if (par) {
#pragma omp for schedule(dynamic, 1)
          for (int64_t f = 0; f < ntile; ++f) tile_body(f);
        } else {
          for (int64_t f = 0; f < ntile; ++f) tile_body(f);
        }
      }
    } else if (schedule == OR_SCHED_REMAINDER) {
      // tile_space_remainder + execute_group (transforms.hpp:35-41,
      // executor.hpp:100-105): 2^n nests main-first (bitmask, dim 1 = low
      // bit), time-step interleaved.  main_i = D_i - D_i mod t_i.
      int64_t mainx[3];
      for (int a = 0; a < 3; ++a) mainx[a] = g.E[a] - g.E[a] % tl[a];
      for (int64_t t = t_begin; t < t_end; ++t) {
        for (int mask = 0; mask < (1 << n); ++mask) {
          int64_t rlo[3], rhi[3], step[3];
          for (int a = 0; a < 3; ++a) { rlo[a] = 0; rhi[a] = g.E[a]; step[a] = g.E[a]; }
          for (int i = 0; i < n; ++i) {
            int a = axis_of(n, i);
            if (mask & (1 << i)) { rlo[a] = mainx[a]; rhi[a] = g.E[a]; step[a] = g.E[a]; }
            else { rlo[a] = 0; rhi[a] = mainx[a]; step[a] = tl[a]; }
          }
          int64_t nb[3];
          for (int a = 0; a < 3; ++a)
            nb[a] = rhi[a] > rlo[a] ? (rhi[a] - rlo[a] + step[a] - 1) / step[a] : 0;
          const int64_t ntile = nb[0] * nb[1] * nb[2];
          auto tile_body = [&](int64_t f) {
            int64_t b[3] = {f / (nb[1] * nb[2]), (f / nb[2]) % nb[1], f % nb[2]};
            int64_t lo[3], hi[3];
            for (int a = 0; a < 3; ++a) {
              lo[a] = rlo[a] + b[a] * step[a];
              hi[a] = std::min(rhi[a], lo[a] + step[a]);
            }
            ex.box(t, lo, hi, zero, -1, false, false);
          };
          if (rev) {
            for (int64_t f = ntile - 1; f >= 0; --f) tile_body(f);
          } else if (par) {
#pragma omp for schedule(dynamic, 1)
            for (int64_t f = 0; f < ntile; ++f) tile_body(f);
          } else {
            for (int64_t f = 0; f < ntile; ++f) tile_body(f);
          }
        }
      }
    } else {
      // tile_time: t_blk in [0, D_t) step t_t;
      // xi_blk in [0, D_i + s*D_t) step t_i (sequential);
      // t in [max(0, t_blk), min(D_t, t_blk + t_t));
      // xi in [max(s*t, xi_blk), min(D_i + s*t, xi_blk + t_i)), body at xi - s*t;
      // the outermost incremental spatial loop is parallel.
      const int64_t sk = skew;
      int64_t nb[3];
      for (int a = 0; a < 3; ++a) {
        bool real = a >= 3 - n;
        nb[a] = real ? (g.E[a] + sk * Dt + tl[a] - 1) / tl[a] : 1;
      }
      for (int64_t tb = 0; tb < Dt; tb += time_tile) {
        for (int64_t b0 = 0; b0 < nb[0]; ++b0)
          for (int64_t b1 = 0; b1 < nb[1]; ++b1)
            for (int64_t b2 = 0; b2 < nb[2]; ++b2) {
              const int64_t b[3] = {b0, b1, b2};
              const int64_t te = std::min(Dt, tb + time_tile);
              for (int64_t tt = std::max<int64_t>(0, tb); tt < te; ++tt) {
                int64_t lo[3], hi[3], sh[3];
                for (int a = 0; a < 3; ++a) {
                  bool real = a >= 3 - n;
                  if (real) {
                    int64_t blk = b[a] * tl[a];
                    lo[a] = std::max(sk * tt, blk);
                    hi[a] = std::min(g.E[a] + sk * tt, blk + tl[a]);
                    sh[a] = sk * tt;
                  } else {
                    lo[a] = 0; hi[a] = 1; sh[a] = 0;
                  }
                }
                ex.box(t_begin + tt, lo, hi, sh, pa, rev, par);
              }
            }
      }
    }
  }
  auto t1 = std::chrono::steady_clock::now();
  if (wall_seconds) *wall_seconds = std::chrono::duration<double>(t1 - t0).count();
  if (points_updated) *points_updated = Dt * g.E[0] * g.E[1] * g.E[2];
  return OR_OK;
}

static int level_range(const Geo& g, int64_t slots_a, int64_t slots_b,
                       int64_t last_level, int64_t compare_levels) {
  if (compare_levels < 1) return -1;
  if (compare_levels > slots_a || compare_levels > slots_b) return -2;  // not retained
  if (last_level - compare_levels + 1 < 0) return -2;
  (void)g;
  return 0;
}

int or_verify_bitwise(const or_spec* s, const int64_t* extents, const float* a,
                      int64_t slots_a, const float* b, int64_t slots_b,
                      int64_t last_level, int64_t compare_levels) {
  Geo g;
  if (!make_geo(s, extents, g)) return -1;
  int rc = level_range(g, slots_a, slots_b, last_level, compare_levels);
  if (rc) return rc;
  for (int64_t lv = last_level - compare_levels + 1; lv <= last_level; ++lv) {
    const float* pa = a + (lv % slots_a) * g.plane;
    const float* pb = b + (lv % slots_b) * g.plane;
    for (int64_t z = 0; z < g.E[0]; ++z)
      for (int64_t y = 0; y < g.E[1]; ++y) {
        int64_t o = row_off(g, z, y);
        if (std::memcmp(pa + o, pb + o, sizeof(float) * g.E[2]) != 0) return 0;
      }
  }
  return 1;
}

double or_max_rel_err(const or_spec* s, const int64_t* extents, const float* a,
                      int64_t slots_a, const float* b, int64_t slots_b,
                      int64_t last_level, int64_t compare_levels) {
  Geo g;
  if (!make_geo(s, extents, g)) return -1.0;
  if (level_range(g, slots_a, slots_b, last_level, compare_levels)) return -1.0;
  double maxa = 0.0, maxd = 0.0;
  for (int64_t lv = last_level - compare_levels + 1; lv <= last_level; ++lv) {
    const float* pa = a + (lv % slots_a) * g.plane;
    const float* pb = b + (lv % slots_b) * g.plane;
    for (int64_t z = 0; z < g.E[0]; ++z)
      for (int64_t y = 0; y < g.E[1]; ++y) {
        int64_t o = row_off(g, z, y);
        for (int64_t x = 0; x < g.E[2]; ++x) {
          double va = pa[o + x], vb = pb[o + x];
          if (!(std::fabs(va) <= maxa)) maxa = std::fabs(va);
          double d = std::fabs(va - vb);
          if (!(d <= maxd)) maxd = d;  // NaN propagates as +inf below
          if (std::isnan(d)) return INFINITY;
        }
      }
  }
  if (maxa == 0.0) return maxd == 0.0 ? 0.0 : INFINITY;
  return maxd / maxa;
}

}  // extern "C"
