// st_host.cpp -- host side of the C-ABI: stencil model, plans, device grids,
// layout conversion, kernel selection and launch.  The compute itself is in
// the sm_100a kernels (st_kernels.cuh); there is no CPU compute path here --
// a grid that cannot be run on the device fails with an error.
#include <cuda.h>
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <list>
#include <unordered_map>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "st_internal.h"
#include "stencil_tiler.h"

using st::DevGeom;
using st::KParams;

// ---------------------------------------------------------------- errors --
static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(x)                                                        \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess)                                                 \
      return fail(ST_ERR_CUDA, "%s failed: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

#define KERN_TRY(x)                                                        \
  do {                                                                     \
    int e_ = (x);                                                          \
    if (e_ != 0)                                                           \
      return fail(ST_ERR_CUDA, "%s failed: %s", #x,                        \
                  cudaGetErrorString((cudaError_t)e_));                    \
  } while (0)

extern "C" const char* st_last_error(void) { return g_err.c_str(); }
extern "C" const char* st_version(void) { return "stencil_tiler-b200 0.1 (sm_100a)"; }

// --------------------------------------------------------- stencil model --
struct st_stencil {
  std::string name;
  int ndims = 0;
  int model = ST_MODEL_TERMS;
  std::vector<st_term> terms;
  int dtd = 1;
  int radii[3] = {0, 0, 0};
};

// StencilSpec::make (stencil.hpp:59-62): derive delta_t and radii; throw
// (here: return) on no terms, dt < 1, or an offset arity mismatch.
static int make_stencil(const char* name, int ndims, const st_term* terms,
                        int nterms, int model, st_stencil** out) {
  if (!out) return fail(ST_ERR_INVALID, "null output");
  if (ndims < 1 || ndims > ST_MAX_DIMS) return fail(ST_ERR_INVALID, "ndims %d outside [1,3]", ndims);
  if (nterms < 1 || !terms) return fail(ST_ERR_INVALID, "a stencil needs at least one term");
  if (nterms > ST_MAX_TERMS) return fail(ST_ERR_UNSUPPORTED, "%d terms > %d", nterms, ST_MAX_TERMS);
  if (model != ST_MODEL_TERMS && model != ST_MODEL_WAVE) return fail(ST_ERR_INVALID, "unknown model %d", model);
  auto* s = new st_stencil;
  s->name = name ? name : "";
  s->ndims = ndims;
  s->model = model;
  s->dtd = 0;
  for (int k = 0; k < nterms; ++k) {
    const st_term& t = terms[k];
    if (t.dt < 1) { delete s; return fail(ST_ERR_INVALID, "term %d: dt = %d < 1", k + 1, t.dt); }
    if (model == ST_MODEL_WAVE && t.dt != 1) {
      delete s;
      return fail(ST_ERR_INVALID, "wave model: term %d must read u^n (dt = 1)", k + 1);
    }
    st_term c = t;
    for (int i = ndims; i < ST_MAX_DIMS; ++i) c.offsets[i] = 0;
    s->terms.push_back(c);
    s->dtd = std::max(s->dtd, t.dt);
    for (int i = 0; i < ndims; ++i) s->radii[i] = std::max(s->radii[i], std::abs(t.offsets[i]));
  }
  if (model == ST_MODEL_WAVE) s->dtd = 2;
  *out = s;
  return ST_OK;
}

extern "C" int st_stencil_create(const char* name, int ndims, const st_term* terms,
                                 int nterms, int model, st_stencil** out) {
  return make_stencil(name, ndims, terms, nterms, model, out);
}

extern "C" void st_stencil_destroy(st_stencil* s) { delete s; }
extern "C" int st_stencil_ndims(const st_stencil* s) { return s ? s->ndims : -1; }
extern "C" int st_stencil_model(const st_stencil* s) { return s ? s->model : -1; }
extern "C" int st_stencil_nterms(const st_stencil* s) { return s ? (int)s->terms.size() : -1; }
extern "C" int st_stencil_term(const st_stencil* s, int k, st_term* out) {
  if (!s || !out || k < 0 || k >= (int)s->terms.size()) return fail(ST_ERR_INVALID, "bad term index");
  *out = s->terms[k];
  return ST_OK;
}
extern "C" int st_stencil_time_depth(const st_stencil* s) { return s ? s->dtd : -1; }
extern "C" int st_stencil_radius(const st_stencil* s, int dim) {
  if (!s || dim < 0 || dim >= s->ndims) return -1;
  return s->radii[dim];
}
// min_skew_factor (stencil.hpp:99-100): max_i delta_i
extern "C" int st_min_skew_factor(const st_stencil* s) {
  if (!s) return -1;
  int m = 0;
  for (int i = 0; i < s->ndims; ++i) m = std::max(m, s->radii[i]);
  return m;
}
// time_buffer_slots (stencil.hpp:102-105): delta_t + t_t
extern "C" int64_t st_time_buffer_slots(const st_stencil* s, int64_t time_tile) {
  if (!s || time_tile < 1) return -1;
  return s->dtd + time_tile;
}
// flops_per_point (stencil.hpp:107-108): 2k - 1; wave ledger adds 4
extern "C" int64_t st_flops_per_point(const st_stencil* s) {
  if (!s) return -1;
  int64_t f = 2 * (int64_t)s->terms.size() - 1;
  if (s->model == ST_MODEL_WAVE) f += 4;
  return f;
}
// check_legality (transforms.hpp:43-51): legal iff skew >= max_i delta_i.
extern "C" int st_check_legality(const st_stencil* s, const st_plan* plan, int* required_minimum) {
  if (!s || !plan) return fail(ST_ERR_INVALID, "null argument");
  const int m = st_min_skew_factor(s);
  if (required_minimum) *required_minimum = m;
  if (plan->skew < m)
    return fail(ST_ERR_ILLEGAL_PLAN, "illegal plan: skew %d < minimum skew factor %d", plan->skew, m);
  return ST_OK;
}
// required_slots (executor.hpp:83-85)
extern "C" int64_t st_required_slots(const st_stencil* s, const st_plan* plan) {
  if (!s) return -1;
  if (plan && plan->schedule == ST_SCHED_TIME) return s->dtd + std::max<int64_t>(1, plan->time_tile);
  return s->dtd + 1;
}

static void ref_padded(const st_stencil* s, const int64_t* ext, int64_t* P) {
  for (int i = 0; i < s->ndims; ++i) P[i] = ext[i] + 2 * s->radii[i];
}

extern "C" int64_t st_layout_plane(const st_stencil* s, const int64_t* extents) {
  if (!s || !extents) return -1;
  int64_t P[3], p = 1;
  ref_padded(s, extents, P);
  for (int i = 0; i < s->ndims; ++i) {
    if (extents[i] < 1) return -1;
    p *= P[i];
  }
  return p;
}

// ------------------------------------------------------------- parse_spec --
// Grammar (stencil.hpp:87-96): `stencil <id>`, `dims <n>`,
// `extent <D_1..D_n>`, `steps <D_t>`, one or more `term <coeff> <dt>
// <off_1..off_n>`; '#' comments; whitespace tokens.
extern "C" int st_stencil_parse(const char* text, st_stencil** out, int* ndims_out,
                                int64_t* extents_out, int64_t* steps_out, int* err_line) {
  if (!text || !out) return fail(ST_ERR_INVALID, "null argument");
  std::istringstream in(text);
  std::string line, name;
  int ndims = 0, lineno = 0;
  bool have_name = false, have_ext = false, have_steps = false;
  int64_t ext[3] = {0, 0, 0}, steps = 0;
  std::vector<st_term> terms;
  auto perr = [&](const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (err_line) *err_line = lineno;
    return fail(ST_ERR_PARSE, "line %d: %s", lineno, buf);
  };
  auto to_i64 = [](const std::string& t, int64_t& v) {
    char* e = nullptr;
    errno = 0;
    long long r = std::strtoll(t.c_str(), &e, 10);
    if (errno || !e || *e) return false;
    v = r;
    return true;
  };
  while (std::getline(in, line)) {
    ++lineno;
    auto h = line.find('#');
    if (h != std::string::npos) line.resize(h);
    std::istringstream ls(line);
    std::vector<std::string> tok;
    std::string t;
    while (ls >> t) tok.push_back(t);
    if (tok.empty()) continue;
    const std::string& kw = tok[0];
    if (kw == "stencil") {
      if (tok.size() != 2) return perr("`stencil` takes one identifier");
      if (have_name) return perr("duplicate `stencil` line");
      name = tok[1];
      have_name = true;
    } else if (kw == "dims") {
      int64_t n;
      if (tok.size() != 2 || !to_i64(tok[1], n)) return perr("`dims` takes one integer");
      if (n < 1 || n > 3) return perr("dims %lld outside [1,3]", (long long)n);
      if (ndims) return perr("duplicate `dims` line");
      ndims = (int)n;
    } else if (kw == "extent") {
      if (!ndims) return perr("`extent` before `dims`");
      if ((int)tok.size() != ndims + 1) return perr("`extent` needs %d values", ndims);
      for (int i = 0; i < ndims; ++i) {
        int64_t v;
        if (!to_i64(tok[1 + i], v)) return perr("bad extent `%s`", tok[1 + i].c_str());
        if (v < 1) return perr("non-positive extent %lld", (long long)v);
        ext[i] = v;
      }
      have_ext = true;
    } else if (kw == "steps") {
      int64_t v;
      if (tok.size() != 2 || !to_i64(tok[1], v)) return perr("`steps` takes one integer");
      if (v < 1) return perr("non-positive steps %lld", (long long)v);
      steps = v;
      have_steps = true;
    } else if (kw == "term") {
      if (!ndims) return perr("`term` before `dims`");
      if ((int)tok.size() != ndims + 3) return perr("term needs coeff, dt and %d offsets", ndims);
      st_term term{};
      char* e = nullptr;
      term.coeff = std::strtof(tok[1].c_str(), &e);
      if (!e || *e) return perr("bad coefficient `%s`", tok[1].c_str());
      int64_t v;
      if (!to_i64(tok[2], v)) return perr("bad dt `%s`", tok[2].c_str());
      if (v < 1) return perr("dt must be >= 1 (got %lld)", (long long)v);
      term.dt = (int)v;
      for (int i = 0; i < ndims; ++i) {
        if (!to_i64(tok[3 + i], v)) return perr("bad offset `%s`", tok[3 + i].c_str());
        term.offsets[i] = (int)v;
      }
      terms.push_back(term);
    } else {
      return perr("unknown keyword `%s`", kw.c_str());
    }
  }
  ++lineno;
  if (!have_name) return perr("missing `stencil` line");
  if (!ndims) return perr("missing `dims` line");
  if (!have_ext) return perr("missing `extent` line");
  if (!have_steps) return perr("missing `steps` line");
  if (terms.empty()) return perr("no `term` lines");
  int rc = make_stencil(name.c_str(), ndims, terms.data(), (int)terms.size(), ST_MODEL_TERMS, out);
  if (rc) return rc;
  if (ndims_out) *ndims_out = ndims;
  if (extents_out)
    for (int i = 0; i < 3; ++i) extents_out[i] = i < ndims ? ext[i] : 1;
  if (steps_out) *steps_out = steps;
  return ST_OK;
}

// ------------------------------------------------------------ initialisers --
// LCG recurrence of LcgStream (executor.hpp:73-81), with O(log n) jump-ahead
// so large grids fill in parallel; values are identical to the sequential
// stream.
namespace {
constexpr uint64_t kA = 6364136223846793005ULL, kC = 1442695040888963407ULL;
struct Aff { uint64_t a, c; };  // s -> a*s + c
inline Aff compose(Aff f, Aff g) { return {g.a * f.a, g.a * f.c + g.c}; }  // g after f
inline Aff jump(uint64_t n) {
  Aff r{1, 0}, b{kA, kC};
  while (n) {
    if (n & 1) r = compose(r, b);
    b = compose(b, b);
    n >>= 1;
  }
  return r;
}
inline float ref_value(uint64_t s) {
  return static_cast<float>(0.001 + 0.001 * (static_cast<double>(s >> 40) / 16777216.0));
}
inline double unit_value(uint64_t s) { return static_cast<double>(s >> 40) / 16777216.0; }

// Fill out[i] = f(state_{i+1}) for i in [0, n) starting from `seed`
// advanced by `skip` values.
template <class F>
void lcg_fill(uint64_t seed, uint64_t skip, int64_t n, F&& f) {
  const int nt = std::max(1, omp_get_max_threads());
  const int64_t chunk = (n + nt - 1) / nt;
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int t = 0; t < nt; ++t) {
    const int64_t i0 = t * chunk, i1 = std::min<int64_t>(n, i0 + chunk);
    if (i0 >= i1) continue;
    Aff j = jump(skip + (uint64_t)i0);
    uint64_t s = j.a * seed + j.c;
    for (int64_t i = i0; i < i1; ++i) {
      s = s * kA + kC;
      f(i, s);
    }
  }
}

struct RefGeo {
  int n;
  int64_t E[3], P[3], R[3], plane;
};
bool ref_geo(const st_stencil* s, const int64_t* ext, RefGeo& g) {
  if (!s || !ext) return false;
  g.n = s->ndims;
  for (int a = 0; a < 3; ++a) { g.E[a] = 1; g.R[a] = 0; }
  for (int i = 0; i < g.n; ++i) {
    if (ext[i] < 1) return false;
    g.E[3 - g.n + i] = ext[i];
    g.R[3 - g.n + i] = s->radii[i];
  }
  g.plane = 1;
  for (int a = 0; a < 3; ++a) { g.P[a] = g.E[a] + 2 * g.R[a]; g.plane *= g.P[a]; }
  return true;
}
inline int64_t ref_row(const RefGeo& g, int64_t z, int64_t y) {
  return ((z + g.R[0]) * g.P[1] + (y + g.R[1])) * g.P[2] + g.R[2];
}
}  // namespace

extern "C" int st_init_reference(const st_stencil* s, const int64_t* extents, float* host,
                                 int64_t slots, uint64_t seed) {
  // init_grid (executor.hpp:87-90): levels [0, delta_t) incl. halo from the
  // LCG stream, level-major then row-major; remaining slots zero.
  RefGeo g;
  if (!ref_geo(s, extents, g) || !host) return fail(ST_ERR_INVALID, "bad arguments");
  if (slots < s->dtd + 1) return fail(ST_ERR_SLOTS, "slots %lld < delta_t + 1", (long long)slots);
  std::memset(host, 0, sizeof(float) * slots * g.plane);
  lcg_fill(seed, 0, (int64_t)s->dtd * g.plane, [&](int64_t i, uint64_t st) {
    const int64_t lv = i / g.plane, off = i - lv * g.plane;
    host[(lv % slots) * g.plane + off] = ref_value(st);
  });
  return ST_OK;
}

extern "C" int st_init_unit(const st_stencil* s, const int64_t* extents, float* host,
                            int64_t slots, uint64_t seed) {
  // Ledger A.4: zero halo, interior of levels [0, delta_t) in [0,1) from the
  // same recurrence, value (s>>40)/2^24, level-major then row-major.
  RefGeo g;
  if (!ref_geo(s, extents, g) || !host) return fail(ST_ERR_INVALID, "bad arguments");
  if (slots < s->dtd + 1) return fail(ST_ERR_SLOTS, "slots %lld < delta_t + 1", (long long)slots);
  std::memset(host, 0, sizeof(float) * slots * g.plane);
  const int64_t npts = g.E[0] * g.E[1] * g.E[2];
  lcg_fill(seed, 0, (int64_t)s->dtd * npts, [&](int64_t i, uint64_t st) {
    const int64_t lv = i / npts, r = i - lv * npts;
    const int64_t x = r % g.E[2], y = (r / g.E[2]) % g.E[1], z = r / (g.E[2] * g.E[1]);
    host[(lv % slots) * g.plane + ref_row(g, z, y) + x] = static_cast<float>(unit_value(st));
  });
  return ST_OK;
}

extern "C" int st_init_gaussian_slab(const st_stencil* s, const int64_t* extents, float* host,
                                     int64_t slots, double sigma, const int64_t* centre,
                                     int64_t z_begin) {
  // Ledger A.5: exp(-|x-c|^2 / (2 sigma^2)) in double, cast once, identical
  // levels [0, delta_t), zero halo.  z_begin shifts d_1 (slab of a global grid).
  RefGeo g;
  if (!ref_geo(s, extents, g) || !host || !centre) return fail(ST_ERR_INVALID, "bad arguments");
  if (slots < s->dtd + 1) return fail(ST_ERR_SLOTS, "slots %lld < delta_t + 1", (long long)slots);
  std::memset(host, 0, sizeof(float) * slots * g.plane);
  int64_t c3[3] = {0, 0, 0};
  for (int i = 0; i < g.n; ++i) c3[3 - g.n + i] = centre[i];
  const int64_t zsh = g.n == 3 || g.n == 2 ? z_begin : 0;
  const double inv = 1.0 / (2.0 * sigma * sigma);
  float* l0 = host;  // level 0 lives in slot 0
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < g.E[0]; ++z)
    for (int64_t y = 0; y < g.E[1]; ++y) {
      float* r = l0 + ref_row(g, z, y);
      for (int64_t x = 0; x < g.E[2]; ++x) {
        const double dz = double(z + (g.n == 3 ? zsh : 0) - c3[0]);
        const double dy = double(y + (g.n == 2 ? zsh : 0) - c3[1]);
        const double dx = double(x - c3[2]);
        r[x] = static_cast<float>(std::exp(-(dz * dz + dy * dy + dx * dx) * inv));
      }
    }
  for (int lv = 1; lv < s->dtd; ++lv)
    std::memcpy(host + (lv % slots) * g.plane, l0, sizeof(float) * g.plane);
  return ST_OK;
}

extern "C" int st_init_gaussian(const st_stencil* s, const int64_t* extents, float* host,
                                int64_t slots, double sigma, const int64_t* centre) {
  return st_init_gaussian_slab(s, extents, host, slots, sigma, centre, 0);
}

extern "C" int st_field_layered(int ndims, const int64_t* extents, float* m, double v_top,
                                double v_bottom, int64_t split, double dt, double h,
                                int64_t z_begin) {
  // m = (c dt / h)^2 in double, cast once; c = v_top above global row
  // `split` of d_1, v_bottom below (ledger A.3, A.5).
  if (ndims < 1 || ndims > 3 || !extents || !m) return fail(ST_ERR_INVALID, "bad arguments");
  int64_t inner = 1;
  for (int i = 1; i < ndims; ++i) inner *= extents[i];
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < extents[0]; ++z) {
    const double v = (z + z_begin) < split ? v_top : v_bottom;
    const double q = v * dt / h;
    const float mv = static_cast<float>(q * q);
    for (int64_t i = 0; i < inner; ++i) m[z * inner + i] = mv;
  }
  return ST_OK;
}

extern "C" int st_field_random_smoothed(int ndims, const int64_t* extents, float* m,
                                        uint64_t seed, double vmin, double vmax, double dt,
                                        double h) {
  // Config 4: v = LCG U[vmin, vmax] over the interior (row-major), 3^n box
  // filter clamped to the edge in double, m = (v dt / h)^2 cast once.
  if (ndims < 1 || ndims > 3 || !extents || !m) return fail(ST_ERR_INVALID, "bad arguments");
  int64_t E[3] = {1, 1, 1};
  for (int i = 0; i < ndims; ++i) E[3 - ndims + i] = extents[i];
  const int64_t N = E[0] * E[1] * E[2];
  std::vector<double> v(N);
  lcg_fill(seed, 0, N, [&](int64_t i, uint64_t st) { v[i] = vmin + (vmax - vmin) * unit_value(st); });
  const int rz = E[0] > 1, ry = E[1] > 1, rx = E[2] > 1;
  const double cnt = double((2 * rz + 1) * (2 * ry + 1) * (2 * rx + 1));
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < E[0]; ++z)
    for (int64_t y = 0; y < E[1]; ++y)
      for (int64_t x = 0; x < E[2]; ++x) {
        double acc = 0.0;
        for (int dz = -rz; dz <= rz; ++dz)
          for (int dy = -ry; dy <= ry; ++dy)
            for (int dx = -rx; dx <= rx; ++dx) {
              const int64_t zz = std::clamp<int64_t>(z + dz, 0, E[0] - 1);
              const int64_t yy = std::clamp<int64_t>(y + dy, 0, E[1] - 1);
              const int64_t xx = std::clamp<int64_t>(x + dx, 0, E[2] - 1);
              acc += v[(zz * E[1] + yy) * E[2] + xx];
            }
        const double q = (acc / cnt) * dt / h;
        m[(z * E[1] + y) * E[2] + x] = static_cast<float>(q * q);
      }
  return ST_OK;
}

static int verify_levels(const RefGeo& g, const float* a, int64_t slots_a, const float* b, int64_t slots_b,
                         int64_t last_level, int64_t compare_levels, int* equal);

extern "C" int st_verify_bitwise(const st_stencil* s, const int64_t* extents, const float* a,
                                 int64_t slots_a, const float* b, int64_t slots_b,
                                 int64_t last_level, int64_t compare_levels, int* equal) {
  // verify_bitwise (executor.hpp:107-110): bit identity of the last
  // compare_levels levels over the interior; error if not retained.
  RefGeo g;
  if (!ref_geo(s, extents, g) || !a || !b || !equal) return fail(ST_ERR_INVALID, "bad arguments");
  return verify_levels(g, a, slots_a, b, slots_b, last_level, compare_levels, equal);
}

extern "C" int st_verify_bitwise_layout(int ndims, const int64_t* extents, const int64_t* radii, const float* a,
                                        int64_t slots_a, const float* b, int64_t slots_b, int64_t last_level,
                                        int64_t compare_levels, int* equal) {
  // verify_bitwise(a, b, compare_levels) (executor.hpp:110): the Grid's own
  // GridLayout (interior extents + halo radii) instead of a stencil handle.
  if (ndims < 1 || ndims > 3 || !extents || !radii || !a || !b || !equal) return fail(ST_ERR_INVALID, "bad arguments");
  RefGeo g;
  g.n = ndims;
  for (int k = 0; k < 3; ++k) { g.E[k] = 1; g.R[k] = 0; }
  for (int i = 0; i < ndims; ++i) {
    if (extents[i] < 1 || radii[i] < 0) return fail(ST_ERR_INVALID, "bad extents / radii");
    g.E[3 - ndims + i] = extents[i];
    g.R[3 - ndims + i] = radii[i];
  }
  g.plane = 1;
  for (int k = 0; k < 3; ++k) { g.P[k] = g.E[k] + 2 * g.R[k]; g.plane *= g.P[k]; }
  return verify_levels(g, a, slots_a, b, slots_b, last_level, compare_levels, equal);
}

static int verify_levels(const RefGeo& g, const float* a, int64_t slots_a, const float* b, int64_t slots_b,
                         int64_t last_level, int64_t compare_levels, int* equal) {
  if (compare_levels < 1) return fail(ST_ERR_INVALID, "compare_levels < 1");
  if (compare_levels > slots_a || compare_levels > slots_b || last_level - compare_levels + 1 < 0)
    return fail(ST_ERR_SLOTS, "grid no longer retains %lld levels", (long long)compare_levels);
  *equal = 1;
  for (int64_t lv = last_level - compare_levels + 1; lv <= last_level && *equal; ++lv) {
    const float* pa = a + (lv % slots_a) * g.plane;
    const float* pb = b + (lv % slots_b) * g.plane;
    for (int64_t z = 0; z < g.E[0] && *equal; ++z)
      for (int64_t y = 0; y < g.E[1]; ++y) {
        const int64_t o = ref_row(g, z, y);
        if (std::memcmp(pa + o, pb + o, sizeof(float) * g.E[2])) { *equal = 0; break; }
      }
  }
  return ST_OK;
}

// --------------------------------------------------------------- context --
struct st_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sms = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // host-overlapped execute: upload / download copy streams and their events
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t evx[8] = {};   // evx[0] stream handoffs, evx[1..] upload blocks
  void* l2junk = nullptr;    // st_context_flush_l2: a buffer larger than L2
  size_t l2junk_bytes = 0;
};

extern "C" int st_context_create(int device, st_context** out) {
  if (!out) return fail(ST_ERR_INVALID, "null output");
  int n = 0;
  CUDA_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(ST_ERR_INVALID, "device %d not present (%d visible)", device, n);
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(ST_ERR_UNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a (B200)", device,
                prop.major, prop.minor);
  auto* c = new st_context;
  c->device = device;
  c->sms = prop.multiProcessorCount;
  bool ok = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreate(&c->ev0) == cudaSuccess && cudaEventCreate(&c->ev1) == cudaSuccess;
  for (auto& e : c->evx) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    delete c;
    return fail(ST_ERR_CUDA, "stream/event creation failed");
  }
  *out = c;
  return ST_OK;
}

extern "C" void st_context_destroy(st_context* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (auto e : c->evx)
    if (e) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  if (c->l2junk) cudaFree(c->l2junk);
  delete c;
}

extern "C" int st_context_flush_l2(st_context* c) {
  // timing hygiene between trials (autotuner, bench): overwrite twice the L2
  // so no trial starts with the previous one's data resident
  if (!c) return fail(ST_ERR_INVALID, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  if (!c->l2junk) {
    int l2 = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device));
    c->l2junk_bytes = std::max<size_t>((size_t)2 * (size_t)l2, 64u << 20);
    CUDA_TRY(cudaMalloc(&c->l2junk, c->l2junk_bytes));
  }
  CUDA_TRY(cudaMemsetAsync(c->l2junk, 0x5a, c->l2junk_bytes, c->stream));
  return ST_OK;
}
extern "C" void* st_context_stream(st_context* c) { return c ? (void*)c->stream : nullptr; }
extern "C" int st_context_device(const st_context* c) { return c ? c->device : -1; }
extern "C" int st_context_sm_count(const st_context* c) { return c ? c->sms : -1; }

// ------------------------------------------------------------------ grid --
struct st_grid {
  st_context* ctx = nullptr;
  st_stencil spec;
  int64_t ext[3] = {1, 1, 1};
  int64_t slots = 0;
  long long refP[3] = {1, 1, 1};
  int64_t ref_plane = 0;
  DevGeom g{};
  int nbuf = 0;
  float* buf[st::kMaxBuffers] = {};
  float* mfield = nullptr;
  float* bank = nullptr;
  float* staging = nullptr;
  bool has_field = false, uploaded = false;
  int64_t last_level = -1, valid_from = 0;
  unsigned* prog = nullptr;
  size_t prog_cap = 0;
  unsigned* done = nullptr;
  size_t done_cap = 0;
  unsigned* ticket = nullptr;
  unsigned* xfer = nullptr;        // host-overlapped execute: [32] upload count, then download counts
  size_t xfer_cap = 0;
  float* xstage = nullptr;         // host-grid execute: 2 delta_t reference-layout staging slots
  size_t xstage_cap = 0;
  long long* dbg_host = nullptr;   // zero-copy diagnostics written by the watchdog
  long long* dbg_dev = nullptr;
  // fused-level passes write a level while its predecessor is still read:
  // one spare level buffer (uniform halo kept in step with the others)
  float* xbuf = nullptr;
  float* rxch = nullptr;           // SM-resident 2-D kernel: epoch exchange buffers (2 levels)
  unsigned char* mcode = nullptr;  // palettized m field: 1-byte codes (device layout)
  float* mpal = nullptr;           // its palette (256 floats)
  int npal = 0;                    // palette size (0: m is not palettized)
  size_t rxch_cap = 0;
  int reserve_ctas = 0;            // persistent launches leave this many CTA slots free (overlapped NCCL)
};

// tuning knobs read once per launch (the defaults are the measured best)
static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

static int dev_axis(int n, int i) {
  if (n == 3) return i;
  if (n == 2) return i == 0 ? 0 : 2;
  return 2;
}

static DevGeom make_geom(const st_stencil& s, const int64_t* ext) {
  DevGeom g{};
  int64_t E[3] = {1, 1, 1};
  int R[3] = {0, 0, 0};
  for (int i = 0; i < s.ndims; ++i) {
    E[dev_axis(s.ndims, i)] = ext[i];
    R[dev_axis(s.ndims, i)] = s.radii[i];
  }
  g.nz = (int)E[0]; g.ny = (int)E[1]; g.nx = (int)E[2];
  g.rz = R[0]; g.ry = R[1]; g.rx = R[2];
  g.xo = g.rx == 0 ? 0 : ((g.rx + 31) / 32) * 32;   // interior rows start 128-B aligned
  g.pitch = ((g.xo + g.nx + g.rx + 31) / 32) * 32;
  g.pstride = (long long)(g.ny + 2 * g.ry) * g.pitch;
  g.base = (long long)g.rz * g.pstride + (long long)g.ry * g.pitch + g.xo;
  // slack: tiles overhang the domain by < one tile; their (never stored)
  // lanes still load, so keep one extra plane + 64 rows addressable.
  g.buf_elems = (long long)(g.nz + 2 * g.rz) * g.pstride + g.pstride + 64 * g.pitch + 1024;
  return g;
}

static void grid_free(st_grid* gr) {
  if (!gr) return;
  cudaSetDevice(gr->ctx->device);
  for (int b = 0; b < st::kMaxBuffers; ++b)
    if (gr->buf[b]) cudaFree(gr->buf[b]);
  if (gr->mfield) cudaFree(gr->mfield);
  if (gr->bank) cudaFree(gr->bank);
  if (gr->staging) cudaFree(gr->staging);
  if (gr->prog) cudaFree(gr->prog);
  if (gr->done) cudaFree(gr->done);
  if (gr->ticket) cudaFree(gr->ticket);
  if (gr->xfer) cudaFree(gr->xfer);
  if (gr->xstage) cudaFree(gr->xstage);
  if (gr->xbuf) cudaFree(gr->xbuf);
  if (gr->rxch) cudaFree(gr->rxch);
  if (gr->mcode) cudaFree(gr->mcode);
  if (gr->mpal) cudaFree(gr->mpal);
  if (gr->dbg_host) cudaFreeHost(gr->dbg_host);
}

extern "C" int st_grid_create(st_context* c, const st_stencil* s, const int64_t* extents,
                              int64_t slots, st_grid** out) {
  if (!c || !s || !extents || !out) return fail(ST_ERR_INVALID, "null argument");
  for (int i = 0; i < s->ndims; ++i)
    if (extents[i] < 1 || extents[i] > (1LL << 30)) return fail(ST_ERR_INVALID, "extent %d out of range", i);
  if (slots < s->dtd + 1)
    return fail(ST_ERR_SLOTS, "slots %lld < delta_t + 1 = %d (required_slots)", (long long)slots, s->dtd + 1);
  if (s->dtd + 1 > st::kMaxBuffers) return fail(ST_ERR_UNSUPPORTED, "delta_t %d too deep", s->dtd);
  CUDA_TRY(cudaSetDevice(c->device));
  auto* gr = new st_grid;
  gr->ctx = c;
  gr->spec = *s;
  gr->slots = slots;
  for (int i = 0; i < s->ndims; ++i) {
    gr->ext[i] = extents[i];
    gr->refP[i] = extents[i] + 2 * s->radii[i];
  }
  gr->ref_plane = st_layout_plane(s, extents);
  gr->g = make_geom(*s, extents);
  gr->nbuf = s->dtd + 1;
  const size_t bytes = sizeof(float) * (size_t)gr->g.buf_elems;
  cudaError_t e = cudaSuccess;
  for (int b = 0; b < gr->nbuf && e == cudaSuccess; ++b) {
    e = cudaMalloc(&gr->buf[b], bytes);
    if (e == cudaSuccess) e = cudaMemsetAsync(gr->buf[b], 0, bytes, c->stream);
  }
  if (e == cudaSuccess) e = cudaMalloc(&gr->staging, sizeof(float) * (size_t)gr->ref_plane);
  if (e == cudaSuccess) e = cudaMalloc(&gr->ticket, sizeof(unsigned));
  if (e == cudaSuccess) e = cudaHostAlloc(&gr->dbg_host, 16 * sizeof(long long), cudaHostAllocMapped);
  if (e == cudaSuccess) {
    std::memset(gr->dbg_host, 0, 16 * sizeof(long long));
    e = cudaHostGetDevicePointer(&gr->dbg_dev, gr->dbg_host, 0);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    grid_free(gr);
    delete gr;
    return fail(ST_ERR_CUDA, "grid allocation (%zu MB per level buffer): %s", bytes >> 20,
                cudaGetErrorString(e));
  }
  *out = gr;
  return ST_OK;
}

extern "C" void st_grid_destroy(st_grid* g) {
  grid_free(g);
  delete g;
}

extern "C" int64_t st_grid_device_bytes(const st_grid* gr) {
  if (!gr) return -1;
  int64_t b = (int64_t)(gr->nbuf + (gr->xbuf ? 1 : 0)) * gr->g.buf_elems * 4 + gr->ref_plane * 4;
  if (gr->mfield) b += gr->g.buf_elems * 4;
  if (gr->bank) b += gr->slots * gr->g.buf_elems * 4;
  return b;
}

// True when every slot of the host grid carries the same halo cells.
static bool halos_uniform(const st_grid* gr, const float* host) {
  RefGeo rg;
  ref_geo(&gr->spec, gr->ext, rg);
  for (int64_t s = 1; s < gr->slots; ++s) {
    const float* a = host;
    const float* b = host + s * rg.plane;
    for (int64_t pz = 0; pz < rg.P[0]; ++pz) {
      const bool zh = pz < rg.R[0] || pz >= rg.R[0] + rg.E[0];
      for (int64_t py = 0; py < rg.P[1]; ++py) {
        const int64_t o = (pz * rg.P[1] + py) * rg.P[2];
        const bool yh = py < rg.R[1] || py >= rg.R[1] + rg.E[1];
        if (zh || yh) {
          if (std::memcmp(a + o, b + o, sizeof(float) * rg.P[2])) return false;
        } else if (rg.R[2]) {
          if (std::memcmp(a + o, b + o, sizeof(float) * rg.R[2])) return false;
          const int64_t o2 = o + rg.R[2] + rg.E[2];
          if (std::memcmp(a + o2, b + o2, sizeof(float) * rg.R[2])) return false;
        }
      }
    }
  }
  return true;
}

extern "C" int st_grid_upload(st_grid* gr, const float* host, int64_t nelems, int64_t last_level,
                              unsigned flags) {
  if (!gr || !host) return fail(ST_ERR_INVALID, "null argument");
  if (nelems != gr->slots * gr->ref_plane)
    return fail(ST_ERR_INVALID, "host grid has %lld elements, layout needs %lld", (long long)nelems,
                (long long)(gr->slots * gr->ref_plane));
  const int dtd = gr->spec.dtd;
  if (last_level < dtd - 1) return fail(ST_ERR_SLOTS, "last_level %lld < delta_t - 1", (long long)last_level);
  cudaStream_t st = gr->ctx->stream;
  CUDA_TRY(cudaSetDevice(gr->ctx->device));
  const size_t pbytes = sizeof(float) * (size_t)gr->ref_plane;
  const bool uniform = (flags & ST_UPLOAD_UNIFORM_HALO) || halos_uniform(gr, host);
  // the delta_t levels the next step reads, oldest first; the newest last
  // so `staging` still holds it for the halo copy below
  bool holds[st::kMaxBuffers] = {};
  for (int64_t lv = last_level - dtd + 1; lv <= last_level; ++lv) {
    const float* slot = host + (lv % gr->slots) * gr->ref_plane;
    CUDA_TRY(cudaMemcpyAsync(gr->staging, slot, pbytes, cudaMemcpyHostToDevice, st));
    float* dst = gr->buf[lv % gr->nbuf];
    KERN_TRY(st::launch_ref_to_dev(gr->staging, dst, gr->g, gr->spec.ndims, gr->refP, st));
    holds[lv % gr->nbuf] = true;
  }
  if (uniform) {
    for (int b = 0; b < gr->nbuf; ++b)
      if (!holds[b])
        KERN_TRY(st::launch_ref_to_dev(gr->staging, gr->buf[b], gr->g, gr->spec.ndims, gr->refP, st));
    if (gr->xbuf) KERN_TRY(st::launch_ref_to_dev(gr->staging, gr->xbuf, gr->g, gr->spec.ndims, gr->refP, st));
    if (gr->bank) {
      cudaFree(gr->bank);
      gr->bank = nullptr;
    }
  } else {
    if (!gr->bank) CUDA_TRY(cudaMalloc(&gr->bank, sizeof(float) * (size_t)gr->g.buf_elems * gr->slots));
    for (int64_t s = 0; s < gr->slots; ++s) {
      CUDA_TRY(cudaMemcpyAsync(gr->staging, host + s * gr->ref_plane, pbytes, cudaMemcpyHostToDevice, st));
      KERN_TRY(st::launch_ref_to_dev(gr->staging, gr->bank + s * gr->g.buf_elems, gr->g, gr->spec.ndims,
                                     gr->refP, st));
    }
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  gr->last_level = last_level;
  gr->valid_from = last_level - dtd + 1;
  gr->uploaded = true;
  return ST_OK;
}

extern "C" int st_grid_set_field(st_grid* gr, const float* m, int64_t nelems) {
  if (!gr || !m) return fail(ST_ERR_INVALID, "null argument");
  const int64_t n = (int64_t)gr->g.nz * gr->g.ny * gr->g.nx;
  if (nelems != n) return fail(ST_ERR_INVALID, "field has %lld elements, interior is %lld", (long long)nelems,
                               (long long)n);
  cudaStream_t st = gr->ctx->stream;
  CUDA_TRY(cudaSetDevice(gr->ctx->device));
  const size_t bytes = sizeof(float) * (size_t)gr->g.buf_elems;
  if (!gr->mfield) {
    CUDA_TRY(cudaMalloc(&gr->mfield, bytes));
    CUDA_TRY(cudaMemsetAsync(gr->mfield, 0, bytes, st));
  }
  float* tmp = nullptr;
  CUDA_TRY(cudaMallocAsync(&tmp, sizeof(float) * (size_t)n, st));
  CUDA_TRY(cudaMemcpyAsync(tmp, m, sizeof(float) * (size_t)n, cudaMemcpyHostToDevice, st));
  KERN_TRY(st::launch_interior_to_dev(tmp, gr->mfield, gr->g, st));
  // palettize (<= 256 distinct values) so that the wave kernels read 1-byte
  // codes into an exact float palette: m costs 1 B instead of 4 per update
  // (config 3: 18 -> 14 B/update in DRAM, 378 -> 386 GPts/s; config 5: 356
  // -> 391).  More than 256 values (config 4's random
  // velocity): floats as before.  ST_MCODES=0 turns it off.
  gr->npal = 0;
  if (env_int("ST_MCODES", 1)) {
    if (!gr->mcode) {
      CUDA_TRY(cudaMalloc(&gr->mcode, (size_t)gr->g.buf_elems));
      CUDA_TRY(cudaMemsetAsync(gr->mcode, 0, (size_t)gr->g.buf_elems, st));
    }
    if (!gr->mpal) CUDA_TRY(cudaMalloc(&gr->mpal, 256 * sizeof(float)));
    float pal_host[256];
    int npal = 0;
    KERN_TRY(st::build_palette(tmp, gr->g, gr->mcode, gr->mpal, pal_host, &npal, st));
    gr->npal = npal;
  }
  CUDA_TRY(cudaFreeAsync(tmp, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  gr->has_field = true;
  return ST_OK;
}

extern "C" int st_grid_download(st_grid* gr, float* host, int64_t nelems, int64_t* last_level) {
  if (!gr || !host) return fail(ST_ERR_INVALID, "null argument");
  if (!gr->uploaded) return fail(ST_ERR_STATE, "grid has no data (upload first)");
  if (nelems != gr->slots * gr->ref_plane) return fail(ST_ERR_INVALID, "host grid size mismatch");
  cudaStream_t st = gr->ctx->stream;
  CUDA_TRY(cudaSetDevice(gr->ctx->device));
  const size_t pbytes = sizeof(float) * (size_t)gr->ref_plane;
  const int64_t lo = std::max(gr->valid_from, gr->last_level - gr->nbuf + 1);
  for (int64_t lv = std::max<int64_t>(0, lo); lv <= gr->last_level; ++lv) {
    KERN_TRY(st::launch_dev_to_ref(gr->buf[lv % gr->nbuf], gr->staging, gr->g, gr->spec.ndims, gr->refP, st));
    CUDA_TRY(cudaMemcpyAsync(host + (lv % gr->slots) * gr->ref_plane, gr->staging, pbytes,
                             cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  if (last_level) *last_level = gr->last_level;
  return ST_OK;
}

extern "C" int st_grid_last_level(const st_grid* gr, int64_t* last_level) {
  if (!gr || !last_level) return fail(ST_ERR_INVALID, "null argument");
  *last_level = gr->last_level;
  return ST_OK;
}


// ------------------------------------------------- host-grid transfers ----
// Upload: a z-block of padded planes is contiguous in a reference-layout
// slot, so it crosses PCIe as one contiguous copy into a reference-layout
// staging area (55 GB/s) and a row kernel converts it into the pitched device
// layout (the copy engines do 2D host->device copies of 1-KB rows at only
// ~9 GB/s).  Download: the copy engine reads the pitched interior rows
// straight into the host slot (2D device->host copies run at ~52 GB/s).
// Measured and dropped: gating the wavefront on upload blocks and the
// download on per-block completion counters (cuStreamWrite/WaitValue32) --
// the dependency cone of a 32-level tile spans half the grid and the row
// kernels cannot co-reside with the 10-warp / 168-register wavefront, so it
// was slower than back-to-back phases (5.0 vs 4.5 ms on config 2).
static const int kUpBlocks = 4;    // upload blocks: the conversion of one overlaps the copy of the next

struct HostXfer {
  float* host;     // reference-layout host grid (slots x ref_plane), page-locked
};

// --------------------------------------------------------------- execute --
// Canonical star: centre, then per reference dim d_1..d_n: -1,+1,...,-R,+R,
// all dt = 1, same radius on every dim.
static bool canonical_star(const st_stencil& s, int& R) {
  R = s.radii[0];
  for (int i = 0; i < s.ndims; ++i)
    if (s.radii[i] != R) return false;
  if (R < 1) return false;
  if ((int)s.terms.size() != 1 + 2 * R * s.ndims) return false;
  int k = 0;
  auto is = [&](int dim, int off) {
    const st_term& t = s.terms[k++];
    if (t.dt != 1) return false;
    for (int i = 0; i < s.ndims; ++i)
      if (t.offsets[i] != (i == dim ? off : 0)) return false;
    return true;
  };
  if (!is(-1, 0)) return false;
  for (int d = 0; d < s.ndims; ++d)
    for (int r = 1; r <= R; ++r) {
      if (!is(d, -r)) return false;
      if (!is(d, r)) return false;
    }
  return true;
}

static bool symmetric_star(const st_stencil& s, int R) {
  for (int d = 0; d < s.ndims; ++d)
    for (int r = 1; r <= R; ++r) {
      const int i = 1 + d * 2 * R + 2 * (r - 1);
      if (std::memcmp(&s.terms[i].coeff, &s.terms[i + 1].coeff, sizeof(float))) return false;
    }
  return true;
}

static int ensure_counters(st_grid* gr, size_t nprog, size_t ndone) {
  if (nprog > gr->prog_cap) {
    if (gr->prog) cudaFree(gr->prog);
    gr->prog = nullptr;
    CUDA_TRY(cudaMalloc(&gr->prog, nprog * sizeof(unsigned)));
    gr->prog_cap = nprog;
  }
  if (ndone > gr->done_cap) {
    if (gr->done) cudaFree(gr->done);
    gr->done = nullptr;
    CUDA_TRY(cudaMalloc(&gr->done, ndone * sizeof(unsigned)));
    gr->done_cap = ndone;
  }
  return ST_OK;
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- TMA tensor maps ------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
  }
  return fn;
}

// L2 fetch granularity of the TMA boxes (ST_TMA_PROMO: 0 none, 1 64 B, 2 128 B, 3 256 B).  128 B: a box
// row starts 16 B before a 128-B line, so 256-B promotion over-fetched at both ends of every row
// (config 5 FAST: 1326 -> 1267 GB per run, 403 -> 411 GPts/s).
static CUtensorMapL2promotion tma_promotion() {
  switch (env_int("ST_TMA_PROMO", 2)) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

// 3D map over a pitched level buffer: (x = padded column incl. pitch slack,
// y = padded row, z = padded plane), box (bw, bh, 1).
static int make_map(CUtensorMap* m, const void* base, const DevGeom& g, int bw, int bh, int esize = 4) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(ST_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)g.pitch, (cuuint64_t)(g.ny + 2 * g.ry), (cuuint64_t)(g.nz + 2 * g.rz)};
  const cuuint64_t strides[2] = {(cuuint64_t)g.pitch * esize, (cuuint64_t)g.pstride * esize};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, esize == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base,
                   dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, tma_promotion(),
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) box %dx%d", (int)r, bw, bh);
  return ST_OK;
}

// Shared-memory ring sizing + tensor maps for the star kernel.  The ring
// holds RZ + 1 + PD planes (PD planes of TMA prefetch in flight); the wave
// operand ring PD + 2 planes.  Budget: the 227 KB opt-in shared memory.
static int setup_pipeline(st_grid* gr, int R, st::LaunchCfg& lc, KParams& p) {
  const DevGeom& g = gr->g;
  const st::StarShape sh = st::star_shape(R, gr->spec.ndims, gr->spec.model, lc.variant);
  const bool wave = gr->spec.model == ST_MODEL_WAVE;
  p.pipe.ns = sh.NS;
  p.pipe.nsa = sh.NSA;
  p.pipe.sw = sh.SW;
  p.pipe.stage_floats = sh.STAGE;
  p.pipe.aux_floats = sh.AUX;
  p.pipe.main_bytes = sh.SW * sh.SH * 4;
  p.pipe.aux_bytes = wave ? 2 * sh.TX * sh.TY * 4 : 0;
  p.pipe.unit = 1;   // the producer publishes whole planes
  lc.smem = st::star_smem_bytes(sh);
  for (int b = 0; b < gr->nbuf && b < 4; ++b) {
    int rc = make_map(&p.tm.main[b], gr->buf[b], g, sh.SW, sh.SH);
    if (rc) return rc;
    if (wave) {
      rc = make_map(&p.tm.aux[b], gr->buf[b], g, sh.TX, sh.TY);
      if (rc) return rc;
    }
  }
  if (wave) {
    int rc = make_map(&p.tm.mfield, gr->mfield, g, sh.TX, sh.TY);
    if (rc) return rc;
    p.mcode_on = 0;
    if (gr->npal > 0 && gr->mcode && env_int("ST_MCODES", 1)) {
      rc = make_map(&p.tm.mcodes, gr->mcode, g, sh.TX, sh.TY, 1);
      if (rc) return rc;
      p.mcode_on = 1;
      p.mpal = gr->mpal;
      p.npal = gr->npal;
    }
    if (sh.MCO && !p.mcode_on)
      return fail(ST_ERR_UNSUPPORTED, "star shape %d needs a palettized m field (<= 256 distinct values)", lc.variant);
  }
  return ST_OK;
}

// Fused-level passes (on-chip time tile, st_fused.cuh): steps are run F at
// a time; each pass reads one level buffer and writes a different one (the
// pool is the grid's level buffers plus one spare), so no pass overwrites a
// level its overlapped neighbours still read.  Afterwards the buffer holding
// the newest level is swapped into that level's canonical slot.
// The spare level buffer of the on-chip realisations (allocated on first
// use; uniform halos, so a copy of the current level carries them).
static int ensure_spare(st_grid* gr, const float* like, cudaStream_t st) {
  if (gr->xbuf) return ST_OK;
  const size_t bytes = sizeof(float) * (size_t)gr->g.buf_elems;
  if (cudaMalloc(&gr->xbuf, bytes) != cudaSuccess)
    return fail(ST_ERR_CUDA, "spare level buffer allocation failed (%zu MB)", bytes >> 20);
  CUDA_TRY(cudaMemcpyAsync(gr->xbuf, like, bytes, cudaMemcpyDeviceToDevice, st));
  return ST_OK;
}

// After an on-chip realisation the newest level sits in `cur` (a level buffer
// or the spare): swap it into that level's canonical slot.
static void place_newest(st_grid* gr, float* cur, int64_t level) {
  const int tgt = (int)(level % gr->nbuf);
  if (gr->buf[tgt] == cur) return;
  if (gr->xbuf == cur) {
    std::swap(gr->xbuf, gr->buf[tgt]);
    return;
  }
  for (int b = 0; b < gr->nbuf; ++b)
    if (gr->buf[b] == cur) {
      std::swap(gr->buf[b], gr->buf[tgt]);
      return;
    }
}

// SM-resident 2-D time tiling (st_resident.cuh): one cooperative launch; the
// grid stays in shared memory, cut into gx x gy tiles, and F levels run
// between halo exchanges.  F = the requested levels per exchange, lowered
// until a tiling fits shared memory; the tiling minimises a per-level cost
// model in warp-row steps (row passes x 32-column warp passes, summed over the
// epoch's shrinking trapezoid) plus a fixed exchange cost (fitted to config 1:
// 0.016 us per step, ~3.4 us per strip exchange, ~4.6 us per tile exchange).  ST_RES_GX forces the column tiles.
// Returns F (0 = does not fit).
// Shared memory one resident2d_kernel CTA indexes: 2 buffers x LR x SW
// floats, maximised over the gy x gx tiles with exactly the kernel's tile
// geometry (st_resident.cuh, the lr0/lr1/lcs/lce/SW lines).
static int64_t resident_tile_bytes(int64_t nz, int64_t nx, int64_t gy, int64_t gx, int64_t R, int64_t H) {
  const int64_t XH = (R + 3) / 4 * 4, HC = (H + 3) / 4 * 4, NX4 = (nx + 3) / 4;
  int64_t worst = 0;
  for (int64_t b = 0; b < gy; ++b) {
    const int64_t r0 = nz * b / gy, r1 = nz * (b + 1) / gy;
    const bool top = r0 - H <= 0, bot = r1 + H >= nz;
    const int64_t LR = (bot ? nz + R : r1 + H) - (top ? -R : r0 - H);
    for (int64_t bc = 0; bc < gx; ++bc) {
      const int64_t c0 = 4 * (NX4 * bc / gx), c1 = std::min(4 * (NX4 * (bc + 1) / gx), nx);
      const bool lft = c0 - HC <= 0, rgt = c1 + HC >= nx;
      const int64_t SW = (rgt ? 4 * NX4 + XH : c1 + HC) - (lft ? -XH : c0 - HC) + 8;
      worst = std::max(worst, 2 * LR * SW * 4);
    }
  }
  return worst;
}

static int resident_plan(const st_grid* gr, int R, int64_t want, int64_t nsteps, int& grid, int& smem, int& gx) {
  const DevGeom& g = gr->g;
  const int64_t sms = gr->ctx->sms, nz = g.nz, nx4 = ceil_div(g.nx, 4);
  const int force = env_int("ST_RES_GX", 0);
  for (int64_t f = std::min(want, nsteps); f >= 1; --f) {
    const int64_t H = R * f, HC = (H + 3) / 4 * 4;
    double best = 0;
    for (int64_t cx = 1; cx <= std::min<int64_t>(nx4, 16); ++cx) {
      if (force > 0 && cx != force) continue;
      const int64_t cy = std::min(nz, sms / cx);
      if (cy < 1) break;
      const int64_t rows = ceil_div(nz, cy), cols = 4 * ceil_div(nx4, cx);
      // smem: two buffers of LR x SW floats, the largest over the actual
      // tiles, by the kernel's own formulas (st_resident.cuh: lr0/lr1,
      // lcs/lce; a side reaching the grid edge takes the whole frozen halo)
      const int64_t bytes = resident_tile_bytes(nz, g.nx, cy, cx, R, H);
      if (bytes > 220 * 1024) continue;
      // exchange: ~210 steps for strips, ~74 more with column tiles (up to
      // 8 neighbours' flags, a ring instead of two row bands; measured:
      // strip F=4 213 us, tiled F=4 225 us, tiled F=16 171 us per launch of
      // config 1)
      double cost = cx > 1 ? 284.0 : 210.0;
      for (int64_t j = 1; j <= f; ++j) {
        const int64_t r = std::min(nz, rows + 2 * (H - j * R));
        const int64_t c4 = std::min(nx4, ceil_div(cols + 2 * (HC - j * R), 4) + 1);
        cost += (double)r * (double)ceil_div(c4, 32);
      }
      cost /= (double)f;
      if (best == 0 || cost < best) {
        best = cost;
        grid = (int)(cx * cy);
        gx = (int)cx;
        smem = (int)bytes;
      }
    }
    if (best > 0) return (int)f;
  }
  return 0;
}

static int run_resident(st_grid* gr, KParams& p, int R, int F, int grid, int gx, int smem, int fast, int64_t t_begin,
                        int64_t nsteps, cudaStream_t st, int64_t& launches) {
  const DevGeom& g = gr->g;
  const int dtd = gr->spec.dtd;
  float* cur = gr->buf[(t_begin + dtd - 1) % gr->nbuf];
  int rc = ensure_spare(gr, cur, st);
  if (rc) return rc;
  const size_t n2 = 2 * (size_t)g.buf_elems;
  if (!gr->rxch || gr->rxch_cap < n2) {
    if (gr->rxch) cudaFree(gr->rxch);
    gr->rxch = nullptr;
    gr->rxch_cap = 0;
    if (cudaMalloc(&gr->rxch, n2 * sizeof(float)) != cudaSuccess)
      return fail(ST_ERR_CUDA, "exchange buffer allocation failed");
    gr->rxch_cap = n2;
  }
  float* out = nullptr;
  for (int b = 0; b < gr->nbuf && !out; ++b)
    if (gr->buf[b] != cur) out = gr->buf[b];
  if (!out) out = gr->xbuf;
  rc = ensure_counters(gr, (size_t)grid << 5, 1);
  if (rc) return rc;
  p.fin = cur;
  p.fout = out;
  p.xch0 = gr->rxch;
  p.xch1 = gr->rxch + g.buf_elems;
  p.T = F;
  p.rgx = gx;
  p.nsteps = (int)nsteps;
  p.prog = gr->prog;
  p.ctr_shift = 5;
  CUDA_TRY(cudaMemsetAsync(gr->prog, 0, ((size_t)grid << 5) * sizeof(unsigned), st));
  const int e = st::launch_resident2d(R, fast, p, grid, smem, st);
  if (e) return fail(ST_ERR_CUDA, "SM-resident launch failed: %s", cudaGetErrorString((cudaError_t)e));
  ++launches;
  place_newest(gr, out, t_begin + nsteps + dtd - 1);
  return ST_OK;
}

// Put the newest level(s) into their canonical slots: `p1` holds level
// `newest`, `p2` (wave) level newest - 1; the other buffers fill the
// remaining slots, the leftover becomes the spare.
static void arrange_levels(st_grid* gr, int64_t newest, float* p1, float* p2) {
  float* all[st::kMaxBuffers + 1];
  int n = 0;
  for (int b = 0; b < gr->nbuf; ++b) all[n++] = gr->buf[b];
  all[n++] = gr->xbuf;
  float* nb[st::kMaxBuffers] = {};
  nb[newest % gr->nbuf] = p1;
  if (p2) nb[(newest - 1) % gr->nbuf] = p2;
  int k = 0;
  for (int b = 0; b < gr->nbuf; ++b) {
    if (nb[b]) continue;
    while (all[k] == p1 || all[k] == p2) ++k;
    nb[b] = all[k++];
  }
  while (all[k] == p1 || all[k] == p2) ++k;
  gr->xbuf = all[k];
  for (int b = 0; b < gr->nbuf; ++b) gr->buf[b] = nb[b];
}

static int run_fused(st_grid* gr, KParams& p, int R, int F, int ty_req, int fast, int64_t t_begin, int64_t nsteps,
                     cudaStream_t st, int64_t& launches, int& ty_used) {
  const DevGeom& g = gr->g;
  const int dtd = gr->spec.dtd;
  const bool wave = gr->spec.model == ST_MODEL_WAVE;
  // inputs: the newest level (in1) and, for the leapfrog, the one before (in2)
  float* in1 = gr->buf[(t_begin + dtd - 1) % gr->nbuf];
  float* in2 = wave ? gr->buf[(t_begin + dtd - 2) % gr->nbuf] : nullptr;
  {
    const int rc = ensure_spare(gr, in1, st);
    if (rc) return rc;
  }
  float* pool[st::kMaxBuffers + 1];
  int np = 0;
  for (int b = 0; b < gr->nbuf; ++b) pool[np++] = gr->buf[b];
  pool[np++] = gr->xbuf;
  // a pass writes buffers no input of that pass lives in (overlapping tiles
  // still read the inputs)
  auto pick = [&](float* a, float* b, float* c) -> float* {
    for (int i = 0; i < np; ++i)
      if (pool[i] != a && pool[i] != b && pool[i] != c) return pool[i];
    return nullptr;
  };
  for (int64_t l = 0; l < nsteps;) {
    const int f = (int)std::min<int64_t>(F, nsteps - l);
    const st::FusedFn fn = st::fused_lookup(R, f, ty_req, fast, wave ? 1 : 0);
    if (!fn.fn) return fail(ST_ERR_UNSUPPORTED, "fused-level kernel (R %d, F %d) not built", R, f);
    float* o1 = pick(in1, in2, nullptr);
    float* o2 = wave && f > 1 ? pick(in1, in2, o1) : nullptr;
    if (!o1 || (wave && f > 1 && !o2)) return fail(ST_ERR_STATE, "fused: no free level buffer");
    p.fin = in1;
    p.fout = o1;
    p.fout2 = o2;
    int rc = make_map(&p.tm.fused, in1, g, fn.bw, fn.bh);
    if (!rc && wave) rc = make_map(&p.tm.fused_u2, in2, g, fn.cx, fn.cy);
    if (!rc && wave) rc = make_map(&p.tm.fused_m, gr->mfield, g, fn.cx, fn.cy);
    if (rc) return rc;
    p.it.tx = 128;
    p.it.ty = fn.ty;
    p.it.nxb = (int)ceil_div(g.nx, 128);
    p.it.nyb = (int)ceil_div(g.ny, fn.ty);
    p.it.ncol = p.it.nxb * p.it.nyb;
    p.zlo = 0;
    p.zhi = g.nz;
    const int gmax = st::fused_grid(fn, gr->ctx->sms);
    if (gmax <= 0) return fail(ST_ERR_CUDA, "fused occupancy query failed: %s", cudaGetErrorString((cudaError_t)-gmax));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(gmax, (int64_t)p.it.ncol * g.nz));
    const int e = st::launch_fused(fn, p, grid, st);
    if (e) return fail(ST_ERR_CUDA, "fused launch failed: %s", cudaGetErrorString((cudaError_t)e));
    ++launches;
    if (f == F) ty_used = fn.ty;
    if (wave) {
      in2 = f > 1 ? o2 : in1;
      in1 = o1;
    } else {
      in1 = o1;
    }
    l += f;
  }
  arrange_levels(gr, t_begin + nsteps + dtd - 1, in1, in2);
  return ST_OK;
}

// zr (optional): per relative level, the interior plane range [lo, hi) to
// compute -- z-slab ghosts shrink level by level (st_dist_*).  Sweep
// schedules only.
static int apply_impl(st_grid* gr, int64_t t_begin, int64_t t_end, const st_plan* plan_in, int mode,
                      st_report* rep, const std::vector<std::pair<int, int>>* zr, const HostXfer* hx = nullptr);

extern "C" int st_apply(st_grid* gr, int64_t t_begin, int64_t t_end, const st_plan* plan_in, int mode,
                        st_report* rep) {
  return apply_impl(gr, t_begin, t_end, plan_in, mode, rep, nullptr);
}

// Staged (conversion-kernel) download of levels [lo, hi) into their slots.
static int download_levels(st_grid* gr, float* host, int64_t lo, int64_t hi) {
  cudaStream_t st = gr->ctx->stream;
  const size_t pbytes = sizeof(float) * (size_t)gr->ref_plane;
  for (int64_t lv = lo; lv < hi; ++lv) {
    KERN_TRY(st::launch_dev_to_ref(gr->buf[lv % gr->nbuf], gr->staging, gr->g, gr->spec.ndims, gr->refP, st));
    CUDA_TRY(cudaMemcpyAsync(host + (lv % gr->slots) * gr->ref_plane, gr->staging, pbytes,
                             cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return ST_OK;
}

extern "C" int st_execute_host(st_grid* gr, float* host, int64_t nelems, int64_t t_begin, int64_t t_end,
                               const st_plan* plan, int mode, unsigned flags, st_report* rep) {
  if (!gr || !host || !plan) return fail(ST_ERR_INVALID, "null argument");
  if (nelems != gr->slots * gr->ref_plane)
    return fail(ST_ERR_INVALID, "host grid has %lld elements, layout needs %lld", (long long)nelems,
                (long long)(gr->slots * gr->ref_plane));
  if (t_begin < 0 || t_end < t_begin)
    return fail(ST_ERR_INVALID, "bad step range [%lld, %lld)", (long long)t_begin, (long long)t_end);
  const int dtd = gr->spec.dtd;
  CUDA_TRY(cudaSetDevice(gr->ctx->device));
  const bool uniform = (flags & ST_UPLOAD_UNIFORM_HALO) || halos_uniform(gr, host);
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();   // pageable pointers report an error on some drivers
  if (!uniform || !pinned || t_end == t_begin) {
    // per-slot halos need the halo bank; pageable memory cannot be copied
    // asynchronously: the staged upload / apply / download phases
    int rc = st_grid_upload(gr, host, nelems, t_begin + dtd - 1, flags);
    if (!rc) rc = apply_impl(gr, t_begin, t_end, plan, mode, rep, nullptr);
    if (!rc) rc = download_levels(gr, host, t_end, t_end + dtd);
    return rc;
  }
  if (gr->bank) {
    cudaFree(gr->bank);
    gr->bank = nullptr;
  }
  // the input levels land inside apply_impl (upload stream)
  gr->last_level = t_begin + dtd - 1;
  gr->valid_from = t_begin;
  gr->uploaded = true;
  const HostXfer hx{host};
  return apply_impl(gr, t_begin, t_end, plan, mode, rep, nullptr, &hx);
}

static int apply_impl(st_grid* gr, int64_t t_begin, int64_t t_end, const st_plan* plan_in, int mode,
                      st_report* rep, const std::vector<std::pair<int, int>>* zr, const HostXfer* hx) {
  if (!gr) return fail(ST_ERR_INVALID, "null grid");
  if (!gr->uploaded) return fail(ST_ERR_STATE, "apply before upload");
  if (t_end < t_begin || t_begin < 0) return fail(ST_ERR_INVALID, "bad step range [%lld, %lld)",
                                                  (long long)t_begin, (long long)t_end);
  const st_stencil& s = gr->spec;
  const int dtd = s.dtd;
  if (t_begin + dtd - 1 != gr->last_level)
    return fail(ST_ERR_SLOTS, "step %lld reads levels [%lld, %lld] but the grid holds levels up to %lld",
                (long long)t_begin, (long long)t_begin, (long long)(t_begin + dtd - 1),
                (long long)gr->last_level);
  st_plan plan{};
  if (plan_in) plan = *plan_in;
  else plan.schedule = ST_SCHED_CANONICAL;
  if (plan.schedule < ST_SCHED_CANONICAL || plan.schedule > ST_SCHED_TIME)
    return fail(ST_ERR_INVALID, "unknown schedule %d", plan.schedule);
  if (plan.schedule == ST_SCHED_TIME) {
    int rc = st_check_legality(&s, &plan, nullptr);
    if (rc) return rc;
    if (plan.time_tile < 1) return fail(ST_ERR_INVALID, "time_tile %lld < 1", (long long)plan.time_tile);
  }
  for (int i = 0; i < s.ndims; ++i)
    if (plan.space_tiles[i] < 0) return fail(ST_ERR_INVALID, "negative space tile");
  if (plan.band_rows < 0 || plan.band_skew < 0) return fail(ST_ERR_INVALID, "negative band_rows / band_skew");
  const int64_t need = st_required_slots(&s, &plan);
  if (gr->slots < need)
    return fail(ST_ERR_SLOTS, "grid has %lld slots, the plan requires %lld (required_slots)",
                (long long)gr->slots, (long long)need);
  if (s.model == ST_MODEL_WAVE && !gr->has_field) return fail(ST_ERR_STATE, "wave model needs st_grid_set_field");
  if (mode != ST_MODE_REFERENCE && mode != ST_MODE_FAST) return fail(ST_ERR_INVALID, "unknown mode %d", mode);

  const int64_t nsteps = t_end - t_begin;
  st_report r{};
  r.mode_used = ST_MODE_REFERENCE;
  if (nsteps == 0) {
    if (rep) *rep = r;
    return ST_OK;
  }
  if (nsteps > (1LL << 30)) return fail(ST_ERR_INVALID, "too many steps");

  // ---- kernel and tile selection
  const DevGeom& g = gr->g;
  int R = 0;
  const bool star = canonical_star(s, R) && st::star_supported(R, s.ndims);
  st::LaunchCfg lc{};
  lc.star = star;
  lc.R = R;
  lc.dims = s.ndims;
  lc.model = s.model;
  lc.fast = star && mode == ST_MODE_FAST && symmetric_star(s, R);
  // The canonical and space-tiled schedules (all of level t before t+1) run
  // on the star kernel as ONE persistent launch with level-major tickets and
  // a time tile of 1: an item of level t+1 starts once its neighbour columns
  // of level t have the planes it reads -- the same dependences as one
  // launch per level, without 2 x nsteps launch boundaries (config 2: 508 ->
  // 644 GPts/s bit-exact, 545 -> 731 FAST).  3-D only: a 2-D level is one
  // plane, whose row items chain through the level-to-level dependence (config
  // 1: 163 per-level vs 94 persistent).  ST_CANON_SWEEP=1 restores one launch
  // per level.
  const bool persist = star && s.ndims == 3 && plan.schedule != ST_SCHED_TIME && !env_int("ST_CANON_SWEEP", 0);
  lc.wf = plan.schedule == ST_SCHED_TIME || persist;
  // plan tiles in device axes (z-chunk, y, x)
  int64_t treq[3] = {0, 0, 0};
  for (int i = 0; i < s.ndims; ++i) treq[dev_axis(s.ndims, i)] = plan.space_tiles[i];
  if (plan.schedule == ST_SCHED_CANONICAL) treq[0] = treq[1] = treq[2] = 0;
  if (persist) treq[0] = g.nz;   // whole-depth items
  st::Items it{};
  if (star) {
    // x/y CTA tile is compiled per (R, dims, model) (st::star_shape); the
    // z-chunk, time tile and skew stay runtime parameters.
    // the d_2 space tile picks the compiled CTA tile height (R = 2, 4 build
    // 8 / 16 / 32-row shapes; see st::star_shape); 0 = per-schedule default
    lc.variant = 0;
    if (s.ndims == 3 && (R == 2 || R == 4)) {
      if (treq[1] == 0) lc.variant = (lc.wf || (R == 2 && s.model != ST_MODEL_WAVE)) ? 1 : 0;
      else if (treq[1] <= 8) lc.variant = 2;
      else if (treq[1] <= 16) lc.variant = 0;
      else lc.variant = 1;
      if (s.model == ST_MODEL_WAVE && lc.variant == 1) lc.variant = 0;   // 32-row wave tile does not fit smem
      // r = 4 wave (configs 3 / 5): the 24-row tile as 12 warps x 2 rows -- three
      // consumer warps per scheduler at 128 registers instead of two at 156
      // (config 3: 371 -> 397 GPts/s, config 5: 375 -> 405, full clock).  With a
      // palettized m field the wave operand stage holds 1-byte codes (V11), which
      // frees the shared memory for a 3-plane prefetch: 407 / 423.
      if (s.model == ST_MODEL_WAVE && R == 4 && (treq[1] == 0 || treq[1] > 16))
        lc.variant = (gr->npal > 0 && gr->mcode && env_int("ST_MCODES", 1)) ? 11 : 8;
      // r = 2 heat: the 32-row tile as 8 warps x 4 rows (V4, 10 warps, 168
      // registers) beats 16 warps x 2 rows (V1, 18 warps: capped at 96
      // registers by the per-SMSP register file, spills) by 4%
      if (lc.variant == 1 && R == 2) lc.variant = 4;
      // r = 2 heat, bit-exact wavefront: the 16-row tile as 4 warps x 4 rows
      // at 2 CTAs/SM (V5) -- two independent items per SM hide the level
      // chain's latency: config 2 584 -> 637 GPts/s (FAST: no change, V4)
      if (R == 2 && s.model != ST_MODEL_WAVE && lc.wf && !lc.fast && treq[1] > 8 && treq[1] <= 16) lc.variant = 5;
      // ... and better still the 24-row tile as 12 warps x 2 rows (V8, three
      // consumer warps per scheduler): config 2 bit-exact 638 -> 700 GPts/s
      // (FAST stays on V4: 774 vs 660)
      if (R == 2 && s.model != ST_MODEL_WAVE && lc.wf && !lc.fast && (treq[1] == 0 || (treq[1] > 16 && treq[1] <= 24)))
        lc.variant = 8;
    }
    // radius 8: 12 warps x 1 row (V7) unless the plan asks for <= 8 rows
    if (s.ndims == 3 && R == 8) lc.variant = (treq[1] > 0 && treq[1] <= 8) ? 0 : 7;
    if (const char* ev = std::getenv("ST_STAR_VARIANT")) {   // tuning override
      const int v = std::atoi(ev);
      if (s.ndims == 3 && (R == 2 || R == 4) && v >= 0 && v <= 3) lc.variant = v;
      if (s.ndims == 3 && R == 4 && (v == 6 || v == 8 || v == 11)) lc.variant = v;
      if (s.ndims == 3 && R == 8 && (v == 0 || v == 7)) lc.variant = v;
      if (s.ndims == 3 && R == 2 && (v == 4 || v == 5 || v == 8) && s.model != ST_MODEL_WAVE) lc.variant = v;
    }
    const st::StarShape sh = st::star_shape(R, s.ndims, s.model, lc.variant);
    lc.bx = 32;
    lc.byt = sh.NC;
    it.tx = sh.TX;
    it.ty = sh.TY;
    lc.smem = 0;  // set with the pipeline below
  } else {
    int tx = treq[2] ? (int)std::clamp<int64_t>(ceil_div(treq[2], 32) * 32, 32, 256) : 32;
    int ty = treq[1] ? (int)std::clamp<int64_t>(treq[1], 1, 256) : (g.ny > 1 ? 8 : 1);
    lc.bx = tx;
    lc.byt = std::max(1, std::min(ty, 256 / tx));
    it.tx = tx;
    it.ty = ty;
    lc.smem = 0;
    if (it.ty < g.ry || it.tx < g.rx) {
      it.ty = std::max(it.ty, g.ry);
    }
  }
  if (it.tx < g.rx || it.ty < g.ry)
    return fail(ST_ERR_UNSUPPORTED, "tile (%d, %d) smaller than the halo", it.ty, it.tx);
  it.nyb = (int)ceil_div(g.ny, it.ty);
  it.nxb = (int)ceil_div(g.nx, it.tx);
  it.ncol = it.nyb * it.nxb;
  const int T = persist ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(plan.time_tile, nsteps));
  // on-chip time tile (plan.fused_levels): 3-D heat star, uniform halos
  int F = 0;
  if (plan.schedule == ST_SCHED_TIME && plan.fused_levels >= 1 && star && s.ndims == 3 && !zr &&
      (hx || !gr->bank) && (s.model == ST_MODEL_TERMS || gr->mfield)) {
    const int wave = s.model == ST_MODEL_WAVE;
    // deepest compiled shapes: heat r=1 F<=4, r=2 F<=3; wave r=1 F<=3, r=2 and 4 F<=2
    F = (int)std::min<int64_t>(plan.fused_levels, wave ? (R == 1 ? 3 : 2) : (R == 1 ? 4 : 3));
    if (!st::fused_lookup(R, F, (int)treq[1], lc.fast, wave).fn) F = 0;
  }
  int fused_ty = 0;
  // SM-resident 2-D time tiling (plan.fused_levels = levels per halo exchange)
  int RF = 0, res_grid = 0, res_smem = 0, res_gx = 1;
  if (plan.schedule == ST_SCHED_TIME && plan.fused_levels >= 1 && star && s.ndims == 2 &&
      s.model == ST_MODEL_TERMS && !zr && (hx || !gr->bank) && st::resident2d_supported(R))
    RF = resident_plan(gr, R, plan.fused_levels, nsteps, res_grid, res_smem, res_gx);
  const int skew = std::max(plan.skew, g.rz);
  if (lc.wf) {
    // chunk of the skewed time tile (d_1 space tile); default keeps T levels
    // of a chunk comfortably inside L2 while leaving enough items in flight
    it.cz = treq[0] > 0 ? (int)std::min<int64_t>(treq[0], g.nz + (int64_t)skew * (T - 1)) : std::min(g.nz, 64);
    it.cz = std::max(it.cz, 1);
    it.nch = (int)ceil_div((int64_t)g.nz + (int64_t)skew * (T - 1), it.cz);
    // y-chunks: keep one chunk's live set (level buffers + m field) within
    // ~1/3 of L2; plan.space_tiles[d_2] (rows) overrides.
    {
      const int64_t arrays = gr->nbuf + (gr->mfield ? 1 : 0);
      const int64_t row_bytes = (int64_t)g.pitch * 4 * arrays * it.cz;
      // default: no y-chunking (measured faster on B200 than L2-sized
      // y-chunks); `row_bytes` sizes a requested chunk.
      (void)row_bytes;
      int64_t cy_rows = (int64_t)it.nyb * it.ty;   // full-width chunks
      if (plan.band_rows > 0) cy_rows = plan.band_rows;                       // st_plan.band_rows
      if (const int ev = env_int("ST_WF_CY_ROWS", 0); ev > 0) cy_rows = ev;   // y-chunk study knob
      // row-skewed y-bands (the L2 time tile): the level with index lt in its
      // time tile runs on the tile grid shifted to rows yb*ty - ysk*lt, so a
      // band of cy tiles advances T levels while its planes are still in L2
      // and only ~4r rows per level cross a band boundary through HBM.  Legal
      // for ysk >= ry (a tile then depends on tiles <= its own index of the
      // previous level: ticket order stays topological) and 2 ry <= ty (the
      // rows a tile reads span <= 3 tiles: wait_plane's 3 x 3 watch block).
      int ysk = env_int("ST_WF_YSKEW", plan.band_rows > 0 ? std::max(plan.band_skew, 1) : 0);
      if (ysk > 0 && star && s.ndims == 3 && T > 1 && !(gr->bank && !hx) && 2 * g.ry <= it.ty) {
        ysk = std::max(ysk, g.ry);
        it.ysk = ysk;
        it.nyb = (int)ceil_div((int64_t)g.ny + (int64_t)ysk * (T - 1), it.ty);
        it.ncol = it.nyb * it.nxb;
        it.cy = (int)std::clamp<int64_t>(ceil_div(cy_rows, it.ty), 1, it.nyb);
        it.nyc = (int)ceil_div(it.nyb, it.cy);
      } else {
        it.cy = (int)std::clamp<int64_t>(ceil_div(cy_rows, it.ty), 1, it.nyb);
        it.nyc = it.cy >= it.nyb ? 1 : (int)ceil_div((int64_t)it.nyb + T - 1, it.cy);
      }
    }
    const int64_t ntiles = ceil_div(nsteps, T);
    it.ntickets = ntiles * it.nch * it.nyc * T * (int64_t)it.cy * it.nxb;
    if (it.ntickets >= (1LL << 31)) return fail(ST_ERR_UNSUPPORTED, "too many wavefront items");
  } else {
    it.cz = g.nz;  // sweep: balanced column-plane ranges per CTA
    it.nch = 1;
    it.cy = it.nyb;
    it.nyc = 1;
    it.ntickets = 0;
  }
  if ((int64_t)it.ncol * g.nz >= (1LL << 40)) return fail(ST_ERR_UNSUPPORTED, "grid too large");

  KParams* pp = new KParams;
  std::memset(pp, 0, sizeof(KParams));
  KParams& p = *pp;
  p.g = g;
  p.it = it;
  for (int b = 0; b < gr->nbuf; ++b) p.buf[b] = gr->buf[b];
  p.nbuf = gr->nbuf;
  p.dtd = dtd;
  p.mfield = gr->mfield;
  p.bank = gr->bank;
  p.bank_slots = gr->slots;
  p.level0 = t_begin + dtd;
  p.nsteps = (int)nsteps;
  p.T = T;
  p.skew = skew;
  p.sleep_pub = env_int("ST_PUB_SLEEP", 256);
  p.sleep_dep = env_int("ST_DEP_SLEEP", 256);
  p.zlo = 0;
  p.zhi = g.nz;
  if (zr && lc.wf) {   // one wavefront over the tile's levels, each on its z-slab range
    if (nsteps > st::kMaxZrLevels || !star) {
      delete pp;
      return fail(ST_ERR_UNSUPPORTED, "z-slab wavefront: at most %d levels per launch, star stencils", st::kMaxZrLevels);
    }
    p.zr_on = 1;
    for (int64_t l = 0; l < nsteps; ++l) {
      p.zr_lo[l] = std::max(0, (*zr)[l].first);
      p.zr_hi[l] = std::min(g.nz, (*zr)[l].second);
    }
  }
  if (star) {
    for (size_t k = 0; k < s.terms.size(); ++k) p.coef[k] = s.terms[k].coeff;
  }
  p.nterms = (int)s.terms.size();
  p.nzero = -0.0f;
  for (size_t k = 0; k < s.terms.size(); ++k) {
    const st_term& t = s.terms[k];
    long long o[3] = {0, 0, 0};
    for (int i = 0; i < s.ndims; ++i) o[dev_axis(s.ndims, i)] = t.offsets[i];
    p.terms[k].c = t.coeff;
    p.terms[k].dt = t.dt;
    p.terms[k].off = o[0] * g.pstride + o[1] * g.pitch + o[2];
  }

  cudaStream_t st = gr->ctx->stream;
  int rc = ST_OK;
  int64_t launches = 0;
  auto w0 = std::chrono::steady_clock::now();
  if (cudaSetDevice(gr->ctx->device) != cudaSuccess) rc = fail(ST_ERR_CUDA, "cudaSetDevice failed");
  if (!rc && star) rc = setup_pipeline(gr, R, lc, p);
  if (!rc) {
    // persistent grid: every resident CTA slot on the device
    const int grid = st::wavefront_grid(lc, gr->ctx->sms);
    if (grid <= 0) rc = fail(ST_ERR_CUDA, "occupancy query failed: %s", cudaGetErrorString((cudaError_t)-grid));
    const int64_t work = lc.wf ? it.ntickets : (int64_t)it.ncol * g.nz;
    lc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid - gr->reserve_ctas, work));
  }
  if (!star) p.pipe.unit = 1;
  p.dbg = gr->dbg_dev;
  size_t nctr = 0;
  if (lc.wf) nctr = (size_t)nsteps * it.nch * it.ncol;
  // one 128-B L2 line per progress counter: packed counters put ~150
  // pollers and the publishers on a handful of lines (measured 623 -> 687
  // GPts/s on config 2)
  p.ctr_shift = env_int("ST_CTR_SHIFT", 5);
  nctr <<= p.ctr_shift;
  if (!rc && nctr) {
    rc = ensure_counters(gr, nctr, 1);
    if (!rc) {
      p.prog = gr->prog;
      p.ticket = gr->ticket;
    }
  }
  // host-grid execute: the input levels cross PCIe on the upload stream in
  // kUpBlocks contiguous blocks; the compute stream converts each block as it
  // lands (and gives the buffers the kernel writes the uniform halo), then runs
  // the step; the download stream pulls the newest levels after it.
  st_context* cx = gr->ctx;
  if (!rc && hx) {
    const size_t nstage = (size_t)dtd * gr->ref_plane;
    if (nstage > gr->xstage_cap) {
      if (gr->xstage) cudaFree(gr->xstage);
      gr->xstage = nullptr;
      gr->xstage_cap = 0;
      if (cudaMalloc(&gr->xstage, nstage * sizeof(float)) != cudaSuccess)
        rc = fail(ST_ERR_CUDA, "transfer staging allocation failed (%zu MB)", (nstage * 4) >> 20);
      else
        gr->xstage_cap = nstage;
    }
    const int64_t Pz = (int64_t)g.nz + 2 * g.rz;
    const int64_t rowp = (int64_t)(g.ny + 2 * g.ry) * (g.nx + 2 * g.rx);   // floats per padded plane (ref)
    const int64_t zb = std::max<int64_t>(1, ceil_div(Pz, kUpBlocks));
    bool holds[st::kMaxBuffers] = {};
    for (int64_t lv = t_begin; lv < t_begin + dtd; ++lv) holds[lv % gr->nbuf] = true;
    cudaError_t e = cudaSuccess;
    // the upload must not overwrite a buffer a previous call still reads
    if (!rc) e = cudaEventRecord(cx->evx[0], st);
    if (!e) e = cudaStreamWaitEvent(cx->h2d, cx->evx[0], 0);
    for (int64_t z0 = 0, b = 0; !rc && !e && z0 < Pz; z0 += zb, ++b) {
      const int64_t z1 = std::min(Pz, z0 + zb);
      for (int64_t lv = t_begin; lv < t_begin + dtd && !e; ++lv)
        e = cudaMemcpyAsync(gr->xstage + (lv - t_begin) * gr->ref_plane + z0 * rowp,
                            hx->host + (lv % gr->slots) * gr->ref_plane + z0 * rowp,
                            sizeof(float) * (size_t)((z1 - z0) * rowp), cudaMemcpyHostToDevice, cx->h2d);
      if (!e) e = cudaEventRecord(cx->evx[1 + b], cx->h2d);
      if (!e) e = cudaStreamWaitEvent(st, cx->evx[1 + b], 0);
      for (int64_t lv = t_begin; lv < t_begin + dtd && !e; ++lv)
        e = (cudaError_t)st::launch_rows(true, gr->xstage + (lv - t_begin) * gr->ref_plane, gr->buf[lv % gr->nbuf],
                                         g, z0, z1, 4 * cx->sms, st);
      for (int bb = 0; bb < gr->nbuf && !e; ++bb)
        if (!holds[bb])
          e = (cudaError_t)st::launch_rows(true, gr->xstage + (size_t)(dtd - 1) * gr->ref_plane, gr->buf[bb], g, z0,
                                           z1, 4 * cx->sms, st, true);
      if (gr->xbuf && !e)
        e = (cudaError_t)st::launch_rows(true, gr->xstage + (size_t)(dtd - 1) * gr->ref_plane, gr->xbuf, g, z0, z1,
                                         4 * cx->sms, st, true);
    }
    if (!rc && e) rc = fail(ST_ERR_CUDA, "host-grid upload: %s", cudaGetErrorString(e));
    p.bank = nullptr;   // uniform halos: set above, never refreshed
  }
  if (!rc) {
    cudaError_t e = cudaEventRecord(gr->ctx->ev0, st);
    if (!e && RF) {
      rc = run_resident(gr, p, R, RF, res_grid, res_gx, res_smem, lc.fast, t_begin, nsteps, st, launches);
      if (rc) e = cudaErrorUnknown;
    } else if (!e && F) {
      rc = run_fused(gr, p, R, F, (int)treq[1], lc.fast, t_begin, nsteps, st, launches, fused_ty);
      if (rc) e = cudaErrorUnknown;
    } else if (!e && lc.wf) {
      e = cudaMemsetAsync(gr->prog, 0, nctr * sizeof(unsigned), st);
      if (!e) e = cudaMemsetAsync(gr->ticket, 0, sizeof(unsigned), st);
      if (!e) e = (cudaError_t)st::launch_wavefront(lc, p, st);
      launches = 1;
    } else if (!e) {
      {
        for (int64_t l = 0; l < nsteps && !e; ++l) {
          if (zr) {
            p.zlo = (*zr)[l].first;
            p.zhi = (*zr)[l].second;
            if (p.zhi <= p.zlo) continue;
          }
          e = (cudaError_t)st::launch_sweep(lc, p, (int)l, st);
          ++launches;
        }
      }
    }
    if (!e) e = cudaEventRecord(gr->ctx->ev1, st);
    if (!e && hx) {
      // newest delta_t levels back into their slots: the interior columns of
      // every row of the interior planes (the y-halo rows' interior columns
      // carry the uniform halo, identical to the host's), pitched device rows
      // -> reference rows, <= 65535 rows per 2D copy
      e = cudaEventRecord(cx->evx[0], st);
      if (!e) e = cudaStreamWaitEvent(cx->d2h, cx->evx[0], 0);
      const int64_t Px = g.nx + 2 * g.rx, Py = g.ny + 2 * g.ry;
      const int64_t nrows = (int64_t)g.nz * Py;
      for (int i = 0; i < dtd && !e; ++i) {
        const int64_t lv = t_end + i;
        float* hs = hx->host + (lv % gr->slots) * gr->ref_plane + (int64_t)g.rz * Py * Px + g.rx;
        const float* ds = gr->buf[lv % gr->nbuf] + (int64_t)g.rz * g.pstride + g.xo;
        for (int64_t r0 = 0; r0 < nrows && !e; r0 += 65535) {
          const int64_t nr = std::min<int64_t>(65535, nrows - r0);
          e = cudaMemcpy2DAsync(hs + r0 * Px, sizeof(float) * Px, ds + r0 * g.pitch, sizeof(float) * g.pitch,
                                sizeof(float) * g.nx, (size_t)nr, cudaMemcpyDeviceToHost, cx->d2h);
        }
      }
    }
    if (!e) e = cudaStreamSynchronize(st);
    if (!e && hx) e = cudaStreamSynchronize(cx->h2d);
    if (!e && hx) e = cudaStreamSynchronize(cx->d2h);
    if (!e) e = cudaGetLastError();
    if (e && !rc) {
      if (gr->dbg_host && gr->dbg_host[0])
        rc = fail(ST_ERR_CUDA, "stencil launch failed: %s (watchdog: kind %lld cta %lld thread %lld counter %lld need %lld have %lld)",
                  cudaGetErrorString(e), gr->dbg_host[1], gr->dbg_host[2], gr->dbg_host[3], gr->dbg_host[4],
                  gr->dbg_host[5], gr->dbg_host[6]);
      else
        rc = fail(ST_ERR_CUDA, "stencil launch failed: %s", cudaGetErrorString(e));
    }
  }
  auto w1 = std::chrono::steady_clock::now();
  delete pp;
  if (rc) return rc;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, gr->ctx->ev0, gr->ctx->ev1);
  r.points_updated = nsteps * (int64_t)g.nz * g.ny * g.nx;
  r.flops = r.points_updated * st_flops_per_point(&s);
  r.wall_seconds = std::chrono::duration<double>(w1 - w0).count();
  r.device_seconds = ms * 1e-3;
  r.time_tile_used = RF ? RF : (F ? F : (lc.wf ? T : 1));
  r.kernel_launches = launches;
  r.tile[0] = RF ? ceil_div(g.nz, res_grid / res_gx) : (F ? g.nz : it.cz);
  r.tile[1] = RF ? 1 : (F ? fused_ty : it.ty);
  r.tile[2] = RF ? 4 * ceil_div(ceil_div(g.nx, 4), res_gx) : (F ? 128 : it.tx);
  r.mode_used = lc.fast ? ST_MODE_FAST : ST_MODE_REFERENCE;
  r.kernel_kind = RF ? 3 : (F ? 2 : (star ? 1 : 0));
  if (rep) *rep = r;
  gr->last_level += nsteps;
  if (F || RF) gr->valid_from = gr->last_level - dtd + 1;   // intermediate levels stay on-chip
  return ST_OK;
}

// ------------------------------------------------------------ z-slabs ----
// Config 5: the global grid is split along d_1 (z) into slabs, one per GPU.
// Each rank holds a *local* grid = its slab plus ghost planes (depth
// ghost = r * T) on the sides that have a neighbour.  Once per time tile of
// T levels the delta_t newest levels' boundary planes are exchanged (NCCL
// send/recv over NVLink, or device copies in the in-process loopback
// backend used for tests); then level j of the tile is computed on the
// local planes that are still valid, [lo_j, hi_j), shrinking by r per level
// into the ghosts (overlapped / trapezoidal tiling along z).  Each exchange
// is one contiguous block per side per level (z is the slowest axis).
#include <dlfcn.h>
#include <nccl.h>

namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// NCCL is resolved at run time: the process may already hold torch's
// libnccl.so.2 (same soname), which is then reused.
const NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("/usr/lib/x86_64-linux-gnu/libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
  api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
  api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.GroupStart &&
           api.GroupEnd && api.GetErrorString;
  return api;
}
}  // namespace

struct st_dist {
  st_grid* local = nullptr;   // not owned
  int rank = 0, world = 1;
  int64_t ghost_lo = 0, ghost_hi = 0;
  ncclComm_t comm = nullptr;  // NCCL backend
  st_dist** group = nullptr;  // loopback backend: all ranks, same process
  // overlapped exchange: the ghost exchange of the next time tile runs on
  // `xs` (NCCL kernels / copy engines) while the interior runs on the grid's
  // compute stream; evb = boundary stripes done, evx = exchange done
  cudaStream_t xs = nullptr;
  cudaEvent_t evb = nullptr, evx = nullptr;
};

extern "C" int st_dist_partition(int64_t global_nz, int world, int rank, int64_t ghost, int64_t* z_begin,
                                 int64_t* z_count, int64_t* ghost_lo, int64_t* ghost_hi) {
  if (world < 1 || rank < 0 || rank >= world || global_nz < world || ghost < 0)
    return fail(ST_ERR_INVALID, "bad partition (nz %lld, world %d, rank %d)", (long long)global_nz, world, rank);
  const int64_t b = global_nz * rank / world, e = global_nz * (rank + 1) / world;
  if (ghost > e - b) return fail(ST_ERR_INVALID, "ghost depth %lld exceeds slab %lld", (long long)ghost,
                                 (long long)(e - b));
  if (z_begin) *z_begin = b;
  if (z_count) *z_count = e - b;
  if (ghost_lo) *ghost_lo = rank > 0 ? ghost : 0;
  if (ghost_hi) *ghost_hi = rank < world - 1 ? ghost : 0;
  return ST_OK;
}

extern "C" int st_nccl_unique_id(unsigned char* id128) {
  const NcclApi& api = nccl();
  if (!api.ok) return fail(ST_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(ST_ERR_NCCL, "ncclGetUniqueId: %s", api.GetErrorString(r));
  std::memcpy(id128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return ST_OK;
}

extern "C" int st_dist_create(st_grid* local, int rank, int world, const unsigned char* nccl_id,
                              int64_t ghost_lo, int64_t ghost_hi, st_dist** out) {
  if (!local || !out || world < 1 || rank < 0 || rank >= world) return fail(ST_ERR_INVALID, "bad arguments");
  if (ghost_lo < 0 || ghost_hi < 0 || ghost_lo + ghost_hi >= local->g.nz)
    return fail(ST_ERR_INVALID, "ghosts (%lld, %lld) leave no slab", (long long)ghost_lo, (long long)ghost_hi);
  auto* d = new st_dist;
  d->local = local;
  d->rank = rank;
  d->world = world;
  d->ghost_lo = ghost_lo;
  d->ghost_hi = ghost_hi;
  cudaSetDevice(local->ctx->device);
  if (cudaStreamCreateWithFlags(&d->xs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->evb, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->evx, cudaEventDisableTiming) != cudaSuccess) {
    st_dist_destroy(d);
    return fail(ST_ERR_CUDA, "dist stream / event creation failed");
  }
  if (nccl_id && world > 1) {
    const NcclApi& api = nccl();
    if (!api.ok) {
      st_dist_destroy(d);
      return fail(ST_ERR_NCCL, "libnccl.so.2 not loadable");
    }
    ncclUniqueId id;
    std::memcpy(id.internal, nccl_id, NCCL_UNIQUE_ID_BYTES);
    cudaSetDevice(local->ctx->device);
    ncclResult_t r = api.CommInitRank(&d->comm, world, id, rank);
    if (r != ncclSuccess) {
      d->comm = nullptr;
      st_dist_destroy(d);
      return fail(ST_ERR_NCCL, "ncclCommInitRank: %s", api.GetErrorString(r));
    }
  }
  *out = d;
  return ST_OK;
}

extern "C" int st_dist_link_loopback(st_dist** ranks, int world) {
  if (!ranks || world < 1) return fail(ST_ERR_INVALID, "bad arguments");
  for (int i = 0; i < world; ++i) {
    if (!ranks[i] || ranks[i]->rank != i || ranks[i]->world != world || ranks[i]->comm)
      return fail(ST_ERR_INVALID, "rank %d is not a loopback member of a world of %d", i, world);
    ranks[i]->group = ranks;
  }
  return ST_OK;
}

extern "C" void st_dist_destroy(st_dist* d) {
  if (!d) return;
  if (d->comm && nccl().ok) nccl().CommDestroy(d->comm);
  if (d->xs) cudaStreamSynchronize(d->xs);
  if (d->evb) cudaEventDestroy(d->evb);
  if (d->evx) cudaEventDestroy(d->evx);
  if (d->xs) cudaStreamDestroy(d->xs);
  delete d;
}

// Plane block [z, z + n) (interior coords, may be ghosts) of level buffer b.
static float* planes(st_grid* gr, int b, int64_t z) { return gr->buf[b] + gr->g.base - gr->g.xo - gr->g.ry * gr->g.pitch + z * gr->g.pstride; }

// Exchange the delta_t newest levels' boundary planes with the z-neighbours,
// on stream `xs` (NCCL: this rank's send/recv; loopback: device copies for
// every rank of the group).
static int dist_exchange(st_dist** ranks, int nr, cudaStream_t xs) {
  // ranks: the calling rank only (NCCL) or every rank (loopback)
  for (int i = 0; i < nr; ++i) {
    st_dist* d = ranks[i];
    st_grid* gr = d->local;
    const int dtd = gr->spec.dtd;
    const size_t blk = (size_t)gr->g.pstride;  // floats per plane
    const int64_t own_lo = d->ghost_lo, own_hi = gr->g.nz - d->ghost_hi;  // own planes [own_lo, own_hi)
    if (d->comm) {
      const NcclApi& api = nccl();
      ncclResult_t r = api.GroupStart();
      for (int64_t lv = gr->last_level - dtd + 1; r == ncclSuccess && lv <= gr->last_level; ++lv) {
        const int b = (int)(lv % gr->nbuf);
        if (d->rank > 0) {
          if (r == ncclSuccess) r = api.Send(planes(gr, b, own_lo), blk * d->ghost_lo, ncclFloat, d->rank - 1, d->comm, xs);
          if (r == ncclSuccess) r = api.Recv(planes(gr, b, 0), blk * d->ghost_lo, ncclFloat, d->rank - 1, d->comm, xs);
        }
        if (d->rank < d->world - 1) {
          if (r == ncclSuccess) r = api.Send(planes(gr, b, own_hi - d->ghost_hi), blk * d->ghost_hi, ncclFloat, d->rank + 1, d->comm, xs);
          if (r == ncclSuccess) r = api.Recv(planes(gr, b, own_hi), blk * d->ghost_hi, ncclFloat, d->rank + 1, d->comm, xs);
        }
      }
      ncclResult_t r2 = api.GroupEnd();
      if (r == ncclSuccess) r = r2;
      if (r != ncclSuccess) return fail(ST_ERR_NCCL, "halo exchange: %s", api.GetErrorString(r));
    } else if (d->group) {
      // loopback: copy my boundary planes into the neighbours' ghosts
      for (int64_t lv = gr->last_level - dtd + 1; lv <= gr->last_level; ++lv) {
        const int b = (int)(lv % gr->nbuf);
        if (d->rank > 0) {
          st_dist* n = d->group[d->rank - 1];
          st_grid* ng = n->local;
          const int nb = (int)(lv % ng->nbuf);
          CUDA_TRY(cudaMemcpyAsync(planes(ng, nb, ng->g.nz - n->ghost_hi), planes(gr, b, own_lo),
                                   sizeof(float) * blk * n->ghost_hi, cudaMemcpyDeviceToDevice, xs));
        }
        if (d->rank < d->world - 1) {
          st_dist* n = d->group[d->rank + 1];
          st_grid* ng = n->local;
          const int nb = (int)(lv % ng->nbuf);
          CUDA_TRY(cudaMemcpyAsync(planes(ng, nb, 0), planes(gr, b, own_hi - d->ghost_hi),
                                   sizeof(float) * blk * n->ghost_lo, cudaMemcpyDeviceToDevice, xs));
        }
      }
    }
  }
  return ST_OK;
}

// Steps [t_begin, t_end) on every rank listed (one for NCCL, all for the
// loopback group).  plan->time_tile = levels per exchange (ghost >= r * T).
//
// Per time tile of n levels, level j = 1..n of a slab with ghosts g below
// and above computes the trapezoid [lo_j, hi_j) (lo_j = g - r(T - j): the
// ghosts shrink by r per level, no exchange inside a tile).  The exchange
// for the NEXT tile needs only the tile's last delta_t levels on the own
// planes [g, 2g) and [own_hi - g, own_hi), whose dependency cone at level j
// is [lo_j, 2g + r(n - j)) (and its mirror).  So each tile runs
//   A: the two boundary stripes (the cones), then
//   B: the interior [2g + r(n - j), own_hi - g - r(n - j)),
// and the exchange runs on the dist's side stream as soon as A is done,
// overlapped with B.  B never touches a ghost plane and
// reads A's stripes only at levels whose buffers A no longer overwrites
// (A's range shrinks by r per level), so the split is bitwise equal to the
// single launch.  ST_DIST_SERIAL=1: exchange, then one launch per tile.
static int dist_apply_ranks(st_dist** ranks, int nr, int64_t t_begin, int64_t t_end, const st_plan* plan, int mode,
                            st_report* rep) {
  st_grid* g0 = ranks[0]->local;
  const int r = std::max(g0->g.rz, 1);
  int64_t T = plan ? std::max<int64_t>(1, plan->time_tile) : 1;
  bool neighbours = false;
  for (int i = 0; i < nr; ++i) {
    const st_dist* d = ranks[i];
    const int64_t gmin = std::min(d->ghost_lo ? d->ghost_lo : INT64_MAX, d->ghost_hi ? d->ghost_hi : INT64_MAX);
    if (gmin != INT64_MAX) T = std::min<int64_t>(T, gmin / r);
    neighbours |= d->ghost_lo > 0 || d->ghost_hi > 0;
  }
  if (T < 1) return fail(ST_ERR_INVALID, "ghost depth below the stencil radius");
  st_plan q{};
  if (plan) q = *plan;
  // time-tiled plans: one wavefront launch per time tile over the trapezoid
  // of z ranges; otherwise per-level sweeps
  q.schedule = plan && (plan->schedule == ST_SCHED_SPACE || plan->schedule == ST_SCHED_TIME) ? plan->schedule
                                                                                          : ST_SCHED_CANONICAL;
  if (q.schedule == ST_SCHED_TIME) q.time_tile = (int)T;
  const bool overlap = neighbours && q.schedule == ST_SCHED_TIME && !env_int("ST_DIST_SERIAL", 0);
  if (!neighbours) {
    // one slab, nothing to exchange: the whole range is one persistent
    // launch (time tiles of T levels inside it) instead of one launch per
    // tile -- no per-tile fill / drain of the wavefront (config 5, N = 1)
    st_report acc{};
    for (int i = 0; i < nr; ++i) {
      st_report rr{};
      const int rc = apply_impl(ranks[i]->local, t_begin, t_end, &q, mode, &rr, nullptr);
      if (rc) return rc;
      if (i == 0) {
        acc = rr;
      } else {
        acc.kernel_launches += rr.kernel_launches;
        acc.device_seconds += rr.device_seconds;
        acc.wall_seconds += rr.wall_seconds;
        acc.points_updated += rr.points_updated;
      }
    }
    acc.flops = acc.points_updated * st_flops_per_point(&g0->spec);
    if (rep) *rep = acc;
    return ST_OK;
  }
  st_report tot{};
  double dev = 0.0;
  // one launch over z ranges zr of levels t+1 .. t+n; every pass of a tile
  // starts from the tile's input levels (the split passes re-enter them)
  auto run = [&](st_dist* d, int64_t t, int64_t n, const std::vector<std::pair<int, int>>& zr) -> int {
    st_grid* gr = d->local;
    gr->last_level = t + gr->spec.dtd - 1;
    bool any = false;
    for (auto& z : zr) any |= z.second > z.first;
    if (!any) {
      gr->last_level = t + n + gr->spec.dtd - 1;
      return ST_OK;
    }
    st_report rr{};
    const int rc = apply_impl(gr, t, t + n, &q, mode, &rr, &zr);
    if (rc) return rc;
    tot.kernel_launches += rr.kernel_launches;
    tot.mode_used = rr.mode_used;
    tot.kernel_kind = rr.kernel_kind;
    for (int a = 0; a < 3; ++a) tot.tile[a] = rr.tile[a];
    tot.wall_seconds += rr.wall_seconds;
    dev += rr.device_seconds;
    return ST_OK;
  };
  // z ranges of a tile of n levels: the whole trapezoid, the two boundary
  // cones (lo / hi) and the interior (mid)
  struct Ranges {
    std::vector<std::pair<int, int>> full, lo, hi, mid;
  };
  auto ranges = [&](const st_dist* d, int64_t n) {
    Ranges z;
    const st_grid* gr = d->local;
    const int64_t own_lo = d->ghost_lo, own_hi = gr->g.nz - d->ghost_hi;
    for (int64_t j = 1; j <= n; ++j) {
      const int a = d->ghost_lo ? (int)(d->ghost_lo - r * (T - j)) : 0;
      const int b = d->ghost_hi ? (int)(gr->g.nz - d->ghost_hi + r * (T - j)) : gr->g.nz;
      const int clo = d->ghost_lo ? (int)std::min<int64_t>(b, own_lo + d->ghost_lo + r * (n - j)) : a;
      const int chi = d->ghost_hi ? (int)std::max<int64_t>(clo, own_hi - d->ghost_hi - r * (n - j)) : b;
      z.full.push_back({a, b});
      z.lo.push_back({a, clo});
      z.hi.push_back({chi, b});
      z.mid.push_back({clo, chi});
    }
    return z;
  };
  // the exchange after the stripes (or the whole tile) of every listed rank
  auto exchange = [&]() -> int {
    for (int i = 0; i < nr; ++i) CUDA_TRY(cudaEventRecord(ranks[i]->evb, ranks[i]->local->ctx->stream));
    for (int i = 0; i < nr; ++i) CUDA_TRY(cudaStreamWaitEvent(ranks[0]->xs, ranks[i]->evb, 0));
    const int rc = dist_exchange(ranks, nr, ranks[0]->xs);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(ranks[0]->evx, ranks[0]->xs));
    return ST_OK;
  };
  auto join = [&]() -> int {
    for (int i = 0; i < nr; ++i) CUDA_TRY(cudaStreamWaitEvent(ranks[i]->local->ctx->stream, ranks[0]->evx, 0));
    return ST_OK;
  };
  int rc = exchange();   // ghosts of the first tile
  if (!rc) rc = join();
  if (rc) return rc;
  for (int64_t t = t_begin; t < t_end; t += T) {
    const int64_t n = std::min<int64_t>(T, t_end - t);
    const bool more = t + n < t_end;
    std::vector<Ranges> zs;
    bool split = overlap && more;
    for (int i = 0; i < nr; ++i) {
      zs.push_back(ranges(ranks[i], n));
      // the two cones must not meet (thin slabs: one launch per tile)
      const int64_t need = (ranks[i]->ghost_lo ? r * n : 0) + (ranks[i]->ghost_hi ? r * n : 0);
      split &= zs[i].mid[0].second - zs[i].mid[0].first >= need;
    }
    for (int i = 0; i < nr; ++i) {
      st_dist* d = ranks[i];
      st_grid* gr = d->local;
      if (split) {
        if (d->ghost_lo && (rc = run(d, t, n, zs[i].lo))) return rc;
        if (d->ghost_hi && (rc = run(d, t, n, zs[i].hi))) return rc;
      } else if ((rc = run(d, t, n, zs[i].full))) {
        return rc;
      }
      tot.points_updated += n * (gr->g.nz - d->ghost_lo - d->ghost_hi) * (int64_t)gr->g.ny * gr->g.nx;
    }
    if (!more) break;
    if ((rc = exchange())) return rc;   // the next tile's ghosts, on the side stream
    if (split) {
      for (int i = 0; i < nr; ++i) {   // ... overlapped with the interiors
        st_dist* d = ranks[i];
        st_grid* gr = d->local;
        // leave CTA slots to NCCL's kernels so the exchange really overlaps
        gr->reserve_ctas = d->comm ? env_int("ST_DIST_RESERVE", 4) : 0;
        rc = run(d, t, n, zs[i].mid);
        gr->reserve_ctas = 0;
        if (rc) return rc;
      }
    }
    if ((rc = join())) return rc;
  }
  tot.flops = tot.points_updated * st_flops_per_point(&g0->spec);
  tot.device_seconds = dev;
  tot.time_tile_used = T;
  if (rep) *rep = tot;
  return ST_OK;
}

extern "C" int st_dist_apply(st_dist* d, int64_t t_begin, int64_t t_end, const st_plan* plan, int mode,
                             st_report* rep) {
  if (!d) return fail(ST_ERR_INVALID, "null dist");
  if (d->group) {
    if (d->rank != 0) return ST_OK;  // loopback: rank 0 drives the whole group
    return dist_apply_ranks(d->group, d->world, t_begin, t_end, plan, mode, rep);
  }
  return dist_apply_ranks(&d, 1, t_begin, t_end, plan, mode, rep);
}

// ------------------------------------------------------------ cache-sim --
// simulate (cache_sim.hpp:28-34): replay the nest's exact
// access stream -- per traced point every term read in term order, then the
// write -- against a fully associative LRU cache (write-allocate,
// write-back) using the reference GridLayout address map (slot-major,
// row-major padded; level l in slot l mod required_slots).  A final flush
// of dirty lines counts as write-back traffic.  The loop nests are the
// reference transforms' bounds: canonical; tile_space
// minmax (t, x_blk.., x..); tile_time (t_blk, x_blk.., t, x.., skewed by
// s*t).  A space tile of 0 means the whole extent.
namespace {
struct LruCache {
  int64_t cap_lines, line;
  std::list<std::pair<int64_t, bool>> order;   // front = most recent; (line, dirty)
  std::unordered_map<int64_t, std::list<std::pair<int64_t, bool>>::iterator> where;
  int64_t loaded = 0, written_back = 0;
  void touch(int64_t addr, bool write) {
    const int64_t ln = addr / line;
    auto it = where.find(ln);
    if (it != where.end()) {
      it->second->second = it->second->second || write;
      order.splice(order.begin(), order, it->second);
      return;
    }
    // write-allocate: a write miss allocates the (dirty) line without a
    // load (identity stencil, D=[4] -> 4 lines loaded, 4 written back)
    if (!write) ++loaded;
    if ((int64_t)order.size() == cap_lines) {
      auto& victim = order.back();
      if (victim.second) ++written_back;
      where.erase(victim.first);
      order.pop_back();
    }
    order.emplace_front(ln, write);
    where[ln] = order.begin();
  }
  void flush() {
    for (auto& e : order)
      if (e.second) ++written_back;
  }
};

// Visit every point of the nest in its execution order: body(t, x[3]).
template <class F>
int64_t visit_nest(const st_stencil& s, const int64_t* D, int64_t Dt, const st_plan& pl, int64_t cap, F&& body) {
  const int n = s.ndims;
  int64_t count = 0;
  int64_t x[3] = {0, 0, 0};
  auto emit = [&](int64_t t) {
    if (++count > cap) return false;
    body(t, x);
    return true;
  };
  if (pl.schedule == ST_SCHED_CANONICAL || pl.schedule == ST_SCHED_SPACE) {
    int64_t ts[3];
    for (int i = 0; i < n; ++i)
      ts[i] = pl.schedule == ST_SCHED_SPACE && pl.space_tiles[i] > 0 ? pl.space_tiles[i] : D[i];
    int64_t b[3] = {0, 0, 0};
    for (int64_t t = 0; t < Dt; ++t) {
      // tile loops (one iteration per dim for the canonical nest), then points
      std::function<bool(int)> tiles = [&](int i) -> bool {
        if (i == n) {
          std::function<bool(int)> pts = [&](int j) -> bool {
            if (j == n) return emit(t);
            for (x[j] = std::max<int64_t>(0, b[j]); x[j] < std::min(D[j], b[j] + ts[j]); ++x[j])
              if (!pts(j + 1)) return false;
            return true;
          };
          return pts(0);
        }
        for (b[i] = 0; b[i] < D[i]; b[i] += ts[i])
          if (!tiles(i + 1)) return false;
        return true;
      };
      if (!tiles(0)) return -1;
    }
    return count;
  }
  // tile_time
  const int64_t sk = pl.skew, T = std::max<int64_t>(1, pl.time_tile);
  int64_t ts[3], b[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i) ts[i] = pl.space_tiles[i] > 0 ? pl.space_tiles[i] : D[i] + sk * Dt;
  for (int64_t tb = 0; tb < Dt; tb += T) {
    std::function<bool(int)> tiles = [&](int i) -> bool {
      if (i == n) {
        for (int64_t t = std::max<int64_t>(0, tb); t < std::min(Dt, tb + T); ++t) {
          std::function<bool(int)> pts = [&](int j) -> bool {
            if (j == n) return emit(t);
            const int64_t lo = std::max(sk * t, b[j]), hi = std::min(D[j] + sk * t, b[j] + ts[j]);
            for (int64_t xs = lo; xs < hi; ++xs) {
              x[j] = xs - sk * t;
              if (!pts(j + 1)) return false;
            }
            return true;
          };
          if (!pts(0)) return false;
        }
        return true;
      }
      for (b[i] = 0; b[i] < D[i] + sk * Dt; b[i] += ts[i])
        if (!tiles(i + 1)) return false;
      return true;
    };
    if (!tiles(0)) return -1;
  }
  return count;
}
}  // namespace

extern "C" int st_simulate(const st_stencil* s, const int64_t* extents, int64_t time_steps, const st_plan* plan,
                           int64_t cache_elems, int64_t line_elems, int64_t cap, st_traffic* out) {
  if (!s || !extents || !plan || !out) return fail(ST_ERR_INVALID, "null argument");
  if (time_steps < 0) return fail(ST_ERR_INVALID, "negative time steps");
  if (line_elems < 1 || cache_elems < line_elems || cache_elems % line_elems)
    return fail(ST_ERR_INVALID, "cache of %lld elements is not a positive multiple of %lld-element lines",
                (long long)cache_elems, (long long)line_elems);
  if (plan->schedule < ST_SCHED_CANONICAL || plan->schedule > ST_SCHED_TIME)
    return fail(ST_ERR_INVALID, "unknown schedule %d", plan->schedule);
  for (int i = 0; i < s->ndims; ++i) {
    if (extents[i] < 1) return fail(ST_ERR_INVALID, "extent %d < 1", i);
    if (plan->space_tiles[i] < 0) return fail(ST_ERR_INVALID, "negative space tile");
  }
  if (plan->schedule == ST_SCHED_TIME) {
    const int rc = st_check_legality(s, plan, nullptr);
    if (rc) return rc;
  }
  // reference GridLayout (executor.hpp:12-41)
  const int n = s->ndims;
  int64_t P[3] = {1, 1, 1};
  ref_padded(s, extents, P);
  int64_t plane = 1;
  for (int i = 0; i < n; ++i) plane *= P[i];
  const int64_t slots = st_required_slots(s, plan);
  LruCache c{cache_elems / line_elems, line_elems, {}, {}, 0, 0};
  c.where.reserve((size_t)std::min<int64_t>(cache_elems / line_elems, 1 << 22) * 2);
  auto offset = [&](int64_t level, const int64_t* x, const int* off) {
    int64_t a = 0;
    for (int i = 0; i < n; ++i) a = a * P[i] + (x[i] + off[i] + s->radii[i]);
    return (level % slots) * plane + a;
  };
  const int zero[3] = {0, 0, 0};
  const int64_t pts = visit_nest(*s, extents, time_steps, *plan, cap, [&](int64_t t, const int64_t* x) {
    const int64_t lw = t + s->dtd;   // step t writes level t + delta_t
    for (const st_term& tm : s->terms) c.touch(offset(lw - tm.dt, x, tm.offsets), false);
    c.touch(offset(lw, x, zero), true);
  });
  if (pts < 0) return fail(ST_ERR_INVALID, "trace cap of %lld points exceeded", (long long)cap);
  c.flush();
  st_traffic r{};
  r.lines_loaded = c.loaded;
  r.lines_written_back = c.written_back;
  r.line_elems = line_elems;
  r.bytes = 4 * line_elems * (c.loaded + c.written_back);
  r.flops = pts * (2 * (int64_t)s->terms.size() - 1);
  r.measured_ai = r.bytes > 0 ? (double)r.flops / (double)r.bytes : 0.0;
  *out = r;
  return ST_OK;
}
