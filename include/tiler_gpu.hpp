// tiler_gpu.hpp -- C++ mirror of the reference operator API (namespace
// tiler, /root/reference/proj/include/tiler/*.hpp) executed on the B200
// through the C-ABI of stencil_tiler.h.  Header-only; link
// paper_1806_08299_b200/libstencil_tiler.so.
//
// Reference -> here (same names, argument meaning and error behaviour):
//   tiler::Error / ParseError            stencil.hpp:11-26   tiler::gpu::Error / ParseError
//   StencilTerm, StencilSpec::make       stencil.hpp:42-63   StencilTerm, StencilSpec::make
//   IterationSpace, TilePlan             stencil.hpp:28-40,65-70
//   parse_spec                           stencil.hpp:87-97
//   min_skew_factor / time_buffer_slots
//   / flops_per_point                    stencil.hpp:99-108
//   build_canonical_nest                 loop_ir.hpp:111-114 (schedule descriptor)
//   tile_space_minmax / tile_time        transforms.hpp:29-59 (schedule descriptors)
//   check_legality                       transforms.hpp:43-51
//   GridLayout, Grid                     executor.hpp:17-56
//   required_slots, init_grid            executor.hpp:83-90
//   execute                              executor.hpp:92-98
//   verify_bitwise                       executor.hpp:107-110
//
// The reference's LoopNest is an IR the CPU interpreter walks; the GPU
// realises the schedule directly, so a LoopNest here is a descriptor
// {schedule, TilePlan}.  Results are bit-identical to the reference
// interpreter for every legal plan (Mode::Reference).
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "stencil_tiler.h"

namespace tiler::gpu {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m, int code = ST_ERR_INVALID) : std::runtime_error(m), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

class ParseError : public Error {
 public:
  ParseError(int line, const std::string& msg) : Error(msg, ST_ERR_PARSE), line_(line) {}
  int line() const { return line_; }

 private:
  int line_;
};

inline void check(int rc) {
  if (rc != ST_OK) throw Error(st_last_error(), rc);
}

struct IterationSpace {
  std::int64_t time_steps = 1;
  std::vector<std::int64_t> extents;
  int ndims() const { return static_cast<int>(extents.size()); }
  std::int64_t points_per_step() const {
    std::int64_t p = 1;
    for (auto e : extents) p *= e;
    return p;
  }
};

struct StencilTerm {
  float coeff = 0.0f;
  int dt = 1;
  std::vector<int> offsets;
};

struct TilePlan {
  int skew = 0;
  std::int64_t time_tile = 1;
  std::vector<std::int64_t> space_tiles;
  std::int64_t fused_levels = 0;   // executor extension: st_plan.fused_levels
  std::int64_t band_rows = 0;      // executor extension: st_plan.band_rows (tile_time along d_2)
  int band_skew = 0;               // ... rows of skew per level (0 = the radius)
};

struct LegalityViolation {
  int skew = 0;
  int required_minimum = 0;
};

enum class Model { Terms = ST_MODEL_TERMS, Wave = ST_MODEL_WAVE };
enum class Mode { Reference = ST_MODE_REFERENCE, Fast = ST_MODE_FAST };

class StencilSpec {
 public:
  std::string name;

  static StencilSpec make(std::string name, int ndims, const std::vector<StencilTerm>& terms,
                          Model model = Model::Terms) {
    std::vector<st_term> t(terms.size());
    for (size_t k = 0; k < terms.size(); ++k) {
      t[k].coeff = terms[k].coeff;
      t[k].dt = terms[k].dt;
      for (int i = 0; i < ST_MAX_DIMS; ++i)
        t[k].offsets[i] = i < static_cast<int>(terms[k].offsets.size()) ? terms[k].offsets[i] : 0;
      if (static_cast<int>(terms[k].offsets.size()) != ndims)
        throw Error("term " + std::to_string(k + 1) + ": offset arity != ndims");
    }
    st_stencil* h = nullptr;
    check(st_stencil_create(name.c_str(), ndims, t.data(), static_cast<int>(t.size()),
                            static_cast<int>(model), &h));
    return StencilSpec(h, std::move(name));
  }

  int ndims() const { return st_stencil_ndims(h_.get()); }
  int time_depth() const { return st_stencil_time_depth(h_.get()); }
  std::vector<int> radii() const {
    std::vector<int> r;
    for (int i = 0; i < ndims(); ++i) r.push_back(st_stencil_radius(h_.get(), i));
    return r;
  }
  std::vector<StencilTerm> terms() const {
    std::vector<StencilTerm> out;
    for (int k = 0; k < st_stencil_nterms(h_.get()); ++k) {
      st_term t;
      check(st_stencil_term(h_.get(), k, &t));
      out.push_back({t.coeff, t.dt, std::vector<int>(t.offsets, t.offsets + ndims())});
    }
    return out;
  }
  Model model() const { return static_cast<Model>(st_stencil_model(h_.get())); }
  const st_stencil* handle() const { return h_.get(); }

  StencilSpec(st_stencil* h, std::string n) : name(std::move(n)), h_(h, &st_stencil_destroy) {}

 private:
  std::shared_ptr<st_stencil> h_;
};

struct ParsedStencil {
  StencilSpec spec;
  IterationSpace space;
};

inline ParsedStencil parse_spec(std::string_view text) {
  std::string s(text);
  st_stencil* h = nullptr;
  int nd = 0, line = 0;
  std::int64_t ext[ST_MAX_DIMS], steps = 0;
  int rc = st_stencil_parse(s.c_str(), &h, &nd, ext, &steps, &line);
  if (rc == ST_ERR_PARSE) throw ParseError(line, st_last_error());
  check(rc);
  return {StencilSpec(h, ""), IterationSpace{steps, std::vector<std::int64_t>(ext, ext + nd)}};
}

inline int min_skew_factor(const StencilSpec& s) { return st_min_skew_factor(s.handle()); }
inline std::int64_t time_buffer_slots(const StencilSpec& s, std::int64_t t_t) {
  return st_time_buffer_slots(s.handle(), t_t);
}
inline std::int64_t flops_per_point(const StencilSpec& s) { return st_flops_per_point(s.handle()); }

inline st_plan to_plan(int schedule, const TilePlan& p) {
  st_plan q{};
  q.schedule = schedule;
  q.skew = p.skew;
  q.time_tile = p.time_tile;
  for (size_t i = 0; i < p.space_tiles.size() && i < ST_MAX_DIMS; ++i) q.space_tiles[i] = p.space_tiles[i];
  q.fused_levels = p.fused_levels;
  q.band_rows = p.band_rows;
  q.band_skew = p.band_skew;
  return q;
}

inline std::optional<LegalityViolation> check_legality(const StencilSpec& s, const TilePlan& p) {
  st_plan q = to_plan(ST_SCHED_TIME, p);
  int req = 0;
  int rc = st_check_legality(s.handle(), &q, &req);
  if (rc == ST_OK) return std::nullopt;
  if (rc == ST_ERR_ILLEGAL_PLAN) return LegalityViolation{p.skew, req};
  check(rc);
  return std::nullopt;
}

// Schedule descriptor standing in for the reference LoopNest.
struct LoopNest {
  int schedule = ST_SCHED_CANONICAL;
  TilePlan plan;
};

inline LoopNest build_canonical_nest(const StencilSpec&, const IterationSpace&) { return {}; }

inline LoopNest tile_space_minmax(const LoopNest& nest, const std::vector<std::int64_t>& sizes) {
  if (nest.schedule != ST_SCHED_CANONICAL) throw Error("tile_space_minmax: the nest must be canonical");
  for (auto t : sizes)
    if (t < 0) throw Error("tile size < 1");
  return {ST_SCHED_SPACE, TilePlan{0, 1, sizes}};
}

inline LoopNest tile_time(const LoopNest& nest, const StencilSpec& spec, const IterationSpace&,
                          const TilePlan& plan) {
  if (nest.schedule != ST_SCHED_CANONICAL) throw Error("tile_time: the nest must be canonical");
  if (auto v = check_legality(spec, plan))
    throw Error("illegal plan: skew " + std::to_string(v->skew) + " < minimum skew factor " +
                    std::to_string(v->required_minimum),
                ST_ERR_ILLEGAL_PLAN);
  return {ST_SCHED_TIME, plan};
}

inline std::int64_t required_slots(const LoopNest& nest, const StencilSpec& spec) {
  st_plan q = to_plan(nest.schedule, nest.plan);
  return st_required_slots(spec.handle(), &q);
}

struct GridLayout {
  std::int64_t slots = 0;
  int time_depth = 0;
  std::vector<std::int64_t> interior;
  std::vector<int> halo;
  std::vector<std::int64_t> padded;

  static GridLayout make(const StencilSpec& spec, const IterationSpace& space, std::int64_t slots) {
    GridLayout g;
    g.slots = slots;
    g.time_depth = spec.time_depth();
    g.interior = space.extents;
    g.halo = spec.radii();
    for (size_t i = 0; i < g.interior.size(); ++i) g.padded.push_back(g.interior[i] + 2 * g.halo[i]);
    return g;
  }
  std::int64_t plane() const {
    std::int64_t p = 1;
    for (auto e : padded) p *= e;
    return p;
  }
  std::int64_t total_elems() const { return slots * plane(); }
};

struct Grid {
  GridLayout layout;
  std::vector<float> data;
  std::int64_t last_level = 0;
};

struct ExecReport {
  std::int64_t points_updated = 0;
  std::int64_t flops = 0;
  double wall_seconds = 0.0;
  st_report detail{};
};

inline Grid init_grid(const StencilSpec& spec, const IterationSpace& space, std::uint64_t seed, std::int64_t slots) {
  Grid g;
  g.layout = GridLayout::make(spec, space, slots);
  g.data.assign(static_cast<size_t>(g.layout.total_elems()), 0.0f);
  check(st_init_reference(spec.handle(), space.extents.data(), g.data.data(), slots, seed));
  g.last_level = spec.time_depth() - 1;
  return g;
}

// A device (context); execute() creates one per call if none is given.
class Device {
 public:
  explicit Device(int ordinal = 0) {
    st_context* c = nullptr;
    check(st_context_create(ordinal, &c));
    c_.reset(c, &st_context_destroy);
  }
  st_context* handle() const { return c_.get(); }

 private:
  std::shared_ptr<st_context> c_;
};

// ExecOptions (executor.hpp:64-68) plus the GPU extensions.  reverse_parallel
// is accepted and has no effect: the GPU realises every schedule bitwise
// equal to the canonical one whatever order the parallel tiles run in, which
// is exactly the property the reference checks with it.
struct ExecOptions {
  bool reverse_parallel = false;
  Mode mode = Mode::Reference;                 // FAST: re-associated symmetric taps + FFMA
  const std::vector<float>* field = nullptr;   // wave model coefficient field m
  const Device* device = nullptr;              // default: a context on device 0
};

// execute (executor.hpp:92-98): the nest's schedule over steps [0, D_t) of
// `space`, in place on `grid`, on the GPU.  `field` is the wave model's m.
inline ExecReport execute(const LoopNest& nest, const StencilSpec& spec, const IterationSpace& space, Grid& grid,
                          Mode mode, const std::vector<float>* field = nullptr,
                          const Device* dev = nullptr) {
  std::optional<Device> own;
  if (!dev) dev = &own.emplace(0);
  if (grid.layout.slots < required_slots(nest, spec))
    throw Error("insufficient slots for the nest", ST_ERR_SLOTS);
  st_grid* g = nullptr;
  check(st_grid_create(dev->handle(), spec.handle(), space.extents.data(), grid.layout.slots, &g));
  std::unique_ptr<st_grid, void (*)(st_grid*)> guard(g, &st_grid_destroy);
  check(st_grid_upload(g, grid.data.data(), static_cast<std::int64_t>(grid.data.size()), grid.last_level, 0));
  if (spec.model() == Model::Wave) {
    if (!field) throw Error("wave model needs a coefficient field", ST_ERR_STATE);
    check(st_grid_set_field(g, field->data(), static_cast<std::int64_t>(field->size())));
  }
  st_plan q = to_plan(nest.schedule, nest.plan);
  st_report r{};
  const std::int64_t t0 = grid.last_level - spec.time_depth() + 1;
  check(st_apply(g, t0, t0 + space.time_steps, &q, static_cast<int>(mode), &r));
  check(st_grid_download(g, grid.data.data(), static_cast<std::int64_t>(grid.data.size()), &grid.last_level));
  return {r.points_updated, r.flops, r.wall_seconds, r};
}

// The reference signature (executor.hpp:96-98).
inline ExecReport execute(const LoopNest& nest, const StencilSpec& spec, const IterationSpace& space, Grid& grid,
                          const ExecOptions& options = {}) {
  return execute(nest, spec, space, grid, options.mode, options.field, options.device);
}

// verify_bitwise (executor.hpp:110): the grids carry their layout.
inline bool verify_bitwise(const Grid& a, const Grid& b, std::int64_t compare_levels) {
  if (a.layout.interior != b.layout.interior || a.layout.halo != b.layout.halo)
    throw Error("verify_bitwise: shape mismatch");
  if (a.last_level != b.last_level) return false;
  std::vector<std::int64_t> radii(a.layout.halo.begin(), a.layout.halo.end());
  int eq = 0;
  check(st_verify_bitwise_layout(static_cast<int>(a.layout.interior.size()), a.layout.interior.data(), radii.data(),
                                 a.data.data(), a.layout.slots, b.data.data(), b.layout.slots, a.last_level,
                                 compare_levels, &eq));
  return eq != 0;
}

inline bool verify_bitwise(const StencilSpec& spec, const Grid& a, const Grid& b, std::int64_t compare_levels) {
  if (a.layout.interior != b.layout.interior) throw Error("verify_bitwise: shape mismatch");
  if (a.last_level != b.last_level) return false;
  int eq = 0;
  check(st_verify_bitwise(spec.handle(), a.layout.interior.data(), a.data.data(), a.layout.slots, b.data.data(),
                          b.layout.slots, a.last_level, compare_levels, &eq));
  return eq != 0;
}

}  // namespace tiler::gpu
