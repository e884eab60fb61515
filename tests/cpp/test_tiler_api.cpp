// C++ client of the drop-in API (include/tiler_gpu.hpp), written the way a
// reference caller uses namespace tiler: parse a spec, build
// canonical and time-tiled nests, init grids, execute, verify_bitwise.
// Host-only checks always run; `--gpu` also executes on device 0.
#include <cstdio>
#include <cstring>
#include <string>

#include "tiler_gpu.hpp"

using namespace tiler::gpu;

#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                     \
    }                                                               \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  // parse_spec examples
  auto ps = parse_spec("stencil s\ndims 1\nextent 8\nsteps 4\nterm 1.0 1 0\n");
  EXPECT(ps.spec.ndims() == 1 && ps.spec.time_depth() == 1 && ps.spec.radii()[0] == 0);
  EXPECT(ps.space.time_steps == 4 && ps.space.extents[0] == 8);
  auto ps2 = parse_spec("stencil s\ndims 1\nextent 8\nsteps 4\nterm 0.5 1 -1\nterm 0.5 1 1\n");
  EXPECT(ps2.spec.radii()[0] == 1);
  bool threw = false;
  try {
    parse_spec("stencil s\ndims 1\nextent 8\nsteps 4\nterm 1.0 0 0\n");
  } catch (const ParseError& e) {
    threw = e.line() == 5;
  }
  EXPECT(threw);
  // derived quantities
  auto s3 = StencilSpec::make("s3", 3, {{0.1f, 1, {2, 0, 0}}, {0.1f, 1, {0, 1, 0}}, {0.1f, 2, {0, 0, -2}}});
  EXPECT(min_skew_factor(s3) == 2 && s3.time_depth() == 2 && flops_per_point(s3) == 5);
  EXPECT(time_buffer_slots(s3, 16) == 18);
  EXPECT(check_legality(s3, TilePlan{2, 2, {4, 4, 4}}) == std::nullopt);
  EXPECT(check_legality(s3, TilePlan{1, 2, {4, 4, 4}})->required_minimum == 2);
  threw = false;
  try {
    tile_time(build_canonical_nest(s3, {}), s3, {}, TilePlan{1, 2, {4, 4, 4}});
  } catch (const Error& e) {
    threw = e.code() == ST_ERR_ILLEGAL_PLAN;
  }
  EXPECT(threw);
  // 2D diffusion, reference flow
  auto lap = parse_spec(
      "stencil lap\ndims 2\nextent 37 61\nsteps 11\n"
      "term 0.6 1 0 0\nterm 0.1 1 -1 0\nterm 0.1 1 1 0\nterm 0.1 1 0 -1\nterm 0.1 1 0 1\n");
  auto canon = build_canonical_nest(lap.spec, lap.space);
  auto tt = tile_time(canon, lap.spec, lap.space, TilePlan{min_skew_factor(lap.spec), 4, {8, 8}});
  EXPECT(required_slots(canon, lap.spec) == 2 && required_slots(tt, lap.spec) == 5);
  Grid a = init_grid(lap.spec, lap.space, 7, required_slots(canon, lap.spec));
  Grid b = init_grid(lap.spec, lap.space, 7, required_slots(tt, lap.spec));
  EXPECT(a.data[0] > 0.001f && a.data[0] < 0.002f && a.last_level == 0);
  // verify_bitwise(a, b, levels) with the reference signature (executor.hpp:110)
  EXPECT(verify_bitwise(a, b, 1));
  {
    Grid d = a;
    d.data[a.layout.plane() * (a.last_level % a.layout.slots) + 4 * (61 + 2) + 7] += 1e-3f;
    EXPECT(!verify_bitwise(a, d, 1));
    threw = false;
    try {
      verify_bitwise(a, b, 3);   // more levels than a canonical grid retains
    } catch (const Error& e) {
      threw = e.code() == ST_ERR_SLOTS;
    }
    EXPECT(threw);
  }
  if (!gpu) {
    std::printf("host checks ok\n");
    return 0;
  }
  // uniform halos so different slot counts are comparable (DESIGN.md ledger)
  for (Grid* g : {&a, &b}) {
    const auto P = g->layout.padded;
    for (std::int64_t s = 1; s < g->layout.slots; ++s)
      for (std::int64_t y = 0; y < P[0]; ++y)
        for (std::int64_t x = 0; x < P[1]; ++x)
          if (y == 0 || x == 0 || y == P[0] - 1 || x == P[1] - 1)
            g->data[s * g->layout.plane() + y * P[1] + x] = g->data[y * P[1] + x];
  }
  Grid c = b;   // for the host-grid entry point below
  Grid f = b;   // for the on-chip realisation below
  auto ra = execute(canon, lap.spec, lap.space, a);   // executor.hpp:96-98 signature, default options
  ExecOptions rev;
  rev.reverse_parallel = true;                        // accepted; bitwise-neutral by contract
  auto rb = execute(tt, lap.spec, lap.space, b, rev);
  EXPECT(ra.points_updated == 11 * 37 * 61 && rb.points_updated == ra.points_updated);
  EXPECT(ra.flops == ra.points_updated * flops_per_point(lap.spec));
  EXPECT(verify_bitwise(lap.spec, a, b, 1) && verify_bitwise(a, b, 1));
  {  // st_execute_host: execute on the host grid through the C-ABI
    Device dev(0);
    st_grid* g = nullptr;
    check(st_grid_create(dev.handle(), lap.spec.handle(), lap.space.extents.data(), c.layout.slots, &g));
    st_plan q = to_plan(tt.schedule, tt.plan);
    st_report r{};
    const int rc = st_execute_host(g, c.data.data(), static_cast<std::int64_t>(c.data.size()), 0,
                                   lap.space.time_steps, &q, ST_MODE_REFERENCE, ST_UPLOAD_UNIFORM_HALO, &r);
    st_grid_destroy(g);
    check(rc);
    c.last_level = lap.space.time_steps;
    EXPECT(r.points_updated == ra.points_updated);
    EXPECT(verify_bitwise(lap.spec, a, c, 1));
  }
  {  // the same time tile realised on-chip (TilePlan::fused_levels): the 2-D
     // grid stays SM-resident, one halo exchange per 4 levels
    TilePlan fp{min_skew_factor(lap.spec), 4, {0, 0}};
    fp.fused_levels = 4;
    auto tf = tile_time(canon, lap.spec, lap.space, fp);
    auto rf = execute(tf, lap.spec, lap.space, f);
    EXPECT(rf.detail.kernel_kind == 3 && rf.detail.kernel_launches == 1);
    EXPECT(verify_bitwise(lap.spec, a, f, 1));
  }
  b.data[b.layout.plane() * (b.last_level % b.layout.slots) + 3 * (61 + 2) + 5] += 1e-3f;
  EXPECT(!verify_bitwise(lap.spec, a, b, 1));
  std::printf("gpu checks ok (%lld updates, %.3f ms device)\n", (long long)rb.points_updated,
              rb.detail.device_seconds * 1e3);
  return 0;
}
