/*
 * oracle.h -- CPU restatement of the reference stencil executor.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker and the
 * CPU baseline; it is loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, never by the product
 * path (paper_1806_08299_b200/).
 *
 * It restates, from the reference headers and spec (the reference ships
 * declarations only; every non-inline definition is absent):
 *   - GridLayout address map          executor.hpp:12-41
 *   - LcgStream / init_grid           executor.hpp:70-90
 *   - required_slots                  executor.hpp:83-85
 *   - execute (fp32, in-order, no FMA) executor.hpp:92-98
 *   - execute_group (remainder mode)  executor.hpp:100-105, transforms.hpp:35-41
 *   - canonical nest                  loop_ir.hpp:111-114
 *   - tile_space_minmax bounds        transforms.hpp:29-33
 *   - tile_time bounds + legality     transforms.hpp:43-59
 *   - mark_parallel placement         transforms.hpp:61-66
 *   - verify_bitwise                  executor.hpp:107-110
 *   - FP contract (-ffp-contract=off) proj/CMakeLists.txt:12-13
 * plus the ledger extensions of SURVEY.md Appendix A (wave model with a
 * per-point m field, [0,1) interior init, Gaussian pulse, velocity models).
 *
 * Parity pins: LcgStream is inline in the reference (executor.hpp:73-81);
 * oracle/ref_golden.sh compiles it from /root/reference and the vectors are
 * committed in tests/golden/.  Field values have no reference goldens
 * (SURVEY.md 8c): they are pinned by this restatement plus the
 * schedule-invariance properties the spec states.
 *
 * All grids use the reference layout: slot-major, then row-major over the
 * halo-padded box, last axis contiguous.  n < 3 dims are embedded as 3D with
 * leading extents 1 and radius 0 (identical memory layout).
 */
#ifndef STENCIL_ORACLE_H
#define STENCIL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_MODEL_TERMS = 0, OR_MODEL_WAVE = 1 };
enum {
  OR_SCHED_CANONICAL = 0,   /* build_canonical_nest            */
  OR_SCHED_SPACE = 1,       /* tile_space_minmax               */
  OR_SCHED_TIME = 2,        /* tile_time (skew + min/max)      */
  OR_SCHED_REMAINDER = 3    /* tile_space_remainder + execute_group */
};
enum { OR_OK = 0, OR_EINVAL = 1, OR_EILLEGAL = 2, OR_ESLOTS = 3 };

typedef struct {
  float coeff;
  int dt;
  int off[3]; /* offsets[0..ndims), rest ignored */
} or_term;

typedef struct {
  int ndims;            /* 1..3 */
  int model;            /* OR_MODEL_* */
  int nterms;
  const or_term* terms; /* spec order = evaluation order */
} or_spec;

/* Derived quantities (stencil.hpp:56-57, 99-108). Returns OR_EINVAL on a
 * violated invariant (no terms, dt<1, bad ndims, wave terms with dt!=1). */
int or_time_depth(const or_spec* s);
int or_radius(const or_spec* s, int dim);
int64_t or_flops_per_point(const or_spec* s);
int or_validate(const or_spec* s);

/* Layout (executor.hpp:17-41) */
int64_t or_plane(const or_spec* s, const int64_t* extents);

/* Inits.  grid has slots*plane floats; levels [0, time_depth) filled. */
void or_init_reference(const or_spec* s, const int64_t* extents, float* grid,
                       int64_t slots, uint64_t seed);
void or_init_unit(const or_spec* s, const int64_t* extents, float* grid,
                  int64_t slots, uint64_t seed);
void or_init_gaussian(const or_spec* s, const int64_t* extents, float* grid,
                      int64_t slots, double sigma, const int64_t* centre);
/* m field (interior only, row-major D_1..D_n) */
void or_mfield_layered(int ndims, const int64_t* extents, float* m,
                       double v_top, double v_bottom, int64_t split, double dt,
                       double h);
void or_mfield_random_smoothed(int ndims, const int64_t* extents, float* m,
                               uint64_t seed, double vmin, double vmax,
                               double dt, double h);
/* LCG known-answer helper: n values of LcgStream(seed).next() */
void or_lcg_reference(uint64_t seed, int64_t n, float* out);

/* Legality (transforms.hpp:50): returns 0 if ok else the required minimum */
int or_check_legality(const or_spec* s, int skew, int* required_min);

/* execute over steps [t_begin, t_end): step t writes level t + delta_t into
 * slot (t + delta_t) mod slots.  tiles: one per dim (spatial / time-tiled).
 * nthreads: OpenMP threads for the parallel-marked loop (1 = sequential).
 * reverse_parallel: iterate the parallel-marked loop in reverse, sequentially
 * (executor.hpp:64-68).  Returns OR_* status. */
int or_execute(const or_spec* s, const int64_t* extents, float* grid,
               int64_t slots, int64_t t_begin, int64_t t_end,
               const float* mfield, int schedule, int skew, int64_t time_tile,
               const int64_t* tiles, int reverse_parallel, int nthreads,
               double* wall_seconds, int64_t* points_updated);

/* verify_bitwise over the interior of the last compare_levels levels
 * ending at last_level.  Returns 1 equal, 0 differ, <0 error. */
int or_verify_bitwise(const or_spec* s, const int64_t* extents,
                      const float* a, int64_t slots_a, const float* b,
                      int64_t slots_b, int64_t last_level,
                      int64_t compare_levels);
/* max|a-b| / max|a| over the same levels (a = oracle) */
double or_max_rel_err(const or_spec* s, const int64_t* extents, const float* a,
                      int64_t slots_a, const float* b, int64_t slots_b,
                      int64_t last_level, int64_t compare_levels);

#ifdef __cplusplus
}
#endif
#endif
