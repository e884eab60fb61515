/*
 * stencil_tiler.h -- C-ABI of the B200 stencil executor.
 *
 * Drop-in boundary for the reference's executor path (namespace tiler,
 * /root/reference/proj/include/tiler/).  Plain C types only: no exceptions,
 * no torch, no STL.  Every entry point returns an st_status (0 = ST_OK) and
 * leaves a thread-local message for st_last_error() on failure -- the
 * reference's `tiler::Error` / `ParseError(line)` (stencil.hpp:11-26)
 * become ST_ERR_* codes.  One st_context = one device + one stream; a
 * context is not re-entrant (the reference's execute is sequential by
 * contract); independent contexts may run concurrently.
 *
 * Entry point  -> reference interface it replaces
 *   st_stencil_create       StencilSpec::make            stencil.hpp:59-62
 *   st_stencil_parse        parse_spec                   stencil.hpp:87-97
 *   st_stencil_time_depth   StencilSpec::time_depth      stencil.hpp:56
 *   st_stencil_radius       StencilSpec::radii           stencil.hpp:57
 *   st_min_skew_factor      min_skew_factor              stencil.hpp:99-100
 *   st_time_buffer_slots    time_buffer_slots            stencil.hpp:102-105
 *   st_flops_per_point      flops_per_point              stencil.hpp:107-108
 *   st_check_legality       check_legality               transforms.hpp:43-51
 *   st_required_slots       required_slots               executor.hpp:83-85
 *   st_layout_plane         GridLayout::plane            executor.hpp:27-31
 *   st_init_reference       init_grid (+ LcgStream)      executor.hpp:70-90
 *   st_grid_create/upload   Grid (device copy)           executor.hpp:43-56
 *   st_apply                execute / execute_group      executor.hpp:92-105
 *                           over a tile_time /
 *                           tile_space_minmax plan       transforms.hpp:29-59
 *   st_grid_download        Grid (host view)             executor.hpp:43-56
 *   st_execute_host         execute on a host Grid       executor.hpp:92-98
 *   st_verify_bitwise       verify_bitwise               executor.hpp:107-110
 *
 * Extensions the reference lacks: the wave model
 * (ST_MODEL_WAVE, per-point coefficient field m), the [0,1)/Gaussian/
 * velocity initialisers, t_begin (resume from last_level) and z-slab
 * decomposition over several GPUs (st_dist_*).
 */
#ifndef STENCIL_TILER_H
#define STENCIL_TILER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ST_MAX_DIMS 3
#define ST_MAX_TERMS 128

typedef enum {
  ST_OK = 0,
  ST_ERR_INVALID = 1,       /* violated invariant (tiler::Error)            */
  ST_ERR_ILLEGAL_PLAN = 2,  /* skew < min_skew_factor (check_legality)      */
  ST_ERR_SLOTS = 3,         /* insufficient / missing slots or levels       */
  ST_ERR_CUDA = 4,          /* CUDA runtime failure                         */
  ST_ERR_NCCL = 5,          /* NCCL failure                                 */
  ST_ERR_UNSUPPORTED = 6,   /* outside the built kernel set                 */
  ST_ERR_PARSE = 7,         /* parse_spec failure (tiler::ParseError)       */
  ST_ERR_STATE = 8          /* call out of order (e.g. apply before upload) */
} st_status;

typedef enum {
  ST_MODEL_TERMS = 0,  /* A[t] = sum_k c_k A[t-dt_k][x+off_k] (reference)   */
  ST_MODEL_WAVE = 1    /* u' = (2u - u_prev) + m * sum_k c_k u[x+off_k]     */
} st_model;

typedef enum {
  ST_MODE_REFERENCE = 0, /* bit-identical to the reference (no FMA)       */
  ST_MODE_FAST = 1       /* <= 1e-5 rel error over the BASELINE runs: FFMA +
                          * symmetric pairing; for the radius-4 leapfrog the
                          * reference's summation order with only the products
                          * of the taps at distance >= 2 fused */
} st_mode;

typedef enum {
  ST_SCHED_CANONICAL = 0, /* build_canonical_nest                          */
  ST_SCHED_SPACE = 1,     /* tile_space_minmax                             */
  ST_SCHED_TIME = 2       /* tile_time: skewed wavefront, T levels in flight */
} st_schedule;

typedef struct {
  float coeff;
  int dt;                      /* >= 1 (stencil.hpp:43)                    */
  int offsets[ST_MAX_DIMS];    /* offsets[0..ndims) used                   */
} st_term;

/* TilePlan (stencil.hpp:65-70) + which nest it tiles.  space_tiles[i] is
 * the tile extent of reference dimension i (0 = let the executor choose).
 * For ST_SCHED_TIME, skew is the wavefront lag between consecutive levels
 * along d_1 (legal iff >= max_i delta_i) and time_tile is the number of
 * levels kept in flight (the time tile t_t).
 * fused_levels (executor extension, 0 = off): for ST_SCHED_TIME, advance F
 * levels on-chip per pass over memory (overlapped x/y tiles with redundant
 * halo compute, trapezoidal z ranges) instead of the wavefront; results
 * are bitwise those of the wavefront.  Realised for 3-D star stencils on
 * uniform-halo grids: heat model radius 1 (F <= 4) and 2 (F <= 3), wave
 * model radius 1 (F <= 3), 2 (F <= 2) and 4 (F <= 2; register-bound, slower
 * than the wavefront); for
 * 2-D ones (radius <= 4) whose rows fit the SMs'
 * shared memory, F is the number of levels between halo exchanges of the
 * SM-resident kernel (the grid stays on-chip for the whole run).  Other
 * stencils fall back to the wavefront (st_report.kernel_kind tells which
 * ran). */
typedef struct {
  int schedule;
  int skew;
  int64_t time_tile;
  int64_t space_tiles[ST_MAX_DIMS];
  int64_t fused_levels;
  /* executor extension (0 = off): tile_time applied to d_2 as well, with a
   * skew of band_skew rows per level (clamped up to the radius; legality as
   * for d_1: skew >= delta_2).  The wavefront then advances bands of
   * band_rows rows through the T levels of a time tile back to back, so a
   * band's levels re-read one another from L2 and only ~4 r rows per level
   * cross a band boundary through HBM.  3-D star stencils
   * with uniform halos and a CTA tile of >= 2 r rows; other plans ignore
   * it.  Bitwise equal to the canonical nest for every value. */
  int64_t band_rows;
  int band_skew;
} st_plan;

/* ExecReport (executor.hpp:58-62) plus device-side detail. */
typedef struct {
  int64_t points_updated;
  int64_t flops;            /* points_updated * flops_per_point             */
  double wall_seconds;      /* host wall clock around the launch sequence  */
  double device_seconds;    /* CUDA events on the context stream            */
  int64_t time_tile_used;   /* levels in flight actually realised           */
  int64_t kernel_launches;  /* kernels this call launched                   */
  int64_t tile[3];          /* CTA tile (z-chunk, y, x) used, device axes   */
  int mode_used;            /* st_mode actually evaluated                   */
  int kernel_kind;          /* 3 = SM-resident 2-D time tiling,             
                             2 = fused levels (on-chip time tile),        
                             1 = star (registers+smem), 0 = generic       */
} st_report;

typedef struct st_stencil st_stencil;
typedef struct st_context st_context;
typedef struct st_grid st_grid;

const char* st_last_error(void);
const char* st_version(void);

/* ---- stencil-model (host) ------------------------------------------- */
int st_stencil_create(const char* name, int ndims, const st_term* terms,
                      int nterms, int model, st_stencil** out);
/* parse_spec grammar (stencil.hpp:87-96). extents_out has
 * room for ST_MAX_DIMS; err_line receives the 1-based line on ST_ERR_PARSE. */
int st_stencil_parse(const char* text, st_stencil** out, int* ndims_out,
                     int64_t* extents_out, int64_t* steps_out, int* err_line);
void st_stencil_destroy(st_stencil* s);
int st_stencil_ndims(const st_stencil* s);
int st_stencil_model(const st_stencil* s);
int st_stencil_nterms(const st_stencil* s);
int st_stencil_term(const st_stencil* s, int k, st_term* out);
int st_stencil_time_depth(const st_stencil* s);
int st_stencil_radius(const st_stencil* s, int dim);
int st_min_skew_factor(const st_stencil* s);
int64_t st_time_buffer_slots(const st_stencil* s, int64_t time_tile);
int64_t st_flops_per_point(const st_stencil* s);
/* ST_OK or ST_ERR_ILLEGAL_PLAN; *required_minimum = min_skew_factor */
int st_check_legality(const st_stencil* s, const st_plan* plan,
                      int* required_minimum);
int64_t st_required_slots(const st_stencil* s, const st_plan* plan);
int64_t st_layout_plane(const st_stencil* s, const int64_t* extents);

/* ---- host initialisers (reference layout, deterministic) ------------ */
int st_init_reference(const st_stencil* s, const int64_t* extents,
                      float* host, int64_t slots, uint64_t seed);
int st_init_unit(const st_stencil* s, const int64_t* extents, float* host,
                 int64_t slots, uint64_t seed);
int st_init_gaussian(const st_stencil* s, const int64_t* extents, float* host,
                     int64_t slots, double sigma, const int64_t* centre);
/* z-slab window of a global Gaussian: rows [z_begin, z_begin + extents[0])
 * of the global grid (for the sharded config). */
int st_init_gaussian_slab(const st_stencil* s, const int64_t* extents,
                          float* host, int64_t slots, double sigma,
                          const int64_t* centre, int64_t z_begin);
int st_field_layered(int ndims, const int64_t* extents, float* m,
                     double v_top, double v_bottom, int64_t split, double dt,
                     double h, int64_t z_begin);
int st_field_random_smoothed(int ndims, const int64_t* extents, float* m,
                             uint64_t seed, double vmin, double vmax,
                             double dt, double h);
int st_verify_bitwise(const st_stencil* s, const int64_t* extents,
                      const float* a, int64_t slots_a, const float* b,
                      int64_t slots_b, int64_t last_level,
                      int64_t compare_levels, int* equal);
/* verify_bitwise(a, b, compare_levels) (executor.hpp:110) without a
 * stencil: the grids' GridLayout (interior extents, halo radii per axis). */
int st_verify_bitwise_layout(int ndims, const int64_t* extents,
                             const int64_t* radii, const float* a,
                             int64_t slots_a, const float* b, int64_t slots_b,
                             int64_t last_level, int64_t compare_levels,
                             int* equal);

/* ---- cache-sim (cache_sim.hpp:28-34) -------------------------------- */
/* TrafficReport (cache_sim.hpp:19-26). */
typedef struct {
  int64_t lines_loaded;
  int64_t lines_written_back;
  int64_t line_elems;
  int64_t bytes;         /* 4 * line_elems * (loaded + written back) */
  int64_t flops;
  double measured_ai;    /* flops / bytes (0 without traffic) */
} st_traffic;
/* simulate: the nest's exact access stream (term reads in term order, then
 * the write, per traced point) against a fully associative LRU cache of
 * cache_elems float32 elements in line_elems-element lines, write-allocate
 * + write-back, final dirty flush counted.  Host-only (CPU model of the
 * reference nest; the autotuner's sim_traffic cost).  ST_ERR_INVALID once
 * more than `cap` points are traced. */
int st_simulate(const st_stencil* s, const int64_t* extents, int64_t time_steps,
                const st_plan* plan, int64_t cache_elems, int64_t line_elems,
                int64_t cap, st_traffic* out);

/* ---- device context ------------------------------------------------- */
int st_context_create(int device, st_context** out);
void st_context_destroy(st_context* c);
/* cudaStream_t of the context (for event timing by the caller). */
void* st_context_stream(st_context* c);
int st_context_device(const st_context* c);
int st_context_sm_count(const st_context* c);
/* Overwrite a buffer of twice the L2 size on the context's stream (timing
 * hygiene between measured trials: autotuner, bench). */
int st_context_flush_l2(st_context* c);

/* ---- device grid ---------------------------------------------------- */
int st_grid_create(st_context* c, const st_stencil* s, const int64_t* extents,
                   int64_t slots, st_grid** out);
void st_grid_destroy(st_grid* g);
/* Host buffer in the reference GridLayout (slots * plane floats).  Levels
 * last_level-delta_t+1 .. last_level are taken from slot (level mod slots).
 * flags: ST_UPLOAD_UNIFORM_HALO asserts every slot carries the same halo. */
#define ST_UPLOAD_UNIFORM_HALO 1u
int st_grid_upload(st_grid* g, const float* host, int64_t nelems,
                   int64_t last_level, unsigned flags);
/* Wave model coefficient field m, interior row-major D_1..D_n. */
int st_grid_set_field(st_grid* g, const float* m, int64_t nelems);
/* Writes the retained levels (the last delta_t + 1) into slot (level mod
 * slots) of the host reference-layout buffer; other slots untouched. */
int st_grid_download(st_grid* g, float* host, int64_t nelems,
                     int64_t* last_level);
int st_grid_last_level(const st_grid* g, int64_t* last_level);
int64_t st_grid_device_bytes(const st_grid* g);
/* Steps t in [t_begin, t_end) (step t writes level t + delta_t).  t_begin
 * must continue the grid: t_begin + delta_t - 1 == last_level. */
int st_apply(st_grid* g, int64_t t_begin, int64_t t_end, const st_plan* plan,
             int mode, st_report* report);

/* execute on a HOST grid (executor.hpp:92-98: execute(nest, spec, space,
 * grid) with the Grid in host memory), through the device grid g: uploads
 * levels [t_begin, t_begin + delta_t) from their slots (level mod slots),
 * runs steps [t_begin, t_end) like st_apply and writes the interior of the
 * newest delta_t levels [t_end, t_end + delta_t) back into their slots
 * (halos and other slots untouched).  With a page-locked host buffer and
 * uniform halos the copies run on the copy engines (contiguous upload
 * blocks converted on the GPU as they land, pitched 2D download); calls on
 * grids of different contexts overlap one another's copies and kernels.
 * Otherwise it is st_grid_upload + st_apply + a staged download.
 * flags: ST_UPLOAD_UNIFORM_HALO (as st_grid_upload). */
int st_execute_host(st_grid* g, float* host, int64_t nelems, int64_t t_begin,
                    int64_t t_end, const st_plan* plan, int mode,
                    unsigned flags, st_report* report);

/* ---- z-slab decomposition (config 5; the reference has none) -------- */
/* Slab of rank `rank` among `world` along d_1, plus ghost depths (0 on the
 * global boundary): the local grid has z_count + ghost_lo + ghost_hi planes
 * and starts at global plane z_begin - ghost_lo. */
int st_dist_partition(int64_t global_nz, int world, int rank, int64_t ghost,
                      int64_t* z_begin, int64_t* z_count, int64_t* ghost_lo,
                      int64_t* ghost_hi);
typedef struct st_dist st_dist;
/* 128-byte NCCL unique id (rank 0 creates it, every rank receives it). */
int st_nccl_unique_id(unsigned char* id128);
/* nccl_id == NULL: in-process loopback member (see st_dist_link_loopback). */
int st_dist_create(st_grid* local, int rank, int world,
                   const unsigned char* nccl_id, int64_t ghost_lo,
                   int64_t ghost_hi, st_dist** out);
int st_dist_link_loopback(st_dist** ranks, int world);
/* Steps [t_begin, t_end): exchange the delta_t newest levels' ghost planes
 * every plan->time_tile levels, compute the shrinking valid ranges. */
int st_dist_apply(st_dist* d, int64_t t_begin, int64_t t_end,
                  const st_plan* plan, int mode, st_report* report);
void st_dist_destroy(st_dist* d);

#ifdef __cplusplus
}
#endif
#endif /* STENCIL_TILER_H */
