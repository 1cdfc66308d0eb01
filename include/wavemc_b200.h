/* wavemc-b200: C ABI of the B200-native batched LF / LF-LTS sample evaluator.
 *
 * This is the drop-in boundary for the reference's sample-parallel hot path.
 * The reference plugs a per-sample solver into its MLMC driver through
 *
 *   struct MlmcProblem { grid; max_levels_available; model_cost; draw; solve; }
 *                                          reference include/wavemc/mlmc.hpp:41-47
 *
 * and evaluates job lists (level, index) in run_jobs (src/mlmc.cpp:107-149),
 * one sample_delta_q (src/mlmc.cpp:21-37) per job.  Here one call evaluates a
 * contiguous index range of coupled (fine, coarse) pairs on a B200:
 *
 *   wmc_level_create   replaces the per-level context build of make_problem /
 *                      build_state_2d (src/experiments.cpp:132-148, :194-237):
 *                      mesh -> operator tables, selector P, R = rows(A P),
 *                      initial data, QoI weights, resident in HBM.
 *   wmc_eval_pairs     replaces run_jobs' loop over sample_delta_q for one
 *                      level: draw (RngStream(seed, level, index), src/rng.cpp:14-32)
 *                      -> solve fine and coarse (assemble + run_wave + QoI,
 *                      src/experiments.cpp:150-172) -> dQ, Q_fine per index.
 *   wmc_run_mlmc_fixed / wmc_run_mlmc
 *                      the fixed-N sweep and the adaptive Giles driver
 *                      (run_mlmc, src/mlmc.cpp:165-233) over batched pairs,
 *                      folding results in (level, index) order like
 *                      src/mlmc.cpp:145-147.
 *
 * Conventions:
 *   - status codes, no exceptions: 0 ok, 2 config error (reference
 *     ConfigError), 3 numerical error (NumericalError / InstabilityError with
 *     err->sample and err->step), 4 device/runtime error;
 *   - host buffers are caller-owned, device memory is handle-owned;
 *   - calls are synchronous; one host thread per device.
 * The message of the last failure on the calling thread: wmc_last_error().
 */
#ifndef WAVEMC_B200_H
#define WAVEMC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WMC_OK 0
#define WMC_CONFIG_ERROR 2
#define WMC_NUMERICAL_ERROR 3
#define WMC_DEVICE_ERROR 4

#define WMC_LEAPFROG 0
#define WMC_LOCAL_TIME_STEPPING 1

#define WMC_FIELD_UNIFORM 0        /* c_k = next_uniform(lo, hi) per cell */
#define WMC_FIELD_LOGNORMAL_KL 1   /* c = exp(g), g a truncated KL expansion sampled at cell centres */
#define WMC_FIELD_LOGNORMAL_KL_ELEMENT 2 /* the same g at every triangle's centroid: one coefficient per element, as
                                            the reference's assemble evaluates speed2 (src/fem.cpp:103-104); cells_x /
                                            cells_y unused; the levels of a pair evaluate one draw on their own elements */

typedef struct wmc_mesh wmc_mesh;
typedef struct wmc_level wmc_level;

/* Unit square, structured right triangles, refined square at h/ratio with
 * 2:1 balanced transitions (no reference counterpart: SURVEY.md Appendix A
 * item 4; transition cells follow src/mesh2d.cpp:96-130, fine flags
 * src/mesh2d.cpp:285-301). */
typedef struct {
    int n_coarse;        /* cells per side, h = 1/n_coarse */
    int ratio;           /* h / h_min, power of two */
    double fine_lo, fine_hi;  /* refined square [lo, hi]^2 */
    double snap;         /* snap grid for the square (0 -> coarse grid) */
    double small_factor; /* small triangle: longest edge < small_factor*sqrt(2)*h (0: none) */
} wmc_square_mesh_spec;

int wmc_mesh_build_square(const wmc_square_mesh_spec* spec, wmc_mesh** out);

/* Graded L-shape [-1,1]^2 minus [0,1]x[-1,0] (BASELINE config 2; no
 * reference counterpart -- the reference L-shape, src/mesh_graded.cpp:48-112,
 * carries no fine flags): balanced quadtree at h = 1/n_per_unit, leaves split
 * while side > h sqrt(r / grade_radius) (r = distance to the corner (0,0)),
 * down to h / 2^tiers.  Triangle flag = refinement tier plus one adjacent
 * layer per tier; P_k = vertices of triangles with flag >= k. */
typedef struct {
    int n_per_unit;      /* h = 1 / n_per_unit */
    int tiers;           /* 0..6 */
    double grade_radius; /* 0.25 */
} wmc_lshape_mesh_spec;

int wmc_mesh_build_lshape(const wmc_lshape_mesh_spec* spec, wmc_mesh** out);
/* A mesh from arrays, e.g. a reference TriMesh (include/wavemc/mesh.hpp:48-74). */
int wmc_mesh_create(int n_vertices, int n_triangles, const double* xy, const int* tri, const unsigned char* fine,
                    const unsigned char* boundary, double coarse_h, double fine_h, wmc_mesh** out);
int wmc_mesh_info(const wmc_mesh* mesh, int* n_vertices, int* n_triangles, double* coarse_h, double* fine_h);
int wmc_mesh_export(const wmc_mesh* mesh, double* xy, int* tri, unsigned char* fine, unsigned char* boundary);
/* Reference fixture text format (src/mesh_io.cpp:1-9). */
int wmc_mesh_dump(const wmc_mesh* mesh, const char* path);
void wmc_mesh_destroy(wmc_mesh* mesh);

typedef struct {
    int cells_x, cells_y;        /* piecewise-constant coefficient grid on [0,1]^2 */
    double coef_lo, coef_hi;     /* c_k = next_uniform(lo, hi), row-major cell order */
    double final_time;           /* T */
    double dt;                   /* requested coarse step (snapped, integrators.cpp:188-189) */
    int substeps;                /* p */
    double nu;                   /* stabilisation, reference default 0.01 */
    int integrator;              /* WMC_LEAPFROG or WMC_LOCAL_TIME_STEPPING */
    double ic_x, ic_y, ic_width2;  /* u0 = exp(-((x-ic_x)^2 + (y-ic_y)^2) / ic_width2), v0 = 0 */
    double qoi_box[4];           /* x0, x1, y0, y1: Q = lumped integral of u(T) over the box */
    int device;                  /* CUDA device ordinal */
    int batch;                   /* samples per device batch, 0 = automatic */
    int field;                   /* WMC_FIELD_UNIFORM, WMC_FIELD_LOGNORMAL_KL or WMC_FIELD_LOGNORMAL_KL_ELEMENT */
    double kl_sigma;             /* KL: standard deviation of g */
    double kl_corr_len;          /* KL: correlation length of exp(-|dx|/l - |dy|/l) */
    int kl_modes;                /* KL: number of terms, xi_m ~ N(0,1) by Box-Muller over next_unit pairs */
    int tiers;                   /* nested LTS tiers (0 or 1: single-tier LF-LTS); tier k substeps with
                                    p per tier on P_k = vertices of triangles with flag >= k */
    double domain[4];            /* x0, x1, y0, y1 of the coefficient grid (all 0: unit square) */
    int qoi_mean;                /* 1: Q = mean of u(T) over the box (weights / their sum) */
    double cfl_safety;           /* > 0: per-sample dt = the reference's stable_dt recipe (src/experiments.cpp:30-43:
                                    power iteration tol 1e-4 from the level's c = 1 warm starts, margin 1.05,
                                    safety factor cfl_safety), snapped to T / n_steps per sample; dt is ignored */
} wmc_level_desc;

void wmc_level_desc_default(wmc_level_desc* desc);

typedef struct {
    int n;                    /* interior DOFs */
    int n_r;                  /* |R|, rows of A P with a nonzero */
    int n_p;                  /* |P| */
    int p;                    /* substeps */
    long n_steps;
    double dt;
    long nnz;                 /* stored operator entries (exact zeros dropped) */
    long ap_nnz;              /* A P entries on R */
    long n_recipes;
    int batch;                /* samples per device batch */
    double dof_updates_per_solve;  /* n + (n_steps-1)(n + sum_k (p^k - p^(k-1))|R_k|) for LTS, n_steps*n for LF */
    int lattice;              /* 1: substeps use the structured refined-square kernel */
    int substep_path;         /* 0 none (LF or p = 1), 1 lattice, 2 generic on-chip, 3 HBM-resident,
                                 4 HBM-resident nested tiers, 5 tiled (R in spatial tiles, every
                                 substep of a step on chip); -1 plan only */
    int tiers;                /* nested LTS tiers in use */
    int n_r_tier[8];          /* |R_k| for tiers k = 1..tiers (n_r_tier[0] == n_r), rows [0, |R_k|) */
    long n_structured;        /* sweep rows taking the structured 5-point path (0 before device setup) */
    int nq;                   /* QoI outputs per sample (1: scalar; the experiments' output grid) */
    int fused;                /* 1: each batch runs as one fused lattice-solve kernel (z_n, z_{n-1} on chip),
                                 2: the same with z_{n-1} in a per-sample global buffer, 0: per-step kernels */
} wmc_level_info;

int wmc_level_create(const wmc_mesh* mesh, const wmc_level_desc* desc, wmc_level** out);
/* A 1D mesh of the reference's sampling experiments: the reference's
 * Mesh1D (include/wavemc/mesh.hpp:21-33) passed through as arrays -- sorted
 * vertices (n_vertices), fine flags per element (n_vertices - 1), coarse and
 * fine sizes.  The adapter feeds it level by level from the reference's own
 * build_hierarchy (src/mesh1d.cpp:76-125), as build_state_1d does
 * (src/experiments.cpp:62-85). */
typedef struct wmc_mesh1d wmc_mesh1d;
int wmc_mesh1d_create(int n_vertices, const double* vertices, const unsigned char* fine_flags, double coarse_h,
                      double fine_h, wmc_mesh1d** out);
void wmc_mesh1d_destroy(wmc_mesh1d* mesh);

/* The reference's own 1D sampling experiments (
 * reference make_problem, src/experiments.cpp:56-106, 194-237): level `level`
 * on `mesh`, the level's mesh of the reference hierarchy, with `substeps` its
 * ratio p_l (MeshHierarchy::ratios; LTS) -- LF uses 1; fine region [5 - h0, 5]
 * (smooth) or [4 - h0, 4] (jump), Neumann, u0 = exp(-(x-3)^2/0.09),
 * per-sample CFL step (stable_dt with the given safety); field sample_kl
 * (smooth: c^2 = 1 + KL, 100 cos + 100 sin terms) or sample_jump (c^2 = 1
 * left of J ~ U[4 - h0, 4), 4 right of it); QoI = u(T) on grid_n points of
 * [0, 6] (restrict_to_grid), norm with trapezoid weights. */
#define WMC_EXP_SMOOTH1D 1
#define WMC_EXP_JUMP1D 2
#define WMC_EXP_CHANNEL2D 3
typedef struct {
    int experiment;
    int integrator;
    double h0, fine_h, final_time, nu, safety;
    int grid_n, max_level;
    int device, batch;
} wmc_experiment_desc;

/* the reference's default_config (src/config_io.cpp:49-73) for the experiment */
void wmc_experiment_desc_default(wmc_experiment_desc* desc, int experiment);
int wmc_level_create_experiment(const wmc_mesh1d* mesh, int substeps, const wmc_experiment_desc* desc, int level,
                                wmc_level** out);
/* The reference's narrow-channel experiment (make_problem Channel2d,
 * src/experiments.cpp:108-172): level `level` on `mesh`, the reference's
 * build_channel_mesh(max(h0 / 2^level, fine_h), fine_h) (src/mesh2d.cpp:
 * 319-359; the adapter passes its TriMesh through wmc_mesh_create).  Per
 * sample the width b = next_uniform(0.001, 0.007) (sample_width,
 * src/rng.cpp:59-64) moves the mesh by ChannelGeometry::map; Neumann (every
 * vertex a DOF), speed 1, bump u0 at (1/2, 0), per-sample CFL step with warm
 * starts from the reference mesh, p = ceil(h0 2^-level / fine_h) (LF-LTS) or
 * 1 (LF), QoI = u(T) on grid_n points of the line x = -0.4, y in [-1/2, 1/2]
 * (extract_line_qoi), trapezoid norm.  desc->experiment = WMC_EXP_CHANNEL2D;
 * wmc_experiment_desc_default gives the reference's default_config. */
int wmc_level_create_channel(const wmc_mesh* mesh, const wmc_experiment_desc* desc, int level, wmc_level** out);
/* Host-only plan of a channel level (sizes, no device work). */
int wmc_channel_plan(const wmc_mesh* mesh, const wmc_experiment_desc* desc, int level, wmc_level_info* info);
/* Host-only plan of an experiment level (sizes, no device work). */
int wmc_experiment_plan(const wmc_mesh1d* mesh, int substeps, const wmc_experiment_desc* desc, int level,
                        wmc_level_info* info);
/* The experiment's model cost per level, the reference's closed-form cost
 * model (model_params, src/experiments.cpp:177-192; cost_lts_level /
 * cost_lf_level, src/cost_model.cpp:40-58): the run_mlmc weights. */
double wmc_experiment_model_cost(const wmc_experiment_desc* desc, int level);

/* Host-only: build the level tables and report their sizes, no device work. */
int wmc_level_plan(const wmc_mesh* mesh, const wmc_level_desc* desc, wmc_level_info* info);
int wmc_level_get_info(const wmc_level* level, wmc_level_info* info);
void wmc_level_destroy(wmc_level* level);

/* Host-only: the temporally blocked step's plan for a box level (spatial
 * tiles around the box ring, streamed slabs inside), no device work.
 * ok = 0 with `reason` when the level does not take the tiled step. */
typedef struct {
    int ok;
    int n_tiles, n_slabs;
    int max_gen;             /* generic rows per tile */
    double work_factor;      /* region positions per box node */
    double streamed_frac;    /* box nodes owned by slabs / box nodes */
    char layout[32];
    char reason[256];
} wmc_tile_plan_info;
int wmc_tile_plan(const wmc_mesh* mesh, const wmc_level_desc* desc, int stream, wmc_tile_plan_info* info);

typedef struct {
    long matvec_full, matvec_fine, matvec_coarse;  /* reference CostRecord, mlmc.hpp:25-32 */
    long weighted_work;
    double dof_updates;
} wmc_cost;

typedef struct {
    long sample;  /* global index of the first failing sample, -1 if none */
    long step;    /* reference InstabilityError::step */
    int level;
} wmc_error;

/* Coupled pairs for indices first .. first+count-1 of MLMC level `level`:
 * c drawn once from RngStream(seed, level, index) and shared by the fine
 * solve (on `fine`) and the coarse solve (on `coarse`; NULL on level 0).
 * dq[i] = Q_fine - Q_coarse (Q_fine on level 0), q_fine[i] = Q_fine.
 * cost and err may be NULL. */
int wmc_eval_pairs(wmc_level* fine, wmc_level* coarse, uint64_t seed, uint32_t level, uint64_t first, uint64_t count,
                   double* dq, double* q_fine, wmc_cost* cost, wmc_error* err);

/* Same work with the per-sample results left in device memory (d_dq, d_q_fine:
 * device pointers, or NULL to keep them in the handle) and no host
 * synchronisation: the device-resident leg used for kernel-level timing. */
int wmc_eval_pairs_device(wmc_level* fine, wmc_level* coarse, uint64_t seed, uint32_t level, uint64_t first,
                          uint64_t count, double* d_dq, double* d_q_fine);

/* The handle's CUDA stream (cudaStream_t) for event timing; all work of a
 * level pair is issued on the fine level's stream. */
void* wmc_level_stream(wmc_level* level);
/* Waits for the level's stream.  Every batch of wmc_eval_pairs_device folds
 * its check_finite flags (reference src/integrators.cpp:12-18) into a record
 * on the fine level; synchronize reads it: the first failing sample (lowest
 * index) since the previous call is reported in err (sample, step, level)
 * with status 3 (NumericalError, as src/mlmc.cpp:31-35), and the record is
 * cleared. */
int wmc_synchronize(wmc_level* level, wmc_error* err);

/* KL table of the log-normal field: table[cell * modes + m] =
 * sigma sqrt(lambda_m) phi_m(centre of cell), lambda[m] (unit variance). */
int wmc_kl_table(int cells_x, int cells_y, double sigma, double corr_len, int modes, double* table, double* lambda);
/* The expansion's modes for a pointwise evaluator (WMC_FIELD_LOGNORMAL_KL_ELEMENT on the reference side,
   where speed2(x, y) is a callable, src/fem.cpp:91-104): out[7 m ..] = amp, omega_x, even_x, norm_x, omega_y,
   even_y, norm_y; mode m is amp * phi_x(x) * phi_y(y), phi(t) = (even ? cos : sin)(omega (t - 1/2)) / norm. */
int wmc_kl_modes(double sigma, double corr_len, int modes, double* out);

/* The level's per-sample cell coefficients for indices first..first+count-1,
 * out[i * n_cells + k], exactly as the solves use them. */
int wmc_level_draw(wmc_level* level, uint64_t seed, uint32_t level_index, uint64_t first, uint64_t count,
                   double* out);

/* Per-sample CFL step (level created with cfl_safety > 0): the device power
 * iterations for indices first..first+count-1 of MLMC level `level_index`,
 * per sample the snapped step dt[i] = T / steps[i] (reference stable_dt,
 * src/experiments.cpp:30-43, then run_wave's snapping). */
int wmc_level_cfl(wmc_level* level, uint64_t seed, uint32_t level_index, uint64_t first, uint64_t count, double* dt,
                  long* steps);

/* Per-sample coefficients exactly as the device draws them (RNG parity). */
int wmc_draw_cells(uint64_t seed, uint32_t level, uint64_t first, uint64_t count, int n_cells, double lo, double hi,
                   int device, double* out);

typedef struct {
    int level;
    long n_samples;
    double sum_dq, sum_dq2, sum_q, sum_q2;  /* LevelAccumulator, mlmc.hpp:53-66 */
    double variance;     /* estimate_variance, mlmc.cpp:61-66 */
    double mc_variance;  /* estimate_mc_variance, mlmc.cpp:68-73 */
    double mean_dq;
    double model_cost;
    wmc_cost cost;
} wmc_level_stats;

/* Fixed sample counts on levels 0..n_levels-1 (BASELINE config 1): indices
 * first[l] .. first[l]+counts[l]-1 of level l (first may be NULL = 0), i.e.
 * one rank's shard; stats hold the shard's LevelAccumulator sums. */
int wmc_run_mlmc_fixed(wmc_level** levels, int n_levels, const long* first, const long* counts, uint64_t seed,
                       wmc_level_stats* stats, wmc_error* err);

typedef struct {
    double eps;             /* root-MSE target */
    double alpha;           /* bias decay exponent */
    int initial_samples;    /* 16 */
    int initial_levels;     /* 2 */
    int max_level;
    uint64_t master_seed;
    int bias_window;        /* 1 */
} wmc_mlmc_config;

void wmc_mlmc_config_default(wmc_mlmc_config* cfg);

typedef struct {
    double estimate;
    int converged;
    int levels_used;
    double total_variance;
    double bias;
    double total_model_cost;
    double rmse;            /* sqrt(total_variance + bias) */
} wmc_mlmc_result;

/* Adaptive Giles driver (reference run_mlmc, src/mlmc.cpp:165-233) with
 * model_cost[l] per level; stats must hold n_levels entries. */
int wmc_run_mlmc(wmc_level** levels, int n_levels, const double* model_cost, const wmc_mlmc_config* cfg,
                 wmc_mlmc_result* result, wmc_level_stats* stats, wmc_error* err);

/* Same driver for QoI vectors (the reference experiments' grid QoIs): also
 * writes the estimate vector (nq outputs, wmc_level_info.nq) to `estimate`;
 * result->estimate then holds its norm. */
int wmc_run_mlmc_vec(wmc_level** levels, int n_levels, const double* model_cost, const wmc_mlmc_config* cfg,
                     wmc_mlmc_result* result, wmc_level_stats* stats, double* estimate, wmc_error* err);

/* Multi-device drivers (the reference's worker pool
 * run_jobs, src/mlmc.cpp:107-149, one level set per device): levels holds
 * n_devices groups of n_levels levels, level l of group d at
 * levels[d * n_levels + l] (each group on its own device, the same level
 * definitions).  Every wave's index range of a level is split into
 * contiguous 64-sample granules per device; each device group runs on its
 * own host thread; the per-sample results are folded on the host in (level,
 * index) order, so stats, estimate and sample counts are bitwise those of
 * the one-device drivers, whatever n_devices. */
int wmc_run_mlmc_fixed_multi(wmc_level** levels, int n_devices, int n_levels, const long* counts, uint64_t seed,
                             wmc_level_stats* stats, wmc_error* err);
int wmc_run_mlmc_multi(wmc_level** levels, int n_devices, int n_levels, const double* model_cost,
                       const wmc_mlmc_config* cfg, wmc_mlmc_result* result, wmc_level_stats* stats, double* estimate,
                       wmc_error* err);

/* Host-only helpers of the adaptive driver, as the reference's
 * optimal_samples (src/mlmc.cpp:75-92) and bias_proxy_sq (:94-98). */
int wmc_optimal_samples(const double* variances, const double* costs, int n_levels, double eps, long min_samples,
                        long* out);
double wmc_bias_proxy_sq(double mean_dq, double alpha);

/* Device-side per-level fold: d_out[0..3] += {sum dq, sum dq^2, sum q, sum q^2}
 * over count device values, one fixed-order block (deterministic).  Scalar
 * QoI levels only (nq == 1; QoI vectors fold on the host): status 2 else. */
int wmc_moments_device(wmc_level* level, const double* d_dq, const double* d_q, uint64_t count, double* d_out);

/* Kernel-level timing: with profiling on, every sweep, substep and R-update
 * launch of the level is bracketed by CUDA events on its stream; read
 * returns the summed device time and launch counts and resets. */
int wmc_profile_enable(wmc_level* level, int on);
int wmc_profile_read(wmc_level* level, double* sweep_ms, long* sweep_launches, double* sub_ms, long* sub_launches,
                     double* upd_ms, long* upd_launches);

/* Number of kernels this library has launched in the process. */
long wmc_launch_count(void);

const char* wmc_last_error(void);
int wmc_device_count(void);

#ifdef __cplusplus
}
#endif
#endif
