// Device kernels of the batched LF / LF-LTS sample evaluator (sm_100a, FP64).
//
// Layout in HBM (per level, per batch of S samples, S a multiple of 64):
//   z[i * S + s]      nodal state, node-major with samples interleaved, so a
//                     warp reads one row for 64 samples as 32 x 16 B
//   gd[s * G + r]     per-sample rows of R (r < n_r, G = n_r rounded up to 8):
//                     A z_n written by the sweep (transposed through shared
//                     memory), read by the substep kernel, overwritten with
//                     d_p, read by the R update -- sample-major so the
//                     one-sample-per-CTA substep kernel moves it coalesced
//   cells[k * S + s]  per-sample coefficient of cell k
// The geometric operator tables are shared by all samples.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace wmc {

// operator entries pack the column (23 bits) and the coefficient cell (9 bits)
constexpr int kColBits = 23;
constexpr int kColMask = (1 << kColBits) - 1;
constexpr int kMaxCells = 511;
constexpr unsigned kMultiCell = 0xffffu;  // slot weight with several cells (on-chip generic kernel)
constexpr unsigned kOvfFlag = 0x8000u;    // lattice kernel: slot weight in the overflow list

constexpr int kSweepChunk = 64;  // samples per warp in the sweep (2 per lane)
constexpr int kSweepWarps = 8;   // rows per sweep block
constexpr int kNsMax = 12;       // fused solve: entries of a TMEM-held row outside R
constexpr int kSubThreads = 1024;
constexpr int kSubMaxRpt = 8;    // rows per thread in the substep kernel

// Structured sweep rows: a row whose stored entries are exactly the 5-point
// pattern {i - dS, i - 1, i, i + 1, i + dN} (column order), all in one
// coefficient cell, with off-diagonal a0 == w.x and diagonal a0 == w.y of a
// small per-level table, is swept from its descriptor alone (no per-entry
// index or weight loads).  Same products in the same order as the generic
// single-cell path: bit-identical results.
constexpr int kMaxRowTypes = 8;

// Narrow-channel experiment (host/channel.hpp): per-sample operator entries
// c_k = A_ij(b), k >= 1, from the moved reference mesh; cell 0 is the unit
// coefficient of the sample-independent entries.
struct ChannelArgs {
    int n_ent;                   // per-sample cells 1 .. n_ent
    const double* vx;            // local vertices: reference position, blend(x)
    const double* vy;
    const double* vblend;
    const int* tri;              // moving triangles, 3 local vertices each
    const double* ms;            // local vertex: mass of its fixed triangles
    const int* m_ptr;
    const int* m_tri;
    const int* e_li;             // entry endpoints (local vertex, or -1 with the fixed mass)
    const int* e_lj;
    const double* e_mi;
    const double* e_mj;
    const double* e_ks;          // fixed triangles' stiffness
    const int* k_ptr;            // moving triangles coupling the pair: t * 9 + a * 3 + b
    const int* k_tri;
};

struct SweepArgs {
    int n;           // rows
    int split;       // rows < split stash g (LTS); 0 for leapfrog
    int S;           // batch stride
    int count;       // live samples
    const int* row_ptr;
    const int* ent;      // col | cell << col_bits (23, or 16 when there are more than 511 cells)
    int col_bits, col_mask;
    const int* cell_ix;          // per-entry cell when it is not packed above the column (NULL: packed)
    const double* a0;
    // per row {info, row_ptr begin, dS, dN}; info = cell | type << 16 |
    // pfull << 24 for a structured row (type >= 1; pfull = deepest tier whose
    // P holds all five columns), cell for another single-cell row, -1 for a
    // row spanning several cells (may be NULL: generic gather everywhere)
    const int4* row_desc;
    const double2* wtype;  // [kMaxRowTypes]: (off-diagonal a0, diagonal a0) of type t + 1 (device table)
    const double* cells;
    const double* z0;    // init only
    const double* zc;    // z_n
    double* zp;          // z_{n-1} in, z_{n+1} out; init: z0 out
    double* zc_out;      // init only: z_1 out
    double* g;           // gd buffer, rows < split
    int g_stride;        // G
    int g_node_major;    // 1: g[r * S + s] (global substep path), 0: gd[s * G + r]
    double factor;       // init_factor or coarse_factor
    int step;
    int* fail;
    const double* rel;   // per-sample CFL: (dt_s / dt)^2 scales every dt^2 constant (NULL: 1)
    const int* nsteps;   // per-sample CFL: steps of sample s; later steps leave it untouched (NULL: all)
    int wide;            // step sweep form: 10 R + MINB of sweep_wide_kernel (fixed dt, S % 128 == 0), 0: sweep_rows_kernel
    int row_begin;       // step sweeps: rows [row_begin, n) only (the tiled step owns R); 0: all rows
    int sample_major;    // 1: z[s * n + i] (tiled levels: one sample's rows contiguous), 0: z[i * S + s]
    int sm_groups;       // sample-major sweep: groups of four samples a thread walks through (set by the launch)
};

struct SubArgs {
    int n_r, S, count, p;
    int n_wid, n_cells, n_ent;
    int cl_smem;                // 1: cell coefficients staged in shared memory, 0: recipes read them from global
    const std::uint32_t* ent;   // SELL: [slice][width][32], col | wid << 16
    const int* slice_off;       // per slice: entry offset; width = (off[s+1]-off[s]) / 32
    const int* rc_ptr;
    const int* rc_cell;
    const double* rc_a0;
    const double* cells;
    double* gd;           // [s][g_stride]: g in, d_p out
    int g_stride;
    const double* beta;   // p-1
    const double* cm;     // p-1
    double c0;
    int step;             // global step being formed (per-sample CFL: skip finished samples)
    const double* rel;
    const int* nsteps;
};

// lattice substep kernel variants (threads, rows per thread, generic rows per
// thread): (1024, 4, 1) and (512, 8, 2); generic SELL rows hold <= 8 entries
constexpr int kLatGenWidth = 8;

// Substep kernel with the structured fast path: the refined-square lattice
// L = [1, m-1]^2 (5-point stencil from cell coefficients, state v = d / h)
// plus generic rows from a per-sample weighted SELL; see kernels.cu.
struct LatArgs {
    int threads, strip_k;        // kernel variant
    int n_r, S, count, p, n_cells, cells_x;
    int m, cw, n_strips;
    int n_gen, n_slots;
    double inv_h, c0;
    const int* strip_j0;
    const int* strip_len;
    const unsigned char* lat_smask;  // per thread: bit k set if the strip's node k is read through shared memory
    const int* cellx;            // m entries
    const int* celly;            // m entries
    const int* gen_rows;         // n_gen dofs
    const double* gen_rs;        // 1/sqrt(M)
    const int* gen_soff;         // slot offset of each 32-row slice (rows sorted by length), n_slices + 1
    const int* gen_warp_slice;   // [warp][G]: slice of the warp's u-th generic role (-1: none), balanced by width
    const std::uint16_t* gen_col;  // per slot: [slice][width / 2][32][2] (slot pairs), padding: col 0, weight 0
    const double* slot_a0;       // per slot: a0 of the single term
    const std::uint16_t* slot_cell;  // per slot: its cell, or kOvfFlag | k: terms ovf_start[k] .. ovf_start[k+1]
    int n_ovf, n_ovf_terms;          // slots whose weight spans several cells (edge on a coefficient line)
    const int* ovf_start;
    const std::uint16_t* ovf_cell;
    const double* ovf_a0;
    const double* cells;
    double* gd;                  // [s][g_stride]: g in, d_p out
    int g_stride;
    const double* beta;
    const double* cm;
    int step;
    const double* rel;
    const int* nsteps;
};

// z_{n+1} = 2 z_n - z_{n-1} + 2 d_p on the R rows (reference
// src/integrators.cpp:149-153), d_p transposed back through shared memory.
struct RUpdateArgs {
    int n_r, S, count, g_stride;
    const double* gd;
    const double* zc;
    double* zp;
    int step;
    int* fail;
    const int* nsteps;
};

// One LTS substep of the HBM-resident path (|R| too large for one SM): warp
// per (row, 64 samples) over the R rows, d in node-major global buffers.
// d_m / d_{m-1} come from a buffer, from -c0 g (d_1) or are zero (d_0).
struct GSubArgs {
    int n_r, S, count;
    const int* ptr;
    const int* ent;       // col | cell << kColBits, columns in P
    const int* cell_ix;   // not NULL: ent holds the column alone and the cell is cell_ix[entry]
                          // (levels with more than kMaxCells coefficient cells: per-element fields)
    const double* a0;
    const double* cells;
    const double* g;      // [r][S]
    const double* dcur;   // d_m (cur_mode 0)
    double* dprev;        // d_{m-1} in (prev_mode 0), d_{m+1} out
    int cur_mode;         // 0 buffer, 1 = -c0 g
    int prev_mode;        // 0 buffer, 1 = -c0 g, 2 = zero
    double c0, beta, cm;
    int last;             // fuse z_{n+1} = 2 z_n - z_{n-1} + 2 d_p
    const int4* row_desc;  // sweep descriptors: rows with pfull >= 1 gather structured
    const double2* wtype;  // device table, see SweepArgs
    const double* zc;
    double* zp;
    int step;
    int* fail;
    const double* rel;
    const int* nsteps;
};

// Nested tiers (BASELINE config 2, no reference counterpart; DESIGN.md
// section "Nested LTS"): one stage m of tier k over the rows of R_k, warp per
// (row, 64 samples).  rho = r_k + A P_k E^k_m (the product only for m >= 1);
// rows < split (R_k+1) hand rho to tier k+1 as its right-hand side, the
// others apply the tier-k update and, when m is the tier's last stage, carry
// the result up through the ancestors' updates (r~ = back_j E^j_p) down to
// z_{n+1} = 2 z_n - z_{n-1} + 2 E^1_p.  Tier j keeps E^j_m in e[j][m & 1].
constexpr int kMaxTiers = 8;

struct TierArgs {
    int k, m, p;                 // tier (1-based), stage, substeps per tier
    int row_begin, row_end, split;
    int S, count;
    const int* ptr;              // A P_k on R_k rows: col | cell << kColBits, a0
    const int* ent;
    const double* a0;
    const double* cells;
    const double* rhs;           // r_k [row][S]
    double* rhs_next;            // r_k+1 [row][S] (rows < split)
    const double* src;           // E^k_m (gathered, m >= 1)
    // the row update and its carry through the ancestors whose stage ends
    // with this one, fixed per launch: link t (tier k - t) forms
    // en = A E_m - B E_{m-1} - C v (E_m of link 0 from the gather window),
    // then either stores en to out, or (out == NULL, tier 1 ending) forms
    // z_{n+1}, or passes v = back en to link t + 1
    int depth;
    struct Link {
        const double* em;        // NULL: E_m == 0 (stage 0)
        const double* emm;       // NULL: E_{m-1} == 0 (stages 0, 1)
        double* out;
        double A, B, C, back;
    } link[kMaxTiers];
    const int4* row_desc;        // sweep descriptors: rows with pfull >= k gather structured
    const double2* wtype;  // device table, see SweepArgs
    const double* zc;
    double* zp;
    int step;
    int* fail;
    const double* rel;
    const int* nsteps;
};

// Fused small-mesh solve: one CTA owns one sample at a time (persistent over
// the batch) and runs the whole solve -- start-up, every global step's sweep,
// LF-LTS substeps on R and update, check_finite, QoI -- with the state in
// shared memory.  For levels whose state fits one SM (the 1D experiments,
// config 0, small MLMC levels) and small batches, where the per-step kernel
// launches of the batched path dominate.  Same arithmetic as the batched
// kernels (generic gathers), per-sample CFL scale and horizon included.
constexpr int kSmallThreads = 512;

struct SmallArgs {
    int n, n_r, p, S, count, n_cells;
    int split;                   // rows < split take the substeps (0: leap-frog everywhere)
    const int* row_ptr;          // full operator (sweep tables, as SweepArgs)
    const int* ent;
    int col_bits, col_mask;
    const int* cell_ix;          // per-entry cell when it is not packed above the column (NULL: packed)
    const double* a0;
    const int4* row_desc;
    const double2* wtype;
    // A P on R rows exactly as the on-chip generic substep kernel holds it:
    // SELL entries col | wid << 16 per 32-row slice, recipes of the weights
    const std::uint32_t* sub_ent;
    const int* slice_off;
    int n_wid;
    const int* rc_ptr;
    const int* rc_cell;
    const double* rc_a0;
    const double* cells;         // [k * S + s]
    const double* z0;
    double init_factor, factor, c0;  // factor: leap-frog / coarse-row factor
    const double* beta;          // p - 1
    const double* cm;            // p - 1
    long n_steps;                // fixed-dt horizon
    const double* rel;           // per-sample CFL (NULL: fixed dt)
    const int* nsteps;
    int nq;                      // QoI matrix (as QoIArgs)
    const int* qptr;
    const int* qdof;
    const double* qw;
    const double* qsm;
    double* q;                   // [k * S + s]
    int* fail;                   // per sample: first non-finite step (INT_MAX: none)
};

void launch_draw_channel(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S,
                         const ChannelArgs& a, double* cells, void* stream);
int small_smem_bytes(const SmallArgs& a);

// Fused lattice solve: the whole solve of one sample per CTA (persistent over
// the batch) for lattice levels whose state fits one SM -- start-up, every
// global step's sweep (g = A z_n on all rows from the sweep descriptors,
// leap-frog update of the rows outside R), the p - 1 substeps of the lattice
// kernel and the R update, check_finite and the QoI.  z_n lives in shared
// memory, z_{n-1} too when it fits (else in a per-sample global buffer read
// and written only by the row's owner).  No HBM traffic per step, and the
// per-sample set-up (cell coefficients, generic weights) once per solve
// instead of once per step.  Arithmetic: see kernels.cu (K6).
struct LatSolveArgs {
    LatArgs lat;                 // substep tables and constants (gd unused)
    int n;                       // all rows; rows [n_r, n) are outside R
    const int* row_ptr;          // sweep tables (as SweepArgs)
    const int* ent;
    int col_bits, col_mask;
    const int* cell_ix;          // per-entry cell when it is not packed above the column (NULL: packed)
    const double* a0;
    const int4* row_desc;
    const double2* wtype;
    const double* z0;
    double init_factor, factor;  // start-up and coarse-row (leap-frog) factors
    long n_steps;
    double* zp_global;           // z_{n-1} at [s * n + i] when it does not fit on chip (NULL: shared)
    // A (I - P) entries of the generic rows (sorted SELL order): g = A z_n on
    // a generic row is the SELL gather on v = z / sqrt(M) (the A P part) plus
    // these (columns outside P)
    // rows outside R that are not structured (CSR rows of <= kNsMax entries),
    // thread t owning ns_rows[t] and ns_rows[t + threads]: their entries live
    // in the thread's TMEM columns (TMEM form 2; n_ns = 0: gathered from the
    // CSR arrays in the round-robin sweep like the structured rows)
    const int* ns_rows;
    int n_ns;
    const int* rem_ptr;
    const int* rem_col;
    const int* rem_cell;
    const double* rem_a0;
    int nq;
    const int* qptr;
    const int* qdof;
    const double* qw;
    const double* qsm;
    double* q;                   // [k * S + s]
    int* fail;                   // per sample: first non-finite step (INT_MAX: none)
    int strips_k_or_k1;          // every lattice strip holds K or K - 1 rows
    int tmem;                    // 0: shared memory; 1: generic weights/columns and d_{m-1} in tensor memory; 2: weights/columns only (default)
    int stagger;                 // substeps: half of each scheduler's warps run their lattice nodes before their generic rows
};

int lattice_solve_smem_bytes(const LatSolveArgs& a);
int lattice_solve_max_smem(int device);
int launch_lattice_solve(const LatSolveArgs& a, int grid, void* stream);  // returns cudaError_t
int small_max_smem(int device);  // largest dynamic shared memory the kernel can take
int launch_small_solve(const SmallArgs& a, int grid, void* stream);  // returns cudaError_t

struct QoIArgs {
    int nq, S, count;     // nq outputs; output k sums entries ptr[k] .. ptr[k+1]
    const int* ptr;
    const int* dof;
    const double* w;
    const double* sqrt_mass;
    const double* z;
    const int* fail;
    double* q;
    const double* z_alt;  // per-sample CFL: a sample that ended (n_max - nsteps[s]) odd steps early
    const int* nsteps;    // holds its state in the other buffer
    int n_max;
    int n;                // sample_major: z[s * n + i]
    int sample_major;
};

// Per-sample CFL step (reference stable_dt, src/experiments.cpp:30-43): batched
// power iteration on A(omega) (full, and A (I-P) on rows outside P) from the
// level's warm starts, per-sample Rayleigh quotients and stopping rule of
// max_eigenvalue (src/fem.cpp:132-175).
struct EigArgs {
    int n, S, count;
    const int* row_ptr;
    const int* ent;
    int col_bits, col_mask;
    const int* cell_ix;          // per-entry cell when it is not packed above the column (NULL: packed)
    const double* a0;
    const double* cells;
    const unsigned char* in_p;
    int coarse;           // 1: masked columns in P, zero rows in P
    const double* v;      // [i][S]
    double* av;
    int n_blocks;         // row blocks of the dot-product partials
    double* part;         // [2][n_blocks][S]: v.av, av.av
    double* norm;         // per sample: |A v| of this iteration
    double* lam;          // per sample: result
    double* lam_prev;
    int* settled;
    int* iters;
    int* done;            // 0 running, 1 settled, 2 zero operator
    int* active_count;    // samples still running after this iteration
    double tol;
};

// log-normal KL field on the cell grid: xi_m ~ N(0,1) by Box-Muller over
// consecutive next_unit() pairs, g_k = sum_m table[k*modes+m] xi_m, c_k = exp(g_k)
constexpr int kMaxKLModes = 64;
void launch_draw_kl(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S, int n_cells,
                    int modes, const double* table, double* cells, void* stream);
void launch_draw_cells(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S, int n_cells,
                       double lo, double hi, double* cells, void* stream);
// the reference's 1D experiment fields, one coefficient per element
// (rng.cpp:42-89): Kl1D: c_e = 1 + sum_m table[e][m] xi_m, xi_m = 2 unit - 1
// (next_symmetric) from words 0..terms-1; Jump1D: J = next_uniform(4 - h0, 4)
// from word 0, c_e = x_e < J ? 1 : 4
void launch_draw_kl1d(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S, int n_cells,
                      int terms, const double* table, double* cells, void* stream);
void launch_draw_jump1d(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S, int n_cells,
                        double h0, const double* x, double* cells, void* stream);
void launch_sweep_init(const SweepArgs& a, void* stream);
void launch_sweep_step(const SweepArgs& a, void* stream);
int substep_smem_bytes(const SubArgs& a);
int launch_substeps(const SubArgs& a, int grid, void* stream);  // returns cudaError_t
void launch_qoi(const QoIArgs& a, void* stream);
void launch_r_update(const RUpdateArgs& a, void* stream);

// Temporally blocked LF-LTS step on R (host/tiles.hpp): one CTA per (tile,
// sample) work item, persistent over items; the tile's region (kTileWz x
// kTileHz box positions, or the transposed shape, plus generic rows) stays
// on chip for the whole step:
// z_n in, g = A z_n, the p - 1 substeps, z_{n+1} = 2 z_n - z_{n-1} + 2 d_p on
// the owned rows out.  Rows outside R are left to the sweep.
constexpr int kTileThreads = 256;  // two CTAs per SM: one's barriers and latencies overlap the other's work
constexpr int kTileK = 8;     // rows per strip (thread = 2 columns x kTileK rows)
constexpr int kTileWz = 128;  // region columns
constexpr int kTileHz = 32;   // region rows (shape 1 is the transpose, shape 2 the square of the same area)
constexpr int kTileSq = 64;
static_assert(kTileSq * kTileSq == kTileWz * kTileHz, "square shape");
struct TileArgs {
    int S, count, p, m, n_cells, cells_x;
    int box_slots, max_app, max_ent, max_gen, n_tiles;
    double inv_h, h, inv_h2, c0;
    const int4* tile_rect;   // per tile: region origin i0, j0; owned columns [oi0, oi1)
    const int4* tile_oj;     // owned rows [oj0, oj1), shape (0: kTileWz x kTileHz, 1: kTileHz x kTileWz, 2: kTileSq x kTileSq)
    const int4* thr_geo;     // per tile and thread: first column, first row, lattice | owned << 16
    const int* gen_off;      // per tile: generic rows [gen_off[t], gen_off[t+1])
    const int* g_slot;
    const int* g_dof;
    const int* g_owned;
    const double* g_rs;      // 1 / sqrt(M)
    const int* g_ent_off;    // SELL entries [off[r], off[r+1]) (P columns, local slots)
    const int* g_rem_off;    // remainder entries [off[r], off[r+1]) (other columns, dofs)
    const int* e_slot;
    const int* e_rc_off;     // recipe of entry e: [e_rc_off[e], e_rc_off[e+1])
    const int* rc_cell;
    const double* rc_a0;     // a0 sqrt(M_col)
    const int* r_dof;
    const int* r_rc_off;
    const int* rr_cell;
    const double* rr_a0;
    const unsigned char* line_row;  // per box row: starts a coefficient row
    const int* cellx;        // per square column / row: coefficient column / row
    const int* celly;
    const double* cells;     // [k * S + s]
    const double* beta;      // p - 1
    const double* cm;        // p - 1
    const double* zc;        // z_n, sample-major: z[s * n + i]
    double* zp;              // z_{n-1} in, z_{n+1} out (owned R rows)
    int n;
    int* fail;
    int step;
};
// Streamed interior of the tiled step (stream.cu): the box interior away
// from the ring in horizontal slabs of kStreamThreads rows (one thread per
// row), each slab swept column by column with all p levels in flight (a
// wavefront: level m one column behind level m - 1), so a slab's region is
// unbounded along the sweep and its halo is p columns at the two ends only.
constexpr int kStreamThreads = 256;
constexpr int kStreamMaxP = 8;
struct StreamArgs {
    int S, count, p, m, n, cells_x, n_slabs, max_nx;
    int threads;             // CTA size: the slabs' rows rounded up to a warp (<= kStreamThreads)
    int chunks, chunk_cols;  // a slab's owned columns in `chunks` runs of chunk_cols (work items of even length)
    double inv_h, h, inv_h2, c0;
    double opb[kStreamMaxP], beta[kStreamMaxP], cm[kStreamMaxP];  // substep m at [m - 1]: 1 + beta_m, beta_m, c_m
    const int4* slab;      // region: first column I0, columns NX, first row J0, rows NY (box coordinates)
    const int4* slab_own;  // owned region columns [x0, x1), rows [y0, y1)
    const int* cellx;
    const int* celly;
    const double* cells;   // [k * S + s]
    const double* zc;      // z_n, sample-major
    double* zp;            // z_{n-1} in, z_{n+1} out (owned rows)
    int* fail;
    int step;
};
int stream_smem_bytes(const StreamArgs& a);
int launch_stream_step(const StreamArgs& a, int grid, void* stream);  // returns cudaError_t

int tile_smem_bytes(const TileArgs& a);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
int set_max_dynamic_smem(const void* kernel, int bytes, bool max_carveout = false);
int launch_tile_step(const TileArgs& a, int grid, void* stream);  // returns cudaError_t
void launch_global_substep(const GSubArgs& a, void* stream);
void launch_tier_stage(const TierArgs& a, void* stream);
void launch_fill_int(int* p, int value, int n, void* stream);
void launch_eig_init(const double* warm, double warm_norm, int n, int S, double* v, void* stream);
void launch_eig_iteration(const EigArgs& a, void* stream);
// per sample: dt = safety min(2 / sqrt(1.05 lc), p_fine 2 / sqrt(1.05 lf)) (or the LF form), snapped to
// T / ceil(T / dt - 1e-12); rel = (dt / dt_ref)^2, nsteps; padding lanes get rel 1 and 1 step
void launch_cfl_finalize(const double* lf, const double* lc, int use_coarse, int p_fine, double safety, double T,
                         double dt_ref, int count, int S, double* rel, int* nsteps, void* stream);
// per-sample results, sample-major: dq[i*nq + k] = qf[k*S + i] - qc[k*S + i]
// (qc NULL: level 0), q_out[i*nq + k] = qf[k*S + i] (q_out may be NULL)
void launch_pair_diff(const double* qf, const double* qc, double* dq, double* q_out, int count, int S, int nq,
                      void* stream);
int substep_max_grid(int device, int smem_bytes);
int lattice_smem_bytes(const LatArgs& a);
int launch_lattice_substeps(const LatArgs& a, int grid, void* stream);  // returns cudaError_t
// deterministic single-block fold of (dq, q) into out[0..3] += {sum dq, sum dq^2, sum q, sum q^2}
void launch_moments(const double* dq, const double* q, int count, double* out, void* stream);
void launch_fail_fold(const int* ff, const int* fc, int count, unsigned long long first, unsigned long long* rec,
                      void* stream);

}  // namespace wmc
