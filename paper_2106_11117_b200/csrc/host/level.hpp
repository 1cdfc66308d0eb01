// Per-level operator tables: the sample-independent geometry of one MLMC
// level, laid out for the device kernels.
//
// Reference semantics restated here (all file:line into /root/reference/proj):
//   * element stiffness K_e = c(centroid) * area * grad(phi_i).grad(phi_j) and
//     lumped mass M_ii += area/3                          src/fem.cpp:91-126
//   * A = M^{-1/2} K M^{-1/2}, selector P = vertices of fine-flagged
//     triangles, A P / A (I-P) column masks               src/fem.cpp:42-63
//   * lumped L2 projection of u0 (edge-midpoint rule), z0 = sqrt(M) coef
//                                                          src/fem.cpp:223-269
//   * n_steps = ceil(T/dt - 1e-12), dt = T/n_steps         src/integrators.cpp:188-189
//   * Chebyshev constants and the LTS substep constants   src/integrators.cpp:34-66, :126-141
//
// The per-sample coefficient c is piecewise constant on an nx x ny cell grid
// and enters A linearly, so A(omega)_ij = sum_k c_k(omega) * a0_ijk with the
// geometric a0_ijk shared by all samples (the "parts" representation).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "mesh.hpp"
#include "mesh1d.hpp"

namespace wmc {

enum class Integrator : int { Leapfrog = 0, LocalTimeStepping = 1 };

struct GaussianIC {
    double x0 = 0.3, y0 = 0.5, width2 = 0.01;  // u0 = exp(-((x-x0)^2+(y-y0)^2)/width2)
};

struct QoIBox {
    double x0 = 0.7, x1 = 0.9, y0 = 0.4, y1 = 0.6;
};

// Uniform / LognormalKL: per-cell coefficients on a cells_x x cells_y grid
// (BASELINE); Kl1D / Jump1D: the reference's 1D experiment fields
// (rng.cpp:42-89), one coefficient per element; Channel: the narrow-channel
// experiment's per-sample geometry (channel.hpp), one cell per moving entry
// LognormalKLElem: the KL field at every triangle's centroid (one coefficient
// cell per element, as the reference's assemble evaluates it, fem.cpp:103-104)
enum class Field : int { Uniform = 0, LognormalKL = 1, Kl1D = 2, Jump1D = 3, Channel = 4, LognormalKLElem = 5 };

struct LevelSpec {
    int cells_x = 4, cells_y = 4;  // coefficient grid on the domain box, cell k = iy*cells_x + ix
    double coef_lo = 0.5, coef_hi = 1.5;  // c_k ~ U[coef_lo, coef_hi)
    Field field = Field::Uniform;
    double kl_sigma = 0.5, kl_corr_len = 0.1;  // log-normal KL (BASELINE config 4)
    int kl_modes = 64;
    double final_time = 1.0;
    double dt = 0.0;  // requested coarse step (snapped so n_steps*dt == T)
    int substeps = 1;
    double nu = 0.01;
    Integrator kind = Integrator::LocalTimeStepping;
    GaussianIC ic;
    QoIBox qoi;
    bool qoi_mean = false;  // Q = mean over the box (weights normalised by their sum)
    int tiers = 1;          // nested LTS tiers (config 2); 1 = the reference's single-tier LF-LTS
    double cfl_safety = 0.0;  // > 0: per-sample dt from the reference's stable_dt recipe (experiments.cpp:30-43)
    double jump_h0 = 0.0;     // Jump1D: jump position ~ U[4 - h0, 4) (rng.cpp:53-58)
    double grid_lo = 0.0, grid_hi = 1.0;  // 1D experiments: QoI output grid (reference OutputGrid)
    int grid_n = 0;
    double dom_x0 = 0.0, dom_x1 = 1.0, dom_y0 = 0.0, dom_y1 = 1.0;  // coefficient grid extent

    // cell k = iy * cells_x + ix of the coefficient grid, ix = floor((x - x0) / (x1 - x0) * cells_x)
    int cell_col(double x) const;
    int cell_row(double y) const;
    int cell_of(double x, double y) const { return cell_row(y) * cells_x + cell_col(x); }
};

struct ChebyshevConstants {
    int p = 1;
    double nu = 0.0, delta = 1.0, omega = 2.0;
    std::vector<double> beta_int, beta_half;
};

ChebyshevConstants chebyshev_constants(int p, double nu);

struct LevelTables {
    int n = 0;       // interior DOFs (Dirichlet boundary eliminated)
    int n_r = 0;     // DOFs [0, n_r) are R = rows of A P with a nonzero
    int n_p = 0;     // |P|
    int n_cells = 0;
    std::vector<int> dof_vertex;        // dof -> mesh vertex
    std::vector<std::uint8_t> in_p;     // per dof
    std::vector<std::uint8_t> dof_tier; // per dof: deepest P_k holding it (0: none; single tier: in_p)

    // full operator, row-wise "parts": A_ij(omega) = sum over the row's
    // entries e with col[e] == j of c[cell[e]] * a0[e]; exact zeros dropped
    std::vector<int> row_ptr;
    std::vector<int> col;
    std::vector<int> cell;
    std::vector<double> a0;
    // the reference's nnz of A (normalized) and of A P (a_fine): explicit
    // zeros kept, as its CSR stores them (cost records' weighted_work)
    long ref_nnz = 0, ref_nnz_fine = 0;

    // A P restricted to R rows, as recipes: entry (row r, col j in P, wid);
    // recipe wid = sum_t c[rc_cell[t]] * rc_a0[t] for t in [rc_ptr[wid], rc_ptr[wid+1])
    std::vector<int> ap_row_ptr;
    std::vector<int> ap_col;
    std::vector<int> ap_wid;
    std::vector<int> rc_ptr;
    std::vector<int> rc_cell;
    std::vector<double> rc_a0;

    // A P on R rows as sweep-style parts (col | cell << apg_col_bits, a0):
    // the HBM-resident substep path for sets R too large for one SM
    std::vector<int> apg_ptr, apg_ent;
    std::vector<int> apg_col, apg_cell;  // the same entries unpacked (levels with more than 511 cells)
    std::vector<double> apg_a0;
    int apg_col_bits = 23;

    std::vector<double> mass;       // lumped mass per dof
    std::vector<double> z0;         // sqrt(M) * projected u0, per dof
    // QoI: nq outputs, output k = sum over entries t in [qoi_ptr[k], qoi_ptr[k+1])
    // of qoi_w[t] * (z[qoi_dof[t]] / sqrt_mass_qoi[t]); the QoI norm is
    // sqrt(sum_k qoi_norm_w[k] Q_k^2) (reference QoIVector::norm, fem.cpp:15-19).
    // BASELINE configs: one output (the box integral), weight 1.
    int nq = 1;
    std::vector<int> qoi_ptr{0, 0};
    std::vector<int> qoi_dof;
    std::vector<double> qoi_w;
    std::vector<double> sqrt_mass_qoi;
    std::vector<double> qoi_norm_w{1.0};

    std::vector<int> elem_cell;     // per triangle (diagnostics)

    // Structured block of the refined square for the substep fast path.  The
    // box has (m+1)^2 nodes with dof = i*(m+1) + j (Q-local i, j; column
    // major); lattice nodes are (i, j) in [1, m-1]^2 off horizontal
    // coefficient lines: their six triangles are h_min lattice triangles, so
    // (A d)_i = (1/h) sum_dir kappa_dir (v_i - v_dir) with v = d / sqrt(M)
    // and kappa = mean coefficient of the two triangles on an edge; every
    // other R row ("generic") keeps explicit per-entry recipes.
    bool lattice = false;
    bool box = false;                       // box geometry valid (dofs [0, (m+1)^2) = box, column major)
    std::vector<int> dof_lx, dof_ly;        // box-local lattice coordinates of every dof (when box)
    int lat_m = 0;
    double lat_inv_h = 0.0;
    std::vector<int> lat_cellx, lat_celly;  // coefficient column / row of square column i / row j
    std::vector<std::uint8_t> lat_row;     // per box row j: 1 if its interior nodes are lattice nodes
    std::vector<int> strip_j0, strip_len;   // row strips of lattice nodes (no coefficient line inside)
    int lat_cw = 0;                         // threads per strip row (columns, rounded up to 32)
    int lat_threads = 0, lat_k = 0;         // kernel variant: CTA size, max rows per thread
    std::string lattice_reason;             // why the fast path is off (diagnostics)
    std::vector<int> gen_rows;              // generic R rows (dofs)
    std::vector<double> gen_rs;             // 1/sqrt(M) of each generic row
    std::vector<int> gen_ptr, gen_col;      // CSR over gen_rows, columns in P
    std::vector<int> gen_rc_ptr, gen_rc_cell;  // per entry: terms of w = sum c_k a0_k sqrt(M_j)
    std::vector<double> gen_rc_a0;

    // nested tiers (config 2): rows are ordered deepest tier first, so
    // R_k = rows [0, n_r_tier[k-1]) with R_1 = [0, n_r) ⊇ R_2 ⊇ ...; per tier
    // A P_k on R_k rows in parts form (col | cell << 23, a0) and the tier's
    // substep constants (its "dt" is dt / p^(k-1)); back = -2 / dt_k^2 turns
    // the tier's d_p into the effective right-hand side of tier k-1
    int tiers = 1;
    std::vector<int> n_r_tier;
    std::vector<std::vector<int>> tier_ptr, tier_ent;
    std::vector<std::vector<double>> tier_a0;
    std::vector<double> tier_c0, tier_back;
    std::vector<std::vector<double>> tier_cm;

    // 1D experiment fields: element midpoints, and for Kl1D the table
    // field_table[e * field_terms + m] with c_e = 1 + sum_m table xi_m over
    // xi = (kl_cos_1..K, kl_sin_1..K), xi ~ next_symmetric()
    std::vector<double> field_x, field_table;
    int field_terms = 0;

    // per-sample CFL (cfl_safety > 0): warm starts of the power iterations,
    // the dominant eigenvectors of the c = 1 operator (full, and A (I-P) on
    // rows outside P), as the reference's level contexts (experiments.cpp:132-148)
    double cfl_safety = 0.0;
    std::vector<double> warm_full, warm_coarse;
    int p_fine = 1;                  // substeps of the finest tier (p^tiers)

    // time stepping
    long n_steps = 0;
    double dt = 0.0;
    int p = 1;
    Integrator kind = Integrator::LocalTimeStepping;
    double c0 = 0.0;                 // d_1 = -c0 (A z_n)
    std::vector<double> beta;        // beta_int[m-1], m = 1..p-1
    std::vector<double> cm;          // c_m, m = 1..p-1
    double coarse_factor = 0.0;      // rows outside R: z+ = 2z - z- - coarse_factor * (A z)
    double init_factor = 0.0;        // start-up: z1 = z0 - init_factor * (A z0)
};

LevelTables build_level_tables(const TriMesh& mesh, const LevelSpec& spec);

/// One level of the reference's 1D sampling experiments (smooth1d / jump1d,
/// experiments.cpp:56-106): Neumann (every vertex a DOF), P1 with c^2 per
/// element at its midpoint (fem.cpp:66-89), u0 projected with two-point Gauss
/// (fem.cpp:206-220), QoI = the solution on spec.grid_n points of
/// [grid_lo, grid_hi] (restrict_to_grid, fem.cpp:277-293).
LevelTables build_level_tables_1d(const Mesh1D& mesh, const LevelSpec& spec);

/// DOF-updates per solve: steps * (n + (p-1)|R|) for LTS, steps * n for LF
/// (SURVEY.md section 8(d)); the start-up step counts as one sweep.  Nested
/// tiers: a row of R_k \ R_k+1 advances p^k times per step.
double dof_updates_per_solve(const LevelTables& t);

}  // namespace wmc
