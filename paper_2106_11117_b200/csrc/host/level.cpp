#include "level.hpp"

#include "channel.hpp"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>

namespace wmc {

namespace {
std::uint64_t mix64_host(std::uint64_t z) {  // reference rng.hpp:14-19
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
}  // namespace

// Chebyshev stabilisation constants, restating reference
// src/integrators.cpp:34-66: delta = 1 + nu/p^2, T_k(delta) by the three-term
// recurrence, omega = 2 p U_{p-1}(delta) / T_p(delta),
// beta_int[k-1] = T_{k-1}/T_{k+1}, beta_half[k-1] = T_k/T_{k+1}.
ChebyshevConstants chebyshev_constants(int p, double nu) {
    if (p < 1) throw std::invalid_argument("chebyshev_constants: p >= 1 required");
    if (nu < 0.0 || nu > 1.0) throw std::invalid_argument("chebyshev_constants: nu in [0,1]");
    ChebyshevConstants c;
    c.p = p;
    c.nu = nu;
    c.delta = 1.0 + nu / (double(p) * p);
    const double d = c.delta;
    std::vector<double> t(p + 1);
    t[0] = 1.0;
    t[1] = d;
    for (int k = 2; k <= p; ++k) t[k] = 2.0 * d * t[k - 1] - t[k - 2];
    double u_prev = 1.0, u = 2.0 * d;
    for (int k = 2; k <= p - 1; ++k) {
        const double next = 2.0 * d * u - u_prev;
        u_prev = u;
        u = next;
    }
    const double u_pm1 = (p == 1) ? 1.0 : u;
    c.omega = 2.0 * p * u_pm1 / t[p];
    c.beta_int.resize(p - 1);
    c.beta_half.resize(p - 1);
    for (int k = 1; k <= p - 1; ++k) {
        c.beta_int[k - 1] = t[k - 1] / t[k + 1];
        c.beta_half[k - 1] = t[k] / t[k + 1];
    }
    return c;
}

int LevelSpec::cell_col(double x) const {
    return std::clamp(static_cast<int>(std::floor((x - dom_x0) / (dom_x1 - dom_x0) * cells_x)), 0, cells_x - 1);
}

int LevelSpec::cell_row(double y) const {
    return std::clamp(static_cast<int>(std::floor((y - dom_y0) / (dom_y1 - dom_y0) * cells_y)), 0, cells_y - 1);
}

namespace {

// lattice substep kernel variants: (threads, max rows per thread)
constexpr int kLatticeVariants[3][2] = {{512, 8}, {768, 6}, {1024, 4}};

using StiffMap = std::map<std::tuple<int, int, int>, double>;

// Geometry of one level before DOF numbering: what a mesh (2D triangles or
// 1D elements) contributes to the tables
struct Geometry {
    int nv = 0;
    std::vector<std::uint8_t> boundary;   // Dirichlet vertices (eliminated)
    std::vector<double> mass;             // lumped mass per vertex
    StiffMap stiff;                       // (vi, vj, cell) -> geometric stiffness
    std::vector<std::uint8_t> sel, vt;    // P_1 and the vertex tier
    std::vector<double> coef0;            // projected u0 coefficients (load / mass)
    bool qoi_dof_order = false;           // one output, vertex weights qoi_vertex_w[0], DOF order
    std::vector<std::vector<double>> qoi_vertex_w;
    std::vector<std::vector<std::pair<int, double>>> qoi_entries;  // else: per output (vertex, weight)
    std::vector<double> qoi_norm_w;
    bool unit_cells = false;              // channel: cells >= 1 are whole per-sample entries (a0 = 1)
    std::vector<double> cell_ref;         // channel: reference-geometry value of every cell (warm starts)
};

// Finds the structured block of the refined square and checks, numerically
// against the assembled element stiffness, that every lattice node
// (i, j) in [1, m-1]^2 has the 5-point stencil with edge conductances
// (c_a + c_b) / 2 and lumped mass h^2.  Rows j on a horizontal coefficient
// line (squares j-1 and j in different cells) are left to the generic path,
// so every lattice node of a strip sees one coefficient row above and below.
// Fills the lattice fields of L and returns the box vertices in column-major
// order (box index i*(m+1) + j), or an empty vector (with lattice_reason).
std::vector<int> lattice_block(const TriMesh& mesh, const LevelSpec& spec, const std::vector<double>& mass,
                               const StiffMap& stiff, const std::vector<std::uint8_t>& in_r, LevelTables& L) {
    auto fail = [&](const std::string& why) {
        L.lattice = false;
        L.lattice_reason = why;
        return std::vector<int>{};
    };
    if (spec.field == Field::LognormalKLElem) return fail("per-element coefficient");
    if (mesh.fine_box_lo < 0 || mesh.lattice.size() != mesh.vertices.size()) return fail("no refined box");
    const int qa = mesh.fine_box_lo, m = mesh.fine_box_hi - mesh.fine_box_lo;
    if (m < 4) return fail("refined box too small");
    if ((m + 1) % 2 == 0) return fail("even box width (shared-memory bank conflicts)");
    const int W = m + 1;
    const double h = mesh.fine_h;
    std::map<std::pair<int, int>, int> at;
    for (int v = 0; v < mesh.n_vertices(); ++v) at[{mesh.lattice[v][0], mesh.lattice[v][1]}] = v;
    std::vector<int> box;
    box.reserve(static_cast<std::size_t>(W) * W);
    for (int i = 0; i <= m; ++i)
        for (int j = 0; j <= m; ++j) {
            const auto it = at.find({qa + i, qa + j});
            if (it == at.end()) return fail("box node missing");
            if (mesh.boundary_vertex[it->second] || !in_r[it->second]) return fail("box node not in R");
            box.push_back(it->second);
        }
    auto node = [&](int i, int j) { return box[i * W + j]; };
    std::vector<int> cx(m), cy(m);
    for (int i = 0; i < m; ++i) {
        const double x = (qa + i + 0.5) * h;
        cx[i] = spec.cell_col(x);
        cy[i] = spec.cell_row(x);
    }
    // distinct test coefficients per cell
    const int nc = spec.cells_x * spec.cells_y;
    std::vector<double> ct(nc);
    for (int k = 0; k < nc; ++k) ct[k] = 1.0 + 0.371 * k + 0.013 * k * k;
    auto csq = [&](int i, int j) { return ct[cy[j] * spec.cells_x + cx[i]]; };
    for (int i = 1; i <= m - 1; ++i)
        for (int j = 1; j <= m - 1; ++j) {
            const int v = node(i, j);
            if (std::abs(mass[v] - h * h) > 1e-12 * h * h) return fail("lumped mass != h^2 in L");
            const int nb[4] = {node(i + 1, j), node(i - 1, j), node(i, j + 1), node(i, j - 1)};
            const double kap[4] = {0.5 * (csq(i, j) + csq(i, j - 1)), 0.5 * (csq(i - 1, j) + csq(i - 1, j - 1)),
                                   0.5 * (csq(i - 1, j) + csq(i, j)), 0.5 * (csq(i - 1, j - 1) + csq(i, j - 1))};
            double want_diag = 0.0, got_diag = 0.0;
            double got[4] = {0.0, 0.0, 0.0, 0.0};
            int others = 0;
            for (auto it = stiff.lower_bound({v, -1, -1}); it != stiff.end() && std::get<0>(it->first) == v; ++it) {
                const int u = std::get<1>(it->first);
                const double val = it->second * ct[std::get<2>(it->first)];
                if (it->second == 0.0) continue;
                if (u == v) {
                    got_diag += val;
                    continue;
                }
                int d = 0;
                while (d < 4 && nb[d] != u) ++d;
                if (d == 4) {
                    ++others;
                    continue;
                }
                got[d] += val;
            }
            if (others) return fail("non 5-point stencil in L");
            for (int d = 0; d < 4; ++d) {
                want_diag += kap[d];
                if (std::abs(got[d] + kap[d]) > 1e-12 * kap[d]) return fail("edge conductance mismatch in L");
            }
            if (std::abs(got_diag - want_diag) > 1e-12 * want_diag) return fail("diagonal mismatch in L");
        }
    // lattice rows: [1, m-1] minus rows on a horizontal coefficient line;
    // strips of <= K consecutive lattice rows, K from the first kernel
    // variant whose CTA holds them
    std::vector<std::uint8_t> lat_row(m + 1, 0);
    for (int j = 1; j <= m - 1; ++j) lat_row[j] = cy[j] == cy[j - 1];
    const int cw = (m - 1 + 31) / 32 * 32;
    std::vector<int> j0s, lens;
    int threads = 0, kmax = 0;
    const char* force = std::getenv("WMC_LATTICE_THREADS");  // tuning: force a variant
    for (const auto& var : kLatticeVariants) {
        if (force && std::atoi(force) != var[0]) continue;
        j0s.clear();
        lens.clear();
        for (int j = 1; j <= m - 1;) {
            if (!lat_row[j]) {
                ++j;
                continue;
            }
            // a run of lattice rows, cut into the fewest strips of <= K rows,
            // lengths balanced (31 rows: 8 8 8 7 at K = 8)
            int e = j;
            while (e <= m - 1 && lat_row[e]) ++e;
            const int run = e - j, ns = (run + var[1] - 1) / var[1];
            for (int q = 0; q < ns; ++q) {
                const int l = run / ns + (q < run % ns ? 1 : 0);
                j0s.push_back(j);
                lens.push_back(l);
                j += l;
            }
        }
        if (static_cast<int>(j0s.size()) * cw <= var[0]) {
            threads = var[0];
            kmax = var[1];
            break;
        }
    }
    // the box geometry holds either way (the tiled step kernel uses it);
    // the single-CTA lattice kernels need every strip in one CTA
    L.box = true;
    L.lat_m = m;
    L.lat_inv_h = 1.0 / h;
    L.lat_cellx = cx;
    L.lat_celly = cy;
    L.lat_row = lat_row;
    if (!threads) {
        L.lattice = false;
        L.lattice_reason = "too many strips for the CTA";
        return box;
    }
    L.lat_threads = threads;
    L.lat_k = kmax;
    L.lattice = true;
    L.lat_m = m;
    L.lat_inv_h = 1.0 / h;
    L.lat_cellx = cx;
    L.lat_celly = cy;
    L.lat_row = lat_row;
    L.strip_j0 = j0s;
    L.strip_len = lens;
    L.lat_cw = cw;
    return box;
}

}  // namespace

static Geometry geometry_2d(const TriMesh& mesh, const LevelSpec& spec, LevelTables& L) {
    if (spec.cells_x < 1 || spec.cells_y < 1) throw std::invalid_argument("level: coefficient grid");
    if (spec.final_time <= 0.0 || spec.dt <= 0.0) throw std::invalid_argument("level: T and dt must be positive");
    if (spec.substeps < 1) throw std::invalid_argument("level: substeps >= 1");
    const bool per_elem = spec.field == Field::LognormalKLElem;
    if (!per_elem && spec.cells_x * spec.cells_y > 32767)
        throw std::invalid_argument("level: at most 32767 coefficient cells");

    const int nv = mesh.n_vertices();
    const int nt = mesh.n_triangles();
    L.n_cells = per_elem ? nt : spec.cells_x * spec.cells_y;

    Geometry g;
    g.nv = nv;
    g.boundary = mesh.boundary_vertex;
    // lumped mass and element stiffness by cell (fem.cpp:91-116)
    std::vector<double>& mass = g.mass;
    mass.assign(nv, 0.0);
    StiffMap& stiff = g.stiff;  // (vi, vj, cell) -> sum area*grad.grad
    L.elem_cell.resize(nt);
    for (int t = 0; t < nt; ++t) {
        const auto& tri = mesh.triangles[t];
        const auto& p0 = mesh.vertices[tri[0]];
        const auto& p1 = mesh.vertices[tri[1]];
        const auto& p2 = mesh.vertices[tri[2]];
        const double area = mesh.signed_area(t);
        if (!(area > 0.0)) throw std::runtime_error("level: nonpositive triangle area");
        const auto cc = mesh.centroid(t);
        const int k = per_elem ? t : spec.cell_of(cc[0], cc[1]);
        L.elem_cell[t] = k;
        if (per_elem) {  // the field's evaluation points (capi: kl_point_table)
            L.field_x.push_back(cc[0]);
            L.field_x.push_back(cc[1]);
        }
        const double gx[3] = {(p1[1] - p2[1]) / (2.0 * area), (p2[1] - p0[1]) / (2.0 * area),
                              (p0[1] - p1[1]) / (2.0 * area)};
        const double gy[3] = {(p2[0] - p1[0]) / (2.0 * area), (p0[0] - p2[0]) / (2.0 * area),
                              (p1[0] - p0[0]) / (2.0 * area)};
        for (int i = 0; i < 3; ++i) {
            mass[tri[i]] += area / 3.0;
            if (mesh.boundary_vertex[tri[i]]) continue;
            for (int j = 0; j < 3; ++j) {
                if (mesh.boundary_vertex[tri[j]]) continue;
                stiff[{tri[i], tri[j], k}] += area * (gx[i] * gx[j] + gy[i] * gy[j]);
            }
        }
    }

    // selector: interior vertices of fine-flagged triangles (fem.cpp:119-122);
    // with nested tiers, vertex tier vt = largest flag of its triangles and
    // P_k = {vt >= k}
    if (spec.tiers < 1 || spec.tiers > 8) throw std::invalid_argument("level: tiers in [1, 8]");
    if (spec.tiers > 1 && (spec.kind != Integrator::LocalTimeStepping || spec.substeps < 2))
        throw std::invalid_argument("level: nested tiers need local time stepping with p >= 2");
    std::vector<std::uint8_t>& sel = g.sel;
    std::vector<std::uint8_t>& vt = g.vt;
    sel.assign(nv, 0);
    vt.assign(nv, 0);
    for (int t = 0; t < nt; ++t)
        if (mesh.fine_flags[t])
            for (int v : mesh.triangles[t])
                if (!mesh.boundary_vertex[v]) {
                    sel[v] = 1;
                    vt[v] = std::max<std::uint8_t>(vt[v], std::min<int>(mesh.fine_flags[t], spec.tiers));
                }

    // initial data: lumped L2 projection with the edge-midpoint rule, then
    // z0 = sqrt(M) coef (fem.cpp:223-241, :243-255); v0 = 0
    std::vector<double> load(nv, 0.0);
    auto u0 = [&](double x, double y) {
        const double dx = x - spec.ic.x0, dy = y - spec.ic.y0;
        return std::exp(-(dx * dx + dy * dy) / spec.ic.width2);
    };
    for (int t = 0; t < nt; ++t) {
        const auto& tri = mesh.triangles[t];
        const double area = mesh.signed_area(t);
        for (int e = 0; e < 3; ++e) {
            const auto& a = mesh.vertices[tri[e]];
            const auto& b = mesh.vertices[tri[(e + 1) % 3]];
            const double value = u0(0.5 * (a[0] + b[0]), 0.5 * (a[1] + b[1]));
            load[tri[e]] += area / 3.0 * value * 0.5;
            load[tri[(e + 1) % 3]] += area / 3.0 * value * 0.5;
        }
    }
    g.coef0.resize(nv);
    for (int v = 0; v < nv; ++v) g.coef0[v] = load[v] / mass[v];

    // QoI: lumped quadrature of u(T) over the triangles whose centroid lies
    // in the box, Q = sum_i w_i u_i with u = z / sqrt(M) (fem.cpp:271-275)
    std::vector<double> qw(nv, 0.0);
    for (int t = 0; t < nt; ++t) {
        const auto cc = mesh.centroid(t);
        if (cc[0] < spec.qoi.x0 || cc[0] > spec.qoi.x1 || cc[1] < spec.qoi.y0 || cc[1] > spec.qoi.y1) continue;
        const double area = mesh.signed_area(t);
        for (int v : mesh.triangles[t]) qw[v] += area / 3.0;
    }
    if (spec.qoi_mean) {  // mean over the box: divide by the area of its triangles
        double total = 0.0;
        for (int v = 0; v < nv; ++v) total += qw[v];
        if (!(total > 0.0)) throw std::invalid_argument("level: QoI box contains no triangle");
        for (int v = 0; v < nv; ++v) qw[v] /= total;
    }
    // one output: the box functional, entries in DOF order (finish_tables)
    g.qoi_vertex_w = {qw};
    g.qoi_norm_w = {1.0};
    g.qoi_dof_order = true;
    return g;
}


static LevelTables finish_tables(Geometry& g, const LevelSpec& spec, LevelTables& L, const TriMesh* mesh) {
    const int nv = g.nv;
    const std::vector<double>& mass = g.mass;
    const StiffMap& stiff = g.stiff;
    const std::vector<std::uint8_t>& sel = g.sel;
    const std::vector<std::uint8_t>& vt = g.vt;
    // rows of A P with a nonzero: R; row tier rt = deepest P_k it couples to
    std::vector<std::uint8_t> in_r(nv, 0), rt(nv, 0);
    for (const auto& [key, s] : stiff) {
        const auto [vi, vj, k] = key;
        (void)k;
        if (s != 0.0 && sel[vj]) {
            in_r[vi] = 1;
            rt[vi] = std::max(rt[vi], vt[vj]);
        }
    }
    int tiers = 1;
    if (spec.tiers > 1)
        for (int v = 0; v < nv; ++v) tiers = std::max<int>(tiers, rt[v]);
    L.tiers = tiers;

    // structured lattice block (substep fast path), decided in vertex space
    std::vector<int> box_vertex;  // (m+1)^2 box nodes in (j, i) order, or empty
    if (spec.kind == Integrator::LocalTimeStepping && tiers == 1)
        if (mesh) box_vertex = lattice_block(*mesh, spec, mass, stiff, in_r, L);

    // dof order: the lattice box (row-major), the other R rows (deepest tier
    // first), then the rest, each in mesh vertex order
    std::vector<int> vdof(nv, -1);
    for (int v : box_vertex) {
        vdof[v] = static_cast<int>(L.dof_vertex.size());
        L.dof_vertex.push_back(v);
        ++L.n_r;
    }
    for (int pass = tiers; pass >= 0; --pass)
        for (int v = 0; v < nv; ++v) {
            if (g.boundary[v] || vdof[v] >= 0) continue;
            if (pass > 0 ? (!in_r[v] || (tiers > 1 && rt[v] != pass) || (tiers == 1 && pass != 1)) : in_r[v])
                continue;
            vdof[v] = static_cast<int>(L.dof_vertex.size());
            L.dof_vertex.push_back(v);
            if (pass > 0) ++L.n_r;
        }
    L.n_r_tier.assign(tiers, 0);
    for (int k = 1; k <= tiers; ++k)
        for (int v = 0; v < nv; ++v)
            if (!g.boundary[v] && in_r[v] && (tiers == 1 || rt[v] >= k)) ++L.n_r_tier[k - 1];
    L.n = static_cast<int>(L.dof_vertex.size());
    if (L.n == 0) throw std::invalid_argument("level: mesh has no interior vertices");
    if (L.box) {  // box-local lattice coordinates of every dof (tiled step kernel)
        L.dof_lx.resize(L.n);
        L.dof_ly.resize(L.n);
        for (int i = 0; i < L.n; ++i) {
            L.dof_lx[i] = mesh->lattice[L.dof_vertex[i]][0] - mesh->fine_box_lo;
            L.dof_ly[i] = mesh->lattice[L.dof_vertex[i]][1] - mesh->fine_box_lo;
        }
    }
    // the reference's stored entries: from_triplets keeps every (row, col)
    // pair an element couples, zero sums included (include/wavemc/sparse.hpp:17-40),
    // restricted to interior rows and columns; a_fine keeps the P columns
    {
        long full = 0, fine = 0;
        int pi = -1, pj = -1;
        for (const auto& [key, s] : stiff) {  // ordered by (vi, vj, cell)
            const auto [vi, vj, k] = key;
            (void)s;
            (void)k;
            if (vi == pi && vj == pj) continue;
            pi = vi;
            pj = vj;
            if (g.boundary[vi] || g.boundary[vj]) continue;
            ++full;
            if (sel[vj]) ++fine;
        }
        L.ref_nnz = full;
        L.ref_nnz_fine = fine;
    }
    L.in_p.assign(L.n, 0);
    L.dof_tier.assign(L.n, 0);
    L.mass.resize(L.n);
    for (int i = 0; i < L.n; ++i) {
        L.in_p[i] = sel[L.dof_vertex[i]];
        L.dof_tier[i] = tiers > 1 ? vt[L.dof_vertex[i]] : sel[L.dof_vertex[i]];
        L.n_p += L.in_p[i];
        L.mass[i] = mass[L.dof_vertex[i]];
    }

    // row-wise parts: (row, col, cell) -> a0 = s / sqrt(M_i M_j)  (fem.cpp:59-63)
    std::vector<std::vector<std::tuple<int, int, double>>> rows(L.n);
    for (const auto& [key, s] : stiff) {
        const auto [vi, vj, k] = key;
        if (s == 0.0) continue;
        const int i = vdof[vi], j = vdof[vj];
        rows[i].emplace_back(j, k, (g.unit_cells && k > 0) ? 1.0 : s / std::sqrt(mass[vi] * mass[vj]));
    }
    // sweep tables: each row's entries in column order (cell-split entries
    // of one column adjacent)
    L.row_ptr.assign(L.n + 1, 0);
    for (int i = 0; i < L.n; ++i) {
        auto& r = rows[i];
        std::sort(r.begin(), r.end());
        for (const auto& [j, k, a] : r) {
            L.col.push_back(j);
            L.cell.push_back(k);
            L.a0.push_back(a);
        }
        L.row_ptr[i + 1] = static_cast<int>(L.col.size());
    }

    // A P on R rows, parts form (HBM-resident and fused small-mesh paths);
    // col | cell << 23, or << 16 when there are more than 511 cells
    L.apg_col_bits = 23;
    if (L.n_cells > 511) {  // as many column bits as the DOFs need (at least 16), the rest for cells
        L.apg_col_bits = 16;
        while ((1L << L.apg_col_bits) < L.n) ++L.apg_col_bits;
        if (L.apg_col_bits > 31 || static_cast<long>(L.n_cells) > (1L << (32 - L.apg_col_bits)))
            L.apg_col_bits = 0;  // no packed form (the HBM-resident paths refuse such levels)
    }
    L.apg_ptr.assign(L.n_r + 1, 0);
    const bool apg_unpacked = L.n_cells > 511;  // the HBM-resident substep kernel reads (column, cell) apart
    for (int i = 0; i < L.n_r && (L.apg_col_bits > 0 || apg_unpacked); ++i) {
        for (const auto& [j, k, a] : rows[i]) {
            if (!L.in_p[j]) continue;
            if (L.apg_col_bits > 0)
                L.apg_ent.push_back(static_cast<int>(static_cast<unsigned>(j) |
                                                     (static_cast<unsigned>(k) << L.apg_col_bits)));
            if (apg_unpacked) {
                L.apg_col.push_back(j);
                L.apg_cell.push_back(k);
            }
            L.apg_a0.push_back(a);
        }
        L.apg_ptr[i + 1] = static_cast<int>(L.apg_a0.size());
    }

    // nested tiers: A P_k on R_k rows, parts form
    if (tiers > 1) {
        for (int k = 1; k <= tiers; ++k) {
            std::vector<int> ptr{0}, ent;
            std::vector<double> a0;
            for (int i = 0; i < L.n_r_tier[k - 1]; ++i) {
                for (const auto& [j, c, a] : rows[i]) {
                    if (vt[L.dof_vertex[j]] < k) continue;
                    ent.push_back(j | (c << 23));  // kColBits
                    a0.push_back(a);
                }
                ptr.push_back(static_cast<int>(ent.size()));
            }
            L.tier_ptr.push_back(std::move(ptr));
            L.tier_ent.push_back(std::move(ent));
            L.tier_a0.push_back(std::move(a0));
        }
    }

    // A P on R rows as deduplicated recipes
    std::map<std::vector<std::pair<int, double>>, int> recipe_id;
    std::vector<std::vector<std::pair<int, double>>> recipes;
    L.ap_row_ptr.assign(L.n_r + 1, 0);
    for (int i = 0; i < L.n_r; ++i) {
        const auto& r = rows[i];
        for (std::size_t e = 0; e < r.size();) {
            const int j = std::get<0>(r[e]);
            std::vector<std::pair<int, double>> terms;
            while (e < r.size() && std::get<0>(r[e]) == j) {
                terms.emplace_back(std::get<1>(r[e]), std::get<2>(r[e]));
                ++e;
            }
            if (!L.in_p[j]) continue;
            auto it = recipe_id.find(terms);
            int wid;
            if (it == recipe_id.end()) {
                wid = static_cast<int>(recipes.size());
                recipe_id.emplace(terms, wid);
                recipes.push_back(terms);
            } else {
                wid = it->second;
            }
            L.ap_col.push_back(j);
            L.ap_wid.push_back(wid);
        }
        L.ap_row_ptr[i + 1] = static_cast<int>(L.ap_col.size());
    }
    if (L.lattice) {
        const int W = L.lat_m + 1;
        L.gen_ptr.push_back(0);
        L.gen_rc_ptr.push_back(0);
        for (int i = 0; i < L.n_r; ++i) {
            const int bi = i / W, bj = i % W;  // column-major box
            if (i < W * W && bi >= 1 && bi <= L.lat_m - 1 && bj >= 1 && bj <= L.lat_m - 1 && L.lat_row[bj])
                continue;  // a lattice node
            L.gen_rows.push_back(i);
            L.gen_rs.push_back(1.0 / std::sqrt(L.mass[i]));
            const auto& r = rows[i];
            for (std::size_t e = 0; e < r.size();) {
                const int j = std::get<0>(r[e]);
                const std::size_t e0 = e;
                while (e < r.size() && std::get<0>(r[e]) == j) ++e;
                if (!L.in_p[j]) continue;
                L.gen_col.push_back(j);
                const double sq = std::sqrt(L.mass[j]);
                for (std::size_t t = e0; t < e; ++t) {
                    L.gen_rc_cell.push_back(std::get<1>(r[t]));
                    L.gen_rc_a0.push_back(std::get<2>(r[t]) * sq);
                }
                L.gen_rc_ptr.push_back(static_cast<int>(L.gen_rc_cell.size()));
            }
            L.gen_ptr.push_back(static_cast<int>(L.gen_col.size()));
        }
    }
    L.rc_ptr.assign(recipes.size() + 1, 0);
    for (std::size_t w = 0; w < recipes.size(); ++w) {
        for (const auto& [k, a] : recipes[w]) {
            L.rc_cell.push_back(k);
            L.rc_a0.push_back(a);
        }
        L.rc_ptr[w + 1] = static_cast<int>(L.rc_cell.size());
    }

    // initial data z0 = sqrt(M) coef (fem.cpp:243-255); v0 = 0
    L.z0.resize(L.n);
    for (int i = 0; i < L.n; ++i) {
        const int v = L.dof_vertex[i];
        L.z0[i] = std::sqrt(mass[v]) * g.coef0[v];
    }
    // QoI tables: output k's entries (DOF order for the box functional, the
    // given order for explicit entry lists)
    L.nq = g.qoi_dof_order ? 1 : static_cast<int>(g.qoi_entries.size());
    L.qoi_norm_w = g.qoi_norm_w;
    L.qoi_ptr.assign(1, 0);
    std::vector<int> vdof_of(nv, -1);
    for (int i = 0; i < L.n; ++i) vdof_of[L.dof_vertex[i]] = i;
    if (g.qoi_dof_order) {
        const auto& qw = g.qoi_vertex_w[0];
        for (int i = 0; i < L.n; ++i) {
            const int v = L.dof_vertex[i];
            if (qw[v] != 0.0) {
                L.qoi_dof.push_back(i);
                L.qoi_w.push_back(qw[v]);
                L.sqrt_mass_qoi.push_back(std::sqrt(mass[v]));
            }
        }
        L.qoi_ptr.push_back(static_cast<int>(L.qoi_dof.size()));
    } else {
        for (const auto& out : g.qoi_entries) {
            for (const auto& [v, w] : out) {
                if (vdof_of[v] < 0) continue;  // a Dirichlet vertex: u = 0
                L.qoi_dof.push_back(vdof_of[v]);
                L.qoi_w.push_back(w);
                L.sqrt_mass_qoi.push_back(std::sqrt(mass[v]));
            }
            L.qoi_ptr.push_back(static_cast<int>(L.qoi_dof.size()));
        }
    }

    // time stepping (integrators.cpp:176-210, :117-157)
    L.kind = spec.kind;
    L.n_steps = static_cast<long>(std::ceil(spec.final_time / spec.dt - 1e-12));
    L.dt = spec.final_time / static_cast<double>(L.n_steps);
    const double dt = L.dt;
    L.init_factor = 0.5 * dt * dt;
    if (spec.kind == Integrator::Leapfrog) {
        L.p = 1;
        L.coarse_factor = dt * dt;
        L.n_r = L.n_r;  // R is still reported; every row takes the leapfrog update
    } else {
        const int p = spec.substeps;
        L.p = p;
        const ChebyshevConstants cc = chebyshev_constants(p, spec.nu);
        const double tau2 = (dt / p) * (dt / p);
        L.c0 = 0.5 * tau2 * 2.0 * p * p / (cc.omega * cc.delta);
        L.beta = cc.beta_int;
        L.cm.resize(p - 1);
        for (int m = 1; m <= p - 1; ++m) L.cm[m - 1] = tau2 * 2.0 * p * p / cc.omega * cc.beta_half[m - 1];
        // the recursion with A P d == 0 and unit forcing: d_p = -kappa
        double dprev = 0.0, dcur = -L.c0 * 1.0;
        for (int m = 1; m <= p - 1; ++m) {
            const double next = (1.0 + L.beta[m - 1]) * dcur - L.beta[m - 1] * dprev - L.cm[m - 1] * 1.0;
            dprev = dcur;
            dcur = next;
        }
        L.coarse_factor = -2.0 * dcur;
        if (tiers > 1) {
            double dt_k = dt;  // tier k advances in steps of dt / p^k; its interval is dt_k = dt / p^(k-1)
            for (int k = 1; k <= tiers; ++k) {
                const double tk2 = (dt_k / p) * (dt_k / p);
                L.tier_c0.push_back(0.5 * tk2 * 2.0 * p * p / (cc.omega * cc.delta));
                std::vector<double> cmk(p - 1);
                for (int m = 1; m <= p - 1; ++m) cmk[m - 1] = tk2 * 2.0 * p * p / cc.omega * cc.beta_half[m - 1];
                L.tier_cm.push_back(cmk);
                L.tier_back.push_back(-2.0 / (dt_k * dt_k));
                dt_k /= p;
            }
        }
    }
    L.p_fine = 1;
    for (int k = 0; k < L.tiers; ++k) L.p_fine *= L.p;
    L.cfl_safety = spec.cfl_safety;
    if (spec.cfl_safety > 0.0) {
        // power iteration as reference max_eigenvalue (src/fem.cpp:132-175):
        // mix64 start vector, tol 1e-4, three settled Rayleigh quotients
        std::vector<double> a1;  // c = 1 operator, one value per stored (row, col)
        std::vector<int> c1, p1{0};
        for (int i = 0; i < L.n; ++i) {
            for (int e = L.row_ptr[i]; e < L.row_ptr[i + 1];) {
                const int j = L.col[e];
                double v = 0.0;
                for (; e < L.row_ptr[i + 1] && L.col[e] == j; ++e)
                    v += g.cell_ref.empty() ? L.a0[e] : g.cell_ref[L.cell[e]] * L.a0[e];
                c1.push_back(j);
                a1.push_back(v);
            }
            p1.push_back(static_cast<int>(c1.size()));
        }
        // the start vector is keyed by the reference's DOF index (interior
        // vertices in vertex order), not by this level's DOF permutation
        std::vector<int> ref_index(nv, -1);
        for (int v = 0, k = 0; v < nv; ++v)
            if (!g.boundary[v]) ref_index[v] = k++;
        auto power = [&](bool coarse) {
            const int n = L.n;
            std::vector<double> v(n), av(n);
            for (int i = 0; i < n; ++i)
                v[i] = static_cast<double>(
                           mix64_host(static_cast<std::uint64_t>(ref_index[L.dof_vertex[i]]) + 1) >> 11) *
                           0x1.0p-53 -
                       0.5;
            double norm = 0.0;
            for (double x : v) norm += x * x;
            norm = std::sqrt(norm);
            if (norm == 0.0) {
                v[0] = 1.0;
                norm = 1.0;
            }
            for (double& x : v) x /= norm;
            double prev = 0.0;
            int settled = 0;
            for (int it = 1; it <= 20000; ++it) {
                for (int i = 0; i < n; ++i) {
                    double acc = 0.0;
                    if (!(coarse && L.in_p[i]))
                        for (int e = p1[i]; e < p1[i + 1]; ++e)
                            if (!(coarse && L.in_p[c1[e]])) acc += a1[e] * v[c1[e]];
                    av[i] = acc;
                }
                double ray = 0.0, nn = 0.0;
                for (int i = 0; i < n; ++i) ray += v[i] * av[i];
                for (int i = 0; i < n; ++i) nn += av[i] * av[i];
                const double avn = std::sqrt(nn);
                if (avn == 0.0) return v;
                for (int i = 0; i < n; ++i) v[i] = av[i] / avn;
                if (std::abs(ray - prev) <= 1e-4 * std::abs(ray)) {
                    if (++settled >= 3) return v;
                } else {
                    settled = 0;
                }
                prev = ray;
            }
            throw std::runtime_error("level: warm-start power iteration did not converge");
        };
        L.warm_full = power(false);
        if (spec.kind == Integrator::LocalTimeStepping && L.n_p > 0) L.warm_coarse = power(true);
    }
    return L;
}


LevelTables build_level_tables(const TriMesh& mesh, const LevelSpec& spec) {
    LevelTables L;
    Geometry g = geometry_2d(mesh, spec, L);
    return finish_tables(g, spec, L, &mesh);
}

LevelTables build_level_tables_1d(const Mesh1D& mesh, const LevelSpec& spec) {
    if (spec.final_time <= 0.0 || spec.dt <= 0.0) throw std::invalid_argument("level: T and dt must be positive");
    if (spec.grid_n < 2 || !(spec.grid_hi > spec.grid_lo)) throw std::invalid_argument("level: bad output grid");
    const int ne = mesh.n_elements(), nv = mesh.n_vertices();
    if (ne < 1) throw std::invalid_argument("level: empty 1D mesh");
    LevelTables L;
    L.n_cells = ne;
    Geometry g;
    g.nv = nv;
    g.boundary.assign(nv, 0);  // the reference's experiments are Neumann
    g.mass.assign(nv, 0.0);
    g.sel.assign(nv, 0);
    for (int e = 0; e < ne; ++e) {
        const double h = mesh.element_size(e);
        const double k = 1.0 / h;  // times c_e^2 per sample
        g.stiff[{e, e, e}] += k;
        g.stiff[{e + 1, e + 1, e}] += k;
        g.stiff[{e, e + 1, e}] += -k;
        g.stiff[{e + 1, e, e}] += -k;
        g.mass[e] += 0.5 * h;
        g.mass[e + 1] += 0.5 * h;
        if (mesh.fine_flags[e]) g.sel[e] = g.sel[e + 1] = 1;
        L.field_x.push_back(mesh.midpoint(e));
    }
    g.vt = g.sel;
    // u0 = exp(-(x - x0)^2 / width2) by two-point Gauss on every element
    std::vector<double> load(nv, 0.0);
    for (int e = 0; e < ne; ++e) {
        const double lo = mesh.vertices[e], hi = mesh.vertices[e + 1];
        const double h = hi - lo;
        const double mid = 0.5 * (lo + hi), off = 0.5 * (hi - lo) / std::sqrt(3.0);
        for (double x : {mid - off, mid + off}) {
            const double f = std::exp(-(x - spec.ic.x0) * (x - spec.ic.x0) / spec.ic.width2);
            const double phi_right = (x - lo) / h;
            load[e] += 0.5 * h * f * (1.0 - phi_right);
            load[e + 1] += 0.5 * h * f * phi_right;
        }
    }
    g.coef0.resize(nv);
    for (int v = 0; v < nv; ++v) g.coef0[v] = load[v] / g.mass[v];
    // restrict_to_grid: linear interpolation at the grid points, trapezoid norm weights
    const double glo = spec.grid_lo, ghi = spec.grid_hi;
    const int gn = spec.grid_n;
    const double spacing = (ghi - glo) / (gn - 1);
    const double lo = mesh.vertices.front(), hi = mesh.vertices.back();
    for (int i = 0; i < gn; ++i) {
        double x = i == gn - 1 ? ghi : glo + spacing * i;
        if (x < lo - 1e-9 || x > hi + 1e-9) throw std::invalid_argument("level: output grid outside the mesh");
        x = std::clamp(x, lo, hi);
        const auto it = std::upper_bound(mesh.vertices.begin(), mesh.vertices.end(), x);
        int e = static_cast<int>(it - mesh.vertices.begin()) - 1;
        e = std::clamp(e, 0, ne - 1);
        const double t = (x - mesh.vertices[e]) / mesh.element_size(e);
        g.qoi_entries.push_back({{e, 1.0 - t}, {e + 1, t}});
        g.qoi_norm_w.push_back((i == 0 || i == gn - 1) ? 0.5 * spacing : spacing);
    }
    // the reference's KL field (rng.cpp:64-77): amp_k = 1 / (4 pi^2 k^2),
    // arg = k pi x / 6, c^2 = 1 + sum_k amp (cos arg xi_k + sin arg eta_k)
    if (spec.field == Field::Kl1D) {
        const int K = 100;  // kKlTerms (rng.hpp:50)
        const double pi = 3.14159265358979323846;
        L.field_terms = 2 * K;
        L.field_table.resize(static_cast<std::size_t>(ne) * 2 * K);
        for (int e = 0; e < ne; ++e)
            for (int k = 1; k <= K; ++k) {
                const double arg = k * pi * L.field_x[e] / 6.0;
                const double amp = 1.0 / (4.0 * pi * pi * k * k);
                L.field_table[static_cast<std::size_t>(e) * 2 * K + (k - 1)] = amp * std::cos(arg);
                L.field_table[static_cast<std::size_t>(e) * 2 * K + K + (k - 1)] = amp * std::sin(arg);
            }
    }
    return finish_tables(g, spec, L, nullptr);
}

double dof_updates_per_solve(const LevelTables& t) {
    const double n = t.n;
    if (t.kind == Integrator::Leapfrog) return static_cast<double>(t.n_steps) * n;
    if (t.tiers > 1) {
        double per_step = n, pk = 1.0;
        for (int k = 1; k <= t.tiers; ++k) {
            per_step += (pk * t.p - pk) * static_cast<double>(t.n_r_tier[k - 1]);
            pk *= t.p;
        }
        return n + static_cast<double>(t.n_steps - 1) * per_step;
    }
    return n + static_cast<double>(t.n_steps - 1) * (n + (t.p - 1) * static_cast<double>(t.n_r));
}


// ---------------------------------------------------------------------------
// Narrow-channel experiment (see channel.hpp)

double channel_blend(double x) {  // src/mesh2d.cpp:361-367
    const double a = std::abs(x);
    if (a <= kChannelHalfLength) return 1.0;
    if (a >= kChannelBlendOuter) return 0.0;
    return 0.5 * (1.0 + std::cos(3.14159265358979323846 * (a - kChannelHalfLength) /
                                 (kChannelBlendOuter - kChannelHalfLength)));
}

double channel_profile(double y, double width) {  // src/mesh2d.cpp:369-377
    const double half_ref = 0.5 * kChannelRefWidth;
    const double peak = 0.5 * (width - kChannelRefWidth);
    const double a = std::abs(y);
    double value;
    if (a <= half_ref)
        value = peak * (a / half_ref);
    else
        value = peak * (kChannelRectHalfHeight - a) / (kChannelRectHalfHeight - half_ref);
    return y < 0.0 ? -value : value;
}

LevelTables build_level_tables_channel(const TriMesh& mesh, const LevelSpec& spec, ChannelTables& ch) {
    if (spec.final_time <= 0.0 || spec.dt <= 0.0) throw std::invalid_argument("level: T and dt must be positive");
    if (spec.substeps < 1) throw std::invalid_argument("level: substeps >= 1");
    if (spec.tiers != 1) throw std::invalid_argument("channel: single-tier LTS only");
    if (spec.grid_n < 2) throw std::invalid_argument("channel: grid_n >= 2");
    LevelTables L;
    const int nv = mesh.n_vertices();
    const int nt = mesh.n_triangles();
    // moving vertices: blend(x) profile(y) != 0 for a width other than the
    // reference one (profile vanishes on y = 0 and |y| = 1/2 only)
    std::vector<std::uint8_t> moving(nv, 0), tri_mov(nt, 0), mass_mov(nv, 0);
    for (int v = 0; v < nv; ++v)
        moving[v] = channel_blend(mesh.vertices[v][0]) != 0.0 &&
                    channel_profile(mesh.vertices[v][1], kChannelWidthLo) != 0.0;
    for (int t = 0; t < nt; ++t) {
        for (int v : mesh.triangles[t]) tri_mov[t] |= moving[v];
        if (tri_mov[t])
            for (int v : mesh.triangles[t]) mass_mov[v] = 1;
    }

    Geometry g;
    g.nv = nv;
    g.boundary.assign(nv, 0);  // Neumann: assemble(transformed mesh), no restriction (experiments.cpp:158)
    g.unit_cells = true;
    g.mass.assign(nv, 0.0);
    std::vector<double> ms(nv, 0.0);  // mass of fixed triangles only
    std::map<std::pair<int, int>, double> kref, kfix;  // reference stiffness: all / fixed triangles
    auto elem = [&](int t, double* gx, double* gy) {  // assemble, fem.cpp:97-116 (speed^2 = 1)
        const auto& tri = mesh.triangles[t];
        const auto& p0 = mesh.vertices[tri[0]];
        const auto& p1 = mesh.vertices[tri[1]];
        const auto& p2 = mesh.vertices[tri[2]];
        const double area = mesh.signed_area(t);
        if (!(area > 0.0)) throw std::runtime_error("channel: nonpositive triangle area");
        gx[0] = (p1[1] - p2[1]) / (2.0 * area);
        gx[1] = (p2[1] - p0[1]) / (2.0 * area);
        gx[2] = (p0[1] - p1[1]) / (2.0 * area);
        gy[0] = (p2[0] - p1[0]) / (2.0 * area);
        gy[1] = (p0[0] - p2[0]) / (2.0 * area);
        gy[2] = (p1[0] - p0[0]) / (2.0 * area);
        return area;
    };
    std::map<std::pair<int, int>, int> cell_of;  // unordered per-sample pair -> cell
    for (int t = 0; t < nt; ++t) {
        double gx[3], gy[3];
        const double area = elem(t, gx, gy);
        const auto& tri = mesh.triangles[t];
        for (int i = 0; i < 3; ++i) {
            g.mass[tri[i]] += area / 3.0;
            if (!tri_mov[t]) ms[tri[i]] += area / 3.0;
            for (int j = 0; j < 3; ++j) {
                const double kij = 1.0 * area * (gx[i] * gx[j] + gy[i] * gy[j]);
                kref[{tri[i], tri[j]}] += kij;
                if (!tri_mov[t]) kfix[{tri[i], tri[j]}] += kij;
                const int a = std::min(tri[i], tri[j]), b = std::max(tri[i], tri[j]);
                if (tri_mov[t] || mass_mov[a] || mass_mov[b]) cell_of[{a, b}] = 0;
            }
        }
    }
    int next_cell = 1;
    for (auto& kv : cell_of) kv.second = next_cell++;
    L.n_cells = next_cell;
    // the stiffness map: fixed pairs by element (cell 0), per-sample pairs as
    // one unit entry of their cell
    for (int t = 0; t < nt; ++t) {
        double gx[3], gy[3];
        const double area = elem(t, gx, gy);
        const auto& tri = mesh.triangles[t];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                const int a = std::min(tri[i], tri[j]), b = std::max(tri[i], tri[j]);
                const auto it = cell_of.find({a, b});
                if (it != cell_of.end())
                    g.stiff[{tri[i], tri[j], it->second}] = 1.0;
                else
                    g.stiff[{tri[i], tri[j], 0}] += 1.0 * area * (gx[i] * gx[j] + gy[i] * gy[j]);
            }
    }
    g.cell_ref.assign(L.n_cells, 1.0);
    for (const auto& [ab, k] : cell_of)
        g.cell_ref[k] = kref[ab] / std::sqrt(g.mass[ab.first] * g.mass[ab.second]);

    // selector: vertices of fine-flagged triangles (fem.cpp:119-122)
    g.sel.assign(nv, 0);
    g.vt.assign(nv, 0);
    for (int t = 0; t < nt; ++t)
        if (mesh.fine_flags[t])
            for (int v : mesh.triangles[t]) g.sel[v] = g.vt[v] = 1;

    // u0 = bump (experiments.cpp:118-124) by the edge-midpoint lumped
    // projection (fem.cpp:223-241); its support (|(x - 1/2, y)| < 0.2) lies
    // where the geometry never moves, so z0 is sample-independent
    auto u0 = [](double x, double y) {
        constexpr double radius = 0.2;
        const double dx = x - 0.5;
        const double rho2 = dx * dx + y * y;
        if (rho2 >= radius * radius) return 0.0;
        return std::exp(1.0 - radius * radius / (radius * radius - rho2));
    };
    std::vector<double> load(nv, 0.0);
    for (int t = 0; t < nt; ++t) {
        const auto& tri = mesh.triangles[t];
        const double area = mesh.signed_area(t);
        for (int e = 0; e < 3; ++e) {
            const auto& a = mesh.vertices[tri[e]];
            const auto& b = mesh.vertices[tri[(e + 1) % 3]];
            const double value = u0(0.5 * (a[0] + b[0]), 0.5 * (a[1] + b[1]));
            load[tri[e]] += area / 3.0 * value * 0.5;
            load[tri[(e + 1) % 3]] += area / 3.0 * value * 0.5;
        }
    }
    g.coef0.resize(nv);
    for (int v = 0; v < nv; ++v) {
        g.coef0[v] = load[v] / g.mass[v];
        if (g.coef0[v] != 0.0 && mass_mov[v]) throw std::runtime_error("channel: u0 support meets the moving region");
    }

    // QoI: u(T) on the line x = -0.4 at the grid points of [-1/2, 1/2]
    // (extract_line_qoi, fem.cpp:295-340): the first candidate triangle (in
    // mesh order, x-range containing the line) holding the point, else the
    // least-missed one; barycentric weights on its corners.  The line lies
    // where the geometry never moves.
    std::vector<int> cand;
    for (int t = 0; t < nt; ++t) {
        double xmin = 1e30, xmax = -1e30;
        for (int v : mesh.triangles[t]) {
            xmin = std::min(xmin, mesh.vertices[v][0]);
            xmax = std::max(xmax, mesh.vertices[v][0]);
        }
        if (xmin - 1e-12 <= kChannelLineX && kChannelLineX <= xmax + 1e-12) cand.push_back(t);
    }
    const double lo = -kChannelRectHalfHeight, hi = kChannelRectHalfHeight;
    const int n_out = spec.grid_n;
    const double spacing = (hi - lo) / (n_out - 1);
    g.qoi_entries.resize(n_out);
    g.qoi_norm_w.resize(n_out);
    for (int i = 0; i < n_out; ++i) {
        const double y = i == n_out - 1 ? hi : lo + spacing * i;  // OutputGrid::point
        g.qoi_norm_w[i] = (i == 0 || i == n_out - 1) ? 0.5 * spacing : spacing;
        double best_miss = 1e30;
        std::vector<std::pair<int, double>> best;
        bool found = false;
        for (int t : cand) {
            const auto& tri = mesh.triangles[t];
            const auto& p0 = mesh.vertices[tri[0]];
            const auto& p1 = mesh.vertices[tri[1]];
            const auto& p2 = mesh.vertices[tri[2]];
            const double x = kChannelLineX;
            const double area2 = (p1[0] - p0[0]) * (p2[1] - p0[1]) - (p2[0] - p0[0]) * (p1[1] - p0[1]);
            const double l0 = ((p1[0] - x) * (p2[1] - y) - (p2[0] - x) * (p1[1] - y)) / area2;
            const double l1 = ((p2[0] - x) * (p0[1] - y) - (p0[0] - x) * (p2[1] - y)) / area2;
            const double l2 = 1.0 - l0 - l1;
            const double miss = -std::min({l0, l1, l2});
            if (miss < best_miss) {
                best_miss = miss;
                best = {{tri[0], l0}, {tri[1], l1}, {tri[2], l2}};
            }
            if (miss <= 1e-9) {
                found = true;
                break;
            }
        }
        if (!found && best_miss > 1e-6) throw std::runtime_error("channel: QoI point outside the mesh");
        for (const auto& [v, w] : best)
            if (mass_mov[v]) throw std::runtime_error("channel: QoI line meets the moving region");
        g.qoi_entries[i] = best;
    }

    // device tables of the per-sample entries
    std::vector<int> loc(nv, -1);
    for (int v = 0; v < nv; ++v)
        if (mass_mov[v]) {
            loc[v] = ch.n_local++;
            ch.vx.push_back(mesh.vertices[v][0]);
            ch.vy.push_back(mesh.vertices[v][1]);
            ch.vblend.push_back(channel_blend(mesh.vertices[v][0]));
            ch.ms.push_back(ms[v]);
        }
    std::vector<int> tloc(nt, -1);
    std::vector<std::vector<int>> vtri(ch.n_local);
    for (int t = 0; t < nt; ++t)
        if (tri_mov[t]) {
            tloc[t] = static_cast<int>(ch.tri.size() / 3);
            for (int v : mesh.triangles[t]) {
                ch.tri.push_back(loc[v]);
                vtri[loc[v]].push_back(tloc[t]);
            }
        }
    ch.m_ptr.assign(1, 0);
    for (int l = 0; l < ch.n_local; ++l) {
        ch.m_tri.insert(ch.m_tri.end(), vtri[l].begin(), vtri[l].end());
        ch.m_ptr.push_back(static_cast<int>(ch.m_tri.size()));
    }
    std::vector<std::vector<int>> pair_tri(L.n_cells);
    for (int t = 0; t < nt; ++t) {
        if (!tri_mov[t]) continue;
        const auto& tri = mesh.triangles[t];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                if (tri[a] <= tri[b]) pair_tri[cell_of.at({tri[a], tri[b]})].push_back(tloc[t] * 9 + a * 3 + b);
    }
    ch.k_ptr.assign(1, 0);
    for (const auto& [ab, k] : cell_of) {
        const auto [a, b] = ab;
        ch.e_li.push_back(loc[a]);
        ch.e_lj.push_back(loc[b]);
        ch.e_mi.push_back(g.mass[a]);
        ch.e_mj.push_back(g.mass[b]);
        const auto it = kfix.find(ab);
        ch.e_ks.push_back(it == kfix.end() ? 0.0 : it->second);
        ch.k_tri.insert(ch.k_tri.end(), pair_tri[k].begin(), pair_tri[k].end());
        ch.k_ptr.push_back(static_cast<int>(ch.k_tri.size()));
    }
    return finish_tables(g, spec, L, nullptr);
}

}  // namespace wmc
