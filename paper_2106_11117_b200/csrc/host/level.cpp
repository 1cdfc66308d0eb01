#include "level.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <stdexcept>
#include <tuple>

namespace wmc {

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

namespace {

int cell_of(double x, double y, int nx, int ny) {
    int ix = static_cast<int>(std::floor(x * nx));
    int iy = static_cast<int>(std::floor(y * ny));
    ix = std::clamp(ix, 0, nx - 1);
    iy = std::clamp(iy, 0, ny - 1);
    return iy * nx + ix;
}

}  // namespace

LevelTables build_level_tables(const TriMesh& mesh, const LevelSpec& spec) {
    if (spec.cells_x < 1 || spec.cells_y < 1) throw std::invalid_argument("level: coefficient grid");
    if (spec.final_time <= 0.0 || spec.dt <= 0.0) throw std::invalid_argument("level: T and dt must be positive");
    if (spec.substeps < 1) throw std::invalid_argument("level: substeps >= 1");
    if (spec.cells_x * spec.cells_y > 255) throw std::invalid_argument("level: at most 255 coefficient cells");

    LevelTables L;
    const int nv = mesh.n_vertices();
    const int nt = mesh.n_triangles();
    L.n_cells = spec.cells_x * spec.cells_y;

    // lumped mass and element stiffness by cell (fem.cpp:91-116)
    std::vector<double> mass(nv, 0.0);
    std::map<std::tuple<int, int, int>, double> stiff;  // (vi, vj, cell) -> sum area*grad.grad
    L.elem_cell.resize(nt);
    for (int t = 0; t < nt; ++t) {
        const auto& tri = mesh.triangles[t];
        const auto& p0 = mesh.vertices[tri[0]];
        const auto& p1 = mesh.vertices[tri[1]];
        const auto& p2 = mesh.vertices[tri[2]];
        const double area = mesh.signed_area(t);
        if (!(area > 0.0)) throw std::runtime_error("level: nonpositive triangle area");
        const auto cc = mesh.centroid(t);
        const int k = cell_of(cc[0], cc[1], spec.cells_x, spec.cells_y);
        L.elem_cell[t] = k;
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

    // selector: interior vertices of fine-flagged triangles (fem.cpp:119-122)
    std::vector<std::uint8_t> sel(nv, 0);
    for (int t = 0; t < nt; ++t)
        if (mesh.fine_flags[t])
            for (int v : mesh.triangles[t])
                if (!mesh.boundary_vertex[v]) sel[v] = 1;

    // rows of A P with a nonzero: R
    std::vector<std::uint8_t> in_r(nv, 0);
    for (const auto& [key, s] : stiff) {
        const auto [vi, vj, k] = key;
        (void)k;
        if (s != 0.0 && sel[vj]) in_r[vi] = 1;
    }

    // dof order: R rows first, then the rest, each in mesh vertex order
    std::vector<int> vdof(nv, -1);
    for (int pass = 0; pass < 2; ++pass)
        for (int v = 0; v < nv; ++v) {
            if (mesh.boundary_vertex[v]) continue;
            if ((pass == 0) != (in_r[v] != 0)) continue;
            vdof[v] = static_cast<int>(L.dof_vertex.size());
            L.dof_vertex.push_back(v);
            if (pass == 0) ++L.n_r;
        }
    L.n = static_cast<int>(L.dof_vertex.size());
    if (L.n == 0) throw std::invalid_argument("level: mesh has no interior vertices");
    L.in_p.assign(L.n, 0);
    L.mass.resize(L.n);
    for (int i = 0; i < L.n; ++i) {
        L.in_p[i] = sel[L.dof_vertex[i]];
        L.n_p += L.in_p[i];
        L.mass[i] = mass[L.dof_vertex[i]];
    }

    // row-wise parts: (row, col, cell) -> a0 = s / sqrt(M_i M_j)  (fem.cpp:59-63)
    std::vector<std::vector<std::tuple<int, int, double>>> rows(L.n);
    for (const auto& [key, s] : stiff) {
        const auto [vi, vj, k] = key;
        if (s == 0.0) continue;
        const int i = vdof[vi], j = vdof[vj];
        rows[i].emplace_back(j, k, s / std::sqrt(mass[vi] * mass[vj]));
    }
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
    L.rc_ptr.assign(recipes.size() + 1, 0);
    for (std::size_t w = 0; w < recipes.size(); ++w) {
        for (const auto& [k, a] : recipes[w]) {
            L.rc_cell.push_back(k);
            L.rc_a0.push_back(a);
        }
        L.rc_ptr[w + 1] = static_cast<int>(L.rc_cell.size());
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
    L.z0.resize(L.n);
    for (int i = 0; i < L.n; ++i) {
        const int v = L.dof_vertex[i];
        L.z0[i] = std::sqrt(mass[v]) * (load[v] / mass[v]);
    }

    // QoI: lumped quadrature of u(T) over the triangles whose centroid lies
    // in the box, Q = sum_i w_i u_i with u = z / sqrt(M) (fem.cpp:271-275)
    std::vector<double> qw(nv, 0.0);
    for (int t = 0; t < nt; ++t) {
        const auto cc = mesh.centroid(t);
        if (cc[0] < spec.qoi.x0 || cc[0] > spec.qoi.x1 || cc[1] < spec.qoi.y0 || cc[1] > spec.qoi.y1) continue;
        const double area = mesh.signed_area(t);
        for (int v : mesh.triangles[t]) qw[v] += area / 3.0;
    }
    for (int i = 0; i < L.n; ++i) {
        const int v = L.dof_vertex[i];
        if (qw[v] != 0.0) {
            L.qoi_dof.push_back(i);
            L.qoi_w.push_back(qw[v]);
            L.sqrt_mass_qoi.push_back(std::sqrt(mass[v]));
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
    }
    return L;
}

double dof_updates_per_solve(const LevelTables& t) {
    const double n = t.n;
    if (t.kind == Integrator::Leapfrog) return static_cast<double>(t.n_steps) * n;
    return n + static_cast<double>(t.n_steps - 1) * (n + (t.p - 1) * static_cast<double>(t.n_r));
}

}  // namespace wmc
