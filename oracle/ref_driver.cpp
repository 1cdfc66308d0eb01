// Oracle driver: composes the BASELINE.json problems from the UNMODIFIED
// reference library's public API (test infrastructure; see oracle/README.md).
//
// Composition:
//   mesh            load_trimesh (reference src/mesh_io.cpp:60-81) of a mesh
//                   written by the shared problem definition
//   coefficient     RngStream(seed, level, index) (src/rng.cpp:14-32),
//                   next_uniform(lo, hi) per cell in row-major cell order
//   operator        assemble(TriMesh, speed2) (src/fem.cpp:91-126), then
//                   Dirichlet by interior restriction through
//                   make_operator(mass_int, K_int, sel_int) (src/fem.cpp:42-57)
//   initial data    project_initial (src/fem.cpp:264-269), restricted
//   time stepping   run_wave with a fixed requested dt (src/integrators.cpp:176-210)
//   QoI             sum_i w_i u_i, u = nodal_values (src/fem.cpp:271-275),
//                   w_i = lumped area of the triangles with centroid in the box
//   MLMC            MlmcProblem + sample_delta_q + LevelAccumulator +
//                   estimate_variance (src/mlmc.cpp:21-73), and run_mlmc for
//                   the adaptive driver (src/mlmc.cpp:165-233)
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "wavemc/errors.hpp"
#include "wavemc/experiments.hpp"
#include "wavemc/fem.hpp"
#include "wavemc/integrators.hpp"
#include "wavemc/mesh.hpp"
#include "wavemc/mlmc.hpp"
#include "wavemc/rng.hpp"

using namespace wavemc;

namespace {

struct Args {
    std::map<std::string, std::vector<std::string>> kv;
    std::string get(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() || it->second.empty() ? def : it->second.back();
    }
    double num(const std::string& k, double def) const {
        const std::string v = get(k);
        return v.empty() ? def : std::strtod(v.c_str(), nullptr);
    }
    long integer(const std::string& k, long def) const {
        const std::string v = get(k);
        return v.empty() ? def : std::strtol(v.c_str(), nullptr, 10);
    }
    std::uint64_t u64(const std::string& k, std::uint64_t def) const {
        const std::string v = get(k);
        return v.empty() ? def : std::strtoull(v.c_str(), nullptr, 0);
    }
    const std::vector<std::string>& all(const std::string& k) const {
        static const std::vector<std::string> none;
        auto it = kv.find(k);
        return it == kv.end() ? none : it->second;
    }
};

Args parse(int argc, char** argv, int start) {
    Args a;
    for (int i = start; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) throw ConfigError("expected --key, got " + k);
        k = k.substr(2);
        std::string v = (i + 1 < argc && std::strncmp(argv[i + 1], "--", 2) != 0) ? argv[++i] : "1";
        a.kv[k].push_back(v);
    }
    return a;
}

struct ProblemDef {
    int cells_x = 4, cells_y = 4;
    double coef_lo = 0.5, coef_hi = 1.5;
    double final_time = 1.0;
    double nu = 0.01;
    Integrator kind = Integrator::LocalTimeStepping;
    double ic_x = 0.3, ic_y = 0.5, ic_w2 = 0.01;
    double box_x0 = 0.7, box_x1 = 0.9, box_y0 = 0.4, box_y1 = 0.6;
    std::vector<double> kl;  // log-normal KL table [cell * kl_modes + m] (empty: uniform cells)
    int kl_modes = 0;
    // pointwise log-normal KL (per-element field): mode m is amp * phi_x(x) * phi_y(y) with
    // phi(t) = (even ? cos : sin)(omega (t - 1/2)) / norm; rows of 7 numbers
    // (amp, omega_x, even_x, norm_x, omega_y, even_y, norm_y), from wmc_kl_modes
    std::vector<double> klp;
    double dom_x0 = 0.0, dom_x1 = 1.0, dom_y0 = 0.0, dom_y1 = 1.0;  // coefficient grid extent
    bool qoi_mean = false;   // Q = mean over the box
    double cfl = 0.0;        // > 0: per-sample dt = cfl-scaled stable step (experiments.cpp:30-43)
};

std::vector<double> num_list(const std::string& s) {
    std::vector<double> out;
    std::stringstream ss(s);
    std::string part;
    while (std::getline(ss, part, ',')) out.push_back(std::strtod(part.c_str(), nullptr));
    return out;
}

ProblemDef problem_from(const Args& a) {
    ProblemDef d;
    d.cells_x = static_cast<int>(a.integer("cells-x", 4));
    d.cells_y = static_cast<int>(a.integer("cells-y", 4));
    d.coef_lo = a.num("coef-lo", 0.5);
    d.coef_hi = a.num("coef-hi", 1.5);
    d.final_time = a.num("T", 1.0);
    d.nu = a.num("nu", 0.01);
    d.kind = a.get("kind", "lts") == "lf" ? Integrator::Leapfrog : Integrator::LocalTimeStepping;
    if (!a.get("ic").empty()) {  // x,y,width2
        const auto v = num_list(a.get("ic"));
        if (v.size() != 3) throw ConfigError("--ic x,y,width2");
        d.ic_x = v[0], d.ic_y = v[1], d.ic_w2 = v[2];
    }
    if (!a.get("box").empty()) {  // x0,x1,y0,y1
        const auto v = num_list(a.get("box"));
        if (v.size() != 4) throw ConfigError("--box x0,x1,y0,y1");
        d.box_x0 = v[0], d.box_x1 = v[1], d.box_y0 = v[2], d.box_y1 = v[3];
    }
    if (!a.get("domain").empty()) {  // coefficient grid x0,x1,y0,y1
        const auto v = num_list(a.get("domain"));
        if (v.size() != 4) throw ConfigError("--domain x0,x1,y0,y1");
        d.dom_x0 = v[0], d.dom_x1 = v[1], d.dom_y0 = v[2], d.dom_y1 = v[3];
    }
    d.qoi_mean = a.integer("qoi-mean", 0) != 0;
    d.cfl = a.num("cfl", 0.0);
    const std::string kl = a.get("kl-table");
    if (!kl.empty()) {  // "<cells> <modes>" then cells*modes values (written by the shared problem definition)
        std::ifstream in(kl);
        int cells = 0;
        in >> cells >> d.kl_modes;
        if (!in || cells != d.cells_x * d.cells_y) throw ConfigError("kl-table: header does not match the cell grid");
        d.kl.resize(static_cast<std::size_t>(cells) * d.kl_modes);
        for (double& v : d.kl) in >> v;
        if (!in) throw ConfigError("kl-table: truncated");
    }
    const std::string klm = a.get("kl-modes");
    if (!klm.empty()) {  // "<modes>" then 7 numbers per mode
        std::ifstream in(klm);
        in >> d.kl_modes;
        if (!in || d.kl_modes < 1) throw ConfigError("kl-modes: bad header");
        d.klp.resize(static_cast<std::size_t>(7) * d.kl_modes);
        for (double& v : d.klp) in >> v;
        if (!in) throw ConfigError("kl-modes: truncated");
    }
    return d;
}

// g(x, y) of the pointwise KL field for the normals xi
double kl_point_value(const ProblemDef& d, const std::vector<double>& xi, double x, double y) {
    auto phi = [](double omega, double even, double norm, double t) {
        return (even != 0.0 ? std::cos(omega * t) : std::sin(omega * t)) / norm;
    };
    double g = 0.0;
    for (int m = 0; m < d.kl_modes; ++m) {
        const double* r = d.klp.data() + 7 * m;
        g += (r[0] * phi(r[1], r[2], r[3], x - 0.5) * phi(r[4], r[5], r[6], y - 0.5)) * xi[m];
    }
    return g;
}

// one level: mesh + interior restriction + sample-independent data
struct Level {
    TriMesh mesh;
    std::vector<int> interior;        // interior vertex ids in vertex order
    std::vector<int> dof_of;          // vertex -> dof or -1
    std::vector<double> qoi_w;        // per dof
    InitialData init;                 // restricted to dofs
    double dt = 0.0;
    int substeps = 1;
    long n_r = 0;                     // rows of A P with entries (for DOF-update counts)
    long n_steps = 0;
    std::vector<double> warm_full, warm_coarse;  // per-sample CFL: c = 1 eigenvectors (experiments.cpp:132-148)
};

TriMesh load_mesh(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ConfigError("cannot open mesh " + path);
    TriMesh m = load_trimesh(in);
    // Dirichlet boundary: vertices of the edges that belong to one triangle
    // (on the unit square these are exactly the vertices with x or y in {0, 1})
    std::map<std::pair<int, int>, int> edges;
    for (const auto& t : m.triangles)
        for (int e = 0; e < 3; ++e) {
            const int a = t[e], b = t[(e + 1) % 3];
            ++edges[{std::min(a, b), std::max(a, b)}];
        }
    m.boundary_vertex.assign(m.n_vertices(), 0);
    for (const auto& [e, count] : edges)
        if (count == 1) m.boundary_vertex[e.first] = m.boundary_vertex[e.second] = 1;
    return m;
}

int cell_of(const ProblemDef& d, double x, double y) {
    int ix = static_cast<int>(std::floor((x - d.dom_x0) / (d.dom_x1 - d.dom_x0) * d.cells_x));
    int iy = static_cast<int>(std::floor((y - d.dom_y0) / (d.dom_y1 - d.dom_y0) * d.cells_y));
    ix = std::clamp(ix, 0, d.cells_x - 1);
    iy = std::clamp(iy, 0, d.cells_y - 1);
    return iy * d.cells_x + ix;
}

DiscreteOperator interior_operator(const Level& lv, const DiscreteOperator& full) {
    const int n = static_cast<int>(lv.interior.size());
    std::vector<double> mass(n);
    std::vector<std::uint8_t> sel(n);
    for (int i = 0; i < n; ++i) {
        mass[i] = full.mass_diag[lv.interior[i]];
        sel[i] = full.selector[lv.interior[i]];
    }
    std::vector<std::tuple<int, int, double>> trip;
    const auto& rp = full.stiffness.row_ptr();
    const auto& ci = full.stiffness.col_idx();
    const auto& va = full.stiffness.values();
    for (int i = 0; i < n; ++i) {
        const int r = lv.interior[i];
        for (int k = rp[r]; k < rp[r + 1]; ++k) {
            const int j = lv.dof_of[ci[k]];
            if (j >= 0) trip.emplace_back(i, j, va[k]);
        }
    }
    return make_operator(std::move(mass), CsrMatrix::from_triplets(n, n, std::move(trip)), std::move(sel));
}

Level make_level(const ProblemDef& d, const std::string& mesh_path, double dt, int substeps) {
    Level lv;
    lv.mesh = load_mesh(mesh_path);
    lv.dt = dt;
    lv.substeps = substeps;
    lv.dof_of.assign(lv.mesh.n_vertices(), -1);
    for (int v = 0; v < lv.mesh.n_vertices(); ++v)
        if (!lv.mesh.boundary_vertex[v]) {
            lv.dof_of[v] = static_cast<int>(lv.interior.size());
            lv.interior.push_back(v);
        }
    const DiscreteOperator full = assemble(lv.mesh, 1.0);
    auto u0 = [&](double x, double y) {
        const double dx = x - d.ic_x, dy = y - d.ic_y;
        return std::exp(-(dx * dx + dy * dy) / d.ic_w2);
    };
    const InitialData init_full = project_initial(lv.mesh, u0, [](double, double) { return 0.0; }, full);
    const int n = static_cast<int>(lv.interior.size());
    lv.init.z0.resize(n);
    lv.init.mhalf_v0.resize(n);
    for (int i = 0; i < n; ++i) {
        lv.init.z0[i] = init_full.z0[lv.interior[i]];
        lv.init.mhalf_v0[i] = init_full.mhalf_v0[lv.interior[i]];
    }
    std::vector<double> w(lv.mesh.n_vertices(), 0.0);
    for (int t = 0; t < lv.mesh.n_triangles(); ++t) {
        const auto c = lv.mesh.centroid(t);
        if (c[0] < d.box_x0 || c[0] > d.box_x1 || c[1] < d.box_y0 || c[1] > d.box_y1) continue;
        const double area = lv.mesh.signed_area(t);
        for (int v : lv.mesh.triangles[t]) w[v] += area / 3.0;
    }
    double total = 0.0;
    for (double v : w) total += v;
    lv.qoi_w.resize(n);
    for (int i = 0; i < n; ++i) lv.qoi_w[i] = d.qoi_mean ? w[lv.interior[i]] / total : w[lv.interior[i]];
    const DiscreteOperator op = interior_operator(lv, full);
    // |R| = rows of A P holding a nonzero value (explicit zeros do not couple)
    for (int r = 0; r < op.a_fine.rows(); ++r)
        for (int k = op.a_fine.row_ptr()[r]; k < op.a_fine.row_ptr()[r + 1]; ++k)
            if (op.a_fine.values()[k] != 0.0) {
                ++lv.n_r;
                break;
            }
    lv.n_steps = static_cast<long>(std::ceil(d.final_time / dt - 1e-12));
    if (d.cfl > 0.0) {  // the reference's per-level warm starts (experiments.cpp:141-145)
        lv.warm_full = max_eigenvalue(op.normalized, 1e-4, 20000).eigenvector;
        if (op.n_fine > 0) lv.warm_coarse = coarse_max_eigenvalue(op, 1e-4, 20000).eigenvector;
    }
    return lv;
}

std::vector<double> draw_cells(const ProblemDef& d, RngStream& stream) {
    std::vector<double> c(d.cells_x * d.cells_y);
    if (d.kl.empty() && d.klp.empty()) {
        for (double& v : c) v = stream.next_uniform(d.coef_lo, d.coef_hi);
        return c;
    }
    // log-normal KL (BASELINE config 4; no reference counterpart): Box-Muller
    // over consecutive next_unit() pairs, c_k = exp(sum_m T[k][m] xi_m)
    std::vector<double> xi(d.kl_modes);
    const double two_pi = 6.283185307179586;
    for (int i = 0; 2 * i < d.kl_modes; ++i) {
        const double u1 = stream.next_unit(), u2 = stream.next_unit();
        const double r = std::sqrt(-2.0 * std::log(1.0 - u1)), th = two_pi * u2;
        xi[2 * i] = r * std::cos(th);
        if (2 * i + 1 < d.kl_modes) xi[2 * i + 1] = r * std::sin(th);
    }
    if (!d.klp.empty()) return xi;  // pointwise field: the sample is its normals (solve_level evaluates g)
    for (std::size_t k = 0; k < c.size(); ++k) {
        double g = 0.0;
        for (int m = 0; m < d.kl_modes; ++m) g += d.kl[k * d.kl_modes + m] * xi[m];
        c[k] = std::exp(g);
    }
    return c;
}

double solve_level(const ProblemDef& d, const Level& lv, const std::vector<double>& cells, CostRecord* cost) {
    // the reference evaluates the squared speed at every triangle's centroid (fem.cpp:103-104)
    const DiscreteOperator full =
        d.klp.empty() ? assemble(lv.mesh, [&](double x, double y) { return cells[cell_of(d, x, y)]; })
                      : assemble(lv.mesh, [&](double x, double y) { return std::exp(kl_point_value(d, cells, x, y)); });
    const DiscreteOperator op = interior_operator(lv, full);
    RunOptions options;
    options.kind = d.kind;
    options.final_time = d.final_time;
    options.dt = lv.dt;
    if (d.cfl > 0.0) {
        // stable_dt (src/experiments.cpp:30-43; file-local there, restated
        // over the public max_eigenvalue / coarse_max_eigenvalue)
        const double margin = 1.05, tol = 1e-4;
        const auto fullv = max_eigenvalue(op.normalized, tol, 20000, &lv.warm_full);
        if (cost) cost->weighted_work += static_cast<long>(fullv.iterations) * op.normalized.nnz();
        if (d.kind == Integrator::LocalTimeStepping && op.n_fine > 0) {
            const auto coarse = coarse_max_eigenvalue(op, tol, 20000, &lv.warm_coarse);
            if (cost) cost->weighted_work += static_cast<long>(coarse.iterations) * op.a_coarse.nnz();
            const double dt_coarse = 2.0 / std::sqrt(margin * coarse.lambda);
            const double dt_fine = lv.substeps * 2.0 / std::sqrt(margin * fullv.lambda);
            options.dt = d.cfl * std::min(dt_coarse, dt_fine);
        } else {
            options.dt = d.cfl * 2.0 / std::sqrt(margin * fullv.lambda);
        }
    }
    options.substeps = lv.substeps;
    options.nu = d.nu;
    const RunResult run = run_wave(op, lv.init, options);
    if (cost) {
        cost->matvec_full += run.counters.full;
        cost->matvec_fine += run.counters.fine;
        cost->matvec_coarse += run.counters.coarse;
        cost->weighted_work += run.counters.full * op.normalized.nnz() +
                               run.counters.fine * op.a_fine.nnz() + run.counters.coarse * op.a_coarse.nnz();
    }
    const std::vector<double> u = nodal_values(op, run.state.z_curr);
    double q = 0.0;
    for (std::size_t i = 0; i < u.size(); ++i) q += lv.qoi_w[i] * u[i];
    return q;
}

double dof_updates(const ProblemDef& d, const Level& lv) {
    const double n = static_cast<double>(lv.interior.size());
    if (d.kind == Integrator::Leapfrog) return static_cast<double>(lv.n_steps) * n;
    return n + static_cast<double>(lv.n_steps - 1) * (n + (lv.substeps - 1) * static_cast<double>(lv.n_r));
}

// scalar QoI as a 2-point QoIVector on the grid {0, 2}: norm() == |Q|
// (the reference tests' own encoding, tests/test_mlmc.cpp:16-20)
const OutputGrid kScalarGrid{0.0, 2.0, 2};

// the reference's run_jobs pattern (src/mlmc.cpp:107-149): atomic cursor,
// per-index result slots, first failure stops the wave and is rethrown
template <class Fn>
void parallel_for(long count, int threads, Fn fn) {
    std::atomic<long> cursor{0};
    std::exception_ptr failure;
    std::mutex failure_mutex;
    auto worker = [&]() {
        for (long i; (i = cursor.fetch_add(1)) < count;) {
            try {
                fn(i);
            } catch (...) {
                std::scoped_lock lock(failure_mutex);
                if (!failure) failure = std::current_exception();
                cursor.store(count);
                break;
            }
        }
    };
    if (threads <= 1) {
        worker();
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
    }
    if (failure) std::rethrow_exception(failure);
}

int default_threads(const Args& a) {
    const long t = a.integer("threads", 0);
    if (t > 0) return static_cast<int>(t);
    const unsigned hc = std::thread::hardware_concurrency();
    return hc ? static_cast<int>(hc) : 1;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct LevelArg {
    std::string mesh;
    double dt;
    int p;
};

std::vector<LevelArg> level_args(const Args& a) {
    std::vector<LevelArg> out;
    for (const auto& s : a.all("level-spec")) {
        LevelArg l;
        std::stringstream ss(s);
        std::string part;
        std::getline(ss, l.mesh, ',');
        std::getline(ss, part, ',');
        l.dt = std::strtod(part.c_str(), nullptr);
        std::getline(ss, part, ',');
        l.p = static_cast<int>(std::strtol(part.c_str(), nullptr, 10));
        out.push_back(l);
    }
    return out;
}

// per-sample Q on one level: "solve --level-spec mesh,dt,p --stream-level L --first I --count N"
int cmd_solve(const Args& a) {
    const ProblemDef d = problem_from(a);
    const auto specs = level_args(a);
    if (specs.size() != 1) throw ConfigError("solve: exactly one --level-spec");
    const Level lv = make_level(d, specs[0].mesh, specs[0].dt, specs[0].p);
    const std::uint64_t seed = a.u64("seed", 0);
    const auto slevel = static_cast<std::uint32_t>(a.integer("stream-level", 0));
    const long first = static_cast<long>(a.u64("first", 0)), count = a.integer("count", 1);
    std::vector<double> q(count);
    const double t0 = now_s();
    parallel_for(count, default_threads(a), [&](long i) {
        RngStream s = derive_stream(seed, slevel, static_cast<std::uint64_t>(first + i));
        q[i] = solve_level(d, lv, draw_cells(d, s), nullptr);
    });
    const double t1 = now_s();
    std::printf("# n=%zu n_r=%ld n_steps=%ld dof_updates_per_solve=%.17g seconds=%.6f\n", lv.interior.size(),
                lv.n_r, lv.n_steps, dof_updates(d, lv), t1 - t0);
    for (long i = 0; i < count; ++i) std::printf("%ld %.17g\n", first + i, q[i]);
    return 0;
}

// fixed-N MLMC over the level hierarchy through the reference's own
// sample_delta_q / LevelAccumulator: "mlmc --level-spec ... --N n0,n1,..."
int cmd_mlmc(const Args& a) {
    const ProblemDef d = problem_from(a);
    const auto specs = level_args(a);
    std::vector<long> counts;
    {
        std::stringstream ss(a.get("N"));
        std::string part;
        while (std::getline(ss, part, ',')) counts.push_back(std::strtol(part.c_str(), nullptr, 10));
    }
    if (counts.size() != specs.size()) throw ConfigError("mlmc: --N needs one count per --level-spec");
    auto levels = std::make_shared<std::vector<Level>>();
    for (const auto& s : specs) levels->push_back(make_level(d, s.mesh, s.dt, s.p));

    MlmcProblem problem;
    problem.grid = kScalarGrid;
    problem.max_levels_available = static_cast<int>(levels->size()) - 1;
    problem.model_cost = [levels, d](int l) { return dof_updates(d, (*levels)[l]); };
    problem.draw = [d](RngStream& s) {
        FieldSample f;
        f.kl_cos = draw_cells(d, s);  // generic random numbers, as tests/test_mlmc.cpp:33-62
        return f;
    };
    problem.solve = [levels, d](const FieldSample& f, int level, CostRecord& cost) {
        const double q = solve_level(d, (*levels)[level], f.kl_cos, &cost);
        return QoIVector{kScalarGrid, {q, 0.0}};
    };

    const std::uint64_t seed = a.u64("seed", 0);
    const int threads = default_threads(a);
    const bool per_sample = a.integer("per-sample", 0) != 0;
    // one job list over all levels, level-major and index-ascending, run by
    // one worker pool and folded in (level, index) order -- the reference's
    // run_jobs (src/mlmc.cpp:107-149, :181-183)
    struct Job {
        int level;
        long index;
    };
    std::vector<Job> jobs;
    for (std::size_t l = 0; l < levels->size(); ++l)
        for (long i = 0; i < counts[l]; ++i) jobs.push_back({static_cast<int>(l), i});
    std::vector<SampleResult> results(jobs.size());
    const double t0 = now_s();
    parallel_for(static_cast<long>(jobs.size()), threads, [&](long k) {
        results[k] = sample_delta_q(problem, jobs[k].level,
                                    derive_stream(seed, static_cast<std::uint32_t>(jobs[k].level),
                                                  static_cast<std::uint64_t>(jobs[k].index)));
    });
    const double total_s = now_s() - t0;
    double total_upd = 0.0;
    std::printf("{\"threads\": %d, \"levels\": [\n", threads);
    std::size_t k0 = 0;
    for (std::size_t l = 0; l < levels->size(); ++l) {
        const long N = counts[l];
        LevelAccumulator acc(static_cast<int>(l), kScalarGrid);
        for (long i = 0; i < N; ++i) acc.add(results[k0 + i]);
        const double upd = N * (dof_updates(d, (*levels)[l]) + (l > 0 ? dof_updates(d, (*levels)[l - 1]) : 0.0));
        total_upd += upd;
        std::printf("  {\"level\": %zu, \"N\": %ld, \"sum_dq\": %.17g, \"sum_dq2\": %.17g, \"sum_q\": %.17g, "
                    "\"sum_q2\": %.17g, \"variance\": %.17g, \"mc_variance\": %.17g, \"mean_dq\": %.17g, "
                    "\"dof_updates\": %.17g, \"n\": %zu, \"n_r\": %ld, \"n_steps\": %ld",
                    l, N, acc.sum_dq.values[0], acc.sum_norm2_dq, acc.sum_q.values[0], acc.sum_norm2_q,
                    N >= 2 ? estimate_variance(acc) : 0.0, N >= 2 ? estimate_mc_variance(acc) : 0.0,
                    acc.mean_dq().values[0], upd, (*levels)[l].interior.size(), (*levels)[l].n_r,
                    (*levels)[l].n_steps);
        if (per_sample) {
            std::printf(", \"dq\": [");
            for (long i = 0; i < N; ++i) std::printf("%s%.17g", i ? ", " : "", results[k0 + i].delta_q.values[0]);
            std::printf("], \"q\": [");
            for (long i = 0; i < N; ++i) std::printf("%s%.17g", i ? ", " : "", results[k0 + i].q_fine.values[0]);
            std::printf("]");
        }
        std::printf("}%s\n", l + 1 < levels->size() ? "," : "");
        k0 += static_cast<std::size_t>(N);
    }
    std::printf("], \"seconds\": %.6f, \"dof_updates\": %.17g}\n", total_s, total_upd);
    return 0;
}

// adaptive Giles driver through the reference's run_mlmc
int cmd_adaptive(const Args& a) {
    const ProblemDef d = problem_from(a);
    const auto specs = level_args(a);
    auto levels = std::make_shared<std::vector<Level>>();
    for (const auto& s : specs) levels->push_back(make_level(d, s.mesh, s.dt, s.p));
    MlmcProblem problem;
    problem.grid = kScalarGrid;
    problem.max_levels_available = static_cast<int>(levels->size()) - 1;
    problem.model_cost = [levels, d](int l) { return dof_updates(d, (*levels)[l]); };
    problem.draw = [d](RngStream& s) {
        FieldSample f;
        f.kl_cos = draw_cells(d, s);
        return f;
    };
    problem.solve = [levels, d](const FieldSample& f, int level, CostRecord& cost) {
        return QoIVector{kScalarGrid, {solve_level(d, (*levels)[level], f.kl_cos, &cost), 0.0}};
    };
    MlmcConfig cfg;
    cfg.eps = a.num("eps", 1e-3);
    cfg.workers = default_threads(a);
    cfg.max_level = static_cast<int>(a.integer("max-level", 6));
    cfg.master_seed = a.u64("seed", 0);
    const double t0 = now_s();
    const MlmcResult r = run_mlmc(problem, cfg);
    const double t1 = now_s();
    std::printf("{\"estimate\": %.17g, \"converged\": %s, \"total_variance\": %.17g, \"bias\": %.17g, "
                "\"seconds\": %.6f, \"threads\": %d, \"levels\": [",
                r.estimate.values[0], r.converged ? "true" : "false", r.total_variance, r.bias, t1 - t0, cfg.workers);
    for (std::size_t l = 0; l < r.levels.size(); ++l)
        std::printf("%s{\"level\": %d, \"N\": %ld, \"variance\": %.17g, \"mean_dq_norm\": %.17g}", l ? ", " : "",
                    r.levels[l].level, r.levels[l].n_samples, r.levels[l].variance, r.levels[l].mean_dq_norm);
    std::printf("]}\n");
    return 0;
}

// The reference's artifact files of a sampling experiment (run_experiment,
// src/experiments.cpp:365-409, 523-545): the config file is parsed by the
// reference's own parse_config_file, the CSVs land in its out_dir.
//   artifacts --config FILE
int cmd_artifacts(const Args& a) {
    const ExperimentConfig cfg = parse_config_file(a.get("config"), std::nullopt);
    std::ostringstream log;
    const int rc = run_experiment(cfg, log);
    std::fprintf(stderr, "%s", log.str().c_str());
    return rc;
}

// The reference's narrow-channel mesh of one level (build_state_2d,
// src/experiments.cpp:137-139: build_channel_mesh(max(h0 2^-l, fine_h), fine_h))
// in its fixture format (dump_mesh, src/mesh_io.cpp:47-55).
//   channel-mesh --h0 H --fine-h F --level L --out PATH
int cmd_channel_mesh(const Args& a) {
    const double h0 = a.num("h0", 1.0 / 60.0), fine_h = a.num("fine-h", 7.6e-4);
    const int level = static_cast<int>(a.integer("level", 0));
    const double coarse = h0 / std::pow(2.0, level);
    const TriMesh m = build_channel_mesh(std::max(coarse, fine_h), fine_h);
    std::ofstream out(a.get("out"));
    if (!out) throw ConfigError("channel-mesh: cannot open --out");
    dump_mesh(m, out);
    return 0;
}

// The reference's 1D mesh hierarchy of a sampling experiment, exactly as
// build_state_1d builds it (src/experiments.cpp:62-85: domain [0, 6], fine
// window [anchor - h0, anchor], build_hierarchy src/mesh1d.cpp:76-125): per
// level the vertices, fine flags, coarse / fine sizes and the ratio p_l.
//   hierarchy1d --name smooth1d|jump1d [--h0 H --fine-h F --max-level L]
int cmd_hierarchy1d(const Args& a) {
    const std::string name = a.get("name", "smooth1d");
    const auto kind = experiment_from_string(name);
    if (!kind || (*kind != ExperimentKind::Smooth1d && *kind != ExperimentKind::Jump1d))
        throw ConfigError("hierarchy1d: --name smooth1d|jump1d");
    ExperimentConfig cfg = default_config(*kind);
    cfg.max_level = static_cast<int>(a.integer("max-level", cfg.max_level));
    if (!a.get("h0").empty()) cfg.h0 = a.num("h0", cfg.h0);
    if (!a.get("fine-h").empty()) cfg.fine_h = a.num("fine-h", cfg.fine_h);
    const double anchor = *kind == ExperimentKind::Jump1d ? 4.0 : 5.0;
    const MeshHierarchy h = build_hierarchy({0.0, 6.0}, cfg.h0, Interval{anchor - cfg.h0, anchor}, cfg.fine_h,
                                            cfg.max_level);
    std::printf("{\"experiment\": \"%s\", \"h0\": %.17g, \"fine_h\": %.17g, \"max_level\": %d, \"levels\": [",
                name.c_str(), cfg.h0, cfg.fine_h, cfg.max_level);
    for (int l = 0; l < h.n_levels(); ++l) {
        const Mesh1D& m = h.levels[l];
        std::printf("%s{\"ratio\": %d, \"coarse_h\": %.17g, \"fine_h\": %.17g, \"vertices\": [", l ? ", " : "",
                    h.ratios[l], m.coarse_h, m.fine_h);
        for (std::size_t i = 0; i < m.vertices.size(); ++i) std::printf("%s%.17g", i ? ", " : "", m.vertices[i]);
        std::printf("], \"fine_flags\": [");
        for (std::size_t i = 0; i < m.fine_flags.size(); ++i) std::printf("%s%d", i ? ", " : "", m.fine_flags[i]);
        std::printf("]}");
    }
    std::printf("]}\n");
    return 0;
}

// The reference's own sampling experiments through its public make_problem
// (src/experiments.cpp:194-237): per-sample QoI vectors of coupled pairs
// (sample_delta_q) and, with --eps, run_mlmc at the reference's config.
//   experiment --name smooth1d|jump1d --kind lts|lf --level L --first I --count N [--eps E]
int cmd_experiment(const Args& a) {
    const std::string name = a.get("name", "smooth1d");
    const auto kind = experiment_from_string(name);
    if (!kind) throw ConfigError("experiment: unknown --name " + name);
    ExperimentConfig cfg = default_config(*kind);
    cfg.max_level = static_cast<int>(a.integer("max-level", cfg.max_level));
    cfg.grid_n = static_cast<int>(a.integer("grid-n", cfg.grid_n));
    if (!a.get("h0").empty()) cfg.h0 = a.num("h0", cfg.h0);
    if (!a.get("fine-h").empty()) cfg.fine_h = a.num("fine-h", cfg.fine_h);
    if (!a.get("final-time").empty()) cfg.final_time = a.num("final-time", cfg.final_time);
    cfg.workers = default_threads(a);
    const Integrator integ = a.get("kind", "lts") == "lf" ? Integrator::Leapfrog : Integrator::LocalTimeStepping;
    const MlmcProblem problem = make_problem(cfg, integ);
    std::printf("{\"experiment\": \"%s\", \"kind\": \"%s\", \"max_level\": %d, \"grid_n\": %d, \"model_cost\": [",
                name.c_str(), a.get("kind", "lts").c_str(), cfg.max_level, cfg.grid_n);
    for (int l = 0; l <= problem.max_levels_available; ++l) std::printf("%s%.17g", l ? ", " : "", problem.model_cost(l));
    std::printf("]");
    if (!a.get("eps").empty()) {
        MlmcConfig m;
        m.eps = a.num("eps", 4e-3);
        m.alpha = cfg.alpha;
        m.initial_samples = cfg.initial_samples;
        m.max_level = cfg.max_level;
        m.master_seed = a.u64("seed", cfg.seed);
        m.workers = cfg.workers;
        m.bias_window = cfg.bias_window;
        const double t0 = now_s();
        const MlmcResult r = run_mlmc(problem, m);
        const double t1 = now_s();
        std::printf(", \"eps\": %.17g, \"seconds\": %.6f, \"converged\": %s, \"total_variance\": %.17g, \"bias\": %.17g, "
                    "\"estimate_norm\": %.17g, \"estimate\": [",
                    m.eps, t1 - t0, r.converged ? "true" : "false", r.total_variance, r.bias, r.estimate.norm());
        for (std::size_t i = 0; i < r.estimate.values.size(); ++i)
            std::printf("%s%.17g", i ? ", " : "", r.estimate.values[i]);
        std::printf("], \"levels\": [");
        for (std::size_t l = 0; l < r.levels.size(); ++l)
            std::printf("%s{\"level\": %d, \"N\": %ld, \"variance\": %.17g, \"mean_dq_norm\": %.17g}", l ? ", " : "",
                        r.levels[l].level, r.levels[l].n_samples, r.levels[l].variance, r.levels[l].mean_dq_norm);
        std::printf("]");
    }
    if (!a.get("level").empty()) {
        const int level = static_cast<int>(a.integer("level", 0));
        const long first = static_cast<long>(a.u64("first", 0)), count = a.integer("count", 1);
        const std::uint64_t seed = a.u64("seed", 0);
        std::vector<SampleResult> res(count);
        parallel_for(count, default_threads(a), [&](long i) {
            res[i] = sample_delta_q(problem, level,
                                    derive_stream(seed, static_cast<std::uint32_t>(level),
                                                  static_cast<std::uint64_t>(first + i)));
        });
        std::printf(", \"level\": %d, \"first\": %ld, \"samples\": [", level, first);
        for (long i = 0; i < count; ++i) {
            std::printf("%s{\"dq\": [", i ? ", " : "");
            for (std::size_t k = 0; k < res[i].delta_q.values.size(); ++k)
                std::printf("%s%.17g", k ? ", " : "", res[i].delta_q.values[k]);
            std::printf("], \"q\": [");
            for (std::size_t k = 0; k < res[i].q_fine.values.size(); ++k)
                std::printf("%s%.17g", k ? ", " : "", res[i].q_fine.values[k]);
            const CostRecord& c = res[i].cost;
            std::printf("], \"cost\": [%ld, %ld, %ld, %ld]}", c.matvec_full, c.matvec_fine, c.matvec_coarse,
                        c.weighted_work);
        }
        std::printf("]");
    }
    std::printf("}\n");
    return 0;
}

int cmd_rng(const Args& a) {
    RngStream s = derive_stream(a.u64("seed", 0),
                                static_cast<std::uint32_t>(a.integer("level", 0)),
                                a.u64("index", 0));
    const long count = a.integer("count", 4);
    const bool uniform = a.integer("uniform", 0) != 0;
    for (long i = 0; i < count; ++i) {
        if (uniform)
            std::printf("%.17g\n", s.next_uniform(a.num("lo", 0.5), a.num("hi", 1.5)));
        else
            std::printf("0x%016llx\n", static_cast<unsigned long long>(s.next_u64()));
    }
    return 0;
}

int cmd_consts(const Args& a) {
    const int p = static_cast<int>(a.integer("p", 2));
    const ChebyshevConstants c = chebyshev_constants(p, a.num("nu", 0.01));
    std::printf("%.17g %.17g\n", c.delta, c.omega);
    for (int k = 0; k < p - 1; ++k) std::printf("%.17g %.17g\n", c.beta_int[k], c.beta_half[k]);
    return 0;
}

int cmd_meshcheck(const Args& a) {
    const TriMesh m = load_mesh(a.get("mesh"));
    const MeshReport r = check_mesh(m);
    long fine = 0;
    for (auto f : m.fine_flags) fine += f;
    std::printf("{\"conforming\": %s, \"positive_areas\": %s, \"total_area\": %.17g, \"boundary_area\": %.17g, "
                "\"euler\": %d, \"n_vertices\": %d, \"n_triangles\": %d, \"n_fine\": %ld}\n",
                r.conforming ? "true" : "false", r.positive_areas ? "true" : "false", r.total_area,
                r.boundary_area, r.euler_characteristic, m.n_vertices(), m.n_triangles(), fine);
    return 0;
}

// sample-independent level data: interior z0 and lumped mass (dof order)
int cmd_level(const Args& a) {
    const ProblemDef d = problem_from(a);
    const auto specs = level_args(a);
    const Level lv = make_level(d, specs.at(0).mesh, specs.at(0).dt, specs.at(0).p);
    const DiscreteOperator full = assemble(lv.mesh, 1.0);
    std::printf("# n=%zu n_r=%ld n_steps=%ld\n", lv.interior.size(), lv.n_r, lv.n_steps);
    for (std::size_t i = 0; i < lv.interior.size(); ++i)
        std::printf("%d %.17g %.17g %.17g\n", lv.interior[i], lv.init.z0[i], full.mass_diag[lv.interior[i]],
                    lv.qoi_w[i]);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: wavemc_ref_driver solve|mlmc|adaptive|experiment|artifacts|channel-mesh|rng|consts|meshcheck|level --key value...\n");
        return 2;
    }
    try {
        const std::string cmd = argv[1];
        const Args a = parse(argc, argv, 2);
        if (cmd == "solve") return cmd_solve(a);
        if (cmd == "mlmc") return cmd_mlmc(a);
        if (cmd == "adaptive") return cmd_adaptive(a);
        if (cmd == "rng") return cmd_rng(a);
        if (cmd == "consts") return cmd_consts(a);
        if (cmd == "meshcheck") return cmd_meshcheck(a);
        if (cmd == "level") return cmd_level(a);
        if (cmd == "experiment") return cmd_experiment(a);
        if (cmd == "hierarchy1d") return cmd_hierarchy1d(a);
        if (cmd == "artifacts") return cmd_artifacts(a);
        if (cmd == "channel-mesh") return cmd_channel_mesh(a);
        throw ConfigError("unknown command " + cmd);
    } catch (const InstabilityError& e) {
        std::fprintf(stderr, "instability at step %ld: %s\n", e.step, e.what());
        return 3;
    } catch (const NumericalError& e) {
        std::fprintf(stderr, "numerical error: %s\n", e.what());
        return 3;
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
