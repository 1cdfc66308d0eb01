// The reference-side binding of the B200 path, compiled and tested
// (oracle/Makefile target `adapter`, tests/test_gpu_adapter.py): the
// reference's own run_mlmc (proj/src/mlmc.cpp:165-233) -- unmodified,
// linked from the reference library -- driving the B200 evaluator through its
// plug-in interface MlmcProblem (proj/include/wavemc/mlmc.hpp:41-47).
//
// The interface is per sample (draw, solve); the device wants batches.  The
// problem below bridges the two without touching the reference:
//   * draw(RngStream& s) records the stream's identity, s.id() = (seed,
//     level, sample_index) (include/wavemc/rng.hpp:21-45), in the FieldSample;
//   * solve(field, l, cost) looks the sample up in a per-level cache of coupled
//     pairs; a miss evaluates a whole block of indices [i, i + block) of that
//     level with one wmc_eval_pairs call (run_mlmc asks for each level's
//     indices in ascending order, src/mlmc.cpp:181-183, so the block is the
//     next samples it will want).  A sample's results depend only on (seed,
//     level, index), so blocks never change them.
//   * the fine solve returns Q_l, the coarse one Q_l - dQ; sample_delta_q
//     (src/mlmc.cpp:21-37) forms dQ = Q_l - Q_{l-1} from them.
// Errors keep the reference's convention: a failing sample raises
// NumericalError("level L, sample I: ...") (src/mlmc.cpp:31-35).
//
// main() runs BASELINE config 1 (the product's own mesh builder and level
// tables, the reference's run_mlmc) and prints one JSON line.
//   reference_adapter --eps E [--block B] [--max-level L]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "wavemc/errors.hpp"
#include "wavemc/mlmc.hpp"
#include "wavemc/rng.hpp"
#include "wavemc_b200.h"

using namespace wavemc;

namespace {

const OutputGrid kScalarGrid{0.0, 2.0, 2};  // scalar QoI as a 2-point vector (tests/test_mlmc.cpp:16-20)

struct Pairs {
    long first = 0;
    std::vector<double> dq, q;
};

class B200Problem {
public:
    B200Problem(std::vector<wmc_level*> levels, std::uint64_t seed, long block)
        : levels_(std::move(levels)), seed_(seed), block_(block), cache_(levels_.size()) {}

    MlmcProblem problem(const std::vector<double>& model_cost) {
        MlmcProblem p;
        p.grid = kScalarGrid;
        p.max_levels_available = static_cast<int>(levels_.size()) - 1;
        p.model_cost = [model_cost](int l) { return model_cost[l]; };
        p.draw = [](RngStream& s) {
            FieldSample f;
            f.kl_cos = {static_cast<double>(s.id().level), static_cast<double>(s.id().sample_index)};
            return f;
        };
        p.solve = [this](const FieldSample& f, int l, CostRecord& cost) {
            const int level = static_cast<int>(f.kl_cos[0]);
            const long index = static_cast<long>(f.kl_cos[1]);
            double dq = 0.0, q = 0.0;
            lookup(level, index, dq, q, cost, l == level);
            return QoIVector{kScalarGrid, {l == level ? q : q - dq, 0.0}};
        };
        return p;
    }

    long device_calls() const { return calls_; }
    long device_pairs() const { return pairs_; }

private:
    void lookup(int level, long index, double& dq, double& q, CostRecord& cost, bool fine) {
        std::lock_guard<std::mutex> lock(mu_);
        Pairs& c = cache_[level];
        if (index < c.first || index >= c.first + static_cast<long>(c.q.size())) {
            const long count = block_;
            c.first = index;
            c.dq.assign(count, 0.0);
            c.q.assign(count, 0.0);
            wmc_cost wc{};
            wmc_error err{};
            const int rc = wmc_eval_pairs(levels_[level], level > 0 ? levels_[level - 1] : nullptr, seed_,
                                          static_cast<std::uint32_t>(level), static_cast<std::uint64_t>(index),
                                          static_cast<std::uint64_t>(count), c.dq.data(), c.q.data(), &wc, &err);
            if (rc == WMC_NUMERICAL_ERROR) throw NumericalError(wmc_last_error());
            if (rc == WMC_CONFIG_ERROR) throw ConfigError(wmc_last_error());
            if (rc != WMC_OK) throw std::runtime_error(wmc_last_error());
            per_pair_[level] = wc;
            ++calls_;
            pairs_ += count;
        }
        dq = c.dq[index - c.first];
        q = c.q[index - c.first];
        // the pair's cost record, uniform per pair on fixed-dt levels: the
        // fine solve books it (the coarse solve of sample_delta_q adds none)
        if (fine) {
            const wmc_cost& wc = per_pair_[level];
            cost.matvec_full += wc.matvec_full / block_;
            cost.matvec_fine += wc.matvec_fine / block_;
            cost.matvec_coarse += wc.matvec_coarse / block_;
            cost.weighted_work += wc.weighted_work / block_;
        }
    }

    std::vector<wmc_level*> levels_;
    std::uint64_t seed_;
    long block_;
    std::vector<Pairs> cache_;
    std::map<int, wmc_cost> per_pair_;
    std::mutex mu_;
    long calls_ = 0, pairs_ = 0;
};

void ok(int rc, const char* what) {
    if (rc != WMC_OK) {
        std::fprintf(stderr, "%s: %s\n", what, wmc_last_error());
        std::exit(2);
    }
}

}  // namespace

int main(int argc, char** argv) {
    double eps = 2e-4;
    long block = 1024;
    int max_level = 4;
    for (int i = 1; i + 1 < argc; i += 2) {
        if (!std::strcmp(argv[i], "--eps")) eps = std::atof(argv[i + 1]);
        if (!std::strcmp(argv[i], "--block")) block = std::atol(argv[i + 1]);
        if (!std::strcmp(argv[i], "--max-level")) max_level = std::atoi(argv[i + 1]);
    }
    // BASELINE config 1 (paper_2106_11117_b200/configs.py): h_l = 1/16 2^-l,
    // refined square [0.45, 0.55]^2 snapped to the level-0 grid at h_min = 1/512,
    // p_l = h_l / h_min, dt = 0.2 h_l, T = 1
    std::vector<wmc_level*> levels;
    std::vector<double> model_cost;
    for (int l = 0; l <= max_level; ++l) {
        const int n = 16 << l, ratio = 512 / n;
        wmc_square_mesh_spec ms{n, ratio, 0.45, 0.55, 1.0 / 16, 0.7};
        wmc_mesh* mesh = nullptr;
        ok(wmc_mesh_build_square(&ms, &mesh), "wmc_mesh_build_square");
        wmc_level_desc d;
        wmc_level_desc_default(&d);
        d.dt = 0.2 / n;
        d.substeps = ratio;
        d.integrator = WMC_LOCAL_TIME_STEPPING;
        wmc_level* lv = nullptr;
        ok(wmc_level_create(mesh, &d, &lv), "wmc_level_create");
        wmc_mesh_destroy(mesh);
        wmc_level_info info{};
        ok(wmc_level_get_info(lv, &info), "wmc_level_get_info");
        levels.push_back(lv);
        model_cost.push_back(info.dof_updates_per_solve);
    }
    B200Problem b200(levels, 0, block);
    MlmcConfig cfg;
    cfg.eps = eps;
    cfg.max_level = max_level;
    cfg.master_seed = 0;
    cfg.workers = 1;
    const MlmcResult r = run_mlmc(b200.problem(model_cost), cfg);  // the reference's driver
    std::printf("{\"eps\": %.17g, \"converged\": %s, \"estimate\": %.17g, \"total_variance\": %.17g, \"bias\": %.17g, "
                "\"device_calls\": %ld, \"device_pairs\": %ld, \"levels\": [",
                eps, r.converged ? "true" : "false", r.estimate.values[0], r.total_variance, r.bias,
                b200.device_calls(), b200.device_pairs());
    for (std::size_t l = 0; l < r.levels.size(); ++l)
        std::printf("%s{\"level\": %d, \"N\": %ld, \"variance\": %.17g}", l ? ", " : "", r.levels[l].level,
                    r.levels[l].n_samples, r.levels[l].variance);
    std::printf("]}\n");
    for (auto* lv : levels) wmc_level_destroy(lv);
    return 0;
}
