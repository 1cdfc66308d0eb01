// C ABI of the batched evaluator (include/wavemc_b200.h): per-level device
// contexts, the pair evaluator that replaces the reference's run_jobs loop
// over sample_delta_q, and the host MLMC drivers.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/wavemc_b200.h"
#include "host/channel.hpp"
#include "host/field.hpp"
#include "host/level.hpp"
#include "host/tiles.hpp"
#include "host/mesh.hpp"
#include "kernels.cuh"

struct wmc_mesh1d {
    wmc::Mesh1D mesh;
};

struct wmc_mesh {
    wmc::TriMesh mesh;
};

namespace {

thread_local std::string g_last_error;
std::atomic<long> g_launches{0};  // kernels launched by this library (all devices)

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return WMC_OK;
    } catch (const ConfigError& e) {
        g_last_error = e.what();
        return WMC_CONFIG_ERROR;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return WMC_CONFIG_ERROR;
    } catch (const NumericalError& e) {
        g_last_error = e.what();
        return WMC_NUMERICAL_ERROR;
    } catch (const DeviceError& e) {
        g_last_error = e.what();
        return WMC_DEVICE_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return WMC_DEVICE_ERROR;
    }
}

template <class T>
T* upload(const std::vector<T>& v) {
    T* d = nullptr;
    const std::size_t bytes = sizeof(T) * std::max<std::size_t>(v.size(), 1);
    check(cudaMalloc(&d, bytes), "cudaMalloc");
    if (!v.empty()) check(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice), "upload");
    return d;
}

}  // namespace

// per-role batch state: a level is solved as the fine level of its own pair
// and as the coarse level of the next one, possibly concurrently on two
// streams, so each role owns its buffers
struct Workspace {
    double* za = nullptr;
    double* zb = nullptr;
    double* g = nullptr;
    double* q = nullptr;
    int* fail = nullptr;
    double* da = nullptr;  // HBM-resident substep path: d buffers [r][S]
    double* db = nullptr;
    std::vector<double*> tier_e;    // nested tiers: E^k buffers, 2 per tier, [row][S] over R_k
    std::vector<double*> tier_rhs;  // r_k for k >= 2, [row][S] over R_k
    // per-sample CFL: (dt_s / dt)^2 and step counts, power-iteration state
    double* rel = nullptr;
    int* nsteps = nullptr;
    double* eig = nullptr;     // part [2][nb][S] | norm | lam | lam_prev | lf | lc  (S each)
    int* eig_i = nullptr;      // settled | iters | done (S each) | active count
    int* h_active = nullptr;   // pinned
    int* h_nsteps = nullptr;   // pinned, S
    int* it_full = nullptr;    // per sample: power iterations of the full / coarse CFL estimate (cost records)
    int* it_coarse = nullptr;
};

constexpr int kEigBlocks = 64;  // row blocks of the power-iteration dot products

enum class SubPath { None, Lattice, OnChip, Global, Tiers, Tiled };

struct wmc_level {
    int device = 0;
    cudaStream_t stream = nullptr;
    wmc::LevelSpec spec;
    wmc::LevelTables tab;
    int batch = 0;  // capacity in samples (multiple of 64)

    // sweep operator
    int* d_row_ptr = nullptr;
    int col_bits = 23;
    int* d_cell_ix = nullptr;  // per-entry cells when they do not fit beside the column bits
    int4* d_row_desc = nullptr;
    double2* d_wtype = nullptr;
    double2 row_types[wmc::kMaxRowTypes] = {};
    int n_row_types = 0;
    long n_structured = 0;
    int* d_ent = nullptr;
    double* d_a0 = nullptr;
    double* d_z0 = nullptr;
    // substep operator (SELL A P on R) and recipes
    std::uint32_t* d_sub_ent = nullptr;
    int* d_slice_off = nullptr;
    int n_sub_ent = 0;
    int* d_rc_ptr = nullptr;
    int* d_rc_cell = nullptr;
    double* d_rc_a0 = nullptr;
    int n_wid = 0;
    double* d_beta = nullptr;
    double* d_cm = nullptr;
    int sub_smem = 0;
    int sub_cl_smem = 1;  // generic substep kernel stages the cell coefficients in shared memory
    int sub_grid = 0;
    int small_smem = 0;  // fused small-mesh solve: shared memory per CTA (0: not eligible)
    int fused_smem = 0;  // fused lattice solve: shared memory per CTA (0: not eligible)
    bool fused_zp_global = false;
    int fused_tmem = 2;            // fused lattice solve: tensor-memory form (fixed at level creation)
    int sweep_wide = 23;           // 256-bit step sweep: 10 rows-per-warp + blocks-per-SM, 0 off (WMC_SWEEP_WIDE)  // fused lattice solve keeps z_{n-1} in a per-sample global buffer
    int n_sms = 148;
    SubPath path = SubPath::None;
    int* d_apg_ptr = nullptr;
    int* d_apg_ent = nullptr;
    int* d_apg_cell = nullptr;
    double* d_apg_a0 = nullptr;
    // temporally blocked step on R (SubPath::Tiled, host/tiles.hpp)
    wmc::TileArgs tile{};          // static part of the kernel arguments
    std::vector<void*> tile_bufs;
    int tile_smem = 0;
    int tile_ctas_per_sm = 1;
    int slab_width = 0;            // owned columns of a streamed slab
    double tile_work = 0.0;        // region positions per box node (diagnostics)
    wmc::StreamArgs slabs{};       // streamed interior of the tiled step (n_slabs = 0: none)
    int stream_smem = 0;
    // nested tiers: A P_k on R_k per tier, substep constants
    std::vector<int*> d_tier_ptr, d_tier_ent;
    std::vector<double*> d_tier_a0;
    double* d_tier_cm = nullptr;
    // per-sample CFL: warm starts and per-dof P membership
    double* d_warm_full = nullptr;
    double* d_warm_coarse = nullptr;
    double warm_full_norm = 0.0, warm_coarse_norm = 0.0;
    unsigned char* d_in_p = nullptr;
    // QoI
    int* d_qptr = nullptr;
    int* d_qdof = nullptr;
    double* d_qw = nullptr;
    double* d_qsm = nullptr;
    // structured substep path
    bool lattice = false;
    int* d_strip_j0 = nullptr;
    unsigned char* d_lat_smask = nullptr;
    int* d_strip_len = nullptr;
    int* d_cellx = nullptr;
    int* d_celly = nullptr;
    int* d_gen_rows = nullptr;
    double* d_gen_rs = nullptr;
    int* d_gen_soff = nullptr;
    int* d_gen_warp_slice = nullptr;
    std::uint16_t* d_gen_col = nullptr;
    int* d_slot_rc = nullptr;  // lattice kernel: overflow start offsets
    std::uint16_t* d_ovf_cell = nullptr;
    int n_ovf = 0, n_ovf_terms = 0;
    double* d_slot_a0 = nullptr;
    std::uint16_t* d_slot_cell = nullptr;
    int* d_grc_cell = nullptr;
    double* d_grc_a0 = nullptr;
    int n_slots = 0;
    // narrow-channel experiment: per-sample entry tables
    wmc::ChannelTables ch;
    wmc::ChannelArgs ch_args{};
    std::vector<void*> ch_bufs;
    int* d_ns_rows = nullptr;  // fused solve: non-structured rows outside R held in TMEM
    int n_ns = 0;
    int* d_rem_ptr = nullptr;  // fused solve: A (I - P) entries of the generic rows
    int* d_rem_col = nullptr;
    int* d_rem_cell = nullptr;
    double* d_rem_a0 = nullptr;
    int lat_smem = 0;
    int lat_grid = 0;
    // batch state: ws[0] as the fine level of a pair, ws[1] as the coarse one
    Workspace ws[2];
    double* d_cells = nullptr;
    double* d_cells_coarse = nullptr;  // per-element fields: this level's coefficients as the coarse of a pair
    double* d_dq = nullptr;
    double* d_kl = nullptr;  // log-normal KL table [cell][mode]
    double* d_field_x = nullptr;      // 1D experiments: element midpoints
    double* d_field_table = nullptr;  // Kl1D table [element][term]
    // per-call results of the pairs whose fine level this is: device and
    // pinned host mirrors, grown on demand (so levels can run concurrently)
    std::size_t r_cap = 0;
    double* r_dq = nullptr;
    double* r_qf = nullptr;
    int* r_ff = nullptr;
    int* r_cnt = nullptr;  // per-sample CFL cost counters [6][r_cap]: n_steps, it_full, it_coarse (fine, coarse)
    int* h_cnt = nullptr;
    int* r_fc = nullptr;
    double* h_dq = nullptr;
    double* h_qf = nullptr;
    int* h_ff = nullptr;
    int* h_fc = nullptr;
    // device-resident pairs: first failing (index << 24 | step) of the fine
    // and coarse solves since the last wmc_synchronize, and the MLMC level
    // index the pairs were issued with
    unsigned long long* d_fail_rec = nullptr;
    int fail_level = 0;
    // optional per-kernel event timing (profiling pass only)
    bool profile = false;
    // captured batch launch sequences, keyed by (workspace, S, count, cells)
    struct BatchGraph {
        bool seen = false;
        cudaGraphExec_t exec = nullptr;
        long nodes = 0;
    };
    std::map<std::tuple<const void*, int, int, const void*>, BatchGraph> graphs;
    std::vector<cudaEvent_t> ev_sweep, ev_sub, ev_upd;  // start/stop pairs

    ~wmc_level() {
        cudaSetDevice(device);
        for (void* p : {(void*)d_row_ptr, (void*)d_row_desc, (void*)d_wtype, (void*)d_ent, (void*)d_a0, (void*)d_z0, (void*)d_sub_ent,
                        (void*)d_slice_off, (void*)d_rc_ptr, (void*)d_rc_cell, (void*)d_rc_a0, (void*)d_beta,
                        (void*)d_cm, (void*)d_qptr, (void*)d_qdof, (void*)d_qw, (void*)d_qsm, (void*)d_cells, (void*)d_cells_coarse, (void*)d_dq,
                        (void*)d_strip_j0, (void*)d_lat_smask, (void*)d_strip_len, (void*)d_cellx, (void*)d_celly, (void*)d_gen_rows,
                        (void*)d_gen_rs, (void*)d_gen_soff, (void*)d_gen_warp_slice, (void*)d_gen_col, (void*)d_slot_rc, (void*)d_slot_a0,
                        (void*)d_slot_cell, (void*)d_ovf_cell, (void*)d_grc_cell,
                        (void*)d_grc_a0, (void*)d_kl, (void*)d_field_x, (void*)d_field_table, (void*)d_apg_ptr, (void*)d_apg_ent, (void*)d_apg_cell, (void*)d_apg_a0,
                        (void*)d_rem_ptr, (void*)d_rem_col, (void*)d_rem_cell, (void*)d_rem_a0, (void*)d_ns_rows,
                        (void*)d_cell_ix})
            if (p) cudaFree(p);
        for (void* p : ch_bufs) cudaFree(p);
        for (void* p : tile_bufs) cudaFree(p);
        for (auto* p : d_tier_ptr) cudaFree(p);
        for (auto* p : d_tier_ent) cudaFree(p);
        for (auto* p : d_tier_a0) cudaFree(p);
        if (d_tier_cm) cudaFree(d_tier_cm);
        for (void* p : {(void*)d_warm_full, (void*)d_warm_coarse, (void*)d_in_p})
            if (p) cudaFree(p);
        for (auto& w : ws) {
            for (void* p : {(void*)w.za, (void*)w.zb, (void*)w.g, (void*)w.q, (void*)w.fail, (void*)w.da, (void*)w.db})
                if (p) cudaFree(p);
            for (void* p : {(void*)w.rel, (void*)w.nsteps, (void*)w.eig, (void*)w.eig_i, (void*)w.it_full,
                            (void*)w.it_coarse})
                if (p) cudaFree(p);
            if (w.h_active) cudaFreeHost(w.h_active);
            if (w.h_nsteps) cudaFreeHost(w.h_nsteps);
            for (auto* p : w.tier_e) cudaFree(p);
            for (auto* p : w.tier_rhs) cudaFree(p);
        }
        for (void* p : {(void*)r_dq, (void*)r_qf, (void*)r_ff, (void*)r_fc, (void*)r_cnt, (void*)d_fail_rec})
            if (p) cudaFree(p);
        for (void* p : {(void*)h_dq, (void*)h_qf, (void*)h_ff, (void*)h_fc, (void*)h_cnt})
            if (p) cudaFreeHost(p);
        for (auto& kv : graphs)
            if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        for (auto e : ev_sweep) cudaEventDestroy(e);
        for (auto e : ev_sub) cudaEventDestroy(e);
        for (auto e : ev_upd) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace {

int round64(long v) { return static_cast<int>((v + 63) / 64 * 64); }

// fused lattice solve: per-thread generic SELL weights / columns in tensor
// memory (2, default; measured best), plus the lattice nodes' d_{m-1} (1),
// or everything in shared memory (0)
int fused_tmem() {
    const char* e = std::getenv("WMC_FUSED_TMEM");  // 0 off, 1 weights + d_{m-1}, 2 weights only (default)
    return e ? std::atoi(e) : 2;
}

// Generic SELL rows of the lattice kernels: lane placement for shared-memory
// banks.  A 64-bit shared access is served per half-warp; it costs as many
// wavefronts as the largest number of distinct addresses that fall into one
// 8-byte bank (address mod 16 doubles).  The gathers v[col] of each slot and
// the store of v[row] are the random accesses, so rows are permuted among
// positions holding the same entry count (slice widths, and every row's
// arithmetic, unchanged) by a seeded local search that lowers the summed
// wavefronts.  Rows past a row's count gather column 0 (padding).
// perm[q][e]: which entry of generic row q sits in SELL slot e
using SlotPerm = std::vector<std::vector<int>>;

int half_cost(const wmc::LevelTables& t, const std::vector<int>& ord, int h, int width, const SlotPerm* perm = nullptr) {
    const int n_gen = static_cast<int>(ord.size());
    int cost = 0;
    int cnt[16];
    int addr[16][16];
    for (int e = -1; e < width; ++e) {  // e = -1: the store of v[row]
        std::fill(cnt, cnt + 16, 0);
        int worst = 0;
        for (int l = 0; l < 16; ++l) {
            const int p = h * 16 + l;
            if (p >= n_gen) break;
            const int q = ord[p];
            int a;
            if (e < 0)
                a = t.gen_rows[q];
            else
                if (perm)  // slot e of the row: an entry, or a hole (weight 0 on column 0)
                    a = e < static_cast<int>((*perm)[q].size()) && (*perm)[q][e] >= 0
                            ? t.gen_col[t.gen_ptr[q] + (*perm)[q][e]]
                            : 0;
                else
                    a = e < t.gen_ptr[q + 1] - t.gen_ptr[q] ? t.gen_col[t.gen_ptr[q] + e] : 0;
            const int b = a & 15;
            bool seen = false;
            for (int k = 0; k < cnt[b]; ++k) seen |= addr[b][k] == a;
            if (!seen) {
                addr[b][cnt[b]++] = a;
                worst = std::max(worst, cnt[b]);
            }
        }
        cost += worst;
    }
    return cost;
}

void optimize_generic_lanes(const wmc::LevelTables& t, std::vector<int>& ord, SlotPerm& perm) {
    const int n_gen = static_cast<int>(ord.size());
    perm.assign(n_gen, {});
    for (int q = 0; q < n_gen; ++q)
        for (int e = 0; e < t.gen_ptr[q + 1] - t.gen_ptr[q]; ++e) perm[q].push_back(e);
    if (n_gen < 2) return;
    const int n_half = (n_gen + 15) / 16;
    std::vector<int> width(n_half, 0), cost(n_half, 0);
    auto w_of = [&](int p) { return t.gen_ptr[ord[p] + 1] - t.gen_ptr[ord[p]]; };
    for (int p = 0; p < n_gen; ++p) width[p / 16] = std::max(width[p / 16], w_of(p));
    for (int h = 0; h + 1 < n_half; h += 2) width[h] = width[h + 1] = std::max(width[h], width[h + 1]);  // slice width
    for (int h = 0; h < n_half; ++h) cost[h] = half_cost(t, ord, h, width[h]);
    long before_total = 0;
    for (int c : cost) before_total += c;
    // positions grouped by the row's entry count: swaps stay inside a group
    std::map<int, std::vector<int>> groups;
    for (int p = 0; p < n_gen; ++p) groups[w_of(p)].push_back(p);
    std::uint64_t x = 0x9e3779b97f4a7c15ull;
    auto rnd = [&](std::size_t n) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        return static_cast<std::size_t>(x % n);
    };
    for (auto& kv : groups) {
        const std::vector<int>& pos = kv.second;
        if (pos.size() < 2) continue;
        const long iters = 400L * static_cast<long>(pos.size());
        for (long it = 0; it < iters; ++it) {
            const int pa = pos[rnd(pos.size())], pb = pos[rnd(pos.size())];
            const int ha = pa / 16, hb = pb / 16;
            if (ha == hb) continue;
            const int before = cost[ha] + cost[hb];
            std::swap(ord[pa], ord[pb]);
            const int ca = half_cost(t, ord, ha, width[ha]), cb = half_cost(t, ord, hb, width[hb]);
            if (ca + cb <= before) {
                cost[ha] = ca;
                cost[hb] = cb;
            } else {
                std::swap(ord[pa], ord[pb]);
            }
        }
    }
    long rows_total = 0;
    for (int c : cost) rows_total += c;
    // then the order of a row's entries over its slots (a warp gathers slot e
    // of its 32 rows at once): swaps of two entries of one row that do not
    // raise the half-warp's wavefront count.  The sum of a row's products is
    // formed in slot order, so this only changes rounding.
    for (int p = 0; p < n_gen; ++p) perm[ord[p]].resize(std::max<std::size_t>(perm[ord[p]].size(), width[p / 16]), -1);
    if (!std::getenv("WMC_GEN_NO_SLOT_PERM")) {
        for (int h = 0; h < n_half; ++h) {
            const int rows_h = std::min(16, n_gen - 16 * h);
            for (long it = 0; it < 6000 && cost[h] > width[h] + 1; ++it) {
                const int q = ord[16 * h + static_cast<int>(rnd(rows_h))];
                const int w = static_cast<int>(perm[q].size());  // the slice width: entries and holes
                if (w < 2) continue;
                const int e1 = static_cast<int>(rnd(w)), e2 = static_cast<int>(rnd(w));
                if (e1 == e2) continue;
                std::swap(perm[q][e1], perm[q][e2]);
                const int c = half_cost(t, ord, h, width[h], &perm);
                if (c <= cost[h])
                    cost[h] = c;
                else
                    std::swap(perm[q][e1], perm[q][e2]);
            }
        }
    }
    if (std::getenv("WMC_BANKS_VERBOSE")) {
        long after_total = 0, ideal = 0;
        for (int c : cost) after_total += c;
        for (int h = 0; h < n_half; ++h) {
            int w = 0;
            for (int p = 16 * h; p < std::min(n_gen, 16 * h + 16); ++p) w = std::max(w, w_of(p));
            ideal += w + 1;
        }
        std::fprintf(stderr, "generic lanes: %d rows, half-warp wavefronts per substep %ld -> %ld (rows) -> %ld (slots); "
                     "conflict-free %ld\n", n_gen, before_total, rows_total, after_total, ideal);
    }
}

void build_device_level(wmc_level& L) {
    const wmc::LevelTables& t = L.tab;
    check(cudaSetDevice(L.device), "cudaSetDevice");
    check(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking), "cudaStreamCreate");

    // sweep entries pack col | cell << col_bits: 23/9 bits, or 16/16 when a
    // level has more than 511 coefficient cells (1D experiments: one per element)
    if (t.n_cells <= wmc::kMaxCells) {
        L.col_bits = wmc::kColBits;
        if (t.n > wmc::kColMask) throw ConfigError("level: more than 2^23 DOFs");
    } else {
        // as many column bits as the DOFs need (at least 16), the rest for
        // cells; past that (narrow-channel levels with ~1e5 per-sample cells)
        // the cells go to a separate per-entry array
        L.col_bits = 16;
        while ((1L << L.col_bits) < t.n) ++L.col_bits;
        if (L.col_bits > 30) throw ConfigError("level: more than 2^30 DOFs");
        if (static_cast<long>(t.n_cells) > (1L << (32 - L.col_bits))) {
            L.col_bits = 31;
            L.d_cell_ix = upload(t.cell);
        }
    }
    std::vector<int> ent(t.col.size());
    for (std::size_t k = 0; k < ent.size(); ++k)
        ent[k] = L.d_cell_ix ? t.col[k]
                             : static_cast<int>(static_cast<unsigned>(t.col[k]) |
                                                (static_cast<unsigned>(t.cell[k]) << L.col_bits));
    L.d_row_ptr = upload(t.row_ptr);
    if (L.spec.field == wmc::Field::Channel) {
        const wmc::ChannelTables& c = L.ch;
        auto up = [&](const auto& v) {
            auto* p = upload(v);
            L.ch_bufs.push_back(static_cast<void*>(p));
            return p;
        };
        wmc::ChannelArgs& a = L.ch_args;
        a.n_ent = static_cast<int>(c.e_li.size());
        a.vx = up(c.vx);
        a.vy = up(c.vy);
        a.vblend = up(c.vblend);
        a.tri = up(c.tri);
        a.ms = up(c.ms);
        a.m_ptr = up(c.m_ptr);
        a.m_tri = up(c.m_tri);
        a.e_li = up(c.e_li);
        a.e_lj = up(c.e_lj);
        a.e_mi = up(c.e_mi);
        a.e_mj = up(c.e_mj);
        a.e_ks = up(c.e_ks);
        a.k_ptr = up(c.k_ptr);
        a.k_tri = up(c.k_tri);
    }
    {
        // sweep row descriptors: single-cell rows, and among them the
        // structured 5-point rows {i - dS, i - 1, i, i + 1, i + dN} whose
        // (off-diagonal, diagonal) a0 pair is one of <= kMaxRowTypes values
        std::vector<int4> desc(t.n);
        std::vector<std::pair<double, double>> types;
        for (int i = 0; i < t.n; ++i) {
            const int b = t.row_ptr[i], e = t.row_ptr[i + 1];
            int c = t.cell[b];
            for (int k = b; k < e; ++k)
                if (t.cell[k] != c) c = -1;
            if (c > 0xffff) c = -1;  // the descriptor holds 16 cell bits
            desc[i] = make_int4(c, b, 0, 0);
            if (c < 0 || e - b != 5 || std::getenv("WMC_SWEEP_GENERIC")) continue;
            const int* col = t.col.data() + b;
            const double* w = t.a0.data() + b;
            if (col[1] != i - 1 || col[2] != i || col[3] != i + 1 || !(col[0] < i - 1) || !(col[4] > i + 1)) continue;
            if (w[0] != w[1] || w[0] != w[3] || w[0] != w[4]) continue;
            int type = -1;
            for (std::size_t q = 0; q < types.size(); ++q)
                if (types[q].first == w[0] && types[q].second == w[2]) type = static_cast<int>(q);
            if (type < 0) {
                if (static_cast<int>(types.size()) == wmc::kMaxRowTypes) continue;
                type = static_cast<int>(types.size());
                types.emplace_back(w[0], w[2]);
            }
            // deepest tier whose P holds all five columns: the substep
            // kernels of tiers <= pfull take the structured gather too
            int pfull = 255;
            for (int q = 0; q < 5; ++q) pfull = std::min<int>(pfull, t.dof_tier[col[q]]);
            desc[i] = make_int4(c | ((type + 1) << 16) | (pfull << 24), b, i - col[0], col[4] - i);
        }
        L.n_row_types = static_cast<int>(types.size());
        for (std::size_t q = 0; q < types.size(); ++q) L.row_types[q] = make_double2(types[q].first, types[q].second);
        for (const auto& d : desc) L.n_structured += d.x >= 0 && ((d.x >> 16) & 0xff) > 0;
        {
            // fused solve (TMEM form 2): the rows outside R that are not
            // structured, at most two per thread of the 512-thread CTA and
            // kNsMax entries each, keep their CSR entries in TMEM
            std::vector<int> ns;
            bool ok = L.d_cell_ix == nullptr;
            for (int i = t.n_r; i < t.n && ok; ++i) {
                const int4 d = desc[i];
                if (d.x >= 0 && ((d.x >> 16) & 0xff) > 0) continue;
                if (t.row_ptr[i + 1] - t.row_ptr[i] > wmc::kNsMax) ok = false;
                ns.push_back(i);
            }
            const char* e = std::getenv("WMC_FUSED_NS_TMEM");  // A/B knob (0: off)
            if (ok && !ns.empty() && static_cast<int>(ns.size()) <= 2 * t.lat_threads && t.lat_threads <= 512 &&
                !(e && std::atoi(e) == 0)) {
                L.d_ns_rows = upload(ns);
                L.n_ns = static_cast<int>(ns.size());
            }
        }
        if (std::getenv("WMC_DEBUG_ROWS")) {  // row-class census (tuning)
            long st = 0, single = 0, multi = 0, len_max = 0, len_sum = 0, long_rows = 0;
            for (int i = t.n_r; i < t.n; ++i) {
                const int4 d = desc[i];
                const int len = t.row_ptr[i + 1] - t.row_ptr[i];
                if (d.x >= 0 && ((d.x >> 16) & 0xff) > 0) { ++st; continue; }
                (d.x >= 0 ? single : multi) += 1;
                len_max = std::max<long>(len_max, len);
                len_sum += len;
                long_rows += len > 9;
            }
            std::fprintf(stderr, "rows outside R: n=%d n_r=%d structured=%ld single-cell=%ld multi-cell=%ld "
                         "generic len max=%ld mean=%.2f (>9: %ld) types=%zu\n", t.n, t.n_r, st, single, multi,
                         len_max, (single + multi) ? double(len_sum) / double(single + multi) : 0.0, long_rows,
                         types.size());
        }
        L.d_row_desc = upload(desc);
        L.d_wtype = upload(std::vector<double2>(L.row_types, L.row_types + wmc::kMaxRowTypes));
    }
    L.d_ent = upload(ent);
    L.d_a0 = upload(t.a0);
    L.d_z0 = upload(t.z0);

    // substep path: structured lattice kernel, generic on-chip kernel, or the
    // HBM-resident kernel when R is too large for one SM (WMC_SUBSTEP_PATH
    // = lattice|onchip|global forces one, for tests)
    const bool lts = t.kind == wmc::Integrator::LocalTimeStepping && t.n_r > 0 && t.p > 1;
    const char* force_path = std::getenv("WMC_SUBSTEP_PATH");
    const std::string fp = force_path ? force_path : "";
    L.n_wid = static_cast<int>(t.rc_ptr.size()) - 1;
    const bool onchip_rows = t.n_r <= wmc::kSubThreads * wmc::kSubMaxRpt && t.n_r < 65536 && L.n_wid < 65535;
    // (one weight per SELL entry and sample on chip: per-element fields on a
    // large R leave no room for the substep state; they take the HBM-resident
    // substeps, whose entries then carry their cells in a separate array)
    const bool onchip_fits = onchip_rows && 8.0 * L.n_wid + 16.0 * t.n_r < 200.0 * 1024.0;
    if (lts && t.n_cells > wmc::kMaxCells && t.tiers > 1)
        throw ConfigError("level: nested tiers support at most 511 coefficient cells");
    auto upload_global = [&] {  // tables of the HBM-resident substeps
        L.d_apg_ptr = upload(t.apg_ptr);
        if (t.n_cells > wmc::kMaxCells) {
            L.d_apg_ent = upload(t.apg_col);
            L.d_apg_cell = upload(t.apg_cell);
        } else {
            L.d_apg_ent = upload(t.apg_ent);
        }
        L.d_apg_a0 = upload(t.apg_a0);
    };
    if (lts && t.tiers > 1) {
        // nested tiers: HBM-resident stage kernels
        if (t.tiers > wmc::kMaxTiers) throw ConfigError("level: too many tiers");
        L.path = SubPath::Tiers;
        for (int k = 0; k < t.tiers; ++k) {
            L.d_tier_ptr.push_back(upload(t.tier_ptr[k]));
            L.d_tier_ent.push_back(upload(t.tier_ent[k]));
            L.d_tier_a0.push_back(upload(t.tier_a0[k]));
        }
        std::vector<double> cm;
        for (const auto& v : t.tier_cm) cm.insert(cm.end(), v.begin(), v.end());
        L.d_tier_cm = upload(cm);
        L.d_beta = upload(t.beta);
    } else if (lts && (fp == "global" || fp == "tiled" || !onchip_fits ||
                       // p = 2 levels too large for the fused solve: the single
                       // substep of the HBM/L2-resident kernel also forms z_{n+1}
                       // (no per-sample weight set-up, no separate R update);
                       // measured 1.17x on config-1 level 4
                       (fp.empty() && t.p == 2 && t.n_cells <= wmc::kMaxCells &&
                        16.0 * t.n + 16.0 * (t.n_r + 16) > 227.0 * 1024.0))) {
        if (t.n > wmc::kColMask) throw ConfigError("level: more than 2^23 DOFs");
        L.path = SubPath::Global;
        // the temporally blocked step when the level has a refined box (R in
        // tiles, every substep on chip); WMC_TILED=0 keeps the HBM-resident
        // substeps (A/B), WMC_SUBSTEP_PATH=global as well
        // (automatic only where R does not fit one SM: small boxes take the
        // HBM/L2-resident substeps, whose halo-free layout wins there)
        const char* tiled_env = std::getenv("WMC_TILED");
        if ((fp == "tiled" || (fp.empty() && !onchip_fits)) && !(tiled_env && std::atoi(tiled_env) == 0) &&
            !L.d_cell_ix) {
            // WMC_STREAM=0: tiles only (no streamed interior)
            const char* stream_env = std::getenv("WMC_STREAM");
            const bool stream = !(stream_env && std::atoi(stream_env) == 0);
            wmc::TilePlan plan = wmc::plan_tiles(t, wmc::kTileWz, wmc::kTileHz, wmc::kTileK,
                                                 stream ? wmc::kStreamThreads : 0, wmc::kStreamMaxP);
            if (std::getenv("WMC_DEBUG_TILES"))
                std::fprintf(stderr, "tile plan: ok=%d layout=%s reason=%s tiles=%d slabs=%d max_gen=%d max_app=%d "
                             "max_ent=%d work=%.3f notes=%s\n", plan.ok, plan.layout.c_str(), plan.reason.c_str(),
                             plan.n_tiles, plan.n_slabs, plan.max_gen, plan.max_app, plan.max_ent, plan.work_factor,
                             plan.notes.c_str());
            if (plan.ok) {
                auto up = [&](const auto& v) {
                    auto* p = upload(v);
                    L.tile_bufs.push_back(static_cast<void*>(p));
                    return p;
                };
                wmc::TileArgs& a = L.tile;
                std::vector<int4> rect(plan.n_tiles), oj(plan.n_tiles);
                for (int q = 0; q < plan.n_tiles; ++q) {
                    rect[q] = make_int4(plan.i0[q], plan.j0[q], plan.oi0[q], plan.oi1[q]);
                    oj[q] = make_int4(plan.oj0[q], plan.oj1[q], plan.tiles_shape[q], 0);
                }
                a.p = t.p;
                a.m = t.lat_m;
                a.n_cells = t.n_cells;
                a.cells_x = L.spec.cells_x;
                a.box_slots = plan.box_slots;
                a.max_app = plan.max_app;
                a.max_ent = plan.max_ent;
                a.max_gen = plan.max_gen;
                a.n_tiles = plan.n_tiles;
                a.inv_h = t.lat_inv_h;
                a.h = 1.0 / t.lat_inv_h;
                a.inv_h2 = t.lat_inv_h * t.lat_inv_h;
                a.c0 = t.c0;
                a.tile_rect = up(rect);
                a.tile_oj = up(oj);
                {
                    std::vector<int4> tg(plan.thr_geo.size() / 4);
                    for (std::size_t q = 0; q < tg.size(); ++q)
                        tg[q] = make_int4(plan.thr_geo[4 * q], plan.thr_geo[4 * q + 1], plan.thr_geo[4 * q + 2], 0);
                    a.thr_geo = up(tg);
                }
                a.gen_off = up(plan.gen_off);
                a.g_slot = up(plan.g_slot);
                a.g_dof = up(plan.g_dof);
                a.g_owned = up(plan.g_owned);
                a.g_rs = up(plan.g_rs);
                a.g_ent_off = up(plan.g_ent_off);
                a.g_rem_off = up(plan.g_rem_off);
                a.e_slot = up(plan.e_slot);
                a.e_rc_off = up(plan.e_rc_off);
                a.rc_cell = up(plan.rc_cell.empty() ? std::vector<int>{0} : plan.rc_cell);
                a.rc_a0 = up(plan.rc_a0.empty() ? std::vector<double>{0.0} : plan.rc_a0);
                a.r_dof = up(plan.r_dof.empty() ? std::vector<int>{0} : plan.r_dof);
                a.r_rc_off = up(plan.r_rc_off);
                a.rr_cell = up(plan.rr_cell.empty() ? std::vector<int>{0} : plan.rr_cell);
                a.rr_a0 = up(plan.rr_a0.empty() ? std::vector<double>{0.0} : plan.rr_a0);
                std::vector<unsigned char> lr(plan.line_row.begin(), plan.line_row.end());
                a.line_row = up(lr);
                a.cellx = up(t.lat_cellx);
                a.celly = up(t.lat_celly);
                a.beta = up(t.beta);
                a.cm = up(t.cm);
                L.tile_smem = wmc::tile_smem_bytes(a);
                L.tile_work = plan.work_factor;
                if (plan.n_slabs > 0) {
                    wmc::StreamArgs& sa = L.slabs;
                    std::vector<int4> sg(plan.n_slabs), so(plan.n_slabs);
                    for (int q = 0; q < plan.n_slabs; ++q) {
                        sg[q] = make_int4(plan.slab[4 * q], plan.slab[4 * q + 1], plan.slab[4 * q + 2],
                                          plan.slab[4 * q + 3]);
                        so[q] = make_int4(plan.slab_own[4 * q], plan.slab_own[4 * q + 1], plan.slab_own[4 * q + 2],
                                          plan.slab_own[4 * q + 3]);
                    }
                    sa.p = t.p;
                    sa.m = t.lat_m;
                    sa.cells_x = L.spec.cells_x;
                    sa.n_slabs = plan.n_slabs;
                    sa.threads = plan.slab_threads;
                    sa.chunks = 1;
                    sa.chunk_cols = plan.slab_own[1] - plan.slab_own[0];
                    L.slab_width = sa.chunk_cols;
                    sa.max_nx = plan.max_nx;
                    sa.inv_h = a.inv_h;
                    sa.h = a.h;
                    sa.inv_h2 = a.inv_h2;
                    sa.c0 = t.c0;
                    for (int q = 0; q + 1 < t.p; ++q) {
                        sa.opb[q] = 1.0 + t.beta[q];
                        sa.beta[q] = t.beta[q];
                        sa.cm[q] = t.cm[q];
                    }
                    sa.slab = up(sg);
                    sa.slab_own = up(so);
                    sa.cellx = a.cellx;
                    sa.celly = a.celly;
                    L.stream_smem = wmc::stream_smem_bytes(sa);
                }
                int optin = 0;
                cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, L.device);
                if (L.tile_smem + 64 <= optin) L.path = SubPath::Tiled;
                // CTAs per SM: registers allow 512 / threads; each takes its shared memory plus 1 KB
                int smem_per_sm = 0;
                cudaDeviceGetAttribute(&smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, L.device);
                L.tile_ctas_per_sm = std::max(1, std::min(512 / wmc::kTileThreads, smem_per_sm / (L.tile_smem + 1024)));
            }
        }
        if (L.path == SubPath::Global) upload_global();
    }
    if (lts && L.path != SubPath::Global && L.path != SubPath::Tiers && L.path != SubPath::Tiled) {
        const int n_slices = (t.n_r + 31) / 32;
        std::vector<int> soff(n_slices + 1, 0);
        std::vector<std::uint32_t> sent;
        const std::uint32_t pad = static_cast<std::uint32_t>(L.n_wid) << 16;
        for (int sl = 0; sl < n_slices; ++sl) {
            int width = 0;
            for (int l = 0; l < 32; ++l) {
                const int r = sl * 32 + l;
                if (r < t.n_r) width = std::max(width, t.ap_row_ptr[r + 1] - t.ap_row_ptr[r]);
            }
            const std::size_t base = sent.size();
            sent.resize(base + static_cast<std::size_t>(width) * 32, pad);
            for (int l = 0; l < 32; ++l) {
                const int r = sl * 32 + l;
                if (r >= t.n_r) continue;
                for (int e = t.ap_row_ptr[r]; e < t.ap_row_ptr[r + 1]; ++e) {
                    const int slot = e - t.ap_row_ptr[r];
                    sent[base + slot * 32 + l] =
                        static_cast<std::uint32_t>(t.ap_col[e]) | (static_cast<std::uint32_t>(t.ap_wid[e]) << 16);
                }
            }
            soff[sl + 1] = static_cast<int>(sent.size());
        }
        L.n_sub_ent = static_cast<int>(sent.size());
        L.d_sub_ent = upload(sent);
        L.d_slice_off = upload(soff);
        L.d_rc_ptr = upload(t.rc_ptr);
        L.d_rc_cell = upload(t.rc_cell);
        L.d_rc_a0 = upload(t.rc_a0);
        L.d_beta = upload(t.beta);
        L.d_cm = upload(t.cm);
        wmc::SubArgs probe{};
        probe.n_r = t.n_r;
        probe.p = t.p;
        probe.n_wid = L.n_wid;
        probe.n_cells = t.n_cells;
        probe.n_ent = L.n_sub_ent;
        probe.cl_smem = 1;
        L.sub_smem = wmc::substep_smem_bytes(probe);
        L.sub_grid = wmc::substep_max_grid(L.device, L.sub_smem);
        if (L.sub_grid <= 0) {  // many cells (channel): recipes read the coefficients from global memory
            probe.cl_smem = 0;
            L.sub_smem = wmc::substep_smem_bytes(probe);
            L.sub_grid = wmc::substep_max_grid(L.device, L.sub_smem);
            L.sub_cl_smem = 0;
        }
    }
    if (!t.field_x.empty() && L.spec.field != wmc::Field::LognormalKLElem) L.d_field_x = upload(t.field_x);
    if (!t.field_table.empty()) L.d_field_table = upload(t.field_table);
    if (L.spec.field == wmc::Field::LognormalKLElem) {
        // one table row per triangle, at its centroid (level.cpp keeps them in field_x)
        const wmc::KLTable kl = wmc::kl_point_table(t.field_x, L.spec.kl_sigma, L.spec.kl_corr_len, L.spec.kl_modes);
        L.d_kl = upload(kl.t);
    }
    if (L.spec.field == wmc::Field::LognormalKL) {
        const wmc::KLTable kl =
            wmc::kl_cell_table(L.spec.cells_x, L.spec.cells_y, L.spec.kl_sigma, L.spec.kl_corr_len, L.spec.kl_modes);
        L.d_kl = upload(kl.t);
    }
    if (t.cfl_safety > 0.0) {
        // the reference normalises the warm start before iterating (fem.cpp:137-146)
        auto norm = [](const std::vector<double>& v) {
            double acc = 0.0;
            for (double x : v) acc += x * x;
            const double n = std::sqrt(acc);
            return n == 0.0 ? 1.0 : n;
        };
        L.d_warm_full = upload(t.warm_full);
        L.warm_full_norm = norm(t.warm_full);
        if (!t.warm_coarse.empty()) {
            L.d_warm_coarse = upload(t.warm_coarse);
            L.warm_coarse_norm = norm(t.warm_coarse);
        }
        L.d_in_p = upload(t.in_p);
    }
    L.d_qptr = upload(t.qoi_ptr);
    L.d_qdof = upload(t.qoi_dof);
    L.d_qw = upload(t.qoi_w);
    L.d_qsm = upload(t.sqrt_mass_qoi);

    int max_gen_width = 0;
    for (std::size_t q = 0; q + 1 < t.gen_ptr.size(); ++q)
        max_gen_width = std::max(max_gen_width, t.gen_ptr[q + 1] - t.gen_ptr[q]);
    if (lts && L.path == SubPath::None && t.lattice && static_cast<int>(t.gen_rows.size()) <= 1024 &&
        max_gen_width <= wmc::kLatGenWidth) {
        // SELL-32 over the generic rows, per slot: column and recipe range
        const int n_gen = static_cast<int>(t.gen_rows.size());
        const int n_slices = (n_gen + 31) / 32;
        // rows sorted by entry count (descending) so each 32-row slice is
        // padded only to its own widest row
        std::vector<int> ord(n_gen);
        for (int q = 0; q < n_gen; ++q) ord[q] = q;
        const char* pad8 = std::getenv("WMC_GEN_PAD8");  // tuning: unsorted, every slice 8 wide
        const bool fixed_width = pad8 && std::atoi(pad8);
        if (!fixed_width)
            std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
                return t.gen_ptr[x + 1] - t.gen_ptr[x] > t.gen_ptr[y + 1] - t.gen_ptr[y];
            });
        SlotPerm perm(n_gen);
        for (int q = 0; q < n_gen; ++q)
            for (int e = 0; e < t.gen_ptr[q + 1] - t.gen_ptr[q]; ++e) perm[q].push_back(e);
        if (!fixed_width && !std::getenv("WMC_GEN_NO_BANKS")) optimize_generic_lanes(t, ord, perm);
        std::vector<int> grows(n_gen);
        std::vector<double> grs(n_gen);
        for (int q = 0; q < n_gen; ++q) {
            grows[q] = t.gen_rows[ord[q]];
            grs[q] = t.gen_rs[ord[q]];
        }
        std::vector<int> soff(n_slices + 1, 0), ovf_start{0};
        std::vector<std::uint16_t> gcol, ovf_cell;
        std::vector<double> ovf_a0, slot_a0;
        std::vector<std::uint16_t> slot_cell;
        for (int sl = 0; sl < n_slices; ++sl) {
            int width = fixed_width ? wmc::kLatGenWidth : 0;
            for (int l = 0; l < 32; ++l) {
                const int q = sl * 32 + l;
                if (q < n_gen) width = std::max(width, static_cast<int>(perm[ord[q]].size()));  // entries and holes
            }
            // slots go in pairs, [slice][pair][lane][2]: a lane's two weights
            // are one 16-byte load and its two columns one 32-bit load
            width = (width + 1) & ~1;
            for (int pr = 0; pr < width / 2; ++pr)
                for (int l2 = 0; l2 < 64; ++l2) {
                    const int l = l2 >> 1, e = 2 * pr + (l2 & 1);
                    const int q = sl * 32 + l;
                    std::uint16_t c = 0;
                    double a1 = 0.0;
                    std::uint16_t k1 = 0;
                    if (q < n_gen && e < static_cast<int>(perm[ord[q]].size()) && perm[ord[q]][e] >= 0) {
                        const int ent = t.gen_ptr[ord[q]] + perm[ord[q]][e];
                        c = static_cast<std::uint16_t>(t.gen_col[ent]);
                        const int nt = t.gen_rc_ptr[ent + 1] - t.gen_rc_ptr[ent];
                        if (nt == 1) {
                            a1 = t.gen_rc_a0[t.gen_rc_ptr[ent]];
                            k1 = static_cast<std::uint16_t>(t.gen_rc_cell[t.gen_rc_ptr[ent]]);
                        } else {
                            k1 = static_cast<std::uint16_t>(wmc::kOvfFlag | (ovf_start.size() - 1));
                            for (int k = t.gen_rc_ptr[ent]; k < t.gen_rc_ptr[ent + 1]; ++k) {
                                ovf_cell.push_back(static_cast<std::uint16_t>(t.gen_rc_cell[k]));
                                ovf_a0.push_back(t.gen_rc_a0[k]);
                            }
                            ovf_start.push_back(static_cast<int>(ovf_cell.size()));
                        }
                    }
                    gcol.push_back(c);
                    slot_a0.push_back(a1);
                    slot_cell.push_back(k1);
                }
            soff[sl + 1] = static_cast<int>(gcol.size());
        }
        L.n_slots = static_cast<int>(gcol.size());
        L.d_strip_j0 = upload(t.strip_j0);
        {
            // nodes read through shared memory by another thread: warp-edge
            // lanes (E/W shuffles stop there), strip ends (N/S across
            // strips) and every lattice node a generic row gathers
            const int W = t.lat_m + 1;
            std::vector<std::uint8_t> gen_read(static_cast<std::size_t>(W) * W, 0);
            for (int c : t.gen_col)
                if (c < W * W) gen_read[c] = 1;
            std::vector<unsigned char> mask(t.lat_threads, 0);
            for (int tid = 0; tid < t.lat_threads; ++tid) {
                const int col = tid % t.lat_cw, strip = tid / t.lat_cw, ci = 1 + col;
                if (ci > t.lat_m - 1 || strip >= static_cast<int>(t.strip_j0.size())) continue;
                const int lane = tid & 31, j0 = t.strip_j0[strip], len = t.strip_len[strip];
                for (int k = 0; k < len; ++k) {
                    const bool ext = lane == 0 || lane == 31 || k == 0 || k == len - 1 ||
                                     gen_read[static_cast<std::size_t>(ci) * W + j0 + k];
                    if (ext) mask[tid] |= static_cast<unsigned char>(1u << k);
                }
            }
            L.d_lat_smask = upload(mask);
        }
        L.d_strip_len = upload(t.strip_len);
        L.d_cellx = upload(t.lat_cellx);
        L.d_celly = upload(t.lat_celly);
        L.d_gen_rows = upload(grows);
        {
            // fused solve: A (I - P) entries of the generic rows (the A P part of
            // g = A z_n comes from the SELL on v = z / sqrt(M)), sorted order
            std::vector<int> rp{0}, rcol, rcell;
            std::vector<double> ra0;
            for (int q = 0; q < n_gen; ++q) {
                const int r = grows[q];
                for (int e = t.row_ptr[r]; e < t.row_ptr[r + 1]; ++e)
                    if (!t.in_p[t.col[e]]) {
                        rcol.push_back(t.col[e]);
                        rcell.push_back(t.cell[e]);
                        ra0.push_back(t.a0[e]);
                    }
                rp.push_back(static_cast<int>(rcol.size()));
            }
            L.d_rem_ptr = upload(rp);
            L.d_rem_col = upload(rcol);
            L.d_rem_cell = upload(rcell);
            L.d_rem_a0 = upload(ra0);
        }
        L.d_gen_rs = upload(grs);
        L.d_gen_soff = upload(soff);
        {
            // balanced warp -> slice assignment (longest slice first onto the
            // least-loaded warp with a free role), so no warp carries two
            // wide slices while others idle at the substep barrier
            const int warps = t.lat_threads / 32, G = t.lat_threads == 1024 ? 1 : 2;
            std::vector<int> table(static_cast<std::size_t>(warps) * G, -1), load(warps, 0), used(warps, 0);
            const char* plain = std::getenv("WMC_GEN_PLAIN_ASSIGN");  // A/B knob: slice q of role u to warp q % warps
            for (int sl = 0; sl < n_slices; ++sl) {
                const int width = (soff[sl + 1] - soff[sl]) / 32;
                int best = -1;
                if (plain) {
                    best = sl % warps;
                    if (used[best] >= G) best = -1;
                } else {
                    for (int w = 0; w < warps; ++w)
                        if (used[w] < G && (best < 0 || load[w] < load[best])) best = w;
                }
                if (best < 0) throw ConfigError("level: generic rows exceed the lattice kernel's roles");
                table[static_cast<std::size_t>(best) * G + used[best]++] = sl;
                load[best] += width;
            }
            L.d_gen_warp_slice = upload(table);
        }
        L.d_gen_col = upload(gcol);
        L.d_slot_rc = upload(ovf_start);
        L.d_slot_a0 = upload(slot_a0);
        L.d_slot_cell = upload(slot_cell);
        L.n_ovf = static_cast<int>(ovf_start.size()) - 1;
        L.n_ovf_terms = static_cast<int>(ovf_cell.size());
        L.d_ovf_cell = upload(ovf_cell);
        L.d_grc_a0 = upload(ovf_a0);
        wmc::LatArgs probe{};
        probe.threads = t.lat_threads;
        probe.strip_k = t.lat_k;
        probe.n_r = t.n_r;
        probe.p = t.p;
        probe.n_cells = t.n_cells;
        probe.m = t.lat_m;
        probe.n_strips = static_cast<int>(t.strip_j0.size());
        probe.n_gen = n_gen;
        probe.n_slots = L.n_slots;
        probe.n_ovf = L.n_ovf;
        probe.n_ovf_terms = L.n_ovf_terms;
        L.lat_smem = wmc::lattice_smem_bytes(probe);
        L.lat_grid = wmc::substep_max_grid(L.device, L.lat_smem);
        L.lattice = L.lat_grid > 0;
    }
    if (lts && L.path == SubPath::None) {
        L.path = (L.lattice && fp != "onchip") ? SubPath::Lattice : SubPath::OnChip;
        if (L.path == SubPath::OnChip && L.sub_grid <= 0) {
            // the SELL of R does not fit one SM (per-element coefficients: every
            // entry its own weight): the HBM-resident substeps instead
            if (t.n > wmc::kColMask) throw ConfigError("level: substep working set exceeds shared memory");
            L.path = SubPath::Global;
            upload_global();
        }
    }
    L.lattice = L.path == SubPath::Lattice;
    {
        const char* e = std::getenv("WMC_SWEEP_WIDE");  // A/B knob, fixed per level
        L.sweep_wide = e ? std::atoi(e) : 23;
    }
    {
        // fused small-mesh solve: the batched arithmetic is mirrored for the
        // leap-frog / p = 1 and on-chip generic substep paths
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, L.device);
        L.n_sms = sms > 0 ? sms : 148;
        if ((L.path == SubPath::None || L.path == SubPath::OnChip) && t.tiers == 1 && t.n_r < 65536) {
            wmc::SmallArgs probe{};
            probe.n = t.n;
            probe.n_r = t.n_r;
            probe.n_cells = t.n_cells;
            probe.n_wid = L.path == SubPath::OnChip ? L.n_wid : 0;
            const int bytes = wmc::small_smem_bytes(probe);
            if (bytes <= wmc::small_max_smem(L.device)) L.small_smem = bytes;
        }
        // fused lattice solve: lattice levels whose z_n (and z_{n-1} when it
        // fits) stay on chip next to the substep state; WMC_FUSED=0 disables
        const char* fz = std::getenv("WMC_FUSED");
        if (L.path == SubPath::Lattice && t.tiers == 1 && t.lat_threads == 512 && t.lat_k == 8 &&
            !(fz && std::atoi(fz) == 0)) {
            wmc::LatSolveArgs probe{};
            probe.lat.n_r = t.n_r;
            probe.lat.p = t.p;
            probe.lat.n_cells = t.n_cells;
            probe.lat.m = t.lat_m;
            probe.lat.n_strips = static_cast<int>(t.strip_j0.size());
            probe.lat.n_slots = L.n_slots;
            probe.n = t.n;
            L.fused_tmem = fused_tmem();
            probe.tmem = L.fused_tmem;
            // taken when z_{n-1} fits on chip too: config-1 levels 0, 1 and,
            // with the generic weights in tensor memory (which frees their
            // shared-memory table), level 2 (n = 8 433; 1.09x over the
            // per-step kernels although 3 752 rows lie outside R).  Without
            // tensor memory the rows outside R must be at most two per
            // thread (round-robin, latency-bound gathers).
            // WMC_FUSED_ZP_GLOBAL=1 forces the layout with z_{n-1} in global
            // memory (tests; it is slower where the rows outside R are many)
            const int cap = wmc::lattice_solve_max_smem(L.device);
            const char* zg = std::getenv("WMC_FUSED_ZP_GLOBAL");
            if (zg && std::atoi(zg) != 0) {
                probe.zp_global = reinterpret_cast<double*>(16);  // layout without z_{n-1}
                L.fused_zp_global = true;
            }
            const int bytes = wmc::lattice_solve_smem_bytes(probe);
            const char* ff = std::getenv("WMC_FUSED_FORCE");  // tuning knob: ignore the rows-outside-R limit
            const bool force = ff && std::atoi(ff) != 0;
            if (bytes <= cap &&
                (force || L.fused_tmem || L.fused_zp_global || t.n - t.n_r <= 2 * t.lat_threads))
                L.fused_smem = bytes;
        }
    }
    L.d_cells = nullptr;
    check(cudaMalloc(&L.d_cells, sizeof(double) * std::max<std::size_t>(static_cast<std::size_t>(L.batch) * t.n_cells, 1)),
          "cudaMalloc batch");
    check(cudaMalloc(&L.d_dq, sizeof(double) * std::max(L.batch, 1)), "cudaMalloc batch");
}

int g_stride(const wmc::LevelTables& t) { return std::max(8, (t.n_r + 7) / 8 * 8); }

Workspace& workspace(wmc_level& L, int role) {
    Workspace& w = L.ws[role];
    if (!w.za) {
        const std::size_t S = static_cast<std::size_t>(L.batch);
        const wmc::LevelTables& t = L.tab;
        auto alloc = [&](auto** p, std::size_t elems) {
            check(cudaMalloc(p, sizeof(**p) * std::max<std::size_t>(elems, 1)), "cudaMalloc batch");
        };
        alloc(&w.za, S * t.n);
        alloc(&w.zb, S * t.n);
        if (L.path != SubPath::Tiled) alloc(&w.g, S * static_cast<std::size_t>(g_stride(t)));  // tiled: g on chip
        alloc(&w.fail, S);
        alloc(&w.q, S * t.nq);
        if (L.path == SubPath::Global) {
            alloc(&w.da, S * t.n_r);
            alloc(&w.db, S * t.n_r);
        }
        if (t.cfl_safety > 0.0) {
            alloc(&w.rel, S);
            alloc(&w.nsteps, S);
            alloc(&w.eig, S * (2 * kEigBlocks + 5));
            alloc(&w.eig_i, S * 3 + 1);
            alloc(&w.it_full, S);
            alloc(&w.it_coarse, S);
            check(cudaMallocHost(&w.h_active, sizeof(int)), "cudaMallocHost");
            check(cudaMallocHost(&w.h_nsteps, sizeof(int) * S), "cudaMallocHost");
        }
        if (L.path == SubPath::Tiers) {
            w.tier_e.assign(2 * t.tiers, nullptr);
            w.tier_rhs.assign(t.tiers, nullptr);
            for (int k = 0; k < t.tiers; ++k) {
                const std::size_t rows = static_cast<std::size_t>(t.n_r_tier[k]);
                alloc(&w.tier_e[2 * k], S * rows);
                alloc(&w.tier_e[2 * k + 1], S * rows);
                if (k > 0) alloc(&w.tier_rhs[k], S * rows);
            }
        }
    }
    return w;
}

// one batch of solves on level L with coefficients `cells` (stride S), result
// Q per sample in L.d_q; asynchronous on `stream`
cudaEvent_t mark(wmc_level& L, std::vector<cudaEvent_t>& v, cudaStream_t st) {
    cudaEvent_t e;
    check(cudaEventCreate(&e), "cudaEventCreate");
    check(cudaEventRecord(e, st), "cudaEventRecord");
    v.push_back(e);
    (void)L;
    return e;
}

// Nested tiers, one global step after the sweep: depth-first over the
// stage tree, tier k's stage m followed by the whole tier-(k+1) solve that
// replaces the stage's right-hand side on R_k+1.  At stage 0 the right-hand
// side of tier k+1 is r_k itself (no product yet), so tier k+1 reads r_k.
void run_tiers(wmc_level& L, Workspace& ws, const double* cells, int S, int count, const double* zc, double* zp,
               int step, const double* rel, const int* nsteps, cudaStream_t stream) {
    const wmc::LevelTables& t = L.tab;
    const int K = t.tiers, p = t.p;
    wmc::TierArgs a{};
    a.p = p;
    a.S = S;
    a.count = count;
    a.cells = cells;
    a.row_desc = L.d_row_desc;
    a.wtype = L.d_wtype;
    a.zc = zc;
    a.zp = zp;
    a.step = step;
    a.fail = ws.fail;
    a.rel = rel;
    a.nsteps = nsteps;
    std::vector<int> stage(K + 1, 0);
    auto buf = [&](int j, int m) { return ws.tier_e[2 * (j - 1) + (m & 1)]; };
    auto run = [&](auto&& self, int k, const double* rhs) -> void {
        const int n_rk = t.n_r_tier[k - 1];
        const int split = k < K ? t.n_r_tier[k] : 0;
        for (int m = 0; m < p; ++m) {
            stage[k] = m;
            a.k = k;
            a.m = m;
            a.rhs = rhs;
            a.rhs_next = k < K ? ws.tier_rhs[k] : nullptr;
            a.src = m > 0 ? buf(k, m) : nullptr;
            a.ptr = L.d_tier_ptr[k - 1];
            a.ent = L.d_tier_ent[k - 1];
            a.a0 = L.d_tier_a0[k - 1];
            a.row_begin = m == 0 ? split : 0;
            a.row_end = n_rk;
            a.split = split;
            // the update chain of a row finishing at tier k stage m
            a.depth = 0;
            for (int j = k; j >= 1; --j) {
                const int mj = stage[j];
                auto& ln = a.link[a.depth++];
                ln = {};
                if (mj == 0) {
                    ln.C = t.tier_c0[j - 1];
                } else {
                    ln.A = 1.0 + t.beta[mj - 1];
                    ln.B = t.beta[mj - 1];
                    ln.C = t.tier_cm[j - 1][mj - 1];
                    ln.em = buf(j, mj);
                    ln.emm = mj >= 2 ? buf(j, mj + 1) : nullptr;
                }
                if (mj + 1 < p) {
                    ln.out = buf(j, mj + 1);
                    break;
                }
                if (j == 1) break;  // out == NULL: z_{n+1}
                ln.back = t.tier_back[j - 1];
            }
            if (a.row_end > a.row_begin) {
                wmc::launch_tier_stage(a, stream);
                ++g_launches;
                static const bool sync_debug = std::getenv("WMC_SYNC_DEBUG") != nullptr;  // debugging aid
                if (sync_debug) {
                    const cudaError_t e = cudaStreamSynchronize(stream);
                    if (e != cudaSuccess)
                        throw DeviceError(std::string("tier stage k=") + std::to_string(k) + " m=" + std::to_string(m) +
                                          ": " + cudaGetErrorString(e));
                }
            }
            if (split > 0) self(self, k + 1, m == 0 ? rhs : ws.tier_rhs[k]);
        }
    };
    run(run, 1, ws.g);
}

// Per-sample CFL (reference stable_dt, src/experiments.cpp:30-43): power
// iterations for the whole batch from the level's warm starts, then per
// sample dt, steps and the dt^2 scale of every constant.  Returns the largest
// step count of the live samples (the batch's horizon).
long cfl_phase(wmc_level& L, Workspace& ws, const double* cells, int S, int count, cudaStream_t stream) {
    const wmc::LevelTables& t = L.tab;
    const std::size_t SS = static_cast<std::size_t>(S);
    double* part = ws.eig;
    double* norm = part + 2 * kEigBlocks * SS;
    double* lam = norm + SS;
    double* lam_prev = lam + SS;
    double* lf = lam_prev + SS;
    double* lc = lf + SS;
    int* settled = ws.eig_i;
    int* iters = settled + SS;
    int* done = iters + SS;
    int* active = done + SS;
    auto power = [&](bool coarse, double* out) {
        wmc::EigArgs e{};
        e.n = t.n;
        e.S = S;
        e.count = count;
        e.row_ptr = L.d_row_ptr;
        e.ent = L.d_ent;
        e.col_bits = L.col_bits;
        e.cell_ix = L.d_cell_ix;
        e.col_mask = static_cast<int>((1u << L.col_bits) - 1u);
        e.a0 = L.d_a0;
        e.cells = cells;
        e.in_p = L.d_in_p;
        e.coarse = coarse ? 1 : 0;
        e.v = ws.za;
        e.av = ws.zb;
        e.n_blocks = kEigBlocks;
        e.part = part;
        e.norm = norm;
        e.lam = lam;
        e.lam_prev = lam_prev;
        e.settled = settled;
        e.iters = iters;
        e.done = done;
        e.active_count = active;
        e.tol = 1e-4;
        check(cudaMemsetAsync(lam_prev, 0, sizeof(double) * SS, stream), "memset");
        check(cudaMemsetAsync(settled, 0, sizeof(int) * 3 * SS, stream), "memset");
        wmc::launch_eig_init(coarse ? L.d_warm_coarse : L.d_warm_full, coarse ? L.warm_coarse_norm : L.warm_full_norm,
                             t.n, S, ws.za, stream);
        ++g_launches;
        // iterations are issued in groups between host checks: a settled
        // sample is frozen (done flag), so extra iterations do not change it
        int group = 4;
        for (int it = 0;;) {
            for (int k = 0; k < group && it < 20000; ++k, ++it) {
                check(cudaMemsetAsync(active, 0, sizeof(int), stream), "memset");
                wmc::launch_eig_iteration(e, stream);
                g_launches += 4;
            }
            check(cudaMemcpyAsync(ws.h_active, active, sizeof(int), cudaMemcpyDeviceToHost, stream), "copy");
            check(cudaStreamSynchronize(stream), "power iteration");
            if (*ws.h_active == 0) break;
            if (it >= 20000) throw NumericalError("max_eigenvalue: power iteration did not converge");
            group = std::min(2 * group, 32);
        }
        check(cudaMemcpyAsync(out, lam, sizeof(double) * SS, cudaMemcpyDeviceToDevice, stream), "copy");
    };
    power(false, lf);
    check(cudaMemcpyAsync(ws.it_full, iters, sizeof(int) * SS, cudaMemcpyDeviceToDevice, stream), "copy");
    const bool use_coarse = t.kind == wmc::Integrator::LocalTimeStepping && t.n_p > 0 && L.d_warm_coarse;
    if (use_coarse) {
        power(true, lc);
        check(cudaMemcpyAsync(ws.it_coarse, iters, sizeof(int) * SS, cudaMemcpyDeviceToDevice, stream), "copy");
    } else {
        check(cudaMemsetAsync(ws.it_coarse, 0, sizeof(int) * SS, stream), "memset");
    }
    wmc::launch_cfl_finalize(lf, lc, use_coarse ? 1 : 0, t.p_fine, t.cfl_safety, L.spec.final_time, t.dt, count, S,
                             ws.rel, ws.nsteps, stream);
    ++g_launches;
    check(cudaMemcpyAsync(ws.h_nsteps, ws.nsteps, sizeof(int) * S, cudaMemcpyDeviceToHost, stream), "copy");
    check(cudaStreamSynchronize(stream), "cfl");
    long n_max = 1;
    for (int s = 0; s < count; ++s) n_max = std::max<long>(n_max, ws.h_nsteps[s]);
    return n_max;
}

wmc::LatArgs lattice_args(const wmc_level& L, Workspace& ws, const double* cells, int S, int count) {
    const wmc::LevelTables& t = L.tab;
    wmc::LatArgs la{};
    la.threads = t.lat_threads;
    la.strip_k = t.lat_k;
    la.n_r = t.n_r;
    la.S = S;
    la.count = count;
    la.p = t.p;
    la.n_cells = t.n_cells;
    la.cells_x = L.spec.cells_x;
    la.m = t.lat_m;
    la.cw = t.lat_cw;
    la.n_strips = static_cast<int>(t.strip_j0.size());
    la.n_gen = static_cast<int>(t.gen_rows.size());
    la.n_slots = L.n_slots;
    la.inv_h = t.lat_inv_h;
    la.c0 = t.c0;
    la.strip_j0 = L.d_strip_j0;
    la.lat_smask = L.d_lat_smask;
    la.strip_len = L.d_strip_len;
    la.cellx = L.d_cellx;
    la.celly = L.d_celly;
    la.gen_rows = L.d_gen_rows;
    la.gen_rs = L.d_gen_rs;
    la.gen_soff = L.d_gen_soff;
    la.gen_warp_slice = L.d_gen_warp_slice;
    la.gen_col = L.d_gen_col;
    la.ovf_start = L.d_slot_rc;
    la.ovf_cell = L.d_ovf_cell;
    la.ovf_a0 = L.d_grc_a0;
    la.n_ovf = L.n_ovf;
    la.n_ovf_terms = L.n_ovf_terms;
    la.slot_a0 = L.d_slot_a0;
    la.slot_cell = L.d_slot_cell;
    la.cells = cells;
    la.gd = ws.g;
    la.g_stride = g_stride(t);
    la.beta = L.d_beta;
    la.cm = L.d_cm;
    return la;
}

void solve_batch_launches(wmc_level& L, Workspace& ws, const double* cells, int S, int count, cudaStream_t stream,
                          long n_steps, const double* rel, const int* nsteps) {
    const wmc::LevelTables& t = L.tab;
    const bool lts = L.path != SubPath::None;
    const bool global = L.path == SubPath::Global;
    const bool tiers = L.path == SubPath::Tiers;
    const bool tiled = L.path == SubPath::Tiled;
    wmc::launch_fill_int(ws.fail, INT_MAX, S, stream);

    wmc::SweepArgs sw{};
    sw.sample_major = tiled ? 1 : 0;  // the tiled step reads one sample's region contiguously
    sw.wide = L.sweep_wide;
    sw.n = t.n;
    sw.S = S;
    sw.count = count;
    sw.row_ptr = L.d_row_ptr;
    sw.col_bits = L.col_bits;
    sw.cell_ix = L.d_cell_ix;
    sw.col_mask = static_cast<int>((1u << L.col_bits) - 1u);
    sw.row_desc = L.d_row_desc;
    sw.wtype = L.d_wtype;
    sw.ent = L.d_ent;
    sw.a0 = L.d_a0;
    sw.cells = cells;
    sw.z0 = L.d_z0;
    sw.zp = ws.zb;
    sw.zc_out = ws.za;
    sw.factor = t.init_factor;
    sw.step = 1;
    sw.fail = ws.fail;
    sw.rel = rel;
    sw.nsteps = nsteps;
    wmc::launch_sweep_init(sw, stream);
    g_launches += 2;

    double* cur = ws.za;
    double* prev = ws.zb;
    wmc::LatArgs la{};
    if (lts && L.lattice) la = lattice_args(L, ws, cells, S, count);
    wmc::SubArgs sb{};
    if (lts) {
        sb.n_r = t.n_r;
        sb.S = S;
        sb.count = count;
        sb.p = t.p;
        sb.n_wid = L.n_wid;
        sb.n_cells = t.n_cells;
        sb.cl_smem = L.sub_cl_smem;
        sb.n_ent = L.n_sub_ent;
        sb.ent = L.d_sub_ent;
        sb.slice_off = L.d_slice_off;
        sb.rc_ptr = L.d_rc_ptr;
        sb.rc_cell = L.d_rc_cell;
        sb.rc_a0 = L.d_rc_a0;
        sb.cells = cells;
        sb.gd = ws.g;
        sb.g_stride = g_stride(t);
        sb.beta = L.d_beta;
        sb.cm = L.d_cm;
        sb.c0 = t.c0;
    }
    const int sub_grid = std::max(1, std::min(L.lattice ? L.lat_grid : L.sub_grid, count));
    la.rel = rel;
    la.nsteps = nsteps;
    sb.rel = rel;
    sb.nsteps = nsteps;
    for (long s = 1; s < n_steps; ++s) {
        la.step = static_cast<int>(s + 1);
        sb.step = static_cast<int>(s + 1);
        sw.zc = cur;
        sw.zp = prev;
        sw.zc_out = nullptr;
        sw.g = ws.g;
        sw.g_stride = g_stride(t);
        sw.g_node_major = (global || tiers) ? 1 : 0;
        sw.split = lts ? t.n_r : 0;
        sw.row_begin = tiled ? t.n_r : 0;  // the tiled step owns R
        sw.factor = t.coarse_factor;
        sw.step = static_cast<int>(s + 1);
        if (L.profile) mark(L, L.ev_sweep, stream);
        wmc::launch_sweep_step(sw, stream);
        if (std::getenv("WMC_SYNC_DEBUG")) {
            const cudaError_t e = cudaStreamSynchronize(stream);
            if (e != cudaSuccess) throw DeviceError(std::string("sweep: ") + cudaGetErrorString(e));
        }
        if (L.profile) mark(L, L.ev_sweep, stream);
        ++g_launches;
        if (tiled) {
            if (L.profile) mark(L, L.ev_sub, stream);
            wmc::TileArgs ta = L.tile;
            ta.S = S;
            ta.count = count;
            ta.cells = cells;
            ta.zc = cur;
            ta.zp = prev;
            ta.n = t.n;
            ta.fail = ws.fail;
            ta.step = static_cast<int>(s + 1);
            const long items = static_cast<long>(ta.n_tiles) * count;
            const int e = wmc::launch_tile_step(
                ta, static_cast<int>(std::min<long>(items, static_cast<long>(L.tile_ctas_per_sm) * L.n_sms)), stream);
            if (e != 0) check(static_cast<cudaError_t>(e), "tiled step launch");
            ++g_launches;
            if (L.slabs.n_slabs > 0) {
                wmc::StreamArgs sa = L.slabs;
                sa.S = S;
                sa.count = count;
                sa.n = t.n;
                sa.cells = cells;
                sa.zc = cur;
                sa.zp = prev;
                sa.fail = ws.fail;
                sa.step = static_cast<int>(s + 1);
                // column chunks: the split of the slabs' owned columns that
                // needs the fewest column iterations over the grid's rounds
                // (every chunk leads and trails by p columns and drains p levels)
                const long grid_max = static_cast<long>(512 / sa.threads) * L.n_sms;  // 128 registers per thread
                const int width = L.slab_width, lead = 3 * sa.p;
                long best = -1;
                static const char* force = std::getenv("WMC_STREAM_CHUNKS");  // A/B knob
                const int c_lo = force ? std::atoi(force) : 1, c_hi = force ? c_lo : 8;
                for (int c = c_lo; c <= c_hi && (c == c_lo || width / c >= 4 * lead); ++c) {
                    const int cols = (width + c - 1) / c;
                    const long rounds = (static_cast<long>(sa.n_slabs) * c * count + grid_max - 1) / grid_max;
                    const long cost = rounds * (cols + lead);
                    if (best < 0 || cost < best) {
                        best = cost;
                        sa.chunks = c;
                        sa.chunk_cols = cols;
                    }
                }
                const long sitems = static_cast<long>(sa.n_slabs) * sa.chunks * count;
                const int es = wmc::launch_stream_step(sa, static_cast<int>(std::min<long>(sitems, grid_max)), stream);
                if (es != 0) check(static_cast<cudaError_t>(es), "streamed step launch");
                ++g_launches;
            }
            if (L.profile) mark(L, L.ev_sub, stream);
        } else if (tiers) {
            if (L.profile) mark(L, L.ev_sub, stream);
            run_tiers(L, ws, cells, S, count, cur, prev, static_cast<int>(s + 1), rel, nsteps, stream);
            if (L.profile) mark(L, L.ev_sub, stream);
        } else if (global) {
            if (L.profile) mark(L, L.ev_sub, stream);
            wmc::GSubArgs ga{};
            ga.n_r = t.n_r;
            ga.S = S;
            ga.count = count;
            ga.ptr = L.d_apg_ptr;
            ga.ent = L.d_apg_ent;
            ga.cell_ix = L.d_apg_cell;
            ga.a0 = L.d_apg_a0;
            ga.cells = cells;
            ga.g = ws.g;
            ga.c0 = t.c0;
            ga.row_desc = L.d_row_desc;
            ga.wtype = L.d_wtype;
            ga.zc = cur;
            ga.zp = prev;
            ga.step = static_cast<int>(s + 1);
            ga.rel = rel;
            ga.nsteps = nsteps;
            ga.fail = ws.fail;
            for (int m = 1; m <= t.p - 1; ++m) {
                // d_m / d_{m-1}: m = 1 -> (-c0 g, 0); m = 2 -> (A, -c0 g); then A/B alternate
                ga.cur_mode = m == 1 ? 1 : 0;
                ga.prev_mode = m == 1 ? 2 : (m == 2 ? 1 : 0);
                ga.dcur = m == 1 ? nullptr : ((m % 2 == 0) ? ws.da : ws.db);
                ga.dprev = m == 1 ? ws.da : ((m % 2 == 0) ? ws.db : ws.da);
                ga.beta = t.beta[m - 1];
                ga.cm = t.cm[m - 1];
                ga.last = m == t.p - 1;
                wmc::launch_global_substep(ga, stream);
                ++g_launches;
            }
            if (L.profile) mark(L, L.ev_sub, stream);
        } else if (lts) {
            if (L.profile) mark(L, L.ev_sub, stream);
            const int e = L.lattice ? wmc::launch_lattice_substeps(la, sub_grid, stream)
                                    : wmc::launch_substeps(sb, sub_grid, stream);
            if (e != 0) check(static_cast<cudaError_t>(e), "substep launch");
            if (L.profile) mark(L, L.ev_sub, stream);
            wmc::RUpdateArgs ru{};
            ru.n_r = t.n_r;
            ru.S = S;
            ru.count = count;
            ru.g_stride = g_stride(t);
            ru.gd = ws.g;
            ru.zc = cur;
            ru.zp = prev;
            ru.step = static_cast<int>(s + 1);
            ru.fail = ws.fail;
            ru.nsteps = nsteps;
            if (L.profile) mark(L, L.ev_upd, stream);
            wmc::launch_r_update(ru, stream);
            if (L.profile) mark(L, L.ev_upd, stream);
            g_launches += 2;
        }
        std::swap(cur, prev);
    }
    wmc::QoIArgs qa{};
    qa.nq = t.nq;
    qa.ptr = L.d_qptr;
    qa.S = S;
    qa.count = count;
    qa.dof = L.d_qdof;
    qa.w = L.d_qw;
    qa.sqrt_mass = L.d_qsm;
    qa.z = cur;
    qa.fail = ws.fail;
    qa.q = ws.q;
    qa.z_alt = prev;
    qa.nsteps = nsteps;
    qa.n_max = static_cast<int>(n_steps);
    qa.n = t.n;
    qa.sample_major = tiled ? 1 : 0;
    wmc::launch_qoi(qa, stream);
    ++g_launches;
    check(cudaGetLastError(), "kernel launch");
}

// One batch of solves.  The whole launch sequence of a batch (start-up
// sweep, n_steps x {sweep, substeps, update}, QoI) depends only on the
// level, the workspace, the batch shape and the coefficient buffer, so from
// its second use it is replayed as a CUDA graph captured once: one launch
// per batch instead of ~3 n_steps (small batches of the adaptive driver are
// launch-bound).  Per-sample CFL batches (host-synchronised power
// iterations) and profiled runs take the plain path; WMC_NO_GRAPH=1 forces it.
// Fused small-mesh solve for small batches (bitwise the same results as the
// batched kernels; SmallArgs).  WMC_SMALL=0 disables it, WMC_SMALL=N sets the
// largest batch that takes it (default two samples per SM).
bool small_path(const wmc_level& L, int count) {
    if (L.small_smem <= 0) return false;
    static const int limit = [] {
        const char* v = std::getenv("WMC_SMALL");
        return v ? std::atoi(v) : -1;
    }();
    const int cap = limit >= 0 ? limit : 2 * L.n_sms;
    return count <= cap;
}

void small_solve(wmc_level& L, Workspace& ws, const double* cells, int S, int count, cudaStream_t stream,
                 const double* rel, const int* nsteps) {
    const wmc::LevelTables& t = L.tab;
    wmc::SmallArgs a{};
    a.n = t.n;
    a.n_r = t.n_r;
    a.p = t.p;
    a.S = S;
    a.count = count;
    a.n_cells = t.n_cells;
    a.split = L.path == SubPath::OnChip ? t.n_r : 0;
    a.row_ptr = L.d_row_ptr;
    a.ent = L.d_ent;
    a.col_bits = L.col_bits;
    a.cell_ix = L.d_cell_ix;
    a.col_mask = static_cast<int>((1u << L.col_bits) - 1u);
    a.a0 = L.d_a0;
    a.row_desc = L.d_row_desc;
    a.wtype = L.d_wtype;
    a.sub_ent = L.d_sub_ent;
    a.slice_off = L.d_slice_off;
    a.n_wid = L.path == SubPath::OnChip ? L.n_wid : 0;
    a.rc_ptr = L.d_rc_ptr;
    a.rc_cell = L.d_rc_cell;
    a.rc_a0 = L.d_rc_a0;
    a.cells = cells;
    a.z0 = L.d_z0;
    a.init_factor = t.init_factor;
    a.factor = t.coarse_factor;
    a.c0 = t.c0;
    a.beta = L.d_beta;
    a.cm = L.d_cm;
    a.n_steps = t.n_steps;
    a.rel = rel;
    a.nsteps = nsteps;
    a.nq = t.nq;
    a.qptr = L.d_qptr;
    a.qdof = L.d_qdof;
    a.qw = L.d_qw;
    a.qsm = L.d_qsm;
    a.q = ws.q;
    a.fail = ws.fail;
    const int e = wmc::launch_small_solve(a, std::min(count, L.n_sms), stream);
    ++g_launches;
    if (e != 0) check(static_cast<cudaError_t>(e), "small solve launch");
}

// Fused lattice solve of a whole batch (one launch; LatSolveArgs).
void fused_solve(wmc_level& L, Workspace& ws, const double* cells, int S, int count, cudaStream_t stream,
                 const double* rel, const int* nsteps) {
    const wmc::LevelTables& t = L.tab;
    wmc::LatSolveArgs a{};
    a.lat = lattice_args(L, ws, cells, S, count);
    a.lat.rel = rel;
    a.lat.nsteps = nsteps;
    a.n = t.n;
    a.row_ptr = L.d_row_ptr;
    a.ent = L.d_ent;
    a.col_bits = L.col_bits;
    a.cell_ix = L.d_cell_ix;
    a.col_mask = static_cast<int>((1u << L.col_bits) - 1u);
    a.a0 = L.d_a0;
    a.row_desc = L.d_row_desc;
    a.wtype = L.d_wtype;
    a.z0 = L.d_z0;
    a.init_factor = t.init_factor;
    a.factor = t.coarse_factor;
    a.n_steps = t.n_steps;
    a.zp_global = L.fused_zp_global ? ws.zb : nullptr;
    a.tmem = L.fused_tmem;
    {
        static const char* e = std::getenv("WMC_FUSED_STAGGER");  // A/B knob (0: off)
        a.stagger = e ? std::atoi(e) : 1;
    }
    a.strips_k_or_k1 = 1;
    for (int len : t.strip_len)
        if (len < t.lat_k - 1) a.strips_k_or_k1 = 0;
    a.ns_rows = L.d_ns_rows;
    a.n_ns = (L.fused_tmem == 2 && t.lat_threads == 512) ? L.n_ns : 0;
    a.rem_ptr = L.d_rem_ptr;
    a.rem_col = L.d_rem_col;
    a.rem_cell = L.d_rem_cell;
    a.rem_a0 = L.d_rem_a0;
    a.nq = t.nq;
    a.qptr = L.d_qptr;
    a.qdof = L.d_qdof;
    a.qw = L.d_qw;
    a.qsm = L.d_qsm;
    a.q = ws.q;
    a.fail = ws.fail;
    if (L.profile) mark(L, L.ev_sub, stream);
    const int e = wmc::launch_lattice_solve(a, std::max(1, std::min(count, L.n_sms)), stream);
    ++g_launches;
    if (e != 0) check(static_cast<cudaError_t>(e), "fused lattice solve launch");
    if (L.profile) mark(L, L.ev_sub, stream);
}

void solve_batch(wmc_level& L, Workspace& ws, const double* cells, int S, int count, cudaStream_t stream) {
    const wmc::LevelTables& t = L.tab;
    if (L.fused_smem > 0) {
        if (t.cfl_safety > 0.0) {
            cfl_phase(L, ws, cells, S, count, stream);
            fused_solve(L, ws, cells, S, count, stream, ws.rel, ws.nsteps);
        } else {
            fused_solve(L, ws, cells, S, count, stream, nullptr, nullptr);
        }
        return;
    }
    if (t.cfl_safety > 0.0) {
        const long n_steps = cfl_phase(L, ws, cells, S, count, stream);
        if (small_path(L, count))
            small_solve(L, ws, cells, S, count, stream, ws.rel, ws.nsteps);
        else
            solve_batch_launches(L, ws, cells, S, count, stream, n_steps, ws.rel, ws.nsteps);
        return;
    }
    if (small_path(L, count) && !L.profile) {
        small_solve(L, ws, cells, S, count, stream, nullptr, nullptr);
        return;
    }
    static const bool no_graph = std::getenv("WMC_NO_GRAPH") != nullptr || std::getenv("WMC_SYNC_DEBUG") != nullptr;
    if (no_graph || L.profile) {
        solve_batch_launches(L, ws, cells, S, count, stream, t.n_steps, nullptr, nullptr);
        return;
    }
    auto& g = L.graphs[std::make_tuple(static_cast<const void*>(&ws), S, count, static_cast<const void*>(cells))];
    if (!g.seen) {  // first use: plain launches (one-time attribute setup, allocations)
        g.seen = true;
        solve_batch_launches(L, ws, cells, S, count, stream, t.n_steps, nullptr, nullptr);
        return;
    }
    if (!g.exec) {
        cudaGraph_t graph = nullptr;
        const long before = g_launches.load();
        check(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "graph capture");
        solve_batch_launches(L, ws, cells, S, count, stream, t.n_steps, nullptr, nullptr);
        check(cudaStreamEndCapture(stream, &graph), "graph capture");
        g.nodes = g_launches.load() - before;
        g_launches -= g.nodes;  // counted when replayed
        const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        check(e, "graph instantiate");
    }
    check(cudaGraphLaunch(g.exec, stream), "graph launch");
    g_launches += g.nodes;
}

void launch_draw(const wmc_level& L, std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S,
                 double* cells, cudaStream_t st) {
    if (L.spec.field == wmc::Field::LognormalKL || L.spec.field == wmc::Field::LognormalKLElem)
        wmc::launch_draw_kl(seed, level, first, count, S, L.tab.n_cells, L.spec.kl_modes, L.d_kl, cells, st);
    else if (L.spec.field == wmc::Field::Kl1D)
        wmc::launch_draw_kl1d(seed, level, first, count, S, L.tab.n_cells, L.tab.field_terms, L.d_field_table, cells,
                              st);
    else if (L.spec.field == wmc::Field::Channel)
        wmc::launch_draw_channel(seed, level, first, count, S, L.ch_args, cells, st);
    else if (L.spec.field == wmc::Field::Jump1D)
        wmc::launch_draw_jump1d(seed, level, first, count, S, L.tab.n_cells, L.spec.jump_h0, L.d_field_x, cells, st);
    else
        wmc::launch_draw_cells(seed, level, first, count, S, L.tab.n_cells, L.spec.coef_lo, L.spec.coef_hi, cells,
                               st);
}

// the 1D experiments' fields are evaluated per element: the coarse level of a
// pair draws its own coefficients from the same stream (rng.cpp:42-89)
bool per_element_field(const wmc_level& L) {
    return L.spec.field == wmc::Field::Kl1D || L.spec.field == wmc::Field::Jump1D ||
           L.spec.field == wmc::Field::Channel || L.spec.field == wmc::Field::LognormalKLElem;
}

void check_pair_compat(const wmc_level* fine, const wmc_level* coarse) {
    if (!fine) throw ConfigError("eval_pairs: fine level is NULL");
    if (coarse && coarse->tab.nq != fine->tab.nq) throw ConfigError("wmc_eval_pairs: QoI sizes differ");
    if (!coarse) return;
    if (fine->device != coarse->device) throw ConfigError("eval_pairs: levels on different devices");
    const auto& a = fine->spec;
    const auto& b = coarse->spec;
    if (a.field != b.field) throw ConfigError("eval_pairs: coefficient fields of the pair differ");
    if (per_element_field(*fine)) {
        // one draw per pair, evaluated on each level's own elements
        if (a.jump_h0 != b.jump_h0 || fine->tab.field_terms != coarse->tab.field_terms ||
            (a.field == wmc::Field::LognormalKLElem &&
             (a.kl_sigma != b.kl_sigma || a.kl_corr_len != b.kl_corr_len || a.kl_modes != b.kl_modes)))
            throw ConfigError("eval_pairs: coefficient fields of the pair differ");
        return;
    }
    if (fine->tab.n_cells != coarse->tab.n_cells || a.coef_lo != b.coef_lo || a.coef_hi != b.coef_hi ||
        a.kl_sigma != b.kl_sigma || a.kl_corr_len != b.kl_corr_len || a.kl_modes != b.kl_modes)
        throw ConfigError("eval_pairs: coefficient fields of the pair differ");
}

// Cost record of `solves` solves of one level, as the reference accumulates
// it per solve (accumulate_cost + stable_dt's power iterations,
// src/experiments.cpp:22-43): StepCounters of run_wave -- LF: n_steps full
// products; LF-LTS: one full (start-up) and per later step one coarse and p
// fine products (src/integrators.cpp:117-157) -- weighted by the reference's
// nnz of A, A P and A (I - P), plus the power iterations weighted by the nnz
// of the operator they apply.
void solve_counts(const wmc::LevelTables& t, wmc_cost& c, long solves, long n_steps, long it_full = 0,
                  long it_coarse = 0) {
    const bool lts = t.kind == wmc::Integrator::LocalTimeStepping;
    const long nnz = t.ref_nnz, nnz_f = t.ref_nnz_fine, nnz_c = t.ref_nnz - t.ref_nnz_fine;
    if (lts && t.tiers > 1) {
        // nested tiers (no reference counterpart): p^k stage products A P_k per step on tier k
        long fine = 0, work = 0, pk = 1;
        for (int k = 0; k < t.tiers; ++k) {
            pk *= t.p;
            fine += pk;
            work += pk * static_cast<long>(t.tier_ent[k].size());
        }
        c.matvec_full += solves;
        c.matvec_coarse += solves * (n_steps - 1);
        c.matvec_fine += solves * (n_steps - 1) * fine;
        c.weighted_work += solves * (nnz + (n_steps - 1) * (nnz_c + work));
    } else if (lts) {
        c.matvec_full += solves;
        c.matvec_coarse += solves * (n_steps - 1);
        c.matvec_fine += solves * (n_steps - 1) * t.p;
        c.weighted_work += solves * (nnz + (n_steps - 1) * (nnz_c + t.p * nnz_f));
    } else {
        c.matvec_full += solves * n_steps;
        c.weighted_work += solves * n_steps * nnz;
    }
    c.weighted_work += solves * (it_full * nnz + it_coarse * nnz_c);
    c.dof_updates += static_cast<double>(solves) * wmc::dof_updates_per_solve(t);
}

void solve_counts(const wmc::LevelTables& t, wmc_cost& c, long solves) { solve_counts(t, c, solves, t.n_steps); }

// Cost of pair i of a per-sample CFL level from the counters issue_pairs
// copied back (fine: fields 0-2, coarse: 3-5 of the fine level's h_cnt).
void pair_cost_sample(const wmc_level* fine, const wmc_level* coarse, std::size_t i, wmc_cost& c) {
    const int* h = fine->h_cnt;
    const std::size_t cap = fine->r_cap;
    solve_counts(fine->tab, c, 1, h[i], h[cap + i], h[2 * cap + i]);
    if (coarse) solve_counts(coarse->tab, c, 1, h[3 * cap + i], h[4 * cap + i], h[5 * cap + i]);
}

// evaluates pairs; host_dq/host_qf may be NULL (device-resident mode: the
// results for index first+i are written to dev_dq/dev_qf + i when given)
void ensure_results(wmc_level& L, std::size_t count) {
    if (count <= L.r_cap) return;
    check(cudaSetDevice(L.device), "cudaSetDevice");
    check(cudaStreamSynchronize(L.stream), "synchronize");
    for (void* p : {(void*)L.r_dq, (void*)L.r_qf, (void*)L.r_ff, (void*)L.r_fc, (void*)L.r_cnt})
        if (p) cudaFree(p);
    for (void* p : {(void*)L.h_dq, (void*)L.h_qf, (void*)L.h_ff, (void*)L.h_fc, (void*)L.h_cnt})
        if (p) cudaFreeHost(p);
    const std::size_t cap = std::max<std::size_t>(count, 256);
    const std::size_t nq = static_cast<std::size_t>(L.tab.nq);
    check(cudaMalloc(&L.r_dq, sizeof(double) * cap * nq), "cudaMalloc results");
    check(cudaMalloc(&L.r_qf, sizeof(double) * cap * nq), "cudaMalloc results");
    check(cudaMalloc(&L.r_ff, sizeof(int) * cap), "cudaMalloc results");
    check(cudaMalloc(&L.r_fc, sizeof(int) * cap), "cudaMalloc results");
    check(cudaMallocHost(&L.h_dq, sizeof(double) * cap * nq), "cudaMallocHost");
    check(cudaMallocHost(&L.h_qf, sizeof(double) * cap * nq), "cudaMallocHost");
    check(cudaMallocHost(&L.h_ff, sizeof(int) * cap), "cudaMallocHost");
    check(cudaMallocHost(&L.h_fc, sizeof(int) * cap), "cudaMallocHost");
    check(cudaMalloc(&L.r_cnt, sizeof(int) * 6 * cap), "cudaMalloc results");
    check(cudaMallocHost(&L.h_cnt, sizeof(int) * 6 * cap), "cudaMallocHost");
    L.r_cap = cap;
}

// Issues the pairs of one index range asynchronously on the fine level's
// stream.  Results land in dev_dq / dev_qf when given (device-resident
// mode), else in the fine level's result buffers, copied to its pinned host
// mirrors together with the fail flags (finish_pairs reads them).
void issue_pairs(wmc_level* fine, wmc_level* coarse, std::uint64_t seed, std::uint32_t level, std::uint64_t first,
                 std::uint64_t count, double* dev_dq, double* dev_qf) {
    check_pair_compat(fine, coarse);
    check(cudaSetDevice(fine->device), "cudaSetDevice");
    const bool to_host = dev_dq == nullptr;
    if (to_host) ensure_results(*fine, count);
    const int cap = coarse ? std::min(fine->batch, coarse->batch) : fine->batch;
    cudaStream_t st = fine->stream;
    for (std::uint64_t off = 0; off < count; off += cap) {
        const int c = static_cast<int>(std::min<std::uint64_t>(cap, count - off));
        const int S = round64(c);
        launch_draw(*fine, seed, level, first + off, c, S, fine->d_cells, st);
        g_launches += 2;  // draw + pair difference
        Workspace& wf = workspace(*fine, 0);
        solve_batch(*fine, wf, fine->d_cells, S, c, st);
        Workspace* wc = nullptr;
        if (coarse) {
            wc = &workspace(*coarse, 1);
            const double* coarse_cells = fine->d_cells;
            if (per_element_field(*fine)) {
                // the coarse role has its own buffer: the level may run its own
                // pair concurrently on its stream
                if (!coarse->d_cells_coarse)
                    check(cudaMalloc(&coarse->d_cells_coarse,
                                     sizeof(double) * static_cast<std::size_t>(coarse->batch) * coarse->tab.n_cells),
                          "cudaMalloc cells");
                launch_draw(*coarse, seed, level, first + off, c, S, coarse->d_cells_coarse, st);
                ++g_launches;
                coarse_cells = coarse->d_cells_coarse;
            }
            solve_batch(*coarse, *wc, coarse_cells, S, c, st);
        }
        const int nq = fine->tab.nq;
        double* dq_dst = (to_host ? fine->r_dq : dev_dq) + off * nq;
        double* qf_dst = to_host ? fine->r_qf + off * nq : (dev_qf ? dev_qf + off * nq : nullptr);
        wmc::launch_pair_diff(wf.q, wc ? wc->q : nullptr, dq_dst, qf_dst, c, S, nq, st);
        if (to_host && fine->tab.cfl_safety > 0.0) {
            const std::size_t cap_r = fine->r_cap;
            const int* src[6] = {wf.nsteps, wf.it_full, wf.it_coarse, wc ? wc->nsteps : nullptr,
                                 wc ? wc->it_full : nullptr, wc ? wc->it_coarse : nullptr};
            for (int f = 0; f < 6; ++f)
                if (src[f])
                    check(cudaMemcpyAsync(fine->r_cnt + f * cap_r + off, src[f], sizeof(int) * c,
                                          cudaMemcpyDeviceToDevice, st), "counters");
        }
        if (!to_host) {  // device-resident: fold the batch's failures into the level's record
            if (!fine->d_fail_rec) {
                check(cudaMalloc(&fine->d_fail_rec, 2 * sizeof(unsigned long long)), "cudaMalloc fail record");
                check(cudaMemsetAsync(fine->d_fail_rec, 0xff, 2 * sizeof(unsigned long long), st), "fail record");
            }
            fine->fail_level = static_cast<int>(level);
            wmc::launch_fail_fold(wf.fail, wc ? wc->fail : nullptr, c, first + off, fine->d_fail_rec, st);
            ++g_launches;
        }
        if (to_host) {
            check(cudaMemcpyAsync(fine->r_ff + off, wf.fail, sizeof(int) * c, cudaMemcpyDeviceToDevice, st), "fail");
            if (wc)
                check(cudaMemcpyAsync(fine->r_fc + off, wc->fail, sizeof(int) * c, cudaMemcpyDeviceToDevice, st),
                      "fail");
        }
    }
    if (to_host) {
        const std::size_t nq = static_cast<std::size_t>(fine->tab.nq);
        check(cudaMemcpyAsync(fine->h_dq, fine->r_dq, sizeof(double) * count * nq, cudaMemcpyDeviceToHost, st), "dq");
        check(cudaMemcpyAsync(fine->h_qf, fine->r_qf, sizeof(double) * count * nq, cudaMemcpyDeviceToHost, st), "q");
        check(cudaMemcpyAsync(fine->h_ff, fine->r_ff, sizeof(int) * count, cudaMemcpyDeviceToHost, st), "fail");
        if (fine->tab.cfl_safety > 0.0)
            for (int f = 0; f < (coarse ? 6 : 3); ++f)
                check(cudaMemcpyAsync(fine->h_cnt + f * fine->r_cap, fine->r_cnt + f * fine->r_cap,
                                      sizeof(int) * count, cudaMemcpyDeviceToHost, st), "counters");
        if (coarse)
            check(cudaMemcpyAsync(fine->h_fc, fine->r_fc, sizeof(int) * count, cudaMemcpyDeviceToHost, st), "fail");
    }
}

// Waits for issue_pairs' host results and reports the first failing sample
// (lowest index) like sample_delta_q's wrapped error (src/mlmc.cpp:31-35).
void finish_pairs(wmc_level* fine, bool has_coarse, std::uint32_t level, std::uint64_t first, std::uint64_t count,
                  wmc_error* err) {
    check(cudaSetDevice(fine->device), "cudaSetDevice");
    check(cudaStreamSynchronize(fine->stream), "synchronize");
    if (err) {
        err->sample = -1;
        err->step = 0;
        err->level = static_cast<int>(level);
    }
    for (std::uint64_t i = 0; i < count; ++i) {
        const bool bad_f = fine->h_ff[i] != INT_MAX, bad_c = has_coarse && fine->h_fc[i] != INT_MAX;
        if (bad_f || bad_c) {
            if (err) {
                err->sample = static_cast<long>(first + i);
                err->step = bad_f ? fine->h_ff[i] : fine->h_fc[i];
                err->level = bad_f ? static_cast<int>(level) : static_cast<int>(level) - 1;
            }
            g_last_error = "level " + std::to_string(level) + ", sample " + std::to_string(first + i) +
                           ": time integration unstable";
            throw NumericalError(g_last_error);
        }
    }
}

void pair_cost(const wmc_level* fine, const wmc_level* coarse, std::uint64_t count, wmc_cost* cost) {
    std::memset(cost, 0, sizeof(*cost));
    solve_counts(fine->tab, *cost, static_cast<long>(count));
    if (coarse) solve_counts(coarse->tab, *cost, static_cast<long>(count));
}

// Cost of pairs [from, from + count) of the fine level's host results: per
// sample (its own step count and power iterations) on per-sample CFL levels,
// else the fixed-horizon counts.
void results_cost(const wmc_level* fine, const wmc_level* coarse, std::size_t from, std::size_t count, wmc_cost* cost) {
    if (fine->tab.cfl_safety <= 0.0 || !fine->h_cnt) {
        pair_cost(fine, coarse, count, cost);
        return;
    }
    std::memset(cost, 0, sizeof(*cost));
    for (std::size_t i = from; i < from + count; ++i) pair_cost_sample(fine, coarse, i, *cost);
}

// evaluates pairs; host_dq/host_qf may be NULL (device-resident mode: the
// results for index first+i are written to dev_dq/dev_qf + i when given)
void eval_pairs_impl(wmc_level* fine, wmc_level* coarse, std::uint64_t seed, std::uint32_t level, std::uint64_t first,
                     std::uint64_t count, double* host_dq, double* host_qf, double* dev_dq, double* dev_qf,
                     wmc_cost* cost, wmc_error* err) {
    if (dev_dq) {
        issue_pairs(fine, coarse, seed, level, first, count, dev_dq, dev_qf);
    } else {
        issue_pairs(fine, coarse, seed, level, first, count, nullptr, nullptr);
        finish_pairs(fine, coarse != nullptr, level, first, count, err);
        const std::size_t nq = static_cast<std::size_t>(fine->tab.nq);
        if (host_dq) std::memcpy(host_dq, fine->h_dq, sizeof(double) * count * nq);
        if (host_qf) std::memcpy(host_qf, fine->h_qf, sizeof(double) * count * nq);
        if (cost) results_cost(fine, coarse, 0, count, cost);
        return;
    }
    if (cost) pair_cost(fine, coarse, count, cost);
}

// LevelAccumulator (reference src/mlmc.cpp:39-73) on QoI vectors of nq
// outputs with the norm weights w (QoIVector::norm, fem.cpp:15-19: sqrt of
// sum_k w_k v_k^2); the BASELINE scalar QoI is nq = 1, w = 1.
struct Acc {
    long n = 0;
    std::vector<double> s_dq, s_q, w;
    double s_dq2 = 0.0, s_q2 = 0.0;
    wmc_cost cost{};
    void init(const std::vector<double>& weights) {
        if (!w.empty()) return;
        w = weights;
        s_dq.assign(w.size(), 0.0);
        s_q.assign(w.size(), 0.0);
    }
    double norm(const double* v) const {
        double acc = 0.0;
        for (std::size_t k = 0; k < w.size(); ++k) acc += w[k] * v[k] * v[k];
        return std::sqrt(acc);
    }
    void add(const double* dq, const double* q) {
        ++n;
        const double a = norm(dq), b = norm(q);
        s_dq2 += a * a;
        s_q2 += b * b;
        for (std::size_t k = 0; k < w.size(); ++k) {
            s_dq[k] += dq[k];
            s_q[k] += q[k];
        }
    }
    // estimate_variance / estimate_mc_variance (src/mlmc.cpp:61-73)
    double variance() const {
        if (n < 2) throw NumericalError("estimate_variance: need at least two samples");
        const double nn = static_cast<double>(n), sn = norm(s_dq.data());
        return std::max(0.0, (s_dq2 - sn * sn / nn) / (nn - 1.0));
    }
    double mc_variance() const {
        if (n < 2) throw NumericalError("estimate_mc_variance: need at least two samples");
        const double nn = static_cast<double>(n), sn = norm(s_q.data());
        return std::max(0.0, (s_q2 - sn * sn / nn) / nn);
    }
    std::vector<double> mean_dq() const {
        std::vector<double> m(s_dq);
        const double f = n > 0 ? 1.0 / static_cast<double>(n) : 0.0;
        for (double& x : m) x *= f;
        return m;
    }
    double mean_dq_norm() const { return w.empty() ? 0.0 : norm(mean_dq().data()); }
};

void fill_stats(int level, const Acc& a, double model_cost, wmc_level_stats& s) {
    s.level = level;
    s.n_samples = a.n;
    // scalar QoI: the sums themselves; QoI vectors: their norms
    s.sum_dq = a.w.size() == 1 ? a.s_dq[0] : (a.w.empty() ? 0.0 : a.norm(a.s_dq.data()));
    s.sum_dq2 = a.s_dq2;
    s.sum_q = a.w.size() == 1 ? a.s_q[0] : (a.w.empty() ? 0.0 : a.norm(a.s_q.data()));
    s.sum_q2 = a.s_q2;
    s.variance = a.n >= 2 ? a.variance() : 0.0;
    s.mc_variance = a.n >= 2 ? a.mc_variance() : 0.0;
    s.mean_dq = a.w.size() == 1 ? a.mean_dq()[0] : a.mean_dq_norm();
    s.model_cost = model_cost;
    s.cost = a.cost;
}

// Runs the index ranges of several levels concurrently (each pair on its fine
// level's stream; a level's workspaces per role keep neighbouring pairs
// apart), then folds every level's results in index order
// (src/mlmc.cpp:145-147).
struct LevelJob {
    int level;
    long first, count;
};

void run_levels(wmc_level** levels, const std::vector<LevelJob>& jobs, std::uint64_t seed, std::vector<Acc>& acc,
                wmc_error* err) {
    for (const auto& j : jobs)
        if (j.count > 0) ensure_results(*levels[j.level], static_cast<std::size_t>(j.count));
    for (const auto& j : jobs)
        if (j.count > 0)
            issue_pairs(levels[j.level], j.level > 0 ? levels[j.level - 1] : nullptr, seed,
                        static_cast<std::uint32_t>(j.level), static_cast<std::uint64_t>(j.first),
                        static_cast<std::uint64_t>(j.count), nullptr, nullptr);
    for (const auto& j : jobs) {
        if (j.count <= 0) continue;
        wmc_level* fine = levels[j.level];
        finish_pairs(fine, j.level > 0, static_cast<std::uint32_t>(j.level), static_cast<std::uint64_t>(j.first),
                     static_cast<std::uint64_t>(j.count), err);
        Acc& a = acc[j.level];
        a.init(fine->tab.qoi_norm_w);
        const int nq = fine->tab.nq;
        for (long i = 0; i < j.count; ++i) a.add(fine->h_dq + i * nq, fine->h_qf + i * nq);
        wmc_cost c{};
        results_cost(fine, j.level > 0 ? levels[j.level - 1] : nullptr, 0, static_cast<std::size_t>(j.count), &c);
        a.cost.matvec_full += c.matvec_full;
        a.cost.matvec_fine += c.matvec_fine;
        a.cost.matvec_coarse += c.matvec_coarse;
        a.cost.weighted_work += c.weighted_work;
        a.cost.dof_updates += c.dof_updates;
    }
}

// Per-level cache of evaluated pairs for the adaptive driver: results for
// indices [0, computed) in index order.  A sample's (dQ, Q) depends only on
// (seed, level, index) -- bitwise, whatever the batch it ran in -- so the
// driver may evaluate ahead of its targets (batches are padded to 64 lanes
// anyway, and the next level's warm-up can run beside the current wave) and
// fold exactly the samples the reference's run_mlmc would (src/mlmc.cpp:165-233).
struct PairCache {
    std::vector<double> dq, qf;
    std::vector<int> ff, fc;  // fail steps (INT_MAX: fine)
    std::vector<wmc_cost> cost;  // per pair (reference CostRecord of sample_delta_q)
    long computed = 0;
};

// Evaluates index ranges of several levels into the per-level caches (results
// appended in index order).  With n_dev device groups (levels[d * n_levels +
// l] is level l on group d) every range is split into contiguous 64-sample
// granules per group and each group runs on its own host thread (issue,
// synchronise, copy out); the ranges of one group run concurrently on their
// level streams.  A sample's results depend only on (seed, level, index), so
// the caches -- and every fold of them -- are independent of n_dev, bitwise.
struct Issue {
    int level;
    long first, count;
};

void eval_into_cache(wmc_level** levels, int n_dev, int n_levels, const std::vector<Issue>& issues,
                     std::uint64_t seed, std::vector<PairCache>& cache) {
    struct Part {
        int level;
        long first, count;
        PairCache out;
    };
    // parts[d]: device group d's sub-ranges, in issue order
    std::vector<std::vector<Part>> parts(n_dev);
    for (const auto& j : issues) {
        const long granules = (j.count + 63) / 64;
        for (int d = 0; d < n_dev; ++d) {
            const long g0 = granules * d / n_dev, g1 = granules * (d + 1) / n_dev;
            const long f = j.first + 64 * g0, c = std::min(j.first + j.count, j.first + 64 * g1) - f;
            if (c > 0) parts[d].push_back({j.level, f, c, {}});
        }
    }
    auto run_group = [&](int d) {
        wmc_level** lv = levels + static_cast<std::size_t>(d) * n_levels;
        for (auto& pt : parts[d]) {
            ensure_results(*lv[pt.level], static_cast<std::size_t>(pt.count));
            issue_pairs(lv[pt.level], pt.level > 0 ? lv[pt.level - 1] : nullptr, seed,
                        static_cast<std::uint32_t>(pt.level), static_cast<std::uint64_t>(pt.first),
                        static_cast<std::uint64_t>(pt.count), nullptr, nullptr);
        }
        for (auto& pt : parts[d]) {
            wmc_level* fine = lv[pt.level];
            check(cudaSetDevice(fine->device), "cudaSetDevice");
            check(cudaStreamSynchronize(fine->stream), "synchronize");
            PairCache& c = pt.out;
            const long nq = fine->tab.nq;
            c.dq.assign(fine->h_dq, fine->h_dq + pt.count * nq);
            c.qf.assign(fine->h_qf, fine->h_qf + pt.count * nq);
            c.ff.assign(fine->h_ff, fine->h_ff + pt.count);
            if (pt.level > 0)
                c.fc.assign(fine->h_fc, fine->h_fc + pt.count);
            else
                c.fc.assign(pt.count, INT_MAX);
            for (long i = 0; i < pt.count; ++i) {
                wmc_cost pc{};
                results_cost(fine, pt.level > 0 ? lv[pt.level - 1] : nullptr, static_cast<std::size_t>(i), 1, &pc);
                c.cost.push_back(pc);
            }
        }
    };
    if (n_dev == 1) {
        run_group(0);
    } else {
        std::vector<std::thread> threads;
        std::vector<std::exception_ptr> errs(n_dev);
        for (int d = 0; d < n_dev; ++d)
            threads.emplace_back([&, d] {
                try {
                    run_group(d);
                } catch (...) {
                    errs[d] = std::current_exception();
                }
            });
        for (auto& t : threads) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    }
    // append in index order: issue order, device-group order within an issue
    for (std::size_t k = 0; k < issues.size(); ++k)
        for (int d = 0; d < n_dev; ++d)
            for (auto& pt : parts[d]) {
                if (pt.level != issues[k].level || pt.first < issues[k].first ||
                    pt.first >= issues[k].first + issues[k].count)
                    continue;
                PairCache& c = cache[pt.level];
                if (pt.first != c.computed) throw DeviceError("eval_into_cache: results out of order");
                c.dq.insert(c.dq.end(), pt.out.dq.begin(), pt.out.dq.end());
                c.qf.insert(c.qf.end(), pt.out.qf.begin(), pt.out.qf.end());
                c.ff.insert(c.ff.end(), pt.out.ff.begin(), pt.out.ff.end());
                c.fc.insert(c.fc.end(), pt.out.fc.begin(), pt.out.fc.end());
                c.cost.insert(c.cost.end(), pt.out.cost.begin(), pt.out.cost.end());
                c.computed += pt.count;
            }
}

// One wave: evaluate, on every level that needs more than its cache holds,
// the missing indices rounded up to the 64-lane batch granule (plus `spec`:
// the first 64 pairs of a level not yet in use), levels concurrently on their
// streams (device groups on their host threads); then fold into acc up to
// the targets in (level, index) order.
void cached_wave(wmc_level** levels, int n_dev, int n_levels, const std::vector<long>& targets, int spec,
                 std::uint64_t seed, std::vector<Acc>& acc, std::vector<PairCache>& cache, wmc_error* err) {
    std::vector<Issue> issues;
    for (int l = 0; l < static_cast<int>(targets.size()); ++l)
        if (targets[l] > cache[l].computed) {
            const long need = targets[l] - cache[l].computed;
            issues.push_back({l, cache[l].computed, (need + 63) / 64 * 64});
        }
    if (spec >= 0 && spec < n_levels && cache[spec].computed == 0) issues.push_back({spec, 0, 64});
    eval_into_cache(levels, n_dev, n_levels, issues, seed, cache);
    if (err) err->sample = -1;
    for (int l = 0; l < static_cast<int>(targets.size()); ++l) {
        Acc& a = acc[l];
        a.init(levels[l]->tab.qoi_norm_w);
        const PairCache& c = cache[l];
        const long nq = levels[l]->tab.nq;
        const long from = a.n;
        for (long i = from; i < targets[l]; ++i) {
            const bool bad_f = c.ff[i] != INT_MAX, bad_c = c.fc[i] != INT_MAX;
            if (bad_f || bad_c) {
                if (err) {
                    err->sample = i;
                    err->step = bad_f ? c.ff[i] : c.fc[i];
                    err->level = bad_f ? l : l - 1;
                }
                g_last_error = "level " + std::to_string(l) + ", sample " + std::to_string(i) +
                               ": time integration unstable";
                throw NumericalError(g_last_error);
            }
            a.add(c.dq.data() + i * nq, c.qf.data() + i * nq);
        }
        if (targets[l] > from) {
            wmc_cost cc{};
            for (long i = from; i < targets[l]; ++i) {
                const wmc_cost& pc = c.cost[i];
                cc.matvec_full += pc.matvec_full;
                cc.matvec_fine += pc.matvec_fine;
                cc.matvec_coarse += pc.matvec_coarse;
                cc.weighted_work += pc.weighted_work;
                cc.dof_updates += pc.dof_updates;
            }
            a.cost.matvec_full += cc.matvec_full;
            a.cost.matvec_fine += cc.matvec_fine;
            a.cost.matvec_coarse += cc.matvec_coarse;
            a.cost.weighted_work += cc.weighted_work;
            a.cost.dof_updates += cc.dof_updates;
        }
    }
}

}  // namespace

namespace {
// reference optimal_samples (src/mlmc.cpp:75-92):
// N_l = max(min, ceil((2/eps^2) sqrt(V_l/C_l) sum sqrt(V C) - 1e-9))
std::vector<long> optimal_samples_impl(const double* v, const double* c, int n, double eps, long min_samples) {
    double total = 0.0;
    for (int l = 0; l < n; ++l) {
        if (!(c[l] > 0.0)) throw ConfigError("optimal_samples: costs must be positive");
        if (v[l] < 0.0) throw ConfigError("optimal_samples: negative variance");
        total += std::sqrt(v[l] * c[l]);
    }
    std::vector<long> out(n);
    for (int l = 0; l < n; ++l) {
        const double nl = 2.0 / (eps * eps) * std::sqrt(v[l] / c[l]) * total;
        out[l] = std::max(min_samples, static_cast<long>(std::ceil(nl - 1e-9)));
    }
    return out;
}

// reference bias_proxy_sq (src/mlmc.cpp:94-98) on the scalar QoI
double bias_proxy_norm(double mean_dq_norm, double alpha) {
    const double denom = std::pow(2.0, alpha) - 1.0;
    const double norm = mean_dq_norm / denom;
    return norm * norm;
}
double bias_proxy_impl(double mean_dq, double alpha) { return bias_proxy_norm(std::sqrt(mean_dq * mean_dq), alpha); }

// batch capacity: the requested one (rounded to 64) or automatic: at most
// 4096 samples, both workspaces of the level within 15 % of device memory
void set_batch(wmc_level& L, int requested) {
    if (requested > 0) {
        L.batch = round64(requested);
        return;
    }
    check(cudaSetDevice(L.device), "cudaSetDevice");
    std::size_t free_b = 0, total_b = 0;
    check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    const auto& t = L.tab;
    double tier_rows = 0.0;
    if (t.tiers > 1)
        for (int k = 0; k < t.tiers; ++k) tier_rows += (k > 0 ? 3.0 : 2.0) * t.n_r_tier[k];
    const double per_sample =
        2.0 * 8.0 * (2.0 * t.n + g_stride(t) + t.n_cells + 4.0 * t.nq + 2.0 * t.n_r + tier_rows);
    const long cap = static_cast<long>(0.15 * static_cast<double>(total_b) / per_sample) / 64 * 64;
    L.batch = static_cast<int>(std::max(64L, std::min(4096L, cap)));
}

// one level of the reference's 1D experiments: hierarchy, spec and tables
// (make_problem / build_state_1d, src/experiments.cpp:56-106)
void experiment_tables(const wmc::Mesh1D& mesh, int substeps, const wmc_experiment_desc* desc, wmc::LevelSpec& s,
                       wmc::LevelTables& t) {
    if (desc->experiment != WMC_EXP_SMOOTH1D && desc->experiment != WMC_EXP_JUMP1D)
        throw ConfigError("experiment: unknown experiment");
    if (substeps < 1) throw ConfigError("experiment: substeps >= 1");
    if (desc->integrator != WMC_LEAPFROG && desc->integrator != WMC_LOCAL_TIME_STEPPING)
        throw ConfigError("experiment: unknown integrator");
    if (!(desc->safety > 0.0 && desc->safety <= 1.0)) throw ConfigError("experiment: safety in (0, 1]");
    if (desc->nu < 0.0 || desc->nu > 1.0) throw ConfigError("experiment: nu in [0, 1]");
    const bool jump = desc->experiment == WMC_EXP_JUMP1D;
    s = wmc::LevelSpec{};
    s.kind = desc->integrator == WMC_LEAPFROG ? wmc::Integrator::Leapfrog : wmc::Integrator::LocalTimeStepping;
    s.substeps = s.kind == wmc::Integrator::Leapfrog ? 1 : substeps;
    s.nu = desc->nu;
    s.final_time = desc->final_time;
    s.dt = mesh.coarse_h;  // nominal: every sample takes its own CFL step
    s.cfl_safety = desc->safety;
    s.field = jump ? wmc::Field::Jump1D : wmc::Field::Kl1D;
    s.jump_h0 = desc->h0;
    s.ic.x0 = 3.0;  // experiments.cpp:64: u0 = exp(-(x - 3)^2 / 0.09)
    s.ic.y0 = 0.0;
    s.ic.width2 = 0.09;
    s.grid_lo = 0.0;
    s.grid_hi = 6.0;  // kDomain1dLength
    s.grid_n = desc->grid_n;
    s.cells_x = mesh.n_elements();
    s.cells_y = 1;
    t = wmc::build_level_tables_1d(mesh, s);
}

// One level of the reference's narrow-channel experiment on the reference
// mesh of that level (make_problem Channel2d / build_state_2d,
// src/experiments.cpp:132-148): p = ceil(h0 2^-l / fine_h) (LF-LTS) or 1,
// per-sample CFL step, QoI on grid_n points of [-1/2, 1/2].
void channel_level_tables(const wmc::TriMesh& mesh, const wmc_experiment_desc* desc, int level, wmc::LevelSpec& s,
                          wmc::LevelTables& t, wmc::ChannelTables& ch) {
    if (desc->experiment != WMC_EXP_CHANNEL2D) throw ConfigError("channel: experiment must be WMC_EXP_CHANNEL2D");
    if (desc->integrator != WMC_LEAPFROG && desc->integrator != WMC_LOCAL_TIME_STEPPING)
        throw ConfigError("channel: unknown integrator");
    if (!(desc->safety > 0.0 && desc->safety <= 1.0)) throw ConfigError("channel: safety in (0, 1]");
    if (desc->nu < 0.0 || desc->nu > 1.0) throw ConfigError("channel: nu in [0, 1]");
    if (!(desc->h0 > 0.0) || !(desc->fine_h > 0.0)) throw ConfigError("channel: h0 and fine_h must be positive");
    if (level < 0 || level > desc->max_level) throw ConfigError("channel: level out of range");
    const double coarse = desc->h0 / std::pow(2.0, level);
    s = wmc::LevelSpec{};
    s.kind = desc->integrator == WMC_LEAPFROG ? wmc::Integrator::Leapfrog : wmc::Integrator::LocalTimeStepping;
    s.substeps = s.kind == wmc::Integrator::Leapfrog
                     ? 1
                     : std::max(1, static_cast<int>(std::ceil(coarse / desc->fine_h - 1e-9)));
    s.nu = desc->nu;
    s.final_time = desc->final_time;
    s.dt = coarse;  // nominal: every sample takes its own CFL step
    s.cfl_safety = desc->safety;
    s.field = wmc::Field::Channel;
    s.grid_lo = -wmc::kChannelRectHalfHeight;
    s.grid_hi = wmc::kChannelRectHalfHeight;
    s.grid_n = desc->grid_n;
    try {
        t = wmc::build_level_tables_channel(mesh, s, ch);
    } catch (const std::invalid_argument& e) {
        throw ConfigError(e.what());
    }
    s.cells_x = t.n_cells;
    s.cells_y = 1;
}

wmc::LevelSpec spec_from_desc(const wmc_level_desc* desc) {
    if (desc->integrator != WMC_LEAPFROG && desc->integrator != WMC_LOCAL_TIME_STEPPING)
        throw ConfigError("wmc_level_create: unknown integrator");
    if (!(desc->coef_lo > 0.0) || !(desc->coef_hi >= desc->coef_lo))
        throw ConfigError("wmc_level_create: coefficient range must be positive");
    if (desc->nu < 0.0 || desc->nu > 1.0) throw ConfigError("wmc_level_create: nu in [0,1]");
    wmc::LevelSpec s;
    s.cells_x = desc->cells_x;
    s.cells_y = desc->cells_y;
    s.coef_lo = desc->coef_lo;
    s.coef_hi = desc->coef_hi;
    s.final_time = desc->final_time;
    s.dt = desc->dt;
    s.substeps = desc->substeps;
    s.nu = desc->nu;
    s.kind = desc->integrator == WMC_LEAPFROG ? wmc::Integrator::Leapfrog : wmc::Integrator::LocalTimeStepping;
    s.ic.x0 = desc->ic_x;
    s.ic.y0 = desc->ic_y;
    s.ic.width2 = desc->ic_width2;
    s.qoi.x0 = desc->qoi_box[0];
    s.qoi.x1 = desc->qoi_box[1];
    s.qoi.y0 = desc->qoi_box[2];
    s.qoi.y1 = desc->qoi_box[3];
    if (desc->field != WMC_FIELD_UNIFORM && desc->field != WMC_FIELD_LOGNORMAL_KL &&
        desc->field != WMC_FIELD_LOGNORMAL_KL_ELEMENT)
        throw ConfigError("wmc_level_create: unknown coefficient field");
    s.field = desc->field == WMC_FIELD_LOGNORMAL_KL           ? wmc::Field::LognormalKL
              : desc->field == WMC_FIELD_LOGNORMAL_KL_ELEMENT ? wmc::Field::LognormalKLElem
                                                              : wmc::Field::Uniform;
    s.kl_sigma = desc->kl_sigma;
    s.kl_corr_len = desc->kl_corr_len;
    s.kl_modes = desc->kl_modes;
    s.tiers = desc->tiers > 1 ? desc->tiers : 1;
    if (desc->tiers < 0 || desc->tiers > wmc::kMaxTiers) throw ConfigError("wmc_level_create: tiers in [0, 8]");
    if (desc->domain[0] != 0.0 || desc->domain[1] != 0.0 || desc->domain[2] != 0.0 || desc->domain[3] != 0.0) {
        if (!(desc->domain[1] > desc->domain[0]) || !(desc->domain[3] > desc->domain[2]))
            throw ConfigError("wmc_level_create: empty coefficient domain");
        s.dom_x0 = desc->domain[0];
        s.dom_x1 = desc->domain[1];
        s.dom_y0 = desc->domain[2];
        s.dom_y1 = desc->domain[3];
    }
    s.qoi_mean = desc->qoi_mean != 0;
    if (desc->cfl_safety < 0.0 || desc->cfl_safety > 1.0) throw ConfigError("wmc_level_create: cfl_safety in [0, 1]");
    s.cfl_safety = desc->cfl_safety;
    if ((s.field == wmc::Field::LognormalKL || s.field == wmc::Field::LognormalKLElem) &&
        (s.kl_modes < 1 || s.kl_modes > wmc::kMaxKLModes || !(s.kl_corr_len > 0.0) || !(s.kl_sigma >= 0.0)))
        throw ConfigError("wmc_level_create: KL field needs 1..64 modes, corr_len > 0, sigma >= 0");
    return s;
}

void fill_info(const wmc::LevelTables& t, int batch, bool lattice, wmc_level_info* info, int path = -1) {
    info->lattice = lattice ? 1 : 0;
    info->substep_path = path;
    info->n = t.n;
    info->n_r = t.n_r;
    info->n_p = t.n_p;
    info->p = t.p;
    info->n_steps = t.n_steps;
    info->dt = t.dt;
    info->nnz = static_cast<long>(t.col.size());
    info->ap_nnz = static_cast<long>(t.ap_col.size());
    info->n_recipes = static_cast<long>(t.rc_ptr.size()) - 1;
    info->batch = batch;
    info->dof_updates_per_solve = wmc::dof_updates_per_solve(t);
    info->tiers = t.tiers;
    info->n_structured = 0;
    info->fused = 0;
    info->nq = t.nq;
    for (int k = 0; k < 8; ++k) info->n_r_tier[k] = k < static_cast<int>(t.n_r_tier.size()) ? t.n_r_tier[k] : 0;
}
}  // namespace

extern "C" {

const char* wmc_last_error(void) { return g_last_error.c_str(); }

int wmc_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int wmc_mesh_build_square(const wmc_square_mesh_spec* spec, wmc_mesh** out) {
    return guarded([&] {
        if (!spec || !out) throw ConfigError("wmc_mesh_build_square: NULL argument");
        wmc::SquareMeshSpec s;
        s.n_coarse = spec->n_coarse;
        s.ratio = spec->ratio;
        s.fine_lo = spec->fine_lo;
        s.fine_hi = spec->fine_hi;
        s.snap = spec->snap;
        s.small_factor = spec->small_factor;
        auto m = std::make_unique<wmc_mesh>();
        m->mesh = wmc::build_refined_square(s);
        *out = m.release();
    });
}

int wmc_mesh_build_lshape(const wmc_lshape_mesh_spec* spec, wmc_mesh** out) {
    return guarded([&] {
        if (!spec || !out) throw ConfigError("wmc_mesh_build_lshape: NULL argument");
        wmc::LShapeMeshSpec s;
        s.n_per_unit = spec->n_per_unit;
        s.tiers = spec->tiers;
        s.grade_radius = spec->grade_radius;
        auto m = std::make_unique<wmc_mesh>();
        m->mesh = wmc::build_graded_lshape(s);
        *out = m.release();
    });
}

int wmc_mesh_create(int n_vertices, int n_triangles, const double* xy, const int* tri, const unsigned char* fine,
                    const unsigned char* boundary, double coarse_h, double fine_h, wmc_mesh** out) {
    return guarded([&] {
        if (n_vertices <= 0 || n_triangles <= 0 || !xy || !tri || !out) throw ConfigError("wmc_mesh_create: bad arguments");
        auto m = std::make_unique<wmc_mesh>();
        auto& M = m->mesh;
        M.coarse_h = coarse_h;
        M.fine_h = fine_h;
        M.vertices.resize(n_vertices);
        M.boundary_vertex.assign(n_vertices, 0);
        for (int v = 0; v < n_vertices; ++v) {
            M.vertices[v] = {xy[2 * v], xy[2 * v + 1]};
            if (boundary) M.boundary_vertex[v] = boundary[v] ? 1 : 0;
        }
        M.triangles.resize(n_triangles);
        M.fine_flags.assign(n_triangles, 0);
        for (int t = 0; t < n_triangles; ++t) {
            for (int k = 0; k < 3; ++k) {
                const int v = tri[3 * t + k];
                if (v < 0 || v >= n_vertices) throw ConfigError("wmc_mesh_create: vertex index out of range");
                M.triangles[t][k] = v;
            }
            if (fine) M.fine_flags[t] = fine[t];  // tier value (0 coarse, k >= 1: in P_1..P_k)
        }
        *out = m.release();
    });
}

int wmc_mesh_info(const wmc_mesh* mesh, int* nv, int* nt, double* coarse_h, double* fine_h) {
    return guarded([&] {
        if (!mesh) throw ConfigError("wmc_mesh_info: NULL mesh");
        if (nv) *nv = mesh->mesh.n_vertices();
        if (nt) *nt = mesh->mesh.n_triangles();
        if (coarse_h) *coarse_h = mesh->mesh.coarse_h;
        if (fine_h) *fine_h = mesh->mesh.fine_h;
    });
}

int wmc_mesh_export(const wmc_mesh* mesh, double* xy, int* tri, unsigned char* fine, unsigned char* boundary) {
    return guarded([&] {
        if (!mesh) throw ConfigError("wmc_mesh_export: NULL mesh");
        const auto& M = mesh->mesh;
        for (int v = 0; v < M.n_vertices(); ++v) {
            if (xy) {
                xy[2 * v] = M.vertices[v][0];
                xy[2 * v + 1] = M.vertices[v][1];
            }
            if (boundary) boundary[v] = M.boundary_vertex[v];
        }
        for (int t = 0; t < M.n_triangles(); ++t) {
            if (tri)
                for (int k = 0; k < 3; ++k) tri[3 * t + k] = M.triangles[t][k];
            if (fine) fine[t] = M.fine_flags[t];
        }
    });
}

int wmc_mesh_dump(const wmc_mesh* mesh, const char* path) {
    return guarded([&] {
        if (!mesh || !path) throw ConfigError("wmc_mesh_dump: NULL argument");
        wmc::dump_mesh_text(mesh->mesh, path);
    });
}

void wmc_mesh_destroy(wmc_mesh* mesh) { delete mesh; }

void wmc_level_desc_default(wmc_level_desc* d) {
    if (!d) return;
    std::memset(d, 0, sizeof(*d));
    d->cells_x = 4;
    d->cells_y = 4;
    d->coef_lo = 0.5;
    d->coef_hi = 1.5;
    d->final_time = 1.0;
    d->dt = 0.2 / 32.0;
    d->substeps = 4;
    d->nu = 0.01;
    d->integrator = WMC_LOCAL_TIME_STEPPING;
    d->ic_x = 0.3;
    d->ic_y = 0.5;
    d->ic_width2 = 0.01;
    d->qoi_box[0] = 0.7;
    d->qoi_box[1] = 0.9;
    d->qoi_box[2] = 0.4;
    d->qoi_box[3] = 0.6;
    d->device = 0;
    d->batch = 0;
    d->field = WMC_FIELD_UNIFORM;
    d->kl_sigma = 0.5;
    d->kl_corr_len = 0.1;
    d->kl_modes = 64;
}

int wmc_level_create(const wmc_mesh* mesh, const wmc_level_desc* desc, wmc_level** out) {
    return guarded([&] {
        if (!mesh || !desc || !out) throw ConfigError("wmc_level_create: NULL argument");
        auto L = std::make_unique<wmc_level>();
        L->device = desc->device;
        L->spec = spec_from_desc(desc);
        L->tab = wmc::build_level_tables(mesh->mesh, L->spec);
        if (L->tab.n_steps >= INT_MAX) throw ConfigError("wmc_level_create: too many steps");
        int ndev = 0;
        check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (L->device < 0 || L->device >= ndev) throw ConfigError("wmc_level_create: no such device");
        set_batch(*L, desc->batch);
        build_device_level(*L);
        *out = L.release();
    });
}

int wmc_mesh1d_create(int n_vertices, const double* vertices, const unsigned char* fine_flags, double coarse_h,
                      double fine_h, wmc_mesh1d** out) {
    return guarded([&] {
        if (!vertices || !fine_flags || !out) throw ConfigError("wmc_mesh1d_create: NULL argument");
        if (n_vertices < 2) throw ConfigError("wmc_mesh1d_create: at least one element");
        auto m = std::make_unique<wmc_mesh1d>();
        m->mesh.vertices.assign(vertices, vertices + n_vertices);
        m->mesh.fine_flags.assign(fine_flags, fine_flags + n_vertices - 1);
        for (int i = 0; i + 1 < n_vertices; ++i)
            if (!(vertices[i + 1] > vertices[i])) throw ConfigError("wmc_mesh1d_create: vertices not increasing");
        m->mesh.coarse_h = coarse_h;
        m->mesh.fine_h = fine_h;
        *out = m.release();
    });
}

void wmc_mesh1d_destroy(wmc_mesh1d* mesh) { delete mesh; }

int wmc_level_create_experiment(const wmc_mesh1d* mesh, int substeps, const wmc_experiment_desc* desc, int level,
                                wmc_level** out) {
    return guarded([&] {
        if (!mesh || !desc || !out) throw ConfigError("wmc_level_create_experiment: NULL argument");
        if (level < 0 || level > desc->max_level) throw ConfigError("wmc_level_create_experiment: level out of range");
        auto L = std::make_unique<wmc_level>();
        L->device = desc->device;
        experiment_tables(mesh->mesh, substeps, desc, L->spec, L->tab);
        int ndev = 0;
        check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (L->device < 0 || L->device >= ndev) throw ConfigError("wmc_level_create_experiment: no such device");
        set_batch(*L, desc->batch);
        build_device_level(*L);
        *out = L.release();
    });
}

int wmc_level_create_channel(const wmc_mesh* mesh, const wmc_experiment_desc* desc, int level, wmc_level** out) {
    return guarded([&] {
        if (!mesh || !desc || !out) throw ConfigError("wmc_level_create_channel: NULL argument");
        auto L = std::make_unique<wmc_level>();
        L->device = desc->device;
        channel_level_tables(mesh->mesh, desc, level, L->spec, L->tab, L->ch);
        int ndev = 0;
        check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (L->device < 0 || L->device >= ndev) throw ConfigError("wmc_level_create_channel: no such device");
        set_batch(*L, desc->batch);
        build_device_level(*L);
        *out = L.release();
    });
}

int wmc_channel_plan(const wmc_mesh* mesh, const wmc_experiment_desc* desc, int level, wmc_level_info* info) {
    return guarded([&] {
        if (!mesh || !desc || !info) throw ConfigError("wmc_channel_plan: NULL argument");
        wmc::LevelSpec s;
        wmc::LevelTables t;
        wmc::ChannelTables ch;
        channel_level_tables(mesh->mesh, desc, level, s, t, ch);
        fill_info(t, 0, false, info);
    });
}

int wmc_experiment_plan(const wmc_mesh1d* mesh, int substeps, const wmc_experiment_desc* desc, int level,
                        wmc_level_info* info) {
    return guarded([&] {
        if (!mesh || !desc || !info) throw ConfigError("wmc_experiment_plan: NULL argument");
        if (level < 0 || level > desc->max_level) throw ConfigError("wmc_experiment_plan: level out of range");
        wmc::LevelSpec s;
        wmc::LevelTables t;
        experiment_tables(mesh->mesh, substeps, desc, s, t);
        fill_info(t, 0, false, info);
    });
}

double wmc_experiment_model_cost(const wmc_experiment_desc* d, int level) {
    if (!d || level < 0) return 0.0;
    // model_params (experiments.cpp:177-192): 1D r = h0 / 6; channel r = channel
    // area / (two rectangles + channel), dim 2; p0 = max(1, ceil(h0 / fine_h - 1e-9))
    const bool channel = d->experiment == WMC_EXP_CHANNEL2D;
    const double channel_area = 2.0 * wmc::kChannelHalfLength * wmc::kChannelRefWidth;
    const double r = channel ? channel_area / (2.0 * wmc::kChannelRectWidth * 2.0 * wmc::kChannelRectHalfHeight +
                                               channel_area)
                             : d->h0 / 6.0;
    const double p0 = std::max(1.0, std::ceil(d->h0 / d->fine_h - 1e-9));
    const int dim = channel ? 2 : 1;
    const double pre = d->final_time * std::pow(1.0, 2 * (dim + 1)) / std::pow(d->h0, dim + 1);  // degree 1
    if (d->integrator == WMC_LEAPFROG) {  // cost_lf_level (cost_model.cpp:40-48)
        if (level == 0) return pre * ((1.0 - r) * p0 + r * std::pow(p0, dim + 1));
        const double coarse =
            (1.0 - r) * (std::pow(2.0, dim) + 1.0) / std::pow(2.0, dim) * std::pow(2.0, dim * level) * p0;
        return pre * (coarse + 2.0 * r * std::pow(p0, dim + 1));
    }
    // cost_lts_level (cost_model.cpp:50-58)
    if (level == 0) return pre * ((1.0 - r) + r * std::pow(p0, dim + 1));
    const double coarse = (1.0 - r) * (std::pow(2.0, dim + 1) + 1.0) / std::pow(2.0, dim + 1) *
                          std::pow(2.0, (dim + 1) * level);
    return pre * (coarse + 2.0 * r * std::pow(p0, dim + 1));
}

void wmc_experiment_desc_default(wmc_experiment_desc* d, int experiment) {
    if (!d) return;
    std::memset(d, 0, sizeof(*d));
    d->experiment = experiment;
    d->integrator = WMC_LOCAL_TIME_STEPPING;
    d->h0 = 1.0 / 16.0;
    d->fine_h = experiment == WMC_EXP_JUMP1D ? 1.0 / 512.0 : 1.0 / 256.0;
    d->final_time = experiment == WMC_EXP_JUMP1D ? 6.0 : 11.0;
    if (experiment == WMC_EXP_CHANNEL2D) {  // src/config_io.cpp:67-73
        d->h0 = 1.0 / 60.0;
        d->fine_h = 7.6e-4;
        d->final_time = 1.0;
    }
    d->nu = 0.01;
    d->safety = 0.9;
    d->grid_n = 512;
    d->max_level = 4;
}

int wmc_level_plan(const wmc_mesh* mesh, const wmc_level_desc* desc, wmc_level_info* info) {
    return guarded([&] {
        if (!mesh || !desc || !info) throw ConfigError("wmc_level_plan: NULL argument");
        const wmc::LevelTables t = wmc::build_level_tables(mesh->mesh, spec_from_desc(desc));
        fill_info(t, 0, t.lattice, info);
    });
}

int wmc_tile_plan(const wmc_mesh* mesh, const wmc_level_desc* desc, int stream, wmc_tile_plan_info* info) {
    return guarded([&] {
        if (!mesh || !desc || !info) throw ConfigError("wmc_tile_plan: NULL argument");
        const wmc::LevelTables t = wmc::build_level_tables(mesh->mesh, spec_from_desc(desc));
        // WMC_PLAN_WIDE / WMC_PLAN_NARROW: planning studies of other region shapes (host only)
        const char* pw = std::getenv("WMC_PLAN_WIDE");
        const char* pn = std::getenv("WMC_PLAN_NARROW");
        const wmc::TilePlan plan = wmc::plan_tiles(t, pw ? std::atoi(pw) : wmc::kTileWz, pn ? std::atoi(pn) : wmc::kTileHz,
                                                   wmc::kTileK, stream ? wmc::kStreamThreads : 0, wmc::kStreamMaxP);
        if (std::getenv("WMC_DEBUG_TILES"))
            std::fprintf(stderr, "tile plan: ok=%d layout=%s reason=%s tiles=%d slabs=%d max_gen=%d max_app=%d "
                         "max_ent=%d work=%.3f notes=%s\n", plan.ok, plan.layout.c_str(), plan.reason.c_str(),
                         plan.n_tiles, plan.n_slabs, plan.max_gen, plan.max_app, plan.max_ent, plan.work_factor,
                         plan.notes.c_str());
        *info = wmc_tile_plan_info{};
        info->ok = plan.ok ? 1 : 0;
        info->n_tiles = plan.n_tiles;
        info->n_slabs = plan.n_slabs;
        info->max_gen = plan.max_gen;
        info->work_factor = plan.work_factor;
        long streamed = 0;
        for (int q = 0; q < plan.n_slabs; ++q)
            streamed += static_cast<long>(plan.slab_own[4 * q + 1] - plan.slab_own[4 * q]) *
                        (plan.slab_own[4 * q + 3] - plan.slab_own[4 * q + 2]);
        const double box = t.box ? static_cast<double>(t.lat_m + 1) * (t.lat_m + 1) : 1.0;
        info->streamed_frac = static_cast<double>(streamed) / box;
        std::snprintf(info->layout, sizeof(info->layout), "%s", plan.layout.c_str());
        std::snprintf(info->reason, sizeof(info->reason), "%s", plan.ok ? plan.notes.c_str() : plan.reason.c_str());
    });
}

int wmc_level_get_info(const wmc_level* L, wmc_level_info* info) {
    return guarded([&] {
        if (!L || !info) throw ConfigError("wmc_level_get_info: NULL argument");
        fill_info(L->tab, L->batch, L->lattice, info, static_cast<int>(L->path));
        info->n_structured = L->n_structured;
        info->fused = L->fused_smem > 0 ? (L->fused_zp_global ? 2 : 1) : 0;
    });
}

void wmc_level_destroy(wmc_level* L) { delete L; }

void* wmc_level_stream(wmc_level* L) { return L ? static_cast<void*>(L->stream) : nullptr; }

// Waits for the level's stream and reports the first failing sample of the
// device-resident pairs issued since the last call (wmc_eval_pairs_device
// folds every batch's check_finite flags into the level's record), as
// finish_pairs does for the host path; the record is cleared.
int wmc_synchronize(wmc_level* L, wmc_error* err) {
    return guarded([&] {
        if (!L) throw ConfigError("wmc_synchronize: NULL level");
        check(cudaSetDevice(L->device), "cudaSetDevice");
        check(cudaStreamSynchronize(L->stream), "synchronize");
        if (err) {
            err->sample = -1;
            err->step = 0;
            err->level = L->fail_level;
        }
        if (!L->d_fail_rec) return;
        unsigned long long rec[2];
        check(cudaMemcpy(rec, L->d_fail_rec, sizeof(rec), cudaMemcpyDeviceToHost), "fail record");
        if (rec[0] == ~0ull && rec[1] == ~0ull) return;
        check(cudaMemset(L->d_fail_rec, 0xff, sizeof(rec)), "fail record");
        // the lower sample index first (the fine solve of a pair runs first)
        const bool fine_first = rec[0] >> 24 <= rec[1] >> 24;
        const unsigned long long r = fine_first ? rec[0] : rec[1];
        const long sample = static_cast<long>(r >> 24);
        if (err) {
            err->sample = sample;
            err->step = static_cast<int>(r & 0xffffff);
            err->level = fine_first ? L->fail_level : L->fail_level - 1;
        }
        g_last_error = "level " + std::to_string(L->fail_level) + ", sample " + std::to_string(sample) +
                       ": time integration unstable";
        throw NumericalError(g_last_error);
    });
}

int wmc_eval_pairs(wmc_level* fine, wmc_level* coarse, uint64_t seed, uint32_t level, uint64_t first, uint64_t count,
                   double* dq, double* q_fine, wmc_cost* cost, wmc_error* err) {
    return guarded([&] { eval_pairs_impl(fine, coarse, seed, level, first, count, dq, q_fine, nullptr, nullptr, cost, err); });
}

int wmc_eval_pairs_device(wmc_level* fine, wmc_level* coarse, uint64_t seed, uint32_t level, uint64_t first,
                          uint64_t count, double* d_dq, double* d_q_fine) {
    return guarded([&] {
        if (fine && count > static_cast<std::uint64_t>(coarse ? std::min(fine->batch, coarse->batch) : fine->batch) &&
            !(d_dq && d_q_fine))
            throw ConfigError("wmc_eval_pairs_device: results of more than one batch need device buffers");
        eval_pairs_impl(fine, coarse, seed, level, first, count, nullptr, nullptr, d_dq, d_q_fine, nullptr, nullptr);
    });
}

int wmc_kl_table(int cells_x, int cells_y, double sigma, double corr_len, int modes, double* table, double* lambda) {
    return guarded([&] {
        if (modes > wmc::kMaxKLModes) throw ConfigError("wmc_kl_table: at most 64 modes");
        const wmc::KLTable kl = wmc::kl_cell_table(cells_x, cells_y, sigma, corr_len, modes);
        if (table) std::copy(kl.t.begin(), kl.t.end(), table);
        if (lambda) std::copy(kl.lambda.begin(), kl.lambda.end(), lambda);
    });
}

int wmc_kl_modes(double sigma, double corr_len, int modes, double* out) {
    return guarded([&] {
        if (!out) throw ConfigError("wmc_kl_modes: NULL argument");
        if (modes > wmc::kMaxKLModes) throw ConfigError("wmc_kl_modes: at most 64 modes");
        const std::vector<double> v = wmc::kl_mode_list(sigma, corr_len, modes);
        std::copy(v.begin(), v.end(), out);
    });
}

int wmc_level_draw(wmc_level* L, uint64_t seed, uint32_t level_index, uint64_t first, uint64_t count, double* out) {
    return guarded([&] {
        if (!L || !out) throw ConfigError("wmc_level_draw: NULL argument");
        check(cudaSetDevice(L->device), "cudaSetDevice");
        const int S = round64(static_cast<long>(count));
        const int nc = L->tab.n_cells;
        double* d = nullptr;
        check(cudaMalloc(&d, sizeof(double) * S * nc), "cudaMalloc");
        launch_draw(*L, seed, level_index, first, static_cast<int>(count), S, d, L->stream);
        std::vector<double> h(static_cast<std::size_t>(S) * nc);
        cudaError_t e = cudaMemcpyAsync(h.data(), d, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, L->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(L->stream);
        cudaFree(d);
        check(e, "draw copy");
        for (std::uint64_t i = 0; i < count; ++i)
            for (int k = 0; k < nc; ++k) out[i * nc + k] = h[static_cast<std::size_t>(k) * S + i];
    });
}

int wmc_level_cfl(wmc_level* L, uint64_t seed, uint32_t level_index, uint64_t first, uint64_t count, double* dt,
                  long* steps) {
    return guarded([&] {
        if (!L || !dt || !steps) throw ConfigError("wmc_level_cfl: NULL argument");
        if (!(L->tab.cfl_safety > 0.0)) throw ConfigError("wmc_level_cfl: level has no per-sample CFL");
        check(cudaSetDevice(L->device), "cudaSetDevice");
        Workspace& w = workspace(*L, 0);
        for (std::uint64_t off = 0; off < count; off += L->batch) {
            const int c = static_cast<int>(std::min<std::uint64_t>(L->batch, count - off));
            const int S = round64(c);
            launch_draw(*L, seed, level_index, first + off, c, S, L->d_cells, L->stream);
            cfl_phase(*L, w, L->d_cells, S, c, L->stream);
            for (int i = 0; i < c; ++i) {
                steps[off + i] = w.h_nsteps[i];
                dt[off + i] = L->spec.final_time / static_cast<double>(w.h_nsteps[i]);
            }
        }
    });
}

int wmc_draw_cells(uint64_t seed, uint32_t level, uint64_t first, uint64_t count, int n_cells, double lo, double hi,
                   int device, double* out) {
    return guarded([&] {
        if (!out || n_cells <= 0) throw ConfigError("wmc_draw_cells: bad arguments");
        check(cudaSetDevice(device), "cudaSetDevice");
        const int S = round64(static_cast<long>(count));
        double* d = nullptr;
        check(cudaMalloc(&d, sizeof(double) * S * n_cells), "cudaMalloc");
        wmc::launch_draw_cells(seed, level, first, static_cast<int>(count), S, n_cells, lo, hi, d, nullptr);
        std::vector<double> h(static_cast<std::size_t>(S) * n_cells);
        const cudaError_t e = cudaMemcpy(h.data(), d, sizeof(double) * h.size(), cudaMemcpyDeviceToHost);
        cudaFree(d);
        check(e, "draw_cells copy");
        for (std::uint64_t i = 0; i < count; ++i)
            for (int k = 0; k < n_cells; ++k) out[i * n_cells + k] = h[static_cast<std::size_t>(k) * S + i];
    });
}

int wmc_run_mlmc_fixed(wmc_level** levels, int n_levels, const long* first, const long* counts, uint64_t seed,
                       wmc_level_stats* stats, wmc_error* err) {
    return guarded([&] {
        if (!levels || n_levels < 1 || !counts || !stats) throw ConfigError("wmc_run_mlmc_fixed: bad arguments");
        std::vector<Acc> acc(n_levels);
        std::vector<LevelJob> jobs;
        for (int l = 0; l < n_levels; ++l) jobs.push_back({l, first ? first[l] : 0, counts[l]});
        run_levels(levels, jobs, seed, acc, err);
        for (int l = 0; l < n_levels; ++l) fill_stats(l, acc[l], 0.0, stats[l]);
    });
}

void wmc_mlmc_config_default(wmc_mlmc_config* c) {
    if (!c) return;
    c->eps = 1e-3;
    c->alpha = 2.0;
    c->initial_samples = 16;
    c->initial_levels = 2;
    c->max_level = 6;
    c->master_seed = 0;
    c->bias_window = 1;
}

// Adaptive driver restating reference run_mlmc (src/mlmc.cpp:165-233) with
// optimal_samples (:75-92), bias_proxy_sq (:94-98) and bias_over_window
// (:151-161); jobs of one level run as one batched index range.
int wmc_run_mlmc(wmc_level** levels, int n_levels, const double* model_cost, const wmc_mlmc_config* cfg,
                 wmc_mlmc_result* result, wmc_level_stats* stats, wmc_error* err) {
    return wmc_run_mlmc_vec(levels, n_levels, model_cost, cfg, result, stats, nullptr, err);
}

namespace {
// device groups for the multi-device drivers: level l of group d at
// levels[d * n_levels + l], one device per group, the same level tables
void check_device_groups(wmc_level** levels, int n_dev, int n_levels) {
    if (!levels || n_dev < 1 || n_levels < 1) throw ConfigError("device groups: bad arguments");
    for (int d = 0; d < n_dev; ++d)
        for (int l = 0; l < n_levels; ++l) {
            const wmc_level* a = levels[l];
            const wmc_level* b = levels[static_cast<std::size_t>(d) * n_levels + l];
            if (!a || !b) throw ConfigError("device groups: NULL level");
            if (b->device != levels[static_cast<std::size_t>(d) * n_levels]->device)
                throw ConfigError("device groups: a group spans several devices");
            if (a->tab.n != b->tab.n || a->tab.n_r != b->tab.n_r || a->tab.n_steps != b->tab.n_steps ||
                a->tab.p != b->tab.p || a->tab.nq != b->tab.nq)
                throw ConfigError("device groups: level " + std::to_string(l) + " differs between groups");
        }
}

// the adaptive driver over n_dev device groups (levels[d * n_levels + l])
void run_mlmc_impl(wmc_level** levels, int n_dev, int n_levels, const double* model_cost, const wmc_mlmc_config* cfg,
                   wmc_mlmc_result* result, wmc_level_stats* stats, double* estimate, wmc_error* err) {
        if (!levels || n_levels < 1 || n_dev < 1 || !model_cost || !cfg || !result || !stats)
            throw ConfigError("wmc_run_mlmc: bad arguments");
        if (!(cfg->eps > 0.0)) throw ConfigError("run_mlmc: eps must be positive");
        if (cfg->alpha < 1.0) throw ConfigError("run_mlmc: alpha >= 1 required");
        const int cap = std::min(cfg->max_level, n_levels - 1);
        int top = std::min(cfg->initial_levels, cap);
        std::vector<Acc> acc(top + 1);
        std::vector<long> targets(top + 1, cfg->initial_samples);
        auto bias_proxy = [&](double mean_norm) { return bias_proxy_norm(mean_norm, cfg->alpha); };
        auto bias_window = [&]() {
            double worst = 0.0;
            for (int j = 0; j < cfg->bias_window && top - j >= 1; ++j) {
                const int l = top - j;
                worst = std::max(worst, bias_proxy(acc[l].mean_dq_norm()) * std::pow(2.0, -2.0 * cfg->alpha * (top - l)));
            }
            return worst;
        };
        bool converged = false;
        std::vector<PairCache> cache(n_levels);
        const bool no_ahead = std::getenv("WMC_MLMC_NO_AHEAD") != nullptr;  // A/B knob: plain waves
        {
            while (true) {
                if (no_ahead) {
                    std::vector<LevelJob> jobs;
                    for (int l = 0; l <= top; ++l)
                        if (acc[l].n < targets[l]) jobs.push_back({l, acc[l].n, targets[l] - acc[l].n});
                    run_levels(levels, jobs, cfg->master_seed, acc, err);
                } else {
                    cached_wave(levels, n_dev, n_levels, targets, top + 1 <= cap ? top + 1 : -1, cfg->master_seed,
                                acc, cache, err);
                }
                std::vector<double> v(top + 1);
                for (int l = 0; l <= top; ++l) v[l] = acc[l].variance();
                const std::vector<long> wanted = optimal_samples_impl(v.data(), model_cost, top + 1, cfg->eps, 2);
                bool increased = false;
                for (int l = 0; l <= top; ++l) {
                    if (wanted[l] > targets[l]) {
                        targets[l] = wanted[l];
                        increased = true;
                    }
                }
                if (increased) continue;
                if (top >= 1 && bias_window() < 0.5 * cfg->eps * cfg->eps) {
                    converged = true;
                    break;
                }
                if (top >= cap) break;
                ++top;
                acc.emplace_back();
                targets.push_back(cfg->initial_samples);
            }
        }
        std::memset(result, 0, sizeof(*result));
        result->converged = converged ? 1 : 0;
        result->levels_used = top;
        const int nq = levels[0]->tab.nq;
        std::vector<double> est(nq, 0.0);
        for (int l = 0; l <= top; ++l) {
            fill_stats(l, acc[l], model_cost[l], stats[l]);
            const std::vector<double> m = acc[l].mean_dq();
            for (int k = 0; k < nq && k < static_cast<int>(m.size()); ++k) est[k] += m[k];
            result->total_variance += stats[l].variance / static_cast<double>(stats[l].n_samples);
            result->total_model_cost += model_cost[l] * static_cast<double>(stats[l].n_samples);
        }
        result->bias = bias_window();
        result->rmse = std::sqrt(result->total_variance + result->bias);
        // the MLMC estimate: sum of the levels' mean dQ (reference MlmcResult::estimate);
        // the scalar field holds it for one output, its norm for QoI vectors
        if (estimate) std::copy(est.begin(), est.end(), estimate);
        if (nq == 1) {
            result->estimate = est[0];
        } else {
            Acc norm_of;
            norm_of.init(levels[0]->tab.qoi_norm_w);
            result->estimate = norm_of.norm(est.data());
        }
}
}  // namespace

int wmc_run_mlmc_vec(wmc_level** levels, int n_levels, const double* model_cost, const wmc_mlmc_config* cfg,
                     wmc_mlmc_result* result, wmc_level_stats* stats, double* estimate, wmc_error* err) {
    return guarded([&] { run_mlmc_impl(levels, 1, n_levels, model_cost, cfg, result, stats, estimate, err); });
}

int wmc_run_mlmc_multi(wmc_level** levels, int n_devices, int n_levels, const double* model_cost,
                       const wmc_mlmc_config* cfg, wmc_mlmc_result* result, wmc_level_stats* stats, double* estimate,
                       wmc_error* err) {
    return guarded([&] {
        check_device_groups(levels, n_devices, n_levels);
        run_mlmc_impl(levels, n_devices, n_levels, model_cost, cfg, result, stats, estimate, err);
    });
}

int wmc_run_mlmc_fixed_multi(wmc_level** levels, int n_devices, int n_levels, const long* counts, uint64_t seed,
                             wmc_level_stats* stats, wmc_error* err) {
    return guarded([&] {
        if (!levels || n_levels < 1 || !counts || !stats) throw ConfigError("wmc_run_mlmc_fixed_multi: bad arguments");
        check_device_groups(levels, n_devices, n_levels);
        std::vector<Issue> issues;
        for (int l = 0; l < n_levels; ++l)
            if (counts[l] > 0) issues.push_back({l, 0, counts[l]});
        std::vector<PairCache> cache(n_levels);
        eval_into_cache(levels, n_devices, n_levels, issues, seed, cache);
        // fold in (level, index) order (src/mlmc.cpp:145-147): independent of n_devices
        std::vector<Acc> acc(n_levels);
        std::vector<long> targets(counts, counts + n_levels);
        cached_wave(levels, n_devices, n_levels, targets, -1, seed, acc, cache, err);
        for (int l = 0; l < n_levels; ++l) fill_stats(l, acc[l], 0.0, stats[l]);
    });
}

long wmc_launch_count(void) { return g_launches.load(); }

int wmc_optimal_samples(const double* variances, const double* costs, int n_levels, double eps, long min_samples,
                        long* out) {
    return guarded([&] {
        if (!variances || !costs || !out || n_levels < 1) throw ConfigError("wmc_optimal_samples: bad arguments");
        if (!(eps > 0.0)) throw ConfigError("wmc_optimal_samples: eps must be positive");
        const std::vector<long> r = optimal_samples_impl(variances, costs, n_levels, eps, min_samples);
        std::copy(r.begin(), r.end(), out);
    });
}

double wmc_bias_proxy_sq(double mean_dq, double alpha) { return bias_proxy_impl(mean_dq, alpha); }

int wmc_moments_device(wmc_level* level, const double* d_dq, const double* d_q, uint64_t count, double* d_out) {
    return guarded([&] {
        if (!level || !d_dq || !d_q || !d_out) throw ConfigError("wmc_moments_device: NULL argument");
        if (count > static_cast<std::uint64_t>(INT_MAX)) throw ConfigError("wmc_moments_device: count too large");
        if (level->tab.nq != 1)
            throw ConfigError("wmc_moments_device: scalar QoI levels only (QoI vectors fold on the host)");
        check(cudaSetDevice(level->device), "cudaSetDevice");
        wmc::launch_moments(d_dq, d_q, static_cast<int>(count), d_out, level->stream);
        ++g_launches;
        check(cudaGetLastError(), "moments launch");
    });
}

int wmc_profile_enable(wmc_level* level, int on) {
    return guarded([&] {
        if (!level) throw ConfigError("wmc_profile_enable: NULL level");
        level->profile = on != 0;
    });
}

int wmc_profile_read(wmc_level* level, double* sweep_ms, long* sweep_launches, double* sub_ms, long* sub_launches,
                     double* upd_ms, long* upd_launches) {
    return guarded([&] {
        if (!level) throw ConfigError("wmc_profile_read: NULL level");
        check(cudaSetDevice(level->device), "cudaSetDevice");
        check(cudaStreamSynchronize(level->stream), "synchronize");
        auto total = [](std::vector<cudaEvent_t>& v, double* ms, long* n) {
            double acc = 0.0;
            for (std::size_t i = 0; i + 1 < v.size(); i += 2) {
                float f = 0.0f;
                check(cudaEventElapsedTime(&f, v[i], v[i + 1]), "cudaEventElapsedTime");
                acc += f;
            }
            if (ms) *ms = acc;
            if (n) *n = static_cast<long>(v.size() / 2);
            for (auto e : v) cudaEventDestroy(e);
            v.clear();
        };
        total(level->ev_sweep, sweep_ms, sweep_launches);
        total(level->ev_sub, sub_ms, sub_launches);
        total(level->ev_upd, upd_ms, upd_launches);
    });
}

}  // extern "C"
