// sm_100a kernels of the batched LF / LF-LTS sample evaluator.  See
// kernels.cuh for the layout and DESIGN.md for the roofline of each kernel.
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>
#include <cstdint>
#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

#include "kernels.cuh"

#ifndef WMC_GSUB_MINB
#define WMC_GSUB_MINB 4  // 64 registers (measured 1.26x over the unconstrained 120-register build, config 3)
#endif
#ifndef WMC_TIER_MINB
#define WMC_TIER_MINB 6  // 40 registers (measured 1.07x, config 2 level 4)
#endif
#ifndef WMC_SWEEP_MINB
#define WMC_SWEEP_MINB 5  // 48 registers: 5 blocks per SM (measured 1.2x on HBM-bound sweeps over the 64-register build)
#endif

namespace wmc {

namespace {

// The coefficient cell of operator entry q: packed above the column
// (col | cell << col_bits), or, when the level's cells do not fit beside its
// columns (narrow-channel levels), from the separate per-entry array.
__device__ __forceinline__ int ent_cell(const int* __restrict__ cell_ix, int q, int pk, int col_bits) {
    return cell_ix ? __ldg(cell_ix + q) : static_cast<int>(static_cast<unsigned>(pk) >> col_bits);
}

// ---------------------------------------------------------------------------
// K0: per-sample coefficients.  Bit-identical to the reference RngStream
// (include/wavemc/rng.hpp:14-19, src/rng.cpp:14-32): key from
// (seed, level, index), word_c = mix64(key + c * phi), unit = (w >> 11) 2^-53,
// next_uniform = lo + (hi - lo) * unit.  The affine map uses explicitly
// rounded ops so that nvcc cannot contract it into an FMA.

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__global__ void draw_cells_kernel(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S,
                                  int n_cells, double lo, double hi, double* __restrict__ cells) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    if (s >= count) {
        for (int k = 0; k < n_cells; ++k) cells[k * S + s] = 1.0;  // padding lanes: harmless unit coefficient
        return;
    }
    std::uint64_t key = mix64(seed);
    key = mix64(key ^ (0xa511e9b3cc1f25d1ULL + static_cast<std::uint64_t>(level)));
    key = mix64(key ^ (0x63d1c71ad3e29f0bULL + (first + static_cast<std::uint64_t>(s))));
    const double span = __dsub_rn(hi, lo);
    for (int k = 0; k < n_cells; ++k) {
        const std::uint64_t w = mix64(key + static_cast<std::uint64_t>(k) * 0x9e3779b97f4a7c15ULL);
        const double unit = __dmul_rn(static_cast<double>(w >> 11), 0x1.0p-53);
        cells[k * S + s] = __dadd_rn(lo, __dmul_rn(span, unit));
    }
}

// Narrow-channel widths (sample_width, src/rng.cpp:59-64: the stream's first
// word through next_uniform(0.001, 0.007)) and the per-sample entries of the
// moved mesh, one thread per (entry, sample).  Every vertex position, area,
// gradient and element product is formed with explicitly rounded operations
// in the reference's order (ChannelGeometry::map, TriMesh::signed_area,
// assemble: src/mesh2d.cpp:361-389, include/wavemc/mesh.hpp:65-70,
// src/fem.cpp:97-116) so that the moved triangles are the reference's to the
// last bit; only the summation order of a pair's / vertex's triangles differs.
// Padding lanes take the reference width.
__device__ __forceinline__ double channel_y(const ChannelArgs& a, int l, double width) {
    const double y = __ldg(a.vy + l);
    const double half_ref = __dmul_rn(0.5, 0.004);
    const double peak = __dmul_rn(0.5, __dsub_rn(width, 0.004));
    const double ay = fabs(y);
    double value;
    if (ay <= half_ref)
        value = __dmul_rn(peak, __ddiv_rn(ay, half_ref));
    else
        value = __ddiv_rn(__dmul_rn(peak, __dsub_rn(0.5, ay)), __dsub_rn(0.5, half_ref));
    if (y < 0.0) value = -value;
    return __dadd_rn(y, __dmul_rn(__ldg(a.vblend + l), value));
}

// area, and gradients of the barycentric basis of moving triangle t
__device__ __forceinline__ double channel_tri(const ChannelArgs& a, int t, double width, double* gx, double* gy) {
    const int v0 = __ldg(a.tri + 3 * t), v1 = __ldg(a.tri + 3 * t + 1), v2 = __ldg(a.tri + 3 * t + 2);
    const double x0 = __ldg(a.vx + v0), x1 = __ldg(a.vx + v1), x2 = __ldg(a.vx + v2);
    const double y0 = channel_y(a, v0, width), y1 = channel_y(a, v1, width), y2 = channel_y(a, v2, width);
    const double area = __dmul_rn(0.5, __dsub_rn(__dmul_rn(__dsub_rn(x1, x0), __dsub_rn(y2, y0)),
                                                 __dmul_rn(__dsub_rn(x2, x0), __dsub_rn(y1, y0))));
    if (gx) {
        const double a2 = __dmul_rn(2.0, area);
        gx[0] = __ddiv_rn(__dsub_rn(y1, y2), a2);
        gx[1] = __ddiv_rn(__dsub_rn(y2, y0), a2);
        gx[2] = __ddiv_rn(__dsub_rn(y0, y1), a2);
        gy[0] = __ddiv_rn(__dsub_rn(x2, x1), a2);
        gy[1] = __ddiv_rn(__dsub_rn(x0, x2), a2);
        gy[2] = __ddiv_rn(__dsub_rn(x1, x0), a2);
    }
    return area;
}

__device__ __forceinline__ double channel_mass(const ChannelArgs& a, int l, double width) {
    double m = __ldg(a.ms + l);
    for (int q = __ldg(a.m_ptr + l); q < __ldg(a.m_ptr + l + 1); ++q)
        m = __dadd_rn(m, __ddiv_rn(channel_tri(a, __ldg(a.m_tri + q), width, nullptr, nullptr), 3.0));
    return m;
}

__global__ void __launch_bounds__(128) draw_channel_kernel(std::uint64_t seed, std::uint32_t level,
                                                           std::uint64_t first, int count, int S, ChannelArgs a,
                                                           double* __restrict__ cells) {
    const int chunks = (S + 127) / 128;
    const int k = blockIdx.x / chunks;
    const int s = (blockIdx.x % chunks) * 128 + threadIdx.x;
    if (s >= S || k > a.n_ent) return;
    const std::size_t SS = static_cast<std::size_t>(S);
    if (k == 0) {
        cells[s] = 1.0;
        return;
    }
    double width = 0.004;  // padding lanes: the reference geometry
    if (s < count) {
        std::uint64_t key = mix64(seed);
        key = mix64(key ^ (0xa511e9b3cc1f25d1ULL + static_cast<std::uint64_t>(level)));
        key = mix64(key ^ (0x63d1c71ad3e29f0bULL + (first + static_cast<std::uint64_t>(s))));
        const std::uint64_t w = mix64(key);
        const double unit = __dmul_rn(static_cast<double>(w >> 11), 0x1.0p-53);
        width = __dadd_rn(0.001, __dmul_rn(__dsub_rn(0.007, 0.001), unit));
    }
    const int e = k - 1;
    const int li = __ldg(a.e_li + e), lj = __ldg(a.e_lj + e);
    const double mi = li >= 0 ? channel_mass(a, li, width) : __ldg(a.e_mi + e);
    const double mj = lj >= 0 ? channel_mass(a, lj, width) : __ldg(a.e_mj + e);
    double kij = __ldg(a.e_ks + e);
    for (int q = __ldg(a.k_ptr + e); q < __ldg(a.k_ptr + e + 1); ++q) {
        const int code = __ldg(a.k_tri + q);
        const int t = code / 9, ca = (code / 3) % 3, cb = code % 3;
        double gx[3], gy[3];
        const double area = channel_tri(a, t, width, gx, gy);
        kij = __dadd_rn(kij, __dmul_rn(__dmul_rn(1.0, area),
                                       __dadd_rn(__dmul_rn(gx[ca], gx[cb]), __dmul_rn(gy[ca], gy[cb]))));
    }
    cells[static_cast<std::size_t>(k) * SS + s] = __ddiv_rn(kij, __dsqrt_rn(__dmul_rn(mi, mj)));
}

// 1D grid over (row group of kSweepWarps rows, 64-sample chunk), row group
// fastest: concurrently resident blocks cover a contiguous band of rows, so
// the N/S neighbour rows of a gather are L2 hits (measured faster than
// chunk-fastest order, which favours DRAM page locality)
__device__ __forceinline__ int n_groups(int rows) { return (rows + kSweepWarps - 1) / kSweepWarps; }
__device__ __forceinline__ int grid_chunk(int rows) { return blockIdx.x / n_groups(rows); }
__device__ __forceinline__ int grid_rowgroup(int rows) { return blockIdx.x % n_groups(rows); }

// Log-normal KL coefficients (BASELINE config 4, no reference counterpart):
// per sample the stream's words 2i, 2i+1 give u1, u2 = next_unit(), then
// r = sqrt(-2 log(1 - u1)), xi_2i = r cos(2 pi u2), xi_2i+1 = r sin(2 pi u2);
// g_k = sum_m T[k][m] xi_m, c_k = exp(g_k).  One thread per sample, the
// normals in shared memory.
constexpr int kKLThreads = 64;
constexpr int kKLMaxModes = 64;

__global__ void __launch_bounds__(kKLThreads) draw_kl_kernel(std::uint64_t seed, std::uint32_t level,
                                                             std::uint64_t first, int count, int S, int n_cells,
                                                             int modes, const double* __restrict__ table,
                                                             double* __restrict__ cells) {
    __shared__ double xi_s[kKLMaxModes][kKLThreads];
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    // blockIdx.y: a chunk of the cells (per-element fields have one cell per
    // triangle; every chunk's CTA forms the sample's normals again)
    const int per = (n_cells + gridDim.y - 1) / gridDim.y;
    const int k_lo = blockIdx.y * per, k_hi = min(n_cells, k_lo + per);
    if (s >= count) {
        for (int k = k_lo; k < k_hi; ++k) cells[static_cast<std::size_t>(k) * S + s] = 1.0;
        return;
    }
    std::uint64_t key = mix64(seed);
    key = mix64(key ^ (0xa511e9b3cc1f25d1ULL + static_cast<std::uint64_t>(level)));
    key = mix64(key ^ (0x63d1c71ad3e29f0bULL + (first + static_cast<std::uint64_t>(s))));
    const double two_pi = 6.283185307179586;
    for (int i = 0; 2 * i < modes; ++i) {
        const std::uint64_t w1 = mix64(key + static_cast<std::uint64_t>(2 * i) * 0x9e3779b97f4a7c15ULL);
        const std::uint64_t w2 = mix64(key + static_cast<std::uint64_t>(2 * i + 1) * 0x9e3779b97f4a7c15ULL);
        const double u1 = __dmul_rn(static_cast<double>(w1 >> 11), 0x1.0p-53);
        const double u2 = __dmul_rn(static_cast<double>(w2 >> 11), 0x1.0p-53);
        const double r = sqrt(-2.0 * log(1.0 - u1));
        const double th = __dmul_rn(two_pi, u2);
        xi_s[2 * i][threadIdx.x] = r * cos(th);
        if (2 * i + 1 < modes) xi_s[2 * i + 1][threadIdx.x] = r * sin(th);
    }
    for (int k = k_lo; k < k_hi; ++k) {
        double g = 0.0;
        for (int m = 0; m < modes; ++m) g += __ldg(table + static_cast<std::size_t>(k) * modes + m) * xi_s[m][threadIdx.x];
        cells[static_cast<std::size_t>(k) * S + s] = exp(g);
    }
}

__device__ __forceinline__ std::uint64_t stream_key(std::uint64_t seed, std::uint32_t level, std::uint64_t index) {
    std::uint64_t key = mix64(seed);
    key = mix64(key ^ (0xa511e9b3cc1f25d1ULL + static_cast<std::uint64_t>(level)));
    return mix64(key ^ (0x63d1c71ad3e29f0bULL + index));
}

// one block per sample: the stream's symmetric words in shared memory, the
// element coefficients from the table (rows of `terms` entries)
constexpr int kKl1dMaxTerms = 256;
__global__ void __launch_bounds__(128) draw_kl1d_kernel(std::uint64_t seed, std::uint32_t level, std::uint64_t first,
                                                       int count, int S, int n_cells, int terms,
                                                       const double* __restrict__ table, double* __restrict__ cells) {
    __shared__ double xi[kKl1dMaxTerms];
    const int s = blockIdx.x;
    if (s >= count) {  // padding lanes: unit coefficient
        for (int e = threadIdx.x; e < n_cells; e += blockDim.x) cells[static_cast<std::size_t>(e) * S + s] = 1.0;
        return;
    }
    const std::uint64_t key = stream_key(seed, level, first + static_cast<std::uint64_t>(s));
    for (int m = threadIdx.x; m < terms; m += blockDim.x) {
        const std::uint64_t w = mix64(key + static_cast<std::uint64_t>(m) * 0x9e3779b97f4a7c15ULL);
        const double unit = __dmul_rn(static_cast<double>(w >> 11), 0x1.0p-53);
        xi[m] = __dsub_rn(__dmul_rn(2.0, unit), 1.0);  // next_symmetric (rng.cpp:34-36)
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n_cells; e += blockDim.x) {
        const double* row = table + static_cast<std::size_t>(e) * terms;
        double acc = 0.0;
        for (int m = 0; m < terms; ++m) acc += __ldg(row + m) * xi[m];
        cells[static_cast<std::size_t>(e) * S + s] = 1.0 + acc;
    }
}

__global__ void draw_jump1d_kernel(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S,
                                   int n_cells, double h0, const double* __restrict__ x, double* __restrict__ cells) {
    const int s = blockIdx.x;
    double jump = 10.0;  // padding lanes: unit coefficient everywhere on [0, 6]
    if (s < count) {
        const std::uint64_t w = mix64(stream_key(seed, level, first + static_cast<std::uint64_t>(s)));
        const double unit = __dmul_rn(static_cast<double>(w >> 11), 0x1.0p-53);
        const double lo = __dsub_rn(4.0, h0);
        jump = __dadd_rn(lo, __dmul_rn(__dsub_rn(4.0, lo), unit));  // next_uniform(4 - h0, 4)
    }
    for (int e = threadIdx.x; e < n_cells; e += blockDim.x)
        cells[static_cast<std::size_t>(e) * S + s] = __ldg(x + e) < jump ? 1.0 : 4.0;
}

__device__ __forceinline__ void flag_fail(int* fail, int s, int count, int step) {
    if (s < count) atomicMin(fail + s, step);
}

// per-sample CFL: the lane's two samples' dt^2 scale and whether `step` is
// still inside their horizons
__device__ __forceinline__ double2 lane_rel(const double* rel, int s0) {
    return rel ? __ldg(reinterpret_cast<const double2*>(rel + s0)) : make_double2(1.0, 1.0);
}
__device__ __forceinline__ int2 lane_live(const int* nsteps, int s0, int step) {
    if (!nsteps) return make_int2(1, 1);
    const int2 n = __ldg(reinterpret_cast<const int2*>(nsteps + s0));
    return make_int2(step <= n.x, step <= n.y);
}
// z_{n+1} store + check_finite for the live samples of the lane
__device__ __forceinline__ void store_z(double* p, double2 out, int2 live, int* fail, int s0, int count, int step) {
    if (live.x && live.y) {
        *reinterpret_cast<double2*>(p) = out;
    } else {
        if (live.x) p[0] = out.x;
        if (live.y) p[1] = out.y;
    }
    if (live.x && !(fabs(out.x) <= 1e100)) flag_fail(fail, s0, count, step);
    if (live.y && !(fabs(out.y) <= 1e100)) flag_fail(fail, s0 + 1, count, step);
}

// ---------------------------------------------------------------------------
// K1: the full sweep g = A(omega) z over every row, one warp per (row, 64
// samples), 16-byte loads per lane.  A(omega)_ij = sum_k c_k a0_ijk
// ("parts"), gathered node-centrically: no atomics, deterministic.
// Rows < split stash g for the substep kernel; the others take the
// leapfrog update z+ = 2 z - z- - factor * g in place of z-
// (reference src/integrators.cpp:89-115; for LTS rows outside R the
// recursion collapses to factor = -2 d_p(g = 1), :117-157).

template <bool kInit, bool kParts, bool kSplit = false>
__global__ void __launch_bounds__(kSweepWarps * 32) sweep_kernel(SweepArgs a) {
    __shared__ double2 tile[kSweepWarps][32];  // g of the block's R rows: [row][lane] = samples 2 lane, 2 lane + 1
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row0 = grid_rowgroup(a.n) * kSweepWarps;
    const int row = row0 + warp;
    const int s0 = grid_chunk(a.n) * kSweepChunk + 2 * lane;
    const std::size_t S = static_cast<std::size_t>(a.S);
    if (row < a.n) {
        const int4 d = a.row_desc ? __ldg(a.row_desc + row) : make_int4(-1, 0, 0, 0);
        const bool structured = !kInit && !kParts && d.x >= 0 && ((d.x >> 16) & 0xff) > 0;
        int b = 0, e = 0;
        if (!structured) {
            b = __ldg(a.row_ptr + row);
            e = __ldg(a.row_ptr + row + 1);
        }
        double acc0 = 0.0, acc1 = 0.0;
        double2 zself = make_double2(0.0, 0.0);
        // z_{n-1} of a leap-frog row issued before the gather (latency overlap)
        double2 zm_early = make_double2(0.0, 0.0);
        if (!kInit && row >= a.split) zm_early = *reinterpret_cast<const double2*>(a.zp + row * S + s0);
        if (kParts) {
            // entries grouped by cell: sum a0 z_j within a part, then scale by
            // the part's coefficient (one coefficient load per part)
            double p0 = 0.0, p1 = 0.0;
            int pcell = ent_cell(kSplit ? a.cell_ix : nullptr, b, __ldg(a.ent + b), a.col_bits);
            double2 c = __ldg(reinterpret_cast<const double2*>(a.cells + pcell * S + s0));
            for (int k = b; k < e; ++k) {
                const int pk = __ldg(a.ent + k);
                const double w = __ldg(a.a0 + k);
                const int j = pk & a.col_mask;
                const int cell = ent_cell(kSplit ? a.cell_ix : nullptr, k, pk, a.col_bits);
                if (cell != pcell) {  // warp-uniform
                    acc0 += c.x * p0;
                    acc1 += c.y * p1;
                    p0 = p1 = 0.0;
                    pcell = cell;
                    c = __ldg(reinterpret_cast<const double2*>(a.cells + cell * S + s0));
                }
                if (kInit) {
                    const double zj = __ldg(a.z0 + j);
                    p0 += w * zj;
                    p1 += w * zj;
                } else {
                    const double2 z = __ldg(reinterpret_cast<const double2*>(a.zc + j * S + s0));
                    if (j == row) zself = z;
                    p0 += w * z.x;
                    p1 += w * z.y;
                }
            }
            acc0 += c.x * p0;
            acc1 += c.y * p1;
        } else if (structured) {
            // structured 5-point row: descriptor only
            const double2 w = __ldg(a.wtype + ((d.x >> 16) & 0xff) - 1);
            const double2 c = __ldg(reinterpret_cast<const double2*>(a.cells + (d.x & 0xffff) * S + s0));
            const double2 zs = __ldg(reinterpret_cast<const double2*>(a.zc + (row - d.z) * S + s0));
            const double2 zw = __ldg(reinterpret_cast<const double2*>(a.zc + (row - 1) * S + s0));
            zself = __ldg(reinterpret_cast<const double2*>(a.zc + row * S + s0));
            const double2 ze = __ldg(reinterpret_cast<const double2*>(a.zc + (row + 1) * S + s0));
            const double2 zn = __ldg(reinterpret_cast<const double2*>(a.zc + (row + d.w) * S + s0));
            double p0 = 0.0, p1 = 0.0;
            p0 += w.x * zs.x;
            p1 += w.x * zs.y;
            p0 += w.x * zw.x;
            p1 += w.x * zw.y;
            p0 += w.y * zself.x;
            p1 += w.y * zself.y;
            p0 += w.x * ze.x;
            p1 += w.x * ze.y;
            p0 += w.x * zn.x;
            p1 += w.x * zn.y;
            acc0 = c.x * p0;
            acc1 = c.y * p1;
        } else if (d.x >= 0) {
            // the row's elements all lie in one coefficient cell: one
            // coefficient load, A(omega)_ij = c * a0_ij
            const double2 c = __ldg(reinterpret_cast<const double2*>(a.cells + (d.x & 0xffff) * S + s0));
            double p0 = 0.0, p1 = 0.0;
#pragma unroll 4
            for (int k = b; k < e; ++k) {
                const int j = __ldg(a.ent + k) & a.col_mask;
                const double w = __ldg(a.a0 + k);
                if (kInit) {
                    const double zj = __ldg(a.z0 + j);
                    p0 += w * zj;
                    p1 += w * zj;
                } else {
                    const double2 z = __ldg(reinterpret_cast<const double2*>(a.zc + j * S + s0));
                    if (j == row) zself = z;
                    p0 += w * z.x;
                    p1 += w * z.y;
                }
            }
            acc0 = c.x * p0;
            acc1 = c.y * p1;
        } else {
#pragma unroll 4
            for (int k = b; k < e; ++k) {
                const int pk = __ldg(a.ent + k);
                const double w = __ldg(a.a0 + k);
                const int j = pk & a.col_mask;
                const int cell = ent_cell(kSplit ? a.cell_ix : nullptr, k, pk, a.col_bits);
                const double2 c = __ldg(reinterpret_cast<const double2*>(a.cells + cell * S + s0));
                if (kInit) {
                    const double zj = __ldg(a.z0 + j);
                    acc0 += (c.x * w) * zj;
                    acc1 += (c.y * w) * zj;
                } else {
                    const double2 z = __ldg(reinterpret_cast<const double2*>(a.zc + j * S + s0));
                    if (j == row) zself = z;
                    acc0 += (c.x * w) * z.x;
                    acc1 += (c.y * w) * z.y;
                }
            }
        }
        const std::size_t idx = row * S + s0;
        if (kInit) {
            // z1 = z0 + dt M^{1/2} v0 + dt^2/2 (F0 - A z0), v0 = F = 0 (integrators.cpp:68-87)
            const double z0 = __ldg(a.z0 + row);
            const double2 r = lane_rel(a.rel, s0);
            double2 out;
            out.x = z0 + (a.factor * r.x) * (0.0 - acc0);
            out.y = z0 + (a.factor * r.y) * (0.0 - acc1);
            *reinterpret_cast<double2*>(a.zp + idx) = make_double2(z0, z0);
            *reinterpret_cast<double2*>(a.zc_out + idx) = out;
            if (!(fabs(out.x) <= 1e100)) flag_fail(a.fail, s0, a.count, a.step);
            if (!(fabs(out.y) <= 1e100)) flag_fail(a.fail, s0 + 1, a.count, a.step);
        } else if (row < a.split) {
            if (a.g_node_major)
                *reinterpret_cast<double2*>(a.g + idx) = make_double2(acc0, acc1);
            else
                tile[warp][lane] = make_double2(acc0, acc1);
        } else {
            const double2 zn = zself;  // every row holds its diagonal entry
            const double2 zm = zm_early;
            const double2 r = lane_rel(a.rel, s0);
            double2 out;
            out.x = 2.0 * zn.x - zm.x - (a.factor * r.x) * acc0;
            out.y = 2.0 * zn.y - zm.y - (a.factor * r.y) * acc1;
            // check_finite (integrators.cpp:12-18): non-finite or |z| > 1e100
            store_z(a.zp + idx, out, lane_live(a.nsteps, s0, a.step), a.fail, s0, a.count, a.step);
        }
    }
    if (kInit || row0 >= a.split || a.g_node_major) return;  // block-uniform
    // store the block's g rows sample-major: warp w writes samples 8w..8w+7,
    // four lanes per sample, two rows (16 B) per lane
    __syncthreads();
    const int sl = 8 * warp + (lane >> 2), rr = 2 * (lane & 3);
    const int s = grid_chunk(a.n) * kSweepChunk + sl;
    const double2 t0 = tile[rr][sl >> 1], t1 = tile[rr + 1][sl >> 1];
    const double g0 = (sl & 1) ? t0.y : t0.x, g1 = (sl & 1) ? t1.y : t1.x;
    double* dst = a.g + static_cast<std::size_t>(s) * a.g_stride + row0 + rr;
    if (row0 + rr + 1 < a.split)
        *reinterpret_cast<double2*>(dst) = make_double2(g0, g1);
    else if (row0 + rr < a.split)
        dst[0] = g0;
}

// K1 (step sweep, default): each warp sweeps R consecutive rows for its 64
// samples, keeping the window z_{i-1}, z_i, z_{i+1} in registers, so a
// structured row loads only z_{i+1}, z_{i-dS} and z_{i+dN} (3 of its 5
// values) and reuses the coefficient of the previous row when the cell is
// the same.  Generic rows gather as in sweep_kernel.  Products and sums in
// the same order as sweep_kernel: bit-identical results.
constexpr int kSweepRows = 4;         // rows per warp of the HBM-resident substep kernel
constexpr int kSweepRowsDefault = 2;  // rows per warp of the step sweep (measured best with 48 registers)
#ifndef WMC_TIER_ROWS
#define WMC_TIER_ROWS 1
#endif
constexpr int kTierRows = WMC_TIER_ROWS;

template <int R>
__global__ void __launch_bounds__(kSweepWarps * 32, WMC_SWEEP_MINB) sweep_rows_kernel(SweepArgs a) {
    __shared__ double2 tile[kSweepWarps * R][32];  // g of the block's R rows: [row][lane]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int groups = (a.n - a.row_begin + kSweepWarps * R - 1) / (kSweepWarps * R);
    const int row0 = a.row_begin + (blockIdx.x % groups) * kSweepWarps * R;
    const int chunk = blockIdx.x / groups;
    const int s0 = chunk * kSweepChunk + 2 * lane;
    const std::size_t S = static_cast<std::size_t>(a.S);
    const int first = row0 + warp * R;
    auto zrow = [&](int r) {
        return __ldg(reinterpret_cast<const double2*>(a.zc + static_cast<std::size_t>(r) * S + s0));
    };
    double2 zprev = make_double2(0.0, 0.0), zcur = zprev;
    if (first < a.n) {
        if (first > 0) zprev = zrow(first - 1);
        zcur = zrow(first);
    }
    int ccell = -1;
    double2 c = make_double2(0.0, 0.0);
    const double2 fac = a.rel ? lane_rel(a.rel, s0) : make_double2(1.0, 1.0);
    const double2 factor = make_double2(a.factor * fac.x, a.factor * fac.y);
    const int2 live = lane_live(a.nsteps, s0, a.step);
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int row = first + k;
        if (row >= a.n) break;
        const std::size_t idx = static_cast<std::size_t>(row) * S + s0;
        double2 zm = make_double2(0.0, 0.0);
        if (row >= a.split) zm = *reinterpret_cast<const double2*>(a.zp + idx);
        const double2 znext = row + 1 < a.n ? zrow(row + 1) : make_double2(0.0, 0.0);
        const int4 d = __ldg(a.row_desc + row);
        double acc0 = 0.0, acc1 = 0.0;
        if (d.x >= 0 && ((d.x >> 16) & 0xff) > 0) {
            const double2 w = __ldg(a.wtype + ((d.x >> 16) & 0xff) - 1);
            if ((d.x & 0xffff) != ccell) {
                ccell = d.x & 0xffff;
                c = __ldg(reinterpret_cast<const double2*>(a.cells + ccell * S + s0));
            }
            const double2 zs = zrow(row - d.z);
            const double2 zn = zrow(row + d.w);
            double p0 = 0.0, p1 = 0.0;
            p0 += w.x * zs.x;
            p1 += w.x * zs.y;
            p0 += w.x * zprev.x;
            p1 += w.x * zprev.y;
            p0 += w.y * zcur.x;
            p1 += w.y * zcur.y;
            p0 += w.x * znext.x;
            p1 += w.x * znext.y;
            p0 += w.x * zn.x;
            p1 += w.x * zn.y;
            acc0 = c.x * p0;
            acc1 = c.y * p1;
        } else {
            const int b = d.y, e = __ldg(a.row_ptr + row + 1);
            if (d.x >= 0) {
                const double2 cc = __ldg(reinterpret_cast<const double2*>(a.cells + (d.x & 0xffff) * S + s0));
                double p0 = 0.0, p1 = 0.0;
#pragma unroll 4
                for (int q = b; q < e; ++q) {
                    const int j = __ldg(a.ent + q) & a.col_mask;
                    const double w = __ldg(a.a0 + q);
                    const double2 z = zrow(j);
                    p0 += w * z.x;
                    p1 += w * z.y;
                }
                acc0 = cc.x * p0;
                acc1 = cc.y * p1;
            } else {
#pragma unroll 4
                for (int q = b; q < e; ++q) {
                    const int pk = __ldg(a.ent + q);
                    const double w = __ldg(a.a0 + q);
                    const int j = pk & a.col_mask;
                    const int cell = ent_cell(nullptr, q, pk, a.col_bits)  /* packed: split levels take sweep_kernel */;
                    const double2 cc = __ldg(reinterpret_cast<const double2*>(a.cells + cell * S + s0));
                    const double2 z = zrow(j);
                    acc0 += (cc.x * w) * z.x;
                    acc1 += (cc.y * w) * z.y;
                }
            }
        }
        if (row < a.split) {
            if (a.g_node_major)
                *reinterpret_cast<double2*>(a.g + idx) = make_double2(acc0, acc1);
            else
                tile[warp * R + k][lane] = make_double2(acc0, acc1);
        } else {
            double2 out;
            out.x = 2.0 * zcur.x - zm.x - factor.x * acc0;
            out.y = 2.0 * zcur.y - zm.y - factor.y * acc1;
            store_z(a.zp + idx, out, live, a.fail, s0, a.count, a.step);
        }
        zprev = zcur;
        zcur = znext;
    }
    if (row0 >= a.split || a.g_node_major) return;  // block-uniform
    // the block's g rows sample-major: thread -> sample tid / 4, 8 rows each
    __syncthreads();
    constexpr int kRowsPerThread = kSweepWarps * R * kSweepChunk / (kSweepWarps * 32);
    const int sl = threadIdx.x / (kSweepWarps * R / kRowsPerThread);
    const int r0 = (threadIdx.x % (kSweepWarps * R / kRowsPerThread)) * kRowsPerThread;
    const int s = chunk * kSweepChunk + sl;
    double* dst = a.g + static_cast<std::size_t>(s) * a.g_stride + row0 + r0;
#pragma unroll
    for (int q = 0; q < kRowsPerThread; q += 2) {
        const double2 t0 = tile[r0 + q][sl >> 1], t1 = tile[r0 + q + 1][sl >> 1];
        const double g0 = (sl & 1) ? t0.y : t0.x, g1 = (sl & 1) ? t1.y : t1.x;
        if (row0 + r0 + q + 1 < a.split)
            *reinterpret_cast<double2*>(dst + q) = make_double2(g0, g1);
        else if (row0 + r0 + q < a.split)
            dst[q] = g0;
    }
}

// K1, sample-major form (tiled levels, z[s * n + i]): thread per (row,
// sample), consecutive rows in a warp, so a structured row's five loads are
// coalesced along the rows of one sample.  Rows [row_begin, n) (the tiled
// step owns R); kInit: every row, the start-up step.  Same products in the
// same order as sweep_kernel.
constexpr int kSmSamples = 4;  // samples per thread: the row's descriptor and entries serve four
// sample groups a thread walks through (WMC_SM_GROUPS: tuning knob)
static int sm_groups() {
    static const int v = [] {
        const char* e = std::getenv("WMC_SM_GROUPS");
        return e && std::atoi(e) == 4 ? 4 : 8;  // the two compiled forms (8: 1.37 vs 1.40 ms per config-3 step)
    }();
    return v;
}
template <bool kInit, int kGroups>
__global__ void __launch_bounds__(256) sweep_sm_kernel(SweepArgs a) {
    const int row = (kInit ? 0 : a.row_begin) + blockIdx.x * 256 + threadIdx.x;
    if (row >= a.n) return;
    const std::size_t n = static_cast<std::size_t>(a.n);
    const int4 d = __ldg(a.row_desc + row);
    // kSmGroups sample groups per thread, one after the other: the row's
    // descriptor is read once and its entries stay in L1 for all of them
    // (read per group they were 17 % of the kernel's DRAM bytes)
#pragma unroll 1
    for (int grp = 0; grp < kGroups; ++grp) {
    const int s0 = (blockIdx.y * kGroups + grp) * kSmSamples;
    if (s0 >= a.S) break;
    double acc[kSmSamples], zself[kSmSamples], zm[kSmSamples];
    auto zat = [&](int u, int i) { return kInit ? __ldg(a.z0 + i) : __ldg(a.zc + (s0 + u) * n + i); };
#pragma unroll
    for (int u = 0; u < kSmSamples; ++u) {
        acc[u] = 0.0;
        zself[u] = zat(u, row);
        zm[u] = kInit ? 0.0 : a.zp[(s0 + u) * n + row];
    }
    if (d.x >= 0 && ((d.x >> 16) & 0xff) > 0) {
        const double2 w = __ldg(a.wtype + ((d.x >> 16) & 0xff) - 1);
        const double* cp = a.cells + static_cast<std::size_t>(d.x & 0xffff) * a.S + s0;
#pragma unroll
        for (int u = 0; u < kSmSamples; ++u) {
            double p0 = 0.0;
            p0 += w.x * zat(u, row - d.z);
            p0 += w.x * zat(u, row - 1);
            p0 += w.y * zself[u];
            p0 += w.x * zat(u, row + 1);
            p0 += w.x * zat(u, row + d.w);
            acc[u] = __ldg(cp + u) * p0;
        }
    } else {
        const int b = d.y, e = __ldg(a.row_ptr + row + 1);
        if (d.x >= 0) {
            const double* cp = a.cells + static_cast<std::size_t>(d.x & 0xffff) * a.S + s0;
            double p0[kSmSamples] = {};
            for (int q = b; q < e; ++q) {
                const double w = __ldg(a.a0 + q);
                const int j = __ldg(a.ent + q) & a.col_mask;
#pragma unroll
                for (int u = 0; u < kSmSamples; ++u) p0[u] += w * zat(u, j);
            }
#pragma unroll
            for (int u = 0; u < kSmSamples; ++u) acc[u] = __ldg(cp + u) * p0[u];
        } else {
            for (int q = b; q < e; ++q) {
                const int pk = __ldg(a.ent + q);
                const double w = __ldg(a.a0 + q);
                const double* cp =
                    a.cells + static_cast<std::size_t>(ent_cell(nullptr, q, pk, a.col_bits)) * a.S + s0;
#pragma unroll
                for (int u = 0; u < kSmSamples; ++u) acc[u] += (__ldg(cp + u) * w) * zat(u, pk & a.col_mask);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < kSmSamples; ++u) {
        const int s = s0 + u;
        if (s >= a.count) break;
        if (kInit) {
            // z1 = z0 + dt M^{1/2} v0 + dt^2/2 (F0 - A z0), v0 = F = 0 (integrators.cpp:68-87)
            const double out = zself[u] + a.factor * (0.0 - acc[u]);
            a.zp[s * n + row] = zself[u];
            a.zc_out[s * n + row] = out;
            if (!(fabs(out) <= 1e100)) flag_fail(a.fail, s, a.count, a.step);
        } else {
            const double out = 2.0 * zself[u] - zm[u] - a.factor * acc[u];
            a.zp[s * n + row] = out;
            if (!(fabs(out) <= 1e100)) flag_fail(a.fail, s, a.count, a.step);  // check_finite (integrators.cpp:12-18)
        }
    }
    }
}

// K1, wide form (fixed dt, S a multiple of 128): four samples per lane with
// 256-bit loads and stores (LDG/STG.E.ENL2.256), 128 samples per warp, so
// each load instruction moves 1 KB per warp and a warp's rows keep twice the
// bytes in flight of sweep_rows_kernel for the same instruction count.  Same
// per-sample products and sums in the same order: bit-identical.
struct D4 {
    double x, y, z, w;
};
__device__ __forceinline__ D4 ld4_nc(const double* p) {
    D4 r;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ D4 ld4(const double* p) {
    D4 r;
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void st4(double* p, const D4& v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}
constexpr int kSweepChunkW = 128;  // samples per warp of the wide sweep

template <int R, int MINB>
__global__ void __launch_bounds__(kSweepWarps * 32, MINB) sweep_wide_kernel(SweepArgs a) {
    __shared__ D4 tile[kSweepWarps * R][32];  // g of the block's R rows: [row][lane] = samples 4 lane .. 4 lane + 3
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int groups = (a.n - a.row_begin + kSweepWarps * R - 1) / (kSweepWarps * R);
    const int row0 = a.row_begin + (blockIdx.x % groups) * kSweepWarps * R;
    const int chunk = blockIdx.x / groups;
    const int s0 = chunk * kSweepChunkW + 4 * lane;
    const std::size_t S = static_cast<std::size_t>(a.S);
    const int first = row0 + warp * R;
    auto zrow = [&](int r) { return ld4_nc(a.zc + static_cast<std::size_t>(r) * S + s0); };
    const D4 zero{0.0, 0.0, 0.0, 0.0};
    D4 zprev = zero, zcur = zero;
    if (first < a.n) {
        if (first > 0) zprev = zrow(first - 1);
        zcur = zrow(first);
    }
    int ccell = -1;
    D4 c = zero;
    const double f = a.factor;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int row = first + k;
        if (row >= a.n) break;
        const std::size_t idx = static_cast<std::size_t>(row) * S + s0;
        D4 zm = zero;
        if (row >= a.split) zm = ld4(a.zp + idx);
        const D4 znext = row + 1 < a.n ? zrow(row + 1) : zero;
        const int4 d = __ldg(a.row_desc + row);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (d.x >= 0 && ((d.x >> 16) & 0xff) > 0) {
            const double2 w = __ldg(a.wtype + ((d.x >> 16) & 0xff) - 1);
            if ((d.x & 0xffff) != ccell) {
                ccell = d.x & 0xffff;
                c = ld4_nc(a.cells + ccell * S + s0);
            }
            const D4 zs = zrow(row - d.z);
            const D4 zn = zrow(row + d.w);
            const double* ps = &zs.x;
            const double* pw = &zprev.x;
            const double* pc = &zcur.x;
            const double* pe = &znext.x;
            const double* pn = &zn.x;
            const double* cc = &c.x;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double p0 = 0.0;
                p0 += w.x * ps[q];
                p0 += w.x * pw[q];
                p0 += w.y * pc[q];
                p0 += w.x * pe[q];
                p0 += w.x * pn[q];
                acc[q] = cc[q] * p0;
            }
        } else {
            const int b = d.y, e = __ldg(a.row_ptr + row + 1);
            if (d.x >= 0) {
                const D4 c1 = ld4_nc(a.cells + (d.x & 0xffff) * S + s0);
                double p[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 2
                for (int q = b; q < e; ++q) {
                    const int j = __ldg(a.ent + q) & a.col_mask;
                    const double w = __ldg(a.a0 + q);
                    const D4 z = zrow(j);
                    p[0] += w * z.x;
                    p[1] += w * z.y;
                    p[2] += w * z.z;
                    p[3] += w * z.w;
                }
                acc[0] = c1.x * p[0];
                acc[1] = c1.y * p[1];
                acc[2] = c1.z * p[2];
                acc[3] = c1.w * p[3];
            } else {
#pragma unroll 2
                for (int q = b; q < e; ++q) {
                    const int pk = __ldg(a.ent + q);
                    const double w = __ldg(a.a0 + q);
                    const int j = pk & a.col_mask;
                    const int cell = ent_cell(nullptr, q, pk, a.col_bits);
                    const D4 c1 = ld4_nc(a.cells + cell * S + s0);
                    const D4 z = zrow(j);
                    acc[0] += (c1.x * w) * z.x;
                    acc[1] += (c1.y * w) * z.y;
                    acc[2] += (c1.z * w) * z.z;
                    acc[3] += (c1.w * w) * z.w;
                }
            }
        }
        if (row < a.split) {
            const D4 g{acc[0], acc[1], acc[2], acc[3]};
            if (a.g_node_major)
                st4(a.g + idx, g);
            else
                tile[warp * R + k][lane] = g;
        } else {
            D4 out;
            out.x = 2.0 * zcur.x - zm.x - f * acc[0];
            out.y = 2.0 * zcur.y - zm.y - f * acc[1];
            out.z = 2.0 * zcur.z - zm.z - f * acc[2];
            out.w = 2.0 * zcur.w - zm.w - f * acc[3];
            st4(a.zp + idx, out);
            // check_finite (integrators.cpp:12-18)
            if (!(fabs(out.x) <= 1e100)) flag_fail(a.fail, s0, a.count, a.step);
            if (!(fabs(out.y) <= 1e100)) flag_fail(a.fail, s0 + 1, a.count, a.step);
            if (!(fabs(out.z) <= 1e100)) flag_fail(a.fail, s0 + 2, a.count, a.step);
            if (!(fabs(out.w) <= 1e100)) flag_fail(a.fail, s0 + 3, a.count, a.step);
        }
        zprev = zcur;
        zcur = znext;
    }
    if (row0 >= a.split || a.g_node_major) return;  // block-uniform
    // the block's g rows sample-major: 128 samples x (kSweepWarps R) rows,
    // thread -> sample tid / 2, half the rows each
    __syncthreads();
    constexpr int kRows = kSweepWarps * R, kTpS = kSweepWarps * 32 / kSweepChunkW, kRpt = kRows / kTpS;
    const int sl = threadIdx.x / kTpS;
    const int r0 = (threadIdx.x % kTpS) * kRpt;
    const int s = chunk * kSweepChunkW + sl;
    double* dst = a.g + static_cast<std::size_t>(s) * a.g_stride + row0 + r0;
#pragma unroll
    for (int q = 0; q < kRpt; q += 2) {
        const double* t0 = &tile[r0 + q][sl >> 2].x;
        const double* t1 = &tile[r0 + q + 1][sl >> 2].x;
        const double g0 = t0[sl & 3], g1 = t1[sl & 3];
        if (row0 + r0 + q + 1 < a.split)
            *reinterpret_cast<double2*>(dst + q) = make_double2(g0, g1);
        else if (row0 + r0 + q < a.split)
            dst[q] = g0;
    }
}

// K2 (HBM-resident): one substep over the R rows, warp per (row, 64
// samples) as in the sweep; A(omega) P d gathered node-centrically from the
// current d buffer, d_{m+1} written over d_{m-1} (own row only), the last
// substep forms z_{n+1} directly (reference src/integrators.cpp:137-153).
template <int R>
__global__ void __launch_bounds__(kSweepWarps * 32, WMC_GSUB_MINB) global_substep_kernel(GSubArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int groups = (a.n_r + kSweepWarps * R - 1) / (kSweepWarps * R);
    const int first = (blockIdx.x % groups) * kSweepWarps * R + warp * R;
    if (first >= a.n_r) return;
    const int s0 = (blockIdx.x / groups) * kSweepChunk + 2 * lane;
    const std::size_t S = static_cast<std::size_t>(a.S);
    const double* src = a.cur_mode == 0 ? a.dcur : a.g;
    const double2 r = lane_rel(a.rel, s0);
    const double2 c0 = make_double2(a.c0 * r.x, a.c0 * r.y), cm = make_double2(a.cm * r.x, a.cm * r.y);
    const double2 scale = a.cur_mode == 0 ? make_double2(1.0, 1.0) : make_double2(-c0.x, -c0.y);
    const int2 live = lane_live(a.nsteps, s0, a.step);
    auto ld = [&](const double* p, int r) {
        return *reinterpret_cast<const double2*>(p + static_cast<std::size_t>(r) * S + s0);
    };
    // window src[i-1], src[i], src[i+1] over the warp's consecutive rows
    double2 vprev = first > 0 ? ld(src, first - 1) : make_double2(0.0, 0.0);
    double2 vcur = ld(src, first);
    int ccell = -1;
    double2 c = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int row = first + k;
        if (row >= a.n_r) break;
        const std::size_t idx = static_cast<std::size_t>(row) * S + s0;
        const double2 g = __ldg(reinterpret_cast<const double2*>(a.g + idx));
        double2 dm = make_double2(0.0, 0.0), dmm = make_double2(0.0, 0.0), zn = dm, zm = dm;
        if (a.cur_mode == 0) dm = vcur;
        if (a.prev_mode == 0) dmm = *reinterpret_cast<const double2*>(a.dprev + idx);
        if (a.last) {
            zn = *reinterpret_cast<const double2*>(a.zc + idx);
            zm = *reinterpret_cast<const double2*>(a.zp + idx);
        }
        const double2 vnext = row + 1 < a.n_r ? ld(src, row + 1) : make_double2(0.0, 0.0);
        double acc0 = 0.0, acc1 = 0.0;
        const int4 d = __ldg(a.row_desc + row);
        if (d.x >= 0 && (d.x >> 24) >= 1) {
            const double2 w = __ldg(a.wtype + ((d.x >> 16) & 0xff) - 1);
            if ((d.x & 0xffff) != ccell) {
                ccell = d.x & 0xffff;
                c = __ldg(reinterpret_cast<const double2*>(a.cells + ccell * S + s0));
            }
            const double2 vs = ld(src, row - d.z), vn = ld(src, row + d.w);
            double p0 = 0.0, p1 = 0.0;
            p0 += w.x * vs.x;
            p1 += w.x * vs.y;
            p0 += w.x * vprev.x;
            p1 += w.x * vprev.y;
            p0 += w.y * vcur.x;
            p1 += w.y * vcur.y;
            p0 += w.x * vnext.x;
            p1 += w.x * vnext.y;
            p0 += w.x * vn.x;
            p1 += w.x * vn.y;
            acc0 = c.x * p0;
            acc1 = c.y * p1;
        } else {
            const int b = __ldg(a.ptr + row), e = __ldg(a.ptr + row + 1);
#pragma unroll 4
            for (int q = b; q < e; ++q) {
                const int pk = __ldg(a.ent + q);
                const double w = __ldg(a.a0 + q);
                const int j = a.cell_ix ? pk : pk & kColMask;
                const int cell = a.cell_ix ? __ldg(a.cell_ix + q) : static_cast<int>(static_cast<unsigned>(pk) >> kColBits);
                const double2 cc = __ldg(reinterpret_cast<const double2*>(a.cells + cell * S + s0));
                const double2 v = ld(src, j);
                acc0 += (cc.x * w) * v.x;
                acc1 += (cc.y * w) * v.y;
            }
        }
        acc0 *= scale.x;
        acc1 *= scale.y;
        if (a.cur_mode != 0) dm = make_double2(-c0.x * g.x, -c0.y * g.y);
        if (a.prev_mode == 1) dmm = make_double2(-c0.x * g.x, -c0.y * g.y);
        double2 next;
        next.x = (1.0 + a.beta) * dm.x - a.beta * dmm.x - cm.x * (g.x + acc0);
        next.y = (1.0 + a.beta) * dm.y - a.beta * dmm.y - cm.y * (g.y + acc1);
        if (!a.last) {
            *reinterpret_cast<double2*>(a.dprev + idx) = next;
        } else {
            double2 out;
            out.x = 2.0 * zn.x - zm.x + 2.0 * next.x;
            out.y = 2.0 * zn.y - zm.y + 2.0 * next.y;
            store_z(a.zp + idx, out, live, a.fail, s0, a.count, a.step);
        }
        vprev = vcur;
        vcur = vnext;
    }
}

// Nested-tier stage (see TierArgs): the single-tier recursion of reference
// src/integrators.cpp:117-157 applied per tier, with the stage's right-hand
// side on R_k+1 replaced by the tier-(k+1) solve over the stage interval.
template <int R>
__global__ void __launch_bounds__(kSweepWarps * 32, WMC_TIER_MINB) tier_stage_kernel(TierArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nrows = a.row_end - a.row_begin;
    const int groups = (nrows + kSweepWarps * R - 1) / (kSweepWarps * R);
    const int first = a.row_begin + (blockIdx.x % groups) * kSweepWarps * R + warp * R;
    if (first >= a.row_end) return;
    const int s0 = (blockIdx.x / groups) * kSweepChunk + 2 * lane;
    const std::size_t S = static_cast<std::size_t>(a.S);
    const double* src = a.src;
    const double2 rr = lane_rel(a.rel, s0);
    auto ld = [&](const double* p, int r) {
        return *reinterpret_cast<const double2*>(p + static_cast<std::size_t>(r) * S + s0);
    };
    // window E_m[i-1], E_m[i], E_m[i+1] over the warp's consecutive rows
    double2 vprev = make_double2(0.0, 0.0), vcur = vprev;
    if (a.m > 0) {
        if (first > 0) vprev = ld(src, first - 1);
        vcur = ld(src, first);
    }
    int ccell = -1;
    double2 c = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int row = first + q;
        if (row >= a.row_end) break;
        const std::size_t idx = static_cast<std::size_t>(row) * S + s0;
        double2 v = __ldg(reinterpret_cast<const double2*>(a.rhs + idx));
        double2 vnext = make_double2(0.0, 0.0);
        if (a.m > 0) {
            if (row + 1 < a.row_end) vnext = ld(src, row + 1);
            double acc0 = 0.0, acc1 = 0.0;
            const int4 d = __ldg(a.row_desc + row);
            if (d.x >= 0 && (d.x >> 24) >= a.k) {
                const double2 w = __ldg(a.wtype + ((d.x >> 16) & 0xff) - 1);
                if ((d.x & 0xffff) != ccell) {
                    ccell = d.x & 0xffff;
                    c = __ldg(reinterpret_cast<const double2*>(a.cells + ccell * S + s0));
                }
                const double2 vs = ld(src, row - d.z), vn = ld(src, row + d.w);
                double p0 = 0.0, p1 = 0.0;
                p0 += w.x * vs.x;
                p1 += w.x * vs.y;
                p0 += w.x * vprev.x;
                p1 += w.x * vprev.y;
                p0 += w.y * vcur.x;
                p1 += w.y * vcur.y;
                p0 += w.x * vnext.x;
                p1 += w.x * vnext.y;
                p0 += w.x * vn.x;
                p1 += w.x * vn.y;
                acc0 = c.x * p0;
                acc1 = c.y * p1;
            } else {
                const int b = __ldg(a.ptr + row), e = __ldg(a.ptr + row + 1);
#pragma unroll 4
                for (int t = b; t < e; ++t) {
                    const int pk = __ldg(a.ent + t);
                    const double w = __ldg(a.a0 + t);
                    const int j = pk & kColMask;
                    const int cell = static_cast<unsigned>(pk) >> kColBits;
                    const double2 cc = __ldg(reinterpret_cast<const double2*>(a.cells + cell * S + s0));
                    const double2 x = ld(src, j);
                    acc0 += (cc.x * w) * x.x;
                    acc1 += (cc.y * w) * x.y;
                }
            }
            v.x += acc0;
            v.y += acc1;
        }
        const double2 em_row = vcur;  // E^k_m of this row (m > 0)
        vprev = vcur;
        vcur = vnext;
        if (row < a.split) {
            *reinterpret_cast<double2*>(a.rhs_next + idx) = v;
            continue;
        }
        // the tier's update, then up through the ancestors whose stage ends here
#pragma unroll
        for (int t = 0; t < kMaxTiers; ++t) {
            if (t >= a.depth) break;
            const auto& L = a.link[t];
            double2 em = make_double2(0.0, 0.0), emm = em;
            if (t == 0) {
                em = em_row;
            } else if (L.em) {
                em = *reinterpret_cast<const double2*>(L.em + idx);
            }
            if (L.emm) emm = *reinterpret_cast<const double2*>(L.emm + idx);
            double2 en;
            en.x = L.A * em.x - L.B * emm.x - (L.C * rr.x) * v.x;
            en.y = L.A * em.y - L.B * emm.y - (L.C * rr.y) * v.y;
            if (t + 1 < a.depth) {
                v = make_double2((L.back / rr.x) * en.x, (L.back / rr.y) * en.y);
                continue;
            }
            if (L.out) {
                *reinterpret_cast<double2*>(L.out + idx) = en;
            } else {
                const double2 zn = *reinterpret_cast<const double2*>(a.zc + idx);
                const double2 zm = *reinterpret_cast<const double2*>(a.zp + idx);
                double2 out;
                out.x = 2.0 * zn.x - zm.x + 2.0 * en.x;
                out.y = 2.0 * zn.y - zm.y + 2.0 * en.y;
                store_z(a.zp + idx, out, lane_live(a.nsteps, s0, a.step), a.fail, s0, a.count, a.step);
            }
        }
    }
}

// Nested-tier stage, wide form (fixed dt, S a multiple of 128): four samples
// per lane with 256-bit loads and stores like sweep_wide_kernel, the same
// per-sample products and sums as tier_stage_kernel.
template <int R, int MINB>
__global__ void __launch_bounds__(kSweepWarps * 32, MINB) tier_stage_wide_kernel(TierArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nrows = a.row_end - a.row_begin;
    const int groups = (nrows + kSweepWarps * R - 1) / (kSweepWarps * R);
    const int first = a.row_begin + (blockIdx.x % groups) * kSweepWarps * R + warp * R;
    if (first >= a.row_end) return;
    const int s0 = (blockIdx.x / groups) * kSweepChunkW + 4 * lane;
    const std::size_t S = static_cast<std::size_t>(a.S);
    const double* src = a.src;
    auto at = [&](const double* p, int r) { return p + static_cast<std::size_t>(r) * S + s0; };
    const D4 zero{0.0, 0.0, 0.0, 0.0};
    // window E_m[i-1], E_m[i], E_m[i+1] over the warp's consecutive rows
    D4 vprev = zero, vcur = zero;
    if (a.m > 0) {
        if (first > 0) vprev = ld4(at(src, first - 1));
        vcur = ld4(at(src, first));
    }
    int ccell = -1;
    D4 c = zero;
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int row = first + q;
        if (row >= a.row_end) break;
        const std::size_t idx = static_cast<std::size_t>(row) * S + s0;
        D4 v = ld4_nc(a.rhs + idx);
        D4 vnext = zero;
        if (a.m > 0) {
            if (row + 1 < a.row_end) vnext = ld4(at(src, row + 1));
            D4 acc = zero;
            const int4 d = __ldg(a.row_desc + row);
            if (d.x >= 0 && (d.x >> 24) >= a.k) {
                const double2 w = __ldg(a.wtype + ((d.x >> 16) & 0xff) - 1);
                if ((d.x & 0xffff) != ccell) {
                    ccell = d.x & 0xffff;
                    c = ld4_nc(a.cells + ccell * S + s0);
                }
                const D4 vs = ld4(at(src, row - d.z)), vn = ld4(at(src, row + d.w));
#define WMC_TIER_STRUCT(F)          \
    {                               \
        double p0 = 0.0;            \
        p0 += w.x * vs.F;           \
        p0 += w.x * vprev.F;        \
        p0 += w.y * vcur.F;         \
        p0 += w.x * vnext.F;        \
        p0 += w.x * vn.F;           \
        acc.F = c.F * p0;           \
    }
                WMC_TIER_STRUCT(x) WMC_TIER_STRUCT(y) WMC_TIER_STRUCT(z) WMC_TIER_STRUCT(w)
#undef WMC_TIER_STRUCT
            } else {
                const int b = __ldg(a.ptr + row), e = __ldg(a.ptr + row + 1);
#pragma unroll 2
                for (int t = b; t < e; ++t) {
                    const int pk = __ldg(a.ent + t);
                    const double w = __ldg(a.a0 + t);
                    const int j = pk & kColMask;
                    const int cell = static_cast<unsigned>(pk) >> kColBits;
                    const D4 cc = ld4_nc(a.cells + cell * S + s0);
                    const D4 x = ld4(at(src, j));
                    acc.x += (cc.x * w) * x.x;
                    acc.y += (cc.y * w) * x.y;
                    acc.z += (cc.z * w) * x.z;
                    acc.w += (cc.w * w) * x.w;
                }
            }
            v.x += acc.x;
            v.y += acc.y;
            v.z += acc.z;
            v.w += acc.w;
        }
        const D4 em_row = vcur;  // E^k_m of this row (m > 0)
        vprev = vcur;
        vcur = vnext;
        if (row < a.split) {
            st4(a.rhs_next + idx, v);
            continue;
        }
        // the tier's update, then up through the ancestors whose stage ends here
#pragma unroll
        for (int t = 0; t < kMaxTiers; ++t) {
            if (t >= a.depth) break;
            const auto& L = a.link[t];
            D4 em = zero, emm = zero;
            if (t == 0) {
                em = em_row;
            } else if (L.em) {
                em = ld4(L.em + idx);
            }
            if (L.emm) emm = ld4(L.emm + idx);
            D4 en;
            en.x = L.A * em.x - L.B * emm.x - (L.C * 1.0) * v.x;
            en.y = L.A * em.y - L.B * emm.y - (L.C * 1.0) * v.y;
            en.z = L.A * em.z - L.B * emm.z - (L.C * 1.0) * v.z;
            en.w = L.A * em.w - L.B * emm.w - (L.C * 1.0) * v.w;
            if (t + 1 < a.depth) {
                v = D4{L.back * en.x, L.back * en.y, L.back * en.z, L.back * en.w};
                continue;
            }
            if (L.out) {
                st4(L.out + idx, en);
            } else {
                const D4 zn = ld4(a.zc + idx), zm = ld4(a.zp + idx);
                D4 out;
                out.x = 2.0 * zn.x - zm.x + 2.0 * en.x;
                out.y = 2.0 * zn.y - zm.y + 2.0 * en.y;
                out.z = 2.0 * zn.z - zm.z + 2.0 * en.z;
                out.w = 2.0 * zn.w - zm.w + 2.0 * en.w;
                st4(a.zp + idx, out);
                // check_finite (integrators.cpp:12-18)
                if (!(fabs(out.x) <= 1e100)) flag_fail(a.fail, s0, a.count, a.step);
                if (!(fabs(out.y) <= 1e100)) flag_fail(a.fail, s0 + 1, a.count, a.step);
                if (!(fabs(out.z) <= 1e100)) flag_fail(a.fail, s0 + 2, a.count, a.step);
                if (!(fabs(out.w) <= 1e100)) flag_fail(a.fail, s0 + 3, a.count, a.step);
            }
        }
    }
}

// R update: z_{n+1} = 2 z_n - z_{n-1} + 2 d_p on rows < n_r, d_p read
// sample-major and transposed through shared memory (mirror of the sweep's
// g store), then one warp per (row, 64 samples) as in the sweep.
__global__ void __launch_bounds__(kSweepWarps * 32) r_update_kernel(RUpdateArgs a) {
    __shared__ double2 tile[kSweepWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row0 = grid_rowgroup(a.n_r) * kSweepWarps;
    {
        const int sl = 8 * warp + (lane >> 2), rr = 2 * (lane & 3);
        const int s = grid_chunk(a.n_r) * kSweepChunk + sl;
        const double* src = a.gd + static_cast<std::size_t>(s) * a.g_stride + row0 + rr;
        double d0 = 0.0, d1 = 0.0;
        if (row0 + rr + 1 < a.n_r) {
            const double2 v = *reinterpret_cast<const double2*>(src);
            d0 = v.x;
            d1 = v.y;
        } else if (row0 + rr < a.n_r) {
            d0 = src[0];
        }
        double* t = reinterpret_cast<double*>(&tile[0][0]);
        t[(rr * 32 + (sl >> 1)) * 2 + (sl & 1)] = d0;
        t[((rr + 1) * 32 + (sl >> 1)) * 2 + (sl & 1)] = d1;
    }
    __syncthreads();
    const int row = row0 + warp;
    if (row >= a.n_r) return;
    const int s0 = grid_chunk(a.n_r) * kSweepChunk + 2 * lane;
    const std::size_t idx = static_cast<std::size_t>(row) * a.S + s0;
    const double2 d = tile[warp][lane];
    const double2 zn = *reinterpret_cast<const double2*>(a.zc + idx);
    const double2 zm = *reinterpret_cast<const double2*>(a.zp + idx);
    double2 out;
    out.x = 2.0 * zn.x - zm.x + 2.0 * d.x;
    out.y = 2.0 * zn.y - zm.y + 2.0 * d.y;
    store_z(a.zp + idx, out, lane_live(a.nsteps, s0, a.step), a.fail, s0, a.count, a.step);
}

// ---------------------------------------------------------------------------
// K2: the p LTS substeps on the compact set R, one sample per CTA at a time
// (persistent over samples).  State of the sample on R stays on chip for all
// p substeps: d_m double-buffered in shared memory (neighbours read it),
// d_{m-1} and g in registers of the owning thread.  A P on R is a sliced
// ELL (32 rows per slice) of 32-bit entries col | wid << 16 in shared memory,
// loaded once per CTA; the per-sample weights W[wid] = sum c_k a0_k are built
// in shared memory per sample.  Deviation form of reference
// src/integrators.cpp:117-157:
//   d_1 = -c0 g,  d_{m+1} = (1+b_m) d_m - b_m d_{m-1} - c_m (g + A P d_m),
//   z+ = 2 z - z- + 2 d_p.

struct SubSmem {
    double* W;
    double* d0;
    double* d1;
    double* beta;
    double* cm;
    double* cl;
    int* soff;
    std::uint32_t* ent;
};

__host__ __device__ inline std::size_t align16(std::size_t v) { return (v + 15) & ~std::size_t(15); }

__host__ __device__ inline std::size_t sub_layout(const SubArgs& a, char* base, SubSmem* s) {
    const int n_slices = (a.n_r + 31) / 32;
    std::size_t off = 0;
    auto take = [&](std::size_t bytes) {
        const std::size_t o = off;
        off = align16(off + bytes);
        return o;
    };
    const std::size_t oW = take(sizeof(double) * (a.n_wid + 1));
    const std::size_t o0 = take(sizeof(double) * a.n_r);
    const std::size_t o1 = take(sizeof(double) * a.n_r);
    const std::size_t ob = take(sizeof(double) * (a.p > 1 ? a.p - 1 : 1));
    const std::size_t oc = take(sizeof(double) * (a.p > 1 ? a.p - 1 : 1));
    const std::size_t ol = take(sizeof(double) * (a.cl_smem ? a.n_cells : 0));
    const std::size_t os = take(sizeof(int) * (n_slices + 1));
    const std::size_t oe = take(sizeof(std::uint32_t) * a.n_ent);
    if (s) {
        s->W = reinterpret_cast<double*>(base + oW);
        s->d0 = reinterpret_cast<double*>(base + o0);
        s->d1 = reinterpret_cast<double*>(base + o1);
        s->beta = reinterpret_cast<double*>(base + ob);
        s->cm = reinterpret_cast<double*>(base + oc);
        s->cl = reinterpret_cast<double*>(base + ol);
        s->soff = reinterpret_cast<int*>(base + os);
        s->ent = reinterpret_cast<std::uint32_t*>(base + oe);
    }
    return off;
}

template <int RPT>
__global__ void __launch_bounds__(kSubThreads, 1) substep_kernel(SubArgs a) {
    extern __shared__ __align__(16) char smem[];
    SubSmem sm;
    sub_layout(a, smem, &sm);
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int n_slices = (a.n_r + 31) / 32;
    const std::size_t S = static_cast<std::size_t>(a.S);

    for (int i = tid; i < a.n_ent; i += kSubThreads) sm.ent[i] = __ldg(a.ent + i);
    for (int i = tid; i <= n_slices; i += kSubThreads) sm.soff[i] = __ldg(a.slice_off + i);
    for (int i = tid; i < a.p - 1; i += kSubThreads) {
        sm.beta[i] = __ldg(a.beta + i);
        sm.cm[i] = __ldg(a.cm + i);
    }
    if (tid == 0) sm.W[a.n_wid] = 0.0;  // padding entries

    for (int s = blockIdx.x; s < a.count; s += gridDim.x) {
        // per-sample CFL: finished samples are left alone, dt^2 constants scale
        if (a.nsteps && a.step > __ldg(a.nsteps + s)) continue;
        const double rs = a.rel ? __ldg(a.rel + s) : 1.0;
        __syncthreads();  // previous sample done with cl / W / d buffers
        if (a.cl_smem) {
            for (int k = tid; k < a.n_cells; k += kSubThreads) sm.cl[k] = __ldg(a.cells + k * S + s);
            __syncthreads();
        }
        for (int w = tid; w < a.n_wid; w += kSubThreads) {
            double acc = 0.0;
            for (int t = __ldg(a.rc_ptr + w); t < __ldg(a.rc_ptr + w + 1); ++t) {
                const int k = __ldg(a.rc_cell + t);
                acc += (a.cl_smem ? sm.cl[k] : __ldg(a.cells + k * S + s)) * __ldg(a.rc_a0 + t);
            }
            sm.W[w] = acc;
        }

        double g[RPT], dc[RPT], dp[RPT];
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int r = tid + k * kSubThreads;
            g[k] = 0.0;
            dc[k] = 0.0;
            dp[k] = 0.0;
            if (r < a.n_r) {
                g[k] = a.gd[static_cast<std::size_t>(s) * a.g_stride + r];
                dc[k] = -(a.c0 * rs) * g[k];
                sm.d0[r] = dc[k];
            }
        }
        __syncthreads();

        for (int m = 1; m <= a.p - 1; ++m) {
            const double* cur = (m & 1) ? sm.d0 : sm.d1;
            double* nxt = (m & 1) ? sm.d1 : sm.d0;
            const double beta = sm.beta[m - 1];
            const double cm = sm.cm[m - 1] * rs;
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const int r = tid + k * kSubThreads;
                if (r < a.n_r) {
                    const int slice = warp + k * (kSubThreads / 32);
                    const int b = sm.soff[slice], e = sm.soff[slice + 1];
                    double aq = 0.0;
                    for (int q = b + lane; q < e; q += 32) {
                        const std::uint32_t pk = sm.ent[q];
                        aq += sm.W[pk >> 16] * cur[pk & 0xffffu];
                    }
                    const double next = (1.0 + beta) * dc[k] - beta * dp[k] - cm * (g[k] + aq);
                    dp[k] = dc[k];
                    dc[k] = next;
                    nxt[r] = next;
                }
            }
            __syncthreads();
        }

#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int r = tid + k * kSubThreads;
            if (r < a.n_r) a.gd[static_cast<std::size_t>(s) * a.g_stride + r] = dc[k];  // d_p, coalesced
        }
    }
    (void)n_slices;
}


// ---------------------------------------------------------------------------
// K2 (structured): the p LTS substeps on R with the refined-square lattice
// as a register-blocked 5-point stencil.  Thread t owns column i = 1 + t % cw
// of strip t / cw (<= kLatStrip consecutive rows of L = [1, m-1]^2), keeping
// d_m, d_{m-1}, g and v = d / h of its nodes in registers; N/S neighbours
// inside the strip come from registers, E/W and the strip ends from the
// shared-memory copy of v (double-buffered, one barrier per substep).
// Edge conductances kappa = (c_a + c_b)/2 come from the sample's cell
// coefficients; a coefficient line always starts a strip, so a thread needs
// one set of constants for its first row and one for the rest.
// Generic rows (box ring + transition belt) use a SELL of per-sample
// weights w_ij = A_ij(omega) sqrt(M_j) acting on v.

// Generic SELL row of the lattice kernels: sum_e w_e v[col_e] over the
// slice's 2 NP slots, odd slots into a second chain, widest slot first.
// Slots are stored in pairs ([slice][pair][lane][2]; q0 = slice offset + 2
// lane): one 16-byte load brings a pair's weights, one 32-bit load its two
// columns.  One straight-line block per width (selected by a warp-uniform
// switch) so the slot loads issue back to back.
template <int NP>
__device__ __forceinline__ double gen_gather(const double* __restrict__ sd, int ogw, int cur,
                                             const std::uint16_t* __restrict__ gcol, int q0) {
    const unsigned* gc2 = reinterpret_cast<const unsigned*>(gcol);
    double acc = 0.0, acc2 = 0.0;
#pragma unroll
    for (int p = NP - 1; p >= 0; --p) {
        const double2 w = *reinterpret_cast<const double2*>(sd + ogw + q0 + 64 * p);
        const unsigned c = gc2[(q0 + 64 * p) >> 1];
        acc2 += w.y * sd[cur + (c >> 16)];
        acc += w.x * sd[cur + (c & 0xffffu)];
    }
    return acc + acc2;
}

__device__ __forceinline__ double gen_gather_w(int wd, const double* __restrict__ sd, int ogw, int cur,
                                               const std::uint16_t* __restrict__ gcol, int q0) {
    switch (wd) {
        case 8: return gen_gather<4>(sd, ogw, cur, gcol, q0);
        case 6: return gen_gather<3>(sd, ogw, cur, gcol, q0);
        case 4: return gen_gather<2>(sd, ogw, cur, gcol, q0);
        case 2: return gen_gather<1>(sd, ogw, cur, gcol, q0);
        default: return 0.0;
    }
}

// Shared-memory layout of the lattice kernel, in units of doubles from the
// dynamic shared base (integer offsets keep every access a 32-bit shared
// address): v0 | v1 | gw | sa0 | cl | beta | cm | then 8-byte aligned int
// and byte tables.
struct LatOff {
    int v0, v1, gw, sa0, cl, beta, cm, oa0, gcol, scell, ostart, ocell, sj0, slen, cx, cy, total;
};

__host__ __device__ inline LatOff lat_offsets(const LatArgs& a) {
    LatOff o;
    int off = 0;
    auto take = [&](int doubles) {
        const int r = off;
        off += (doubles + 1) & ~1;  // keep 16-byte alignment
        return r;
    };
    const int slots = a.n_slots > 0 ? a.n_slots : 1;
    o.v0 = take(a.n_r + 16);  // rows past a short strip read (never write) up to 8 beyond
    o.v1 = take(a.n_r + 16);
    o.gw = take(slots);
    o.sa0 = take(slots);
    o.cl = take(a.n_cells);
    o.beta = take(a.p > 1 ? a.p - 1 : 1);
    o.cm = take(a.p > 1 ? a.p - 1 : 1);
    o.oa0 = take(a.n_ovf_terms > 0 ? a.n_ovf_terms : 1);
    o.gcol = take((slots * 2 + 7) / 8);  // uint16
    o.scell = take((slots * 2 + 7) / 8);  // uint16
    o.ostart = take((a.n_ovf + 1 + 1) / 2);  // int
    o.ocell = take((a.n_ovf_terms * 2 + 7) / 8);  // uint16
    o.sj0 = take((a.n_strips + 1) / 2);  // int
    o.slen = take((a.n_strips + 1) / 2);
    o.cx = take((a.m + 1) / 2);
    o.cy = take((a.m + 1) / 2);
    o.total = off;
    return o;
}

// K2 (structured): the p LTS substeps on R with the refined-square lattice
// as a register-blocked 5-point stencil.  Thread t owns column i = 1 + t % cw
// of strip t / cw (<= K consecutive rows of L = [1, m-1]^2), keeping d_m,
// d_{m-1} and g of its nodes in registers; N/S neighbours inside the strip
// come from registers, E/W and the strip ends from the shared-memory copy
// of v = d / sqrt(M) (double-buffered, one barrier per substep).  Edge
// conductances kappa = (c_a + c_b)/2 come from the sample's cell
// coefficients; a coefficient line always starts a strip, so a thread needs
// one set of constants for its first row and one for the rest.  Generic rows
// (box ring + transition belt, G per thread) use a SELL of per-sample
// weights w_ij = A_ij(omega) sqrt(M_j) on v; rows are sorted by length and
// each warp-wide slice is padded to its widest row, the gather is predicated
// straight-line code.  Rows past a short strip compute on
// clamped addresses and never store.
template <int T, int K, int G>
__global__ void __launch_bounds__(T, 1) lattice_substep_kernel(LatArgs a) {
    extern __shared__ __align__(16) double sd[];
    const LatOff o = lat_offsets(a);
    std::uint16_t* gcol = reinterpret_cast<std::uint16_t*>(sd + o.gcol);
    std::uint16_t* scell = reinterpret_cast<std::uint16_t*>(sd + o.scell);
    int* ostart = reinterpret_cast<int*>(sd + o.ostart);
    std::uint16_t* ocell = reinterpret_cast<std::uint16_t*>(sd + o.ocell);
    int* sj0 = reinterpret_cast<int*>(sd + o.sj0);
    int* slen = reinterpret_cast<int*>(sd + o.slen);
    int* cx = reinterpret_cast<int*>(sd + o.cx);
    int* cy = reinterpret_cast<int*>(sd + o.cy);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const std::size_t S = static_cast<std::size_t>(a.S);
    const int W = a.m + 1;
    const int nr = a.n_r;
    const double inv_h = a.inv_h;
    const double hh = 1.0 / inv_h;

    // static tables, once per CTA
    for (int i = tid; i < a.n_slots; i += T) {
        gcol[i] = __ldg(a.gen_col + i);
        scell[i] = __ldg(a.slot_cell + i);
        sd[o.sa0 + i] = __ldg(a.slot_a0 + i);
    }
    for (int i = tid; i <= a.n_ovf; i += T) ostart[i] = __ldg(a.ovf_start + i);
    for (int i = tid; i < a.n_ovf_terms; i += T) {
        ocell[i] = __ldg(a.ovf_cell + i);
        sd[o.oa0 + i] = __ldg(a.ovf_a0 + i);
    }
    for (int i = tid; i < a.n_strips; i += T) {
        sj0[i] = __ldg(a.strip_j0 + i);
        slen[i] = __ldg(a.strip_len + i);
    }
    for (int i = tid; i < a.m; i += T) {
        cx[i] = __ldg(a.cellx + i);
        cy[i] = __ldg(a.celly + i);
    }
    for (int i = tid; i < a.p - 1; i += T) {
        sd[o.beta + i] = __ldg(a.beta + i);
        sd[o.cm + i] = __ldg(a.cm + i);
    }

    // structured role: column ci of strip `strip`
    const int col = tid % a.cw, strip = tid / a.cw;
    const int ci = 1 + col;
    const bool lat_on = ci <= a.m - 1 && strip < a.n_strips;
    // generic role: the warp's u-th 32-row slice from the host's balanced
    // assignment (widest slices spread over the warps), slots [slice][width][32]
    int grow[G], gslot[G], gwid[G];
    double grs[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
        const int wsl = __ldg(a.gen_warp_slice + (tid >> 5) * G + u);
        const int q = wsl >= 0 ? wsl * 32 + lane : a.n_gen;
        grow[u] = q < a.n_gen ? __ldg(a.gen_rows + q) : -1;
        grs[u] = q < a.n_gen ? __ldg(a.gen_rs + q) : 0.0;
        const int sl = wsl >= 0 ? wsl : 0;  // idle warps point at slice 0 with width 0
        gslot[u] = __ldg(a.gen_soff + sl) + 2 * lane;
        gwid[u] = wsl >= 0 ? (__ldg(a.gen_soff + sl + 1) - __ldg(a.gen_soff + sl)) >> 5 : 0;
    }
    __syncthreads();
    // column-major box: the strip's nodes are base .. base + len - 1.  Idle
    // lanes of a strip (columns past m - 1) shadow its last column: their
    // loads hit the same addresses (a broadcast, not a bank conflict); they
    // never store (len 0).  Threads past the last strip point at node (1, 1).
    const bool shadow = !lat_on && strip < a.n_strips;
    int j0 = 1, len = 0, span = 0;
    if (lat_on || shadow) {
        j0 = sj0[strip];
        span = slen[strip];
    }
    if (lat_on) len = span;
    const int base = (lat_on || shadow) ? (lat_on ? ci : a.m - 1) * W + j0 : W + 1;

    for (int s = blockIdx.x; s < a.count; s += gridDim.x) {
        // per-sample CFL: finished samples are left alone, dt^2 constants scale
        if (a.nsteps && a.step > __ldg(a.nsteps + s)) continue;
        const double rs = a.rel ? __ldg(a.rel + s) : 1.0;
        // ---- per-sample set-up: g staged coalesced into v1, coefficients,
        // generic weights
        double* gdrow = a.gd + static_cast<std::size_t>(s) * a.g_stride;
        for (int r = tid; r < nr; r += T) sd[o.v1 + r] = gdrow[r];
        for (int k = tid; k < a.n_cells; k += T) sd[o.cl + k] = __ldg(a.cells + k * S + s);
        __syncthreads();
        double gg[K], ggg[G];
#pragma unroll
        for (int k = 0; k < K; ++k) gg[k] = k < len ? sd[o.v1 + base + k] : 0.0;
#pragma unroll
        for (int u = 0; u < G; ++u) ggg[u] = grow[u] >= 0 ? sd[o.v1 + grow[u]] : 0.0;
        for (int e = tid; e < a.n_slots; e += T) {
            const unsigned c = scell[e];
            double w;
            if (!(c & kOvfFlag)) {
                w = sd[o.cl + c] * sd[o.sa0 + e];
            } else {  // several cells share this entry (edge on a coefficient line)
                const int k = c & ~kOvfFlag;
                w = 0.0;
                for (int t = ostart[k]; t < ostart[k + 1]; ++t) w += sd[o.cl + ocell[t]] * sd[o.oa0 + t];
            }
            sd[o.gw + e] = w;
        }
        // edge conductances of this thread's column, scaled by 1/h (v = d/h):
        // squares right (column ci) and left (ci - 1) of the strip, all in
        // the strip's coefficient row
        double kE = 0, kW = 0, kNS = 0, dg = 0;
        if (lat_on) {
            const int row = o.cl + cy[j0] * a.cells_x;
            const double cR = sd[row + cx[ci]], cL = sd[row + cx[ci - 1]];
            kE = cR * inv_h;
            kW = cL * inv_h;
            kNS = (cL + cR) * (0.5 * inv_h);
            dg = kE + kW + 2.0 * kNS;
        }
        // d_{m-1} of a lattice node is not kept in registers: it is the value
        // the node published one substep ago, still in the buffer this
        // substep overwrites (read just before the write; d_0 = 0)
        double d[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            d[k] = -(a.c0 * rs) * gg[k];
            if (k < len) sd[o.v0 + base + k] = d[k] * inv_h;
        }
        double gd[G], gdp[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
            gdp[u] = 0.0;
            gd[u] = -(a.c0 * rs) * ggg[u];
            if (grow[u] >= 0) sd[o.v0 + grow[u]] = gd[u] * grs[u];
        }
        __syncthreads();

        // ---- p - 1 substeps, state on chip
        const int sS = (lat_on || shadow) ? base - 1 : 0, sN = (lat_on || shadow) ? base + span : 0;
        for (int m = 1; m <= a.p - 1; ++m) {
            const int cur = (m & 1) ? o.v0 : o.v1;
            const int nxt = (m & 1) ? o.v1 : o.v0;
            const double beta = sd[o.beta + m - 1];
            const double cmm = sd[o.cm + m - 1] * rs;
            const double onepb = 1.0 + beta;
            double gaq[G];
#pragma unroll
            for (int u = 0; u < G; ++u) {
                gaq[u] = gen_gather_w(gwid[u], sd, o.gw, cur, gcol, gslot[u]);
            }
            const int ce = cur + base + W, cw_ = cur + base - W;
            const double vnl = sd[cur + sN];
            double vs = sd[cur + sS];
            double vk = d[0] * inv_h;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const double ve = sd[ce + k], vw = sd[cw_ + k];
                const double vn = (k + 1 < len) ? d[k + 1] * inv_h : vnl;
                const double aq = dg * vk - kE * ve - kW * vw - kNS * (vn + vs);
                const double dpk = m == 1 ? 0.0 : sd[nxt + base + k] * hh;
                const double next = onepb * d[k] - beta * dpk - cmm * (gg[k] + aq);
                d[k] = next;
                if (k < len) sd[nxt + base + k] = next * inv_h;
                vs = vk;
                vk = vn;
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const double next = onepb * gd[u] - beta * gdp[u] - cmm * (ggg[u] + gaq[u]);
                gdp[u] = gd[u];
                gd[u] = next;
                if (grow[u] >= 0) sd[nxt + grow[u]] = next * grs[u];
            }
            __syncthreads();
        }

        // ---- d_p out, staged through v0 for a coalesced store (the R update
        // kernel forms z_{n+1})
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (k < len) sd[o.v0 + base + k] = d[k];
#pragma unroll
        for (int u = 0; u < G; ++u)
            if (grow[u] >= 0) sd[o.v0 + grow[u]] = gd[u];
        __syncthreads();
        for (int r = tid; r < nr; r += T) gdrow[r] = sd[o.v0 + r];
        __syncthreads();  // cl / gw / v buffers are rewritten for the next sample
    }
}

// ---------------------------------------------------------------------------
// K4: per-sample CFL step.  Power iteration of reference max_eigenvalue
// (src/fem.cpp:132-175) for every sample of the batch at once: av = A(omega) v
// (coarse: v masked on P, rows in P zeroed, :177-189), per-sample Rayleigh
// quotient and |av| from fixed-order partial sums, the stopping rule
// |r - r_prev| <= tol |r| three times in a row, v = av / |av|.

__global__ void eig_init_kernel(const double* __restrict__ warm, double warm_norm, int n, int S, double* v) {
    const std::size_t total = static_cast<std::size_t>(n) * S;
    for (std::size_t q = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; q < total;
         q += static_cast<std::size_t>(gridDim.x) * blockDim.x)
        v[q] = __ldg(warm + q / S) / warm_norm;
}

__global__ void __launch_bounds__(kSweepWarps * 32) eig_matvec_kernel(EigArgs a) {
    const int lane = threadIdx.x & 31;
    const int row = grid_rowgroup(a.n) * kSweepWarps + (threadIdx.x >> 5);
    if (row >= a.n) return;
    const int s0 = grid_chunk(a.n) * kSweepChunk + 2 * lane;
    const std::size_t S = static_cast<std::size_t>(a.S);
    double acc0 = 0.0, acc1 = 0.0;
    if (!(a.coarse && __ldg(a.in_p + row))) {
        const int b = __ldg(a.row_ptr + row), e = __ldg(a.row_ptr + row + 1);
        for (int k = b; k < e; ++k) {
            const int pk = __ldg(a.ent + k);
            const int j = pk & a.col_mask;
            if (a.coarse && __ldg(a.in_p + j)) continue;
            const double w = __ldg(a.a0 + k);
            const int cell = ent_cell(a.cell_ix, k, pk, a.col_bits);
            const double2 c = __ldg(reinterpret_cast<const double2*>(a.cells + cell * S + s0));
            const double2 x = __ldg(reinterpret_cast<const double2*>(a.v + j * S + s0));
            acc0 += (c.x * w) * x.x;
            acc1 += (c.y * w) * x.y;
        }
    }
    *reinterpret_cast<double2*>(a.av + static_cast<std::size_t>(row) * S + s0) = make_double2(acc0, acc1);
}

// partial sums of v.av and av.av over row block blockIdx.y, 64 samples per
// block (2 per lane), rows of the block strided over its 8 warps
__global__ void __launch_bounds__(kSweepWarps * 32) eig_dot_kernel(EigArgs a) {
    __shared__ double2 red[2][kSweepWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s0 = blockIdx.x * kSweepChunk + 2 * lane;
    const std::size_t S = static_cast<std::size_t>(a.S);
    const int rows_per = (a.n + a.n_blocks - 1) / a.n_blocks;
    const int r0 = blockIdx.y * rows_per, r1 = min(a.n, r0 + rows_per);
    double2 va = make_double2(0.0, 0.0), aa = va;
    for (int r = r0 + warp; r < r1; r += kSweepWarps) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(a.v + r * S + s0));
        const double2 x = __ldg(reinterpret_cast<const double2*>(a.av + r * S + s0));
        va.x += v.x * x.x;
        va.y += v.y * x.y;
        aa.x += x.x * x.x;
        aa.y += x.y * x.y;
    }
    red[0][warp][lane] = va;
    red[1][warp][lane] = aa;
    __syncthreads();
    if (warp == 0) {
        for (int w = 1; w < kSweepWarps; ++w) {
            va.x += red[0][w][lane].x;
            va.y += red[0][w][lane].y;
            aa.x += red[1][w][lane].x;
            aa.y += red[1][w][lane].y;
        }
        double* p0 = a.part + static_cast<std::size_t>(blockIdx.y) * S + s0;
        double* p1 = a.part + (static_cast<std::size_t>(a.n_blocks) + blockIdx.y) * S + s0;
        *reinterpret_cast<double2*>(p0) = va;
        *reinterpret_cast<double2*>(p1) = aa;
    }
}

__global__ void eig_update_kernel(EigArgs a) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= a.S || a.done[s]) return;
    const std::size_t S = static_cast<std::size_t>(a.S);
    double ray = 0.0, nn = 0.0;
    for (int b = 0; b < a.n_blocks; ++b) {
        ray += a.part[static_cast<std::size_t>(b) * S + s];
        nn += a.part[(static_cast<std::size_t>(a.n_blocks) + b) * S + s];
    }
    const double av_norm = sqrt(nn);
    a.iters[s] += 1;
    if (av_norm == 0.0) {  // zero operator
        a.lam[s] = 0.0;
        a.done[s] = 2;
        return;
    }
    a.norm[s] = av_norm;
    if (fabs(ray - a.lam_prev[s]) <= a.tol * fabs(ray)) {
        if (++a.settled[s] >= 3) {
            a.lam[s] = ray;
            a.done[s] = 1;
            return;
        }
    } else {
        a.settled[s] = 0;
    }
    a.lam_prev[s] = ray;
    atomicAdd(a.active_count, 1);
}

__global__ void eig_normalize_kernel(EigArgs a) {
    const std::size_t total = static_cast<std::size_t>(a.n) * a.S;
    double* v = const_cast<double*>(a.v);
    for (std::size_t q = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; q < total;
         q += static_cast<std::size_t>(gridDim.x) * blockDim.x) {
        const int s = static_cast<int>(q % a.S);
        if (!a.done[s]) v[q] = a.av[q] / a.norm[s];
    }
}

__global__ void cfl_finalize_kernel(const double* lf, const double* lc, int use_coarse, int p_fine, double safety,
                                    double T, double dt_ref, int count, int S, double* rel, int* nsteps) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    if (s >= count) {  // padding lanes: one step, unit scale (never read)
        rel[s] = 1.0;
        nsteps[s] = 1;
        return;
    }
    const double margin = 1.05;
    double dt;
    if (use_coarse) {
        const double dt_coarse = 2.0 / sqrt(margin * lc[s]);
        const double dt_fine = p_fine * 2.0 / sqrt(margin * lf[s]);
        dt = safety * fmin(dt_coarse, dt_fine);
    } else {
        dt = safety * 2.0 / sqrt(margin * lf[s]);
    }
    const double steps = ceil(T / dt - 1e-12);  // run_wave snapping (integrators.cpp:188-189)
    const double dts = T / steps;
    nsteps[s] = static_cast<int>(steps);
    rel[s] = (dts / dt_ref) * (dts / dt_ref);
}

// ---------------------------------------------------------------------------
// K5: fused small-mesh solve (see SmallArgs): the same arithmetic, row by row
// and in the same order, as the batched path it replaces (sweep_kernel<true>
// start-up, sweep_rows_kernel's structured / single-cell / multi-cell
// gathers, substep_kernel's recipe weights and SELL gather, r_update), so a
// sample's result is bitwise the same whichever path ran it.  Shared
// memory: cell coefficients | recipe weights W | z_a | z_b | g | d_a | d_b.

__host__ __device__ inline int small_layout(const SmallArgs& a, int* oW, int* za, int* zb, int* g, int* da,
                                            int* db) {
    int off = (a.n_cells + 1) & ~1;
    if (oW) *oW = off;
    off += (a.n_wid + 2) & ~1;
    if (za) *za = off;
    off += (a.n + 1) & ~1;
    if (zb) *zb = off;
    off += (a.n + 1) & ~1;
    const int r = (a.n_r + 1) & ~1;
    if (g) *g = off;
    if (da) *da = off + r;
    if (db) *db = off + 2 * r;
    return off + 3 * r;
}

__global__ void __launch_bounds__(kSmallThreads, 1) small_solve_kernel(SmallArgs a) {
    extern __shared__ __align__(16) double sm[];
    int oW, oza, ozb, og, oda, odb;
    small_layout(a, &oW, &oza, &ozb, &og, &oda, &odb);
    double* cl = sm;
    double* W = sm + oW;
    const int tid = threadIdx.x, T = blockDim.x;
    const std::size_t S = static_cast<std::size_t>(a.S);
    __shared__ int fail_step;
    for (int s = blockIdx.x; s < a.count; s += gridDim.x) {
        const long n_steps = a.nsteps ? __ldg(a.nsteps + s) : a.n_steps;
        const double rs = a.rel ? __ldg(a.rel + s) : 1.0;
        for (int k = tid; k < a.n_cells; k += T) cl[k] = __ldg(a.cells + k * S + s);
        if (tid == 0) fail_step = INT_MAX;
        __syncthreads();
        for (int w = tid; w < a.n_wid; w += T) {  // recipe weights (substep_kernel)
            double acc = 0.0;
            for (int t = __ldg(a.rc_ptr + w); t < __ldg(a.rc_ptr + w + 1); ++t)
                acc += cl[__ldg(a.rc_cell + t)] * __ldg(a.rc_a0 + t);
            W[w] = acc;
        }
        if (tid == 0) W[a.n_wid] = 0.0;  // SELL padding weight
        double* zc = sm + oza;  // z_n
        double* zp = sm + ozb;  // z_{n-1}, overwritten with z_{n+1}
        // start-up (sweep_kernel<true>): z1 = z0 + factor (0 - A z0)
        for (int i = tid; i < a.n; i += T) {
            const int4 d = __ldg(a.row_desc + i);
            const int b = __ldg(a.row_ptr + i), e = __ldg(a.row_ptr + i + 1);
            double acc0 = 0.0;
            if (d.x >= 0) {
                const double c = cl[d.x & 0xffff];
                double p0 = 0.0;
                for (int q = b; q < e; ++q) {
                    const double zj = __ldg(a.z0 + (__ldg(a.ent + q) & a.col_mask));
                    p0 += __ldg(a.a0 + q) * zj;
                }
                acc0 = c * p0;
            } else {
                for (int q = b; q < e; ++q) {
                    const unsigned pk = static_cast<unsigned>(__ldg(a.ent + q));
                    const double zj = __ldg(a.z0 + (pk & a.col_mask));
                    acc0 += (cl[ent_cell(a.cell_ix, q, static_cast<int>(pk), a.col_bits)] * __ldg(a.a0 + q)) * zj;
                }
            }
            const double z0 = __ldg(a.z0 + i);
            const double out = z0 + (a.init_factor * rs) * (0.0 - acc0);
            zp[i] = z0;
            zc[i] = out;
            if (!(fabs(out) <= 1e100)) atomicMin(&fail_step, 1);
        }
        __syncthreads();
        const double factor = a.factor * rs;
        for (long st = 1; st < n_steps; ++st) {
            const int step = static_cast<int>(st + 1);
            // sweep (sweep_rows_kernel)
            for (int i = tid; i < a.n; i += T) {
                const int4 d = __ldg(a.row_desc + i);
                double acc0 = 0.0;
                if (d.x >= 0 && ((d.x >> 16) & 0xff) > 0) {
                    const double2 w = __ldg(a.wtype + ((d.x >> 16) & 0xff) - 1);
                    const double c = cl[d.x & 0xffff];
                    double p0 = 0.0;
                    p0 += w.x * zc[i - d.z];
                    p0 += w.x * zc[i - 1];
                    p0 += w.y * zc[i];
                    p0 += w.x * zc[i + 1];
                    p0 += w.x * zc[i + d.w];
                    acc0 = c * p0;
                } else if (d.x >= 0) {
                    const double c = cl[d.x & 0xffff];
                    double p0 = 0.0;
                    for (int q = d.y; q < __ldg(a.row_ptr + i + 1); ++q)
                        p0 += __ldg(a.a0 + q) * zc[__ldg(a.ent + q) & a.col_mask];
                    acc0 = c * p0;
                } else {
                    for (int q = d.y; q < __ldg(a.row_ptr + i + 1); ++q) {
                        const unsigned pk = static_cast<unsigned>(__ldg(a.ent + q));
                        acc0 += (cl[ent_cell(a.cell_ix, q, static_cast<int>(pk), a.col_bits)] * __ldg(a.a0 + q)) *
                                zc[pk & a.col_mask];
                    }
                }
                if (i < a.split) {
                    sm[og + i] = acc0;
                } else {
                    const double out = 2.0 * zc[i] - zp[i] - factor * acc0;
                    zp[i] = out;
                    if (!(fabs(out) <= 1e100)) atomicMin(&fail_step, step);
                }
            }
            __syncthreads();
            if (a.split > 0) {
                // substep_kernel: d_1 = -c0 g, then the SELL gather with recipe weights
                const double c0 = a.c0 * rs;
                for (int i = tid; i < a.split; i += T) sm[oda + i] = -c0 * sm[og + i];
                __syncthreads();
                for (int m = 1; m <= a.p - 1; ++m) {
                    const double* cur = sm + ((m & 1) ? oda : odb);
                    double* nxt = sm + ((m & 1) ? odb : oda);
                    const double beta = __ldg(a.beta + m - 1);
                    const double cm = __ldg(a.cm + m - 1) * rs;
                    for (int i = tid; i < a.split; i += T) {
                        const int slice = i >> 5, lane = i & 31;
                        const int b = __ldg(a.slice_off + slice), e = __ldg(a.slice_off + slice + 1);
                        double aq = 0.0;
                        for (int q = b + lane; q < e; q += 32) {
                            const std::uint32_t pk = __ldg(a.sub_ent + q);
                            aq += W[pk >> 16] * cur[pk & 0xffffu];
                        }
                        const double dp = m == 1 ? 0.0 : nxt[i];
                        nxt[i] = (1.0 + beta) * cur[i] - beta * dp - cm * (sm[og + i] + aq);
                    }
                    __syncthreads();
                }
                // r_update: z_{n+1} = 2 z_n - z_{n-1} + 2 d_p
                const double* dpv = sm + ((a.p & 1) ? oda : odb);
                for (int i = tid; i < a.split; i += T) {
                    const double out = 2.0 * zc[i] - zp[i] + 2.0 * dpv[i];
                    zp[i] = out;
                    if (!(fabs(out) <= 1e100)) atomicMin(&fail_step, step);
                }
            }
            __syncthreads();
            double* t = zc;  // z_{n+1} becomes z_n
            zc = zp;
            zp = t;
        }
        // QoI outputs of the final state (qoi_kernel; NaN for a failed sample)
        for (int k = tid; k < a.nq; k += T) {
            double acc = 0.0;
            for (int q = __ldg(a.qptr + k); q < __ldg(a.qptr + k + 1); ++q)
                acc += __ldg(a.qw + q) * (zc[__ldg(a.qdof + q)] / __ldg(a.qsm + q));
            a.q[k * S + s] = fail_step == INT_MAX ? acc : __longlong_as_double(0x7ff8000000000000LL);
        }
        if (tid == 0) a.fail[s] = fail_step;
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K6: fused lattice solve (see LatSolveArgs).  Thread roles are the lattice
// kernel's: column ci of strip `strip` (<= K consecutive lattice rows) and G
// generic rows of R; rows outside R go round-robin.  The substeps, the R
// update, the leap-frog rows and the QoI are the batched kernels' arithmetic;
// g = A z_n on the lattice rows comes from the substep stencil (v = z / h)
// instead of the sweep's per-row descriptors (the same operator, a different
// rounding: agreement with the per-step path at the 1e-15 level, not
// bitwise).  A level takes one path for every batch, so results still depend
// only on (seed, level, index).  Shared memory (doubles): z_n | z_{n-1}
// (optional) | v0 | v1 | gw | cl | beta | cm | then the integer tables.

struct LatSolveOff {
    int zn, zp, v0, v1, gw, cl, beta, cm, gcol, sj0, slen, cx, cy, total;
};

__host__ __device__ inline LatSolveOff lat_solve_offsets(const LatSolveArgs& A) {
    const LatArgs& a = A.lat;
    LatSolveOff o;
    int off = 0;
    auto take = [&](int doubles) {
        const int r = off;
        off += (doubles + 1) & ~1;
        return r;
    };
    const int slots = a.n_slots > 0 ? a.n_slots : 1;
    o.zn = take(A.n);
    o.zp = A.zp_global ? -1 : take(A.n);
    o.v0 = take(a.n_r + 16);  // rows past a short strip read (never write) up to 8 beyond
    // v1 also holds z_{n+1} of the rows outside R between the sweep and its store
    o.v1 = take(a.n_r + 16 > A.n - a.n_r ? a.n_r + 16 : A.n - a.n_r);
    o.gw = A.tmem ? -1 : take(slots);  // generic weights and columns live in TMEM when tmem is set
    o.cl = take(a.n_cells);
    o.beta = take(a.p > 1 ? a.p - 1 : 1);
    o.cm = take(a.p > 1 ? a.p - 1 : 1);
    o.gcol = A.tmem ? -1 : take((slots * 2 + 7) / 8);  // uint16
    o.sj0 = take((a.n_strips + 1) / 2);  // int
    o.slen = take((a.n_strips + 1) / 2);
    o.cx = take((a.m + 1) / 2);
    o.cy = take((a.m + 1) / 2);
    o.total = off;
    return o;
}

// g_i = (A(omega) z)_i of one row, exactly as sweep_rows_kernel forms it
// (structured 5-point rows from the descriptor; single-cell and multi-cell
// rows from the entries), with z and the cell coefficients on chip
__device__ __forceinline__ double lat_solve_row(const LatSolveArgs& A, int i, const double* zc, const double* cl) {
    const int4 d = __ldg(A.row_desc + i);
    double acc0 = 0.0;
    if (d.x >= 0 && ((d.x >> 16) & 0xff) > 0) {
        const double2 w = __ldg(A.wtype + ((d.x >> 16) & 0xff) - 1);
        const double c = cl[d.x & 0xffff];
        double p0 = 0.0;
        p0 += w.x * zc[i - d.z];
        p0 += w.x * zc[i - 1];
        p0 += w.y * zc[i];
        p0 += w.x * zc[i + 1];
        p0 += w.x * zc[i + d.w];
        acc0 = c * p0;
    } else if (d.x >= 0) {
        const double c = cl[d.x & 0xffff];
        double p0 = 0.0;
        const int e = __ldg(A.row_ptr + i + 1);
        for (int q = d.y; q < e; ++q) p0 += __ldg(A.a0 + q) * zc[__ldg(A.ent + q) & A.col_mask];
        acc0 = c * p0;
    } else {
        const int e = __ldg(A.row_ptr + i + 1);
        for (int q = d.y; q < e; ++q) {
            const unsigned pk = static_cast<unsigned>(__ldg(A.ent + q));
            acc0 += (cl[ent_cell(A.cell_ix, q, static_cast<int>(pk), A.col_bits)] * __ldg(A.a0 + q)) *
                    zc[pk & A.col_mask];
        }
    }
    return acc0;
}

// g = A z_n on the thread's lattice rows by the substep stencil: v = z / sqrt(M)
// of every R row published to v (owners), one barrier, then the 5-point
// stencil of lattice_substep_kernel (edge conductances already / h)
// PUB = false: v is already published (the previous step's R update or the
// start-up wrote it next to z_n, and a barrier followed)
template <int K, int G, bool PUB = true>
__device__ __forceinline__ void lat_solve_g(double* sd, int ov, const double* zn, int base, int len, int W, int sS,
                                            int sN, double inv_h, double kE, double kW, double kNS, double dg,
                                            const int* grow, const double* grs, double* gg) {
    if (PUB) {
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (k < len) sd[ov + base + k] = zn[base + k] * inv_h;
#pragma unroll
        for (int u = 0; u < G; ++u)
            if (grow[u] >= 0) sd[ov + grow[u]] = zn[grow[u]] * grs[u];
        __syncthreads();
    }
    const int ce = ov + base + W, cw_ = ov + base - W;
    const double vnl = sd[ov + sN];
    double vs = sd[ov + sS];
    double vk = sd[ov + base];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double ve = sd[ce + k], vw = sd[cw_ + k];
        const double vn = (k + 1 < len) ? sd[ov + base + k + 1] : vnl;
        gg[k] = k < len ? dg * vk - kE * ve - kW * vw - kNS * (vn + vs) : 0.0;
        vs = vk;
        vk = vn;
    }
}

// ---- Tensor memory as per-thread private storage (fused lattice solve).
// TMEM (256 KB per SM, 128 lanes x 512 columns of 32 bits) is read by
// tcgen05.ld on its own datapath: measured on this B200 at ~390 B/clk/SM
// beside an unchanged 128 B/clk of shared-memory LDS.128 traffic
// (tools/tmem_bench.cu), so what a thread alone reads every substep -- its
// generic rows' SELL weights and columns, and d_{m-1} of its lattice nodes --
// moves out of the shared-memory pipe the kernel is bound by.  Warp w owns
// lanes 32 (w % 4) .. + 31 (its sub-partition's lane quarter) and columns
// 128 (w / 4) .. + 127.  Each tcgen05.ld / st is issued together with its
// wait in one asm statement, so the compiler cannot read the outputs (or
// reuse the inputs) early.  The loads carry no "memory" clobber (TMEM is
// not memory the compiler tracks; asm volatile keeps them ordered with the
// tcgen05.st), so shared-memory accesses may be scheduled around them.
__device__ __forceinline__ void tm_ld16(std::uint32_t addr, std::uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
}
__device__ __forceinline__ void tm_ld16_4(std::uint32_t aw, std::uint32_t (&w)[16], std::uint32_t ac,
                                          std::uint32_t (&c)[4]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%20];\n"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%16,%17,%18,%19}, [%21];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
          "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]),
          "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3])
        : "r"(aw), "r"(ac));
}
__device__ __forceinline__ void tm_st16(std::uint32_t addr, const std::uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
        "tcgen05.wait::st.sync.aligned;\n"
        :
        : "r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tm_st4(std::uint32_t addr, const std::uint32_t (&r)[4]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n"
        "tcgen05.wait::st.sync.aligned;\n"
        :
        : "r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
        : "memory");
}
// N-column forms (N = 2 K for the d_{m-1} columns): x16 / x4 / x2 chunks,
// each with its own wait
__device__ __forceinline__ void tm_ld2(std::uint32_t addr, std::uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(r[0]), "=r"(r[1])
                 : "r"(addr)
                 : "memory");
}
__device__ __forceinline__ void tm_ld4p(std::uint32_t addr, std::uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr)
                 : "memory");
}
__device__ __forceinline__ void tm_st2(std::uint32_t addr, const std::uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n"
                 "tcgen05.wait::st.sync.aligned;\n"
                 :
                 : "r"(addr), "r"(r[0]), "r"(r[1])
                 : "memory");
}
template <int N>
__device__ __forceinline__ void tm_ldn(std::uint32_t addr, std::uint32_t (&r)[N]) {
    static_assert(N % 2 == 0, "even column count");
    int c = 0;
    if constexpr (N >= 16) {
        tm_ld16(addr, *reinterpret_cast<std::uint32_t(*)[16]>(r));
        c = 16;
    }
#pragma unroll
    for (; c + 4 <= N; c += 4) tm_ld4p(addr + c, r + c);
#pragma unroll
    for (; c + 2 <= N; c += 2) tm_ld2(addr + c, r + c);
}
template <int N>
__device__ __forceinline__ void tm_stn(std::uint32_t addr, const std::uint32_t (&r)[N]) {
    static_assert(N % 2 == 0, "even column count");
    int c = 0;
    if constexpr (N >= 16) {
        tm_st16(addr, *reinterpret_cast<const std::uint32_t(*)[16]>(r));
        c = 16;
    }
#pragma unroll
    for (; c + 4 <= N; c += 4) tm_st4(addr + c, *reinterpret_cast<const std::uint32_t(*)[4]>(r + c));
#pragma unroll
    for (; c + 2 <= N; c += 2) tm_st2(addr + c, r + c);
}
// NCOL columns (32..512, a power of two): 128 per four warps, so a
// 512-thread CTA takes the whole TMEM and four 128-thread CTAs share an SM
template <int NCOL>
__device__ __forceinline__ std::uint32_t tm_alloc(std::uint32_t* slot) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 "tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n"
                 :
                 : "r"(static_cast<std::uint32_t>(__cvta_generic_to_shared(slot))), "n"(NCOL)
                 : "memory");
    return 0;
}
template <int NCOL>
__device__ __forceinline__ void tm_dealloc(std::uint32_t base) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" : : "r"(base), "n"(NCOL) : "memory");
}
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// generic SELL row from TMEM-held weight pairs (w: [pair][lo x, hi x, lo y,
// hi y]) and column pairs: gen_gather's products and sums in its order
template <int NP>
__device__ __forceinline__ double gen_gather_r(const double* __restrict__ sd, int cur, const std::uint32_t (&w)[16],
                                               const std::uint32_t (&c)[4]) {
    double acc = 0.0, acc2 = 0.0;
#pragma unroll
    for (int p = NP - 1; p >= 0; --p) {
        const double wx = __hiloint2double(static_cast<int>(w[4 * p + 1]), static_cast<int>(w[4 * p]));
        const double wy = __hiloint2double(static_cast<int>(w[4 * p + 3]), static_cast<int>(w[4 * p + 2]));
        acc2 += wy * sd[cur + (c[p] >> 16)];
        acc += wx * sd[cur + (c[p] & 0xffffu)];
    }
    return acc + acc2;
}

// warp-uniform width wd; TMEM columns tw (weights) and tc (column pairs)
__device__ __forceinline__ double gen_gather_tm(int wd, const double* __restrict__ sd, int cur, std::uint32_t tw,
                                                std::uint32_t tc) {
    if (wd == 0) return 0.0;
    std::uint32_t w[16], c[4];
    tm_ld16_4(tw, w, tc, c);
    switch (wd) {
        case 8: return gen_gather_r<4>(sd, cur, w, c);
        case 6: return gen_gather_r<3>(sd, cur, w, c);
        case 4: return gen_gather_r<2>(sd, cur, w, c);
        case 2: return gen_gather_r<1>(sd, cur, w, c);
        default: return 0.0;
    }
}

// g = A z_n on a generic R row of the fused solve: the row's A P part is the
// SELL gather on v = z / sqrt(M) (published to v0 by every R row's owner),
// the entries with columns outside P come from the small remainder table
__device__ __forceinline__ double gen_full_row(const LatSolveArgs& A, const double* sd, int ogw, int ov,
                                               const std::uint16_t* gcol, int gslot, int gwid, int q,
                                               const double* zn, const double* cl) {
    double rem = 0.0;
    for (int t = __ldg(A.rem_ptr + q); t < __ldg(A.rem_ptr + q + 1); ++t)
        rem += (cl[__ldg(A.rem_cell + t)] * __ldg(A.rem_a0 + t)) * zn[__ldg(A.rem_col + t)];
    return gen_gather_w(gwid, sd, ogw, ov, gcol, gslot) + rem;
}
// TMEM form: the gather is warp-collective (tcgen05.ld), so every lane of
// the warp calls it; the remainder only for lanes holding a row (live)
__device__ __forceinline__ double gen_full_row_tm(const LatSolveArgs& A, const double* sd, int ov, std::uint32_t tw,
                                                  std::uint32_t tc, int gwid, int q, bool live, const double* zn,
                                                  const double* cl) {
    const double gath = gen_gather_tm(gwid, sd, ov, tw, tc);
    double rem = 0.0;
    if (live)
        for (int t = __ldg(A.rem_ptr + q); t < __ldg(A.rem_ptr + q + 1); ++t)
            rem += (cl[__ldg(A.rem_cell + t)] * __ldg(A.rem_a0 + t)) * zn[__ldg(A.rem_col + t)];
    return gath + rem;
}

#ifndef WMC_LAT_PIPE
#define WMC_LAT_PIPE 2
#endif
// TM: generic weights / columns and the lattice nodes' d_{m-1} in tensor
// memory (see tm_ld16); otherwise weights and columns in shared memory and
// d_{m-1} read back from the buffer the substep overwrites.
// VT (with TM): d_{m-1} of the lattice nodes in TMEM too; otherwise read
// back from the shared-memory buffer the substep overwrites.
// PK: every strip holds K or K - 1 rows (host-checked), so the rare path
// for shorter strips is compiled out.
template <int T, int K, int G, bool TM, bool VT = TM, bool PK = false>
__global__ void __launch_bounds__(T, 1) lattice_solve_kernel(LatSolveArgs A) {
    static_assert(!TM || (T % 128 == 0 && T <= 512 && 20 * G + 4 * K <= 128), "TMEM columns per thread");
    extern __shared__ __align__(16) double sd[];
    const LatArgs& a = A.lat;
    const LatSolveOff o = lat_solve_offsets(A);
    std::uint16_t* gcol = reinterpret_cast<std::uint16_t*>(sd + o.gcol);
    int* sj0 = reinterpret_cast<int*>(sd + o.sj0);
    int* slen = reinterpret_cast<int*>(sd + o.slen);
    int* cx = reinterpret_cast<int*>(sd + o.cx);
    int* cy = reinterpret_cast<int*>(sd + o.cy);
    double* zn = sd + o.zn;
    double* cl = sd + o.cl;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const std::size_t S = static_cast<std::size_t>(a.S);
    const int W = a.m + 1;
    const int nr = a.n_r;
    const double inv_h = a.inv_h;
    const double hh = 1.0 / inv_h;
    __shared__ int fail_step;
    __shared__ std::uint32_t tm_slot;

    // tensor memory: the whole 512 columns (one CTA per SM); this thread's
    // columns: weights of generic role u at 16 u, its column pairs at
    // 20 G + 4 u... see tw_/tc_/tv_ below
    if (TM) {
        if ((tid >> 5) == 0) tm_alloc<(T >= 512 ? 512 : 128 * (T / 128))>(&tm_slot);
        tm_fence_before();
        __syncthreads();
        tm_fence_after();
    }
    const std::uint32_t tbase =
        TM ? tm_slot + (static_cast<std::uint32_t>(32 * ((tid >> 5) & 3)) << 16) + 128u * ((tid >> 5) >> 2) : 0u;
    auto tw_ = [&](int u) { return tbase + 16u * u; };            // 16 columns: 4 weight pairs
    auto tc_ = [&](int u) { return tbase + 16u * G + 4u * u; };   // 4 columns: column pairs
    auto tv_ = [&](int set) { return tbase + 20u * G + 2u * K * set; };  // 2 K columns: v_{m-1}
    // non-structured rows outside R (form 2 only, d_{m-1} not in TMEM):
    // role j at 20 G + 38 j: kNsMax entry words, 2 kNsMax weight words, row, count | (cell + 1) << 8
    auto tn_ = [&](int j) { return tbase + 20u * G + 38u * j; };
    static_assert(!TM || VT || 20 * G + 2 * 38 <= static_cast<int>(128), "TMEM columns for the rows outside R");
    if (TM && !VT && A.n_ns > 0) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int q = j * T + tid;
            const int r = q < A.n_ns ? __ldg(A.ns_rows + q) : -1;
            std::uint32_t ew[kNsMax], ww[2 * kNsMax], mw[2];
            int b = 0, cnt = 0, cellp = 0;
            if (r >= 0) {
                b = __ldg(A.row_ptr + r);
                cnt = __ldg(A.row_ptr + r + 1) - b;
                const int4 d = __ldg(A.row_desc + r);
                cellp = d.x >= 0 ? (d.x & 0xffff) + 1 : 0;
            }
#pragma unroll
            for (int t = 0; t < kNsMax; ++t) {
                const double w = t < cnt ? __ldg(A.a0 + b + t) : 0.0;
                ew[t] = t < cnt ? static_cast<std::uint32_t>(__ldg(A.ent + b + t)) : 0u;
                ww[2 * t] = static_cast<std::uint32_t>(__double2loint(w));
                ww[2 * t + 1] = static_cast<std::uint32_t>(__double2hiint(w));
            }
            mw[0] = static_cast<std::uint32_t>(r);
            mw[1] = static_cast<std::uint32_t>(cnt) | (static_cast<std::uint32_t>(cellp) << 8);
            tm_stn<kNsMax>(tn_(j), ew);
            tm_stn<2 * kNsMax>(tn_(j) + kNsMax, ww);
            tm_stn<2>(tn_(j) + 3 * kNsMax, mw);
        }
    }

    // static tables, once per CTA
    if (!TM)
        for (int i = tid; i < a.n_slots; i += T) gcol[i] = __ldg(a.gen_col + i);
    for (int i = tid; i < a.n_strips; i += T) {
        sj0[i] = __ldg(a.strip_j0 + i);
        slen[i] = __ldg(a.strip_len + i);
    }
    for (int i = tid; i < a.m; i += T) {
        cx[i] = __ldg(a.cellx + i);
        cy[i] = __ldg(a.celly + i);
    }
    for (int i = tid; i < a.p - 1; i += T) {
        sd[o.beta + i] = __ldg(a.beta + i);
        sd[o.cm + i] = __ldg(a.cm + i);
    }
    const int col = tid % a.cw, strip = tid / a.cw;
    const int ci = 1 + col;
    const bool lat_on = ci <= a.m - 1 && strip < a.n_strips;
    int grow[G], gslot[G], gwid[G], gq[G];
    double grs[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
        const int wsl = __ldg(a.gen_warp_slice + (tid >> 5) * G + u);
        const int q = wsl >= 0 ? wsl * 32 + lane : a.n_gen;
        gq[u] = q;
        grow[u] = q < a.n_gen ? __ldg(a.gen_rows + q) : -1;
        grs[u] = q < a.n_gen ? __ldg(a.gen_rs + q) : 0.0;
        const int sl = wsl >= 0 ? wsl : 0;
        gslot[u] = __ldg(a.gen_soff + sl) + 2 * lane;
        gwid[u] = wsl >= 0 ? (__ldg(a.gen_soff + sl + 1) - __ldg(a.gen_soff + sl)) >> 5 : 0;
    }
    __syncthreads();
    // idle lanes shadow the strip's last column (see lattice_substep_kernel)
    const bool shadow = !lat_on && strip < a.n_strips;
    int j0 = 1, len = 0, span = 0;
    if (lat_on || shadow) {
        j0 = sj0[strip];
        span = slen[strip];
    }
    if (lat_on) len = span;
    const int base = (lat_on || shadow) ? (lat_on ? ci : a.m - 1) * W + j0 : W + 1;
    const int sS = (lat_on || shadow) ? base - 1 : 0, sN = (lat_on || shadow) ? base + span : 0;

    for (int s = blockIdx.x; s < a.count; s += gridDim.x) {
        const long n_steps = a.nsteps ? __ldg(a.nsteps + s) : A.n_steps;
        const double rs = a.rel ? __ldg(a.rel + s) : 1.0;
        double* zp = A.zp_global ? A.zp_global + static_cast<std::size_t>(s) * A.n : sd + o.zp;
        // ---- per-sample set-up: coefficients, z_0, generic weights
        for (int k = tid; k < a.n_cells; k += T) cl[k] = __ldg(a.cells + k * S + s);
        for (int i = tid; i < A.n; i += T) {
            const double z = __ldg(A.z0 + i);
            zn[i] = z;
            zp[i] = z;
        }
        if (tid == 0) fail_step = INT_MAX;
        __syncthreads();
        auto slot_weight = [&](int e) {
            const unsigned c = __ldg(a.slot_cell + e);
            double w;
            if (!(c & kOvfFlag)) {
                w = cl[c] * __ldg(a.slot_a0 + e);
            } else {
                const int k = c & ~kOvfFlag;
                w = 0.0;
                for (int t = __ldg(a.ovf_start + k); t < __ldg(a.ovf_start + k + 1); ++t)
                    w += cl[__ldg(a.ovf_cell + t)] * __ldg(a.ovf_a0 + t);
            }
            return w;
        };
        if (TM) {
            // each thread forms its own generic rows' weights straight into
            // its TMEM columns (pairs p < width / 2; the rest zero)
            __syncthreads();  // cl complete
            const unsigned* gc2 = reinterpret_cast<const unsigned*>(a.gen_col);
#pragma unroll
            for (int u = 0; u < G; ++u) {
                std::uint32_t wr[16], cr[4];
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    double w0 = 0.0, w1 = 0.0;
                    cr[p] = 0u;
                    if (2 * p < gwid[u]) {
                        w0 = slot_weight(gslot[u] + 64 * p);
                        w1 = slot_weight(gslot[u] + 64 * p + 1);
                        cr[p] = __ldg(gc2 + ((gslot[u] + 64 * p) >> 1));
                    }
                    wr[4 * p] = static_cast<std::uint32_t>(__double2loint(w0));
                    wr[4 * p + 1] = static_cast<std::uint32_t>(__double2hiint(w0));
                    wr[4 * p + 2] = static_cast<std::uint32_t>(__double2loint(w1));
                    wr[4 * p + 3] = static_cast<std::uint32_t>(__double2hiint(w1));
                }
                tm_st16(tw_(u), wr);
                tm_st4(tc_(u), cr);
            }
        } else {
            for (int e = tid; e < a.n_slots; e += T) sd[o.gw + e] = slot_weight(e);
        }
        double kE = 0, kW = 0, kNS = 0, dg = 0;
        if (lat_on) {
            const int row = cy[j0] * a.cells_x;
            const double cR = cl[row + cx[ci]], cL = cl[row + cx[ci - 1]];
            kE = cR * inv_h;
            kW = cL * inv_h;
            kNS = (cL + cR) * (0.5 * inv_h);
            dg = kE + kW + 2.0 * kNS;
        }
        // ---- start-up (sweep_kernel<true>): z_1 = z_0 + f (0 - A z_0)
        double gg[K], ggg[G];
        {
            const double fi = A.init_factor * rs;
            lat_solve_g<K, G>(sd, o.v0, zn, base, len, W, sS, sN, inv_h, kE, kW, kNS, dg, grow, grs, gg);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (k < len) {
                    gg[k] = zn[base + k] + fi * (0.0 - gg[k]);
                    if (!(fabs(gg[k]) <= 1e100)) atomicMin(&fail_step, 1);
                }
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
                ggg[u] = 0.0;
                const double gt =
                    TM ? gen_full_row_tm(A, sd, o.v0, tw_(u), tc_(u), gwid[u], gq[u], grow[u] >= 0, zn, cl) : 0.0;
                if (grow[u] >= 0) {
                    ggg[u] = zn[grow[u]] +
                             fi * (0.0 - (TM ? gt
                                             : gen_full_row(A, sd, o.gw, o.v0, gcol, gslot[u], gwid[u], gq[u], zn,
                                                            cl)));
                    if (!(fabs(ggg[u]) <= 1e100)) atomicMin(&fail_step, 1);
                }
            }
            for (int i = nr + tid; i < A.n; i += T) {
                const double out = zn[i] + fi * (0.0 - lat_solve_row(A, i, zn, cl));
                sd[o.v1 + i - nr] = out;
                if (!(fabs(out) <= 1e100)) atomicMin(&fail_step, 1);
            }
            __syncthreads();
            // z_1, and v = z_1 / sqrt(M) published for the first step's sweep
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (k < len) {
                    zn[base + k] = gg[k];
                    sd[o.v0 + base + k] = gg[k] * inv_h;
                }
#pragma unroll
            for (int u = 0; u < G; ++u)
                if (grow[u] >= 0) {
                    zn[grow[u]] = ggg[u];
                    sd[o.v0 + grow[u]] = ggg[u] * grs[u];
                }
            for (int i = nr + tid; i < A.n; i += T) zn[i] = sd[o.v1 + i - nr];
            __syncthreads();
        }
        const double factor = A.factor * rs;
        const double c0 = a.c0 * rs;
        for (long st = 1; st < n_steps; ++st) {
            const int step = static_cast<int>(st + 1);
            // check_finite (integrators.cpp:12-18): a per-thread flag over the
            // step's stores, one atomic per flagged thread at the step end
            bool bad = false;
            // ---- sweep: g = A z_n on R rows (lattice rows by the substep
            // stencil, the others as sweep_rows_kernel), leap-frog update of
            // the rows outside R (z_{n+1} parked in v1 until every read of
            // z_n is done)
            lat_solve_g<K, G, false>(sd, o.v0, zn, base, len, W, sS, sN, inv_h, kE, kW, kNS, dg, grow, grs, gg);
#pragma unroll
            for (int u = 0; u < G; ++u)
                if (TM) {
                    const double gt =
                        gen_full_row_tm(A, sd, o.v0, tw_(u), tc_(u), gwid[u], gq[u], grow[u] >= 0, zn, cl);
                    ggg[u] = grow[u] >= 0 ? gt : 0.0;
                } else {
                    ggg[u] = grow[u] >= 0 ? gen_full_row(A, sd, o.gw, o.v0, gcol, gslot[u], gwid[u], gq[u], zn, cl)
                                          : 0.0;
                }
            // four rows per pass, every load before any store (z_{n-1} may
            // live in global memory: its latency overlaps instead of chaining)
            for (int i0 = nr + tid; i0 < A.n; i0 += 4 * T) {
                double zi[4], zq[4], gr[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * T;
                    zi[u] = i < A.n ? zn[i] : 0.0;
                    zq[u] = i < A.n ? zp[i] : 0.0;
                }
                bool mine[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * T;
                    mine[u] = i < A.n;
                    if (TM && !VT && A.n_ns > 0 && mine[u]) {  // non-structured rows: the TMEM pass below
                        const int4 dd = __ldg(A.row_desc + i);
                        mine[u] = dd.x >= 0 && ((dd.x >> 16) & 0xff) > 0;
                    }
                    gr[u] = mine[u] ? lat_solve_row(A, i, zn, cl) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * T;
                    if (!mine[u]) continue;
                    const double out = 2.0 * zi[u] - zq[u] - factor * gr[u];
                    sd[o.v1 + i - nr] = out;
                    bad |= !(fabs(out) <= 1e100);
                }
            }
            if (TM && !VT && A.n_ns > 0) {
                // the thread's non-structured rows outside R from its TMEM
                // columns: lat_solve_row's CSR sums in entry order, no global
                // loads, warp-uniform trip count (predicated on the row length)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (j * T + (tid & ~31) >= A.n_ns) continue;  // warp-uniform
                    std::uint32_t mw[2], ew[kNsMax];
                    tm_ldn<2>(tn_(j) + 3 * kNsMax, mw);
                    tm_ldn<kNsMax>(tn_(j), ew);
                    std::uint32_t ww[2 * kNsMax];
                    tm_ldn<2 * kNsMax>(tn_(j) + kNsMax, ww);
                    const int r = static_cast<int>(mw[0]);
                    if (r >= 0) {  // per lane (no warp-collective op inside)
                    const int cnt = static_cast<int>(mw[1] & 0xffu), cellp = static_cast<int>(mw[1] >> 8);
                    double acc0 = 0.0;
                    if (cellp) {
                        double p0 = 0.0;
#pragma unroll
                        for (int t = 0; t < kNsMax; ++t)
                            if (t < cnt)
                                p0 += __hiloint2double(static_cast<int>(ww[2 * t + 1]), static_cast<int>(ww[2 * t])) *
                                      zn[ew[t] & static_cast<unsigned>(A.col_mask)];
                        acc0 = cl[cellp - 1] * p0;
                    } else {
#pragma unroll
                        for (int t = 0; t < kNsMax; ++t)
                            if (t < cnt)
                                acc0 += (cl[ew[t] >> A.col_bits] *
                                         __hiloint2double(static_cast<int>(ww[2 * t + 1]), static_cast<int>(ww[2 * t]))) *
                                        zn[ew[t] & static_cast<unsigned>(A.col_mask)];
                    }
                    const double out = 2.0 * zn[r] - zp[r] - factor * acc0;
                    sd[o.v1 + r - nr] = out;
                    bad |= !(fabs(out) <= 1e100);
                    }
                }
            }
            __syncthreads();
            for (int i = nr + tid; i < A.n; i += T) {  // z_{n-1} <- z_n, z_n <- z_{n+1}
                zp[i] = zn[i];
                zn[i] = sd[o.v1 + i - nr];
            }
            // ---- substeps (lattice_substep_kernel's recursion), d_1 = -c0 g.
            // Lattice nodes recurse on v = d / h itself (what the stencil and
            // the neighbours read): v_{m+1} = (1 + beta) v_m - beta v_{m-1}
            // - (c_m / h)(g + A d_m), three multiplies per node fewer than
            // carrying d; d_p = h v_p at the update
            double d[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                d[k] = (-c0 * gg[k]) * inv_h;
                if (k < len) sd[o.v0 + base + k] = d[k];
            }
            double gd[G], gdp[G];
#pragma unroll
            for (int u = 0; u < G; ++u) {
                gdp[u] = 0.0;
                gd[u] = -c0 * ggg[u];
                if (grow[u] >= 0) sd[o.v0 + grow[u]] = gd[u] * grs[u];
            }
            __syncthreads();
            // buffer offsets carried through the substeps (swapped each one)
            // rather than re-derived from the layout; beta / c_m by pointer
            int cur = o.v0, nxt = o.v1;
            const double* bp = sd + o.beta;
            const double* cp = sd + o.cm;
            const bool lat_first = TM && A.stagger && (((tid >> 5) >> 2) & 1);  // warp-uniform
            for (int m = 1; m <= a.p - 1; ++m) {
                const double beta = bp[m - 1];
                const double cmm = cp[m - 1] * rs;
                const double onepb = 1.0 + beta;
                const double cmh = cmm * inv_h;
                double gaq[G];
                auto gather = [&]() {
#pragma unroll
                    for (int u = 0; u < G; ++u) {
                        gaq[u] = TM ? gen_gather_tm(gwid[u], sd, cur, tw_(u), tc_(u))
                                    : gen_gather_w(gwid[u], sd, o.gw, cur, gcol, gslot[u]);
                    }
                };
                // staggered warps: the generic gather is a latency chain (TMEM
                // load, shared gather, FP64 sums), the lattice nodes are FP64
                // work; half of each scheduler's four warps run the two in the
                // other order so the phases overlap instead of coinciding
                // the strip's two end neighbours, loaded ahead of the gather
                // (level 0: 0.086 -> 0.084 s per 4 096 solves)
                const double vnl_h = sd[cur + base + span], vs_h = sd[cur + base - 1];
                if (!lat_first) gather();
                // TMEM: v_m of the thread's nodes parked for substep m + 1,
                // v_{m-1} back from the other set
                std::uint32_t vp[2 * K];
                if (TM && VT) {
                    if (m < a.p - 1) {
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            vp[2 * k] = static_cast<std::uint32_t>(__double2loint(d[k]));
                            vp[2 * k + 1] = static_cast<std::uint32_t>(__double2hiint(d[k]));
                        }
                        tm_stn<2 * K>(tv_(m & 1), vp);
                    }
                    if (m >= 2) {
                        tm_ldn<2 * K>(tv_((m - 1) & 1), vp);
                    } else {
#pragma unroll
                        for (int k = 0; k < 2 * K; ++k) vp[k] = 0u;
                    }
                }
                if (TM) {
                    // padded strip: a strip shorter than K treats its nodes
                    // k >= len as dummies; node len - 1 reads v_N (the node
                    // above the strip) in place of d[len] -- selected inside
                    // the loop for the common K - 1 case, parked in d[len]
                    // before it for shorter strips -- on one code path;
                    // dummies compute and never store.
                    // Shared-memory rows as pointers (immediate offsets).
                    const double* vc = sd + cur + base;
                    double* vx = sd + nxt + base;
                    const double* vE = vc + W;
                    const double* vW = vc - W;
                    const double vnl = vnl_h;
                    const bool pad_last = span == K - 1;  // the common short strip: v_N read in the loop
                    if (!PK && span < K - 1) {
#pragma unroll
                        for (int k = 0; k < K - 1; ++k)
                            if (k == span) d[k] = vnl;
                    }
                    double vs = vs_h;
                    double vk = d[0];
                    // software-pipelined by kPipe nodes: a node's shared loads are
                    // issued before the store of the node kPipe before it (the
                    // compiler cannot see that the two buffers never alias and
                    // would otherwise chain load -> FP64 -> store node by node)
                    constexpr int kPipe = WMC_LAT_PIPE;
                    double ve_[K], vw_[K], vq_[K];
#pragma unroll
                    for (int k = 0; k < kPipe && k < K; ++k) {
                        ve_[k] = vE[k];
                        vw_[k] = vW[k];
                        vq_[k] = VT ? 0.0 : (m == 1 ? 0.0 : vx[k]);
                    }
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        if (k + kPipe < K) {
                            ve_[k + kPipe] = vE[k + kPipe];
                            vw_[k + kPipe] = vW[k + kPipe];
                            vq_[k + kPipe] = VT ? 0.0 : (m == 1 ? 0.0 : vx[k + kPipe]);
                        }
                        const double ve = ve_[k], vw = vw_[k];
                        const double vn = k + 2 < K ? d[k + 1] : k + 2 == K ? (pad_last ? vnl : d[k + 1]) : vnl;
                        // g + A d as two shallow chains (FP64 dependency depth 5, was 6):
                        // (g + dg v_k - kE v_E) - (kW v_W + kNS (v_N + v_S))
                        const double ga = fma(-kE, ve, fma(dg, vk, gg[k]));
                        const double gb = fma(kW, vw, kNS * (vn + vs));
                        const double vpk =
                            VT ? __hiloint2double(static_cast<int>(vp[2 * k + 1]), static_cast<int>(vp[2 * k]))
                               : vq_[k];
                        const double next = fma(-cmh, ga - gb, fma(onepb, d[k], -(beta * vpk)));
                        d[k] = next;
                        if (k < len) vx[k] = next;
                        vs = vk;
                        vk = vn;
                    }
                } else {
                const int ce = cur + base + W, cw_ = cur + base - W;
                const double vnl = sd[cur + sN];
                double vs = sd[cur + sS];
                double vk = d[0];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const double ve = sd[ce + k], vw = sd[cw_ + k];
                    const double vn = (k + 1 < len) ? d[k + 1] : vnl;
                    // g + A d as two shallow chains (FP64 dependency depth 5, was 6):
                    // (g + dg v_k - kE v_E) - (kW v_W + kNS (v_N + v_S))
                    const double ga = fma(-kE, ve, fma(dg, vk, gg[k]));
                    const double gb = fma(kW, vw, kNS * (vn + vs));
                    const double vpk = m == 1 ? 0.0 : sd[nxt + base + k];
                    const double next = fma(-cmh, ga - gb, fma(onepb, d[k], -(beta * vpk)));
                    d[k] = next;
                    if (k < len) sd[nxt + base + k] = next;
                    vs = vk;
                    vk = vn;
                }
                }
                if (lat_first) gather();
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    const double next = onepb * gd[u] - beta * gdp[u] - cmm * (ggg[u] + gaq[u]);
                    gdp[u] = gd[u];
                    gd[u] = next;
                    if (grow[u] >= 0) sd[nxt + grow[u]] = next * grs[u];
                }
                __syncthreads();
                const int t_ = cur;
                cur = nxt;
                nxt = t_;
            }
            // ---- R update (r_update_kernel): z_{n+1} = 2 z_n - z_{n-1} + 2 d_p;
            // z_{n-1} of the thread's rows loaded before any store
            double zq[K], zgq[G];
#pragma unroll
            for (int k = 0; k < K; ++k) zq[k] = k < len ? zp[base + k] : 0.0;
#pragma unroll
            for (int u = 0; u < G; ++u) zgq[u] = grow[u] >= 0 ? zp[grow[u]] : 0.0;
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (k < len) {
                    const int i = base + k;
                    const double zi = zn[i];
                    const double out = 2.0 * zi - zq[k] + 2.0 * (d[k] * hh);
                    zp[i] = zi;
                    zn[i] = out;
                    sd[o.v0 + i] = out * inv_h;  // v for the next step's sweep (the substeps are done with v0)
                    bad |= !(fabs(out) <= 1e100);
                }
#pragma unroll
            for (int u = 0; u < G; ++u)
                if (grow[u] >= 0) {
                    const int i = grow[u];
                    const double zi = zn[i];
                    const double out = 2.0 * zi - zgq[u] + 2.0 * gd[u];
                    zp[i] = zi;
                    zn[i] = out;
                    sd[o.v0 + i] = out * grs[u];
                    bad |= !(fabs(out) <= 1e100);
                }
            if (bad) atomicMin(&fail_step, step);
            __syncthreads();
        }
        // ---- QoI of the final state (qoi_kernel; NaN for a failed sample)
        for (int k = tid; k < A.nq; k += T) {
            double acc = 0.0;
            for (int q = __ldg(A.qptr + k); q < __ldg(A.qptr + k + 1); ++q)
                acc += __ldg(A.qw + q) * (zn[__ldg(A.qdof + q)] / __ldg(A.qsm + q));
            A.q[k * S + s] = fail_step == INT_MAX ? acc : __longlong_as_double(0x7ff8000000000000LL);
        }
        if (tid == 0) A.fail[s] = fail_step;
        __syncthreads();
    }
    if (TM) {
        tm_fence_before();
        __syncthreads();
        tm_fence_after();
        if ((tid >> 5) == 0) tm_dealloc<(T >= 512 ? 512 : 128 * (T / 128))>(tm_slot);
    }
}

// ---------------------------------------------------------------------------
// K3: QoI per sample, Q = sum_t w_t (z_t / sqrt(M_t)) over the box nodes in a
// fixed order (deterministic); failed samples report NaN.

__global__ void qoi_kernel(QoIArgs a) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (s >= a.count) return;
    const std::size_t S = static_cast<std::size_t>(a.S);
    double acc = 0.0;
    const double* z = (a.nsteps && ((a.n_max - __ldg(a.nsteps + s)) & 1)) ? a.z_alt : a.z;
    for (int t = __ldg(a.ptr + k); t < __ldg(a.ptr + k + 1); ++t) {
        const int i = __ldg(a.dof + t);
        const std::size_t at = a.sample_major ? static_cast<std::size_t>(s) * a.n + i : i * S + s;
        acc += __ldg(a.w + t) * (z[at] / __ldg(a.sqrt_mass + t));
    }
    a.q[k * S + s] = a.fail[s] == INT_MAX ? acc : __longlong_as_double(0x7ff8000000000000LL);
}

// K3, sample-major state (tiled levels): one block per (sample, output), the
// box entries strided over the threads (coalesced along one sample's rows),
// a fixed-order tree over the partial sums (deterministic)
__global__ void __launch_bounds__(256) qoi_sm_kernel(QoIArgs a) {
    __shared__ double part[256];
    const int s = blockIdx.x, k = blockIdx.y;
    const double* z = a.z + static_cast<std::size_t>(s) * a.n;
    double acc = 0.0;
    for (int t = __ldg(a.ptr + k) + threadIdx.x; t < __ldg(a.ptr + k + 1); t += 256)
        acc += __ldg(a.w + t) * (z[__ldg(a.dof + t)] / __ldg(a.sqrt_mass + t));
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        a.q[static_cast<std::size_t>(k) * a.S + s] =
            a.fail[s] == INT_MAX ? part[0] : __longlong_as_double(0x7ff8000000000000LL);
}

__global__ void fill_int_kernel(int* p, int value, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = value;
}

__global__ void pair_diff_kernel(const double* qf, const double* qc, double* dq, double* q_out, int count, int S,
                                 int nq) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (i >= count) return;
    const std::size_t src = static_cast<std::size_t>(k) * S + i, dst = static_cast<std::size_t>(i) * nq + k;
    dq[dst] = qc ? qf[src] - qc[src] : qf[src];
    if (q_out) q_out[dst] = qf[src];
}

// Device-resident results: the first failing sample of a batch (lowest
// index, then step) folded into a per-level record key = index << 24 | step,
// read back by wmc_synchronize (reference check_finite -> InstabilityError,
// src/integrators.cpp:12-18, wrapped per sample as src/mlmc.cpp:31-35)
__global__ void fail_fold_kernel(const int* __restrict__ ff, const int* __restrict__ fc, int count,
                                 unsigned long long first, unsigned long long* rec) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int sf = ff[i], sc = fc ? fc[i] : INT_MAX;
    if (sf != INT_MAX) atomicMin(rec, ((first + i) << 24) | static_cast<unsigned long long>(min(sf, 0xffffff)));
    if (sc != INT_MAX) atomicMin(rec + 1, ((first + i) << 24) | static_cast<unsigned long long>(min(sc, 0xffffff)));
}

// K3b: per-level moment sums, one block, fixed-order tree: deterministic for
// a given count (LevelAccumulator::add, reference src/mlmc.cpp:44-53)
__global__ void __launch_bounds__(1024) moments_kernel(const double* __restrict__ dq, const double* __restrict__ q,
                                                       int count, double* __restrict__ out) {
    __shared__ double red[4][32];
    double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        const double x = dq[i], y = q[i];
        a += x;
        b += x * x;
        c += y;
        d += y * y;
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
        c += __shfl_down_sync(0xffffffffu, c, o);
        d += __shfl_down_sync(0xffffffffu, d, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][warp] = a;
        red[1][warp] = b;
        red[2][warp] = c;
        red[3][warp] = d;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        a = lane < nw ? red[0][lane] : 0.0;
        b = lane < nw ? red[1][lane] : 0.0;
        c = lane < nw ? red[2][lane] : 0.0;
        d = lane < nw ? red[3][lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_down_sync(0xffffffffu, a, o);
            b += __shfl_down_sync(0xffffffffu, b, o);
            c += __shfl_down_sync(0xffffffffu, c, o);
            d += __shfl_down_sync(0xffffffffu, d, o);
        }
        if (lane == 0) {
            out[0] += a;
            out[1] += b;
            out[2] += c;
            out[3] += d;
        }
    }
}

}  // namespace

void launch_fail_fold(const int* ff, const int* fc, int count, unsigned long long first, unsigned long long* rec,
                      void* stream) {
    fail_fold_kernel<<<(count + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(ff, fc, count, first, rec);
}

void launch_moments(const double* dq, const double* q, int count, double* out, void* stream) {
    moments_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(dq, q, count, out);
}

void launch_draw_kl(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S, int n_cells,
                    int modes, const double* table, double* cells, void* stream) {
    // 256 cells per CTA (the normals cost about as much as 32 cells)
    const dim3 grid((S + kKLThreads - 1) / kKLThreads, std::max(1, std::min(65535, (n_cells + 255) / 256)));
    draw_kl_kernel<<<grid, kKLThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        seed, level, first, count, S, n_cells, modes, table, cells);
}

void launch_draw_kl1d(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S, int n_cells,
                      int terms, const double* table, double* cells, void* stream) {
    draw_kl1d_kernel<<<S, 128, 0, static_cast<cudaStream_t>(stream)>>>(seed, level, first, count, S, n_cells, terms,
                                                                       table, cells);
}

void launch_draw_jump1d(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S, int n_cells,
                        double h0, const double* x, double* cells, void* stream) {
    draw_jump1d_kernel<<<S, 128, 0, static_cast<cudaStream_t>(stream)>>>(seed, level, first, count, S, n_cells, h0, x,
                                                                         cells);
}

void launch_draw_cells(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S, int n_cells,
                       double lo, double hi, double* cells, void* stream) {
    draw_cells_kernel<<<(S + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, level, first, count, S,
                                                                                       n_cells, lo, hi, cells);
}

void launch_sweep_init(const SweepArgs& a, void* stream) {
    if (a.sample_major) {
        SweepArgs b = a;
        b.sm_groups = sm_groups();
        const dim3 g(static_cast<unsigned>((a.n + 255) / 256),
                     static_cast<unsigned>((a.S + kSmSamples * b.sm_groups - 1) / (kSmSamples * b.sm_groups)));
        if (b.sm_groups == 8)
            sweep_sm_kernel<true, 8><<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(b);
        else
            sweep_sm_kernel<true, 4><<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(b);
        return;
    }
    const unsigned grid = ((a.n + kSweepWarps - 1) / kSweepWarps) * (a.S / kSweepChunk);
    if (a.cell_ix)
        sweep_kernel<true, false, true><<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
    else
        sweep_kernel<true, false><<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
}

void launch_sweep_step(const SweepArgs& a, void* stream) {
    if (a.sample_major) {
        SweepArgs b = a;
        b.sm_groups = sm_groups();
        const dim3 g(static_cast<unsigned>((a.n - a.row_begin + 255) / 256),
                     static_cast<unsigned>((a.S + kSmSamples * b.sm_groups - 1) / (kSmSamples * b.sm_groups)));
        if (b.sm_groups == 8)
            sweep_sm_kernel<false, 8><<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(b);
        else
            sweep_sm_kernel<false, 4><<<g, 256, 0, static_cast<cudaStream_t>(stream)>>>(b);
        return;
    }
    const unsigned grid = ((a.n + kSweepWarps - 1) / kSweepWarps) * (a.S / kSweepChunk);
    static const int parts = [] {
        const char* v = std::getenv("WMC_SWEEP_PARTS");  // tuning knob
        return v ? std::atoi(v) : 0;
    }();
    static const int one_row = [] {
        const char* v = std::getenv("WMC_SWEEP_ONE_ROW");  // tuning knob: one row per warp
        return v ? std::atoi(v) : 0;
    }();
    const int wide = a.wide;
    // a row range (row_begin > 0) takes the descriptor forms below; the host
    // selects it only for levels with descriptors and packed cells
    if (a.row_begin > 0) {
    } else if (a.cell_ix) {  // cells in a separate per-entry array (narrow-channel levels)
        sweep_kernel<false, false, true><<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
    } else if (parts) {
        sweep_kernel<false, true><<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
    } else if (one_row || !a.row_desc) {
        sweep_kernel<false, false><<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
    }
    if (a.row_begin == 0 && (a.cell_ix || parts || one_row || !a.row_desc)) return;
    if (wide && !a.rel && !a.nsteps && a.S % kSweepChunkW == 0) {
        // wide sweep (default for fixed dt): wide = 10 R + MINB
        const int r = wide / 10;
        const unsigned g2 = ((a.n - a.row_begin + kSweepWarps * r - 1) / (kSweepWarps * r)) * (a.S / kSweepChunkW);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (wide == 14)
            sweep_wide_kernel<1, 4><<<g2, kSweepWarps * 32, 0, st>>>(a);
        else  // 23 (default; measured: level 4 1.22x, level 3 1.15x over sweep_rows_kernel<2>)
            sweep_wide_kernel<2, 3><<<g2, kSweepWarps * 32, 0, st>>>(a);
    } else {
        static const int r = [] {
            const char* v = std::getenv("WMC_SWEEP_ROWS");  // tuning knob: rows per warp (2, 4, 8)
            return v ? std::atoi(v) : kSweepRowsDefault;
        }();
        const int rows = kSweepWarps * r;
        const unsigned g2 = ((a.n - a.row_begin + rows - 1) / rows) * (a.S / kSweepChunk);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (r == 2)
            sweep_rows_kernel<2><<<g2, kSweepWarps * 32, 0, st>>>(a);
        else if (r == 8)
            sweep_rows_kernel<8><<<g2, kSweepWarps * 32, 0, st>>>(a);
        else
            sweep_rows_kernel<4><<<g2, kSweepWarps * 32, 0, st>>>(a);
    }
}

// cudaFuncSetAttribute applies per device: remember what was set for each
// (kernel, device) pair, so a process driving several devices configures each
int set_max_dynamic_smem(const void* kernel, int bytes, bool max_carveout) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_pair(kernel, dev);
    const auto it = done.find(key);
    if (it != done.end()) return it->second;
    const int r = static_cast<int>(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    // the largest shared-memory carveout for kernels that co-reside several
    // CTAs per SM by their shared memory (the tiled step).  Not for the others:
    // an SM configured for them leaves the concurrent levels' sweeps a small
    // L1 (config-1 estimator 2684 -> 2721 ms when every kernel asked for it)
    if (r == 0 && max_carveout)
        cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    done[key] = r;
    return r;
}

int substep_smem_bytes(const SubArgs& a) { return static_cast<int>(sub_layout(a, nullptr, nullptr)); }

template <int RPT>
static int launch_sub_rpt(const SubArgs& a, int grid, int smem, cudaStream_t st) {
    set_max_dynamic_smem(reinterpret_cast<const void*>(substep_kernel<RPT>), 227 * 1024);
    substep_kernel<RPT><<<grid, kSubThreads, smem, st>>>(a);
    return static_cast<int>(cudaGetLastError());
}

int launch_substeps(const SubArgs& a, int grid, void* stream) {
    const int smem = substep_smem_bytes(a);
    const int rpt = (a.n_r + kSubThreads - 1) / kSubThreads;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (rpt) {
        case 0:
        case 1: return launch_sub_rpt<1>(a, grid, smem, st);
        case 2: return launch_sub_rpt<2>(a, grid, smem, st);
        case 3: return launch_sub_rpt<3>(a, grid, smem, st);
        case 4: return launch_sub_rpt<4>(a, grid, smem, st);
        case 5: return launch_sub_rpt<5>(a, grid, smem, st);
        case 6: return launch_sub_rpt<6>(a, grid, smem, st);
        case 7: return launch_sub_rpt<7>(a, grid, smem, st);
        case 8: return launch_sub_rpt<8>(a, grid, smem, st);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

int lattice_smem_bytes(const LatArgs& a) { return lat_offsets(a).total * static_cast<int>(sizeof(double)); }

template <int T, int K, int G>
static int launch_lat(const LatArgs& a, int grid, cudaStream_t st) {
    set_max_dynamic_smem(reinterpret_cast<const void*>(lattice_substep_kernel<T, K, G>), 227 * 1024);
    lattice_substep_kernel<T, K, G><<<grid, T, lattice_smem_bytes(a), st>>>(a);
    return static_cast<int>(cudaGetLastError());
}

int launch_lattice_substeps(const LatArgs& a, int grid, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (a.threads == 1024 && a.strip_k == 4) return launch_lat<1024, 4, 1>(a, grid, st);
    if (a.threads == 768 && a.strip_k == 6) return launch_lat<768, 6, 2>(a, grid, st);
    if (a.threads == 512 && a.strip_k == 8) return launch_lat<512, 8, 2>(a, grid, st);
    return static_cast<int>(cudaErrorInvalidValue);
}

int substep_max_grid(int device, int smem_bytes) {
    int sms = 0, optin = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (smem_bytes > optin) return 0;
    return sms;  // one 1024-thread CTA per SM
}

void launch_global_substep(const GSubArgs& a, void* stream) {
    const int rows = kSweepWarps * kSweepRows;
    const unsigned grid = ((a.n_r + rows - 1) / rows) * (a.S / kSweepChunk);
    global_substep_kernel<kSweepRows><<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
}

void launch_tier_stage(const TierArgs& a, void* stream) {
    const int rows = a.row_end - a.row_begin;
    if (rows <= 0) return;
    static const bool wide = [] {
        const char* e = std::getenv("WMC_TIER_WIDE");  // A/B knob (0: the 16-byte form)
        return !(e && std::atoi(e) == 0);
    }();
    if (wide && !a.rel && !a.nsteps && a.S % kSweepChunkW == 0) {
        constexpr int R = 2;
        const unsigned grid = ((rows + kSweepWarps * R - 1) / (kSweepWarps * R)) * (a.S / kSweepChunkW);
        tier_stage_wide_kernel<R, 3><<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
        return;
    }
    const int per = kSweepWarps * kTierRows;
    const unsigned grid = ((rows + per - 1) / per) * (a.S / kSweepChunk);
    tier_stage_kernel<kTierRows><<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
}

void launch_r_update(const RUpdateArgs& a, void* stream) {
    const unsigned grid = ((a.n_r + kSweepWarps - 1) / kSweepWarps) * (a.S / kSweepChunk);
    r_update_kernel<<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
}

void launch_qoi(const QoIArgs& a, void* stream) {
    if (a.sample_major && !a.nsteps) {
        qoi_sm_kernel<<<dim3(a.count, a.nq), 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
        return;
    }
    qoi_kernel<<<dim3((a.count + 127) / 128, a.nq), 128, 0, static_cast<cudaStream_t>(stream)>>>(a);
}

void launch_eig_init(const double* warm, double warm_norm, int n, int S, double* v, void* stream) {
    eig_init_kernel<<<2 * 148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(warm, warm_norm, n, S, v);
}

void launch_eig_iteration(const EigArgs& a, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned grid = ((a.n + kSweepWarps - 1) / kSweepWarps) * (a.S / kSweepChunk);
    eig_matvec_kernel<<<grid, kSweepWarps * 32, 0, st>>>(a);
    eig_dot_kernel<<<dim3(a.S / kSweepChunk, a.n_blocks), kSweepWarps * 32, 0, st>>>(a);
    eig_update_kernel<<<(a.S + 127) / 128, 128, 0, st>>>(a);
    eig_normalize_kernel<<<2 * 148 * 8, 256, 0, st>>>(a);
}

void launch_cfl_finalize(const double* lf, const double* lc, int use_coarse, int p_fine, double safety, double T,
                         double dt_ref, int count, int S, double* rel, int* nsteps, void* stream) {
    cfl_finalize_kernel<<<(S + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        lf, lc, use_coarse, p_fine, safety, T, dt_ref, count, S, rel, nsteps);
}

void launch_fill_int(int* p, int value, int n, void* stream) {
    fill_int_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(p, value, n);
}

void launch_pair_diff(const double* qf, const double* qc, double* dq, double* q_out, int count, int S, int nq,
                      void* stream) {
    pair_diff_kernel<<<dim3((count + 255) / 256, nq), 256, 0, static_cast<cudaStream_t>(stream)>>>(qf, qc, dq, q_out,
                                                                                                  count, S, nq);
}

int small_smem_bytes(const SmallArgs& a) {
    return small_layout(a, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr) * static_cast<int>(sizeof(double));
}

int small_max_smem(int device) {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, small_solve_kernel) != cudaSuccess) return 0;
    return optin - static_cast<int>(fa.sharedSizeBytes);  // the kernel also holds static shared memory
}

int launch_small_solve(const SmallArgs& a, int grid, void* stream) {
    int device = 0;
    cudaGetDevice(&device);
    const int configured = set_max_dynamic_smem(reinterpret_cast<const void*>(small_solve_kernel), small_max_smem(device));
    if (configured != 0) return configured;
    small_solve_kernel<<<grid, kSmallThreads, small_smem_bytes(a), static_cast<cudaStream_t>(stream)>>>(a);
    return static_cast<int>(cudaGetLastError());
}



int lattice_solve_smem_bytes(const LatSolveArgs& a) {
    return lat_solve_offsets(a).total * static_cast<int>(sizeof(double));
}

int lattice_solve_max_smem(int device) {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, lattice_solve_kernel<512, 8, 2, false>) != cudaSuccess) return 0;
    cudaFuncAttributes fb{};
    if (cudaFuncGetAttributes(&fb, lattice_solve_kernel<512, 8, 2, true>) != cudaSuccess) return 0;
    if (fb.sharedSizeBytes > fa.sharedSizeBytes) fa.sharedSizeBytes = fb.sharedSizeBytes;
    return optin - static_cast<int>(fa.sharedSizeBytes);
}

template <int T, int K, int G, bool TM, bool VT, bool PK = false>
static int launch_lat_solve(const LatSolveArgs& a, int grid, cudaStream_t st) {
    int device = 0;
    cudaGetDevice(&device);
    const int configured = set_max_dynamic_smem(
        reinterpret_cast<const void*>(lattice_solve_kernel<T, K, G, TM, VT, PK>), lattice_solve_max_smem(device));
    if (configured != 0) return configured;
    lattice_solve_kernel<T, K, G, TM, VT, PK><<<grid, T, lattice_solve_smem_bytes(a), st>>>(a);
    return static_cast<int>(cudaGetLastError());
}

int launch_lattice_solve(const LatSolveArgs& a, int grid, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (a.lat.threads == 512 && a.lat.strip_k == 8)
        return a.tmem == 2 ? (a.strips_k_or_k1 ? launch_lat_solve<512, 8, 2, true, false, true>(a, grid, st)
                                               : launch_lat_solve<512, 8, 2, true, false>(a, grid, st))
               : a.tmem    ? launch_lat_solve<512, 8, 2, true, true>(a, grid, st)
                           : launch_lat_solve<512, 8, 2, false, false>(a, grid, st);
    return static_cast<int>(cudaErrorInvalidValue);
}


void launch_draw_channel(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S,
                         const ChannelArgs& a, double* cells, void* stream) {
    const unsigned grid = static_cast<unsigned>((S + 127) / 128) * static_cast<unsigned>(a.n_ent + 1);
    draw_channel_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(seed, level, first, count, S, a, cells);
}

}  // namespace wmc
