// sm_100a kernels of the batched LF / LF-LTS sample evaluator.  See
// kernels.cuh for the layout and DESIGN.md for the roofline of each kernel.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "kernels.cuh"

namespace wmc {

namespace {

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

__device__ __forceinline__ void flag_fail(int* fail, int s, int count, int step) {
    if (s < count) atomicMin(fail + s, step);
}

// ---------------------------------------------------------------------------
// K1: the full sweep g = A(omega) z over every row, one warp per (row, 64
// samples), 16-byte loads per lane.  A(omega)_ij = sum_k c_k a0_ijk
// ("parts"), gathered node-centrically: no atomics, deterministic.
// Rows < split stash g for the substep kernel; the others take the
// leapfrog update z+ = 2 z - z- - factor * g in place of z-
// (reference src/integrators.cpp:89-115; for LTS rows outside R the
// recursion collapses to factor = -2 d_p(g = 1), :117-157).

template <bool kInit>
__global__ void __launch_bounds__(kSweepWarps * 32) sweep_kernel(SweepArgs a) {
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * kSweepWarps + (threadIdx.x >> 5);
    if (row >= a.n) return;
    const int s0 = blockIdx.y * kSweepChunk + 2 * lane;
    const std::size_t S = static_cast<std::size_t>(a.S);
    const int b = __ldg(a.row_ptr + row), e = __ldg(a.row_ptr + row + 1);
    double acc0 = 0.0, acc1 = 0.0;
    for (int k = b; k < e; ++k) {
        const int pk = __ldg(a.ent + k);
        const double w = __ldg(a.a0 + k);
        const int j = pk & 0xffffff;
        const int cell = static_cast<unsigned>(pk) >> 24;
        const double2 c = __ldg(reinterpret_cast<const double2*>(a.cells + cell * S + s0));
        if (kInit) {
            const double zj = __ldg(a.z0 + j);
            acc0 += (c.x * w) * zj;
            acc1 += (c.y * w) * zj;
        } else {
            const double2 z = __ldg(reinterpret_cast<const double2*>(a.zc + j * S + s0));
            acc0 += (c.x * w) * z.x;
            acc1 += (c.y * w) * z.y;
        }
    }
    const std::size_t idx = row * S + s0;
    if (kInit) {
        // z1 = z0 + dt M^{1/2} v0 + dt^2/2 (F0 - A z0), v0 = F = 0 (integrators.cpp:68-87)
        const double z0 = __ldg(a.z0 + row);
        double2 out;
        out.x = z0 + a.factor * (0.0 - acc0);
        out.y = z0 + a.factor * (0.0 - acc1);
        *reinterpret_cast<double2*>(a.zp + idx) = make_double2(z0, z0);
        *reinterpret_cast<double2*>(a.zc_out + idx) = out;
        if (!(fabs(out.x) <= 1e100)) flag_fail(a.fail, s0, a.count, a.step);
        if (!(fabs(out.y) <= 1e100)) flag_fail(a.fail, s0 + 1, a.count, a.step);
        return;
    }
    if (row < a.split) {
        *reinterpret_cast<double2*>(a.g + idx) = make_double2(acc0, acc1);
        return;
    }
    const double2 zn = *reinterpret_cast<const double2*>(a.zc + idx);
    const double2 zm = *reinterpret_cast<const double2*>(a.zp + idx);
    double2 out;
    out.x = 2.0 * zn.x - zm.x - a.factor * acc0;
    out.y = 2.0 * zn.y - zm.y - a.factor * acc1;
    *reinterpret_cast<double2*>(a.zp + idx) = out;
    // check_finite (integrators.cpp:12-18): non-finite or |z| > 1e100
    if (!(fabs(out.x) <= 1e100)) flag_fail(a.fail, s0, a.count, a.step);
    if (!(fabs(out.y) <= 1e100)) flag_fail(a.fail, s0 + 1, a.count, a.step);
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
    const std::size_t ol = take(sizeof(double) * a.n_cells);
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
        __syncthreads();  // previous sample done with cl / W / d buffers
        for (int k = tid; k < a.n_cells; k += kSubThreads) sm.cl[k] = __ldg(a.cells + k * S + s);
        __syncthreads();
        for (int w = tid; w < a.n_wid; w += kSubThreads) {
            double acc = 0.0;
            for (int t = __ldg(a.rc_ptr + w); t < __ldg(a.rc_ptr + w + 1); ++t)
                acc += sm.cl[__ldg(a.rc_cell + t)] * __ldg(a.rc_a0 + t);
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
                g[k] = __ldg(a.g + r * S + s);
                dc[k] = -a.c0 * g[k];
                sm.d0[r] = dc[k];
            }
        }
        __syncthreads();

        for (int m = 1; m <= a.p - 1; ++m) {
            const double* cur = (m & 1) ? sm.d0 : sm.d1;
            double* nxt = (m & 1) ? sm.d1 : sm.d0;
            const double beta = sm.beta[m - 1];
            const double cm = sm.cm[m - 1];
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
            if (r < a.n_r) {
                const std::size_t idx = r * S + s;
                const double zn = a.zc[idx];
                const double zm = a.zp[idx];
                const double out = 2.0 * zn - zm + 2.0 * dc[k];
                a.zp[idx] = out;
                if (!(fabs(out) <= 1e100)) atomicMin(a.fail + s, a.step);
            }
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

struct LatSmem {
    double* v0;
    double* v1;
    double* gw;
    double* cl;
    double* beta;
    double* cm;
    std::uint16_t* gcol;
    int* gsoff;
    int* sj0;
    int* slen;
    int* cx;
    int* cy;
};

__host__ __device__ inline std::size_t lat_layout(const LatArgs& a, char* base, LatSmem* s) {
    const int n_slices = (a.n_gen + 31) / 32;
    std::size_t off = 0;
    auto take = [&](std::size_t bytes) {
        const std::size_t o = off;
        off = align16(off + bytes);
        return o;
    };
    const std::size_t o0 = take(sizeof(double) * a.n_r);
    const std::size_t o1 = take(sizeof(double) * a.n_r);
    const std::size_t ow = take(sizeof(double) * (a.n_slots > 0 ? a.n_slots : 1));
    const std::size_t ol = take(sizeof(double) * a.n_cells);
    const std::size_t ob = take(sizeof(double) * (a.p > 1 ? a.p - 1 : 1));
    const std::size_t oc = take(sizeof(double) * (a.p > 1 ? a.p - 1 : 1));
    const std::size_t og = take(sizeof(std::uint16_t) * (a.n_slots > 0 ? a.n_slots : 1));
    const std::size_t os = take(sizeof(int) * (n_slices + 1));
    const std::size_t oj = take(sizeof(int) * a.n_strips);
    const std::size_t olen = take(sizeof(int) * a.n_strips);
    const std::size_t ox = take(sizeof(int) * a.m);
    const std::size_t oy = take(sizeof(int) * a.m);
    if (s) {
        s->v0 = reinterpret_cast<double*>(base + o0);
        s->v1 = reinterpret_cast<double*>(base + o1);
        s->gw = reinterpret_cast<double*>(base + ow);
        s->cl = reinterpret_cast<double*>(base + ol);
        s->beta = reinterpret_cast<double*>(base + ob);
        s->cm = reinterpret_cast<double*>(base + oc);
        s->gcol = reinterpret_cast<std::uint16_t*>(base + og);
        s->gsoff = reinterpret_cast<int*>(base + os);
        s->sj0 = reinterpret_cast<int*>(base + oj);
        s->slen = reinterpret_cast<int*>(base + olen);
        s->cx = reinterpret_cast<int*>(base + ox);
        s->cy = reinterpret_cast<int*>(base + oy);
    }
    return off;
}

__global__ void __launch_bounds__(kLatThreads, 1) lattice_substep_kernel(LatArgs a) {
    extern __shared__ __align__(16) char smem[];
    LatSmem sm;
    lat_layout(a, smem, &sm);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int n_slices = (a.n_gen + 31) / 32;
    const std::size_t S = static_cast<std::size_t>(a.S);
    const int W = a.m + 1;

    for (int i = tid; i < a.n_slots; i += kLatThreads) sm.gcol[i] = __ldg(a.gen_col + i);
    for (int i = tid; i <= n_slices; i += kLatThreads) sm.gsoff[i] = __ldg(a.gen_soff + i);
    for (int i = tid; i < a.n_strips; i += kLatThreads) {
        sm.sj0[i] = __ldg(a.strip_j0 + i);
        sm.slen[i] = __ldg(a.strip_len + i);
    }
    for (int i = tid; i < a.m; i += kLatThreads) {
        sm.cx[i] = __ldg(a.cellx + i);
        sm.cy[i] = __ldg(a.celly + i);
    }
    for (int i = tid; i < a.p - 1; i += kLatThreads) {
        sm.beta[i] = __ldg(a.beta + i);
        sm.cm[i] = __ldg(a.cm + i);
    }

    // structured role
    const int col = tid % a.cw, strip = tid / a.cw;
    const int ci = 1 + col;
    const bool lat_on = ci <= a.m - 1 && strip < a.n_strips;
    // generic role
    int gq[kLatGen];
#pragma unroll
    for (int u = 0; u < kLatGen; ++u) gq[u] = tid + u * kLatThreads;

    for (int s = blockIdx.x; s < a.count; s += gridDim.x) {
        __syncthreads();
        for (int k = tid; k < a.n_cells; k += kLatThreads) sm.cl[k] = __ldg(a.cells + k * S + s);
        __syncthreads();
        for (int e = tid; e < a.n_slots; e += kLatThreads) {
            double acc = 0.0;
            for (int t = __ldg(a.slot_rc + e); t < __ldg(a.slot_rc + e + 1); ++t)
                acc += sm.cl[__ldg(a.rc_cell + t)] * __ldg(a.rc_a0 + t);
            sm.gw[e] = acc;
        }

        // lattice constants of this thread (scaled by 1/h: v = d/h)
        int j0 = 1, len = 0;
        double kE0 = 0, kW0 = 0, kN0 = 0, kS0 = 0, dg0 = 0, kE = 0, kW = 0, kNS = 0, dg = 0;
        double d[kLatStrip], dp[kLatStrip], gg[kLatStrip];
        if (lat_on) {
            j0 = sm.sj0[strip];
            len = sm.slen[strip];
            const int rowu = sm.cy[j0] * a.cells_x, rowd = sm.cy[j0 - 1] * a.cells_x;
            const double cRu = sm.cl[rowu + sm.cx[ci]], cRd = sm.cl[rowd + sm.cx[ci]];
            const double cLu = sm.cl[rowu + sm.cx[ci - 1]], cLd = sm.cl[rowd + sm.cx[ci - 1]];
            const double f = 0.5 * a.inv_h;
            kE0 = (cRu + cRd) * f;
            kW0 = (cLu + cLd) * f;
            kN0 = (cLu + cRu) * f;
            kS0 = (cLd + cRd) * f;
            dg0 = kE0 + kW0 + kN0 + kS0;
            kE = cRu * a.inv_h;
            kW = cLu * a.inv_h;
            kNS = (cLu + cRu) * f;
            dg = kE + kW + 2.0 * kNS;
        }
#pragma unroll
        for (int k = 0; k < kLatStrip; ++k) {
            d[k] = 0.0;
            dp[k] = 0.0;
            gg[k] = 0.0;
            if (k < len) {
                const int dof = (j0 + k) * W + ci;
                gg[k] = __ldg(a.g + dof * S + s);
                d[k] = -a.c0 * gg[k];
                sm.v0[dof] = d[k] * a.inv_h;
            }
        }
        double gd[kLatGen], gdp[kLatGen], ggg[kLatGen], grs[kLatGen];
        int grow[kLatGen];
#pragma unroll
        for (int u = 0; u < kLatGen; ++u) {
            gd[u] = gdp[u] = ggg[u] = grs[u] = 0.0;
            grow[u] = -1;
            if (gq[u] < a.n_gen) {
                grow[u] = __ldg(a.gen_rows + gq[u]);
                grs[u] = __ldg(a.gen_rs + gq[u]);
                ggg[u] = __ldg(a.g + grow[u] * S + s);
                gd[u] = -a.c0 * ggg[u];
                sm.v0[grow[u]] = gd[u] * grs[u];
            }
        }
        __syncthreads();

        for (int m = 1; m <= a.p - 1; ++m) {
            const double* cur = (m & 1) ? sm.v0 : sm.v1;
            double* nxt = (m & 1) ? sm.v1 : sm.v0;
            const double beta = sm.beta[m - 1];
            const double cmm = sm.cm[m - 1];
            const double onepb = 1.0 + beta;
            if (len > 0) {
                const int base = j0 * W + ci;
                double vs = cur[base - W];  // south neighbour of the first row (old)
                double vk = d[0] * a.inv_h;  // old v of the current node
#pragma unroll
                for (int k = 0; k < kLatStrip; ++k) {
                    if (k < len) {
                        const int dof = base + k * W;
                        const double vn = (k + 1 < len) ? d[k + 1] * a.inv_h : cur[dof + W];
                        const double ve = cur[dof + 1], vw = cur[dof - 1];
                        double aq;
                        if (k == 0)
                            aq = dg0 * vk - kE0 * ve - kW0 * vw - kN0 * vn - kS0 * vs;
                        else
                            aq = dg * vk - kE * ve - kW * vw - kNS * (vn + vs);
                        const double next = onepb * d[k] - beta * dp[k] - cmm * (gg[k] + aq);
                        dp[k] = d[k];
                        d[k] = next;
                        nxt[dof] = next * a.inv_h;
                        vs = vk;
                        vk = vn;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kLatGen; ++u) {
                if (grow[u] >= 0) {
                    const int slice = gq[u] >> 5;
                    const int b = sm.gsoff[slice], e = sm.gsoff[slice + 1];
                    double aq = 0.0;
                    for (int q = b + lane; q < e; q += 32) aq += sm.gw[q] * cur[sm.gcol[q]];
                    const double next = onepb * gd[u] - beta * gdp[u] - cmm * (ggg[u] + aq);
                    gdp[u] = gd[u];
                    gd[u] = next;
                    nxt[grow[u]] = next * grs[u];
                }
            }
            __syncthreads();
        }

        // z_{n+1} = 2 z_n - z_{n-1} + 2 d_p
#pragma unroll
        for (int k = 0; k < kLatStrip; ++k) {
            if (k < len) {
                const std::size_t idx = static_cast<std::size_t>((j0 + k) * W + ci) * S + s;
                const double out = 2.0 * a.zc[idx] - a.zp[idx] + 2.0 * d[k];
                a.zp[idx] = out;
                if (!(fabs(out) <= 1e100)) atomicMin(a.fail + s, a.step);
            }
        }
#pragma unroll
        for (int u = 0; u < kLatGen; ++u) {
            if (grow[u] >= 0) {
                const std::size_t idx = static_cast<std::size_t>(grow[u]) * S + s;
                const double out = 2.0 * a.zc[idx] - a.zp[idx] + 2.0 * gd[u];
                a.zp[idx] = out;
                if (!(fabs(out) <= 1e100)) atomicMin(a.fail + s, a.step);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K3: QoI per sample, Q = sum_t w_t (z_t / sqrt(M_t)) over the box nodes in a
// fixed order (deterministic); failed samples report NaN.

__global__ void qoi_kernel(QoIArgs a) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= a.count) return;
    const std::size_t S = static_cast<std::size_t>(a.S);
    double acc = 0.0;
    for (int t = 0; t < a.nq; ++t) {
        const int i = __ldg(a.dof + t);
        acc += __ldg(a.w + t) * (a.z[i * S + s] / __ldg(a.sqrt_mass + t));
    }
    a.q[s] = a.fail[s] == INT_MAX ? acc : __longlong_as_double(0x7ff8000000000000LL);
}

__global__ void fill_int_kernel(int* p, int value, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = value;
}

__global__ void pair_diff_kernel(const double* qf, const double* qc, double* dq, int count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) dq[i] = qc ? qf[i] - qc[i] : qf[i];
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

void launch_moments(const double* dq, const double* q, int count, double* out, void* stream) {
    moments_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(dq, q, count, out);
}

void launch_draw_cells(std::uint64_t seed, std::uint32_t level, std::uint64_t first, int count, int S, int n_cells,
                       double lo, double hi, double* cells, void* stream) {
    draw_cells_kernel<<<(S + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, level, first, count, S,
                                                                                       n_cells, lo, hi, cells);
}

void launch_sweep_init(const SweepArgs& a, void* stream) {
    dim3 grid((a.n + kSweepWarps - 1) / kSweepWarps, a.S / kSweepChunk);
    sweep_kernel<true><<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
}

void launch_sweep_step(const SweepArgs& a, void* stream) {
    dim3 grid((a.n + kSweepWarps - 1) / kSweepWarps, a.S / kSweepChunk);
    sweep_kernel<false><<<grid, kSweepWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
}

int substep_smem_bytes(const SubArgs& a) { return static_cast<int>(sub_layout(a, nullptr, nullptr)); }

template <int RPT>
static int launch_sub_rpt(const SubArgs& a, int grid, int smem, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(substep_kernel<RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        configured = true;
    }
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

int lattice_smem_bytes(const LatArgs& a) { return static_cast<int>(lat_layout(a, nullptr, nullptr)); }

int launch_lattice_substeps(const LatArgs& a, int grid, void* stream) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(lattice_substep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        configured = true;
    }
    lattice_substep_kernel<<<grid, kLatThreads, lattice_smem_bytes(a), static_cast<cudaStream_t>(stream)>>>(a);
    return static_cast<int>(cudaGetLastError());
}

int substep_max_grid(int device, int smem_bytes) {
    int sms = 0, optin = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (smem_bytes > optin) return 0;
    return sms;  // one 1024-thread CTA per SM
}

void launch_qoi(const QoIArgs& a, void* stream) {
    qoi_kernel<<<(a.count + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(a);
}

void launch_fill_int(int* p, int value, int n, void* stream) {
    fill_int_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(p, value, n);
}

void launch_pair_diff(const double* qf, const double* qc, double* dq, int count, void* stream) {
    pair_diff_kernel<<<(count + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(qf, qc, dq, count);
}

}  // namespace wmc
