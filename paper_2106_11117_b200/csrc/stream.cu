// Streamed interior of the temporally blocked LF-LTS step (sm_100a, FP64):
// one global step of the reference's lts_step (src/integrators.cpp:117-157)
// for the box nodes of R far from the box ring (host/tiles.hpp plans which).
//
// A work item is (slab, sample).  A slab is a band of up to kStreamThreads
// box rows (one thread per row, so a column of the band is one coalesced
// sample-major load) swept along the box columns.  Iteration t:
//   level 0  z_n of column t arrives (prefetched one iteration earlier)
//   level 1  g = A z_n on column t - 1 and d_1 = -c0 g
//   level m  d_m on column t - m (m = 2 .. p): the recursion
//            d_m = (1 + beta) d_{m-1} - beta d_{m-2} - c (g + A P d_{m-1})
//            needs d_{m-1} on columns t - m - 1 .. t - m + 1 of its own row --
//            the last one produced by level m - 1 earlier in this iteration --
//            and on the rows above and below (published by the neighbour
//            threads in the previous iteration)
//   final    z_{n+1} = 2 z_n - z_{n-1} + 2 d_p on column t - p (owned only).
// Every level keeps its last three columns in registers (the phase t mod 3 is
// a template argument, so the window never moves); a level's value for the
// row neighbours goes through shared memory, double-buffered by the iteration
// parity: one barrier per iteration for all p levels.  g waits p iterations
// for its last use in a per-thread ring in tensor memory (stored twice, so
// one 16-column load reads an iteration's eight values).  The CTA size is the
// slabs' row count rounded to four warps (planned per level: 128 threads and
// four CTAs per SM for config 3); a launch may cut a slab's columns into
// chunks (work items of even length over the grid's rounds).  Global
// addresses are running pointers, z_n / z_{n-1} arrive a column ahead in
// registers (consumed raw an iteration later) and six columns ahead in L2.
//
// The region is the owned band grown by p rows / columns; positions near its
// edge see zeros for missing neighbours, an error that moves one column or
// row per level and never reaches the owned positions.  Lattice values are
// v = d / h (h a power of two) with conductances scaled by 1 / h^2, as in the
// tile kernel (tile.cu).
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "kernels.cuh"

namespace wmc {
namespace {

constexpr int kT = kStreamThreads;
constexpr int kPS = kT + 2;  // publish stride (guard rows 0 and kT + 1, always zero)
constexpr int kRing = 16;    // g ring slots per thread (>= p)
static_assert(kRing >= 2 * kStreamMaxP && (kRing & (kRing - 1)) == 0, "g ring");

struct Cond {
    double dg, kE, kW, kN, kS;
};

// conductances (scaled by 1 / h^2) of a node whose W / E squares lie in cell
// columns key & 0xffff / key >> 16, N / S squares in cell rows cu / cd
__device__ __forceinline__ Cond cond_of(const StreamArgs& a, int key, int cu, int cd, int s, double half) {
    const std::size_t S = static_cast<std::size_t>(a.S);
    const int x0 = key & 0xffff, x1 = key >> 16;
    const double U0 = __ldg(a.cells + static_cast<std::size_t>(cu + x0) * S + s);
    const double U1 = __ldg(a.cells + static_cast<std::size_t>(cu + x1) * S + s);
    const double D0 = __ldg(a.cells + static_cast<std::size_t>(cd + x0) * S + s);
    const double D1 = __ldg(a.cells + static_cast<std::size_t>(cd + x1) * S + s);
    Cond c;
    c.kE = (U1 + D1) * half;
    c.kW = (U0 + D0) * half;
    c.kN = (U0 + U1) * half;
    c.kS = (D0 + D1) * half;
    c.dg = c.kE + c.kW + c.kN + c.kS;
    return c;
}

// g ring in tensor memory, 16 slots (a slot = 2 columns of the thread's lane)
// stored twice, at q and q + 16, so the 8 consecutive columns an iteration
// needs never wrap: one 16-column load with the slot base in a uniform
// register instead of a load (and its address arithmetic) per level
__device__ __forceinline__ void ring_put(std::uint32_t tb, int slot, double g) {
    asm volatile("{\n.reg .b32 lo, hi;\nmov.b64 {lo, hi}, %1;\n"
                 "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {lo, hi};\n"
                 "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0 + 32], {lo, hi};\n}\n"
                 :
                 : "r"(tb + 2u * static_cast<std::uint32_t>(slot)), "d"(g)
                 : "memory");
}
// g of columns t - 8 .. t - 1 (g[8 - lv] for level lv; the last one is not
// written yet and unused); the previous iteration's store is waited for first
__device__ __forceinline__ void ring_get8(std::uint32_t tb, int t, double (&g)[8]) {
    const std::uint32_t ad = tb + 2u * static_cast<std::uint32_t>((t - 8) & (kRing - 1));
    asm volatile(
        "{\n.reg .b32 l<16>;\n"
        "tcgen05.wait::st.sync.aligned;\n"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {l0, l1, l2, l3, l4, l5, l6, l7, l8, l9, l10, l11, l12, l13, l14, l15}, "
        "[%8];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        "mov.b64 %0, {l0, l1};\nmov.b64 %1, {l2, l3};\nmov.b64 %2, {l4, l5};\nmov.b64 %3, {l6, l7};\n"
        "mov.b64 %4, {l8, l9};\nmov.b64 %5, {l10, l11};\nmov.b64 %6, {l12, l13};\nmov.b64 %7, {l14, l15};\n}\n"
        : "=d"(g[0]), "=d"(g[1]), "=d"(g[2]), "=d"(g[3]), "=d"(g[4]), "=d"(g[5]), "=d"(g[6]), "=d"(g[7])
        : "r"(ad)
        : "memory");
}

constexpr int kAhead = 6;
__device__ __forceinline__ void l2_prefetch(const double* p) {
    asm volatile("prefetch.global.L2 [%0];\n" : : "l"(p));
}

template <int P>
__global__ void __launch_bounds__(kT, 2) stream_step_kernel(StreamArgs a) {
    static_assert(P >= 2 && P <= kStreamMaxP, "levels");
    extern __shared__ __align__(16) double sd[];
    __shared__ std::uint32_t tm_slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    double* pub = sd;  // [level][parity][kPS]
    int* ckey = reinterpret_cast<int*>(sd + P * 2 * kPS);
    const int nthr = blockDim.x;
    for (int q = tid; q < P * 2 * kPS; q += nthr) pub[q] = 0.0;

    // tensor memory: 128 columns; warps w and w + 4 share lanes 32 (w % 4)..
    // and take columns 0 / 64 (the doubled g ring, 32 doubles)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n"
                     "tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n"
                     :
                     : "r"(static_cast<std::uint32_t>(__cvta_generic_to_shared(&tm_slot)))
                     : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const std::uint32_t tb = tm_slot + (static_cast<std::uint32_t>(32 * (warp & 3)) << 16) + 64u * (warp >> 2);

    const int W = a.m + 1, m = a.m;
    const double half = 0.5 * a.inv_h2, inv_h = a.inv_h, h2 = 2.0 * a.h, c0 = a.c0;
    const int per_sample = a.n_slabs * a.chunks;
    const int items = per_sample * a.count;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        // a sample's slabs (and a slab's column chunks) on neighbouring CTAs
        const int s = item / per_sample, rest = item - s * per_sample;
        const int sl = rest / a.chunks, ch = rest - sl * a.chunks;
        const int4 geo = __ldg(a.slab + sl);
        int4 own = __ldg(a.slab_own + sl);
        // chunk ch of the owned columns (own.x == p: the region leads by p columns)
        const int q0 = ch * a.chunk_cols, q1 = min(own.y - own.x, q0 + a.chunk_cols);
        const int I0 = geo.x + q0, NX = q1 - q0 + 2 * own.x, J0 = geo.z, NY = geo.w;
        own.y = own.x + q1 - q0;
        __syncthreads();  // the previous item's key readers are done
        for (int x = tid; x < NX; x += nthr) {
            const int i = I0 + x;
            ckey[x] = __ldg(a.cellx + min(max(i - 1, 0), m - 1)) | (__ldg(a.cellx + min(max(i, 0), m - 1)) << 16);
        }
        const int y = tid, j = J0 + y;
        const bool row_ok = y < NY;
        const bool own_row = y >= own.z && y < own.w;
        const int cu = __ldg(a.celly + min(max(j, 0), m - 1)) * a.cells_x;
        const int cd = __ldg(a.celly + min(max(j - 1, 0), m - 1)) * a.cells_x;
        const std::size_t base = static_cast<std::size_t>(s) * a.n + (row_ok ? j : J0);
        const double* __restrict__ zs = a.zc + base;  // + column * W
        double* __restrict__ zo = a.zp + base;
        __syncthreads();  // ckey

        auto key = [&](int x) { return ckey[min(max(x, 0), NX - 1)]; };
        double w[P][3];
#pragma unroll
        for (int q = 0; q < P; ++q) w[q][0] = w[q][1] = w[q][2] = 0.0;
        // prefetched one iteration ahead and consumed raw at the start of the
        // next one (any arithmetic on the loaded value here would wait for it)
        double znext = row_ok ? __ldg(zs + static_cast<std::size_t>(I0) * W) : 0.0;
        // running pointers (advanced a column per iteration; recomputing the
        // addresses from t cost ~35 integer instructions per iteration):
        // z_n of column t + 1, and z_n / z_{n-1} of the final's column t + 1 - P
        const std::ptrdiff_t Wd = W;
        const double* pz = zs + static_cast<std::ptrdiff_t>(I0 + 1) * Wd;
        const double* pfz = zs + static_cast<std::ptrdiff_t>(I0 + 1 - P) * Wd;
        double* pzo = zo + static_cast<std::ptrdiff_t>(I0 + 1 - P) * Wd;
        // L2 prefetch lanes: one request per 128-byte line of the warp's rows,
        // lanes 0 / 16 for z_n, 8 / 24 for z_{n-1}
        const bool pf_lane = row_ok && (tid & 7) == 0, pf_zo = (tid & 8) != 0;
        const std::ptrdiff_t ahead = static_cast<std::ptrdiff_t>(kAhead) * Wd;
        double fz_next = 0.0, fp_next = 0.0;  // z_n, z_{n-1} of the final column
        double wv_cur = 0.0;                  // 2 z_n - z_{n-1} of the final column
        int cur_key = -1;
        Cond K{0.0, 0.0, 0.0, 0.0, 0.0};
        bool bad = false;
        const int NT = NX + P;

        auto body = [&](auto ph, auto slow, int t) {
            constexpr int PH = decltype(ph)::value;
            constexpr bool kSlow = decltype(slow)::value;
            constexpr int C = PH, P1 = (PH + 2) % 3, P2 = (PH + 1) % 3;  // window slots: this, previous, before
            double gv[8];
            ring_get8(tb, t, gv);
            // level 0: z_n of column t; prefetch column t + 1 and the final's
            // w of column t + 1 - P
            w[0][C] = znext * inv_h;
            wv_cur = 2.0 * fz_next - fp_next;
            {
                const int xn = t + 1, xf = t + 1 - P;
                znext = row_ok && xn < NX ? __ldg(pz) : 0.0;
                if (own_row && xf >= own.x && xf < own.y) {
                    fz_next = __ldg(pfz);
                    fp_next = *pzo;
                }
                // the columns kAhead iterations on, into L2 (an iteration is
                // about as long as a loaded DRAM access)
                if (pf_lane) {
                    const int xa = (pf_zo ? xf : xn) + kAhead;
                    if (pf_zo ? (xa >= own.x && xa < own.y) : xa < NX) l2_prefetch((pf_zo ? pzo : pz) + ahead);
                }
            }
            const double* rd = pub + ((t - 1) & 1) * kPS + 1 + y;  // published in the previous iteration
            double* wr = pub + (t & 1) * kPS + 1 + y;
            // (the levels' values are published after the last level: a store
            // between two levels' neighbour loads would order them -- the
            // compiler cannot see that the two parity buffers never alias --
            // and chain load -> FP64 -> store level by level)
            // level 1: g on column t - 1
            {
                const Cond k = kSlow ? cond_of(a, key(t - 1), cu, cd, s, half) : K;
                const double g = k.dg * w[0][P1] - k.kE * w[0][C] - k.kW * w[0][P2] - k.kN * rd[1] - k.kS * rd[-1];
                ring_put(tb, (t - 1) & (kRing - 1), g);
                w[1][C] = -c0 * g;
            }
#pragma unroll
            for (int lv = 2; lv <= P; ++lv) {
                const Cond k = kSlow ? cond_of(a, key(t - lv), cu, cd, s, half) : K;
                const double* r = rd + (lv - 1) * 2 * kPS;
                const double vO = w[lv - 1][P1];
                const double vprev = lv >= 3 ? w[lv >= 3 ? lv - 2 : 0][P2] : 0.0;
                // d_lv = (1 + beta) d - beta d_prev - c (g + A d) in 8 FP64
                // operations; the E neighbour -- formed a moment ago by level
                // lv - 1 in this iteration -- enters last, so the levels of
                // one iteration overlap except for two operations each.
                // (Writing the levels' independent parts as seven interleaved
                // chains spilled and ran slower: 3.49 vs 2.84 ms per step.)
                const double rest =
                    fma(-k.kS, r[-1], fma(-k.kN, r[1], fma(-k.kW, w[lv - 1][P2], fma(k.dg, vO, gv[8 - lv]))));
                const double q = fma(a.opb[lv - 2], vO, -(a.beta[lv - 2] * vprev));
                const double nx = fma(-a.cm[lv - 2], fma(-k.kE, w[lv - 1][C], rest), q);
                if (lv < P) {
                    w[lv < P ? lv : 0][C] = nx;
                } else {
                    const int xf = t - P;
                    if (own_row && xf >= own.x && xf < own.y) {
                        const double out = wv_cur + h2 * nx;
                        pzo[-Wd] = out;  // column t - P
                        bad |= !(fabs(out) <= 1e100);
                    }
                }
            }
#pragma unroll
            for (int lv = 0; lv < P; ++lv) wr[lv * 2 * kPS] = w[lv][C];
            pz += Wd;
            pfz += Wd;
            pzo += Wd;
            __syncthreads();
        };
        // fast iterations: every level's column in one run of equal cell
        // columns (cellx is monotone, so the two ends decide) with the
        // conductances held in registers; slow ones read them per level
        auto step = [&](auto ph, int t) {
            const int k1 = key(t - 1), kp = key(t - P);
            if (k1 == kp) {
                if (k1 != cur_key) {
                    K = cond_of(a, k1, cu, cd, s, half);
                    cur_key = k1;
                }
                body(ph, std::false_type{}, t);
            } else {
                body(ph, std::true_type{}, t);
            }
        };
        for (int t0 = 0; t0 < NT; t0 += 3) {
            step(std::integral_constant<int, 0>{}, t0);
            if (t0 + 1 < NT) step(std::integral_constant<int, 1>{}, t0 + 1);
            if (t0 + 2 < NT) step(std::integral_constant<int, 2>{}, t0 + 2);
        }
        if (bad && s < a.count) atomicMin(a.fail + s, a.step);
    }

    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" : : "r"(tm_slot) : "memory");
}

template <int P>
int launch_p(const StreamArgs& a, int grid, void* stream) {
    const int smem = stream_smem_bytes(a);
    // (the device maximum, set once per kernel and device: levels of one
    // process differ in their column-key array)
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem + 64 > optin) return static_cast<int>(cudaErrorInvalidValue);
    const int e = set_max_dynamic_smem(reinterpret_cast<const void*>(stream_step_kernel<P>), optin - 64, true);
    if (e != 0) return e;
    stream_step_kernel<P><<<grid, a.threads, smem, static_cast<cudaStream_t>(stream)>>>(a);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace

int stream_smem_bytes(const StreamArgs& a) {
    return static_cast<int>(sizeof(double)) * a.p * 2 * kPS + static_cast<int>(sizeof(int)) * (a.max_nx + 2);
}

int launch_stream_step(const StreamArgs& a, int grid, void* stream) {
    switch (a.p) {
        case 2: return launch_p<2>(a, grid, stream);
        case 3: return launch_p<3>(a, grid, stream);
        case 4: return launch_p<4>(a, grid, stream);
        case 5: return launch_p<5>(a, grid, stream);
        case 6: return launch_p<6>(a, grid, stream);
        case 7: return launch_p<7>(a, grid, stream);
        case 8: return launch_p<8>(a, grid, stream);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

}  // namespace wmc
