// Temporally blocked LF-LTS step on R (sm_100a, FP64): one global step of
// the reference's lts_step (src/integrators.cpp:117-157) for the rows of R,
// a spatial tile at a time, with every substep on chip.
//
// A work item is (tile, sample).  Its region is kTileWz x kTileHz positions
// of the refined-square lattice around the tile's owned rectangle plus the
// tile's generic rows (box ring, R rows outside the box; host/tiles.hpp).
//   1. z_n of the region in:        v = z / sqrt(M)  (shared memory, buffer 0)
//   2. g = A z_n:                   lattice 5-point stencil / generic SELL on
//                                   v plus the non-P columns from HBM
//   3. d_1 = -c0 g, then p - 1 substeps
//      d_{m+1} = (1 + beta_m) d_m - beta_m d_{m-1} - c_m (g + A P d_m)
//      with v double-buffered in shared memory (one barrier per substep)
//   4. owned rows: z_{n+1} = 2 z_n - z_{n-1} + 2 d_p, check_finite.
// Values near the region's edge are wrong (missing neighbours) but the
// planner proved the error cannot travel to an owned row in p substeps.
//
// Thread = 2 adjacent columns x kTileK rows of the region (a strip).  A
// lattice node keeps v = d / h (h = h_min, a power of two: v and d carry the
// same bits scaled, so the recursion runs on v directly with conductances
// scaled by 1 / h^2) in registers; g and v_{m-1} live in the thread's
// tensor-memory columns (tcgen05.ld / st: their own datapath beside the
// shared-memory pipe the stencil is bound by).  E/W neighbours come from the
// other threads' columns in shared memory (even and odd columns stored apart,
// so a warp's 32 loads hit 32 consecutive column positions: conflict-free),
// N/S neighbours inside the strip from registers.  Generic rows keep d in
// registers and publish v = d / sqrt(M).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <type_traits>

#include "kernels.cuh"

namespace wmc {
namespace {

constexpr int kT = kTileThreads;
constexpr int kK = kTileK;
constexpr int kTPC = kTileWz / 2;          // thread columns per strip row (wide shape)
static_assert(kTPC % 32 == 0 && kT == kTPC * (kTileHz / kK) && kT % 128 == 0, "tile shape");
static_assert(32 % (kTileHz / 2) == 0 || (kTileHz / 2) % 32 == 0, "tall shape: strips per warp");
constexpr int kTmCols = 128 * (kT / 128);  // tensor-memory columns of a CTA (128 per four warps)

__device__ __forceinline__ void t_ld16(std::uint32_t addr, std::uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
}
__device__ __forceinline__ void t_st16(std::uint32_t addr, const std::uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
        "tcgen05.wait::st.sync.aligned;\n"
        :
        : "r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void t_ld8(std::uint32_t addr, std::uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
}
__device__ __forceinline__ void t_st8(std::uint32_t addr, const std::uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                 "tcgen05.wait::st.sync.aligned;\n"
                 :
                 : "r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ double t_dbl(const std::uint32_t* r) {
    return __hiloint2double(static_cast<int>(r[1]), static_cast<int>(r[0]));
}
__device__ __forceinline__ void t_put(std::uint32_t* r, double d) {
    r[0] = static_cast<std::uint32_t>(__double2loint(d));
    r[1] = static_cast<std::uint32_t>(__double2hiint(d));
}
// 4 doubles <-> 8 TMEM columns, the 32-bit halves packed / unpacked inside
// the asm so the doubles land in aligned register pairs (no moves)
__device__ __forceinline__ void t_ld4d(std::uint32_t addr, double (&d)[4]) {
    asm volatile(
        "{\n.reg .b32 t<8>;\n"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {t0,t1,t2,t3,t4,t5,t6,t7}, [%4];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        "mov.b64 %0, {t0,t1};\nmov.b64 %1, {t2,t3};\nmov.b64 %2, {t4,t5};\nmov.b64 %3, {t6,t7};\n}\n"
        : "=d"(d[0]), "=d"(d[1]), "=d"(d[2]), "=d"(d[3])
        : "r"(addr));
}
__device__ __forceinline__ void t_st4d(std::uint32_t addr, double d0, double d1, double d2, double d3) {
    asm volatile(
        "{\n.reg .b32 t<8>;\n"
        "mov.b64 {t0,t1}, %1;\nmov.b64 {t2,t3}, %2;\nmov.b64 {t4,t5}, %3;\nmov.b64 {t6,t7}, %4;\n"
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {t0,t1,t2,t3,t4,t5,t6,t7};\n"
        "tcgen05.wait::st.sync.aligned;\n}\n"
        :
        : "r"(addr), "d"(d0), "d"(d1), "d"(d2), "d"(d3)
        : "memory");
}

// conductances (scaled by 1 / h^2) of the thread's two columns: rows 1 ..
// K-1 of a strip see one coefficient row (squares ia - 1, ia, ib)
struct ColConst {
    double kWa, kEa, kNSa, dga;  // column a (kWb = kEa)
    double kEb, kNSb, dgb;       // column b
};

// row 0 of a strip starting on a coefficient line: conductances from the
// coefficient rows above (U) and below (D) the line, recomputed from the
// shared-memory cell table each time (only such warps take this path)
struct LineCells {
    int cu, cd, x0, x1, x2;
};
__device__ __forceinline__ void line_row0(const double* cl, const LineCells& lc, double s2, double va, double vb,
                                          double vWa, double vEb, double vNa, double vSa, double vNb, double vSb,
                                          double& aqa, double& aqb) {
    const double U0 = cl[lc.cu + lc.x0], U1 = cl[lc.cu + lc.x1], U2 = cl[lc.cu + lc.x2];
    const double D0 = cl[lc.cd + lc.x0], D1 = cl[lc.cd + lc.x1], D2 = cl[lc.cd + lc.x2];
    const double h2 = 0.5 * s2;
    const double kEa = (U1 + D1) * h2, kWa = (U0 + D0) * h2, kNa = (U0 + U1) * h2, kSa = (D0 + D1) * h2;
    const double kEb = (U2 + D2) * h2, kNb = (U1 + U2) * h2, kSb = (D1 + D2) * h2;
    aqa = (kEa + kWa + kNa + kSa) * va - kEa * vb - kWa * vWa - kNa * vNa - kSa * vSa;
    aqb = (kEb + kEa + kNb + kSb) * vb - kEb * vEb - kEa * va - kNb * vNb - kSb * vSb;
}

// A v on the thread's two columns, row k (v units): column a's E neighbour is
// column b and column b's W neighbour column a (registers); the far sides
// from shared memory; S from the previous row (pa / pb: that row's values
// before this substep overwrote them), N from the next row or the strip end
template <int k>
__device__ __forceinline__ void lattice_row(const double (&va)[kK], const double (&vb)[kK], double pa, double pb,
                                            double na_end, double nb_end, double vWa, double vEb, const ColConst& c,
                                            bool line, const double* cl, const LineCells& lc, double s2,
                                            double& aqa, double& aqb) {
    const double vNa = k + 1 < kK ? va[k + 1 < kK ? k + 1 : 0] : na_end;
    const double vNb = k + 1 < kK ? vb[k + 1 < kK ? k + 1 : 0] : nb_end;
    if (k == 0 && line) {
        line_row0(cl, lc, s2, va[k], vb[k], vWa, vEb, vNa, pa, vNb, pb, aqa, aqb);
        return;
    }
    aqa = c.dga * va[k] - c.kEa * vb[k] - c.kWa * vWa - c.kNSa * (vNa + pa);
    aqb = c.dgb * vb[k] - c.kEb * vEb - c.kEa * va[k] - c.kNSb * (vNb + pb);
}

// TMEM layout per thread (128 columns): row pair q at 16 q: g of rows 2q,
// 2q+1 of column a, of column b (8 columns), then v_{m-1} likewise (8);
// then z_n of the next item's positions (64: column a, 80: column b; 16
// columns each) and w = 2 z_n - z_{n-1} of this item's (96, 112)
constexpr unsigned kTmZn = 64, kTmW = 96;

// the thread's view of one work item
struct ItemGeo {
    int tile, s;
    int wz, hz, HS;
    int sa, sb, sWa, sEb;
    int ia, ib, jr0;
    unsigned lat, own;  // bit k: column a row k, bit 8 + k: column b
};

__device__ __forceinline__ ItemGeo item_geo(const TileArgs& a, int item, int warp, int lane) {
    ItemGeo g;
    g.tile = item / a.count;
    g.s = item - g.tile * a.count;
    const int shape = __ldg(&a.tile_oj[g.tile].z);
    const int4 t = __ldg(a.thr_geo + g.tile * kT + warp * 32 + lane);  // planned per (tile, thread)
    // region shape: wide (kTileWz columns), tall (kTileHz columns) or square
    // (the corners); the same number of positions
    g.wz = shape == 0 ? kTileWz : shape == 1 ? kTileHz : kTileSq;
    g.hz = shape == 0 ? kTileHz : shape == 1 ? kTileWz : kTileSq;
    g.HS = g.hz + 3;
    // a strip row of fewer than 32 column pairs (the tall shape) puts
    // 32 / pairs strips in a warp (host/tiles.cpp plans the same mapping)
    const int pairs = g.wz / 2;
    const int strip = pairs >= 32 ? warp / (pairs / 32) : warp * (32 / pairs) + lane / pairs;
    const int tc = pairs >= 32 ? (warp % (pairs / 32)) * 32 + lane : lane % pairs;
    const int pa = tc + 1, pb = g.wz / 2 + 2 + tc;  // column positions of the own columns
    g.sa = pa * g.HS + strip * kK + 1;
    g.sb = pb * g.HS + strip * kK + 1;
    g.sWa = g.sb - g.HS;  // far neighbours: W of column a, E of column b
    g.sEb = g.sa + g.HS;
    g.ia = t.x;
    g.ib = t.x + 1;
    g.jr0 = t.y;
    g.lat = static_cast<unsigned>(t.z) & 0xffffu;
    g.own = static_cast<unsigned>(t.z) >> 16;
    return g;
}

// 8 z values of one column of an item's lattice positions (0 elsewhere)
// (sample-major state: the column's 8 rows are 64 contiguous bytes)
__device__ __forceinline__ void load_col(const double* __restrict__ z, const ItemGeo& g, int col, int W, int n,
                                         double (&out)[kK]) {
    const double* zs = z + static_cast<std::size_t>(g.s) * n + (col ? g.ib : g.ia) * W + g.jr0;
#pragma unroll
    for (int k = 0; k < kK; ++k) out[k] = (g.lat >> (8 * col + k)) & 1u ? __ldg(zs + k) : 0.0;
}
__device__ __forceinline__ void tm_put8(std::uint32_t addr, const double (&d)[kK]) {
    std::uint32_t r[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int k = 0; k < 4; ++k) t_put(r + 2 * k, d[4 * h + k]);
        t_st8(addr + 8 * h, r);
    }
}
__device__ __forceinline__ void tm_get8(std::uint32_t addr, double (&d)[kK]) {
    std::uint32_t r[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        t_ld8(addr + 8 * h, r);
#pragma unroll
        for (int k = 0; k < 4; ++k) d[4 * h + k] = t_dbl(r + 2 * k);
    }
}

__global__ void __launch_bounds__(kT, 512 / kT) tile_step_kernel(TileArgs a) {
    extern __shared__ __align__(16) double sd[];
    __shared__ std::uint32_t tm_slot;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = a.m + 1, m = a.m;
    const int buf = a.box_slots + a.max_app;
    double* B0 = sd;
    double* B1 = sd + buf;
    double* wbuf = sd + 2 * buf;
    double* gst = wbuf + a.max_ent;  // generic rows: d | d_{m-1} | g  (max_gen each)
    double* cl = gst + 3 * a.max_gen;
    double* kbeta = cl + a.n_cells;  // substep constants beta_m, c_m
    double* kcm = kbeta + a.p;
    for (int q = tid; q < a.p - 1; q += kT) {
        kbeta[q] = __ldg(a.beta + q);
        kcm[q] = __ldg(a.cm + q);
    }
    const std::size_t S = static_cast<std::size_t>(a.S);
    const double s2 = a.inv_h2;
    const double* __restrict__ zc = a.zc;
    double* __restrict__ zp = a.zp;

    // tensor memory: 128 columns per four warps (the SM's 512 shared by its
    // CTAs); warp w: lanes 32 (w % 4).., columns 128 (w / 4)..
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                     "tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n"
                     :
                     : "r"(static_cast<std::uint32_t>(__cvta_generic_to_shared(&tm_slot))), "n"(kTmCols)
                     : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const std::uint32_t tb = tm_slot + (static_cast<std::uint32_t>(32 * (warp & 3)) << 16) + 128u * (warp >> 2);

    const int items = a.n_tiles * a.count;
    // software pipeline: an item's z_n and cell coefficients are loaded
    // during the previous item's substeps (prologue: the first item here)
    double cl_next = 0.0;
    if (blockIdx.x < items) {
        const ItemGeo g0 = item_geo(a, blockIdx.x, warp, lane);
        double z[kK];
        load_col(zc, g0, 0, W, a.n, z);
        tm_put8(tb + kTmZn, z);
        load_col(zc, g0, 1, W, a.n, z);
        tm_put8(tb + kTmZn + 16, z);
        if (tid < a.n_cells) cl_next = __ldg(a.cells + static_cast<std::size_t>(tid) * S + g0.s);
    }
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const ItemGeo g = item_geo(a, item, warp, lane);
        const int s = g.s;
        const std::size_t zbase = static_cast<std::size_t>(s) * a.n;  // sample-major state
        const int next_item = item + gridDim.x;
        const bool has_next = next_item < items;
        const int gb = __ldg(a.gen_off + g.tile), ng = __ldg(a.gen_off + g.tile + 1) - gb;
        const bool partial = __any_sync(0xffffffffu, g.lat != 0xffffu);
        const int sa = g.sa, sb = g.sb, sWa = g.sWa, sEb = g.sEb, HS = g.HS, wz = g.wz, hz = g.hz;
        const unsigned lat = g.lat;

        if (tid < a.n_cells) cl[tid] = cl_next;
        __syncthreads();  // cl; and every reader of the previous item's buffers is done
        // guards of this shape (zero; the previous item may have had the other
        // shape): column positions 0, wz/2 + 1, wz + 2 and rows 0, hz + 1, hz + 2
        for (int q = tid; q < 3 * HS; q += kT) {
            const int pos = q / HS, r = q % HS;
            const int col = pos == 0 ? 0 : (pos == 1 ? wz / 2 + 1 : wz + 2);
            B0[col * HS + r] = 0.0;
            B1[col * HS + r] = 0.0;
        }
        for (int q = tid; q < 3 * (wz + 3); q += kT) {
            const int pos = q / 3, r = q % 3 == 0 ? 0 : hz + q % 3;
            B0[pos * HS + r] = 0.0;
            B1[pos * HS + r] = 0.0;
        }

        ColConst cc;
        LineCells lc;
        const bool line = g.jr0 >= 1 && g.jr0 <= m - 1 && __ldg(a.line_row + g.jr0);
        {
            const int q0 = min(max(g.ia - 1, 0), m - 1), q1 = min(max(g.ia, 0), m - 1),
                      q2 = min(max(g.ib, 0), m - 1);
            const int ru = min(max(g.jr0, 0), m - 1), rd = min(max(g.jr0 - 1, 0), m - 1);
            lc.cu = __ldg(a.celly + ru) * a.cells_x;
            lc.cd = __ldg(a.celly + rd) * a.cells_x;
            lc.x0 = __ldg(a.cellx + q0);
            lc.x1 = __ldg(a.cellx + q1);
            lc.x2 = __ldg(a.cellx + q2);
            const double U0 = cl[lc.cu + lc.x0], U1 = cl[lc.cu + lc.x1], U2 = cl[lc.cu + lc.x2];
            cc.kWa = U0 * s2;
            cc.kEa = U1 * s2;
            cc.kNSa = (U0 + U1) * (0.5 * s2);
            cc.dga = cc.kEa + cc.kWa + 2.0 * cc.kNSa;
            cc.kEb = U2 * s2;
            cc.kNSb = (U1 + U2) * (0.5 * s2);
            cc.dgb = cc.kEb + cc.kEa + 2.0 * cc.kNSb;
        }

        // 1. z_n in (prefetched into TMEM): lattice positions v = z / h;
        // positions outside the box 0 (both buffers); box ring positions
        // belong to the generic rows
        double va[kK], vb[kK];
        tm_get8(tb + kTmZn, va);
        tm_get8(tb + kTmZn + 16, vb);
#pragma unroll
        for (int k = 0; k < kK; ++k) {
            const int j = g.jr0 + k;
            const bool jin = j >= 0 && j <= m;
            va[k] *= a.inv_h;
            vb[k] *= a.inv_h;
            if (lat & (1u << k)) {
                B0[sa + k] = va[k];
            } else if (!(jin && g.ia >= 0 && g.ia <= m)) {
                B0[sa + k] = 0.0;
                B1[sa + k] = 0.0;
            }
            if (lat & (1u << (8 + k))) {
                B0[sb + k] = vb[k];
            } else if (!(jin && g.ib >= 0 && g.ib <= m)) {
                B0[sb + k] = 0.0;
                B1[sb + k] = 0.0;
            }
        }
        // generic rows (tid, tid + T, ...): z_n in, per-sample SELL weights
        const int eb = __ldg(a.g_ent_off + gb);
        for (int u = tid; u < ng; u += kT) {
            const int r = gb + u;
            B0[__ldg(a.g_slot + r)] = __ldg(zc + zbase + __ldg(a.g_dof + r)) * __ldg(a.g_rs + r);
        }
        // the weights entry by entry (a thread per entry: the index loads of a
        // warp are consecutive, and two entries' loads are in flight at once)
        {
            const int ee = __ldg(a.g_ent_off + gb + ng);
            for (int e = eb + tid; e < ee; e += 2 * kT) {
                const int e2 = e + kT;
                const bool two = e2 < ee;
                const int t0 = __ldg(a.e_rc_off + e), t1 = __ldg(a.e_rc_off + e + 1);
                const int u0 = two ? __ldg(a.e_rc_off + e2) : 0, u1 = two ? __ldg(a.e_rc_off + e2 + 1) : 0;
                double w = 0.0, w2 = 0.0;
                for (int t = t0, u = u0; t < t1 || u < u1; ++t, ++u) {
                    const bool pa = t < t1, pb = u < u1;
                    const int ca = pa ? __ldg(a.rc_cell + t) : 0, cb = pb ? __ldg(a.rc_cell + u) : 0;
                    const double xa = pa ? __ldg(a.rc_a0 + t) : 0.0, xb = pb ? __ldg(a.rc_a0 + u) : 0.0;
                    if (pa) w += cl[ca] * xa;
                    if (pb) w2 += cl[cb] * xb;
                }
                wbuf[e - eb] = w;
                if (two) wbuf[e2 - eb] = w2;
            }
        }
        __syncthreads();

        // 2. g = A z_n (v units on the lattice), d_1 = -c0 g; TMEM: g, v_0 = 0
        const double c0 = a.c0;
        {
            if (partial) {  // rows / columns outside the lattice read their ring or zero values
#pragma unroll
                for (int k = 0; k < kK; ++k) {
                    if (!(lat & (1u << k))) va[k] = B0[sa + k];
                    if (!(lat & (1u << (8 + k)))) vb[k] = B0[sb + k];
                }
            }
            const double na_end = B0[sa + kK], nb_end = B0[sb + kK];
            double pa_ = B0[sa - 1], pb_ = B0[sb - 1];
#pragma unroll
            for (int q = 0; q < kK / 2; ++q) {
                double g2[2][2];
#define WMC_TILE_G_ROW(K_, R_)                                                                              \
                {                                                                                           \
                    double ga, gbb;                                                                         \
                    lattice_row<K_>(va, vb, pa_, pb_, na_end, nb_end, B0[sWa + K_], B0[sEb + K_], cc, line, \
                                    cl, lc, s2, ga, gbb);                                                   \
                    g2[R_][0] = ga;                                                                         \
                    g2[R_][1] = gbb;                                                                        \
                    pa_ = va[K_];                                                                           \
                    pb_ = vb[K_];                                                                           \
                }
                if (q == 0) { WMC_TILE_G_ROW(0, 0) WMC_TILE_G_ROW(1, 1) }
                if (q == 1) { WMC_TILE_G_ROW(2, 0) WMC_TILE_G_ROW(3, 1) }
                if (q == 2) { WMC_TILE_G_ROW(4, 0) WMC_TILE_G_ROW(5, 1) }
                if (q == 3) { WMC_TILE_G_ROW(6, 0) WMC_TILE_G_ROW(7, 1) }
#undef WMC_TILE_G_ROW
                t_st4d(tb + 16 * q, g2[0][0], g2[1][0], g2[0][1], g2[1][1]);
                va[2 * q] = -c0 * g2[0][0];
                va[2 * q + 1] = -c0 * g2[1][0];
                vb[2 * q] = -c0 * g2[0][1];
                vb[2 * q + 1] = -c0 * g2[1][1];
            }
#pragma unroll
            for (int k = 0; k < kK; ++k) {
                if (lat & (1u << k)) B1[sa + k] = va[k];
                if (lat & (1u << (8 + k))) B1[sb + k] = vb[k];
            }
        }
        for (int u = tid; u < ng; u += kT) {
            const int r = gb + u;
            double acc = 0.0;
            for (int e = __ldg(a.g_ent_off + r); e < __ldg(a.g_ent_off + r + 1); ++e)
                acc += wbuf[e - eb] * B0[__ldg(a.e_slot + e)];
            double rem = 0.0;
            for (int e = __ldg(a.g_rem_off + r); e < __ldg(a.g_rem_off + r + 1); ++e) {
                double w = 0.0;
                for (int t = __ldg(a.r_rc_off + e); t < __ldg(a.r_rc_off + e + 1); ++t)
                    w += cl[__ldg(a.rr_cell + t)] * __ldg(a.rr_a0 + t);
                rem += w * __ldg(zc + zbase + __ldg(a.r_dof + e));
            }
            const double gg = acc + rem, d1 = -c0 * gg;
            gst[u] = d1;
            gst[a.max_gen + u] = 0.0;
            gst[2 * a.max_gen + u] = gg;
            B1[__ldg(a.g_slot + r)] = d1 * __ldg(a.g_rs + r);
        }
        __syncthreads();

        // prefetch stages, overlapped with the substeps: 0 / 1: z_{n-1} of
        // this item's columns a / b -> w = 2 z_n - z_{n-1} (TMEM); 2 / 3: z_n
        // of the next item's columns (TMEM) and its cell coefficients
        // stage q (0..7): rows 4 (q & 1) .. + 3 of column (q >> 1) & 1; q < 4:
        // z_{n-1} of this item -> w, q >= 4: z_n of the next item
        constexpr int kH = kK / 2;
        auto issue = [&](int stage, double (&z)[kH]) {
            const int col = (stage >> 1) & 1, h = stage & 1;
            if (stage < 4) {
                const double* zs = zp + zbase + (col ? g.ib : g.ia) * W + g.jr0 + kH * h;
#pragma unroll
                for (int k = 0; k < kH; ++k) z[k] = (lat >> (8 * col + kH * h + k)) & 1u ? __ldg(zs + k) : 0.0;
            } else if (has_next) {
                const ItemGeo gn = item_geo(a, next_item, warp, lane);  // a table lookup
                const double* zs = zc + static_cast<std::size_t>(gn.s) * a.n + (col ? gn.ib : gn.ia) * W + gn.jr0 +
                                   kH * h;
#pragma unroll
                for (int k = 0; k < kH; ++k) z[k] = (gn.lat >> (8 * col + kH * h + k)) & 1u ? __ldg(zs + k) : 0.0;
                if (stage == 4 && tid < a.n_cells)
                    cl_next = __ldg(a.cells + static_cast<std::size_t>(tid) * S + gn.s);
            }
        };
        auto commit = [&](int stage, const double (&z)[kH]) {
            const int col = (stage >> 1) & 1, h = stage & 1;
            std::uint32_t r[8];
            if (stage < 4) {
                t_ld8(tb + kTmZn + 16 * col + 8 * h, r);
#pragma unroll
                for (int k = 0; k < kH; ++k) t_put(r + 2 * k, 2.0 * t_dbl(r + 2 * k) - z[k]);
                t_st8(tb + kTmW + 16 * col + 8 * h, r);
            } else if (has_next) {
#pragma unroll
                for (int k = 0; k < kH; ++k) t_put(r + 2 * k, z[k]);
                t_st8(tb + kTmZn + 16 * col + 8 * h, r);
            }
        };

        // 3. substeps m = 1 .. p-1 (v_m in buffer m & 1; the parity is a
        // template argument so the buffer addresses are fixed per body)
        auto substep = [&](auto odd, auto first, int mm) {
            constexpr bool kOdd = decltype(odd)::value;
            constexpr bool kFirst = decltype(first)::value;  // m = 1: v_0 = 0
            const double* cur = kOdd ? B1 : B0;
            double* nxt = kOdd ? B0 : B1;
            const double beta = kbeta[mm - 1], cmm = kcm[mm - 1];
            const double onepb = 1.0 + beta;
            double pre[kH];
            if (mm <= 8) issue(mm - 1, pre);
            if (partial) {
#pragma unroll
                for (int k = 0; k < kK; ++k) {
                    if (!(lat & (1u << k))) va[k] = cur[sa + k];
                    if (!(lat & (1u << (8 + k)))) vb[k] = cur[sb + k];
                }
            }
            const double na_end = cur[sa + kK], nb_end = cur[sb + kK];
            double pa_ = cur[sa - 1], pb_ = cur[sb - 1];
#pragma unroll
            for (int q = 0; q < kK / 2; ++q) {
                double tg[4], tv[4];
                t_ld4d(tb + 16 * q, tg);
                // v_{m-1}: still in the buffer this substep overwrites (own slots)
                tv[0] = kFirst ? 0.0 : nxt[sa + 2 * q];
                tv[1] = kFirst ? 0.0 : nxt[sa + 2 * q + 1];
                tv[2] = kFirst ? 0.0 : nxt[sb + 2 * q];
                tv[3] = kFirst ? 0.0 : nxt[sb + 2 * q + 1];
                double nx[2][2];
#define WMC_TILE_S_ROW(K_, R_)                                                                               \
                {                                                                                            \
                    double aqa, aqb;                                                                         \
                    lattice_row<K_>(va, vb, pa_, pb_, na_end, nb_end, cur[sWa + K_], cur[sEb + K_], cc, line, \
                                    cl, lc, s2, aqa, aqb);                                                   \
                    nx[R_][0] = onepb * va[K_] - beta * tv[R_] - cmm * (tg[R_] + aqa);                       \
                    nx[R_][1] = onepb * vb[K_] - beta * tv[2 + R_] - cmm * (tg[2 + R_] + aqb);               \
                    pa_ = va[K_];                                                                            \
                    pb_ = vb[K_];                                                                            \
                }
                if (q == 0) { WMC_TILE_S_ROW(0, 0) WMC_TILE_S_ROW(1, 1) }
                if (q == 1) { WMC_TILE_S_ROW(2, 0) WMC_TILE_S_ROW(3, 1) }
                if (q == 2) { WMC_TILE_S_ROW(4, 0) WMC_TILE_S_ROW(5, 1) }
                if (q == 3) { WMC_TILE_S_ROW(6, 0) WMC_TILE_S_ROW(7, 1) }
#undef WMC_TILE_S_ROW
                va[2 * q] = nx[0][0];
                va[2 * q + 1] = nx[1][0];
                vb[2 * q] = nx[0][1];
                vb[2 * q + 1] = nx[1][1];
            }
            if (!partial) {  // warp-uniform: every position of the warp is a lattice node
#pragma unroll
                for (int k = 0; k < kK; ++k) {
                    nxt[sa + k] = va[k];
                    nxt[sb + k] = vb[k];
                }
            } else {
#pragma unroll
                for (int k = 0; k < kK; ++k) {
                    if (lat & (1u << k)) nxt[sa + k] = va[k];
                    if (lat & (1u << (8 + k))) nxt[sb + k] = vb[k];
                }
            }
            for (int u = tid; u < ng; u += kT) {
                const int r = gb + u;
                // the row's table reads first (independent loads, one latency),
                // then its entries four at a time: slots and weights of a
                // group before its gathers (padding: weight 0 on the zero
                // guard slot 0, so the sum keeps its order and value)
                const int e0 = __ldg(a.g_ent_off + r), e1 = __ldg(a.g_ent_off + r + 1);
                const int gs = __ldg(a.g_slot + r);
                const double rs = __ldg(a.g_rs + r);
                const double d = gst[u], dp = gst[a.max_gen + u], gg = gst[2 * a.max_gen + u];
                double acc = 0.0;
                for (int e = e0; e < e1; e += 4) {
                    int sl[4];
                    double w[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const bool ok = e + q < e1;
                        sl[q] = ok ? __ldg(a.e_slot + e + q) : 0;
                        w[q] = ok ? wbuf[e + q - eb] : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc += w[q] * cur[sl[q]];
                }
                const double next = onepb * d - beta * dp - cmm * (gg + acc);
                gst[a.max_gen + u] = d;
                gst[u] = next;
                nxt[gs] = next * rs;
            }
            if (mm <= 8) commit(mm - 1, pre);
            __syncthreads();
        };
        if (a.p > 1) substep(std::true_type{}, std::true_type{}, 1);
        for (int mm = 2; mm <= a.p - 1; mm += 2) {
            substep(std::false_type{}, std::false_type{}, mm);
            if (mm + 1 <= a.p - 1) substep(std::true_type{}, std::false_type{}, mm + 1);
        }
        for (int stage = a.p - 1; stage < 8; ++stage) {  // short step sequences (p < 9)
            double pre[kH];
            issue(stage, pre);
            commit(stage, pre);
        }

        // 4. owned rows: z_{n+1} = w + 2 d_p (d = v h), check_finite
        bool bad = false;
        {
            double w[kK];
            tm_get8(tb + kTmW, w);
#pragma unroll
            for (int k = 0; k < kK; ++k)
                if (g.own & (1u << k)) {
                    const double out = w[k] + 2.0 * (va[k] * a.h);
                    zp[zbase + g.ia * W + g.jr0 + k] = out;
                    bad |= !(fabs(out) <= 1e100);
                }
            tm_get8(tb + kTmW + 16, w);
#pragma unroll
            for (int k = 0; k < kK; ++k)
                if (g.own & (1u << (8 + k))) {
                    const double out = w[k] + 2.0 * (vb[k] * a.h);
                    zp[zbase + g.ib * W + g.jr0 + k] = out;
                    bad |= !(fabs(out) <= 1e100);
                }
        }
        for (int u = tid; u < ng; u += kT) {
            const int r = gb + u;
            if (!__ldg(a.g_owned + r)) continue;
            const std::size_t idx = zbase + __ldg(a.g_dof + r);
            const double out = 2.0 * __ldg(zc + idx) - zp[idx] + 2.0 * gst[u];
            zp[idx] = out;
            bad |= !(fabs(out) <= 1e100);
        }
        if (bad && s < a.count) atomicMin(a.fail + s, a.step);
    }

    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" : : "r"(tm_slot), "n"(kTmCols) : "memory");
}

}  // namespace

int tile_smem_bytes(const TileArgs& a) {
    return static_cast<int>(sizeof(double)) *
           (2 * (a.box_slots + a.max_app) + a.max_ent + 3 * a.max_gen + a.n_cells + 2 * a.p + 1);
}

int launch_tile_step(const TileArgs& a, int grid, void* stream) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, tile_step_kernel);  // static shared memory (the TMEM address slot)
    const int e = set_max_dynamic_smem(reinterpret_cast<const void*>(tile_step_kernel),
                                       optin - static_cast<int>(fa.sharedSizeBytes), true);
    if (e != 0) return e;
    tile_step_kernel<<<grid, kT, tile_smem_bytes(a), static_cast<cudaStream_t>(stream)>>>(a);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace wmc
