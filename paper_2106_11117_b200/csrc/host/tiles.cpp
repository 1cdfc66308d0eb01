// Tile planner of the temporally blocked LF-LTS step (see tiles.hpp).
#include "tiles.hpp"

#include <algorithm>
#include <cmath>
#include <queue>
#include <unordered_map>

namespace wmc {

namespace {

int ceil_div(int a, int b) { return (a + b - 1) / b; }

struct TileDesc {
    int shape;  // 0: wide (kWide columns x kNarrow rows), 1: tall
    int ri0, rj0;
    int oi0, oi1, oj0, oj1;
};

struct Rect {
    int i0 = 0, i1 = 0, j0 = 0, j1 = 0;  // [i0, i1) x [j0, j1), empty when i0 == i1
};

// Regular grid of wide tiles, halo p (columns) / p rounded up to k (rows).
std::vector<TileDesc> layout_grid(int W, int p, int k, int jres, int wz, int hz) {
    std::vector<TileDesc> out;
    const int hx = p, hy = ceil_div(p, k) * k;
    const int ow = wz - 2 * hx, oh = hz - 2 * hy;
    if (ow < 8 || oh < k) return out;
    const int n_ti = ceil_div(W, ow), owb = ceil_div(W, n_ti);
    const int jb = jres == 0 ? 0 : jres - k;
    const int n_tj = ceil_div(W - jb, oh);
    for (int tj = 0; tj < n_tj; ++tj)
        for (int ti = 0; ti < n_ti; ++ti) {
            TileDesc d;
            d.shape = 0;
            d.oi0 = ti * owb;
            d.oi1 = std::min(W, (ti + 1) * owb);
            d.oj0 = std::max(0, jb + tj * oh);
            d.oj1 = std::min(W, jb + (tj + 1) * oh);
            d.ri0 = d.oi0 - (wz - (d.oi1 - d.oi0)) / 2;
            d.rj0 = jb + tj * oh - hy;
            out.push_back(d);
        }
    return out;
}

// Frame layout for halos that must be wider along the box edges (the R rows
// outside the box are coarser, so a path of p hops through them moves
// farther along the edge than p lattice steps): tall tiles in the left and
// right bands (halo 2 p along the edge), wide tiles with halo 2 p in the
// bottom and top bands, the regular grid inside.  Row origins stay = jres
// (mod k).
// With `inner` the interior grid is left out and its rectangle returned.
// `thin_sides` (streamed interior only): the bottom and top bands span every
// column, corners included, and the side bands between them own tw - p
// columns (their tiles see no corner, so p columns of halo on the inner
// side are enough -- the halo check has the last word).
std::vector<TileDesc> layout_frame(int W, int p, int k, int jres, int wz, int hz, int he, Rect* inner = nullptr,
                                   bool thin_sides = false) {
    std::vector<TileDesc> out;
    auto align_down = [&](int j) {  // largest value <= j that is = jres (mod k)
        int r = ((j - jres) % k + k) % k;
        return j - r;
    };
    const int hi = p;
    const int hye = ceil_div(he, k) * k, hyi = ceil_div(hi, k) * k;
    // side bands: tall tiles (hz columns x wz rows), owned width sb
    const int tw = hz, th = wz;
    thin_sides = thin_sides && inner;
    const int sb = thin_sides ? tw - hi : tw - he;
    if (sb < 8 || 2 * sb >= W) return out;
    const int soh = th - 2 * hye;
    if (soh < k) return out;
    // rows of the side bands: all of them, or (thin sides) those between the
    // bottom and top bands, whose heights follow from the wide tiles below
    int side_j0 = 0, side_j1 = W;
    if (thin_sides) {
        const int rjb_ = align_down(0), rjt_ = align_down(W - hz + k - 1);
        side_j0 = rjb_ + hz - hyi;
        side_j1 = rjt_ + hyi;
        if (side_j0 < p + 1 || W - side_j1 < p + 1 || side_j1 - side_j0 < k) return {};
    }
    for (int side = 0; side < 2; ++side) {
        const int oi0 = side == 0 ? 0 : W - sb, oi1 = side == 0 ? sb : W;
        const int ri0 = side == 0 ? 0 : W - tw;
        for (int oj0 = side_j0; oj0 < side_j1;) {
            const int start = align_down(oj0);
            const int oj1 = std::min(side_j1, start + soh);
            TileDesc d{1, ri0, start - hye, oi0, oi1, oj0, oj1};
            out.push_back(d);
            oj0 = oj1;
        }
    }
    // middle columns [sb, W - sb) (thin sides: every column): bottom / top
    // bands (halo he across columns) and the interior grid (halo hi)
    const int c0 = sb, c1 = W - sb, cw = c1 - c0;
    const int bw = wz - 2 * he;  // band tile owned width
    const int iw = wz - 2 * hi;  // interior owned width
    const int ih = hz - 2 * hyi;  // interior owned height
    if (bw < 8 || iw < 8 || ih < k) return out;
    // band heights: bottom rows [0, bb), top rows [W - bt, W); the interior
    // rows a whole number of ih-row bands, each starting = jres (mod k)
    const int band_max = hz - hyi;  // the region must reach hyi rows past the band
    int bb = -1, bt = -1, n_int = 0;
    // band tile regions: below / above the box by hyi rows (the grid case),
    // or (streamed interior) flush with the box so the bands can be taller
    int rjb = 0, rjt = 0;
    if (inner) {  // streamed interior: any height; the bands as tall as their tiles allow
        rjb = align_down(0);
        rjt = align_down(W - hz + k - 1);  // the first aligned origin whose region reaches row W - 1
        bb = rjb + hz - hyi;
        bt = W - (rjt + hyi);
        if (bb < p + 1 || bt < p + 1 || W - bb - bt < k) return {};
    } else {
        for (n_int = (W - 2) / ih; n_int >= 0 && bb < 0; --n_int)
            for (int b = align_down(band_max); b >= 1; b -= k) {
                const int t = W - b - n_int * ih;
                if (b % k == ((jres % k) + k) % k && t >= 1 && t <= band_max) {
                    bb = b;
                    bt = t;
                    break;
                }
            }
        ++n_int;
    }
    if (bb < 0) return {};
    // thin sides: the corners are square tiles (shape 2, sq x sq positions:
    // paths along both edges' coarser rows stay inside), owning sq - he columns
    int sq = 0;
    while (sq * sq < wz * hz) ++sq;
    const int cown = sq - he;
    if (thin_sides && (sq * sq != wz * hz || sq % 64 || cown < sb || 2 * cown >= W)) return {};
    auto band = [&](int oj0, int oj1, bool bottom) {
        int c0 = thin_sides ? cown : sb, c1 = W - c0;
        const int cw = c1 - c0;
        if (thin_sides) {
            const int rj = bottom ? rjb : align_down(W - sq + k - 1);
            out.push_back(TileDesc{2, 0, rj, 0, cown, oj0, oj1});
            out.push_back(TileDesc{2, W - sq, rj, W - cown, W, oj0, oj1});
        }
        const int n = ceil_div(cw, bw), w = ceil_div(cw, n);
        for (int q = 0; q < n; ++q) {
            TileDesc d;
            d.shape = 0;
            d.oi0 = c0 + q * w;
            d.oi1 = std::min(c1, c0 + (q + 1) * w);
            d.oj0 = oj0;
            d.oj1 = oj1;
            d.ri0 = d.oi0 - (wz - (d.oi1 - d.oi0)) / 2;
            if (inner)
                d.rj0 = bottom ? rjb : rjt;
            else
                d.rj0 = bottom ? align_down(oj0 - hyi) : align_down(oj1 + hyi - hz);
            out.push_back(d);
        }
    };
    band(0, bb, true);
    if (inner) {
        *inner = Rect{sb, W - sb, bb, W - bt};
    } else {
        const int n = ceil_div(cw, iw), w = ceil_div(cw, n);
        for (int r = 0; r < n_int; ++r)
            for (int q = 0; q < n; ++q) {
                TileDesc d;
                d.shape = 0;
                d.oi0 = c0 + q * w;
                d.oi1 = std::min(c1, c0 + (q + 1) * w);
                d.oj0 = bb + r * ih;
                d.oj1 = d.oj0 + ih;
                d.ri0 = d.oi0 - (wz - (d.oi1 - d.oi0)) / 2;
                d.rj0 = d.oj0 - hyi;
                out.push_back(d);
            }
    }
    band(W - bt, W, false);
    return out;
}

// Slabs of the streamed interior: owned row bands of at most slab_rows - 2 p
// rows (the stream kernel's threads), each region grown by p rows and columns.
// The region stays inside the box interior [1, m-1]^2 (checked by the
// caller), so every position is a 5-point lattice row and an owned
// position's p-hop dependency cone lies in its region.  Returns the region
// positions.
long plan_slabs(const Rect& inner, int p, TilePlan& P) {
    P.slab.clear();
    P.slab_own.clear();
    P.n_slabs = P.max_nx = 0;
    if (inner.i0 == inner.i1) return 0;
    // CTA size: the multiple of four warps (at most slab_rows, a thread per region
    // row) that wastes the fewest thread-rows; ties to the larger CTA
    const int rows = inner.j1 - inner.j0;
    int best_t = 0;
    long best_cost = 0;
    // (multiples of four warps only: the SM's four schedulers take a CTA's
    // warps round-robin, and an uneven share made 224 threads no faster than 256)
    for (int T = P.slab_rows; T >= 128 && T > 2 * p + 32; T -= 128) {
        const long cost = static_cast<long>(ceil_div(rows, T - 2 * p)) * T;
        if (best_t == 0 || cost < best_cost) {
            best_t = T;
            best_cost = cost;
        }
    }
    if (best_t == 0) best_t = P.slab_rows;
    P.slab_threads = best_t;
    const int per = best_t - 2 * p;
    const int n = ceil_div(rows, per), each = ceil_div(rows, n);
    const int nx = inner.i1 - inner.i0 + 2 * p;
    long positions = 0;
    for (int q = 0; q < n; ++q) {
        const int oj0 = inner.j0 + q * each, oj1 = std::min(inner.j1, oj0 + each);
        const int ny = oj1 - oj0 + 2 * p;
        P.slab.insert(P.slab.end(), {inner.i0 - p, nx, oj0 - p, ny});
        P.slab_own.insert(P.slab_own.end(), {p, p + inner.i1 - inner.i0, p, p + oj1 - oj0});
        positions += static_cast<long>(nx) * ny;
    }
    P.n_slabs = n;
    P.max_nx = nx;
    return positions;
}

// Builds the tile tables of P for `tiles` and checks the halos; false with
// P.reason when a tile fails.
bool build_tiles(const LevelTables& t, const std::vector<TileDesc>& tiles, const Rect& inner, int wide, int narrow,
                 int k, TilePlan& P) {
    const int m = t.lat_m, W = m + 1, p = t.p, n_r = t.n_r, WW = W * W;
    P.tiles_shape.clear();
    P.thr_geo.clear();
    P.i0.clear(), P.j0.clear(), P.oi0.clear(), P.oi1.clear(), P.oj0.clear(), P.oj1.clear();
    P.gen_off.assign(1, 0);
    P.g_slot.clear(), P.g_dof.clear(), P.g_owned.clear(), P.g_rs.clear();
    P.g_ent_off.assign(1, 0);
    P.g_rem_off.assign(1, 0);
    P.e_slot.clear(), P.e_rc_off.clear(), P.rc_cell.clear(), P.rc_a0.clear();
    P.r_dof.clear(), P.r_rc_off.clear(), P.rr_cell.clear(), P.rr_a0.clear();
    P.max_gen = P.max_app = P.max_ent = 0;
    // owner of every box node, then of every R row outside the box (its
    // lattice position clamped into the box)
    std::vector<int> owner(static_cast<std::size_t>(WW), -1);
    for (int i = inner.i0; i < inner.i1; ++i)
        for (int j = inner.j0; j < inner.j1; ++j) owner[i * W + j] = -2;  // streamed
    for (std::size_t q = 0; q < tiles.size(); ++q)
        for (int i = tiles[q].oi0; i < tiles[q].oi1; ++i)
            for (int j = tiles[q].oj0; j < tiles[q].oj1; ++j) {
                if (owner[i * W + j] >= 0) {
                    P.reason = "tiles overlap";
                    return false;
                }
                owner[i * W + j] = static_cast<int>(q);
            }
    for (int x = 0; x < WW; ++x)
        if (owner[x] == -1) {
            P.reason = "tiles leave a box node unowned";
            return false;
        }
    std::vector<std::vector<int>> belt_owned(tiles.size());
    for (int r = WW; r < n_r; ++r) {
        const int i = std::clamp(t.dof_lx[r], 0, m), j = std::clamp(t.dof_ly[r], 0, m);
        if (owner[i * W + j] < 0) {
            P.reason = "an R row outside the box maps into the streamed interior";
            return false;
        }
        belt_owned[owner[i * W + j]].push_back(r);
    }
    auto is_box = [&](int r) { return r < WW; };
    auto interior = [&](int i, int j) { return i >= 1 && i <= m - 1 && j >= 1 && j <= m - 1; };
    long region_positions = 0;
    for (std::size_t q = 0; q < tiles.size(); ++q) {
        const TileDesc& d = tiles[q];
        int sq = 0;
        while (sq * sq < wide * narrow) ++sq;
        const int wz = d.shape == 0 ? wide : d.shape == 1 ? narrow : sq;
        const int hz = d.shape == 0 ? narrow : d.shape == 1 ? wide : sq;
        const int hs = (hz + 2) | 1;
        const int box_slots = (wz + 3) * hs;
        if (box_slots > P.box_slots || wz * hz != wide * narrow) {  // appended slots start at P.box_slots
            P.reason = "a shape exceeds the plan's slot count";
            return false;
        }
        if (((d.rj0 - P.jres) % k + k) % k != 0) {
            P.reason = "region row origin not aligned to the strips";
            return false;
        }
        const int ri0 = d.ri0, rj0 = d.rj0;
        auto in_rect = [&](int i, int j) { return i >= ri0 && i < ri0 + wz && j >= rj0 && j < rj0 + hz; };
        auto rect_slot = [&](int i, int j) {
            const int c = i - ri0, rr = j - rj0;
            const int cp = (c % 2 == 0) ? c / 2 + 1 : wz / 2 + 2 + c / 2;
            return cp * hs + rr + 1;
        };
        for (int i = d.oi0; i < d.oi1; ++i)
            for (int j = d.oj0; j < d.oj1; ++j)
                if (!in_rect(i, j)) {
                    P.reason = "owned node outside its region";
                    return false;
                }
        // ball: rows needed within p hops of the owned rows ("needs" edges:
        // row x needs its P columns)
        std::unordered_map<int, int> dist;
        std::queue<int> bfs;
        for (int i = d.oi0; i < d.oi1; ++i)
            for (int j = d.oj0; j < d.oj1; ++j) {
                dist[i * W + j] = 0;
                bfs.push(i * W + j);
            }
        for (int r : belt_owned[q]) {
            dist[r] = 0;
            bfs.push(r);
        }
        std::vector<int> belt_ball;
        while (!bfs.empty()) {
            const int x = bfs.front();
            bfs.pop();
            const int dx = dist[x];
            if (!is_box(x)) belt_ball.push_back(x);
            if (dx >= p) continue;
            for (int e = t.row_ptr[x]; e < t.row_ptr[x + 1]; ++e) {
                const int y = t.col[e];
                if (y >= n_r || !t.in_p[y] || dist.count(y)) continue;
                dist[y] = dx + 1;
                bfs.push(y);
            }
        }
        std::sort(belt_ball.begin(), belt_ball.end());
        // generic rows: box ring nodes inside the region, and the rows of the
        // ball with no region position: R rows outside the box (owned ones
        // included) and box nodes beyond the region (paths through the
        // coarser rows outside the box run farther along the edge than p
        // lattice steps)
        std::unordered_map<int, int> slot_of;
        std::vector<int> gens;
        for (int i = std::max(0, ri0); i < std::min(W, ri0 + wz); ++i)
            for (int j = std::max(0, rj0); j < std::min(W, rj0 + hz); ++j)
                if (!interior(i, j)) gens.push_back(i * W + j);
        int n_app = 0;
        for (int x : belt_ball) {
            slot_of[x] = P.box_slots + n_app++;
            gens.push_back(x);
        }
        {
            std::vector<int> far;
            for (const auto& [x, dx] : dist)
                if (is_box(x) && !in_rect(x / W, x % W)) far.push_back(x);
            std::sort(far.begin(), far.end());
            for (int x : far) {
                slot_of[x] = P.box_slots + n_app++;
                gens.push_back(x);
            }
        }
        auto local_slot = [&](int x) -> int {  // -1: not on chip
            if (is_box(x) && in_rect(x / W, x % W)) return rect_slot(x / W, x % W);
            const auto it = slot_of.find(x);
            return it == slot_of.end() ? -1 : it->second;
        };
        // halo check on the implemented graph: multi-source BFS from the
        // positions whose values are wrong from the first substep on (a
        // lattice stencil leaving the region, a generic row missing a P
        // column); an owned row must be >= p hops away
        std::unordered_map<int, std::vector<int>> readers;  // slot -> slots reading it
        std::vector<int> sources;
        for (int i = std::max(1, ri0); i < std::min(m, ri0 + wz); ++i)
            for (int j = std::max(1, rj0); j < std::min(m, rj0 + hz); ++j) {
                const int s = rect_slot(i, j);
                const int nb[4][2] = {{i + 1, j}, {i - 1, j}, {i, j + 1}, {i, j - 1}};
                bool bad = false;
                for (const auto& n : nb) {
                    if (!in_rect(n[0], n[1])) {
                        bad = true;
                        continue;
                    }
                    readers[rect_slot(n[0], n[1])].push_back(s);
                }
                if (bad) sources.push_back(s);
            }
        const int g0 = static_cast<int>(P.g_slot.size());
        for (int x : gens) {
            const int s = local_slot(x);
            bool bad = false;
            for (int e = t.row_ptr[x]; e < t.row_ptr[x + 1];) {
                const int col = t.col[e];
                int e1 = e;
                while (e1 < t.row_ptr[x + 1] && t.col[e1] == col) ++e1;
                if (col >= n_r || !t.in_p[col]) {  // remainder: z_n from HBM
                    P.r_dof.push_back(col);
                    P.r_rc_off.push_back(static_cast<int>(P.rr_cell.size()));
                    for (int u = e; u < e1; ++u) {
                        P.rr_cell.push_back(t.cell[u]);
                        P.rr_a0.push_back(t.a0[u]);
                    }
                } else {
                    const int cs = local_slot(col);
                    if (cs < 0)
                        bad = true;
                    else
                        readers[cs].push_back(s);
                    P.e_slot.push_back(cs < 0 ? 0 : cs);  // slot 0: a guard (always zero)
                    P.e_rc_off.push_back(static_cast<int>(P.rc_cell.size()));
                    const double sq = std::sqrt(t.mass[col]);
                    for (int u = e; u < e1; ++u) {
                        P.rc_cell.push_back(t.cell[u]);
                        P.rc_a0.push_back(t.a0[u] * sq);
                    }
                }
                e = e1;
            }
            if (bad) sources.push_back(s);
            P.g_slot.push_back(s);
            P.g_dof.push_back(x);
            P.g_rs.push_back(1.0 / std::sqrt(t.mass[x]));
            const auto it = dist.find(x);
            P.g_owned.push_back(it != dist.end() && it->second == 0 ? 1 : 0);
            P.g_ent_off.push_back(static_cast<int>(P.e_slot.size()));
            P.g_rem_off.push_back(static_cast<int>(P.r_dof.size()));
        }
        std::unordered_map<int, int> bd;
        std::queue<int> bq;
        for (int s : sources)
            if (!bd.count(s)) {
                bd[s] = 0;
                bq.push(s);
            }
        while (!bq.empty()) {
            const int s = bq.front();
            bq.pop();
            const int ds = bd[s];
            if (ds + 1 >= p) continue;
            const auto it = readers.find(s);
            if (it == readers.end()) continue;
            for (int r : it->second)
                if (!bd.count(r)) {
                    bd[r] = ds + 1;
                    bq.push(r);
                }
        }
        for (int i = d.oi0; i < d.oi1; ++i)
            for (int j = d.oj0; j < d.oj1; ++j)
                if (bd.count(rect_slot(i, j))) {
                    P.reason = "tile " + std::to_string(q) + ": halo too narrow at box node (" + std::to_string(i) +
                               "," + std::to_string(j) + ")";
                    return false;
                }
        for (std::size_t u = 0; u < gens.size(); ++u)
            if (P.g_owned[g0 + u] && bd.count(P.g_slot[g0 + u])) {
                P.reason = "tile " + std::to_string(q) + ": halo too narrow at generic row " + std::to_string(gens[u]);
                return false;
            }
        {
            // thread geometry (tile_step_kernel's item view): thread = 2
            // columns x k rows; wz / 64 warps per strip row
            // (a strip row narrower than a warp's 32 column pairs -- the tall
            // shape of a 128 x 32 region -- puts 32 / pairs strips in a warp)
            const int threads = wide / 2 * narrow / k, pairs = wz / 2;
            for (int tid = 0; tid < threads; ++tid) {
                const int warp = tid / 32, lane = tid % 32;
                const int strip = pairs >= 32 ? warp / (pairs / 32) : warp * (32 / pairs) + lane / pairs;
                const int tc = pairs >= 32 ? (warp % (pairs / 32)) * 32 + lane : lane % pairs;
                const int ia = ri0 + 2 * tc, jr0 = rj0 + strip * k;
                unsigned lat = 0, own = 0;
                for (int c = 0; c < 2; ++c)
                    for (int r = 0; r < k; ++r) {
                        const int i = ia + c, j = jr0 + r;
                        if (!interior(i, j)) continue;
                        lat |= 1u << (k * c + r);
                        if (i >= d.oi0 && i < d.oi1 && j >= d.oj0 && j < d.oj1) own |= 1u << (k * c + r);
                    }
                P.thr_geo.push_back(ia);
                P.thr_geo.push_back(jr0);
                P.thr_geo.push_back(static_cast<int>(lat | (own << 16)));
                P.thr_geo.push_back(0);
            }
        }
        P.tiles_shape.push_back(d.shape);
        P.i0.push_back(ri0);
        P.j0.push_back(rj0);
        P.oi0.push_back(d.oi0);
        P.oi1.push_back(d.oi1);
        P.oj0.push_back(d.oj0);
        P.oj1.push_back(d.oj1);
        P.gen_off.push_back(static_cast<int>(P.g_slot.size()));
        P.max_gen = std::max(P.max_gen, static_cast<int>(gens.size()));
        P.max_app = std::max(P.max_app, n_app);
        P.max_ent = std::max(P.max_ent, P.g_ent_off.back() - P.g_ent_off[g0]);
        region_positions += static_cast<long>(wz) * hz;
    }
    // closing offsets: the recipe of entry e spans [rc_off[e], rc_off[e + 1])
    P.e_rc_off.push_back(static_cast<int>(P.rc_cell.size()));
    P.r_rc_off.push_back(static_cast<int>(P.rr_cell.size()));
    P.n_tiles = static_cast<int>(tiles.size());
    region_positions += plan_slabs(inner, p, P);
    P.work_factor = static_cast<double>(region_positions) / static_cast<double>(WW);
    return true;
}

}  // namespace

TilePlan plan_tiles(const LevelTables& t, int wide, int narrow, int k, int slab_rows, int stream_max_p) {
    TilePlan P;
    auto fail = [&](const std::string& why) {
        P.ok = false;
        P.reason = why;
        return P;
    };
    if (!t.box) return fail("no refined box");
    if (t.kind != Integrator::LocalTimeStepping || t.tiers != 1) return fail("single-tier LF-LTS only");
    if (t.p < 2) return fail("p < 2");
    if (t.cfl_safety > 0.0) return fail("per-sample CFL");
    if (wide % 64 || narrow % k || narrow % 32 || (narrow < 64 && 64 % narrow)) return fail("region shape");
    const int m = t.lat_m, W = m + 1, p = t.p;
    const double h = 1.0 / t.lat_inv_h;
    if (std::exp2(std::round(std::log2(h))) != h) return fail("lattice h not a power of two");
    P.wz = wide;
    P.hz = narrow;
    P.k = k;
    P.hs = (narrow + 2) | 1;
    P.box_slots = (wide + 3) * P.hs;
    // coefficient lines: every line row of the box interior starts a strip
    P.line_row.assign(W, 0);
    int jres = -1;
    for (int j = 1; j <= m - 1; ++j) {
        if (t.lat_celly[j] == t.lat_celly[j - 1]) continue;
        P.line_row[j] = 1;
        if (jres < 0) jres = j % k;
        if (j % k != jres) return fail("coefficient lines not aligned to the strip height");
    }
    P.jres = jres < 0 ? 0 : jres;
    // the regular grid first; the frame layout when an edge halo is too narrow
    // (edge halo 2p, 3p, 4p) when an edge halo is too narrow
    std::string why;
    // with streaming: the frame layouts with a streamed interior first
    const bool stream = slab_rows > 2 * p && p <= stream_max_p;
    P.slab_rows = slab_rows;
    for (int attempt = stream ? -6 : 0; attempt < 4; ++attempt) {
        Rect inner;
        const bool streamed = attempt < 0;
        // streamed attempts: halo 2p, 3p, 4p with thin side bands, then the same with full-height ones
        const bool thin = attempt < -3;
        const int he = streamed ? ((attempt + 6) % 3 + 2) * p : (attempt + 1) * p;
        std::vector<TileDesc> tiles = streamed       ? layout_frame(W, p, k, P.jres, wide, narrow, he, &inner, thin)
                                      : attempt == 0 ? layout_grid(W, p, k, P.jres, wide, narrow)
                                                     : layout_frame(W, p, k, P.jres, wide, narrow, he);
        std::string name = attempt == 0 ? "grid" : "frame(" + std::to_string(he) + ")";
        if (streamed) {
            name += thin ? "+thin+stream" : "+stream";
            if (inner.i0 - p < 1 || inner.i1 + p > m || inner.j0 - p < 1 || inner.j1 + p > m) {
                why += name + ": interior too close to the ring; ";
                continue;
            }
        }
        if (tiles.empty()) {
            why += name + ": no layout; ";
            continue;
        }
        if (build_tiles(t, tiles, inner, wide, narrow, k, P)) {
            P.layout = name;
            P.reason.clear();
            P.notes = why;
            P.ok = true;
            return P;
        }
        why += name + ": " + P.reason + "; ";
    }
    return fail(why);
}

}  // namespace wmc
