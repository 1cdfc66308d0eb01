#include "mesh.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <stdexcept>
#include <unordered_map>
#include <unordered_set>

namespace wmc {

double TriMesh::longest_edge(int t) const {
    double best = 0.0;
    for (int e = 0; e < 3; ++e) {
        const auto& a = vertices[triangles[t][e]];
        const auto& b = vertices[triangles[t][(e + 1) % 3]];
        best = std::max(best, std::hypot(b[0] - a[0], b[1] - a[1]));
    }
    return best;
}

namespace {

// Leaves of the quadtree live on the integer lattice of the finest size; a
// leaf of level k has side 2^k units and is keyed by (k, x0 >> k, y0 >> k).
struct Quadtree {
    int levels = 0;  // coarse level K: coarse side = 2^K units
    long extent = 0;  // domain side in units
    long cut = -1;    // L-shape: unit cells with px >= cut and py < cut lie outside (-1: square)
    std::unordered_set<std::uint64_t> leaves;

    bool outside(long px, long py) const {
        return px < 0 || py < 0 || px >= extent || py >= extent || (cut >= 0 && px >= cut && py < cut);
    }

    static std::uint64_t key(int k, long i, long j) {
        return (std::uint64_t(k) << 56) | (std::uint64_t(i) << 28) | std::uint64_t(j);
    }
    bool has(int k, long x0, long y0) const { return leaves.count(key(k, x0 >> k, y0 >> k)) != 0; }

    // side of the leaf covering unit cell (px, py); 0 outside the domain
    long size_at(long px, long py) const {
        if (outside(px, py)) return 0;
        for (int k = 0; k <= levels; ++k)
            if (leaves.count(key(k, px >> k, py >> k))) return 1L << k;
        throw std::logic_error("quadtree: unit cell not covered");
    }

    void split(int k, long x0, long y0) {
        leaves.erase(key(k, x0 >> k, y0 >> k));
        const long h = 1L << (k - 1);
        for (long dy = 0; dy < 2; ++dy)
            for (long dx = 0; dx < 2; ++dx)
                leaves.insert(key(k - 1, (x0 + dx * h) >> (k - 1), (y0 + dy * h) >> (k - 1)));
    }

    struct Leaf {
        int k;
        long x0, y0;
    };
    std::vector<Leaf> list() const {
        std::vector<Leaf> out;
        out.reserve(leaves.size());
        for (std::uint64_t key : leaves) {
            const int k = static_cast<int>(key >> 56);
            const long i = static_cast<long>((key >> 28) & ((1ULL << 28) - 1));
            const long j = static_cast<long>(key & ((1ULL << 28) - 1));
            out.push_back({k, i << k, j << k});
        }
        std::sort(out.begin(), out.end(), [](const Leaf& a, const Leaf& b) {
            if (a.y0 != b.y0) return a.y0 < b.y0;
            if (a.x0 != b.x0) return a.x0 < b.x0;
            return a.k < b.k;
        });
        return out;
    }

    // true if some leaf touching the side of (or a corner of) this leaf is
    // smaller than half its size: 2:1 balance across edges and corners
    bool unbalanced(int k, long x0, long y0) const {
        const long s = 1L << k;
        if (s <= 2) return false;
        const long lim = s / 2;
        for (long t = 0; t < s; ++t) {
            long v;
            if ((v = size_at(x0 + t, y0 - 1)) && v < lim) return true;
            if ((v = size_at(x0 + t, y0 + s)) && v < lim) return true;
            if ((v = size_at(x0 - 1, y0 + t)) && v < lim) return true;
            if ((v = size_at(x0 + s, y0 + t)) && v < lim) return true;
        }
        const long cx[4] = {x0 - 1, x0 + s, x0 - 1, x0 + s};
        const long cy[4] = {y0 - 1, y0 - 1, y0 + s, y0 + s};
        for (int c = 0; c < 4; ++c) {
            const long v = size_at(cx[c], cy[c]);
            if (v && v < lim) return true;
        }
        return false;
    }
};

int ilog2_exact(int v) {
    int k = 0;
    while ((1 << k) < v) ++k;
    if ((1 << k) != v) throw std::invalid_argument("build_refined_square: ratio must be a power of two");
    return k;
}

// triangulate the leaves: plain cells split along the SW-NE diagonal, one
// hanging midpoint -> three triangles (the reference 2:1 cell,
// mesh2d.cpp:96-130), two or more -> fan around the cell centre.  Vertices in
// lattice units, tri_level = quadtree level of each triangle's leaf.
void triangulate(const Quadtree& tree, std::vector<std::array<long, 2>>& lat, std::vector<std::array<int, 3>>& tris,
                 std::vector<int>& tri_level) {
    std::map<std::pair<long, long>, int> vid;
    lat.clear();
    tris.clear();
    tri_level.clear();
    auto vertex = [&](long x, long y) {
        const auto it = vid.find({y, x});
        if (it != vid.end()) return it->second;
        const int id = static_cast<int>(lat.size());
        vid.emplace(std::make_pair(y, x), id);
        lat.push_back({x, y});
        return id;
    };
    for (const auto& leaf : tree.list()) {
        const long s = 1L << leaf.k;
        const long x0 = leaf.x0, y0 = leaf.y0;
        // corners CCW: SW, SE, NE, NW; side e runs from corner e to corner e+1
        const long cx[4] = {x0, x0 + s, x0 + s, x0};
        const long cy[4] = {y0, y0, y0 + s, y0 + s};
        bool hang[4] = {false, false, false, false};
        if (s >= 2) {
            long v;
            hang[0] = (v = tree.size_at(x0 + s / 2, y0 - 1)) && v < s;  // bottom
            hang[1] = (v = tree.size_at(x0 + s, y0 + s / 2)) && v < s;  // right
            hang[2] = (v = tree.size_at(x0 + s / 2, y0 + s)) && v < s;  // top
            hang[3] = (v = tree.size_at(x0 - 1, y0 + s / 2)) && v < s;  // left
        }
        const int nh = hang[0] + hang[1] + hang[2] + hang[3];
        int c[4];
        for (int e = 0; e < 4; ++e) c[e] = vertex(cx[e], cy[e]);
        if (nh == 0) {
            tris.push_back({c[0], c[1], c[2]});
            tris.push_back({c[0], c[2], c[3]});
            tri_level.insert(tri_level.end(), 2, leaf.k);
        } else if (nh == 1) {
            int e = 0;
            while (!hang[e]) ++e;
            const int c0 = c[e], c1 = c[(e + 1) % 4], c2 = c[(e + 2) % 4], c3 = c[(e + 3) % 4];
            const int m = vertex((cx[e] + cx[(e + 1) % 4]) / 2, (cy[e] + cy[(e + 1) % 4]) / 2);
            tris.push_back({c0, m, c3});
            tris.push_back({m, c2, c3});
            tris.push_back({m, c1, c2});
            tri_level.insert(tri_level.end(), 3, leaf.k);
        } else {
            const int o = vertex(x0 + s / 2, y0 + s / 2);
            for (int e = 0; e < 4; ++e) {
                const int a = c[e], b = c[(e + 1) % 4];
                if (hang[e]) {
                    const int m = vertex((cx[e] + cx[(e + 1) % 4]) / 2, (cy[e] + cy[(e + 1) % 4]) / 2);
                    tris.push_back({o, a, m});
                    tris.push_back({o, m, b});
                    tri_level.insert(tri_level.end(), 2, leaf.k);
                } else {
                    tris.push_back({o, a, b});
                    tri_level.push_back(leaf.k);
                }
            }
        }
    }
}

// vertex renumbering row-major (y, then x) for a deterministic order
std::vector<int> row_major_rank(const std::vector<std::array<long, 2>>& lat) {
    std::vector<int> order(lat.size());
    for (std::size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        if (lat[a][1] != lat[b][1]) return lat[a][1] < lat[b][1];
        return lat[a][0] < lat[b][0];
    });
    std::vector<int> rank(lat.size());
    for (std::size_t i = 0; i < order.size(); ++i) rank[order[i]] = static_cast<int>(i);
    return rank;
}

// 2:1 balance across edges and corners
void balance(Quadtree& tree) {
    for (bool changed = true; changed;) {
        changed = false;
        for (const auto& leaf : tree.list())
            if (tree.has(leaf.k, leaf.x0, leaf.y0) && tree.unbalanced(leaf.k, leaf.x0, leaf.y0)) {
                tree.split(leaf.k, leaf.x0, leaf.y0);
                changed = true;
            }
    }
}

}  // namespace

TriMesh build_refined_square(const SquareMeshSpec& spec) {
    if (spec.n_coarse < 2) throw std::invalid_argument("build_refined_square: n_coarse >= 2");
    if (spec.ratio < 1) throw std::invalid_argument("build_refined_square: ratio >= 1");
    if (!(spec.fine_lo < spec.fine_hi) || spec.fine_lo < 0.0 || spec.fine_hi > 1.0)
        throw std::invalid_argument("build_refined_square: bad refined square");
    const int K = ilog2_exact(spec.ratio);
    const long n = spec.n_coarse;
    const long R = spec.ratio;
    const long extent = n * R;
    if (extent >= (1L << 27)) throw std::invalid_argument("build_refined_square: mesh too large");

    // snap the refined square outward to the snap grid, then to the coarse grid
    const double snap = spec.snap > 0.0 ? spec.snap : 1.0 / static_cast<double>(n);
    const double lo = std::floor(spec.fine_lo / snap + 1e-9) * snap;
    const double hi = std::ceil(spec.fine_hi / snap - 1e-9) * snap;
    const long qa = static_cast<long>(std::floor(lo * n + 1e-9)) * R;
    const long qb = static_cast<long>(std::ceil(hi * n - 1e-9)) * R;

    Quadtree tree;
    tree.levels = K;
    tree.extent = extent;
    for (long j = 0; j < n; ++j)
        for (long i = 0; i < n; ++i) tree.leaves.insert(Quadtree::key(K, i, j));

    if (R > 1) {
        // refine the cells inside the square to the finest lattice
        for (long j = 0; j < n; ++j)
            for (long i = 0; i < n; ++i) {
                const long x0 = i * R, y0 = j * R;
                if (x0 >= qa && x0 + R <= qb && y0 >= qa && y0 + R <= qb) {
                    std::vector<Quadtree::Leaf> work{{K, x0, y0}};
                    while (!work.empty()) {
                        const auto leaf = work.back();
                        work.pop_back();
                        if (leaf.k == 0) continue;
                        tree.split(leaf.k, leaf.x0, leaf.y0);
                        const long h = 1L << (leaf.k - 1);
                        for (long dy = 0; dy < 2; ++dy)
                            for (long dx = 0; dx < 2; ++dx)
                                work.push_back({leaf.k - 1, leaf.x0 + dx * h, leaf.y0 + dy * h});
                    }
                }
            }
        balance(tree);
    }

    std::vector<std::array<long, 2>> lat;
    std::vector<std::array<int, 3>> tris;
    std::vector<int> tri_level;
    triangulate(tree, lat, tris, tri_level);
    std::vector<int> rank = row_major_rank(lat);

    TriMesh mesh;
    mesh.coarse_h = 1.0 / static_cast<double>(n);
    mesh.fine_h = mesh.coarse_h / static_cast<double>(R);
    if (R > 1 && qb > qa) {
        mesh.fine_box_lo = static_cast<int>(qa);
        mesh.fine_box_hi = static_cast<int>(qb);
    }
    const double unit = mesh.fine_h;
    mesh.vertices.resize(lat.size());
    mesh.lattice.resize(lat.size());
    mesh.boundary_vertex.assign(lat.size(), 0);
    for (std::size_t i = 0; i < lat.size(); ++i) {
        const int r = rank[i];
        mesh.vertices[r] = {static_cast<double>(lat[i][0]) * unit, static_cast<double>(lat[i][1]) * unit};
        mesh.lattice[r] = {static_cast<int>(lat[i][0]), static_cast<int>(lat[i][1])};
        if (lat[i][0] == 0 || lat[i][1] == 0 || lat[i][0] == extent || lat[i][1] == extent)
            mesh.boundary_vertex[r] = 1;
    }
    mesh.triangles.reserve(tris.size());
    for (const auto& t : tris) {
        std::array<int, 3> tt{rank[t[0]], rank[t[1]], rank[t[2]]};
        mesh.triangles.push_back(tt);
        if (!(mesh.signed_area(mesh.n_triangles() - 1) > 0.0))
            throw std::logic_error("build_refined_square: non-CCW triangle");
    }

    // fine flags: small elements plus one adjacent layer (mesh2d.cpp:285-301)
    const int nt = mesh.n_triangles();
    const double threshold = spec.small_factor * std::sqrt(2.0) * mesh.coarse_h;
    std::vector<std::uint8_t> small(nt, 0), touched(mesh.n_vertices(), 0);
    for (int t = 0; t < nt; ++t)
        if (R > 1 && mesh.longest_edge(t) < threshold) {
            small[t] = 1;
            for (int v : mesh.triangles[t]) touched[v] = 1;
        }
    mesh.fine_flags.assign(nt, 0);
    for (int t = 0; t < nt; ++t) {
        if (small[t]) {
            mesh.fine_flags[t] = 1;
            continue;
        }
        for (int v : mesh.triangles[t])
            if (touched[v]) {
                mesh.fine_flags[t] = 1;
                break;
            }
    }
    return mesh;
}

TriMesh build_graded_lshape(const LShapeMeshSpec& spec) {
    if (spec.n_per_unit < 1) throw std::invalid_argument("build_graded_lshape: n_per_unit >= 1");
    if (spec.tiers < 0 || spec.tiers > 6) throw std::invalid_argument("build_graded_lshape: tiers in [0, 6]");
    if (!(spec.grade_radius > 0.0)) throw std::invalid_argument("build_graded_lshape: grade_radius > 0");
    const int K = spec.tiers;
    const long n = spec.n_per_unit;  // coarse cells per unit length
    const long R = 1L << K;
    const long extent = 2 * n * R;   // [-1, 1] in lattice units
    if (extent >= (1L << 27)) throw std::invalid_argument("build_graded_lshape: mesh too large");
    const long corner = n * R;       // (0, 0) in lattice units
    const double h = 1.0 / static_cast<double>(n);
    const double unit = h / static_cast<double>(R);

    Quadtree tree;
    tree.levels = K;
    tree.extent = extent;
    tree.cut = corner;  // the quadrant x >= 0, y < 0 is not in the domain
    for (long j = 0; j < 2 * n; ++j)
        for (long i = 0; i < 2 * n; ++i)
            if (!tree.outside(i * R, j * R)) tree.leaves.insert(Quadtree::key(K, i, j));

    // grading toward the corner: split a leaf of side s while
    // s > h sqrt(r / rho), i.e. r < rho (s / h)^2, r = leaf-to-corner distance
    std::vector<Quadtree::Leaf> work = tree.list();
    while (!work.empty()) {
        const auto leaf = work.back();
        work.pop_back();
        if (leaf.k == 0) continue;
        const long s = 1L << leaf.k;
        const long dx = std::max({leaf.x0 - corner, 0L, corner - (leaf.x0 + s)});
        const long dy = std::max({leaf.y0 - corner, 0L, corner - (leaf.y0 + s)});
        const double r = std::hypot(static_cast<double>(dx), static_cast<double>(dy)) * unit;
        const double rel = static_cast<double>(s) * unit / h;
        if (!(r < spec.grade_radius * rel * rel)) continue;
        tree.split(leaf.k, leaf.x0, leaf.y0);
        const long hs = s / 2;
        for (long cy = 0; cy < 2; ++cy)
            for (long cx = 0; cx < 2; ++cx) work.push_back({leaf.k - 1, leaf.x0 + cx * hs, leaf.y0 + cy * hs});
    }
    balance(tree);

    std::vector<std::array<long, 2>> lat;
    std::vector<std::array<int, 3>> tris;
    std::vector<int> tri_level;
    triangulate(tree, lat, tris, tri_level);
    const std::vector<int> rank = row_major_rank(lat);

    TriMesh mesh;
    mesh.coarse_h = h;
    mesh.fine_h = unit;
    mesh.vertices.resize(lat.size());
    mesh.lattice.resize(lat.size());
    for (std::size_t i = 0; i < lat.size(); ++i) {
        const int r = rank[i];
        mesh.vertices[r] = {static_cast<double>(lat[i][0] - corner) * unit,
                            static_cast<double>(lat[i][1] - corner) * unit};
        mesh.lattice[r] = {static_cast<int>(lat[i][0]), static_cast<int>(lat[i][1])};
    }
    mesh.triangles.reserve(tris.size());
    for (const auto& t : tris) {
        mesh.triangles.push_back({rank[t[0]], rank[t[1]], rank[t[2]]});
        if (!(mesh.signed_area(mesh.n_triangles() - 1) > 0.0))
            throw std::logic_error("build_graded_lshape: non-CCW triangle");
    }
    // Dirichlet boundary: vertices of edges that belong to one triangle
    std::map<std::pair<int, int>, int> edges;
    for (const auto& t : mesh.triangles)
        for (int e = 0; e < 3; ++e) {
            const int a = t[e], b = t[(e + 1) % 3];
            ++edges[{std::min(a, b), std::max(a, b)}];
        }
    mesh.boundary_vertex.assign(mesh.vertices.size(), 0);
    for (const auto& [e, count] : edges)
        if (count == 1) mesh.boundary_vertex[e.first] = mesh.boundary_vertex[e.second] = 1;

    // tiers: the leaf's depth below the coarse level, then one adjacent layer
    const int nt = mesh.n_triangles();
    std::vector<std::uint8_t> vtier(mesh.vertices.size(), 0);
    for (int t = 0; t < nt; ++t) {
        const auto tier = static_cast<std::uint8_t>(K - tri_level[t]);
        for (int v : mesh.triangles[t]) vtier[v] = std::max(vtier[v], tier);
    }
    mesh.fine_flags.assign(nt, 0);
    for (int t = 0; t < nt; ++t)
        for (int v : mesh.triangles[t]) mesh.fine_flags[t] = std::max(mesh.fine_flags[t], vtier[v]);
    return mesh;
}

void dump_mesh_text(const TriMesh& mesh, const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("dump_mesh_text: cannot open " + path);
    std::fprintf(f, "wavemc-mesh-2d %d %d %.17g %.17g\n", mesh.n_vertices(), mesh.n_triangles(),
                 mesh.coarse_h, mesh.fine_h);
    for (const auto& v : mesh.vertices) std::fprintf(f, "v %.17g %.17g\n", v[0], v[1]);
    for (int t = 0; t < mesh.n_triangles(); ++t)
        std::fprintf(f, "t %d %d %d %d\n", mesh.triangles[t][0], mesh.triangles[t][1],
                     mesh.triangles[t][2], int(mesh.fine_flags[t]));
    std::fclose(f);
}

}  // namespace wmc
