// Host-side geometry for the BASELINE unit-square problems.
//
// The reference has no unit-square generator;
// its only refined 2D mesh is the channel mesh with dyadic 2:1 transition
// frames (reference proj/src/mesh2d.cpp:96-130, :171-283).  This builder keeps
// that idea -- 2:1 grading, 3-triangle transition cells -- but organises it
// as a balanced quadtree over a structured right-triangle grid, so that the
// refined square has a uniform h_min lattice and every vertex lies on that
// lattice.  Fine flags follow the reference rule "small elements plus one
// adjacent layer" (mesh2d.cpp:285-301) with the threshold measured against
// the coarse element's longest edge.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace wmc {

struct TriMesh {
    std::vector<std::array<double, 2>> vertices;
    std::vector<std::array<int, 3>> triangles;  // counter-clockwise
    std::vector<std::uint8_t> fine_flags;       // per triangle: 0 coarse, k >= 1 tier (selector P_k = flag >= k)
    std::vector<std::uint8_t> boundary_vertex;  // per vertex (Dirichlet)
    std::vector<std::array<int, 2>> lattice;    // integer lattice coordinates (units of fine_h)
    int fine_box_lo = -1, fine_box_hi = -1;     // refined square [lo, hi]^2 in lattice units (-1: none)
    double coarse_h = 0.0;
    double fine_h = 0.0;

    int n_vertices() const { return static_cast<int>(vertices.size()); }
    int n_triangles() const { return static_cast<int>(triangles.size()); }
    double signed_area(int t) const {
        const auto& a = vertices[triangles[t][0]];
        const auto& b = vertices[triangles[t][1]];
        const auto& c = vertices[triangles[t][2]];
        return 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1]));
    }
    std::array<double, 2> centroid(int t) const {
        const auto& a = vertices[triangles[t][0]];
        const auto& b = vertices[triangles[t][1]];
        const auto& c = vertices[triangles[t][2]];
        return {(a[0] + b[0] + c[0]) / 3.0, (a[1] + b[1] + c[1]) / 3.0};
    }
    double longest_edge(int t) const;
};

struct SquareMeshSpec {
    int n_coarse = 32;       // coarse cells per side, h = 1 / n_coarse
    int ratio = 4;           // h / h_min, a power of two (1 = uniform mesh)
    double fine_lo = 0.45;   // refined square [fine_lo, fine_hi]^2 ...
    double fine_hi = 0.55;
    double snap = 1.0 / 16;  // ... snapped outward to this grid (level-0 grid)
    double small_factor = 0.7;  // small: longest edge < small_factor * sqrt(2) * h
};

/// Unit square, structured right triangles (SW-NE diagonals), refined square
/// at h / ratio with 2:1 balanced transitions.  Throws std::invalid_argument on
/// bad specs.
TriMesh build_refined_square(const SquareMeshSpec& spec);

struct LShapeMeshSpec {
    int n_per_unit = 16;        // h = 1 / n_per_unit on [-1,1]^2 minus [0,1]x[-1,0]
    int tiers = 3;              // refinement tiers toward the re-entrant corner (0,0): h/2 .. h/2^tiers
    double grade_radius = 0.25;  // element size target h * sqrt(r / grade_radius) near the corner
};

/// Graded L-shape (BASELINE config 2, no reference counterpart: the
/// reference L-shape, src/mesh_graded.cpp:48-112, is a different domain with
/// no fine flags).  Balanced quadtree as build_refined_square; a leaf of side
/// s is split while s > h * sqrt(r / grade_radius), r = distance of the leaf
/// to the corner, down to h / 2^tiers.  fine_flags[t] = refinement tier
/// (0 = coarse) of the triangle, raised to the largest tier among the
/// triangles sharing one of its vertices (the reference's "plus one adjacent
/// layer", mesh2d.cpp:285-301, applied per tier).  Dirichlet on the whole
/// boundary (edges of one triangle).
TriMesh build_graded_lshape(const LShapeMeshSpec& spec);

/// Reference fixture format (reference proj/src/mesh_io.cpp:1-9).
void dump_mesh_text(const TriMesh& mesh, const std::string& path);

}  // namespace wmc
