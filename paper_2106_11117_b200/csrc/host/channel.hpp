// The reference's narrow-channel sampling experiment (make_problem
// Channel2d, src/experiments.cpp:108-172): per sample the channel width b ~
// U[0.001, 0.007] (sample_width, src/rng.cpp:59-64) moves the vertices of the
// reference mesh by y' = y + blend(x) profile(y) (ChannelGeometry,
// src/mesh2d.cpp:361-389), and the solve assembles the transformed mesh
// (speed 1, Neumann: every vertex a DOF), takes the per-sample CFL step with
// warm starts from the reference mesh, starts from the bump u0 and records u
// on the line x = -0.4 (extract_line_qoi, src/fem.cpp:295-340).
//
// The geometry change is confined to triangles with a moving vertex
// (|x| < 0.1), so the level's operator splits into sample-independent entries
// (cell 0, the usual a0 = K_ij / sqrt(M_i M_j)) and per-sample entries: every
// pair coupled by a moving triangle or touching a vertex whose lumped mass
// moves gets its own cell k >= 1 with a0 = 1, and the device evaluates
// c_k = A_ij(b) = K_ij(b) / sqrt(M_i(b) M_j(b)) per sample from the tables
// below (ChannelArgs, draw_channel_kernel).  A_ij = A_ji share a cell.
#pragma once

#include <vector>

#include "level.hpp"
#include "mesh.hpp"

namespace wmc {

// include/wavemc/mesh.hpp:82-86, include/wavemc/rng.hpp:52-53, src/experiments.cpp:170
constexpr double kChannelRefWidth = 0.004;
constexpr double kChannelHalfLength = 0.05;
constexpr double kChannelBlendOuter = 0.1;
constexpr double kChannelRectHalfHeight = 0.5;
constexpr double kChannelRectWidth = 0.95;
constexpr double kChannelWidthLo = 0.001, kChannelWidthHi = 0.007;
constexpr double kChannelLineX = -0.4;

double channel_blend(double x);                  // ChannelGeometry::blend
double channel_profile(double y, double width);  // ChannelGeometry::profile

// Per-sample operator data of a channel level ("local" vertices are those of
// moving triangles; every vertex of the arrays below is local unless marked)
struct ChannelTables {
    int n_local = 0;
    std::vector<double> vx, vy, vblend;  // per local vertex: reference position and blend(x)
    std::vector<int> tri;                // moving triangles: 3 local vertices each, mesh corner order
    std::vector<double> ms;              // per local vertex: lumped mass of its fixed triangles
    std::vector<int> m_ptr, m_tri;       // per local vertex: its moving triangles
    // per per-sample cell k >= 1 (index k - 1): the pair (i, j) as local
    // vertices (-1: not local, fixed mass e_mi / e_mj), the fixed triangles'
    // stiffness, and the moving triangles coupling the pair, t * 9 + a * 3 + b
    // with a, b the pair's corners in triangle t
    std::vector<int> e_li, e_lj;
    std::vector<double> e_mi, e_mj, e_ks;
    std::vector<int> k_ptr, k_tri;
};

// Level tables of one channel level on the reference mesh `mesh` (the
// reference's build_channel_mesh output, passed in by the caller).
LevelTables build_level_tables_channel(const TriMesh& mesh, const LevelSpec& spec, ChannelTables& ch);

}  // namespace wmc
