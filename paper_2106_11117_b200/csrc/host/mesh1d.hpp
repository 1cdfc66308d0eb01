// 1D meshes of the reference's own sampling experiments (smooth1d / jump1d).
// The product takes them from the caller (wmc_mesh1d_create): the adapter
// passes the reference's Mesh1D of each level of its build_hierarchy
// (reference proj/include/wavemc/mesh.hpp:21-33, src/mesh1d.cpp:76-125).
#pragma once

#include <cstdint>
#include <vector>

namespace wmc {

struct Mesh1D {
    std::vector<double> vertices;          // sorted, n + 1
    std::vector<std::uint8_t> fine_flags;  // per element
    double coarse_h = 0.0, fine_h = 0.0;

    int n_elements() const { return static_cast<int>(vertices.size()) - 1; }
    int n_vertices() const { return static_cast<int>(vertices.size()); }
    double element_size(int e) const { return vertices[e + 1] - vertices[e]; }
    double midpoint(int e) const { return 0.5 * (vertices[e] + vertices[e + 1]); }
};

}  // namespace wmc
