// 1D meshes of the reference's own sampling experiments (smooth1d / jump1d):
// restated from reference proj/src/mesh1d.cpp (build_refined_interval,
// build_hierarchy) with the same arithmetic, so vertex coordinates agree
// bit for bit.
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

struct Hierarchy1D {
    std::vector<Mesh1D> levels;
    std::vector<int> ratios;  // substeps p_l
};

/// reference build_refined_interval (mesh1d.cpp:46-77); fine region [fine_lo, fine_hi]
/// (fine_hi <= fine_lo: uniform mesh)
Mesh1D build_refined_interval(double lo, double hi, double coarse_h, double fine_lo, double fine_hi, double fine_h);

/// reference build_hierarchy (mesh1d.cpp:79-125)
Hierarchy1D build_hierarchy_1d(double lo, double hi, double h0, double fine_lo, double fine_hi, double fine_h,
                               int num_levels);

}  // namespace wmc
