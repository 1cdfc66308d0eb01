// Log-normal random coefficient for BASELINE config 4 (no reference
// counterpart: the reference's only KL field is 1D with U(-1,1) weights,
// src/rng.cpp:42-51, 66-84).
//
// g(x) = sigma * sum_{m < modes} sqrt(lambda_m) xi_m phi_m(x), xi_m ~ N(0,1),
// c = exp(g), for the separable exponential covariance
// C(x, y) = exp(-|x1 - y1| / l - |x2 - y2| / l) on the unit square, whose
// eigenpairs are products of the analytic 1D pairs (roots of the even/odd
// transcendental equations, solved by bisection).  The field is sampled at
// the centres of a cells_x x cells_y grid (the coefficient is piecewise
// constant per cell, like the uniform configs), so every kernel keeps its
// cell-coefficient form; the table T[cell][m] = sigma sqrt(lambda_m)
// phi_m(centre) is shared by the device draw and the oracles.
#pragma once

#include <vector>

namespace wmc {

struct KLTable {
    int cells = 0, modes = 0;
    std::vector<double> t;       // [cell * modes + m]
    std::vector<double> lambda;  // 2D eigenvalues (unit variance), descending
};

KLTable kl_cell_table(int cells_x, int cells_y, double sigma, double corr_len, int modes);

// The same expansion at arbitrary points of the unit square (xy interleaved,
// one table row per point): the per-element field, evaluated at every
// triangle's centroid as the reference's assemble does (src/fem.cpp:103-104).
KLTable kl_point_table(const std::vector<double>& xy, double sigma, double corr_len, int modes);

// The expansion's modes for a pointwise evaluator (the reference-side driver):
// 7 numbers per mode -- amp = sigma sqrt(lambda_m), then omega, even (1 / 0)
// and norm of the x and of the y factor, phi(t) = (even ? cos : sin)(omega (t - 1/2)) / norm.
std::vector<double> kl_mode_list(double sigma, double corr_len, int modes);

}  // namespace wmc
