#include "field.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace wmc {

namespace {

struct Mode1D {
    double omega, lambda;
    bool even;
};

// 1D eigenpairs of exp(-|x - y| / l) on [-a, a], a = 1/2:
// lambda = 2c / (omega^2 + c^2), c = 1/l, with
//   even (cos):  c - omega tan(omega a) = 0,  omega a in (k pi, k pi + pi/2)
//   odd  (sin):  omega + c tan(omega a) = 0,  omega a in (k pi + pi/2, (k+1) pi)
std::vector<Mode1D> modes_1d(double corr_len, int count) {
    const double a = 0.5, c = 1.0 / corr_len, pi = 3.14159265358979323846;
    std::vector<Mode1D> out;
    for (int k = 0; static_cast<int>(out.size()) < count; ++k) {
        for (int parity = 0; parity < 2 && static_cast<int>(out.size()) < count; ++parity) {
            const bool even = parity == 0;
            double lo = even ? k * pi : k * pi + pi / 2, hi = even ? k * pi + pi / 2 : (k + 1) * pi;
            lo = (lo + 1e-12) / a;
            hi = (hi - 1e-12) / a;
            auto f = [&](double w) { return even ? c - w * std::tan(w * a) : w + c * std::tan(w * a); };
            double flo = f(lo);
            for (int it = 0; it < 200; ++it) {
                const double mid = 0.5 * (lo + hi);
                const double fm = f(mid);
                if ((fm > 0) == (flo > 0)) {
                    lo = mid;
                    flo = fm;
                } else {
                    hi = mid;
                }
            }
            const double w = 0.5 * (lo + hi);
            out.push_back({w, 2.0 * c / (w * w + c * c), even});
        }
    }
    std::sort(out.begin(), out.end(), [](const Mode1D& x, const Mode1D& y) { return x.lambda > y.lambda; });
    return out;
}

double phi_norm(const Mode1D& m) {
    const double a = 0.5, w = m.omega;
    return m.even ? std::sqrt(a + std::sin(2.0 * w * a) / (2.0 * w)) : std::sqrt(a - std::sin(2.0 * w * a) / (2.0 * w));
}
double phi(const Mode1D& m, double x) {  // x in [-1/2, 1/2], L2-normalised
    return (m.even ? std::cos(m.omega * x) : std::sin(m.omega * x)) / phi_norm(m);
}

}  // namespace

namespace {

struct Pair2D {
    int i, j;
    double lambda;
};

// the `modes` largest products of 1D eigenvalues (stable order)
std::vector<Pair2D> largest_pairs(const std::vector<Mode1D>& m1, int modes) {
    const int n1 = static_cast<int>(m1.size());
    std::vector<Pair2D> pairs;
    for (int i = 0; i < n1; ++i)
        for (int j = 0; j < n1; ++j) pairs.push_back({i, j, m1[i].lambda * m1[j].lambda});
    std::stable_sort(pairs.begin(), pairs.end(), [](const Pair2D& x, const Pair2D& y) { return x.lambda > y.lambda; });
    pairs.resize(modes);
    return pairs;
}

}  // namespace

KLTable kl_point_table(const std::vector<double>& xy, double sigma, double corr_len, int modes) {
    if (xy.size() % 2 || modes < 1 || !(sigma >= 0.0) || !(corr_len > 0.0))
        throw std::invalid_argument("kl_point_table: bad parameters");
    const std::vector<Mode1D> m1 = modes_1d(corr_len, modes + 8);  // enough 1D modes for the largest products
    const std::vector<Pair2D> pairs = largest_pairs(m1, modes);
    KLTable t;
    t.cells = static_cast<int>(xy.size() / 2);
    t.modes = modes;
    t.t.resize(static_cast<std::size_t>(t.cells) * modes);
    for (const auto& p : pairs) t.lambda.push_back(p.lambda);
    for (int c = 0; c < t.cells; ++c) {
        const double x = xy[2 * c] - 0.5, y = xy[2 * c + 1] - 0.5;
        for (int m = 0; m < modes; ++m)
            t.t[static_cast<std::size_t>(c) * modes + m] =
                sigma * std::sqrt(pairs[m].lambda) * phi(m1[pairs[m].i], x) * phi(m1[pairs[m].j], y);
    }
    return t;
}

std::vector<double> kl_mode_list(double sigma, double corr_len, int modes) {
    if (modes < 1 || !(sigma >= 0.0) || !(corr_len > 0.0)) throw std::invalid_argument("kl_mode_list: bad parameters");
    const std::vector<Mode1D> m1 = modes_1d(corr_len, modes + 8);
    const std::vector<Pair2D> pairs = largest_pairs(m1, modes);
    std::vector<double> out;
    for (const auto& p : pairs) {
        const Mode1D &mx = m1[p.i], &my = m1[p.j];
        out.insert(out.end(), {sigma * std::sqrt(p.lambda), mx.omega, mx.even ? 1.0 : 0.0, phi_norm(mx), my.omega,
                               my.even ? 1.0 : 0.0, phi_norm(my)});
    }
    return out;
}

KLTable kl_cell_table(int cells_x, int cells_y, double sigma, double corr_len, int modes) {
    if (cells_x < 1 || cells_y < 1) throw std::invalid_argument("kl_cell_table: bad parameters");
    std::vector<double> xy;
    for (int iy = 0; iy < cells_y; ++iy)
        for (int ix = 0; ix < cells_x; ++ix) {
            xy.push_back((ix + 0.5) / cells_x);
            xy.push_back((iy + 0.5) / cells_y);
        }
    return kl_point_table(xy, sigma, corr_len, modes);
}

}  // namespace wmc
