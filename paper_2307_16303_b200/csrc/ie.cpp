// Host-side pieces of the integral-equation driver (reference solver.cpp /
// kernel.cpp): the collocation grid and the singular cell self-integral of
// 1/r. Restated from the published algorithms; pinned against the reference
// build in tests/test_solver_host.py.
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace h3db {

namespace {

// Gauss-Legendre nodes / weights mapped to [0, 1] by Newton iteration on the
// three-term recurrence (reference solver.cpp:127-148).
void gauss_legendre01(int order, std::vector<double>& nodes, std::vector<double>& weights) {
  nodes.assign(order, 0.0);
  weights.assign(order, 0.0);
  for (int i = 0; i < order; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (order + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p_cur = 1.0, p_prev = 0.0;
      for (int j = 0; j < order; ++j) {
        const double p_old = p_prev;
        p_prev = p_cur;
        p_cur = ((2.0 * j + 1.0) * x * p_prev - j * p_old) / (j + 1.0);
      }
      dp = order * (x * p_cur - p_prev) / (x * x - 1.0);
      const double step = p_cur / dp;
      x -= step;
      if (std::abs(step) < 1e-15) break;
    }
    nodes[i] = 0.5 * (1.0 - x);
    weights[i] = 1.0 / ((1.0 - x * x) * dp * dp);
  }
}

// Tensor Gauss rule for the integral of 1/|u| over the cube [o, o + s]^3
// (reference solver.cpp:150-167).
double box_integral(double ox, double oy, double oz, double s, int order) {
  std::vector<double> t, w;
  gauss_legendre01(order, t, w);
  double sum = 0.0;
  for (int a = 0; a < order; ++a) {
    const double x = ox + s * t[a];
    for (int b = 0; b < order; ++b) {
      const double y = oy + s * t[b];
      double col = 0.0;
      for (int c = 0; c < order; ++c) {
        const double z = oz + s * t[c];
        col += w[c] / std::sqrt(x * x + y * y + z * z);
      }
      sum += w[a] * w[b] * col;
    }
  }
  return sum * s * s * s;
}

// The corner-singular integral over [0,1]^3: the corner octant is the whole
// scaled by 1/4, so I = (sum of the 7 regular octants) * 4/3
// (reference solver.cpp:169-181).
double corner_unit() {
  double shell = 0.0;
  for (int o = 1; o < 8; ++o)
    shell += box_integral(0.5 * (o & 1), 0.5 * ((o >> 1) & 1), 0.5 * ((o >> 2) & 1), 0.5, 40);
  return shell * 4.0 / 3.0;
}

}  // namespace

// integral of 1/|u| over [-1/2, 1/2]^3 (two corner integrals of the half-cell
// scaling, reference solver.cpp:185-188)
double unit_cell_integral_constant() {
  static const double c = 2.0 * corner_unit();
  return c;
}

double cell_self_integral(double h) { return h * h * unit_cell_integral_constant(); }

// Cell centres of the side^3 partition of [-1,1]^3, x-major (reference
// kernel.cpp:96-109).
void tensor_grid_points(std::int64_t n, double* xyz) {
  const auto side = static_cast<std::int64_t>(std::llround(std::cbrt(static_cast<double>(n))));
  if (side * side * side != n)
    throw std::invalid_argument("tensor-grid N must be a perfect cube, got " + std::to_string(n));
  auto centre = [&](std::int64_t k) { return -1.0 + (2.0 * static_cast<double>(k) + 1.0) / static_cast<double>(side); };
  std::int64_t p = 0;
  for (std::int64_t ix = 0; ix < side; ++ix)
    for (std::int64_t iy = 0; iy < side; ++iy)
      for (std::int64_t iz = 0; iz < side; ++iz, ++p) {
        xyz[3 * p] = centre(ix);
        xyz[3 * p + 1] = centre(iy);
        xyz[3 * p + 2] = centre(iz);
      }
}

}  // namespace h3db
