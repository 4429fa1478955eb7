// BASELINE problem generators for the checker side — TEST INFRASTRUCTURE ONLY.
//
// The reference generates none of the five BASELINE matrices (
// its gen_conv_diff is centred with identity Dirichlet rows,
// proj/src/problems.cpp:292-377), so the product ships its own generators
// (paper_2503_22631_b200/csrc/problems.cpp, gen.cu). This file restates the
// same definitions independently of that code so that
//   * bench.py's reference arm builds its inputs without loading the product
//     library (the timed CPU baseline touches oracle/ only), and
//   * the tests check the product generators bit-for-bit against a second
//     implementation instead of trusting the code under test.
// Conventions: lexicographic node order (ix*N + iy)*N + iz
// (problems.cpp:30-32); CSR rows with strictly increasing columns; every value
// is formed by the same floating-point expression as the definition below, so
// the arrays agree bit-for-bit (summation orders are stated).
//
// Build: oracle/Makefile links this TU into liboracle.so.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

extern "C" void orc_gaussian_vector(uint64_t seed, int64_t n, double* out);

namespace {

// rows [0, n) split over the host threads (static blocks)
template <class F>
void rows_parallel(int64_t n, F&& fn) {
  unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  if (n < (int64_t(1) << 16)) nt = 1;
  std::vector<std::thread> ts;
  for (unsigned t = 0; t < nt; ++t) {
    const int64_t a = n * t / nt, b = n * (t + 1) / nt;
    if (a < b) ts.emplace_back([&fn, a, b] { fn(a, b); });
  }
  for (auto& th : ts) th.join();
}

// A stencil row emitter: for each row, the neighbours come out in increasing
// column order, so the prefix sums of the counts are the row pointers.
struct Grid3 {
  int64_t N;
  int64_t id(int64_t x, int64_t y, int64_t z) const { return (x * N + y) * N + z; }
  void xyz(int64_t r, int64_t& x, int64_t& y, int64_t& z) const {
    z = r % N;
    y = (r / N) % N;
    x = r / (N * N);
  }
};

}  // namespace

extern "C" {

// 5-point (dim 2, nodes (ix, iy), id ix*N + iy) or 7-point (dim 3) Dirichlet
// Laplacian on the N^dim interior nodes, h = 1/(N+1), scaled by h^-2:
// diagonal 2*dim/h^2, each existing neighbour -1/h^2.
int orc_gen_laplacian(int dim, int64_t N, int64_t* n_out, int64_t* nnz_out, int64_t* rp,
                      int32_t* ci, double* v) {
  if ((dim != 2 && dim != 3) || N < 1) return 1;
  const int64_t n = dim == 3 ? N * N * N : N * N;
  *n_out = n;
  // each axis loses one neighbour on each of its two boundary layers
  *nnz_out = (2 * dim + 1) * n - 2 * dim * (n / N);
  if (!rp) return 0;
  const double h = 1.0 / double(N + 1);
  const double s = 1.0 / (h * h);
  const double diag = 2.0 * dim * s;
  std::vector<int64_t> strides = dim == 3 ? std::vector<int64_t>{N * N, N, 1}
                                          : std::vector<int64_t>{N, 1};
  auto coord = [&](int64_t r, int a) { return (r / strides[size_t(a)]) % N; };
  rp[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    int64_t cnt = 1;
    for (int a = 0; a < dim; ++a) {
      const int64_t c = coord(r, a);
      cnt += (c > 0 ? 1 : 0) + (c + 1 < N ? 1 : 0);
    }
    rp[r + 1] = rp[r] + cnt;
  }
  rows_parallel(n, [&](int64_t a0, int64_t a1) {
    for (int64_t r = a0; r < a1; ++r) {
      int64_t k = rp[r];
      for (int a = 0; a < dim; ++a)  // below: the largest stride first
        if (coord(r, a) > 0) { ci[k] = int32_t(r - strides[size_t(a)]); v[k++] = -s; }
      ci[k] = int32_t(r);
      v[k++] = diag;
      for (int a = dim - 1; a >= 0; --a)  // above: the smallest stride first
        if (coord(r, a) + 1 < N) { ci[k] = int32_t(r + strides[size_t(a)]); v[k++] = -s; }
    }
  });
  return 0;
}

// Q1 trilinear hexahedral stiffness on N^3 nodes of the unit cube (h =
// 1/(N-1)): A_ij = h * Khat[D] * sum of kappa_e over the elements containing
// both nodes (D = number of differing coordinates; Khat = {1/3, 0, -1/12,
// -1/12}); the element sum runs over element origins (ex, ey, ez) in
// lexicographic order. kappa_e = exp(N(0,1) draw of derive(seed, e)) when
// lognormal, else 1. dirichlet: boundary rows become identity rows and
// couplings to boundary nodes are explicit zeros (27-point pattern kept).
int orc_gen_q1_hex(int64_t N, int lognormal, uint64_t seed, int dirichlet, int64_t* n_out,
                   int64_t* nnz_out, int64_t* rp, int32_t* ci, double* v) {
  if (N < 2) return 1;
  const int64_t n = N * N * N, E = N - 1;
  *n_out = n;
  *nnz_out = (3 * N - 2) * (3 * N - 2) * (3 * N - 2);
  if (!rp) return 0;
  std::vector<double> kap;
  if (lognormal) {
    kap.resize(size_t(E * E * E));
    std::vector<double> g(size_t(E * E * E));
    orc_gaussian_vector(seed, E * E * E, g.data());
    for (size_t e = 0; e < g.size(); ++e) kap[e] = std::exp(g[e]);
  }
  const Grid3 G{N};
  const double h = 1.0 / double(N - 1);
  const double Khat[4] = {1.0 / 3.0, 0.0, -1.0 / 12.0, -1.0 / 12.0};
  auto nb = [&](int64_t c) { return (c > 0 ? 1 : 0) + 1 + (c + 1 < N ? 1 : 0); };
  rp[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    int64_t x, y, z;
    G.xyz(r, x, y, z);
    rp[r + 1] = rp[r] + nb(x) * nb(y) * nb(z);
  }
  auto on_bnd = [&](int64_t x, int64_t y, int64_t z) {
    return std::min({x, y, z}) == 0 || std::max({x, y, z}) == N - 1;
  };
  // element origins along one axis shared by nodes p and q (|p - q| <= 1)
  auto origins = [&](int64_t p, int64_t q, int64_t& lo, int64_t& hi) {
    if (p != q) {
      lo = hi = std::min(p, q);
    } else {
      lo = std::max<int64_t>(p - 1, 0);
      hi = std::min<int64_t>(p, E - 1);
    }
  };
  rows_parallel(n, [&](int64_t a0, int64_t a1) {
    for (int64_t r = a0; r < a1; ++r) {
      int64_t x, y, z;
      G.xyz(r, x, y, z);
      const bool brow = dirichlet && on_bnd(x, y, z);
      int64_t k = rp[r];
      for (int64_t X = std::max<int64_t>(x - 1, 0); X <= std::min(x + 1, N - 1); ++X)
        for (int64_t Y = std::max<int64_t>(y - 1, 0); Y <= std::min(y + 1, N - 1); ++Y)
          for (int64_t Z = std::max<int64_t>(z - 1, 0); Z <= std::min(z + 1, N - 1); ++Z) {
            const int64_t c = G.id(X, Y, Z);
            double val;
            if (dirichlet && (brow || on_bnd(X, Y, Z))) {
              val = c == r ? 1.0 : 0.0;
            } else {
              int64_t xl, xh, yl, yh, zl, zh;
              origins(x, X, xl, xh);
              origins(y, Y, yl, yh);
              origins(z, Z, zl, zh);
              double acc = 0.0;
              for (int64_t ex = xl; ex <= xh; ++ex)
                for (int64_t ey = yl; ey <= yh; ++ey)
                  for (int64_t ez = zl; ez <= zh; ++ez)
                    acc += lognormal ? kap[size_t((ex * E + ey) * E + ez)] : 1.0;
              const int D = int(X != x) + int(Y != y) + int(Z != z);
              val = h * Khat[D] * acc;
            }
            ci[k] = int32_t(c);
            v[k++] = val;
          }
    }
  });
  return 0;
}

// 3D convection-diffusion -eps Lap u + w . grad u on N^3 interior nodes (h =
// 1/(N+1), Dirichlet eliminated): central diffusion eps/h^2, first-order
// upwind convection; eps from the mesh Peclet number max|w_a| h / (2 eps).
// Row: lower neighbour along axis a: -eps/h^2 - max(w_a, 0)/h; upper: -eps/h^2
// + min(w_a, 0)/h; diagonal 6 eps/h^2 + |w_x|/h + |w_y|/h + |w_z|/h (added in
// that order).
int orc_gen_convdiff_upwind(int64_t N, double peclet, double wx, double wy, double wz,
                            int64_t* n_out, int64_t* nnz_out, int64_t* rp, int32_t* ci,
                            double* v) {
  if (N < 1 || !(peclet > 0.0)) return 1;
  const int64_t n = N * N * N;
  *n_out = n;
  *nnz_out = 7 * n - 6 * N * N;
  if (!rp) return 0;
  const double h = 1.0 / double(N + 1);
  const double w[3] = {wx, wy, wz};
  const double wmax = std::max(std::fabs(wx), std::max(std::fabs(wy), std::fabs(wz)));
  const double eps = wmax * h / (2.0 * peclet);
  const double dif = eps / (h * h);
  double diag = 6.0 * dif;
  for (int a = 0; a < 3; ++a) diag += std::fabs(w[a]) / h;
  double lower[3], upper[3];
  for (int a = 0; a < 3; ++a) {
    lower[a] = -dif - (w[a] > 0 ? w[a] / h : 0.0);
    upper[a] = -dif + (w[a] < 0 ? w[a] / h : 0.0);
  }
  const int64_t stride[3] = {N * N, N, 1};
  const Grid3 G{N};
  rp[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    int64_t c[3];
    G.xyz(r, c[0], c[1], c[2]);
    int64_t cnt = 1;
    for (int a = 0; a < 3; ++a) cnt += (c[a] > 0) + (c[a] + 1 < N);
    rp[r + 1] = rp[r] + cnt;
  }
  rows_parallel(n, [&](int64_t a0, int64_t a1) {
    for (int64_t r = a0; r < a1; ++r) {
      int64_t c[3];
      G.xyz(r, c[0], c[1], c[2]);
      int64_t k = rp[r];
      for (int a = 0; a < 3; ++a)
        if (c[a] > 0) { ci[k] = int32_t(r - stride[a]); v[k++] = lower[a]; }
      ci[k] = int32_t(r);
      v[k++] = diag;
      for (int a = 2; a >= 0; --a)
        if (c[a] + 1 < N) { ci[k] = int32_t(r + stride[a]); v[k++] = upper[a]; }
    }
  });
  return 0;
}

}  // extern "C"
