// Synthetic inputs for the BASELINE configs (host side, deterministic).
//
// The reference generates none of the five BASELINE matrices (its
// gen_conv_diff is centred-difference with identity Dirichlet rows,
// proj/src/problems.cpp:292-377), so these are new generators. They share the
// reference's lexicographic node ordering (ix*ny + iy)*nz + iz
// (problems.cpp:30-32) and emit CSR with sorted, duplicate-free columns
// (sparse.hpp:16-24; explicit zeros are allowed). Both the device
// path and the CPU oracle consume the same arrays.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "rkmf_b200.h"

namespace {

template <class F>
void par_rows(int64_t n, F&& fn) {
  unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 65536) hw = 1;
  std::vector<std::thread> pool;
  const int64_t chunk = (n + hw - 1) / hw;
  for (unsigned t = 0; t < hw; ++t) {
    const int64_t lo = int64_t(t) * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

uint64_t sm64_next(uint64_t& s) {  // rng.hpp:21-26
  uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t sm64_derive(uint64_t seed, uint64_t tag) {  // rng.hpp:56-59
  uint64_t s = seed ^ (0xA0761D6478BD642FULL + tag * 0xE7037ED1A0B428DBULL);
  return sm64_next(s);
}
double sm64_unit(uint64_t& s) { return double(sm64_next(s) >> 11) * 0x1.0p-53; }
double gaussian_at(uint64_t seed, uint64_t i) {  // next_gaussian(0,1), rng.hpp:47-53
  uint64_t s = sm64_derive(seed, i);
  double u1 = sm64_unit(s);
  while (u1 <= 0.0) u1 = sm64_unit(s);
  const double u2 = sm64_unit(s);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

}  // namespace

extern "C" {

int rkmf_gen_gaussian(uint64_t seed, int64_t n, double* out) {
  return rkmf_gen_gaussian_range(seed, 0, n, out);
}

// entries [i0, i0 + n) of the same vector: one rank's slice of b
int rkmf_gen_gaussian_range(uint64_t seed, int64_t i0, int64_t n, double* out) {
  if (i0 < 0 || n < 0) return RKMF_PARAMETER_ERROR;
  par_rows(n, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) out[i] = gaussian_at(seed, uint64_t(i0 + i));
  });
  return RKMF_OK;
}

// dim-dimensional (2 or 3) 5/7-point Laplacian on an N^dim interior grid of the
// unit square/cube, Dirichlet boundary eliminated, scaled by h^-2 (h = 1/(N+1)).
int rkmf_gen_laplacian(int32_t dim, int64_t N, int64_t* n_out, int64_t* nnz_out, int64_t* rp,
                       int32_t* ci, double* v) {
  if ((dim != 2 && dim != 3) || N < 1) return RKMF_PARAMETER_ERROR;
  const int64_t n = dim == 2 ? N * N : N * N * N;
  const int64_t nnz = dim == 2 ? 5 * N * N - 4 * N : 7 * N * N * N - 6 * N * N;
  *n_out = n;
  *nnz_out = nnz;
  if (!rp) return RKMF_OK;
  const double h = 1.0 / double(N + 1), s = 1.0 / (h * h);
  auto coords = [&](int64_t r, int64_t* c) {
    if (dim == 2) { c[0] = r / N; c[1] = r % N; c[2] = 0; }
    else { c[0] = r / (N * N); c[1] = (r / N) % N; c[2] = r % N; }
  };
  // row lengths
  std::vector<int64_t> len(static_cast<size_t>(n));
  par_rows(n, [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      int64_t c[3];
      coords(r, c);
      int64_t l = 1;
      for (int a = 0; a < dim; ++a) l += (c[a] > 0) + (c[a] < N - 1);
      len[size_t(r)] = l;
    }
  });
  rp[0] = 0;
  for (int64_t r = 0; r < n; ++r) rp[r + 1] = rp[r] + len[size_t(r)];
  const int64_t stride[3] = {dim == 2 ? N : N * N, dim == 2 ? 1 : N, 1};
  par_rows(n, [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      int64_t c[3];
      coords(r, c);
      int64_t k = rp[r];
      // neighbours in increasing column order: -x, -y, (-z), self, (+z), +y, +x
      for (int a = 0; a < dim; ++a)
        if (c[a] > 0) { ci[k] = int32_t(r - stride[a]); v[k++] = -s; }
      ci[k] = int32_t(r);
      v[k++] = 2.0 * dim * s;
      for (int a = dim - 1; a >= 0; --a)
        if (c[a] < N - 1) { ci[k] = int32_t(r + stride[a]); v[k++] = -s; }
    }
  });
  return RKMF_OK;
}

// Q1 (trilinear) hexahedral stiffness matrix on an N^3 node grid of the unit
// cube (h = 1/(N-1)): full 27-point coupling, A_ij = h * Khat(D) * sum of the
// element coefficients kappa_e over elements containing nodes i and j, where D
// is the number of differing coordinates and Khat = {1/3, 0, -1/12, -1/12} for
// D = 0..3 (the exact unit-cube element matrix K1(x)M1(x)M1 + ...). kappa_e =
// exp(g_e), g_e = N(0,1) drawn from derive(coef_seed, e) when lognormal != 0,
// else 1. With dirichlet != 0 the boundary nodes become identity rows and their
// couplings are zeroed in both directions, keeping the 27-point pattern with
// explicit zeros (nnz = (3N-2)^3 either way).
int rkmf_gen_q1_hex(int64_t N, int32_t lognormal, uint64_t coef_seed, int32_t dirichlet,
                    int64_t* n_out, int64_t* nnz_out, int64_t* rp, int32_t* ci, double* v) {
  if (N < 2) return RKMF_PARAMETER_ERROR;
  const int64_t n = N * N * N;
  const int64_t nnz = (3 * N - 2) * (3 * N - 2) * (3 * N - 2);
  *n_out = n;
  *nnz_out = nnz;
  if (!rp) return RKMF_OK;
  const int64_t E = N - 1;  // elements per dimension
  std::vector<double> kappa;
  if (lognormal) {
    kappa.resize(size_t(E * E * E));
    par_rows(E * E * E, [&](int64_t lo, int64_t hi) {
      for (int64_t e = lo; e < hi; ++e) kappa[size_t(e)] = std::exp(gaussian_at(coef_seed, uint64_t(e)));
    });
  }
  const double h = 1.0 / double(N - 1);
  const double khat[4] = {1.0 / 3.0, 0.0, -1.0 / 12.0, -1.0 / 12.0};
  auto span = [&](int64_t x) { return int64_t(x > 0) + 1 + int64_t(x < N - 1); };
  rp[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t x = r / (N * N), y = (r / N) % N, z = r % N;
    rp[r + 1] = rp[r] + span(x) * span(y) * span(z);
  }
  auto bnd = [&](int64_t x, int64_t y, int64_t z) {
    return x == 0 || y == 0 || z == 0 || x == N - 1 || y == N - 1 || z == N - 1;
  };
  par_rows(n, [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      const int64_t x = r / (N * N), y = (r / N) % N, z = r % N;
      const bool rb = dirichlet && bnd(x, y, z);
      int64_t k = rp[r];
      for (int dx = -1; dx <= 1; ++dx) {
        const int64_t X = x + dx;
        if (X < 0 || X >= N) continue;
        for (int dy = -1; dy <= 1; ++dy) {
          const int64_t Y = y + dy;
          if (Y < 0 || Y >= N) continue;
          for (int dz = -1; dz <= 1; ++dz) {
            const int64_t Z = z + dz;
            if (Z < 0 || Z >= N) continue;
            const int64_t c = (X * N + Y) * N + Z;
            double val;
            if (dirichlet && (rb || bnd(X, Y, Z))) {
              val = (c == r) ? 1.0 : 0.0;
            } else {
              const int D = (dx != 0) + (dy != 0) + (dz != 0);
              // element origins shared by both nodes, per dimension
              double ksum = 0.0;
              const int64_t ox0 = dx ? std::min(x, X) : x - 1, ox1 = dx ? std::min(x, X) : x;
              const int64_t oy0 = dy ? std::min(y, Y) : y - 1, oy1 = dy ? std::min(y, Y) : y;
              const int64_t oz0 = dz ? std::min(z, Z) : z - 1, oz1 = dz ? std::min(z, Z) : z;
              for (int64_t ox = std::max<int64_t>(0, ox0); ox <= std::min(E - 1, ox1); ++ox)
                for (int64_t oy = std::max<int64_t>(0, oy0); oy <= std::min(E - 1, oy1); ++oy)
                  for (int64_t oz = std::max<int64_t>(0, oz0); oz <= std::min(E - 1, oz1); ++oz)
                    ksum += lognormal ? kappa[size_t((ox * E + oy) * E + oz)] : 1.0;
              val = h * khat[D] * ksum;
            }
            ci[k] = int32_t(c);
            v[k++] = val;
          }
        }
      }
    }
  });
  return RKMF_OK;
}

// Non-symmetric 3D convection-diffusion -eps Lap u + v . grad u on an N^3
// interior grid (h = 1/(N+1), Dirichlet eliminated): central differences for
// diffusion, first-order upwind for convection. Mesh Peclet number
// Pe_h = max|v_i| h / (2 eps) fixes eps. 7-point, M-matrix.
int rkmf_gen_convdiff_upwind(int64_t N, double peclet, double vx, double vy, double vz,
                             int64_t* n_out, int64_t* nnz_out, int64_t* rp, int32_t* ci,
                             double* v) {
  if (N < 1 || !(peclet > 0.0)) return RKMF_PARAMETER_ERROR;
  const int64_t n = N * N * N;
  const int64_t nnz = 7 * N * N * N - 6 * N * N;
  *n_out = n;
  *nnz_out = nnz;
  if (!rp) return RKMF_OK;
  const double h = 1.0 / double(N + 1);
  const double vel[3] = {vx, vy, vz};
  const double vmax = std::max({std::fabs(vx), std::fabs(vy), std::fabs(vz)});
  const double eps = vmax * h / (2.0 * peclet);
  const double dif = eps / (h * h);
  const int64_t stride[3] = {N * N, N, 1};
  rp[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t c[3] = {r / (N * N), (r / N) % N, r % N};
    int64_t l = 1;
    for (int a = 0; a < 3; ++a) l += (c[a] > 0) + (c[a] < N - 1);
    rp[r + 1] = rp[r] + l;
  }
  par_rows(n, [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      const int64_t c[3] = {r / (N * N), (r / N) % N, r % N};
      int64_t k = rp[r];
      double diag = 6.0 * dif;
      for (int a = 0; a < 3; ++a) diag += std::fabs(vel[a]) / h;
      for (int a = 0; a < 3; ++a)  // lower neighbours: -x, -y, -z
        if (c[a] > 0) {
          ci[k] = int32_t(r - stride[a]);
          v[k++] = -dif - (vel[a] > 0 ? vel[a] / h : 0.0);
        }
      ci[k] = int32_t(r);
      v[k++] = diag;
      for (int a = 2; a >= 0; --a)  // upper neighbours: +z, +y, +x
        if (c[a] < N - 1) {
          ci[k] = int32_t(r + stride[a]);
          v[k++] = -dif + (vel[a] < 0 ? vel[a] / h : 0.0);
        }
    }
  });
  return RKMF_OK;
}

}  // extern "C"
