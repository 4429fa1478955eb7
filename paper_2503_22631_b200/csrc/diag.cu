// Per-cycle diagnostics of the reference's CycleRecord (restart.cpp:101,103,
// approximants.cpp:29-47): kappa_W = sigma_max / sigma_min of W_m and the
// leftmost Ritz value of R_m. Opt-in (rkmf_restart_options.diagnostics); not
// on the timed hot path.
//
// B200 split: the only n-sized work is the Gram matrix G = W_m^T W_m, one
// pass over the m basis columns (a tall-skinny SYRK in fp64 on the CUDA cores:
// 64-row tiles of W_m staged in shared memory, each thread owning a few (i, j)
// pairs). kappa_W = sqrt(lambda_max(G) / lambda_min(G)) (cyclic Jacobi on the
// host, m x m) — the reference takes the SVD of W_m; for the sketched basis
// (kappa well below 1e6) the Gram route agrees to many digits. The Ritz values
// are the eigenvalues of the m x m upper Hessenberg R_m (Francis double-shift
// QR on the host, as Eigen::EigenSolver computes them).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "rkmf_internal.cuh"

namespace rkmf_b200 {

namespace {

constexpr int kGramThreads = 256;
constexpr int kGramRows = 64;
constexpr int kGramMaxM = 64;
constexpr int kGramPairsPerThread = (kGramMaxM * (kGramMaxM + 1) / 2 + kGramThreads - 1) / kGramThreads;

// part[block][q] = sum over the block's rows of W[r,i] W[r,j] for pair q = (i, j),
// i <= j; column 0 scaled by sigma. gram_finish_kernel sums the blocks in
// block order (no floating-point atomics: kappa_W is bitwise reproducible,
// acceptance.cpp:545-582)
__global__ void __launch_bounds__(kGramThreads)
    gram_kernel(int64_t n, int m, int64_t ldw, const double* __restrict__ W, const SolveState* st,
                double* part) {
  __shared__ double tile[kGramRows][kGramMaxM + 1];
  __shared__ short pi[kGramMaxM * (kGramMaxM + 1) / 2], pj[kGramMaxM * (kGramMaxM + 1) / 2];
  const int P = m * (m + 1) / 2;
  const int t = threadIdx.x;
  for (int q = t; q < P; q += kGramThreads) {  // pair q -> (i, j), i <= j
    int i = 0, rem = q;
    while (rem >= m - i) { rem -= m - i; ++i; }
    pi[q] = short(i);
    pj[q] = short(i + rem);
  }
  const double sigma = st->sigma;
  double acc[kGramPairsPerThread];
#pragma unroll
  for (int a = 0; a < kGramPairsPerThread; ++a) acc[a] = 0.0;
  for (int64_t r0 = int64_t(blockIdx.x) * kGramRows; r0 < n; r0 += int64_t(gridDim.x) * kGramRows) {
    __syncthreads();
    for (int e = t; e < kGramRows * m; e += kGramThreads) {
      const int c = e / kGramRows, r = e % kGramRows;
      const int64_t row = r0 + r;
      double v = row < n ? W[int64_t(c) * ldw + row] : 0.0;
      tile[r][c] = c == 0 ? v * sigma : v;
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < kGramPairsPerThread; ++a) {
      const int q = t + a * kGramThreads;
      if (q < P) {
        const int i = pi[q], j = pj[q];
        double s = 0.0;
        for (int r = 0; r < kGramRows; ++r) s += tile[r][i] * tile[r][j];
        acc[a] += s;
      }
    }
  }
#pragma unroll
  for (int a = 0; a < kGramPairsPerThread; ++a) {
    const int q = t + a * kGramThreads;
    if (q < P) part[int64_t(blockIdx.x) * P + q] = acc[a];
  }
}

__global__ void gram_finish_kernel(int m, int nblocks, const double* __restrict__ part, double* G) {
  const int P = m * (m + 1) / 2;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < P; q += gridDim.x * blockDim.x) {
    int i = 0, rem = q;
    while (rem >= m - i) { rem -= m - i; ++i; }
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += part[int64_t(b) * P + q];
    G[i * m + i + rem] = s;
  }
}

}  // namespace

int gram_grid(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (n + kGramRows - 1) / kGramRows;
  return int(std::max<int64_t>(1, std::min<int64_t>(tiles, 4 * int64_t(sms))));
}

size_t gram_scratch_doubles(int64_t n, int m) {
  return size_t(m) * size_t(m) + size_t(gram_grid(n)) * size_t(m) * size_t(m + 1) / 2;
}

// G = the first m*m doubles of the scratch (gram_scratch_doubles), the block
// partials after them
bool launch_gram(int64_t n, int m, int64_t ldw, const double* W, const SolveState* st_dev,
                 double* G, cudaStream_t st) {
  if (m < 1 || m > kGramMaxM) return false;
  RKMF_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * size_t(m) * size_t(m), st));
  const int grid = gram_grid(n);
  double* part = G + size_t(m) * size_t(m);
  gram_kernel<<<grid, kGramThreads, 0, st>>>(n, m, ldw, W, st_dev, part);
  gram_finish_kernel<<<(m * (m + 1) / 2 + 127) / 128, 128, 0, st>>>(m, grid, part, G);
  RKMF_CUDA(cudaGetLastError());
  return true;
}

// ---- host: small dense eigenvalue problems ----

// eigenvalues of a symmetric m x m matrix (upper triangle of G, row-major),
// cyclic Jacobi
std::vector<double> sym_eigenvalues(const std::vector<double>& Gu, int m) {
  std::vector<double> a(size_t(m) * size_t(m));
  for (int i = 0; i < m; ++i)
    for (int j = i; j < m; ++j) a[size_t(i) * m + j] = a[size_t(j) * m + i] = Gu[size_t(i) * m + j];
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < m; ++i) {
      diag += a[size_t(i) * m + i] * a[size_t(i) * m + i];
      for (int j = i + 1; j < m; ++j) off += a[size_t(i) * m + j] * a[size_t(i) * m + j];
    }
    if (off <= 1e-32 * diag) break;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        const double apq = a[size_t(p) * m + q];
        if (apq == 0.0) continue;
        const double app = a[size_t(p) * m + p], aqq = a[size_t(q) * m + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(tt * tt + 1.0), s = tt * c;
        for (int k = 0; k < m; ++k) {  // columns p, q
          const double akp = a[size_t(k) * m + p], akq = a[size_t(k) * m + q];
          a[size_t(k) * m + p] = c * akp - s * akq;
          a[size_t(k) * m + q] = s * akp + c * akq;
        }
        for (int k = 0; k < m; ++k) {  // rows p, q
          const double apk = a[size_t(p) * m + k], aqk = a[size_t(q) * m + k];
          a[size_t(p) * m + k] = c * apk - s * aqk;
          a[size_t(q) * m + k] = s * apk + c * aqk;
        }
      }
  }
  std::vector<double> ev(static_cast<size_t>(m));
  for (int i = 0; i < m; ++i) ev[size_t(i)] = a[size_t(i) * m + i];
  return ev;
}

// eigenvalues (re, im) of an upper Hessenberg matrix (row-major h[i*m + j]),
// Francis double-shift QR with deflation (EISPACK hqr)
void hessenberg_eigenvalues(std::vector<double> h, int m, std::vector<double>& wr,
                            std::vector<double>& wi) {
  wr.assign(size_t(m), 0.0);
  wi.assign(size_t(m), 0.0);
  auto A = [&](int i, int j) -> double& { return h[size_t(i) * m + j]; };
  double anorm = 0.0;
  for (int i = 0; i < m; ++i)
    for (int j = std::max(i - 1, 0); j < m; ++j) anorm += std::fabs(A(i, j));
  int nn = m - 1;
  double t = 0.0;
  while (nn >= 0) {
    int its = 0, l;
    do {
      for (l = nn; l >= 1; --l) {
        const double s = std::fabs(A(l - 1, l - 1)) + std::fabs(A(l, l));
        const double ss = s == 0.0 ? anorm : s;
        if (std::fabs(A(l, l - 1)) + ss == ss) {
          A(l, l - 1) = 0.0;
          break;
        }
      }
      const double x = A(nn, nn);
      if (l == nn) {  // one root
        wr[size_t(nn)] = x + t;
        wi[size_t(nn)] = 0.0;
        --nn;
      } else {
        const double y = A(nn - 1, nn - 1), w = A(nn, nn - 1) * A(nn - 1, nn);
        if (l == nn - 1) {  // two roots
          const double p = 0.5 * (y - x), q = p * p + w, z = std::sqrt(std::fabs(q));
          const double xx = x + t;
          if (q >= 0.0) {
            const double zz = p + (p >= 0 ? z : -z);
            wr[size_t(nn - 1)] = wr[size_t(nn)] = xx + zz;
            if (zz != 0.0) wr[size_t(nn)] = xx - w / zz;
            wi[size_t(nn - 1)] = wi[size_t(nn)] = 0.0;
          } else {
            wr[size_t(nn - 1)] = wr[size_t(nn)] = xx + p;
            wi[size_t(nn - 1)] = -z;
            wi[size_t(nn)] = z;
          }
          nn -= 2;
        } else {  // no roots yet: a double-shift QR sweep
          if (its == 60) throw Error(RKMF_NUMERICAL_ERROR, "ritz: Hessenberg QR did not converge");
          double xs = x, ys = y, ws = w;
          if (its == 10 || its == 20) {  // exceptional shift
            t += x;
            for (int i = 0; i <= nn; ++i) A(i, i) -= x;
            const double s = std::fabs(A(nn, nn - 1)) + std::fabs(A(nn - 1, nn - 2));
            ys = xs = 0.75 * s;
            ws = -0.4375 * s * s;
          }
          ++its;
          int mm;
          double p = 0, q = 0, r = 0, z;
          for (mm = nn - 2; mm >= l; --mm) {
            z = A(mm, mm);
            r = xs - z;
            const double s2 = ys - z;
            p = (r * s2 - ws) / A(mm + 1, mm) + A(mm, mm + 1);
            q = A(mm + 1, mm + 1) - z - r - s2;
            r = A(mm + 2, mm + 1);
            const double s = std::fabs(p) + std::fabs(q) + std::fabs(r);
            p /= s;
            q /= s;
            r /= s;
            if (mm == l) break;
            const double u = std::fabs(A(mm, mm - 1)) * (std::fabs(q) + std::fabs(r));
            const double v = std::fabs(p) * (std::fabs(A(mm - 1, mm - 1)) + std::fabs(z) +
                                             std::fabs(A(mm + 1, mm + 1)));
            if (u + v == v) break;
          }
          for (int i = mm + 2; i <= nn; ++i) {
            A(i, i - 2) = 0.0;
            if (i != mm + 2) A(i, i - 3) = 0.0;
          }
          for (int k = mm; k <= nn - 1; ++k) {
            if (k != mm) {
              p = A(k, k - 1);
              q = A(k + 1, k - 1);
              r = 0.0;
              if (k != nn - 1) r = A(k + 2, k - 1);
              const double xx = std::fabs(p) + std::fabs(q) + std::fabs(r);
              if (xx != 0.0) {
                p /= xx;
                q /= xx;
                r /= xx;
              }
              if (xx == 0.0) continue;
              const double s = (p >= 0 ? 1.0 : -1.0) * std::sqrt(p * p + q * q + r * r);
              A(k, k - 1) = -s * xx;
              p += s;
              const double xk = p / s, yk = q / s, zk = r / s;
              q /= p;
              r /= p;
              for (int j = k; j <= nn; ++j) {
                double pp = A(k, j) + q * A(k + 1, j);
                if (k != nn - 1) {
                  pp += r * A(k + 2, j);
                  A(k + 2, j) -= pp * zk;
                }
                A(k + 1, j) -= pp * yk;
                A(k, j) -= pp * xk;
              }
              const int mmin = nn < k + 3 ? nn : k + 3;
              for (int i = l; i <= mmin; ++i) {
                double pp = xk * A(i, k) + yk * A(i, k + 1);
                if (k != nn - 1) {
                  pp += zk * A(i, k + 2);
                  A(i, k + 2) -= pp * r;
                }
                A(i, k + 1) -= pp * q;
                A(i, k) -= pp;
              }
            } else {
              const double s = (p >= 0 ? 1.0 : -1.0) * std::sqrt(p * p + q * q + r * r);
              if (s == 0.0) continue;
              if (l != mm) A(k, k - 1) = -A(k, k - 1);
              p += s;
              const double xk = p / s, yk = q / s, zk = r / s;
              q /= p;
              r /= p;
              for (int j = k; j <= nn; ++j) {
                double pp = A(k, j) + q * A(k + 1, j);
                if (k != nn - 1) {
                  pp += r * A(k + 2, j);
                  A(k + 2, j) -= pp * zk;
                }
                A(k + 1, j) -= pp * yk;
                A(k, j) -= pp * xk;
              }
              const int mmin = nn < k + 3 ? nn : k + 3;
              for (int i = l; i <= mmin; ++i) {
                double pp = xk * A(i, k) + yk * A(i, k + 1);
                if (k != nn - 1) {
                  pp += zk * A(i, k + 2);
                  A(i, k + 2) -= pp * r;
                }
                A(i, k + 1) -= pp * q;
                A(i, k) -= pp;
              }
            }
          }
        }
      }
    } while (l < nn - 1);
  }
}

// kappa_W from the (upper-triangle) Gram matrix of W_m
double kappa_from_gram(const std::vector<double>& G, int m) {
  const std::vector<double> ev = sym_eigenvalues(G, m);
  const double lmax = *std::max_element(ev.begin(), ev.end());
  const double lmin = *std::min_element(ev.begin(), ev.end());
  if (!(lmin > 0.0)) return std::numeric_limits<double>::infinity();
  return std::sqrt(lmax / lmin);
}

// all Ritz values of R_m (Rbar column-major with leading dim ldr)
void ritz_values(const std::vector<double>& Rbar, int64_t ldr, int m, std::vector<double>& wr,
                 std::vector<double>& wi) {
  std::vector<double> h(size_t(m) * size_t(m), 0.0);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i <= std::min(j + 1, m - 1); ++i)
      h[size_t(i) * m + j] = Rbar[size_t(j) * size_t(ldr) + size_t(i)];
  hessenberg_eigenvalues(h, m, wr, wi);
}

// leftmost Ritz real part of R_m
double leftmost_ritz(const std::vector<double>& Rbar, int64_t ldr, int m) {
  std::vector<double> wr, wi;
  ritz_values(Rbar, ldr, m, wr, wi);
  return *std::min_element(wr.begin(), wr.end());
}

}  // namespace rkmf_b200
