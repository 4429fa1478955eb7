// rkmf CPU oracle — TEST INFRASTRUCTURE ONLY.
//
// A plain C++17, Eigen-free restatement of the reference solver path of
// arXiv 2503.22631's artifact (`rkmf`, mounted read-only at /root/reference/proj).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// `--impl reference` legs may load this library, and only as the checker or
// the timed CPU baseline. The product (paper_2503_22631_b200) never links it.
//
// Why a restatement: the reference's own build cannot run here (Eigen3 and
// vendor/ are absent; proj/CMakeLists.txt:5,12), so every function below
// follows the cited reference file:line and replaces Eigen calls by explicit
// loops whose summation order is stated.
//
// How it is pinned: `make ref` (oracle/Makefile) compiles the reference's own
// solver-path sources, unmodified and where they lie, against an Eigen-API
// stand-in (oracle/eigen_standin) into oracle/_ref/librkmf_ref.so. Compiled
// contraction-free like that library (liboracle_strict.so), this file
// reproduces it BIT FOR BIT — sketches, decompositions (W, U, Rbar),
// restarted f(A)b with both builders (f_hat, R_accum, update norms, counters),
// funm, breakdown and saturation cases, error classes and messages
// (tests/test_ref_pin.py, live and through the frozen fixture
// tests/golden/ref_pin.npz). What stays unpinned is the rounding order of
// Eigen's own kernels (packet reductions, GEMV/GEMM blocking), which no build
// without Eigen can reproduce: against an Eigen build of the reference, parity
// is at the tolerance level, bit-exact only for the integer sketch generation.
//
// Function kinds: ExpNeg follows densefun.cpp:119-157 (Pade-13 scaling and
// squaring). InvSqrt (f(z) = z^{-1/2}) is NOT in the reference
// (FunctionSpec::Kind, densefun.hpp:20); it is added here for BASELINE cfg3
// via a determinant-scaled Denman-Beavers iteration — parity unpinned.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include <thread>

namespace orc {

// ---- errors: the reference's hierarchy (types.hpp:25-48) as status codes ----
enum Status { kOk = 0, kParameter = 1, kShape = 2, kNumerical = 3 };
struct Err : std::runtime_error {
  int code;
  Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void param(const std::string& m) { throw Err(kParameter, m); }
[[noreturn]] void shape(const std::string& m) { throw Err(kShape, m); }
[[noreturn]] void numer(const std::string& m) { throw Err(kNumerical, m); }

// Static row-block split over std::thread (libgomp is absent in this image).
// threads <= 1 runs inline, so the default oracle is single-threaded like the
// reference solve (restart.cpp is single-threaded per solve).
template <class F>
void par_for(int64_t n, int threads, F&& fn) {  // fn(lo, hi)
  if (threads <= 1 || n < 4096) { fn(int64_t(0), n); return; }
  std::vector<std::thread> pool;
  const int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = int64_t(t) * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

// ---- SplitMix64: rng.hpp:17-63 ----
struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t next_u64() {  // rng.hpp:21-26
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double next_unit() { return double(next_u64() >> 11) * 0x1.0p-53; }  // :29-31
  uint64_t next_below(uint64_t bound) {  // :34-41, unbiased rejection
    const uint64_t limit = bound * (UINT64_MAX / bound);
    uint64_t v;
    do { v = next_u64(); } while (v >= limit);
    return v % bound;
  }
  bool next_sign() { return (next_u64() & 1ULL) != 0; }  // :43
  double next_gaussian(double mean, double sd) {  // :47-53
    double u1 = next_unit();
    while (u1 <= 0.0) u1 = next_unit();
    const double u2 = next_unit();
    const double r = std::sqrt(-2.0 * std::log(u1));
    return mean + sd * r * std::cos(6.283185307179586476925286766559 * u2);
  }
  static uint64_t derive(uint64_t seed, uint64_t tag) {  // :56-59
    SplitMix64 g(seed ^ (0xA0761D6478BD642FULL + tag * 0xE7037ED1A0B428DBULL));
    return g.next_u64();
  }
};

// ---- CSR view (reference: sparse.hpp:16-24; int64 row_ptr, int32 columns) ----
struct Csr {
  int64_t n_rows, n_cols;
  const int64_t* rp;
  const int32_t* ci;
  const double* v;
  int64_t nnz() const { return rp[n_rows]; }
};

// validate: sparse.cpp:61-81
void validate(const Csr& A) {
  if (A.n_rows < 0 || A.n_cols < 0) shape("negative dimension");
  if (A.rp[0] != 0) shape("row_ptr[0] != 0");
  for (int64_t r = 0; r < A.n_rows; ++r) {
    const int64_t lo = A.rp[r], hi = A.rp[r + 1];
    if (hi < lo) shape("row_ptr not nondecreasing");
    for (int64_t k = lo; k < hi; ++k) {
      const int64_t c = A.ci[k];
      if (c < 0 || c >= A.n_cols) shape("column index out of range");
      if (k > lo && c <= A.ci[k - 1]) shape("columns not strictly increasing within a row");
      if (!std::isfinite(A.v[k])) numer("non-finite matrix entry");
    }
  }
}

// spmv: sparse.cpp:83-95 (row-sequential accumulation from 0.0)
void spmv(const Csr& A, const double* x, double* y, int threads) {
  par_for(A.n_rows, threads, [&](int64_t r0, int64_t r1) {
    for (int64_t r = r0; r < r1; ++r) {
      double acc = 0.0;
      const int64_t hi = A.rp[r + 1];
      for (int64_t k = A.rp[r]; k < hi; ++k) acc += A.v[k] * x[A.ci[k]];
      y[r] = acc;
    }
  });
}

// norm1 = max column abs-sum: sparse.cpp:97-102
double norm1(const Csr& A) {
  std::vector<double> cs(static_cast<size_t>(A.n_cols), 0.0);
  const int64_t nz = A.nnz();
  for (int64_t k = 0; k < nz; ++k) cs[size_t(A.ci[k])] += std::fabs(A.v[k]);
  double m = 0.0;
  for (double c : cs) m = std::max(m, c);
  return A.n_cols == 0 ? 0.0 : m;
}

// ---- sketch: sketch.hpp:16-24 ----
struct Sketch {
  int64_t d, n, zeta;
  const int64_t* rows;
  const int8_t* signs;
  double scale;
};

// make_sketch: sketch.cpp:13-49 (per-column derived stream, Floyd sampling,
// ascending sort, signs drawn in sorted order). Bit-exact definition of S.
void make_sketch(int64_t d, int64_t n, int64_t zeta, uint64_t seed, int64_t* rows,
                 int8_t* signs, double* scale) {
  if (zeta < 1) param("sketch: zeta must be >= 1");
  if (zeta > d) param("sketch: zeta must not exceed d");
  if (d > n) param("sketch: d must not exceed n");
  *scale = 1.0 / std::sqrt(double(zeta));
  std::vector<int64_t> chosen;
  chosen.reserve(size_t(zeta));
  for (int64_t j = 0; j < n; ++j) {
    SplitMix64 gen(SplitMix64::derive(seed, uint64_t(j)));
    chosen.clear();
    for (int64_t i = d - zeta; i < d; ++i) {
      const int64_t t = int64_t(gen.next_below(uint64_t(i) + 1));
      if (std::find(chosen.begin(), chosen.end(), t) == chosen.end())
        chosen.push_back(t);
      else
        chosen.push_back(i);
    }
    std::sort(chosen.begin(), chosen.end());
    const size_t base = size_t(j) * size_t(zeta);
    for (int64_t k = 0; k < zeta; ++k) {
      rows[base + size_t(k)] = chosen[size_t(k)];
      signs[base + size_t(k)] = gen.next_sign() ? 1 : -1;
    }
  }
}

// sketch_apply (vector): sketch.cpp:51-63 (column order, zero entries skipped)
void sketch_apply_range(const Sketch& S, const double* x, double* y, int64_t j0, int64_t j1) {
  const size_t z = size_t(S.zeta);
  for (int64_t j = j0; j < j1; ++j) {
    const double xj = S.scale * x[j];
    if (xj == 0.0) continue;
    const size_t base = size_t(j) * z;
    for (size_t k = 0; k < z; ++k) y[S.rows[base + k]] += S.signs[base + k] > 0 ? xj : -xj;
  }
}

// threads <= 1: the reference's column-sequential order exactly. threads > 1
// (the CPU baseline only): contiguous column ranges into per-thread partial
// sketches, summed in range order (deterministic; rounding differs from the
// sequential order at the 1e-16 level).
void sketch_apply(const Sketch& S, const double* x, double* y, int threads = 1) {
  std::fill(y, y + S.d, 0.0);
  if (threads <= 1 || S.n < 65536) {
    sketch_apply_range(S, x, y, 0, S.n);
    return;
  }
  std::vector<std::vector<double>> part(size_t(threads), std::vector<double>(size_t(S.d), 0.0));
  std::vector<std::thread> pool;
  const int64_t chunk = (S.n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = std::min<int64_t>(S.n, int64_t(t) * chunk);
    const int64_t hi = std::min<int64_t>(S.n, lo + chunk);
    pool.emplace_back([&, t, lo, hi] { sketch_apply_range(S, x, part[size_t(t)].data(), lo, hi); });
  }
  for (auto& th : pool) th.join();
  for (int t = 0; t < threads; ++t)
    for (int64_t i = 0; i < S.d; ++i) y[i] += part[size_t(t)][size_t(i)];
}

// ---- small dense helpers (column-major), replacing Eigen ----
struct Mat {
  int64_t r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int64_t rr, int64_t cc) : r(rr), c(cc), a(size_t(rr * cc), 0.0) {}
  double& operator()(int64_t i, int64_t j) { return a[size_t(j * r + i)]; }
  double operator()(int64_t i, int64_t j) const { return a[size_t(j * r + i)]; }
  static Mat eye(int64_t n) { Mat m(n, n); for (int64_t i = 0; i < n; ++i) m(i, i) = 1.0; return m; }
};

Mat gemm(const Mat& A, const Mat& B) {  // C = A*B, k-outer (column axpy) order
  Mat C(A.r, B.c);
  for (int64_t j = 0; j < B.c; ++j)
    for (int64_t k = 0; k < A.c; ++k) {
      const double b = B(k, j);
      if (b == 0.0) continue;
      const double* ak = &A.a[size_t(k * A.r)];
      double* cj = &C.a[size_t(j * C.r)];
      for (int64_t i = 0; i < A.r; ++i) cj[i] += ak[i] * b;
    }
  return C;
}
Mat lin(std::initializer_list<std::pair<double, const Mat*>> terms, int64_t n, double diag = 0.0) {
  Mat M(n, n);
  for (auto& t : terms)
    for (size_t i = 0; i < M.a.size(); ++i) M.a[i] += t.first * t.second->a[i];
  for (int64_t i = 0; i < n; ++i) M(i, i) += diag;
  return M;
}
bool all_finite(const Mat& M) {
  for (double x : M.a) if (!std::isfinite(x)) return false;
  return true;
}
double norm1(const Mat& M) {
  double m = 0.0;
  for (int64_t j = 0; j < M.c; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < M.r; ++i) s += std::fabs(M(i, j));
    m = std::max(m, s);
  }
  return m;
}

// Partial-pivot LU (replaces Eigen::PartialPivLU used at densefun.cpp:150).
struct Lu {
  Mat lu;
  std::vector<int64_t> piv;
  double logabsdet = 0.0;
  bool singular = false;
};
Lu lu_factor(Mat A) {
  const int64_t n = A.r;
  Lu f;
  f.piv.resize(size_t(n));
  for (int64_t k = 0; k < n; ++k) {
    int64_t p = k;
    double best = std::fabs(A(k, k));
    for (int64_t i = k + 1; i < n; ++i)
      if (std::fabs(A(i, k)) > best) { best = std::fabs(A(i, k)); p = i; }
    f.piv[size_t(k)] = p;
    if (p != k)
      for (int64_t j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
    const double d = A(k, k);
    if (d == 0.0) { f.singular = true; continue; }
    f.logabsdet += std::log(std::fabs(d));
    for (int64_t i = k + 1; i < n; ++i) A(i, k) /= d;
    for (int64_t j = k + 1; j < n; ++j) {
      const double akj = A(k, j);
      if (akj == 0.0) continue;
      for (int64_t i = k + 1; i < n; ++i) A(i, j) -= A(i, k) * akj;
    }
  }
  f.lu = std::move(A);
  return f;
}
Mat lu_solve(const Lu& f, Mat B) {
  const int64_t n = f.lu.r;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t p = f.piv[size_t(k)];
    if (p != k)
      for (int64_t j = 0; j < B.c; ++j) std::swap(B(k, j), B(p, j));
  }
  for (int64_t j = 0; j < B.c; ++j) {
    for (int64_t k = 0; k < n; ++k) {  // L y = b (unit diagonal)
      const double bk = B(k, j);
      for (int64_t i = k + 1; i < n; ++i) B(i, j) -= f.lu(i, k) * bk;
    }
    for (int64_t k = n - 1; k >= 0; --k) {  // U x = y
      B(k, j) /= f.lu(k, k);
      const double bk = B(k, j);
      for (int64_t i = 0; i < k; ++i) B(i, j) -= f.lu(i, k) * bk;
    }
  }
  return B;
}

constexpr double kTheta13 = 5.371920351148152;  // densefun.cpp:115

// expm: densefun.cpp:119-157 (Pade-13 scaling and squaring, Higham 2005).
Mat expm(const Mat& X) {
  if (X.r != X.c) shape("shape: expm expects a square matrix");
  if (!all_finite(X)) numer("expm: non-finite input");
  const int64_t n = X.r;
  if (n == 0) return Mat(0, 0);
  const double nrm = norm1(X);
  if (nrm == 0.0) return Mat::eye(n);
  int s = 0;
  if (nrm > kTheta13) s = std::min(int(std::ceil(std::log2(nrm / kTheta13))), 64);
  Mat A = X;
  const double sc = std::ldexp(1.0, -s);
  for (double& x : A.a) x *= sc;
  static const double b[14] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                               1187353796428800.0,  129060195264000.0,   10559470521600.0,
                               670442572800.0,      33522128640.0,       1323241920.0,
                               40840800.0,          960960.0,            16380.0,
                               182.0,               1.0};
  const Mat A2 = gemm(A, A), A4 = gemm(A2, A2), A6 = gemm(A2, A4);
  const Mat t1 = lin({{b[13], &A6}, {b[11], &A4}, {b[9], &A2}}, n);
  Mat in_u = gemm(A6, t1);
  in_u = lin({{1.0, &in_u}, {b[7], &A6}, {b[5], &A4}, {b[3], &A2}}, n, b[1]);
  const Mat U = gemm(A, in_u);
  const Mat t2 = lin({{b[12], &A6}, {b[10], &A4}, {b[8], &A2}}, n);
  Mat V = gemm(A6, t2);
  V = lin({{1.0, &V}, {b[6], &A6}, {b[4], &A4}, {b[2], &A2}}, n, b[0]);
  const Mat VmU = lin({{1.0, &V}, {-1.0, &U}}, n), VpU = lin({{1.0, &V}, {1.0, &U}}, n);
  Mat F = lu_solve(lu_factor(VmU), VpU);
  for (int i = 0; i < s; ++i) {
    F = gemm(F, F);
    if (!all_finite(F)) numer("expm: function overflow");
  }
  if (!all_finite(F)) numer("expm: function overflow");
  return F;
}

// X^{-1/2} by the Denman-Beavers iteration with determinant scaling
// (Higham, Functions of Matrices, Alg. 6.x). NOT in the reference.
Mat inv_sqrtm(const Mat& X) {
  const int64_t n = X.r;
  if (n == 0) return Mat(0, 0);
  Mat Y = X, Z = Mat::eye(n);
  bool scale = true;
  for (int it = 0; it < 100; ++it) {
    const Lu fy = lu_factor(Y), fz = lu_factor(Z);
    if (fy.singular || fz.singular) numer("invsqrt: singular iterate");
    const Mat Yi = lu_solve(fy, Mat::eye(n)), Zi = lu_solve(fz, Mat::eye(n));
    double g = 1.0;
    if (scale) g = std::exp(-(fy.logabsdet + fz.logabsdet) / (2.0 * double(n)));
    Mat Yn = lin({{0.5 * g, &Y}, {0.5 / g, &Zi}}, n);
    Mat Zn = lin({{0.5 * g, &Z}, {0.5 / g, &Yi}}, n);
    Mat dY = lin({{1.0, &Yn}, {-1.0, &Y}}, n);
    const double rel = norm1(dY) / std::max(norm1(Yn), 1e-300);
    Y = std::move(Yn);
    Z = std::move(Zn);
    if (rel < 1e-2) scale = false;
    if (rel < 1e-15 * double(n)) break;
  }
  if (!all_finite(Z)) numer("invsqrt: function overflow");
  return Z;
}

enum Kind { kExpNeg = 0, kInvSqrt = 4 };

// funm dispatch: densefun.cpp:429-450 (ExpNeg → expm(-t X)); InvSqrt added.
Mat funm(const Mat& X, int kind, double t) {
  if (X.r != X.c) shape("shape: funm expects a square matrix");
  Mat F;
  if (kind == kExpNeg) {
    Mat Y = X;
    for (double& x : Y.a) x *= -t;
    F = expm(Y);
  } else if (kind == kInvSqrt) {
    F = inv_sqrtm(X);
  } else {
    param("funm: unknown FunctionSpec kind");
  }
  if (!all_finite(F)) numer("funm: function overflow");
  return F;
}

// ---- Krylov decompositions: basis.hpp:22-41, basis.cpp ----
struct Counters {  // types.hpp:57-75
  long long matvecs = 0, dot_n = 0, dot_d = 0, basis_updates = 0, peak_basis_cols = 0;
  void note(long long c) { peak_basis_cols = std::max(peak_basis_cols, c); }
  void add(const Counters& o) {
    matvecs += o.matvecs; dot_n += o.dot_n; dot_d += o.dot_d; basis_updates += o.basis_updates;
    note(o.peak_basis_cols);
  }
};

struct Dec {
  int64_t n = 0, m = 0, cols = 0, d = 0;  // W is n x cols (m+1, or m on breakdown)
  std::vector<double> W, U;               // col-major, capacity m+1 columns
  Mat Rbar;                               // (m+1) x m, or m x m on breakdown
  double start_norm = 0.0;
  int64_t breakdown_at = 0;               // 0 = none
  Counters ctr;
  double subdiag() const { return cols == m + 1 ? Rbar(m, m - 1) : 0.0; }
};

constexpr double kBreakdownFactor = 1e-14;  // basis.cpp:12

void check_start(const Csr& A, int64_t blen, int64_t m) {  // basis.cpp:14-23
  validate(A);
  if (A.n_rows != A.n_cols) shape("arnoldi: matrix must be square");
  if (blen != A.n_rows) shape("arnoldi: start vector length mismatch");
  if (m < 1) param("arnoldi: m must be >= 1");
  if (m > A.n_rows) param("arnoldi: m exceeds matrix dimension");
}

void shrink(Dec& dec, int64_t kept) {  // basis.cpp:25-31
  dec.cols = kept;
  Mat sq(kept, kept);
  for (int64_t j = 0; j < kept; ++j)
    for (int64_t i = 0; i < kept; ++i) sq(i, j) = dec.Rbar(i, j);
  dec.Rbar = std::move(sq);
  dec.m = kept;
  dec.breakdown_at = kept;
}

double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

// w = (z - Wk r) / rkk with Wk = first kc columns of W (Eigen GEMV at basis.cpp:135;
// here: per row, column-ordered accumulation, then subtract and divide).
void basis_update(const double* W, int64_t n, int64_t kc, const double* r, const double* z,
                  double rkk, double* out, int threads) {
  const int64_t B = 512;
  par_for((n + B - 1) / B, threads, [&](int64_t b0, int64_t b1) {
    double acc[512];
    for (int64_t blk = b0; blk < b1; ++blk) {
      const int64_t i0 = blk * B, i1 = std::min(n, i0 + B);
      for (int64_t i = i0; i < i1; ++i) acc[i - i0] = 0.0;
      for (int64_t c = 0; c < kc; ++c) {
        const double rc = r[c];
        const double* w = W + size_t(c) * size_t(n);
        for (int64_t i = i0; i < i1; ++i) acc[i - i0] += w[i] * rc;
      }
      for (int64_t i = i0; i < i1; ++i) out[i] = (z[i] - acc[i - i0]) / rkk;
    }
  });
}

// randomized_arnoldi: basis.cpp:92-142
Dec randomized_arnoldi(const Csr& A, const Sketch& S, const double* b, int64_t m, int threads,
                       bool do_validate = true) {
  if (do_validate) check_start(A, A.n_rows, m);
  const int64_t n = A.n_rows;
  if (S.n != n) shape("randomized_arnoldi: sketch width mismatch");
  const int64_t need = (m == n) ? m : m + 1;
  if (S.d < need) param("randomized_arnoldi: sketch dimension d too small for m");
  const int64_t d = S.d;
  std::vector<double> sb(static_cast<size_t>(d));
  sketch_apply(S, b, sb.data(), threads);
  const double alpha = std::sqrt(dot(sb.data(), sb.data(), d));
  if (alpha == 0.0) param("randomized_arnoldi: zero start vector after sketching");

  Dec dec;
  dec.n = n; dec.m = m; dec.cols = m + 1; dec.d = d;
  dec.start_norm = alpha;
  dec.W.assign(size_t(n) * size_t(m + 1), 0.0);
  dec.U.assign(size_t(d) * size_t(m + 1), 0.0);
  dec.Rbar = Mat(m + 1, m);
  for (int64_t i = 0; i < n; ++i) dec.W[size_t(i)] = b[i] / alpha;
  for (int64_t i = 0; i < d; ++i) dec.U[size_t(i)] = sb[size_t(i)] / alpha;
  dec.ctr.note(1);

  const double tol = kBreakdownFactor * norm1(A);  // basis.cpp:118
  std::vector<double> z(static_cast<size_t>(n)), p(static_cast<size_t>(d)), r;
  for (int64_t k = 0; k < m; ++k) {
    spmv(A, dec.W.data() + size_t(k) * size_t(n), z.data(), threads);
    dec.ctr.matvecs++;
    sketch_apply(S, z.data(), p.data(), threads);
    r.assign(size_t(k + 1), 0.0);
    for (int64_t i = 0; i <= k; ++i) {  // MGS in sketch space, basis.cpp:123-128
      const double* u = dec.U.data() + size_t(i) * size_t(d);
      r[size_t(i)] = dot(u, p.data(), d);
      for (int64_t q = 0; q < d; ++q) p[size_t(q)] -= r[size_t(i)] * u[q];
    }
    dec.ctr.dot_d += k + 1;
    for (int64_t i = 0; i <= k; ++i) dec.Rbar(i, k) = r[size_t(i)];
    const double rkk = std::sqrt(dot(p.data(), p.data(), d));
    if (rkk <= tol || k + 1 == n) {
      shrink(dec, k + 1);
      return dec;
    }
    basis_update(dec.W.data(), n, k + 1, r.data(), z.data(), rkk,
                 dec.W.data() + size_t(k + 1) * size_t(n), threads);
    dec.ctr.basis_updates++;
    double* u1 = dec.U.data() + size_t(k + 1) * size_t(d);
    for (int64_t q = 0; q < d; ++q) u1[q] = p[size_t(q)] / rkk;
    dec.Rbar(k + 1, k) = rkk;
    dec.ctr.note(k + 2);
  }
  return dec;
}

// classical Arnoldi with one MGS sweep: basis.cpp:34-77 (k_trunc >= m)
Dec arnoldi(const Csr& A, const double* b, int64_t m, int threads, bool do_validate = true) {
  if (do_validate) check_start(A, A.n_rows, m);
  const int64_t n = A.n_rows;
  const double beta = std::sqrt(dot(b, b, n));
  if (beta == 0.0) param("arnoldi: zero start vector");
  Dec dec;
  dec.n = n; dec.m = m; dec.cols = m + 1;
  dec.start_norm = beta;
  dec.W.assign(size_t(n) * size_t(m + 1), 0.0);
  dec.Rbar = Mat(m + 1, m);
  for (int64_t i = 0; i < n; ++i) dec.W[size_t(i)] = b[i] / beta;
  dec.ctr.note(1);
  const double tol = kBreakdownFactor * norm1(A);
  std::vector<double> w(static_cast<size_t>(n));
  for (int64_t k = 0; k < m; ++k) {
    spmv(A, dec.W.data() + size_t(k) * size_t(n), w.data(), threads);
    dec.ctr.matvecs++;
    for (int64_t i = 0; i <= k; ++i) {
      const double* v = dec.W.data() + size_t(i) * size_t(n);
      const double h = dot(v, w.data(), n);
      dec.ctr.dot_n++;
      for (int64_t q = 0; q < n; ++q) w[size_t(q)] -= h * v[q];
      dec.Rbar(i, k) = h;
    }
    const double hnext = std::sqrt(dot(w.data(), w.data(), n));
    if (hnext <= tol || k + 1 == n) {
      shrink(dec, k + 1);
      return dec;
    }
    dec.Rbar(k + 1, k) = hnext;
    double* out = dec.W.data() + size_t(k + 1) * size_t(n);
    for (int64_t q = 0; q < n; ++q) out[q] = w[size_t(q)] / hnext;
    dec.ctr.basis_updates++;
    dec.ctr.note(k + 2);
  }
  return dec;
}

double now_ms() {  // restart.cpp:17-21
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace orc

// =========================== C ABI for tests/bench ===========================
extern "C" {

struct orc_cycle_record {  // restart.hpp:28-40 (kappa_W / ritz not computed: NaN)
  int64_t cycle, total_m, total_matvecs;
  double update_norm, error_vs_reference, kappa_W, leftmost_ritz_re, alpha_dev;
  double elapsed_ms, build_ms, funm_ms;
  double start_norm, subdiag;
};

struct orc_result {  // restart.hpp:56-65
  int64_t converged, cycles, total_m;
  double alpha;
  int64_t matvecs, dot_n, dot_d, basis_updates, peak_basis_cols;
  int64_t n_records;
};

static void put_err(char* err, const char* msg) {
  if (err) { std::snprintf(err, 512, "%s", msg); }
}

#define ORC_TRY(...)                                           \
  try { __VA_ARGS__; return 0; }                                      \
  catch (const orc::Err& e) { put_err(err, e.what()); return e.code; } \
  catch (const std::exception& e) { put_err(err, e.what()); return 5; }

uint64_t orc_splitmix_derive(uint64_t seed, uint64_t tag) { return orc::SplitMix64::derive(seed, tag); }

void orc_splitmix_stream(uint64_t seed, int64_t count, uint64_t* out) {
  orc::SplitMix64 g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = g.next_u64();
}

// b[i] = first next_gaussian(0,1) of the stream derive(seed, i) (counter-based;
// the input convention shared by the product generators and the tests).
void orc_gaussian_vector(uint64_t seed, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    orc::SplitMix64 g(orc::SplitMix64::derive(seed, uint64_t(i)));
    out[i] = g.next_gaussian(0.0, 1.0);
  }
}

int orc_make_sketch(int64_t d, int64_t n, int64_t zeta, uint64_t seed, int64_t* rows,
                    int8_t* signs, double* scale, char* err) {
  ORC_TRY(orc::make_sketch(d, n, zeta, seed, rows, signs, scale));
}

void orc_sketch_apply(int64_t d, int64_t n, int64_t zeta, const int64_t* rows, const int8_t* signs,
                      double scale, const double* x, double* y) {
  orc::Sketch S{d, n, zeta, rows, signs, scale};
  orc::sketch_apply(S, x, y);
}

void orc_spmv(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* ci,
              const double* v, const double* x, double* y, int threads) {
  orc::Csr A{n_rows, n_cols, rp, ci, v};
  orc::spmv(A, x, y, threads);
}

double orc_norm1(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* ci,
                 const double* v) {
  orc::Csr A{n_rows, n_cols, rp, ci, v};
  return orc::norm1(A);
}

int orc_validate(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* ci,
                 const double* v, char* err) {
  orc::Csr A{n_rows, n_cols, rp, ci, v};
  ORC_TRY(orc::validate(A));
}

int orc_funm(int64_t n, const double* X, int kind, double t, double* F, char* err) {
  ORC_TRY({
    orc::Mat M(n, n);
    std::memcpy(M.a.data(), X, sizeof(double) * size_t(n * n));
    orc::Mat R = orc::funm(M, kind, t);
    std::memcpy(F, R.a.data(), sizeof(double) * size_t(n * n));
  });
}

// One decomposition. W: n x (m+1), U: d x (m+1), Rbar: (m+1) x m, all col-major
// and sized for the full m; *cols / *mk report the kept sizes on breakdown.
int orc_arnoldi_decomp(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                       int64_t d, int64_t zeta, const int64_t* rows, const int8_t* signs,
                       double scale, int use_sketch, const double* b, int64_t m, double* W,
                       double* U, double* Rbar, double* start_norm, int64_t* mk,
                       int64_t* cols, int64_t* breakdown_at, int64_t* counters, char* err) {
  ORC_TRY({
    orc::Csr A{n, n, rp, ci, v};
    orc::Sketch S{d, n, zeta, rows, signs, scale};
    orc::Dec dec = use_sketch ? orc::randomized_arnoldi(A, S, b, m, 1)
                              : orc::arnoldi(A, b, m, 1);
    std::memcpy(W, dec.W.data(), sizeof(double) * size_t(n) * size_t(dec.cols));
    if (use_sketch) std::memcpy(U, dec.U.data(), sizeof(double) * size_t(d) * size_t(dec.cols));
    std::fill(Rbar, Rbar + (m + 1) * m, 0.0);
    for (int64_t j = 0; j < dec.Rbar.c; ++j)
      for (int64_t i = 0; i < dec.Rbar.r; ++i) Rbar[j * (m + 1) + i] = dec.Rbar(i, j);
    *start_norm = dec.start_norm;
    *mk = dec.m;
    *cols = dec.cols;
    *breakdown_at = dec.breakdown_at;
    counters[0] = dec.ctr.matvecs; counters[1] = dec.ctr.dot_n; counters[2] = dec.ctr.dot_d;
    counters[3] = dec.ctr.basis_updates; counters[4] = dec.ctr.peak_basis_cols;
  });
}

// restarted_krylov: restart.cpp:27-122. use_sketch=0 selects the classical
// builder (S == nullptr in the reference). R_out (optional) receives R_accum
// (total_m x total_m col-major) when its capacity R_cap >= total_m.
int orc_restarted_krylov(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                         const double* b, int kind, double t, int64_t m_r, double tol,
                         int64_t k_max, int64_t budget_total_m, double divergence_factor,
                         int use_sketch, int64_t d, int64_t zeta, const int64_t* rows,
                         const int8_t* signs, double scale, const double* reference,
                         int threads, double* f_out, orc_result* res, orc_cycle_record* recs,
                         int64_t rec_cap, double* R_out, int64_t R_cap, char* err) {
  ORC_TRY({
    using namespace orc;
    if (m_r < 1) param("restart: m_r must be >= 1");
    if (k_max < 1) param("restart: k_max must be >= 1");
    if (!(tol > 0.0)) param("restart: tol must be > 0");
    if (budget_total_m < m_r) param("restart: total-m budget below one cycle");
    if (kind != kExpNeg && kind != kInvSqrt) param("funm: unknown FunctionSpec kind");
    Csr A{n, n, rp, ci, v};
    Sketch S{d, n, zeta, rows, signs, scale};
    const int64_t m_eff = std::min(m_r, n);
    std::memset(res, 0, sizeof(orc_result));
    std::fill(f_out, f_out + n, 0.0);
    std::vector<double> start(b, b + n), y(static_cast<size_t>(n));
    Mat Racc;
    int64_t M = 0;
    double coupling = 0.0, first_update = -1.0;
    Counters total;
    double ref_norm = 0.0;
    if (reference) ref_norm = std::sqrt(dot(reference, reference, n));
    for (int64_t k = 1; k <= k_max; ++k) {
      if (M + m_eff > budget_total_m) break;
      const double t0 = now_ms();
      Dec dec = use_sketch ? randomized_arnoldi(A, S, start.data(), m_eff, threads)
                           : arnoldi(A, start.data(), m_eff, threads);
      const double t_built = now_ms();
      const int64_t mk = dec.m;
      if (k == 1) res->alpha = dec.start_norm;
      total.add(dec.ctr);
      Mat grown(M + mk, M + mk);  // restart.cpp:61-70
      for (int64_t j = 0; j < M; ++j)
        for (int64_t i = 0; i < M; ++i) grown(i, j) = Racc(i, j);
      if (M > 0) grown(M, M - 1) = coupling * dec.start_norm;
      for (int64_t j = 0; j < mk; ++j)
        for (int64_t i = 0; i < mk; ++i) grown(M + i, M + j) = dec.Rbar(i, j);
      Racc = std::move(grown);
      Mat F;
      try {
        F = funm(Racc, kind, t);
      } catch (const Err& e) {
        numer(std::string("restart: function evaluation failed (cycle ") + std::to_string(k) +
              "): " + e.what());
      }
      const double t_funm = now_ms();
      // y = alpha * (W[:, :mk] * F[M:M+mk, 0]) (restart.cpp:80-81)
      std::vector<double> g(static_cast<size_t>(mk));
      for (int64_t j = 0; j < mk; ++j) g[size_t(j)] = F(M + j, 0);
      {
        const int64_t B = 512;
        par_for((n + B - 1) / B, threads, [&](int64_t b0, int64_t b1) {
          double acc[512];
          for (int64_t blk = b0; blk < b1; ++blk) {
            const int64_t i0 = blk * B, i1 = std::min(n, i0 + B);
            for (int64_t i = i0; i < i1; ++i) acc[i - i0] = 0.0;
            for (int64_t c = 0; c < mk; ++c) {
              const double* w = dec.W.data() + size_t(c) * size_t(n);
              const double gc = g[size_t(c)];
              for (int64_t i = i0; i < i1; ++i) acc[i - i0] += w[i] * gc;
            }
            for (int64_t i = i0; i < i1; ++i) y[size_t(i)] = res->alpha * acc[i - i0];
          }
        });
      }
      bool finite = true;
      for (double q : y) if (!std::isfinite(q)) { finite = false; break; }
      if (!finite) numer("restart divergence (cycle " + std::to_string(k) + ")");
      double yn2 = 0.0;
      for (int64_t i = 0; i < n; ++i) { f_out[i] += y[size_t(i)]; yn2 += y[size_t(i)] * y[size_t(i)]; }
      const double yn = std::sqrt(yn2);
      if (first_update < 0.0)
        first_update = yn;
      else if (yn > divergence_factor * first_update)
        numer("restart divergence (cycle " + std::to_string(k) + ")");
      if (res->n_records < rec_cap) {
        orc_cycle_record& rec = recs[res->n_records];
        rec.cycle = k;
        rec.total_m = M + mk;
        rec.total_matvecs = total.matvecs;
        rec.update_norm = yn;
        rec.error_vs_reference = std::numeric_limits<double>::quiet_NaN();
        if (reference && ref_norm > 0.0) {
          double e2 = 0.0;
          for (int64_t i = 0; i < n; ++i) { const double q = f_out[i] - reference[i]; e2 += q * q; }
          rec.error_vs_reference = std::sqrt(e2) / ref_norm;
        }
        rec.kappa_W = std::numeric_limits<double>::quiet_NaN();
        rec.leftmost_ritz_re = std::numeric_limits<double>::quiet_NaN();
        rec.alpha_dev = (k == 1) ? 0.0 : std::fabs(dec.start_norm - 1.0);
        rec.elapsed_ms = now_ms() - t0;
        rec.build_ms = t_built - t0;
        rec.funm_ms = t_funm - t_built;
        rec.start_norm = dec.start_norm;
        rec.subdiag = dec.subdiag();
        res->n_records++;
      }
      M += mk;
      res->cycles = k;
      res->total_m = M;
      if (yn <= tol || dec.breakdown_at) { res->converged = 1; break; }
      coupling = dec.subdiag();
      std::memcpy(start.data(), dec.W.data() + size_t(mk) * size_t(n), sizeof(double) * size_t(n));
    }
    res->matvecs = total.matvecs; res->dot_n = total.dot_n; res->dot_d = total.dot_d;
    res->basis_updates = total.basis_updates; res->peak_basis_cols = total.peak_basis_cols;
    if (R_out && R_cap >= M)
      for (int64_t j = 0; j < M; ++j)
        for (int64_t i = 0; i < M; ++i) R_out[j * M + i] = Racc(i, j);
  });
}

}  // extern "C"
