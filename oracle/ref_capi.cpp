// C ABI over the REFERENCE'S OWN sources — TEST INFRASTRUCTURE ONLY.
//
// This file is the only code of ours in oracle/_ref/librkmf_ref.so: a thin
// extern "C" layer that calls the reference's public functions
//   sketch::make_sketch / sketch_apply        (sketch.hpp:28-34)
//   sparse::spmv / norm1 / validate / MTX I/O (sparse.hpp:41-66)
//   densefun::funm                            (densefun.hpp:66)
//   basis::randomized_arnoldi / arnoldi       (basis.hpp:46-60)
//   restart::restarted_krylov                 (restart.hpp:74-79)
//   approx::rand_fom                          (approximants.hpp:36)
// with the SAME signatures as the oracle's orc_* entry points
// (rkmf_oracle.cpp), so tests drive both through one Python front-end
// (oracle/ref.py) and compare them. The reference sources are compiled where
// they lie under /root/reference/proj/src, unmodified, by `make ref`
// (oracle/Makefile) against the Eigen-API stand-in in oracle/eigen_standin/
// (Eigen itself is absent from this image; see that header for what the
// stand-in does and does not pin).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <iostream>  // libstdc++ is linked statically here: this TU constructs ios_base::Init
#include <limits>
#include <string>

#include "rkmf/approximants.hpp"
#include "rkmf/basis.hpp"
#include "rkmf/densefun.hpp"
#include "rkmf/restart.hpp"
#include "rkmf/rng.hpp"
#include "rkmf/sketch.hpp"
#include "rkmf/sparse.hpp"

namespace {

using namespace rkmf;

sparse::SparseMatrix make_csr(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* ci,
                              const double* v) {
  sparse::SparseMatrix A;
  A.n_rows = n_rows;
  A.n_cols = n_cols;
  A.row_ptr.assign(rp, rp + n_rows + 1);
  const int64_t nnz = rp[n_rows];
  A.col_idx.assign(ci, ci + nnz);
  A.values.assign(v, v + nnz);
  return A;
}

sketch::SketchOperator make_op(int64_t d, int64_t n, int64_t zeta, const int64_t* rows,
                               const int8_t* signs, double scale) {
  sketch::SketchOperator S;
  S.d = d;
  S.n = n;
  S.zeta = zeta;
  S.rows.assign(rows, rows + n * zeta);
  S.signs.assign(signs, signs + n * zeta);
  S.scale = scale;
  return S;
}

Vector make_vec(const double* x, int64_t n) {
  Vector v(n);
  std::memcpy(v.data(), x, sizeof(double) * size_t(n));
  return v;
}

void put_err(char* err, const char* msg) {
  if (err) std::snprintf(err, 512, "%s", msg);
}

}  // namespace

// status codes of the oracle ABI: 1 Parameter, 2 Shape, 3 Numerical, 4 Parse
#define REF_TRY(...)                                                          \
  try { __VA_ARGS__; return 0; }                                              \
  catch (const rkmf::ParameterError& e) { put_err(err, e.what()); return 1; } \
  catch (const rkmf::ShapeError& e) { put_err(err, e.what()); return 2; }     \
  catch (const rkmf::NumericalError& e) { put_err(err, e.what()); return 3; } \
  catch (const rkmf::ParseError& e) { put_err(err, e.what()); return 4; }     \
  catch (const std::exception& e) { put_err(err, e.what()); return 5; }

extern "C" {

struct ref_cycle_record {  // layout of orc_cycle_record
  int64_t cycle, total_m, total_matvecs;
  double update_norm, error_vs_reference, kappa_W, leftmost_ritz_re, alpha_dev;
  double elapsed_ms, build_ms, funm_ms;
  double start_norm, subdiag;
};

struct ref_result {  // layout of orc_result
  int64_t converged, cycles, total_m;
  double alpha;
  int64_t matvecs, dot_n, dot_d, basis_updates, peak_basis_cols;
  int64_t n_records;
};

uint64_t ref_splitmix_derive(uint64_t seed, uint64_t tag) { return SplitMix64::derive(seed, tag); }

void ref_splitmix_stream(uint64_t seed, int64_t count, uint64_t* out) {
  SplitMix64 g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = g.next_u64();
}

void ref_gaussian_vector(uint64_t seed, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    SplitMix64 g(SplitMix64::derive(seed, uint64_t(i)));
    out[i] = g.next_gaussian(0.0, 1.0);
  }
}

// next_below / next_sign / next_unit streams, for the bit-exact pins
void ref_splitmix_below(uint64_t seed, uint64_t bound, int64_t count, uint64_t* out) {
  SplitMix64 g(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = g.next_below(bound);
}

int ref_make_sketch(int64_t d, int64_t n, int64_t zeta, uint64_t seed, int64_t* rows,
                    int8_t* signs, double* scale, char* err) {
  REF_TRY({
    const sketch::SketchOperator S = sketch::make_sketch(d, n, zeta, seed);
    for (size_t i = 0; i < S.rows.size(); ++i) {
      rows[i] = S.rows[i];
      signs[i] = S.signs[i];
    }
    *scale = S.scale;
  });
}

void ref_sketch_apply(int64_t d, int64_t n, int64_t zeta, const int64_t* rows, const int8_t* signs,
                      double scale, const double* x, double* y) {
  const sketch::SketchOperator S = make_op(d, n, zeta, rows, signs, scale);
  const Vector r = sketch::sketch_apply(S, make_vec(x, n));
  std::memcpy(y, r.data(), sizeof(double) * size_t(d));
}

void ref_spmv(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* ci,
              const double* v, const double* x, double* y, int /*threads*/) {
  const sparse::SparseMatrix A = make_csr(n_rows, n_cols, rp, ci, v);
  const Vector r = sparse::spmv(A, make_vec(x, n_cols), nullptr);
  std::memcpy(y, r.data(), sizeof(double) * size_t(n_rows));
}

double ref_norm1(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* ci,
                 const double* v) {
  return sparse::norm1(make_csr(n_rows, n_cols, rp, ci, v));
}

int ref_validate(int64_t n_rows, int64_t n_cols, const int64_t* rp, const int32_t* ci,
                 const double* v, char* err) {
  REF_TRY(sparse::validate(make_csr(n_rows, n_cols, rp, ci, v)));
}

// kind: 0 = ExpNeg (the oracle ABI's numbering); the reference has no InvSqrt
int ref_funm(int64_t n, const double* X, int kind, double t, double* F, char* err) {
  REF_TRY({
    if (kind != 0) throw ParameterError("funm: unknown FunctionSpec kind");
    Matrix M(n, n);
    std::memcpy(M.data(), X, sizeof(double) * size_t(n * n));
    const Matrix R = densefun::funm(M, densefun::FunctionSpec::exp_neg(t));
    std::memcpy(F, R.data(), sizeof(double) * size_t(n * n));
  });
}

int ref_arnoldi_decomp(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                       int64_t d, int64_t zeta, const int64_t* rows, const int8_t* signs,
                       double scale, int use_sketch, const double* b, int64_t m, double* W,
                       double* U, double* Rbar, double* start_norm, int64_t* mk,
                       int64_t* cols, int64_t* breakdown_at, int64_t* counters, char* err) {
  REF_TRY({
    const sparse::SparseMatrix A = make_csr(n, n, rp, ci, v);
    basis::KrylovDecomposition dec;
    if (use_sketch) {
      const sketch::SketchOperator S = make_op(d, n, zeta, rows, signs, scale);
      dec = basis::randomized_arnoldi(A, S, make_vec(b, n), m);
    } else {
      dec = basis::arnoldi(A, make_vec(b, n), m);
    }
    std::memcpy(W, dec.W.data(), sizeof(double) * size_t(n) * size_t(dec.W.cols()));
    if (use_sketch) std::memcpy(U, dec.U.data(), sizeof(double) * size_t(d) * size_t(dec.U.cols()));
    std::fill(Rbar, Rbar + (m + 1) * m, 0.0);
    for (Index j = 0; j < dec.Rbar.cols(); ++j)
      for (Index i = 0; i < dec.Rbar.rows(); ++i) Rbar[j * (m + 1) + i] = dec.Rbar(i, j);
    *start_norm = dec.start_norm;
    *mk = dec.m();
    *cols = dec.W.cols();
    *breakdown_at = dec.breakdown_at ? *dec.breakdown_at : 0;
    counters[0] = dec.counters.matvecs;
    counters[1] = dec.counters.dot_n;
    counters[2] = dec.counters.dot_d;
    counters[3] = dec.counters.basis_updates;
    counters[4] = dec.counters.peak_basis_cols;
  });
}

int ref_restarted_krylov(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                         const double* b, int kind, double t, int64_t m_r, double tol,
                         int64_t k_max, int64_t budget_total_m, double divergence_factor,
                         int use_sketch, int64_t d, int64_t zeta, const int64_t* rows,
                         const int8_t* signs, double scale, const double* reference,
                         int /*threads*/, double* f_out, ref_result* res, ref_cycle_record* recs,
                         int64_t rec_cap, double* R_out, int64_t R_cap, char* err) {
  REF_TRY({
    if (kind != 0) throw ParameterError("funm: unknown FunctionSpec kind");
    const sparse::SparseMatrix A = make_csr(n, n, rp, ci, v);
    sketch::SketchOperator S;
    if (use_sketch) S = make_op(d, n, zeta, rows, signs, scale);
    restart::RestartOptions opts;
    opts.m_r = m_r;
    opts.tol = tol;
    opts.k_max = k_max;
    opts.budget_total_m = budget_total_m;
    opts.divergence_factor = divergence_factor;
    Vector ref;
    if (reference) ref = make_vec(reference, n);
    const restart::RestartResult r = restart::restarted_krylov(
        A, make_vec(b, n), densefun::FunctionSpec::exp_neg(t), opts, use_sketch ? &S : nullptr,
        restart::CycleObserver{}, reference ? &ref : nullptr);
    std::memset(res, 0, sizeof(ref_result));
    std::memcpy(f_out, r.f_hat.data(), sizeof(double) * size_t(n));
    res->converged = r.converged;
    res->cycles = r.cycles;
    res->total_m = r.total_m;
    res->alpha = r.alpha;
    res->matvecs = r.counters.matvecs;
    res->dot_n = r.counters.dot_n;
    res->dot_d = r.counters.dot_d;
    res->basis_updates = r.counters.basis_updates;
    res->peak_basis_cols = r.counters.peak_basis_cols;
    for (size_t i = 0; i < r.history.size() && int64_t(i) < rec_cap; ++i) {
      const restart::CycleRecord& h = r.history[i];
      ref_cycle_record& o = recs[i];
      o.cycle = h.cycle;
      o.total_m = h.total_m;
      o.total_matvecs = h.total_matvecs;
      o.update_norm = h.update_norm;
      o.error_vs_reference = h.error_vs_reference ? *h.error_vs_reference
                                                  : std::numeric_limits<double>::quiet_NaN();
      o.kappa_W = h.kappa_W;
      o.leftmost_ritz_re = h.leftmost_ritz_re;
      o.alpha_dev = h.alpha_dev;
      o.elapsed_ms = h.elapsed_ms;
      o.build_ms = h.build_ms;
      o.funm_ms = h.funm_ms;
      // the coupling entry R_accum(M, M-1) = subdiag(k-1) * start_norm(k)
      // (restart.cpp:66) is in R_accum; the records carry no separate copy
      o.start_norm = std::numeric_limits<double>::quiet_NaN();
      o.subdiag = std::numeric_limits<double>::quiet_NaN();
      res->n_records++;
    }
    const Index M = r.R_accum.rows();
    if (R_out && R_cap >= M)
      for (Index j = 0; j < M; ++j)
        for (Index i = 0; i < M; ++i) R_out[j * M + i] = r.R_accum(i, j);
  });
}

// One randomized-Arnoldi approximant f_m = alpha W_m f(R_m) e_1 with its
// diagnostics (approximants.cpp:62-70): value [n], kappa_W, ritz (re, im) [m].
int ref_rand_fom(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, int64_t d,
                 int64_t zeta, const int64_t* rows, const int8_t* signs, double scale,
                 const double* b, int64_t m, double t, double* value, double* kappa_W,
                 double* ritz_re, double* ritz_im, char* err) {
  REF_TRY({
    const sparse::SparseMatrix A = make_csr(n, n, rp, ci, v);
    const sketch::SketchOperator S = make_op(d, n, zeta, rows, signs, scale);
    const basis::KrylovDecomposition dec = basis::randomized_arnoldi(A, S, make_vec(b, n), m);
    const approx::Approximant ap = approx::rand_fom(dec, densefun::FunctionSpec::exp_neg(t));
    std::memcpy(value, ap.value.data(), sizeof(double) * size_t(n));
    *kappa_W = ap.diag.kappa_W;
    for (size_t i = 0; i < ap.diag.ritz.size(); ++i) {
      ritz_re[i] = ap.diag.ritz[i].real();
      ritz_im[i] = ap.diag.ritz[i].imag();
    }
  });
}

// Matrix Market / vector files through the reference's reader and writer
// (sparse.cpp:140-242). load: call with null arrays for the sizes first.
int ref_load_mtx(const char* path, int64_t* n_rows, int64_t* n_cols, int64_t* nnz, int64_t* rp,
                 int32_t* ci, double* v, char* err) {
  REF_TRY({
    const sparse::SparseMatrix A = sparse::load_matrix_market(path);
    *n_rows = A.n_rows;
    *n_cols = A.n_cols;
    *nnz = A.nnz();
    if (rp) {
      for (size_t i = 0; i < A.row_ptr.size(); ++i) rp[i] = A.row_ptr[i];
      for (size_t i = 0; i < A.col_idx.size(); ++i) ci[i] = int32_t(A.col_idx[i]);
      for (size_t i = 0; i < A.values.size(); ++i) v[i] = A.values[i];
    }
  });
}

int ref_save_mtx(const char* path, int64_t n_rows, int64_t n_cols, const int64_t* rp,
                 const int32_t* ci, const double* v, char* err) {
  REF_TRY(sparse::save_matrix_market(make_csr(n_rows, n_cols, rp, ci, v), path));
}

int ref_load_vector(const char* path, int64_t* n, double* out, int64_t cap, char* err) {
  REF_TRY({
    const Vector x = sparse::load_vector(path);
    *n = x.size();
    if (out && cap >= x.size()) std::memcpy(out, x.data(), sizeof(double) * size_t(x.size()));
  });
}

int ref_save_vector(const char* path, const double* x, int64_t n, char* err) {
  REF_TRY(sparse::save_vector(make_vec(x, n), path));
}

// restart::convergence_sweep (restart.cpp:124-305) on an external-kind
// problem {L, b, f = ExpNeg(t)} (problems.hpp:32-39; no generator needed).
// The two structs have the layout of the product ABI's rkmf_method_spec /
// rkmf_sweep_record (include/rkmf_b200.h), so one ctypes definition serves both.
struct ref_method_spec {
  char name[32];
  int64_t m, d, zeta;
  double tol;
  int64_t k_max;
  uint64_t seed;
};
struct ref_sweep_record {
  char method[32];
  int64_t n, m_or_totalm, cycle, matvecs;
  double rel_error, update_norm, kappa_W, leftmost_ritz_re, elapsed_ms;
  char note[256];
  double phase_build_ms, phase_eval_ms;
};

int ref_convergence_sweep(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                          const double* b, double t, const double* reference,
                          const ref_method_spec* methods, int64_t n_methods, int with_timing,
                          ref_sweep_record* out, int64_t cap, int64_t* n_out, char* err) {
  REF_TRY({
    problems::ProblemInstance prob;
    prob.L = make_csr(n, n, rp, ci, v);
    prob.b = make_vec(b, n);
    prob.f = densefun::FunctionSpec::exp_neg(t);
    std::vector<restart::MethodSpec> ms;
    for (int64_t i = 0; i < n_methods; ++i) {
      restart::MethodSpec m;
      m.name = methods[i].name;
      m.m = methods[i].m;
      m.d = methods[i].d;
      m.zeta = methods[i].zeta;
      m.tol = methods[i].tol;
      m.k_max = methods[i].k_max;
      m.seed = methods[i].seed;
      ms.push_back(m);
    }
    Vector ref;
    if (reference) ref = make_vec(reference, n);
    const std::vector<restart::SweepRecord> rows =
        restart::convergence_sweep(prob, ms, ref, with_timing != 0, 1);
    *n_out = int64_t(rows.size());
    for (size_t i = 0; i < rows.size() && int64_t(i) < cap; ++i) {
      const restart::SweepRecord& r = rows[i];
      ref_sweep_record& o = out[i];
      std::memset(&o, 0, sizeof(o));
      std::snprintf(o.method, sizeof(o.method), "%s", r.method.c_str());
      std::snprintf(o.note, sizeof(o.note), "%s", r.note.c_str());
      o.n = r.n;
      o.m_or_totalm = r.m_or_totalm;
      o.cycle = r.cycle;
      o.matvecs = r.matvecs;
      o.rel_error = r.rel_error;
      o.update_norm = r.update_norm;
      o.kappa_W = r.kappa_W;
      o.leftmost_ritz_re = r.leftmost_ritz_re;
      o.elapsed_ms = r.elapsed_ms;
      o.phase_build_ms = r.phase_build_ms;
      o.phase_eval_ms = r.phase_eval_ms;
    }
  });
}

}  // extern "C"
