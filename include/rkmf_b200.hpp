// rkmf_b200.hpp — header-only C++ mirror of the reference solver interface
// (proj/include/rkmf/restart.hpp, sketch.hpp, sparse.hpp, densefun.hpp,
// types.hpp) over the C ABI in rkmf_b200.h. Eigen-free: vectors are
// std::vector<double>. Errors are rethrown as the reference's exception types
// with the same message text (types.hpp:25-48).
#ifndef RKMF_B200_HPP
#define RKMF_B200_HPP

#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rkmf_b200.h"

namespace rkmf_b200 {

// ---- types.hpp:25-48 ----
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class ShapeError : public Error {
 public:
  explicit ShapeError(const std::string& m) : Error(m) {}
};
class ParameterError : public Error {
 public:
  explicit ParameterError(const std::string& m) : Error(m) {}
};
class NumericalError : public Error {
 public:
  explicit NumericalError(const std::string& m) : Error(m) {}
};
class DeviceError : public Error {
 public:
  explicit DeviceError(const std::string& m) : Error(m) {}
};
class ParseError : public Error {
 public:
  explicit ParseError(const std::string& m) : Error(m) {}
};

inline void check(rkmf_context* ctx, int code) {
  if (code == RKMF_OK) return;
  const std::string msg = ctx ? rkmf_last_error(ctx) : "rkmf_b200 error";
  switch (code) {
    case RKMF_PARAMETER_ERROR: throw ParameterError(msg);
    case RKMF_SHAPE_ERROR: throw ShapeError(msg);
    case RKMF_NUMERICAL_ERROR: throw NumericalError(msg);
    case RKMF_DEVICE_ERROR: throw DeviceError(msg);
    case RKMF_PARSE_ERROR: throw ParseError(msg);
    default: throw Error(msg);
  }
}
inline void check_msg(int code, const char* msg) {  // host-only calls with an err buffer
  if (code == RKMF_OK) return;
  switch (code) {
    case RKMF_PARAMETER_ERROR: throw ParameterError(msg);
    case RKMF_SHAPE_ERROR: throw ShapeError(msg);
    case RKMF_PARSE_ERROR: throw ParseError(msg);
    default: throw Error(msg);
  }
}

// One device + stream; owns nothing else.
class Context {
 public:
  explicit Context(int device = 0) {
    rkmf_context* c = nullptr;
    const int code = rkmf_context_create(device, &c);
    if (code != RKMF_OK) throw DeviceError("rkmf_context_create failed (no CUDA device?)");
    ctx_.reset(c);
  }
  rkmf_context* get() const { return ctx_.get(); }
  // small matrices: a cycle's steps as one cooperative kernel (default on)
  void set_fused_cycle(bool enable) { check(get(), rkmf_context_set_fused_cycle(get(), enable)); }

 private:
  struct Del {
    void operator()(rkmf_context* c) const { rkmf_context_destroy(c); }
  };
  std::unique_ptr<rkmf_context, Del> ctx_;
};

// ---- sparse.hpp:16-24: host CSR, int64 row pointers, int32 columns ----
struct SparseMatrix {
  int64_t n_rows = 0, n_cols = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col_idx;
  std::vector<double> values;
  int64_t nnz() const { return static_cast<int64_t>(values.size()); }
};

// ---- sparse.hpp:55-66: Matrix Market / vector interchange (host) ----
inline SparseMatrix load_matrix_market(const std::string& path) {
  int64_t nr = 0, nc = 0, nnz = 0;
  int64_t* rp = nullptr;
  int32_t* ci = nullptr;
  double* v = nullptr;
  char err[1024] = {0};
  check_msg(rkmf_mtx_load(path.c_str(), &nr, &nc, &nnz, &rp, &ci, &v, err, sizeof(err)), err);
  SparseMatrix A;
  A.n_rows = nr;
  A.n_cols = nc;
  A.row_ptr.assign(rp, rp + nr + 1);
  A.col_idx.assign(ci, ci + nnz);
  A.values.assign(v, v + nnz);
  rkmf_host_free(rp);
  rkmf_host_free(ci);
  rkmf_host_free(v);
  return A;
}
inline void save_matrix_market(const SparseMatrix& A, const std::string& path) {
  char err[1024] = {0};
  check_msg(rkmf_mtx_save(path.c_str(), A.n_rows, A.n_cols, A.row_ptr.data(), A.col_idx.data(),
                          A.values.data(), err, sizeof(err)),
            err);
}
inline std::vector<double> load_vector(const std::string& path) {
  int64_t n = 0;
  double* p = nullptr;
  char err[1024] = {0};
  check_msg(rkmf_vector_load(path.c_str(), &n, &p, err, sizeof(err)), err);
  std::vector<double> v(p, p + n);
  rkmf_host_free(p);
  return v;
}
inline void save_vector(const std::vector<double>& v, const std::string& path) {
  char err[1024] = {0};
  check_msg(rkmf_vector_save(path.c_str(), static_cast<int64_t>(v.size()), v.data(), err,
                             sizeof(err)),
            err);
}

// Device-resident copy of a SparseMatrix (validated on upload, sparse.cpp:61-81).
class DeviceMatrix {
 public:
  DeviceMatrix(const Context& ctx, const SparseMatrix& A) : ctx_(ctx.get()) {
    rkmf_matrix* m = nullptr;
    check(ctx_, rkmf_matrix_create_host(ctx_, A.n_rows, A.n_cols, A.row_ptr.data(),
                                        A.col_idx.data(), A.values.data(), &m));
    m_.reset(m);
  }
  rkmf_matrix* get() const { return m_.get(); }

 private:
  struct Del {
    void operator()(rkmf_matrix* m) const { rkmf_matrix_destroy(m); }
  };
  rkmf_context* ctx_;
  std::unique_ptr<rkmf_matrix, Del> m_;
};

// ---- sketch.hpp:16-31: make_sketch on device, bit-exact ----
class SketchOperator {
 public:
  SketchOperator(const Context& ctx, int64_t d, int64_t n, int64_t zeta, uint64_t seed)
      : ctx_(ctx.get()), d(d), n(n), zeta(zeta), seed(seed) {
    rkmf_sketch* s = nullptr;
    check(ctx_, rkmf_sketch_create(ctx_, d, n, zeta, seed, &s));
    s_.reset(s);
  }
  void set_scale(double scale) { rkmf_sketch_set_scale(s_.get(), scale); }
  // bytes per 128-column tile of the layout the fused kernel streams
  std::pair<int64_t, int64_t> layout_bytes_per_tile() const {
    int64_t h = 0, e = 0;
    rkmf_sketch_layout_info(s_.get(), &h, &e);
    return {h, e};
  }
  rkmf_sketch* get() const { return s_.get(); }
  const rkmf_context* context() const { return ctx_; }

 private:
  struct Del {
    void operator()(rkmf_sketch* s) const { rkmf_sketch_destroy(s); }
  };
  rkmf_context* ctx_;
  std::unique_ptr<rkmf_sketch, Del> s_;

 public:
  const int64_t d, n, zeta;
  const uint64_t seed;
};

// ---- densefun.hpp:19-32 ----
struct FunctionSpec {
  int32_t kind = RKMF_FN_EXP_NEG;
  double t = 1.0;
  static FunctionSpec exp_neg(double t) {
    if (!(t >= 0.0)) throw ParameterError("FunctionSpec: t must be >= 0");
    return FunctionSpec{RKMF_FN_EXP_NEG, t};
  }
  static FunctionSpec inv_sqrt() { return FunctionSpec{RKMF_FN_INV_SQRT, 1.0}; }
};

// ---- restart.hpp:20-65 ----
struct RestartOptions {
  int64_t m_r = 20;
  double tol = 1e-10;
  int64_t k_max = 100;
  int64_t budget_total_m = 4000;
  double divergence_factor = 1e6;
  int32_t dense_f = RKMF_DENSE_AUTO;
  int32_t quad_nodes = 0;   // InvSqrt: 0 = adaptive (Ritz-designed, node doubling)
  bool diagnostics = false;  // kappa_W / leftmost_ritz_re per cycle
};

// ---- restart.hpp:42-54: test-only observer, fed by device->host copies ----
struct CycleInfo {
  int64_t cycle;
  int64_t n, m_k, w_cols;
  const double* W;  // n x w_cols column-major
  int64_t total_m;
  const double* R_accum;  // total_m x total_m column-major, or nullptr
  const double* update;
  const double* f_hat;
  double alpha;
};
using CycleObserver = std::function<void(const CycleInfo&)>;

struct CycleRecord {
  int64_t cycle = 0, total_m = 0;
  long long total_matvecs = 0;
  double update_norm = 0.0;
  std::optional<double> error_vs_reference;
  double kappa_W = 0.0, leftmost_ritz_re = 0.0, alpha_dev = 0.0;
  double elapsed_ms = 0.0, build_ms = 0.0, funm_ms = 0.0;
};

struct PerfCounters {  // types.hpp:57-75
  long long matvecs = 0, dot_n = 0, dot_d = 0, basis_updates = 0;
  int64_t peak_basis_cols = 0;
};

struct RestartResult {
  std::vector<double> f_hat;
  std::vector<CycleRecord> history;
  std::vector<double> R_accum;  // total_m x total_m, column-major
  bool converged = false;
  double alpha = 0.0;
  int64_t cycles = 0, total_m = 0;
  PerfCounters counters;
};

// restart::restarted_krylov (restart.hpp:74-79): S == nullptr selects the
// classical builder (restart.cpp:53-55), otherwise the randomized one with the
// same sketch every cycle; observer is the reference's test-only CycleObserver.
inline RestartResult restarted_krylov(const Context& ctx, const DeviceMatrix& A,
                                      const std::vector<double>& b, const FunctionSpec& f,
                                      const RestartOptions& opts,
                                      const SketchOperator* S = nullptr,
                                      const CycleObserver& observer = nullptr,
                                      const std::vector<double>* reference = nullptr) {
  rkmf_restart_options o;
  rkmf_restart_options_default(&o);
  o.m_r = opts.m_r;
  o.tol = opts.tol;
  o.k_max = opts.k_max;
  o.budget_total_m = opts.budget_total_m;
  o.divergence_factor = opts.divergence_factor;
  o.dense_f = opts.dense_f;
  o.quad_nodes = opts.quad_nodes;
  o.diagnostics = opts.diagnostics ? 1 : 0;
  RestartResult res;
  res.f_hat.assign(b.size(), 0.0);
  std::vector<rkmf_cycle_record> recs(static_cast<size_t>(std::max<int64_t>(opts.k_max, 1)) + 1);
  rkmf_restart_result r{};
  struct Tramp {
    static void call(void* user, const rkmf_cycle_info* i) {
      const CycleInfo c{i->cycle, i->n,       i->m_k,    i->w_cols, i->W,
                        i->total_m, i->R_accum, i->update, i->f_hat,  i->alpha};
      (*static_cast<const CycleObserver*>(user))(c);
    }
  };
  if (observer)
    check(ctx.get(), rkmf_context_set_observer(ctx.get(), &Tramp::call,
                                               const_cast<CycleObserver*>(&observer)));
  const int code = rkmf_restarted_krylov(ctx.get(), A.get(), S ? S->get() : nullptr, b.data(), 0,
                                         f.kind, f.t, &o, res.f_hat.data(), 0,
                                         reference ? reference->data() : nullptr, &r, recs.data(),
                                         static_cast<int64_t>(recs.size()));
  if (observer) rkmf_context_set_observer(ctx.get(), nullptr, nullptr);
  check(ctx.get(), code);
  res.converged = r.converged != 0;
  res.alpha = r.alpha;
  res.cycles = r.cycles;
  res.total_m = r.total_m;
  res.counters = {r.matvecs, r.dot_n, r.dot_d, r.basis_updates, r.peak_basis_cols};
  for (int64_t i = 0; i < r.n_records; ++i) {
    const rkmf_cycle_record& c = recs[static_cast<size_t>(i)];
    CycleRecord h;
    h.cycle = c.cycle;
    h.total_m = c.total_m;
    h.total_matvecs = c.total_matvecs;
    h.update_norm = c.update_norm;
    if (!std::isnan(c.error_vs_reference)) h.error_vs_reference = c.error_vs_reference;
    h.kappa_W = c.kappa_W;
    h.leftmost_ritz_re = c.leftmost_ritz_re;
    h.alpha_dev = c.alpha_dev;
    h.elapsed_ms = c.elapsed_ms;
    h.build_ms = c.build_ms;
    h.funm_ms = c.funm_ms;
    res.history.push_back(h);
  }
  int64_t M = 0;
  check(ctx.get(), rkmf_last_r_accum(ctx.get(), nullptr, 0, &M));
  if (M > 0) {
    res.R_accum.resize(static_cast<size_t>(M * M));
    check(ctx.get(), rkmf_last_r_accum(ctx.get(), res.R_accum.data(), M, &M));
  }
  return res;
}

// the randomized builder with S by reference (round-1 signature)
inline RestartResult restarted_krylov(const Context& ctx, const DeviceMatrix& A,
                                      const std::vector<double>& b, const FunctionSpec& f,
                                      const RestartOptions& opts, const SketchOperator& S,
                                      const std::vector<double>* reference = nullptr) {
  return restarted_krylov(ctx, A, b, f, opts, &S, nullptr, reference);
}

}  // namespace rkmf_b200

#endif  // RKMF_B200_HPP
