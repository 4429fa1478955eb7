// Convergence sweep over methods and its CSV (host C++ above the C ABI).
//
// Restates restart::convergence_sweep / run_method_cell
// (proj/src/restart.cpp:124-305) and the CLI's CSV writer
// (proj/tools/rkmf_bench.cpp:172-186) for the device path: the restarted
// methods ("restart": classical builder, "restart-rand": randomized builder
// with d = 16 m_r unless given, restart.cpp:229-233) run through
// rkmf_restarted_krylov and become one row per cycle; a failing cell becomes
// a single NaN row carrying the sanitised error text and the sweep goes on
// (restart.cpp:276-286). Of the one-shot approximants, "arnoldi" and "rand"
// are the first cycle of the restarted methods and run as such (one row,
// cycle 0); "incomplete", "rand-ls" and "sfom" are outside the device hot path
// (SURVEY.md §2): their cells become such a note row. Rows keep the config order; with
// with_timing off the output is byte-deterministic (the device solves are
// bitwise reproducible, detred.cuh), as acceptance criterion c14 asks
// (proj/tests/acceptance.cpp:545-582). Cells run one after another on the
// context's device (the reference's threads parallelise host cells).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "rkmf_b200.h"

namespace {

std::string sanitize(std::string s) {  // restart.cpp:128-132
  for (char& c : s)
    if (c == ',' || c == '\n' || c == '\r') c = ';';
  return s;
}

void put(char* dst, size_t cap, const std::string& s) {
  std::strncpy(dst, s.c_str(), cap - 1);
  dst[cap - 1] = '\0';
}

rkmf_sweep_record base_row(const rkmf_method_spec& ms, int64_t n) {
  rkmf_sweep_record r;
  std::memset(&r, 0, sizeof(r));
  put(r.method, sizeof(r.method), ms.name);
  r.n = n;
  r.rel_error = std::numeric_limits<double>::quiet_NaN();
  return r;
}

bool one_shot(const std::string& name) {  // restart.cpp:147-150
  return name == "arnoldi" || name == "incomplete" || name == "rand" || name == "rand-ls" ||
         name == "sfom";
}

struct CellError {
  std::string what;
};

std::vector<rkmf_sweep_record> run_cell(rkmf_context* ctx, const rkmf_matrix* A, int64_t n,
                                        const double* b, int32_t kind, double t,
                                        const double* ref, const rkmf_method_spec& ms,
                                        int with_timing) {
  const std::string name(ms.name);
  // The one-shot approximants f_m = beta W_m f(R_m) e_1 on the classical
  // basis ("arnoldi", approximants.cpp:49-60) and alpha W_m f(R_m) e_1 on the
  // randomized one ("rand", approximants.cpp:62-70; d = 4 m unless given,
  // restart.cpp:170-171) are exactly the first cycle of the corresponding
  // restarted method, so they run as one cycle and become one row with
  // cycle = 0 (restart.cpp:199-221; sampled m = {min(m, n)}, restart.cpp:132-142).
  const bool shot = name == "arnoldi" || name == "rand";
  if (one_shot(name) && !shot)
    throw CellError{"method '" + name + "' is a one-shot approximant: not on the device path"};
  if (!shot && name != "restart" && name != "restart-rand")
    throw CellError{"sweep: unknown method name '" + name + "'"};
  const int64_t m_shot = std::min<int64_t>(ms.m, n);
  if (shot && m_shot < 1) throw CellError{"sweep: sampled m values must be >= 1"};
  rkmf_restart_options o;
  rkmf_restart_options_default(&o);
  o.m_r = shot ? m_shot : ms.m;
  o.tol = shot ? std::numeric_limits<double>::min() : ms.tol;
  o.k_max = shot ? 1 : ms.k_max;
  if (shot) o.budget_total_m = std::max<int64_t>(o.budget_total_m, m_shot);
  o.diagnostics = 1;  // kappa_W and the leftmost Ritz value per cycle (restart.cpp:101,103)
  rkmf_sketch* S = nullptr;
  auto fail = [&](int code) {
    if (code != RKMF_OK) {
      const std::string msg = rkmf_last_error(ctx);
      if (S) rkmf_sketch_destroy(S);
      throw CellError{msg};
    }
  };
  if (name == "restart-rand" || name == "rand") {
    const int64_t d = ms.d > 0 ? ms.d : (shot ? 4 * m_shot : 16 * ms.m);
    fail(rkmf_sketch_create(ctx, d, n, ms.zeta, ms.seed, &S));
  }
  std::vector<double> f(static_cast<size_t>(n));
  std::vector<rkmf_cycle_record> recs(static_cast<size_t>(std::max<int64_t>(ms.k_max, 1)) + 1);
  rkmf_restart_result res;
  fail(rkmf_restarted_krylov(ctx, A, S, b, 0, kind, t, &o, f.data(), 0, ref, &res, recs.data(),
                             int64_t(recs.size())));
  if (S) rkmf_sketch_destroy(S);
  std::vector<rkmf_sweep_record> rows;
  for (int64_t i = 0; i < res.n_records; ++i) {  // restart.cpp:244-261
    const rkmf_cycle_record& c = recs[static_cast<size_t>(i)];
    rkmf_sweep_record r = base_row(ms, n);
    r.m_or_totalm = c.total_m;
    r.cycle = shot ? 0 : c.cycle;
    r.matvecs = c.total_matvecs;
    if (ref && !std::isnan(c.error_vs_reference)) r.rel_error = c.error_vs_reference;
    r.update_norm = c.update_norm;
    r.kappa_W = c.kappa_W;
    r.leftmost_ritz_re = c.leftmost_ritz_re;
    if (with_timing) {
      r.elapsed_ms = c.elapsed_ms;
      r.phase_build_ms = c.build_ms;
      r.phase_eval_ms = c.elapsed_ms - c.build_ms;
    }
    rows.push_back(r);
  }
  return rows;
}

std::string fmt17(double v) {  // rkmf_bench.cpp:166-170
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

}  // namespace

extern "C" {

int rkmf_convergence_sweep(rkmf_context* ctx, const rkmf_matrix* A, const double* h_b,
                           int32_t fn_kind, double fn_t, const double* h_reference,
                           const rkmf_method_spec* methods, int64_t n_methods, int32_t with_timing,
                           rkmf_sweep_record* out, int64_t cap, int64_t* n_out) {
  if (!ctx || !A || !h_b || (n_methods > 0 && !methods) || !n_out) return RKMF_PARAMETER_ERROR;
  int64_t n = 0;
  rkmf_matrix_info(A, &n, nullptr, nullptr, nullptr);
  std::vector<rkmf_sweep_record> all;
  for (int64_t i = 0; i < n_methods; ++i) {
    try {
      const std::vector<rkmf_sweep_record> rows =
          run_cell(ctx, A, n, h_b, fn_kind, fn_t, h_reference, methods[i], with_timing);
      all.insert(all.end(), rows.begin(), rows.end());
    } catch (const CellError& e) {  // restart.cpp:279-285: one NaN row with the note
      rkmf_sweep_record r = base_row(methods[i], n);
      put(r.note, sizeof(r.note), sanitize(e.what));
      all.push_back(r);
    }
  }
  *n_out = int64_t(all.size());
  if (out)
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n_out); ++i) out[i] = all[size_t(i)];
  return RKMF_OK;
}

int rkmf_sweep_write_csv(const rkmf_sweep_record* rows, int64_t n_rows, const char* path,
                         char* err, int64_t err_cap) {
  std::string s =
      "method,n,m_or_totalm,cycle,matvecs,rel_error,update_norm,kappa_W,leftmost_ritz_re,"
      "elapsed_ms,note\n";
  for (int64_t i = 0; i < n_rows; ++i) {
    const rkmf_sweep_record& r = rows[i];
    s += std::string(r.method) + ',' + std::to_string(r.n) + ',' + std::to_string(r.m_or_totalm) +
         ',' + std::to_string(r.cycle) + ',' + std::to_string(r.matvecs) + ',' +
         fmt17(r.rel_error) + ',' + fmt17(r.update_norm) + ',' + fmt17(r.kappa_W) + ',' +
         fmt17(r.leftmost_ritz_re) + ',' + fmt17(r.elapsed_ms) + ',' + std::string(r.note) + '\n';
  }
  FILE* fp = (path && path[0]) ? std::fopen(path, "wb") : stdout;
  if (!fp) {
    if (err && err_cap > 0) {
      std::snprintf(err, size_t(err_cap), "%s: cannot open for writing", path);
    }
    return RKMF_INTERNAL_ERROR;
  }
  const bool ok = std::fwrite(s.data(), 1, s.size(), fp) == s.size();
  if (fp != stdout) std::fclose(fp);
  else std::fflush(fp);
  if (!ok) {
    if (err && err_cap > 0) std::snprintf(err, size_t(err_cap), "%s: write failure", path);
    return RKMF_INTERNAL_ERROR;
  }
  return RKMF_OK;
}

}  // extern "C"
