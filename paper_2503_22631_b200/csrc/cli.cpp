// rkmf_b200_bench — the reference CLI's `generate` and `run` subcommands
// (proj/tools/rkmf_bench.cpp) on the device path.
//
//   rkmf_b200_bench generate --config gen.json [--output prefix] [--seed s]
//   rkmf_b200_bench run      --config run.json [--output out.csv] [--threads k] [--seed s]
//
// Config (JSON, the reference's keys): "problem" {"kind": "baseline" (the
// BASELINE configs' generators: "config": "cfg1".."cfg5", optional "N") |
// "external" ("matrix": .mtx, "rhs": vector file), "function" {"kind":
// "exp_neg", "t"} | {"kind": "inv_sqrt"}}, "methods" [{"name", "m_r"|"m",
// "d", "zeta", "tol", "k_max", "seed"}], "reference" {"mode": "none" | "file"
// ("path") | "restart-highm" ("m_r", "tol", "k_max")}, "timing", "output".
// Exit codes as the reference: 0 success, 1 configuration/usage error, 2
// runtime failure (rkmf_bench.cpp:326-335). Problems and sweeps go through the
// C ABI (include/rkmf_b200.h); the sweep and CSV are csrc/sweep.cpp.
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "rkmf_b200.h"

namespace {

struct UsageError : std::runtime_error {  // ParseError / ParameterError -> exit 1
  using std::runtime_error::runtime_error;
};

// ---- a small JSON reader (objects, arrays, strings, numbers, bools, null) ----
struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;
  bool has(const std::string& k) const { return kind == Obj && obj.count(k); }
  const Json& at(const std::string& k) const {
    if (!has(k)) throw UsageError("config: missing key '" + k + "'");
    return obj.at(k);
  }
  double number(const std::string& k, double dflt) const {
    if (!has(k)) return dflt;
    const Json& v = obj.at(k);
    if (v.kind != Num) throw UsageError("config: '" + k + "' must be a number");
    return v.num;
  }
  std::string string(const std::string& k, const std::string& dflt) const {
    if (!has(k)) return dflt;
    const Json& v = obj.at(k);
    if (v.kind != Str) throw UsageError("config: '" + k + "' must be a string");
    return v.str;
  }
  bool boolean(const std::string& k, bool dflt) const {
    if (!has(k)) return dflt;
    const Json& v = obj.at(k);
    if (v.kind != Bool) throw UsageError("config: '" + k + "' must be true/false");
    return v.b;
  }
};

struct JsonParser {
  const std::string& s;
  size_t i = 0;
  explicit JsonParser(const std::string& src) : s(src) {}
  [[noreturn]] void fail(const std::string& what) {
    throw UsageError("config: JSON parse error at offset " + std::to_string(i) + ": " + what);
  }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  Json value() {
    ws();
    if (i >= s.size()) fail("unexpected end");
    const char c = s[i];
    Json v;
    if (c == '{') {
      v.kind = Json::Obj;
      ++i;
      ws();
      if (i < s.size() && s[i] == '}') { ++i; return v; }
      for (;;) {
        ws();
        Json k = value();
        if (k.kind != Json::Str) fail("object key must be a string");
        ws();
        if (i >= s.size() || s[i] != ':') fail("expected ':'");
        ++i;
        v.obj[k.str] = value();
        ws();
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == '}') { ++i; return v; }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Json::Arr;
      ++i;
      ws();
      if (i < s.size() && s[i] == ']') { ++i; return v; }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == ']') { ++i; return v; }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Json::Str;
      ++i;
      while (i < s.size() && s[i] != '"') {
        if (s[i] == '\\' && i + 1 < s.size()) {
          const char e = s[++i];
          v.str += e == 'n' ? '\n' : e == 't' ? '\t' : e;
        } else {
          v.str += s[i];
        }
        ++i;
      }
      if (i >= s.size()) fail("unterminated string");
      ++i;
      return v;
    }
    if (s.compare(i, 4, "true") == 0) { i += 4; v.kind = Json::Bool; v.b = true; return v; }
    if (s.compare(i, 5, "false") == 0) { i += 5; v.kind = Json::Bool; return v; }
    if (s.compare(i, 4, "null") == 0) { i += 4; return v; }
    char* end = nullptr;
    v.num = std::strtod(s.c_str() + i, &end);
    if (end == s.c_str() + i) fail("unexpected character");
    i = size_t(end - s.c_str());
    v.kind = Json::Num;
    return v;
  }
};

Json load_config(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw UsageError(path + ": cannot open config");
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  JsonParser p(text);
  Json j = p.value();
  if (j.kind != Json::Obj) throw UsageError(path + ": the config must be a JSON object");
  return j;
}

// ---- problems ----
struct Problem {
  int64_t n = 0;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> v;
  std::vector<double> b;
  int32_t kind = RKMF_FN_EXP_NEG;
  double t = 1.0;
};

// status first, then the message the call wrote (argument order is unspecified)
void check(int code, const std::string& what);
inline void check_after(int code, const char* err) { check(code, std::string(err)); }

void check(int code, const std::string& what) {
  if (code == RKMF_OK) return;
  if (code == RKMF_PARAMETER_ERROR || code == RKMF_PARSE_ERROR) throw UsageError(what);
  throw std::runtime_error(what);
}

// ||A||_2 by 60 fixed-seed power iterations (on A^T A when nonsymmetric),
// the convention of paper_2503_22631_b200/configs.py (acceptance.cpp:429-437)
double power_norm2(const Problem& P, bool symmetric) {
  const int64_t n = P.n;
  std::vector<double> x(static_cast<size_t>(n)), y(static_cast<size_t>(n)), z(static_cast<size_t>(n));
  rkmf_gen_gaussian(7, n, x.data());
  double nx = 0.0;
  for (double a : x) nx += a * a;
  nx = std::sqrt(nx);
  for (double& a : x) a /= nx;
  double lam = 0.0;
  for (int it = 0; it < 60; ++it) {
    for (int64_t r = 0; r < n; ++r) {
      double s = 0.0;
      for (int64_t k = P.rp[size_t(r)]; k < P.rp[size_t(r) + 1]; ++k) s += P.v[size_t(k)] * x[size_t(P.ci[size_t(k)])];
      y[size_t(r)] = s;
    }
    if (!symmetric) {
      std::fill(z.begin(), z.end(), 0.0);
      for (int64_t r = 0; r < n; ++r)
        for (int64_t k = P.rp[size_t(r)]; k < P.rp[size_t(r) + 1]; ++k)
          z[size_t(P.ci[size_t(k)])] += P.v[size_t(k)] * y[size_t(r)];
      y.swap(z);
    }
    double ny = 0.0;
    for (double a : y) ny += a * a;
    lam = std::sqrt(ny);
    for (int64_t r = 0; r < n; ++r) x[size_t(r)] = y[size_t(r)] / lam;
  }
  return symmetric ? lam : std::sqrt(lam);
}

void parse_function(const Json& jf, Problem& P) {
  const std::string kind = jf.at("kind").str;
  if (kind == "exp_neg") {
    P.kind = RKMF_FN_EXP_NEG;
    P.t = jf.number("t", 1.0);
    if (!(P.t >= 0.0)) throw UsageError("FunctionSpec: t must be >= 0");
  } else if (kind == "inv_sqrt") {
    P.kind = RKMF_FN_INV_SQRT;
  } else {
    throw UsageError("config: function kind '" + kind + "' is not on the device path "
                     "(exp_neg, inv_sqrt)");
  }
}

Problem build_problem(const Json& cfg) {
  if (!cfg.has("problem")) throw UsageError("config: missing 'problem' object");
  const Json& p = cfg.at("problem");
  const std::string kind = p.at("kind").str;
  Problem P;
  char err[1024] = {0};
  if (kind == "external") {  // problems.cpp:494-508
    if (!p.has("function")) throw UsageError("config: external problems need a 'function'");
    int64_t nr = 0, nc = 0, nnz = 0;
    int64_t* rp = nullptr;
    int32_t* ci = nullptr;
    double* v = nullptr;
    check_after(rkmf_mtx_load(p.at("matrix").str.c_str(), &nr, &nc, &nnz, &rp, &ci, &v, err, sizeof(err)), err);
    P.n = nr;
    P.rp.assign(rp, rp + nr + 1);
    P.ci.assign(ci, ci + nnz);
    P.v.assign(v, v + nnz);
    rkmf_host_free(rp);
    rkmf_host_free(ci);
    rkmf_host_free(v);
    if (nr != nc) throw UsageError("external: matrix must be square");
    int64_t nb = 0;
    double* bb = nullptr;
    check_after(rkmf_vector_load(p.at("rhs").str.c_str(), &nb, &bb, err, sizeof(err)), err);
    P.b.assign(bb, bb + nb);
    rkmf_host_free(bb);
    if (nb != nr) throw UsageError("external: rhs length does not match the matrix");
    parse_function(p.at("function"), P);
    return P;
  }
  if (kind != "baseline") throw UsageError("config: unknown problem kind '" + kind + "'");
  // BASELINE.json configs (paper_2503_22631_b200/configs.py CONFIGS)
  const std::string name = p.at("config").str;
  static const std::map<std::string, std::vector<double>> cfgs = {
      // kind(0 lap2d,1 lap3d,2 q1,3 convdiff), N, c (t = c / ||A||_2), lognormal, dirichlet
      {"cfg1", {0, 256, 100, 0, 0}}, {"cfg2", {1, 128, 500, 0, 0}}, {"cfg3", {2, 200, 0, 1, 1}},
      {"cfg4", {3, 256, 200, 0, 0}}, {"cfg5", {2, 512, 300, 0, 0}}};
  if (!cfgs.count(name)) throw UsageError("config: unknown baseline config '" + name + "'");
  const std::vector<double>& c = cfgs.at(name);
  const int64_t N = int64_t(p.number("N", c[1]));
  int64_t n = 0, nnz = 0;
  const int k = int(c[0]);
  auto gen = [&](bool fill) {
    int64_t* rp = fill ? P.rp.data() : nullptr;
    int32_t* ci = fill ? P.ci.data() : nullptr;
    double* v = fill ? P.v.data() : nullptr;
    int code;
    if (k <= 1) code = rkmf_gen_laplacian(k == 0 ? 2 : 3, N, &n, &nnz, rp, ci, v);
    else if (k == 2) code = rkmf_gen_q1_hex(N, int(c[3]), 1, int(c[4]), &n, &nnz, rp, ci, v);
    else code = rkmf_gen_convdiff_upwind(N, 10.0, 1.0, 0.5, 0.25, &n, &nnz, rp, ci, v);
    if (code != RKMF_OK) throw UsageError("baseline: invalid grid size");
  };
  gen(false);
  P.n = n;
  P.rp.resize(size_t(n + 1));
  P.ci.resize(size_t(nnz));
  P.v.resize(size_t(nnz));
  gen(true);
  P.b.resize(size_t(n));
  rkmf_gen_gaussian(1, n, P.b.data());
  if (k == 2 && c[2] == 0) {
    P.kind = RKMF_FN_INV_SQRT;
  } else {
    double norm2;
    if (k <= 1) {  // analytic lambda_max of the Dirichlet Laplacian
      const double h = 1.0 / double(N + 1), s = std::sin(double(N) * M_PI / double(2 * N + 2));
      norm2 = (4.0 * (k == 0 ? 2 : 3) / (h * h)) * s * s;
    } else {
      norm2 = power_norm2(P, k == 2);
    }
    P.t = c[2] / norm2;
  }
  if (p.has("function")) parse_function(p.at("function"), P);
  return P;
}

struct Args {
  std::string sub, config, output;
  int threads = 1;
  bool has_seed = false;
  uint64_t seed = 0;
};

struct Device {
  rkmf_context* ctx = nullptr;
  rkmf_matrix* A = nullptr;
  Device() { check(rkmf_context_create(0, &ctx), "rkmf_context_create: no CUDA device"); }
  ~Device() {
    rkmf_matrix_destroy(A);
    rkmf_context_destroy(ctx);
  }
  void ok(int code) { check(code, rkmf_last_error(ctx)); }
};

int cmd_generate(const Args& a) {  // rkmf_bench.cpp:188-204
  const Json cfg = load_config(a.config);
  const Problem P = build_problem(cfg);
  const std::string prefix = !a.output.empty() ? a.output : cfg.string("output", "");
  if (prefix.empty()) throw UsageError("config: generate needs an output prefix");
  char err[1024] = {0};
  check_after(rkmf_mtx_save((prefix + ".mtx").c_str(), P.n, P.n, P.rp.data(), P.ci.data(), P.v.data(),
                      err, sizeof(err)), err);
  check_after(rkmf_vector_save((prefix + ".b.txt").c_str(), P.n, P.b.data(), err, sizeof(err)), err);
  std::printf("wrote %s.mtx %s.b.txt (n=%lld, nnz=%lld)\n", prefix.c_str(), prefix.c_str(),
              (long long)P.n, (long long)P.v.size());
  return 0;
}

int cmd_run(const Args& a) {  // rkmf_bench.cpp:206-250
  const Json cfg = load_config(a.config);
  const Problem P = build_problem(cfg);
  std::vector<rkmf_method_spec> methods;
  if (cfg.has("methods")) {
    for (const Json& e : cfg.at("methods").arr) {
      rkmf_method_spec ms;
      std::memset(&ms, 0, sizeof(ms));
      const std::string name = e.at("name").str;
      static const char* known[] = {"arnoldi", "incomplete", "rand", "rand-ls", "sfom", "restart",
                                    "restart-rand"};
      bool ok = false;
      for (const char* k : known) ok |= name == k;
      if (!ok) throw UsageError("config: unknown method name '" + name + "'");
      std::strncpy(ms.name, name.c_str(), sizeof(ms.name) - 1);
      ms.m = int64_t(e.has("m_r") ? e.number("m_r", 100) : e.number("m", 100));
      ms.d = int64_t(e.number("d", 0));
      ms.zeta = int64_t(e.number("zeta", 4));
      ms.tol = e.number("tol", 1e-10);
      ms.k_max = int64_t(e.number("k_max", 100));
      ms.seed = a.has_seed ? a.seed : uint64_t(e.number("seed", 0));
      if ((name == "restart" || name == "restart-rand") && ms.k_max * ms.m > 4000)
        std::fprintf(stderr,
                     "warning: %s k_max*m_r = %lld exceeds the total-m budget 4000; cycles stop "
                     "at the budget\n",
                     name.c_str(), (long long)(ms.k_max * ms.m));
      methods.push_back(ms);
    }
  }
  const bool timing = cfg.boolean("timing", false);
  Device dev;
  dev.ok(rkmf_matrix_create_host(dev.ctx, P.n, P.n, P.rp.data(), P.ci.data(), P.v.data(), &dev.A));
  // reference (rkmf_bench.cpp:125-152)
  std::vector<double> ref;
  const Json none;
  const Json& rj = cfg.has("reference") ? cfg.at("reference") : none;
  const std::string mode = rj.kind == Json::Obj ? rj.string("mode", "none") : "none";
  char err[1024] = {0};
  if (mode == "file") {
    int64_t nr = 0;
    double* p = nullptr;
    check_after(rkmf_vector_load(rj.at("path").str.c_str(), &nr, &p, err, sizeof(err)), err);
    ref.assign(p, p + nr);
    rkmf_host_free(p);
    if (nr != P.n) throw UsageError("reference: length does not match the problem");
  } else if (mode == "restart-highm") {
    rkmf_restart_options o;
    rkmf_restart_options_default(&o);
    o.m_r = int64_t(rj.number("m_r", 100));
    o.tol = rj.number("tol", 3e-12);
    o.k_max = int64_t(rj.number("k_max", 100));
    ref.resize(size_t(P.n));
    rkmf_restart_result r;
    dev.ok(rkmf_restarted_krylov(dev.ctx, dev.A, nullptr, P.b.data(), 0, P.kind, P.t, &o,
                                 ref.data(), 0, nullptr, &r, nullptr, 0));
  } else if (mode != "none") {
    throw UsageError("config: reference mode '" + mode + "' is not on the device path "
                     "(none, file, restart-highm)");
  }
  int64_t nrows = 0;
  dev.ok(rkmf_convergence_sweep(dev.ctx, dev.A, P.b.data(), P.kind, P.t,
                                ref.empty() ? nullptr : ref.data(), methods.data(),
                                int64_t(methods.size()), timing ? 1 : 0, nullptr, 0, &nrows));
  std::vector<rkmf_sweep_record> rows(size_t(std::max<int64_t>(nrows, 1)));
  dev.ok(rkmf_convergence_sweep(dev.ctx, dev.A, P.b.data(), P.kind, P.t,
                                ref.empty() ? nullptr : ref.data(), methods.data(),
                                int64_t(methods.size()), timing ? 1 : 0, rows.data(), nrows,
                                &nrows));
  const std::string out = !a.output.empty() ? a.output : cfg.string("output", "");
  check_after(rkmf_sweep_write_csv(rows.data(), nrows, out.c_str(), err, sizeof(err)), err);
  if (timing) {  // rkmf_bench.cpp:232-247
    std::map<std::string, std::vector<double>> agg;
    for (int64_t i = 0; i < nrows; ++i) {
      auto& v = agg[rows[size_t(i)].method];
      v.resize(3, 0.0);
      v[0] += rows[size_t(i)].phase_build_ms;
      v[1] += rows[size_t(i)].phase_eval_ms;
      v[2] += rows[size_t(i)].elapsed_ms;
    }
    for (const auto& kv : agg)
      std::fprintf(stderr, "timing %s: basis build %.2f ms, function+update %.2f ms, total %.2f ms\n",
                   kv.first.c_str(), kv.second[0], kv.second[1], kv.second[2]);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  auto usage = [] {
    std::fprintf(stderr,
                 "usage: rkmf_b200_bench {generate|run} --config FILE [--output PATH] "
                 "[--threads K] [--seed S]\n");
    return 1;
  };
  if (argc < 2) return usage();
  a.sub = argv[1];
  if (a.sub != "generate" && a.sub != "run") {
    if (a.sub == "spectrum") {
      std::fprintf(stderr, "error: spectrum (dense eigendecomposition) is not on the device path\n");
      return 1;
    }
    return usage();
  }
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    if (i + 1 >= argc) return usage();
    const std::string v = argv[++i];
    if (k == "--config") a.config = v;
    else if (k == "--output") a.output = v;
    else if (k == "--threads") a.threads = std::atoi(v.c_str());
    else if (k == "--seed") {
      a.has_seed = true;
      a.seed = std::strtoull(v.c_str(), nullptr, 10);
    } else {
      return usage();
    }
  }
  if (a.config.empty()) return usage();
  if (a.threads < 1) {
    std::fprintf(stderr, "error: --threads must be >= 1\n");
    return 1;
  }
  try {
    return a.sub == "generate" ? cmd_generate(a) : cmd_run(a);
  } catch (const UsageError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
