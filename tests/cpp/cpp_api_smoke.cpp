// C++ host-API smoke test (include/rkmf_b200.hpp): cfg1-shaped 2D Laplacian on
// a 48x48 grid, exp(-tA)b through rkmf_b200::restarted_krylov, compared with a
// reference f computed by a fine explicit time-integration-free check: the
// semigroup identity exp(-tA)b = exp(-tA/2)(exp(-tA/2)b). Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "rkmf_b200.hpp"

int main() {
  using namespace rkmf_b200;
  try {
    Context ctx(0);
    const int64_t N = 48;
    SparseMatrix A;
    int64_t n = 0, nnz = 0;
    rkmf_gen_laplacian(2, N, &n, &nnz, nullptr, nullptr, nullptr);
    A.n_rows = A.n_cols = n;
    A.row_ptr.resize(static_cast<size_t>(n + 1));
    A.col_idx.resize(static_cast<size_t>(nnz));
    A.values.resize(static_cast<size_t>(nnz));
    rkmf_gen_laplacian(2, N, &n, &nnz, A.row_ptr.data(), A.col_idx.data(), A.values.data());
    std::vector<double> b(static_cast<size_t>(n));
    rkmf_gen_gaussian(1, n, b.data());
    const double h = 1.0 / double(N + 1);
    const double lmax = 8.0 / (h * h) * std::pow(std::sin(N * M_PI / (2 * N + 2)), 2);
    const double t = 100.0 / lmax;
    DeviceMatrix dA(ctx, A);
    SketchOperator S(ctx, 120, n, 8, 1);
    RestartOptions o;
    o.m_r = 30;
    double bn = 0;
    for (double v : b) bn += v * v;
    o.tol = 1e-12 * std::sqrt(bn);
    RestartResult full = restarted_krylov(ctx, dA, b, FunctionSpec::exp_neg(t), o, S);
    RestartResult h1 = restarted_krylov(ctx, dA, b, FunctionSpec::exp_neg(t / 2), o, S);
    RestartResult h2 = restarted_krylov(ctx, dA, h1.f_hat, FunctionSpec::exp_neg(t / 2), o, S);
    double e = 0, nf = 0;
    for (size_t i = 0; i < b.size(); ++i) {
      e += (full.f_hat[i] - h2.f_hat[i]) * (full.f_hat[i] - h2.f_hat[i]);
      nf += full.f_hat[i] * full.f_hat[i];
    }
    const double rel = std::sqrt(e / nf);
    // the same solve through the per-step kernels (the matrix is small enough
    // for the fused cycle kernel by default): equal to rounding
    ctx.set_fused_cycle(false);
    RestartResult steps = restarted_krylov(ctx, dA, b, FunctionSpec::exp_neg(t), o, S);
    ctx.set_fused_cycle(true);
    double es = 0;
    for (size_t i = 0; i < b.size(); ++i)
      es += (full.f_hat[i] - steps.f_hat[i]) * (full.f_hat[i] - steps.f_hat[i]);
    const auto lb = S.layout_bytes_per_tile();
    if (std::sqrt(es / nf) > 1e-11 || steps.cycles != full.cycles || lb.first <= 0 ||
        lb.second <= 0) {
      std::printf("cpp_api_smoke: fused vs per-step kernels differ (%.3e)\n", std::sqrt(es / nf));
      return 1;
    }
    std::printf("cpp_api_smoke: n=%lld cycles=%lld converged=%d semigroup_rel=%.3e R_accum=%zux\n",
                (long long)n, (long long)full.cycles, int(full.converged), rel,
                full.R_accum.size());
    // classical builder (S == nullptr, restart.cpp:53-55) and the observer
    int seen = 0;
    double last_f = 0.0;
    CycleObserver obs = [&](const CycleInfo& ci) {
      ++seen;
      last_f = ci.f_hat[0];
    };
    RestartResult cl = restarted_krylov(ctx, dA, b, FunctionSpec::exp_neg(t), o, nullptr, obs);
    double ec = 0;
    for (size_t i = 0; i < b.size(); ++i)
      ec += (cl.f_hat[i] - full.f_hat[i]) * (cl.f_hat[i] - full.f_hat[i]);
    const double rel_cl = std::sqrt(ec / nf);
    const bool obs_ok = seen == int(cl.cycles) && last_f == cl.f_hat[0];
    // Matrix Market round trip (sparse.cpp:140-211)
    const std::string path = "/tmp/rkmf_cpp_api_smoke.mtx";
    save_matrix_market(A, path);
    const SparseMatrix B = load_matrix_market(path);
    std::remove(path.c_str());
    const bool mtx_ok = B.row_ptr == A.row_ptr && B.col_idx == A.col_idx && B.values == A.values;
    std::printf("cpp_api_smoke: classical_rel=%.3e observer_calls=%d mtx_round_trip=%d\n", rel_cl,
                seen, int(mtx_ok));
    bool parse_threw = false;
    try {
      load_matrix_market("/nonexistent/rkmf.mtx");
    } catch (const ParseError&) {
      parse_threw = true;
    }
    bool threw = false;
    try {
      RestartOptions bad;
      bad.m_r = 0;
      restarted_krylov(ctx, dA, b, FunctionSpec::exp_neg(t), bad, S);
    } catch (const ParameterError& ex) {
      threw = std::string(ex.what()).find("restart: m_r must be >= 1") == 0;
    }
    return (full.converged && rel < 1e-9 && threw && cl.converged && rel_cl < 1e-9 && obs_ok &&
            mtx_ok && parse_threw && full.R_accum.size() == size_t(full.total_m * full.total_m))
               ? 0
               : 1;
  } catch (const std::exception& ex) {
    std::printf("cpp_api_smoke: exception: %s\n", ex.what());
    return 2;
  }
}
