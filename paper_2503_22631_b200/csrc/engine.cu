// Host C++ engine and C ABI of rkmf_b200.
//
// rkmf_restarted_krylov restates restart::restarted_krylov
// (proj/src/restart.cpp:27-122) with the randomized builder
// (proj/src/basis.cpp:92-142) running as device kernels:
//
//   per cycle:  start_init (alpha_k, U[:,0])                          1 block
//               m x [ spmv_sketch (K2) -> rgs_step (K3) -> basis_update (K4) ]
//               dense f (K6: FULL exp(-tR)e1 or restart quadrature)
//               final_update (K5: last basis update + y = alpha W g, f += y)
//               spmv_sketch in sketch-only mode on the next start vector
//
// The host reads a few scalars back once (quadrature) or twice (FULL: the
// squaring count needs ||R_accum||_1) per cycle; everything else stays on the
// device. There is no CPU fallback: without a CUDA device every call fails
// with RKMF_DEVICE_ERROR.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "rkmf_internal.cuh"

using namespace rkmf_b200;

namespace rkmf_b200 {
bool pdl_enabled() {  // RKMF_PDL=0 launches the step kernels without PDL
  static int v = -1;
  if (v < 0) {
    const char* e = knob_env("RKMF_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
}  // namespace rkmf_b200

#include "engine_types.cuh"

namespace {

template <class F>
int guarded(rkmf_context* ctx, F&& fn) {
  try {
    fn();
    if (ctx) ctx->last_error.clear();
    return RKMF_OK;
  } catch (const Error& e) {
    if (ctx) ctx->last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_error = e.what();
    return RKMF_INTERNAL_ERROR;
  }
}

void set_device(rkmf_context* ctx) { RKMF_CUDA(cudaSetDevice(ctx->device)); }

int choose_cap(const std::vector<int64_t>& tile_nnz_max) {
  int64_t mx = 1;
  for (int64_t v : tile_nnz_max) mx = std::max(mx, v);
  return int(std::min<int64_t>(4096, round_up(std::max<int64_t>(mx, 128), 128)));
}

// ---- matrix construction helpers ----
// Validates the CSR on device (sparse.cpp:61-81) and caches norm1
// (sparse.cpp:97-102): once per matrix instead of every cycle (basis.cpp:15,118).
void finish_matrix(rkmf_matrix* M, int64_t max_tile_nnz, bool require_sorted) {
  rkmf_context* ctx = M->ctx;
  M->view.cap = choose_cap({max_tile_nnz});
  M->view.row_ptr = M->rp;
  M->view.col = M->col;
  M->view.val = M->val;
  char* scr = static_cast<char*>(ctx->scratch.ensure(64));
  int32_t* flags = reinterpret_cast<int32_t*>(scr);
  double* out = reinterpret_cast<double*>(scr + 16);
  DevBuf colsum;
  colsum.ensure(sizeof(double) * size_t(2 * M->view.n_cols + 1));
  // validate first: norm1 scatters by column index
  launch_matrix_check(&M->view, flags, require_sorted, ctx->stream);
  int32_t hf[2] = {0, 0};
  RKMF_CUDA(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, ctx->stream));
  RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hf[0]) shape_error("invalid CSR structure (sparse.cpp:61-81 invariants)");
  if (hf[1]) numerical_error("non-finite matrix entry");
  launch_matrix_norm1(&M->view, colsum.as<double>(), out, ctx->stream);
  ctx->launches += 4;
  RKMF_CUDA(cudaMemcpyAsync(&M->norm1, out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
  colsum.release();
  if (dia_enabled_by_env()) build_dia(M);
  if (!M->view.ndiag) build_csr_dict(M);
}

__global__ void rp_narrow_kernel(int64_t n, const int64_t* __restrict__ src, int32_t* dst) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = int32_t(src[i]);
}

__global__ void tile_nnz_max_kernel(int64_t n, const int64_t* __restrict__ rp,
                                    unsigned long long* out) {
  const int64_t tiles = (n + kTileRows - 1) / kTileRows;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < tiles;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r0 = t * kTileRows, r1 = min(n, r0 + kTileRows);
    atomicMax(out, (unsigned long long)(rp[r1] - rp[r0]));
  }
}

double host_norm(const double* x, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += x[i] * x[i];
  return std::sqrt(s);
}

struct SolveBuffers {
  int64_t n, n_global, d, m_eff, ldw, ldr;
  double *W, *U, *Rbar, *G, *z;
};

// n: local rows; n_ext: local rows + halo columns (W columns carry the halo
// tail the partitioned SpMV reads); n_global: rows of the whole problem.
SolveBuffers prepare(rkmf_context* ctx, int64_t n, int64_t n_ext, int64_t n_global, int64_t d,
                     int64_t m_eff) {
  SolveBuffers b;
  b.n = n;
  b.n_global = n_global;
  b.d = d;
  b.m_eff = m_eff;
  b.ldw = round_up(std::max<int64_t>(n_ext, 1), 32);
  b.ldr = m_eff + 1;
  b.W = static_cast<double*>(ctx->W.ensure(sizeof(double) * size_t(b.ldw) * size_t(m_eff + 1)));
  // +2: the Gram-form K3 bulk-copies U[:,0..k] rounded up to 16 bytes
  b.U = static_cast<double*>(ctx->U.ensure(sizeof(double) * (size_t(d) * size_t(m_eff + 1) + 2)));
  b.Rbar = static_cast<double*>(ctx->Rbar.ensure(sizeof(double) * size_t(b.ldr) * size_t(m_eff)));
  b.G = static_cast<double*>(ctx->gram.ensure(sizeof(double) * size_t(b.ldr) * size_t(b.ldr)));
  b.z = static_cast<double*>(ctx->z.ensure(sizeof(double) * size_t(b.ldw)));
  ctx->ensure_red(d);
  RKMF_CUDA(cudaMemsetAsync(b.Rbar, 0, sizeof(double) * size_t(b.ldr) * size_t(m_eff), ctx->stream));
  RKMF_CUDA(cudaMemsetAsync(ctx->st_dev, 0, sizeof(SolveState), ctx->stream));
  return b;
}

void check_builder_args(const rkmf_matrix* A, const rkmf_sketch* S, int64_t m) {
  // basis.cpp:14-23, 96-101 (dimensions of the global problem when partitioned)
  const int64_t ng = A->n_rows_global();
  if (!A->partitioned && A->view.n_rows != A->view.n_cols)
    shape_error("arnoldi: matrix must be square");
  if (m < 1) param_error("arnoldi: m must be >= 1");
  if (m > ng) param_error("arnoldi: m exceeds matrix dimension");
  if (!S) return;  // classical builder (basis.cpp:34-77)
  if (S->n != A->view.n_rows || (A->partitioned && (S->n_global != ng ||
                                                     S->col_begin != A->halo.row_begin)))
    shape_error("randomized_arnoldi: sketch width mismatch");
  const int64_t need = (m == ng) ? m : m + 1;
  if (S->d < need) param_error("randomized_arnoldi: sketch dimension d too small for m");
}

// The sketch of one launch for its consumer: on one rank, the group partials
// as written (the consumer sums them in group order); partitioned, the ranks'
// sums must be added, so the groups are summed on device first (a one-block
// kernel, fixed order) and the d doubles allreduced.
SketchSum sketch_allreduce(rkmf_context* ctx, const DetRed& red, int64_t d, DevBuf& fin) {
  if (!ctx->comm || ctx->nranks <= 1) return SketchSum{red.gpart, red.groups};
  double* out = static_cast<double*>(fin.ensure(sizeof(double) * size_t(d)));
  launch_det_finish(red, d, out, ctx->stream);
  ctx->launches++;
  comm_allreduce_sum(ctx, out, size_t(d));
  return SketchSum{out, 1};
}

// The m_eff steps of one cycle (basis.cpp:119-139). fuse_last: leave the
// last basis update to final_update (K5).
void run_steps(rkmf_context* ctx, const rkmf_matrix* A, const rkmf_sketch* S,
               const SolveBuffers& b, double tol, bool fuse_last) {
  const SketchView sv = S->view();
  if (ctx->fused_cycle && !(ctx->comm && ctx->nranks > 1) && !A->partitioned &&
      cycle_small_applicable(&A->view, &sv, b.m_eff)) {
    bool ok = false;
    ctx->timed(6, [&] {
      ok = launch_cycle_small(&A->view, &sv, int(b.m_eff), fuse_last, b.W, b.ldw, b.z, b.U,
                              b.Rbar, b.ldr, b.G, tol, b.n_global, ctx->st_dev,
                              ctx->red_sketch(b.d), ctx->stream);
    });
    if (ok) {
      ctx->launches++;
      return;
    }
  }
  const int grid = spmv_sketch_grid(&A->view, &sv, 1);
  int32_t* stop = &ctx->st_dev->stopped;
  DetRed& red = ctx->red_sketch(b.d);
  for (int64_t k = 0; k < b.m_eff; ++k) {
    double* x = b.W + k * b.ldw;
    comm_halo_exchange(ctx, A, x);  // multi-GPU: off-rank x entries into the halo tail
    ctx->timed(0, [&] {
      launch_spmv_sketch(&A->view, &sv, 1, x, k == 0 ? &ctx->st_dev->sigma : nullptr, b.z,
                         stop, int(k), grid, red, ctx->stream);
    });
    const SketchSum p = sketch_allreduce(ctx, red, b.d, ctx->pfin_sk);
    ctx->timed(1, [&] {
      launch_rgs_step(b.d, int(k), b.ldr, b.n_global, tol, p.part, p.groups, b.U, b.Rbar,
                      b.G, b.ldr,
                      ctx->st_dev,
                      ctx->stream);
    });
    ctx->launches += 2;
    if (!(fuse_last && k == b.m_eff - 1)) {
      ctx->timed(2, [&] {
        launch_basis_update(b.n, int(k), b.ldw, b.W, b.z, b.Rbar, b.ldr, ctx->st_dev, ctx->stream);
      });
      ctx->launches++;
    }
  }
}

// Classical builder steps (S == nullptr; basis.cpp:47-72 via CGS2, classical.cu).
// cl: [h1 | h2 | nrm2 | rlast (ldr x m_eff)]; fuse_last leaves the last
// update (z' - W h2)/beta to final_update, with (h2, beta) in rlast.
void run_steps_classical(rkmf_context* ctx, const rkmf_matrix* A, const SolveBuffers& b,
                         double tol, bool fuse_last, double* cl) {
  double* h1 = cl;
  double* h2 = cl + b.ldr;
  double* nrm2 = cl + 2 * b.ldr;
  double* rlast = cl + 2 * b.ldr + 2;
  const int grid = spmv_sketch_grid(&A->view, nullptr, 0);
  int32_t* stop = &ctx->st_dev->stopped;
  cudaStream_t st = ctx->stream;
  for (int64_t k = 0; k < b.m_eff; ++k) {
    const bool last = fuse_last && k == b.m_eff - 1;
    double* x = b.W + k * b.ldw;
    comm_halo_exchange(ctx, A, x);
    ctx->timed(0, [&] {
      DetRed none;  // mode 0: no sketch
      launch_spmv_sketch(&A->view, nullptr, 0, x, k == 0 ? &ctx->st_dev->sigma : nullptr, b.z,
                         stop, int(k), grid, none, st);
    });
    const DetRed& rcl = ctx->red_classical(b.m_eff + 1);
    const DetRed& rsc = ctx->red_update();
    ctx->timed(1, [&] { launch_cl_multidot(b.n, int(k), b.ldw, b.W, b.z, h1, ctx->st_dev, rcl, st); });
    comm_allreduce_sum(ctx, h1, size_t(k + 1));
    ctx->timed(2, [&] {
      launch_cl_update(b.n, int(k), b.ldw, b.W, b.z, h1, nullptr, true, ctx->st_dev, rsc, st);
    });
    ctx->timed(1, [&] { launch_cl_multidot(b.n, int(k), b.ldw, b.W, b.z, h2, ctx->st_dev, rcl, st); });
    comm_allreduce_sum(ctx, h2, size_t(k + 1));
    ctx->timed(2, [&] {
      launch_cl_update(b.n, int(k), b.ldw, b.W, b.z, h2, nrm2, !last, ctx->st_dev, rsc, st);
    });
    comm_allreduce_sum(ctx, nrm2, 1);
    ctx->timed(1, [&] {
      launch_cl_decide(int(k), b.ldr, b.n_global, tol, h1, h2, nrm2, b.Rbar,
                       last ? rlast : nullptr, ctx->st_dev, st);
    });
    ctx->launches += 6;
    if (!last) {
      ctx->timed(2, [&] {
        launch_cl_scale(b.n, int(k), b.ldw, b.W, b.z, b.Rbar, b.ldr, ctx->st_dev, st);
      });
      ctx->launches++;
    }
  }
}

// Classical start (basis.cpp:38-43): ||start||_2 over the (local) rows.
void start_classical(rkmf_context* ctx, const SolveBuffers& b, double* cl, bool first) {
  double* nrm2 = cl + 2 * b.ldr;
  ctx->timed(5, [&] {
    launch_cl_start(b.n, b.W, nrm2, ctx->st_dev, first, int(b.m_eff), true, ctx->red_update(),
                    ctx->stream);
  });
  comm_allreduce_sum(ctx, nrm2, 1);
  ctx->timed(5, [&] {
    launch_cl_start(b.n, b.W, nrm2, ctx->st_dev, first, int(b.m_eff), false, ctx->red_update(),
                    ctx->stream);
  });
  ctx->launches += 2;
}

// One node set of the adaptive InvSqrt restart quadrature (densef.cu): the
// nodes of an InvSqrtDesign, their running states, the partial sums and the
// g it produces.
struct QuadSet {
  rkmf_context::QuadBufs* buf = nullptr;
  QuadState q{};
  InvSqrtDesign d;
  double* partial = nullptr;
  double* g = nullptr;
  // stream-ordered (the context stream is non-blocking: a legacy-stream
  // cudaMemcpy would not wait for its kernels)
  void load(const InvSqrtDesign& dd, int64_t m_eff, cudaStream_t st) {
    d = dd;
    std::vector<double> hs, hw;
    invsqrt_nodes(d, hs, hw);
    const std::vector<double> ones(hs.size(), 1.0);
    const size_t nb = sizeof(double) * hs.size();
    q.nq = d.nq;
    q.shift = static_cast<double*>(buf->shift.ensure(nb));
    q.weight = static_cast<double*>(buf->weight.ensure(nb));
    q.pi = static_cast<double*>(buf->pi.ensure(nb));
    q.emx = static_cast<double*>(buf->emx.ensure(nb));
    partial = static_cast<double*>(buf->partial.ensure(nb * size_t(m_eff)));
    g = static_cast<double*>(buf->g.ensure(sizeof(double) * size_t(m_eff)));
    RKMF_CUDA(cudaMemcpyAsync(q.shift, hs.data(), nb, cudaMemcpyHostToDevice, st));
    RKMF_CUDA(cudaMemcpyAsync(q.weight, hw.data(), nb, cudaMemcpyHostToDevice, st));
    RKMF_CUDA(cudaMemcpyAsync(q.pi, ones.data(), nb, cudaMemcpyHostToDevice, st));
    RKMF_CUDA(cudaStreamSynchronize(st));  // the host vectors die here
  }
};

// S * start (basis.cpp:103-104) into the start-sketch group partials
// (ctx->red_st), summed by start_init
void start_sketch(rkmf_context* ctx, const rkmf_sketch* S, const SolveBuffers& b) {
  const SketchView sv = S->view();
  DetRed& red = ctx->red_start(b.d);
  ctx->timed(5, [&] {
    launch_spmv_sketch(nullptr, &sv, 2, b.W, nullptr, nullptr, nullptr, 0, 0, red, ctx->stream);
  });
  ctx->launches++;
  ctx->start_sum = sketch_allreduce(ctx, red, b.d, ctx->pfin_st);
}

void copy_in(rkmf_context* ctx, double* dst, const double* src, int64_t n, bool on_device) {
  if (n <= 0) return;
  RKMF_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * size_t(n),
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            ctx->stream));
}

}  // namespace

// host/device CSR -> validated device matrix (also used by gen.cu)
rkmf_matrix* rkmf_b200::create_from_device_rp64(rkmf_context* ctx, int64_t n_rows, int64_t n_cols,
                                     int64_t nnz, const int64_t* rp64_dev,
                                     const int32_t* col_dev, const double* val_dev,
                                     bool copy_colval, bool require_sorted) {
  auto* M = new rkmf_matrix();
  M->ctx = ctx;
  M->device = ctx->device;
  M->view.n_rows = n_rows;
  M->view.n_cols = n_cols;
  M->view.nnz = nnz;
  try {
    const bool rp64 = nnz >= (int64_t(1) << 31) - 1;
    M->view.rp64 = rp64;
    // tail padding: the TMA-pipelined SpMV rounds its bulk copies up to 16 B
    const size_t rp_elems = size_t(n_rows + 1 + kRpPad);
    if (rp64) {
      RKMF_CUDA(cudaMalloc(&M->rp, sizeof(int64_t) * rp_elems));
      RKMF_CUDA(cudaMemsetAsync(M->rp, 0, sizeof(int64_t) * rp_elems, ctx->stream));
      RKMF_CUDA(cudaMemcpyAsync(M->rp, rp64_dev, sizeof(int64_t) * size_t(n_rows + 1),
                                cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
      RKMF_CUDA(cudaMalloc(&M->rp, sizeof(int32_t) * rp_elems));
      RKMF_CUDA(cudaMemsetAsync(M->rp, 0, sizeof(int32_t) * rp_elems, ctx->stream));
      rp_narrow_kernel<<<256, 256, 0, ctx->stream>>>(n_rows, rp64_dev,
                                                     static_cast<int32_t*>(M->rp));
      RKMF_CUDA(cudaGetLastError());
      ctx->launches++;
    }
    if (!copy_colval) {  // caller-allocated with kNnzPad elements of padding
      M->col = const_cast<int32_t*>(col_dev);
      M->val = const_cast<double*>(val_dev);
    } else {
      RKMF_CUDA(cudaMalloc(&M->col, sizeof(int32_t) * size_t(nnz + kNnzPad)));
      RKMF_CUDA(cudaMalloc(&M->val, sizeof(double) * size_t(nnz + kNnzPad)));
      RKMF_CUDA(cudaMemsetAsync(M->col, 0, sizeof(int32_t) * size_t(nnz + kNnzPad), ctx->stream));
      RKMF_CUDA(cudaMemsetAsync(M->val, 0, sizeof(double) * size_t(nnz + kNnzPad), ctx->stream));
      if (nnz > 0) {
        RKMF_CUDA(cudaMemcpyAsync(M->col, col_dev, sizeof(int32_t) * size_t(nnz),
                                  cudaMemcpyDeviceToDevice, ctx->stream));
        RKMF_CUDA(cudaMemcpyAsync(M->val, val_dev, sizeof(double) * size_t(nnz),
                                  cudaMemcpyDeviceToDevice, ctx->stream));
      }
    }
    unsigned long long* mx = reinterpret_cast<unsigned long long*>(ctx->scratch.ensure(64));
    RKMF_CUDA(cudaMemsetAsync(mx, 0, 8, ctx->stream));
    tile_nnz_max_kernel<<<256, 256, 0, ctx->stream>>>(n_rows, rp64_dev, mx);
    RKMF_CUDA(cudaGetLastError());
    ctx->launches++;
    unsigned long long hmx = 0;
    RKMF_CUDA(cudaMemcpyAsync(&hmx, mx, 8, cudaMemcpyDeviceToHost, ctx->stream));
    RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
    M->view.max_tile_nnz = int64_t(hmx);
    M->view.padded = true;
    finish_matrix(M, int64_t(hmx), require_sorted);
  } catch (...) {
    if (M->rp) cudaFree(M->rp);
    if (copy_colval && M->col) cudaFree(M->col);
    if (copy_colval && M->val) cudaFree(M->val);
    delete M;
    throw;
  }
  return M;
}


// ============================== C ABI ==============================
extern "C" {

int rkmf_context_create(int device, rkmf_context** out) {
  return guarded(nullptr, [&] {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
      throw Error(RKMF_DEVICE_ERROR, "rkmf_b200: no CUDA device available (no CPU fallback)");
    if (device < 0 || device >= count) param_error("rkmf_b200: invalid device index");
    auto* ctx = new rkmf_context();
    ctx->device = device;
    try {
      RKMF_CUDA(cudaSetDevice(device));
      RKMF_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
      ctx->stream = ctx->own_stream;
      RKMF_CUDA(cudaMalloc(&ctx->st_dev, sizeof(SolveState)));
      RKMF_CUDA(cudaMallocHost(&ctx->st_host, sizeof(SolveState)));
    } catch (...) {
      delete ctx;
      throw;
    }
    *out = ctx;
  });
}

int rkmf_context_destroy(rkmf_context* ctx) {
  if (!ctx) return RKMF_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& qb : ctx->isq) qb.release();
  for (DevBuf* b : {&ctx->redbuf, &ctx->redcl, &ctx->pfin_sk, &ctx->pfin_st, &ctx->z, &ctx->W, &ctx->U, &ctx->Rbar, &ctx->Racc,
                    &ctx->ws, &ctx->u, &ctx->g, &ctx->fhat, &ctx->ref, &ctx->partial,
                    &ctx->qshift, &ctx->qweight, &ctx->qpi, &ctx->qemx, &ctx->scratch, &ctx->gram,
                    &ctx->cl, &ctx->diag})
    b->release();
  for (cudaEvent_t e : ctx->events) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->kpool) cudaEventDestroy(e);
  delete ctx->comm;
  if (ctx->st_dev) cudaFree(ctx->st_dev);
  if (ctx->st_host) cudaFreeHost(ctx->st_host);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return RKMF_OK;
}

const char* rkmf_last_error(const rkmf_context* ctx) {
  return ctx ? ctx->last_error.c_str() : "rkmf_b200: null context";
}

int rkmf_context_set_stream(rkmf_context* ctx, void* s) {
  return guarded(ctx, [&] {
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
  });
}

int64_t rkmf_context_launch_count(const rkmf_context* ctx) { return ctx ? ctx->launches : 0; }

int rkmf_context_set_fused_cycle(rkmf_context* ctx, int enable) {
  if (!ctx) return RKMF_PARAMETER_ERROR;
  ctx->fused_cycle = enable != 0;
  return RKMF_OK;
}

int rkmf_context_kernel_timing(rkmf_context* ctx, int enable) {
  return guarded(ctx, [&] {
    ctx->ktime = enable != 0;
    ctx->kpend.clear();
  });
}

int rkmf_context_kernel_times(rkmf_context* ctx, double* ms, int64_t* launches, int reset) {
  return guarded(ctx, [&] {
    for (int c = 0; c < RKMF_KCLASS_COUNT; ++c) {
      if (ms) ms[c] = ctx->kms[c];
      if (launches) launches[c] = ctx->kcnt[c];
      if (reset) {
        ctx->kms[c] = 0.0;
        ctx->kcnt[c] = 0;
      }
    }
  });
}

// Developer diagnostic (not in the public header; tools/trace_steps.py):
// enable != 0 (re)arms the per-step device timeline of K2/K3/K4 (zeroed),
// enable == 0 copies it out (steps x kTraceSlots stamps) and disarms it.
int rkmf_debug_trace(rkmf_context* ctx, int enable, uint64_t* h_out, int64_t steps) {
  static unsigned long long* buf = nullptr;
  static int64_t cap = 0;
  return guarded(ctx, [&] {
    if (enable) {
      if (steps > cap) {
        if (buf) cudaFree(buf);
        RKMF_CUDA(cudaMalloc(&buf, sizeof(unsigned long long) * steps * rkmf_b200::kTraceSlots));
        cap = steps;
      }
      RKMF_CUDA(cudaMemset(buf, 0, sizeof(unsigned long long) * cap * rkmf_b200::kTraceSlots));
      rkmf_b200::trace_bind_krylov(buf);
      rkmf_b200::trace_bind_spmv_pipe(buf);
    } else {
      RKMF_CUDA(cudaDeviceSynchronize());
      if (h_out && buf)
        RKMF_CUDA(cudaMemcpy(h_out, buf,
                             sizeof(unsigned long long) * std::min(steps, cap) * rkmf_b200::kTraceSlots,
                             cudaMemcpyDeviceToHost));
      rkmf_b200::trace_bind_krylov(nullptr);
      rkmf_b200::trace_bind_spmv_pipe(nullptr);
    }
  });
}

void rkmf_restart_options_default(rkmf_restart_options* o) {  // restart.hpp:20-26
  o->m_r = 20;
  o->tol = 1e-10;
  o->k_max = 100;
  o->budget_total_m = 4000;
  o->divergence_factor = 1e6;
  o->dense_f = RKMF_DENSE_AUTO;
  o->quad_nodes = 0;
  o->diagnostics = 0;
  o->reserved = 0;
}

int rkmf_matrix_create_host(rkmf_context* ctx, int64_t n_rows, int64_t n_cols,
                            const int64_t* h_rp, const int32_t* h_ci, const double* h_v,
                            rkmf_matrix** out) {
  return guarded(ctx, [&] {
    *out = rkmf_b200::create_matrix_host(ctx, n_rows, n_cols, h_rp, h_ci, h_v, true);
  });
}

}  // extern "C"

rkmf_matrix* rkmf_b200::create_matrix_host(rkmf_context* ctx, int64_t n_rows, int64_t n_cols,
                                           const int64_t* h_rp, const int32_t* h_ci,
                                           const double* h_v, bool require_sorted) {
  rkmf_matrix** out = nullptr;
  rkmf_matrix* result = nullptr;
  out = &result;
  {
    set_device(ctx);
    if (n_rows < 0 || n_cols < 0) shape_error("negative dimension");
    if (h_rp[0] != 0) shape_error("row_ptr[0] != 0");
    const int64_t nnz = h_rp[n_rows];
    int64_t* rp_dev = nullptr;
    int32_t* col = nullptr;
    double* val = nullptr;
    RKMF_CUDA(cudaMalloc(&rp_dev, sizeof(int64_t) * size_t(n_rows + 1)));
    RKMF_CUDA(cudaMalloc(&col, sizeof(int32_t) * size_t(nnz + kNnzPad)));
    RKMF_CUDA(cudaMalloc(&val, sizeof(double) * size_t(nnz + kNnzPad)));
    RKMF_CUDA(cudaMemsetAsync(col + nnz, 0, sizeof(int32_t) * size_t(kNnzPad), ctx->stream));
    RKMF_CUDA(cudaMemsetAsync(val + nnz, 0, sizeof(double) * size_t(kNnzPad), ctx->stream));
    RKMF_CUDA(cudaMemcpyAsync(rp_dev, h_rp, sizeof(int64_t) * size_t(n_rows + 1),
                              cudaMemcpyHostToDevice, ctx->stream));
    if (nnz > 0) {
      RKMF_CUDA(cudaMemcpyAsync(col, h_ci, sizeof(int32_t) * size_t(nnz), cudaMemcpyHostToDevice,
                                ctx->stream));
      RKMF_CUDA(cudaMemcpyAsync(val, h_v, sizeof(double) * size_t(nnz), cudaMemcpyHostToDevice,
                                ctx->stream));
    }
    rkmf_matrix* M = nullptr;
    try {
      M = create_from_device_rp64(ctx, n_rows, n_cols, nnz, rp_dev, col, val, false,
                                  require_sorted);
    } catch (...) {
      cudaFree(rp_dev);
      cudaFree(col);
      cudaFree(val);
      throw;
    }
    RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
    RKMF_CUDA(cudaFree(rp_dev));
    *out = M;
  }
  return result;
}

extern "C" {

int rkmf_matrix_create_device(rkmf_context* ctx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                              const int64_t* d_rp, const int32_t* d_ci, const double* d_v,
                              rkmf_matrix** out) {
  return guarded(ctx, [&] {
    set_device(ctx);
    if (n_rows < 0 || n_cols < 0) shape_error("negative dimension");
    *out = create_from_device_rp64(ctx, n_rows, n_cols, nnz, d_rp, d_ci, d_v, true, true);
  });
}

int rkmf_matrix_destroy(rkmf_matrix* M) {
  if (!M) return RKMF_OK;
  // does not touch M->ctx: a matrix may be released after its context
  // (cudaFree synchronises the device itself)
  cudaSetDevice(M->device);
  if (M->halo.send_idx) cudaFree(M->halo.send_idx);
  if (M->halo.sendbuf) cudaFree(M->halo.sendbuf);
  drop_dia(M);
  drop_csr_dict(M);
  if (M->rp) cudaFree(M->rp);
  if (M->col) cudaFree(M->col);
  if (M->val) cudaFree(M->val);
  delete M;
  return RKMF_OK;
}

int rkmf_matrix_dia(rkmf_matrix* M, int enable, int* ndiag) {
  if (!M) return RKMF_PARAMETER_ERROR;
  return guarded(M->ctx, [&] {
    set_device(M->ctx);
    if (enable == 1) {  // the diagonal copy, else the CSR row dictionary
      build_dia(M);
      if (!M->view.ndiag) build_csr_dict(M);
      else drop_csr_dict(M);
    } else if (enable == 0) {  // CSR stream only
      drop_dia(M);
      drop_csr_dict(M);
    }  // other values: query only
    if (ndiag) *ndiag = M->view.ndiag;
  });
}

int rkmf_matrix_dia_dict(rkmf_matrix* M, int enable, int* ntuples) {
  if (!M) return RKMF_PARAMETER_ERROR;
  return guarded(M->ctx, [&] {
    set_device(M->ctx);
    // the diagonal copy's dictionary, or without a copy the CSR row dictionary
    if (enable == 1) {
      if (M->view.ndiag) build_dia_dict(M);
      else build_csr_dict(M);
    } else if (enable == 0) {
      drop_dia_dict(M);
      drop_csr_dict(M);
    }  // other values: query only
    if (ntuples) *ntuples = M->view.ndiag ? M->view.ntup : M->view.rntup;
  });
}

int rkmf_matrix_export(rkmf_context* ctx, const rkmf_matrix* M, int64_t* h_rp, int32_t* h_ci,
                       double* h_v) {
  if (!M) return RKMF_PARAMETER_ERROR;
  return guarded(ctx, [&] {
    set_device(ctx);
    const CsrView& v = M->view;
    const int64_t n = v.n_rows, nnz = v.nnz;
    cudaStream_t st = ctx->stream;
    if (h_rp) {
      if (v.rp64) {
        RKMF_CUDA(cudaMemcpyAsync(h_rp, v.row_ptr, sizeof(int64_t) * size_t(n + 1),
                                  cudaMemcpyDeviceToHost, st));
        RKMF_CUDA(cudaStreamSynchronize(st));
      } else {
        std::vector<int32_t> r32(size_t(n + 1));
        RKMF_CUDA(cudaMemcpyAsync(r32.data(), v.row_ptr, sizeof(int32_t) * size_t(n + 1),
                                  cudaMemcpyDeviceToHost, st));
        RKMF_CUDA(cudaStreamSynchronize(st));
        for (int64_t i = 0; i <= n; ++i) h_rp[i] = r32[size_t(i)];
      }
    }
    if (h_ci && nnz > 0)
      RKMF_CUDA(cudaMemcpyAsync(h_ci, v.col, sizeof(int32_t) * size_t(nnz), cudaMemcpyDeviceToHost, st));
    if (h_v && nnz > 0)
      RKMF_CUDA(cudaMemcpyAsync(h_v, v.val, sizeof(double) * size_t(nnz), cudaMemcpyDeviceToHost, st));
    RKMF_CUDA(cudaStreamSynchronize(st));
  });
}

int rkmf_matrix_load_mtx(rkmf_context* ctx, const char* path, rkmf_matrix** out) {
  return guarded(ctx, [&] {
    set_device(ctx);
    int64_t nr = 0, nc = 0, nnz = 0;
    int64_t* rp = nullptr;
    int32_t* ci = nullptr;
    double* v = nullptr;
    char err[512] = {0};
    const int code = rkmf_mtx_load(path, &nr, &nc, &nnz, &rp, &ci, &v, err, sizeof(err));
    if (code != RKMF_OK) throw Error(code, err);
    try {
      *out = create_matrix_host(ctx, nr, nc, rp, ci, v, true);
    } catch (...) {
      rkmf_host_free(rp);
      rkmf_host_free(ci);
      rkmf_host_free(v);
      throw;
    }
    rkmf_host_free(rp);
    rkmf_host_free(ci);
    rkmf_host_free(v);
  });
}

int rkmf_matrix_save_mtx(rkmf_context* ctx, const rkmf_matrix* M, const char* path) {
  if (!M) return RKMF_PARAMETER_ERROR;
  return guarded(ctx, [&] {
    if (M->partitioned) param_error("save_matrix_market: partitioned matrices hold local rows only");
    const int64_t n = M->view.n_rows, nnz = M->view.nnz;
    std::vector<int64_t> rp(size_t(n + 1));
    std::vector<int32_t> ci(size_t(std::max<int64_t>(nnz, 1)));
    std::vector<double> v(size_t(std::max<int64_t>(nnz, 1)));
    const int code = rkmf_matrix_export(ctx, M, rp.data(), ci.data(), v.data());
    if (code != RKMF_OK) throw Error(code, ctx->last_error);
    char err[512] = {0};
    const int c2 = rkmf_mtx_save(path, n, M->view.n_cols, rp.data(), ci.data(), v.data(), err,
                                 sizeof(err));
    if (c2 != RKMF_OK) throw Error(c2, err);
  });
}

__global__ void rp_widen_kernel(int64_t n, const int32_t* __restrict__ src, int64_t* dst) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

int rkmf_matrix_rp64(rkmf_matrix* M, int enable, int* is64) {
  if (!M) return RKMF_PARAMETER_ERROR;
  return guarded(M->ctx, [&] {
    set_device(M->ctx);
    if (enable && !M->view.rp64) {
      const int64_t n = M->view.n_rows;
      const size_t elems = size_t(n + 1 + kRpPad);
      int64_t* rp = nullptr;
      RKMF_CUDA(cudaMalloc(&rp, sizeof(int64_t) * elems));
      cudaStream_t st = M->ctx->stream;
      RKMF_CUDA(cudaMemsetAsync(rp, 0, sizeof(int64_t) * elems, st));
      rp_widen_kernel<<<256, 256, 0, st>>>(n, static_cast<const int32_t*>(M->rp), rp);
      RKMF_CUDA(cudaGetLastError());
      RKMF_CUDA(cudaStreamSynchronize(st));
      RKMF_CUDA(cudaFree(M->rp));
      M->rp = rp;
      M->view.row_ptr = rp;
      M->view.rp64 = true;
      M->ctx->launches++;
      // the point is to run the int64 row-pointer kernels: the CSR stream,
      // not its row dictionary
      drop_csr_dict(M);
    }
    if (is64) *is64 = M->view.rp64 ? 1 : 0;
  });
}

int rkmf_matrix_info(const rkmf_matrix* M, int64_t* n_rows, int64_t* n_cols, int64_t* nnz,
                     double* norm1) {
  if (!M) return RKMF_PARAMETER_ERROR;
  if (n_rows) *n_rows = M->view.n_rows;
  if (n_cols) *n_cols = M->view.n_cols;
  if (nnz) *nnz = M->view.nnz;
  if (norm1) *norm1 = M->norm1;
  return RKMF_OK;
}

int rkmf_sketch_create(rkmf_context* ctx, int64_t d, int64_t n, int64_t zeta, uint64_t seed,
                       rkmf_sketch** out) {
  return rkmf_sketch_create_partitioned(ctx, d, n, zeta, seed, 0, n, out);
}

int rkmf_sketch_create_partitioned(rkmf_context* ctx, int64_t d, int64_t n_global, int64_t zeta,
                                   uint64_t seed, int64_t col_begin, int64_t n,
                                   rkmf_sketch** out) {
  return guarded(ctx, [&] {
    set_device(ctx);
    if (zeta < 1) param_error("sketch: zeta must be >= 1");  // sketch.cpp:14-16
    if (zeta > d) param_error("sketch: zeta must not exceed d");
    if (d > n_global) param_error("sketch: d must not exceed n");
    if (col_begin < 0 || n < 0 || col_begin + n > n_global)
      shape_error("sketch: column range outside [0, n)");
    auto* S = new rkmf_sketch();
    S->ctx = ctx;
    S->device = ctx->device;
    S->d = d;
    S->n = n;
    S->zeta = zeta;
    S->seed = seed;
    S->n_global = n_global;
    S->col_begin = col_begin;
    S->scale = 1.0 / std::sqrt(double(zeta));  // sketch.cpp:23
    try {
      const int64_t tiles = (n + kTileRows - 1) / kTileRows;
      const int64_t off_stride = tile_off_stride(d);
      RKMF_CUDA(cudaMalloc(&S->rows, sizeof(uint16_t) * size_t(std::max<int64_t>(n * zeta, 1))));
      RKMF_CUDA(cudaMalloc(&S->signs, size_t(std::max<int64_t>(n * zeta, 1))));
      launch_sketch_generate(d, n, col_begin, zeta, seed, S->rows, S->signs, ctx->stream);
      // one allocation for the tile layout (header | entries), so a single L2
      // access-policy window can keep it resident across steps
      S->ent_stride = sketch_tiles_stride(d, n, zeta, S->rows, ctx->stream);
      const size_t ob = round_up(int64_t(sizeof(uint16_t)) * std::max<int64_t>(tiles * off_stride, 1), 256);
      const size_t eb = size_t(std::max<int64_t>(tiles * S->ent_stride, 16)) + 16;
      void* tl = nullptr;
      RKMF_CUDA(cudaMalloc(&tl, ob + eb));
      S->tile_off = static_cast<uint16_t*>(tl);
      S->tile_ent = static_cast<uint8_t*>(tl) + ob;
      S->layout_bytes = ob + eb;
      launch_sketch_tiles(d, n, zeta, S->rows, S->signs, S->tile_off, S->tile_ent, S->ent_stride,
                          ctx->stream);
      ctx->launches += 1;
      ctx->launches += 2;
      RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      if (S->rows) cudaFree(S->rows);
      if (S->signs) cudaFree(S->signs);
      if (S->tile_off) cudaFree(S->tile_off);
      delete S;
      throw;
    }
    *out = S;
  });
}

int rkmf_sketch_destroy(rkmf_sketch* S) {
  if (!S) return RKMF_OK;
  cudaSetDevice(S->device);
  cudaFree(S->rows);
  cudaFree(S->signs);
  cudaFree(S->tile_off);  // also holds tile_ent
  delete S;
  return RKMF_OK;
}

int rkmf_sketch_set_scale(rkmf_sketch* S, double scale) {
  if (!S) return RKMF_PARAMETER_ERROR;
  S->scale = scale;
  return RKMF_OK;
}

int rkmf_sketch_layout_info(const rkmf_sketch* S, int64_t* header_bytes, int64_t* entry_bytes) {
  if (!S) return RKMF_PARAMETER_ERROR;
  if (header_bytes) *header_bytes = int64_t(sizeof(uint16_t)) * tile_off_stride(S->d);
  if (entry_bytes) *entry_bytes = S->ent_stride;
  return RKMF_OK;
}

int rkmf_sketch_export(rkmf_context* ctx, const rkmf_sketch* S, int64_t* h_rows, int8_t* h_signs,
                       double* h_scale) {
  return guarded(ctx, [&] {
    set_device(ctx);
    const int64_t cnt = S->n * S->zeta;
    if (h_rows && cnt > 0) {
      DevBuf tmp;
      tmp.ensure(sizeof(int64_t) * size_t(cnt));
      launch_sketch_export(cnt, S->rows, S->signs, tmp.as<int64_t>(), ctx->stream);
      ctx->launches++;
      RKMF_CUDA(cudaMemcpyAsync(h_rows, tmp.p, sizeof(int64_t) * size_t(cnt),
                                cudaMemcpyDeviceToHost, ctx->stream));
      RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
      tmp.release();
    }
    if (h_signs && cnt > 0) {
      RKMF_CUDA(cudaMemcpyAsync(h_signs, S->signs, size_t(cnt), cudaMemcpyDeviceToHost, ctx->stream));
      RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    if (h_scale) *h_scale = S->scale;
  });
}

int rkmf_spmv(rkmf_context* ctx, const rkmf_matrix* A, const double* d_x, double* d_y) {
  return guarded(ctx, [&] {
    set_device(ctx);
    DetRed none;
    launch_spmv_sketch(&A->view, nullptr, 0, d_x, nullptr, d_y, nullptr, 0, 0, none,
                       ctx->stream);
    ctx->launches++;
    RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int rkmf_sketch_apply(rkmf_context* ctx, const rkmf_sketch* S, const double* d_x, double* d_y) {
  return guarded(ctx, [&] {
    set_device(ctx);
    const SketchView sv = S->view();
    DetRed& red = ctx->red_start(S->d);
    launch_spmv_sketch(nullptr, &sv, 2, d_x, nullptr, nullptr, nullptr, 0, 0, red, ctx->stream);
    launch_det_finish(red, S->d, d_y, ctx->stream);
    ctx->launches += 2;
    RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int rkmf_spmv_sketch(rkmf_context* ctx, const rkmf_matrix* A, const rkmf_sketch* S,
                     const double* d_x, double* d_z, double* d_p) {
  return guarded(ctx, [&] {
    set_device(ctx);
    if (S->n != A->view.n_rows) shape_error("spmv_sketch: sketch width mismatch");
    const SketchView sv = S->view();
    DetRed& red = ctx->red_sketch(S->d);
    launch_spmv_sketch(&A->view, &sv, 1, d_x, nullptr, d_z, nullptr, 0, 0, red, ctx->stream);
    launch_det_finish(red, S->d, d_p, ctx->stream);
    ctx->launches += 2;
    RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

bool flush_l2_between() {  // RKMF_BENCH_FLUSH=1: kernel_bench flushes L2 between launches
  const char* e = knob_env("RKMF_BENCH_FLUSH");
  return e && e[0] == '1';
}

int rkmf_kernel_bench(rkmf_context* ctx, const rkmf_matrix* A, const rkmf_sketch* S, int32_t mode,
                      const double* d_x, double* d_z, double* d_p, int32_t reps, double* avg_ms) {
  return guarded(ctx, [&] {
    set_device(ctx);
    if (mode < 0 || mode > 2 || reps < 1) param_error("kernel_bench: bad mode or reps");
    if (mode != 0 && (!S || S->n != A->view.n_rows))
      shape_error("kernel_bench: sketch width mismatch");
    SketchView sv{};
    if (S) sv = S->view();
    const SketchView* svp = mode == 0 ? nullptr : &sv;
    const int grid = spmv_sketch_grid(mode == 2 ? nullptr : &A->view, svp, mode);
    DetRed none;
    DetRed& red = mode == 0 ? none : ctx->red_sketch(S->d);
    auto launch = [&] {
      launch_spmv_sketch(mode == 2 ? nullptr : &A->view, svp, mode, d_x, nullptr, d_z, nullptr,
                         0, grid, red, ctx->stream);
    };
    launch();  // warm-up
    if (flush_l2_between()) {  // cold-L2 variant: a 256 MB write between timed launches
      DevBuf junk;
      junk.ensure(size_t(256) << 20);
      double tot = 0.0;
      for (int i = 0; i < reps; ++i) {
        RKMF_CUDA(cudaMemsetAsync(junk.p, i & 0xff, size_t(256) << 20, ctx->stream));
        RKMF_CUDA(cudaEventRecord(ctx->event(0), ctx->stream));
        launch();
        RKMF_CUDA(cudaEventRecord(ctx->event(1), ctx->stream));
        RKMF_CUDA(cudaEventSynchronize(ctx->event(1)));
        float ms = 0.f;
        RKMF_CUDA(cudaEventElapsedTime(&ms, ctx->event(0), ctx->event(1)));
        tot += ms;
      }
      junk.release();
      *avg_ms = tot / reps;
    } else {
      RKMF_CUDA(cudaEventRecord(ctx->event(0), ctx->stream));
      for (int i = 0; i < reps; ++i) launch();
      RKMF_CUDA(cudaEventRecord(ctx->event(1), ctx->stream));
      RKMF_CUDA(cudaEventSynchronize(ctx->event(1)));
      float ms = 0.f;
      RKMF_CUDA(cudaEventElapsedTime(&ms, ctx->event(0), ctx->event(1)));
      *avg_ms = double(ms) / reps;
    }
    ctx->launches += reps + 1;
    if (mode != 0) {  // the last launch's sketch as a plain d-vector
      launch_det_finish(red, S->d, d_p, ctx->stream);
      ctx->launches++;
      RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  });
}

int rkmf_randomized_arnoldi(rkmf_context* ctx, const rkmf_matrix* A, const rkmf_sketch* S,
                            const double* d_b, int64_t m, double* d_W, int64_t ldw, double* d_U,
                            double* h_Rbar, double* start_norm, int64_t* mk,
                            int64_t* breakdown_at, int64_t* counters) {
  return guarded(ctx, [&] {
    set_device(ctx);
    check_builder_args(A, S, m);
    const int64_t n = A->view.n_rows;
    if (ldw < n) param_error("randomized_arnoldi: ldw < n");
    SolveBuffers b = prepare(ctx, n, A->view.n_cols, A->n_rows_global(), S->d, m);
    copy_in(ctx, b.W, d_b, n, true);
    start_sketch(ctx, S, b);
    launch_start_init_m(b.d, ctx->start_sum.part, ctx->start_sum.groups, b.U, ctx->st_dev, true,
                        int(m), ctx->stream);
    ctx->launches++;
    ctx->sync_state();
    if (ctx->st_host->zero_start)  // basis.cpp:105-106
      param_error("randomized_arnoldi: zero start vector after sketching");
    run_steps(ctx, A, S, b, 1e-14 * A->norm1, false);
    launch_scale_copy(n, b.W, b.W, ctx->st_dev, ctx->stream);  // W[:,0] = b / alpha
    ctx->launches++;
    ctx->sync_state();
    const SolveState& h = *ctx->st_host;
    const int64_t kept = h.stopped;
    const bool next = h.breakdown == 0;
    const int64_t cols = next ? m + 1 : kept;
    RKMF_CUDA(cudaMemcpy2DAsync(d_W, sizeof(double) * size_t(ldw), b.W, sizeof(double) * size_t(b.ldw),
                                sizeof(double) * size_t(n), size_t(cols), cudaMemcpyDeviceToDevice,
                                ctx->stream));
    RKMF_CUDA(cudaMemcpyAsync(d_U, b.U, sizeof(double) * size_t(S->d) * size_t(cols),
                              cudaMemcpyDeviceToDevice, ctx->stream));
    RKMF_CUDA(cudaMemcpyAsync(h_Rbar, b.Rbar, sizeof(double) * size_t(b.ldr) * size_t(m),
                              cudaMemcpyDeviceToHost, ctx->stream));
    RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
    *start_norm = h.alpha_k;
    *mk = kept;
    *breakdown_at = h.breakdown;
    if (counters) {  // types.hpp:57-75, cost formulas of test_basis.cpp:230-254
      counters[0] = kept;
      counters[1] = 0;
      counters[2] = kept * (kept + 1) / 2;
      counters[3] = next ? m : kept - 1;
      counters[4] = next ? m + 1 : kept;
    }
  });
}

int rkmf_restarted_krylov(rkmf_context* ctx, const rkmf_matrix* A, const rkmf_sketch* S,
                          const double* b_in, int b_on_device, int32_t fn_kind, double fn_t,
                          const rkmf_restart_options* opts_in, double* f_out, int f_on_device,
                          const double* reference, rkmf_restart_result* res,
                          rkmf_cycle_record* records, int64_t records_cap) {
  return guarded(ctx, [&] {
    set_device(ctx);
    rkmf_restart_options opts;
    if (opts_in) opts = *opts_in;
    else rkmf_restart_options_default(&opts);
    // restart.cpp:33-37
    if (opts.m_r < 1) param_error("restart: m_r must be >= 1");
    if (opts.k_max < 1) param_error("restart: k_max must be >= 1");
    if (!(opts.tol > 0.0)) param_error("restart: tol must be > 0");
    if (opts.budget_total_m < opts.m_r) param_error("restart: total-m budget below one cycle");
    if (fn_kind != RKMF_FN_EXP_NEG && fn_kind != RKMF_FN_INV_SQRT)
      param_error("funm: unknown FunctionSpec kind");
    if (fn_kind == RKMF_FN_EXP_NEG && !(fn_t >= 0.0)) param_error("FunctionSpec: t must be >= 0");
    const bool classical = S == nullptr;  // restart.cpp:53-55: arnoldi vs randomized_arnoldi
    int dense = opts.dense_f;
    if (dense == RKMF_DENSE_AUTO) dense = fn_kind == RKMF_FN_EXP_NEG ? RKMF_DENSE_FULL : RKMF_DENSE_QUADRATURE;
    if (dense == RKMF_DENSE_FULL && fn_kind != RKMF_FN_EXP_NEG)
      param_error("rkmf_b200: FULL dense f is implemented for exp_neg only");
    const int64_t n = A->view.n_rows;  // local rows when partitioned
    const int64_t m_eff = std::min(opts.m_r, A->n_rows_global());  // restart.cpp:38
    check_builder_args(A, S, m_eff);
    std::memset(res, 0, sizeof(*res));
    ctx->kpend.clear();

    cudaStream_t st = ctx->stream;
    SolveBuffers bb = prepare(ctx, n, A->view.n_cols, A->n_rows_global(), classical ? 1 : S->d,
                              m_eff);
    double* cl = nullptr;
    if (classical) {
      const size_t cnt = size_t(2 * bb.ldr + 2 + bb.ldr * m_eff);
      cl = static_cast<double*>(ctx->cl.ensure(sizeof(double) * cnt));
      RKMF_CUDA(cudaMemsetAsync(cl, 0, sizeof(double) * cnt, ctx->stream));
    }
    double* g = static_cast<double*>(ctx->g.ensure(sizeof(double) * size_t(m_eff)));
    double* fhat = f_on_device ? f_out : static_cast<double*>(ctx->fhat.ensure(sizeof(double) * size_t(std::max<int64_t>(n, 1))));
    RKMF_CUDA(cudaMemsetAsync(fhat, 0, sizeof(double) * size_t(n), st));
    const double* ref_dev = nullptr;
    double ref_norm = 0.0;
    if (reference) {
      std::vector<double> hr;
      if (b_on_device) {
        hr.resize(size_t(n));
        RKMF_CUDA(cudaMemcpyAsync(hr.data(), reference, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, st));
        RKMF_CUDA(cudaStreamSynchronize(st));
        ref_dev = reference;
        ref_norm = host_norm(hr.data(), n);
      } else {
        double* rd = static_cast<double*>(ctx->ref.ensure(sizeof(double) * size_t(n)));
        copy_in(ctx, rd, reference, n, false);
        ref_dev = rd;
        ref_norm = host_norm(reference, n);
      }
      if (ctx->comm && ctx->nranks > 1) {  // global ||reference||
        double* sc = reinterpret_cast<double*>(static_cast<char*>(ctx->scratch.ensure(64)) + 32);
        double r2 = ref_norm * ref_norm;
        RKMF_CUDA(cudaMemcpyAsync(sc, &r2, sizeof(double), cudaMemcpyHostToDevice, st));
        comm_allreduce_sum(ctx, sc, 1);
        RKMF_CUDA(cudaMemcpyAsync(&r2, sc, sizeof(double), cudaMemcpyDeviceToHost, st));
        RKMF_CUDA(cudaStreamSynchronize(st));
        ref_norm = std::sqrt(r2);
      }
    }
    copy_in(ctx, bb.W, b_in, n, b_on_device != 0);  // start = b (restart.cpp:45)

    // dense-f state
    const int64_t Ncap = std::min<int64_t>(opts.budget_total_m, opts.k_max * m_eff);
    // R_accum lives in the context's buffer (capacity ctx->racc_cap, kept
    // across solves so a solve does not allocate, free and synchronise as
    // R_accum grows); the stripes a cycle adds are zeroed on the stream
    int64_t ldR = 0, used = 0;
    double* Racc = nullptr;
    auto ensure_racc = [&](int64_t N) {
      if (N > ctx->racc_cap) {  // grow geometrically, up to the budget
        int64_t newld = std::min<int64_t>(Ncap, std::max<int64_t>(N, 2 * ctx->racc_cap));
        newld = std::max(newld, N);
        DevBuf nb;
        nb.ensure(sizeof(double) * size_t(newld) * size_t(newld));
        if (Racc && used > 0)
          RKMF_CUDA(cudaMemcpy2DAsync(nb.p, sizeof(double) * size_t(newld), Racc,
                                      sizeof(double) * size_t(ldR), sizeof(double) * size_t(used),
                                      size_t(used), cudaMemcpyDeviceToDevice, st));
        RKMF_CUDA(cudaStreamSynchronize(st));
        ctx->Racc.release();
        ctx->Racc = nb;
        nb.p = nullptr;
        ctx->racc_cap = newld;
        Racc = nullptr;
      }
      if (!Racc) {
        Racc = ctx->Racc.as<double>();
        ldR = ctx->racc_cap;
      }
      if (N > used) {  // rows [used, N) of columns [0, N), then columns [used, N) above them
        RKMF_CUDA(cudaMemset2DAsync(Racc + used, sizeof(double) * size_t(ldR), 0,
                                    sizeof(double) * size_t(N - used), size_t(N), st));
        if (used > 0)
          RKMF_CUDA(cudaMemset2DAsync(Racc + used * ldR, sizeof(double) * size_t(ldR), 0,
                                      sizeof(double) * size_t(used), size_t(N - used), st));
        used = N;
      }
    };
    QuadState q{};
    double* partial = nullptr;
    // InvSqrt: quad_nodes > 0 fixes the node count on the interval
    // [0.5 ln(||A||_1 1e-14) - 37, 0.5 ln ||A||_1 + 37]; the default (0) designs
    // the nodes from the Ritz values with node doubling (adaptive below)
    const bool isq_adaptive = fn_kind == RKMF_FN_INV_SQRT && opts.quad_nodes <= 0;
    QuadSet qa, qb;
    qa.buf = &ctx->isq[0];
    qb.buf = &ctx->isq[1];
    double s_lmin = std::numeric_limits<double>::infinity(), s_lmax = 0.0, s_th = 0.0;
    int64_t isq_nodes = 0;
    if (dense == RKMF_DENSE_QUADRATURE && fn_kind == RKMF_FN_INV_SQRT && !isq_adaptive) {
      q.nq = opts.quad_nodes;
      q.shift = static_cast<double*>(ctx->qshift.ensure(sizeof(double) * size_t(q.nq)));
      q.weight = static_cast<double*>(ctx->qweight.ensure(sizeof(double) * size_t(q.nq)));
      q.pi = static_cast<double*>(ctx->qpi.ensure(sizeof(double) * size_t(q.nq)));
      q.emx = static_cast<double*>(ctx->qemx.ensure(sizeof(double) * size_t(q.nq)));
      partial = static_cast<double*>(ctx->partial.ensure(sizeof(double) * size_t(q.nq) * size_t(m_eff)));
      // trapezoid nodes u in [0.5 ln(||A|| * 1e-14) - 37, 0.5 ln(||A||) + 37]
      const double an = std::max(A->norm1, 1e-300);
      const double u0 = 0.5 * std::log(an * 1e-14) - 37.0, u1 = 0.5 * std::log(an) + 37.0;
      const double h = (u1 - u0) / double(q.nq);
      std::vector<double> hs(size_t(q.nq)), hw(size_t(q.nq)), ones(size_t(q.nq), 1.0);
      for (int i = 0; i < q.nq; ++i) {
        const double u = u0 + (double(i) + 0.5) * h;
        hs[size_t(i)] = std::exp(2.0 * u);
        hw[size_t(i)] = (2.0 / M_PI) * h * std::exp(u);
      }
      RKMF_CUDA(cudaMemcpyAsync(q.shift, hs.data(), sizeof(double) * hs.size(), cudaMemcpyHostToDevice, st));
      RKMF_CUDA(cudaMemcpyAsync(q.weight, hw.data(), sizeof(double) * hw.size(), cudaMemcpyHostToDevice, st));
      RKMF_CUDA(cudaMemcpyAsync(q.pi, ones.data(), sizeof(double) * ones.size(), cudaMemcpyHostToDevice, st));
      RKMF_CUDA(cudaStreamSynchronize(st));
    }

    const double tol_break = 1e-14 * A->norm1;  // basis.cpp:118
    ExpContour contour;
    bool exp_fallback = false;
    std::vector<double> ritz_re, ritz_im;  // t-scaled Ritz values of all cycles so far
    std::vector<int64_t> cyc_M, cyc_mk;     // R_accum block offset and size per cycle
    int64_t M = 0;
    double first_update = -1.0;
    long long matvecs = 0, dot_n = 0, dot_d = 0, updates = 0, peak = 0;
    RKMF_CUDA(cudaEventRecord(ctx->event(0), st));
    if (!classical) start_sketch(ctx, S, bb);
    struct CycleEv { size_t e0, e1, e2, e3; };
    size_t next_ev = 1;
    std::vector<CycleEv> evs;
    std::vector<rkmf_cycle_record> recs;
    for (int64_t k = 1; k <= opts.k_max; ++k) {
      if (M + m_eff > opts.budget_total_m) break;  // restart.cpp:50
      const size_t base = next_ev;
      next_ev += 4;
      CycleEv ce{base, base + 1, base + 2, base + 3};
      RKMF_CUDA(cudaEventRecord(ctx->event(ce.e0), st));
      if (classical) {
        start_classical(ctx, bb, cl, k == 1);
      } else {
        ctx->timed(5, [&] {
          launch_start_init_m(bb.d, ctx->start_sum.part, ctx->start_sum.groups, bb.U, ctx->st_dev,
                              k == 1, int(m_eff), st);
        });
        ctx->launches++;
      }
      if (k == 1) {
        ctx->sync_state();
        if (ctx->st_host->zero_start)
          param_error(classical ? "arnoldi: zero start vector"
                                : "randomized_arnoldi: zero start vector after sketching");
      }
      if (classical) run_steps_classical(ctx, A, bb, tol_break, true, cl);
      else run_steps(ctx, A, S, bb, tol_break, true);
      // diagnostics: Gram of W_m before final_update overwrites column 0
      bool diag_ok = false;
      double* Gd = nullptr;
      if (opts.diagnostics) {
        Gd = static_cast<double*>(ctx->diag.ensure(sizeof(double) * gram_scratch_doubles(n, int(m_eff))));
        diag_ok = launch_gram(n, int(m_eff), bb.ldw, bb.W, ctx->st_dev, Gd, st);
        if (diag_ok) {
          ctx->launches += 2;
          comm_allreduce_sum(ctx, Gd, size_t(m_eff) * size_t(m_eff));
        }
      }
      RKMF_CUDA(cudaEventRecord(ctx->event(ce.e1), st));
      // ---- dense f ----
      // FULL exp(-t R_accum) e1 from the appended R_accum (restart.cpp:61-78)
      auto full_expneg = [&] {
        const int64_t N = M + m_eff;
        ctx->timed(3, [&] { launch_dense_norm1(Racc, ldR, N, &ctx->st_dev->rnorm1, st); });
        ctx->launches++;
        ctx->sync_state();
        const double xn = std::fabs(fn_t) * ctx->st_host->rnorm1;
        int s = 0;
        if (xn > 1.0) s = std::min(64, int(std::ceil(std::log2(xn))));
        double* ws = static_cast<double*>(ctx->ws.ensure(sizeof(double) * 6 * size_t(N) * size_t(N)));
        double* u = static_cast<double*>(ctx->u.ensure(sizeof(double) * size_t(N)));
        int64_t nl = 0;
        ctx->timed(3, [&] {
          dense_expneg_e1(Racc, ldR, N, fn_t, s, ws, u, st, &nl);
          launch_make_g(u, M, int(m_eff), g, ctx->st_dev, st);
        });
        ctx->launches += nl + 1;
      };
      if (M + m_eff <= Ncap) {  // R_accum (FULL, the exp fallback, rkmf_last_r_accum)
        ensure_racc(M + m_eff);
        ctx->timed(3, [&] { launch_raccum_append(Racc, ldR, M, bb.Rbar, bb.ldr, ctx->st_dev, st); });
        ctx->launches++;
      }
      if (dense == RKMF_DENSE_FULL || exp_fallback) {
        full_expneg();
      } else if (fn_kind == RKMF_FN_INV_SQRT && !isq_adaptive) {
        ctx->timed(3, [&] {
          launch_quad_invsqrt_cycle(bb.Rbar, bb.ldr, int(m_eff), k, &q, g, ctx->st_dev, partial,
                                    st);
        });
        ctx->launches += 2;
      } else if (fn_kind == RKMF_FN_INV_SQRT) {
        // Adaptive restart quadrature for z^{-1/2}. The
        // spectrum of R_accum is the union of the cycles' Ritz values (it is
        // block lower-bidiagonal): each cycle's are checked against the
        // branch cut (-inf, 0] and, when they leave the node design, the
        // nodes are redesigned from all values seen and the earlier cycles are
        // replayed into the new node states (R_accum kept on device). A new
        // design is verified by node doubling: the cycle's g from the set and
        // from the set at half the step must agree to 1e-12, else the finer
        // set is taken and checked in turn.
        ctx->sync_state();
        const int mk = ctx->st_host->stopped;
        std::vector<double> Rh(size_t(bb.ldr) * size_t(m_eff)), wr, wi;
        RKMF_CUDA(cudaMemcpy(Rh.data(), bb.Rbar, sizeof(double) * Rh.size(), cudaMemcpyDeviceToHost));
        ritz_values(Rh, bb.ldr, mk, wr, wi);
        double clo = std::numeric_limits<double>::infinity(), chi = 0.0, cth = 0.0;
        for (size_t i = 0; i < wr.size(); ++i) {
          const double mod = std::hypot(wr[i], wi[i]), th = std::atan2(std::fabs(wi[i]), wr[i]);
          if (!(mod > 0.0) || !std::isfinite(mod) || th > M_PI - 1e-3) {
            char v[96];
            std::snprintf(v, sizeof(v), "%.6g%+.6gi", wr[i], wi[i]);
            numerical_error("inv_sqrt: a Ritz value of the restart compression lies on the branch "
                            "cut (-inf, 0] (cycle " + std::to_string(k) + ": " + v +
                            "): z^{-1/2} is undefined there");
          }
          clo = std::min(clo, mod);
          chi = std::max(chi, mod);
          cth = std::max(cth, th);
        }
        s_lmin = std::min(s_lmin, clo);
        s_lmax = std::max(s_lmax, chi);
        s_th = std::max(s_th, cth);
        if (k > 1 && M + m_eff > Ncap)
          numerical_error("inv_sqrt: R_accum beyond the budget: the quadrature cannot replay");
        // the earlier cycles' blocks of R_accum into a set's node states
        auto replay = [&](QuadSet& s) {
          for (size_t j = 0; j < cyc_M.size(); ++j) {
            double coup = 0.0;
            if (j > 0) {  // R_accum(M_j, M_j - 1) = coupling * alpha (restart.cpp:67)
              RKMF_CUDA(cudaMemcpyAsync(&coup, Racc + (cyc_M[j] - 1) * ldR + cyc_M[j],
                                        sizeof(double), cudaMemcpyDeviceToHost, st));
              RKMF_CUDA(cudaStreamSynchronize(st));
            }
            launch_quad_invsqrt_cycle(Racc + cyc_M[j] * ldR + cyc_M[j], ldR, int(m_eff),
                                      int64_t(j) + 1, &s.q, nullptr, ctx->st_dev, nullptr, st,
                                      int(cyc_mk[j]), coup);
            ctx->launches++;
          }
        };
        auto current = [&](QuadSet& s) {
          launch_quad_invsqrt_cycle(bb.Rbar, bb.ldr, int(m_eff), k, &s.q, s.g, ctx->st_dev,
                                    s.partial, st);
          ctx->launches += 2;
        };
        ctx->timed(3, [&] {
          if (k == 1 || !qa.d.covers(clo, chi, cth)) {
            qa.load(design_invsqrt(s_lmin, s_lmax, s_th), m_eff, st);
            replay(qa);
            current(qa);
            std::vector<double> ga(static_cast<size_t>(mk)), gb(static_cast<size_t>(mk));
            for (;;) {
              qb.load(qa.d.doubled(), m_eff, st);
              replay(qb);
              current(qb);
              RKMF_CUDA(cudaMemcpyAsync(ga.data(), qa.g, sizeof(double) * size_t(mk),
                                        cudaMemcpyDeviceToHost, st));
              RKMF_CUDA(cudaMemcpyAsync(gb.data(), qb.g, sizeof(double) * size_t(mk),
                                        cudaMemcpyDeviceToHost, st));
              RKMF_CUDA(cudaStreamSynchronize(st));
              double dn = 0.0, bn = 0.0;
              for (int i = 0; i < mk; ++i) {
                dn += (ga[size_t(i)] - gb[size_t(i)]) * (ga[size_t(i)] - gb[size_t(i)]);
                bn += gb[size_t(i)] * gb[size_t(i)];
              }
              if (std::sqrt(dn) <= 1e-12 * std::sqrt(bn)) break;  // qa is accurate
              std::swap(qa, qb);  // the finer set, its states advanced through this cycle
              if (qa.d.nq > (1 << 16))
                numerical_error("inv_sqrt: the restart quadrature does not converge under node "
                                "doubling (cycle " + std::to_string(k) + ")");
            }
          } else {
            current(qa);
          }
          RKMF_CUDA(cudaMemcpyAsync(g, qa.g, sizeof(double) * size_t(m_eff), cudaMemcpyDeviceToDevice, st));
        });
        isq_nodes = qa.d.nq;
      } else {
        // ExpNeg restart quadrature. The contour is designed from the Ritz
        // values seen so far; when a cycle's Ritz values leave it, it is
        // redesigned from all of them and the node states are rebuilt by
        // replaying the earlier cycles' blocks of R_accum (kept on device),
        // O(cycles N_q m^2) once. Only contours that would need > 4096 nodes
        // send the solve to FULL.
        ctx->sync_state();
        const int mk = ctx->st_host->stopped;
        std::vector<double> Rh(size_t(bb.ldr) * size_t(m_eff)), wr, wi;
        RKMF_CUDA(cudaMemcpy(Rh.data(), bb.Rbar, sizeof(double) * Rh.size(), cudaMemcpyDeviceToHost));
        ritz_values(Rh, bb.ldr, mk, wr, wi);
        bool redesign = k == 1;
        for (size_t i = 0; i < wr.size(); ++i) {
          wr[i] *= fn_t;
          wi[i] *= fn_t;
          if (k > 1 && !contour.inside(wr[i], wi[i])) redesign = true;
          ritz_re.push_back(wr[i]);
          ritz_im.push_back(wi[i]);
        }
        if (redesign) {
          contour = design_exp_contour(ritz_re, ritz_im);
          if (contour.K > 4096) exp_fallback = true;
        }
        if (redesign && !exp_fallback) {
          std::vector<double> hs, hw;
          exp_contour_nodes(contour, fn_t, hs, hw);
          q.nq = contour.K + 1;
          q.shift = static_cast<double*>(ctx->qshift.ensure(sizeof(double) * hs.size()));
          q.weight = static_cast<double*>(ctx->qweight.ensure(sizeof(double) * hw.size()));
          q.pi = static_cast<double*>(ctx->qpi.ensure(sizeof(double) * hs.size()));
          q.emx = static_cast<double*>(ctx->qemx.ensure(sizeof(double) * hs.size()));
          partial = static_cast<double*>(ctx->partial.ensure(sizeof(double) * size_t(q.nq) * size_t(m_eff)));
          std::vector<double> ones(hs.size(), 0.0);
          for (size_t i = 0; i < ones.size(); i += 2) ones[i] = 1.0;
          RKMF_CUDA(cudaMemcpyAsync(q.shift, hs.data(), sizeof(double) * hs.size(), cudaMemcpyHostToDevice, st));
          RKMF_CUDA(cudaMemcpyAsync(q.weight, hw.data(), sizeof(double) * hw.size(), cudaMemcpyHostToDevice, st));
          RKMF_CUDA(cudaMemcpyAsync(q.pi, ones.data(), sizeof(double) * ones.size(), cudaMemcpyHostToDevice, st));
          for (size_t j = 0; j < cyc_M.size(); ++j) {  // replay cycles 1..k-1
            double coup = 0.0;
            if (j > 0) {  // R_accum(M_j, M_j - 1) = coupling * alpha (restart.cpp:67)
              RKMF_CUDA(cudaMemcpyAsync(&coup, Racc + (cyc_M[j] - 1) * ldR + cyc_M[j],
                                        sizeof(double), cudaMemcpyDeviceToHost, st));
              RKMF_CUDA(cudaStreamSynchronize(st));
            }
            launch_quad_expneg_cycle(Racc + cyc_M[j] * ldR + cyc_M[j], ldR, int(m_eff),
                                     int64_t(j) + 1, &q, g, ctx->st_dev, partial, st,
                                     int(cyc_mk[j]), coup);
            ctx->launches++;
          }
        }
        if (exp_fallback) {
          full_expneg();
        } else {
          ctx->timed(3, [&] {
            launch_quad_expneg_cycle(bb.Rbar, bb.ldr, int(m_eff), k, &q, g, ctx->st_dev, partial,
                                     st);
          });
          ctx->launches += 2;
        }
      }
      RKMF_CUDA(cudaEventRecord(ctx->event(ce.e2), st));
      // observer (test-only): the basis block as built and f_hat before K5
      // overwrites column 0 with the next start vector
      std::vector<double> obs_W, obs_f0;
      if (ctx->observer) {
        obs_W.assign(size_t(n) * size_t(m_eff + 1), 0.0);
        obs_f0.assign(size_t(n), 0.0);
        RKMF_CUDA(cudaMemcpy2DAsync(obs_W.data(), sizeof(double) * size_t(n), bb.W,
                                    sizeof(double) * size_t(bb.ldw), sizeof(double) * size_t(n),
                                    size_t(m_eff), cudaMemcpyDeviceToHost, st));
        RKMF_CUDA(cudaMemcpyAsync(obs_f0.data(), fhat, sizeof(double) * size_t(n),
                                  cudaMemcpyDeviceToHost, st));
        RKMF_CUDA(cudaStreamSynchronize(st));
      }
      ctx->timed(4, [&] {
        // classical: the last step left z' and (h2, beta) in rlast
        launch_final_update(n, int(m_eff), bb.ldw, bb.W, bb.z,
                            classical ? cl + 2 * bb.ldr + 2 : bb.Rbar, bb.ldr, g, fhat, ref_dev,
                            ctx->st_dev, ctx->red_update(), st);
      });
      ctx->launches++;
      comm_allreduce_sum(ctx, &ctx->st_dev->yn2, 2);  // global ||y||^2, ||f - ref||^2
      RKMF_CUDA(cudaEventRecord(ctx->event(ce.e3), st));
      ctx->sync_state();
      const SolveState& h = *ctx->st_host;
      const int64_t mk = h.stopped;
      const bool next = h.breakdown == 0;
      if (k == 1) res->alpha = h.alpha1;
      matvecs += mk;
      (classical ? dot_n : dot_d) += mk * (mk + 1) / 2;
      updates += next ? m_eff : mk - 1;
      peak = std::max<long long>(peak, next ? m_eff + 1 : mk);
      if (h.nonfinite || !std::isfinite(h.yn2))  // restart.cpp:82-83
        numerical_error("restart divergence (cycle " + std::to_string(k) + ")");
      const double yn = std::sqrt(h.yn2);
      rkmf_cycle_record rec;
      rec.cycle = k;
      rec.total_m = M + mk;
      rec.total_matvecs = matvecs;
      rec.update_norm = yn;
      rec.error_vs_reference = (reference && ref_norm > 0.0) ? std::sqrt(h.err2) / ref_norm
                                                             : std::numeric_limits<double>::quiet_NaN();
      rec.kappa_W = std::numeric_limits<double>::quiet_NaN();
      rec.leftmost_ritz_re = std::numeric_limits<double>::quiet_NaN();
      if (diag_ok) {  // approximants.cpp:29-47 on the mk kept columns
        std::vector<double> Gh(size_t(m_eff) * size_t(m_eff)), Rh(size_t(bb.ldr) * size_t(m_eff));
        RKMF_CUDA(cudaMemcpy(Gh.data(), Gd, sizeof(double) * Gh.size(), cudaMemcpyDeviceToHost));
        RKMF_CUDA(cudaMemcpy(Rh.data(), bb.Rbar, sizeof(double) * Rh.size(),
                             cudaMemcpyDeviceToHost));
        std::vector<double> Gk(size_t(mk) * size_t(mk));
        for (int64_t i = 0; i < mk; ++i)
          for (int64_t j = 0; j < mk; ++j) Gk[size_t(i * mk + j)] = Gh[size_t(i * m_eff + j)];
        rec.kappa_W = kappa_from_gram(Gk, int(mk));
        rec.leftmost_ritz_re = leftmost_ritz(Rh, bb.ldr, int(mk));
      }
      rec.alpha_dev = k == 1 ? 0.0 : std::fabs(h.alpha_k - 1.0);
      rec.start_norm = h.alpha_k;
      rec.subdiag = h.coupling;
      rec.elapsed_ms = rec.build_ms = rec.funm_ms = 0.0;
      recs.push_back(rec);
      evs.push_back(ce);
      if (first_update < 0.0) first_update = yn;
      else if (yn > opts.divergence_factor * first_update)
        numerical_error("restart divergence (cycle " + std::to_string(k) + ")");
      if (ctx->observer) {  // restart.cpp:91-92
        std::vector<double> fh, Rh;
        fh.resize(size_t(n));
        const int64_t wc = next ? mk + 1 : mk;
        if (next)  // w_m, the next start vector, now in column 0
          RKMF_CUDA(cudaMemcpy(obs_W.data() + size_t(mk) * size_t(n), bb.W,
                               sizeof(double) * size_t(n), cudaMemcpyDeviceToHost));
        RKMF_CUDA(cudaMemcpy(fh.data(), fhat, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i) {
          obs_W[size_t(i)] /= h.alpha_k;  // column 0 holds the unscaled start
          obs_f0[size_t(i)] = fh[size_t(i)] - obs_f0[size_t(i)];
        }
        const int64_t Mk = M + mk;
        const bool have_R = Racc != nullptr && ldR >= Mk;
        if (have_R) {
          Rh.resize(size_t(Mk) * size_t(Mk));
          RKMF_CUDA(cudaMemcpy2D(Rh.data(), sizeof(double) * size_t(Mk), Racc,
                                 sizeof(double) * size_t(ldR), sizeof(double) * size_t(Mk),
                                 size_t(Mk), cudaMemcpyDeviceToHost));
        }
        rkmf_cycle_info info;
        info.cycle = k;
        info.n = n;
        info.m_k = mk;
        info.w_cols = wc;
        info.W = obs_W.data();
        info.total_m = Mk;
        info.R_accum = have_R ? Rh.data() : nullptr;
        info.update = obs_f0.data();
        info.f_hat = fh.data();
        info.alpha = res->alpha;
        ctx->observer(ctx->observer_user, &info);
      }
      cyc_M.push_back(M);
      cyc_mk.push_back(mk);
      M += mk;
      res->cycles = k;
      res->total_m = M;
      if (yn <= opts.tol || !next) {  // restart.cpp:113-116
        res->converged = 1;
        break;
      }
      if (!classical) start_sketch(ctx, S, bb);  // next cycle's S * start
    }
    const size_t e_end = next_ev;
    RKMF_CUDA(cudaEventRecord(ctx->event(e_end), st));
    if (!f_on_device)
      RKMF_CUDA(cudaMemcpyAsync(f_out, fhat, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, st));
    RKMF_CUDA(cudaStreamSynchronize(st));
    ctx->collect_ktimes();
    float ms = 0.f;
    RKMF_CUDA(cudaEventElapsedTime(&ms, ctx->event(0), ctx->event(e_end)));
    res->solve_ms = ms;
    for (size_t i = 0; i < recs.size(); ++i) {
      float a = 0.f, b2 = 0.f, c = 0.f;
      RKMF_CUDA(cudaEventElapsedTime(&a, ctx->event(evs[i].e0), ctx->event(evs[i].e3)));
      RKMF_CUDA(cudaEventElapsedTime(&b2, ctx->event(evs[i].e0), ctx->event(evs[i].e1)));
      RKMF_CUDA(cudaEventElapsedTime(&c, ctx->event(evs[i].e1), ctx->event(evs[i].e2)));
      recs[i].elapsed_ms = a;
      recs[i].build_ms = b2;
      recs[i].funm_ms = c;
    }
    res->matvecs = matvecs;
    res->dot_n = dot_n;
    res->dot_d = dot_d;
    res->basis_updates = updates;
    res->peak_basis_cols = peak;
    res->n_records = int64_t(recs.size());
    res->quad_nodes = isq_adaptive ? isq_nodes : (q.nq > 0 ? q.nq : 0);
    if (records)
      for (int64_t i = 0; i < std::min<int64_t>(records_cap, res->n_records); ++i) records[i] = recs[size_t(i)];
    ctx->racc_ld = ldR;
    ctx->last_M = (ldR >= M) ? M : 0;
  });
}

int rkmf_context_set_observer(rkmf_context* ctx, rkmf_cycle_observer fn, void* user) {
  return guarded(ctx, [&] {
    ctx->observer = fn;
    ctx->observer_user = user;
  });
}

int rkmf_last_r_accum(rkmf_context* ctx, double* h_R, int64_t n_cap, int64_t* total_m) {
  return guarded(ctx, [&] {
    set_device(ctx);
    const int64_t M = ctx->last_M;
    *total_m = M;
    if (!h_R || M == 0) return;
    if (n_cap < M) param_error("rkmf_last_r_accum: capacity too small");
    RKMF_CUDA(cudaMemcpy2DAsync(h_R, sizeof(double) * size_t(M), ctx->Racc.p,
                                sizeof(double) * size_t(ctx->racc_ld), sizeof(double) * size_t(M),
                                size_t(M), cudaMemcpyDeviceToHost, ctx->stream));
    RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
