// Multi-GPU plumbing: transports, row-partitioned matrices and sketches, the
// per-step halo exchange and the sketch allreduce.
//
// One process per GPU. Rank r owns rows [row_starts[r], row_starts[r+1]) of A,
// the same rows of every basis vector, of z and of f; its sketch is the same
// column range of the global S (bit-identical to make_sketch on n_global).
// Per Krylov step:
//   halo exchange   pack the owned x entries other ranks reference, then one
//                   personalised exchange; the received values land directly
//                   in the halo tail of the x column (W is allocated with
//                   ld >= n_local + n_halo)
//   local K2        SpMV over [owned | halo] columns + local sketch partial
//   allreduce       sum of the d sketch doubles, in place
//   K3              replicated (every rank holds the same p, hence the same r)
//   K4              local
// Per cycle: allreduce of the start sketch (d) and of ||y||^2, ||f-ref||^2 (2).
//
// Transports: NcclTransport (ncclAllReduce, grouped ncclSend/ncclRecv over
// NVLink/NVSwitch) is the product path. HostTransport stages the same
// collectives through pinned host memory into caller callbacks
// (rkmf_host_comm), so an MPI or gloo host stack can drive the partitioned
// solve, and the multi-rank path can be exercised where fewer GPUs than ranks
// exist: its ranks never wait on each other inside a kernel.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "engine_types.cuh"

extern "C" int rkmf_partition_halo(int32_t nranks, int32_t rank, const int64_t* row_starts,
                                   const int64_t* row_ptr_local, const int32_t* col_global,
                                   int64_t* n_halo, int64_t* halo_global, int64_t* recv_counts,
                                   int32_t* col_local);

namespace rkmf_b200 {

#define RKMF_NCCL(call)                                                                   \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      throw Error(RKMF_DEVICE_ERROR, std::string("NCCL error: ") + ncclGetErrorString(r_) + \
                                         " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

namespace {

class NcclTransport final : public Transport {
 public:
  int kind() const override { return 1; }
  int comm_size() const override {
    int n = 0;
    RKMF_NCCL(ncclCommCount(comm_, &n));
    return n;
  }
  NcclTransport(int nranks, int rank, const ncclUniqueId& id) : me_(rank), p_(nranks) {
    RKMF_NCCL(ncclCommInitRank(&comm_, nranks, id, rank));
  }
  ~NcclTransport() override {
    if (comm_) ncclCommDestroy(comm_);
  }
  void allreduce(double* dev, size_t count, bool max, cudaStream_t st) override {
    RKMF_NCCL(ncclAllReduce(dev, dev, count, ncclFloat64, max ? ncclMax : ncclSum, comm_, st));
  }
  void alltoallv(const void* send, const std::vector<int64_t>& soff,
                 const std::vector<int64_t>& scnt, void* recv, const std::vector<int64_t>& roff,
                 const std::vector<int64_t>& rcnt, bool is_double, cudaStream_t st) override {
    const ncclDataType_t ty = is_double ? ncclFloat64 : ncclInt64;
    const char* s = static_cast<const char*>(send);
    char* r = static_cast<char*>(recv);
    RKMF_NCCL(ncclGroupStart());
    for (int q = 0; q < p_; ++q) {
      if (q == me_) continue;
      if (scnt[q] > 0) RKMF_NCCL(ncclSend(s + 8 * soff[q], size_t(scnt[q]), ty, q, comm_, st));
      if (rcnt[q] > 0) RKMF_NCCL(ncclRecv(r + 8 * roff[q], size_t(rcnt[q]), ty, q, comm_, st));
    }
    RKMF_NCCL(ncclGroupEnd());
  }

 private:
  ncclComm_t comm_ = nullptr;
  int me_, p_;
};

class HostTransport final : public Transport {
 public:
  int kind() const override { return 2; }
  int comm_size() const override { return p_; }
  HostTransport(int nranks, int rank, const rkmf_host_comm& cb) : me_(rank), p_(nranks), cb_(cb) {}
  ~HostTransport() override {
    if (stage_) cudaFreeHost(stage_);
  }
  void allreduce(double* dev, size_t count, bool max, cudaStream_t st) override {
    double* h = static_cast<double*>(host(8 * count));
    RKMF_CUDA(cudaMemcpyAsync(h, dev, 8 * count, cudaMemcpyDeviceToHost, st));
    RKMF_CUDA(cudaStreamSynchronize(st));
    const int rc = max ? cb_.allreduce_max_f64(cb_.user, h, int64_t(count))
                       : cb_.allreduce_sum_f64(cb_.user, h, int64_t(count));
    if (rc != 0) throw Error(RKMF_DEVICE_ERROR, "host comm: allreduce callback failed");
    RKMF_CUDA(cudaMemcpyAsync(dev, h, 8 * count, cudaMemcpyHostToDevice, st));
    RKMF_CUDA(cudaStreamSynchronize(st));  // h is reused by the next call
  }
  void alltoallv(const void* send, const std::vector<int64_t>& soff,
                 const std::vector<int64_t>& scnt, void* recv, const std::vector<int64_t>& roff,
                 const std::vector<int64_t>& rcnt, bool /*is_double*/, cudaStream_t st) override {
    // the callback sees contiguous per-rank segments in rank order
    std::vector<int64_t> sc(scnt), rc(rcnt);
    sc[me_] = 0;
    rc[me_] = 0;
    int64_t stot = 0, rtot = 0;
    for (int q = 0; q < p_; ++q) {
      stot += sc[q];
      rtot += rc[q];
    }
    char* h = static_cast<char*>(host(8 * size_t(stot + rtot)));
    char* hs = h;
    char* hr = h + 8 * stot;
    const char* s = static_cast<const char*>(send);
    char* r = static_cast<char*>(recv);
    int64_t o = 0;
    for (int q = 0; q < p_; ++q) {
      if (sc[q] > 0)
        RKMF_CUDA(cudaMemcpyAsync(hs + 8 * o, s + 8 * soff[q], 8 * size_t(sc[q]),
                                  cudaMemcpyDeviceToHost, st));
      o += sc[q];
    }
    RKMF_CUDA(cudaStreamSynchronize(st));
    if (cb_.alltoallv_b64(cb_.user, hs, sc.data(), hr, rc.data()) != 0)
      throw Error(RKMF_DEVICE_ERROR, "host comm: alltoallv callback failed");
    o = 0;
    for (int q = 0; q < p_; ++q) {
      if (rc[q] > 0)
        RKMF_CUDA(cudaMemcpyAsync(r + 8 * roff[q], hr + 8 * o, 8 * size_t(rc[q]),
                                  cudaMemcpyHostToDevice, st));
      o += rc[q];
    }
    RKMF_CUDA(cudaStreamSynchronize(st));
  }

 private:
  void* host(size_t bytes) {
    if (bytes > cap_) {
      if (stage_) RKMF_CUDA(cudaFreeHost(stage_));
      stage_ = nullptr;
      cap_ = std::max<size_t>(bytes, 4096);
      RKMF_CUDA(cudaMallocHost(&stage_, cap_));
    }
    return stage_;
  }
  int me_, p_;
  rkmf_host_comm cb_;
  void* stage_ = nullptr;
  size_t cap_ = 0;
};

__global__ void pack_kernel(int64_t cnt, const int32_t* __restrict__ idx,
                            const double* __restrict__ x, double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = x[idx[i]];
}

int blocks_for(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096))); }

}  // namespace

void comm_allreduce_sum(rkmf_context* ctx, double* buf, size_t count) {
  if (!ctx->comm || ctx->nranks <= 1 || count == 0) return;
  ctx->comm->allreduce(buf, count, false, ctx->stream);
}

void comm_halo_exchange(rkmf_context* ctx, const rkmf_matrix* A, double* x) {
  if (!A->partitioned || !ctx->comm || ctx->nranks <= 1) return;
  const HaloPlan& h = A->halo;
  if (h.send_total > 0) {
    pack_kernel<<<blocks_for(h.send_total), 256, 0, ctx->stream>>>(h.send_total, h.send_idx, x,
                                                                    h.sendbuf);
    RKMF_CUDA(cudaGetLastError());
    ctx->launches++;
  }
  ctx->comm->alltoallv(h.sendbuf, h.send_off, h.send_cnt, x + h.n_local, h.recv_off, h.recv_cnt,
                       true, ctx->stream);
}

// Global norm1 = max column abs-sum (sparse.cpp:97-102) of a partitioned
// matrix whose halo plan is set, order-independent like the single-GPU one
// (spmv.cu fixed-point words): the global max |a_ij| (allreduce max) fixes
// the scale, local fixed-point column sums, their halo parts returned to the
// owners (the reverse of the halo exchange; the words travel as 8-byte
// payloads) and added with integer atomics, local max, allreduce(max).
void partitioned_norm1(rkmf_context* ctx, rkmf_matrix* M) {
  const HaloPlan& h = M->halo;
  const int64_t n_local = h.n_local, n_halo = h.n_halo, nnz = M->view.nnz;
  const int64_t nc = n_local + n_halo;
  cudaStream_t st = ctx->stream;
  Transport& T = *ctx->comm;
  ScopedBuf cs, back, mx, vm;
  cs.ensure(sizeof(unsigned long long) * size_t(2 * nc + 1));
  back.ensure(sizeof(unsigned long long) * size_t(std::max<int64_t>(h.send_total, 1)));
  mx.ensure(sizeof(double));
  vm.ensure(sizeof(double));
  auto* hi = static_cast<unsigned long long*>(cs.p);
  auto* lo = hi + nc;
  auto* vmax = static_cast<unsigned long long*>(vm.p);
  launch_abs_max_bits(nnz, M->val, vmax, st);
  T.allreduce(vm.as<double>(), 1, true, st);  // non-negative: max of the values = max of the bits
  launch_fx_colsum(nnz, M->col, M->val, vmax, nc, hi, lo, st);
  for (unsigned long long* word : {hi, lo}) {
    T.alltoallv(word + n_local, h.recv_off, h.recv_cnt, back.p, h.send_off, h.send_cnt, false, st);
    launch_fx_scatter_add(h.send_total, h.send_idx, static_cast<unsigned long long*>(back.p), word,
                          st);
  }
  launch_fx_colmax(n_local, hi, lo, vmax, mx.as<double>(), st);
  T.allreduce(mx.as<double>(), 1, true, st);
  RKMF_CUDA(cudaMemcpyAsync(&M->norm1, mx.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaStreamSynchronize(st));
  ctx->launches += 5;
}

}  // namespace rkmf_b200

using namespace rkmf_b200;

namespace {

template <class F>
int guarded_c(rkmf_context* ctx, F&& fn) {
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

void check_ranks(int32_t nranks, int32_t rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) param_error("comm: invalid rank/nranks");
}

}  // namespace

extern "C" {

int rkmf_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return RKMF_DEVICE_ERROR;
  std::memcpy(out128, &id, sizeof(id));
  return RKMF_OK;
}

int rkmf_context_init_comm(rkmf_context* ctx, int32_t nranks, int32_t rank,
                           const void* unique_id128) {
  return guarded_c(ctx, [&] {
    check_ranks(nranks, rank);
    RKMF_CUDA(cudaSetDevice(ctx->device));
    delete ctx->comm;
    ctx->comm = nullptr;
    ctx->nranks = nranks;
    ctx->rank = rank;
    if (nranks == 1) return;
    ncclUniqueId id;
    std::memcpy(&id, unique_id128, sizeof(id));
    ctx->comm = new NcclTransport(nranks, rank, id);
  });
}

int rkmf_context_init_host_comm(rkmf_context* ctx, int32_t nranks, int32_t rank,
                                const rkmf_host_comm* callbacks) {
  return guarded_c(ctx, [&] {
    check_ranks(nranks, rank);
    if (nranks > 1 && (!callbacks || !callbacks->allreduce_sum_f64 ||
                       !callbacks->allreduce_max_f64 || !callbacks->alltoallv_b64))
      param_error("host comm: all three callbacks are required");
    delete ctx->comm;
    ctx->comm = nullptr;
    ctx->nranks = nranks;
    ctx->rank = rank;
    if (nranks == 1) return;
    ctx->comm = new HostTransport(nranks, rank, *callbacks);
  });
}

int rkmf_matrix_create_partitioned(rkmf_context* ctx, int64_t n_global, const int64_t* row_starts,
                                   const int64_t* h_row_ptr_local, const int32_t* h_col_global,
                                   const double* h_values, rkmf_matrix** out) {
  return guarded_c(ctx, [&] {
    RKMF_CUDA(cudaSetDevice(ctx->device));
    const int P = ctx->nranks, me = ctx->rank;
    if (P > 1 && !ctx->comm) param_error("partitioned matrix: initialise the communicator first");
    const int64_t rb = row_starts[me], re = row_starts[me + 1];
    const int64_t n_local = re - rb;
    if (row_starts[0] != 0 || rb < 0 || re < rb || row_starts[P] != n_global)
      shape_error("partition: bad row_starts");
    if (h_row_ptr_local[0] != 0) shape_error("row_ptr[0] != 0");
    const int64_t nnz = h_row_ptr_local[n_local];
    // validate the rows in global numbering (sparse.cpp:61-81)
    for (int64_t r = 0; r < n_local; ++r) {
      const int64_t lo = h_row_ptr_local[r], hi = h_row_ptr_local[r + 1];
      if (hi < lo) shape_error("row_ptr not nondecreasing");
      for (int64_t k = lo; k < hi; ++k) {
        const int64_t c = h_col_global[k];
        if (c < 0 || c >= n_global) shape_error("column index out of range");
        if (k > lo && c <= h_col_global[k - 1])
          shape_error("columns not strictly increasing within a row");
        if (!std::isfinite(h_values[k])) numerical_error("non-finite matrix entry");
      }
    }
    int64_t n_halo = 0;
    rkmf_partition_halo(P, me, row_starts, h_row_ptr_local, h_col_global, &n_halo, nullptr,
                        nullptr, nullptr);
    std::vector<int64_t> halo(static_cast<size_t>(n_halo)), recv_cnt(static_cast<size_t>(P));
    std::vector<int32_t> col_local(static_cast<size_t>(nnz));
    rkmf_partition_halo(P, me, row_starts, h_row_ptr_local, h_col_global, &n_halo, halo.data(),
                        recv_cnt.data(), col_local.data());
    rkmf_matrix* M = create_matrix_host(ctx, n_local, n_local + n_halo, h_row_ptr_local,
                                        col_local.data(), h_values, false);
    try {
      HaloPlan& h = M->halo;
      M->partitioned = true;
      h.n_global = n_global;
      h.row_begin = rb;
      h.n_local = n_local;
      h.n_halo = n_halo;
      h.recv_cnt = recv_cnt;
      h.recv_off.assign(size_t(P), 0);
      for (int q = 1; q < P; ++q) h.recv_off[q] = h.recv_off[q - 1] + h.recv_cnt[q - 1];
      h.send_cnt.assign(size_t(P), 0);
      h.send_off.assign(size_t(P), 0);
      cudaStream_t st = ctx->stream;
      if (P > 1) {
        Transport& T = *ctx->comm;
        std::vector<int64_t> one(static_cast<size_t>(P), 1), idx(static_cast<size_t>(P));
        for (int q = 0; q < P; ++q) idx[q] = q;
        // 1) counts: what each rank needs from me
        DevBuf rc, sc;
        rc.ensure(sizeof(int64_t) * size_t(P));
        sc.ensure(sizeof(int64_t) * size_t(P));
        RKMF_CUDA(cudaMemcpyAsync(rc.p, h.recv_cnt.data(), sizeof(int64_t) * size_t(P),
                                  cudaMemcpyHostToDevice, st));
        RKMF_CUDA(cudaMemsetAsync(sc.p, 0, sizeof(int64_t) * size_t(P), st));
        T.alltoallv(rc.p, idx, one, sc.p, idx, one, false, st);
        RKMF_CUDA(cudaMemcpyAsync(h.send_cnt.data(), sc.p, sizeof(int64_t) * size_t(P),
                                  cudaMemcpyDeviceToHost, st));
        RKMF_CUDA(cudaStreamSynchronize(st));
        h.send_cnt[me] = 0;
        for (int q = 1; q < P; ++q) h.send_off[q] = h.send_off[q - 1] + h.send_cnt[q - 1];
        h.send_total = h.send_off[P - 1] + h.send_cnt[P - 1];
        // 2) index lists: my requests (global ids, grouped by owner) -> owners
        DevBuf req, got;
        req.ensure(sizeof(int64_t) * size_t(std::max<int64_t>(n_halo, 1)));
        got.ensure(sizeof(int64_t) * size_t(std::max<int64_t>(h.send_total, 1)));
        if (n_halo > 0)
          RKMF_CUDA(cudaMemcpyAsync(req.p, halo.data(), sizeof(int64_t) * size_t(n_halo),
                                    cudaMemcpyHostToDevice, st));
        T.alltoallv(req.p, h.recv_off, h.recv_cnt, got.p, h.send_off, h.send_cnt, false, st);
        std::vector<int64_t> sg(static_cast<size_t>(h.send_total));
        if (h.send_total > 0)
          RKMF_CUDA(cudaMemcpyAsync(sg.data(), got.p, sizeof(int64_t) * size_t(h.send_total),
                                    cudaMemcpyDeviceToHost, st));
        RKMF_CUDA(cudaStreamSynchronize(st));
        std::vector<int32_t> sl(static_cast<size_t>(h.send_total));
        for (int64_t i = 0; i < h.send_total; ++i) {
          if (sg[size_t(i)] < rb || sg[size_t(i)] >= re) shape_error("partition: bad halo request");
          sl[size_t(i)] = int32_t(sg[size_t(i)] - rb);
        }
        RKMF_CUDA(cudaMalloc(&h.send_idx, sizeof(int32_t) * size_t(std::max<int64_t>(h.send_total, 1))));
        RKMF_CUDA(cudaMalloc(&h.sendbuf, sizeof(double) * size_t(std::max<int64_t>(h.send_total, 1))));
        if (h.send_total > 0)
          RKMF_CUDA(cudaMemcpyAsync(h.send_idx, sl.data(), sizeof(int32_t) * size_t(h.send_total),
                                    cudaMemcpyHostToDevice, st));
        partitioned_norm1(ctx, M);
      }
    } catch (...) {
      rkmf_matrix_destroy(M);
      throw;
    }
    *out = M;
  });
}

// Rows of the Q1 matrix on N^3 nodes (BASELINE cfg3/cfg5) generated in HBM
// for this rank's plane-aligned block: the same local rows,
// local column numbering [owned | lower plane | upper plane] and halo plan
// that rkmf_matrix_create_partitioned builds from host CSR (rkmf_partition_halo),
// without a host copy of the 27-point matrix. row_starts must be strictly
// increasing multiples of N^2 (every rank owns whole x-planes), so the halo
// is exactly the x-plane below (owned by rank - 1) and above (rank + 1).
int rkmf_matrix_gen_q1_hex_partitioned(rkmf_context* ctx, int64_t N, int32_t lognormal,
                                       uint64_t coef_seed, int32_t dirichlet,
                                       const int64_t* row_starts, rkmf_matrix** out) {
  return guarded_c(ctx, [&] {
    RKMF_CUDA(cudaSetDevice(ctx->device));
    const int P = ctx->nranks, me = ctx->rank;
    if (P > 1 && !ctx->comm) param_error("partitioned matrix: initialise the communicator first");
    if (N < 2) param_error("gen_q1_hex: N must be >= 2");
    const int64_t plane = N * N, n = N * N * N;
    if (row_starts[0] != 0 || row_starts[P] != n) shape_error("partition: bad row_starts");
    for (int q = 0; q < P; ++q)
      if (row_starts[q + 1] <= row_starts[q] || row_starts[q + 1] % plane != 0)
        param_error("gen_q1_hex_partitioned: row_starts must be increasing multiples of N^2");
    const int64_t rb = row_starts[me], re = row_starts[me + 1], n_local = re - rb;
    const int64_t nlo = me > 0 ? plane : 0, nhi = me < P - 1 ? plane : 0;
    rkmf_matrix* M = gen_q1_rows(ctx, N, lognormal, coef_seed, dirichlet, rb, re, nlo, nhi);
    try {
      HaloPlan& h = M->halo;
      M->partitioned = true;
      h.n_global = n;
      h.row_begin = rb;
      h.n_local = n_local;
      h.n_halo = nlo + nhi;
      h.recv_cnt.assign(size_t(P), 0);
      h.send_cnt.assign(size_t(P), 0);
      if (me > 0) h.recv_cnt[size_t(me - 1)] = h.send_cnt[size_t(me - 1)] = plane;
      if (me < P - 1) h.recv_cnt[size_t(me + 1)] = h.send_cnt[size_t(me + 1)] = plane;
      h.recv_off.assign(size_t(P), 0);
      h.send_off.assign(size_t(P), 0);
      for (int q = 1; q < P; ++q) {
        h.recv_off[q] = h.recv_off[q - 1] + h.recv_cnt[q - 1];
        h.send_off[q] = h.send_off[q - 1] + h.send_cnt[q - 1];
      }
      h.send_total = h.send_off[P - 1] + h.send_cnt[P - 1];
      if (P > 1) {
        // my first plane goes to rank - 1, my last plane to rank + 1 (rank order)
        std::vector<int32_t> sl;
        sl.reserve(size_t(h.send_total));
        if (me > 0)
          for (int64_t i = 0; i < plane; ++i) sl.push_back(int32_t(i));
        if (me < P - 1)
          for (int64_t i = n_local - plane; i < n_local; ++i) sl.push_back(int32_t(i));
        RKMF_CUDA(cudaMalloc(&h.send_idx, sizeof(int32_t) * size_t(std::max<int64_t>(h.send_total, 1))));
        RKMF_CUDA(cudaMalloc(&h.sendbuf, sizeof(double) * size_t(std::max<int64_t>(h.send_total, 1))));
        RKMF_CUDA(cudaMemcpy(h.send_idx, sl.data(), sizeof(int32_t) * sl.size(),
                             cudaMemcpyHostToDevice));
        partitioned_norm1(ctx, M);
      }
    } catch (...) {
      rkmf_matrix_destroy(M);
      throw;
    }
    *out = M;
  });
}

int rkmf_context_comm_info(const rkmf_context* ctx, int32_t* nranks, int32_t* rank,
                           int32_t* transport) {
  if (!ctx) return RKMF_PARAMETER_ERROR;
  return guarded_c(const_cast<rkmf_context*>(ctx), [&] {
    const Transport* T = ctx->comm;
    if (nranks) *nranks = T ? T->comm_size() : ctx->nranks;
    if (rank) *rank = ctx->rank;
    if (transport) *transport = T ? T->kind() : 0;
  });
}

}  // extern "C"
