// Private definitions shared by engine.cu and comm.cu (context, matrix and
// sketch objects behind the opaque C-ABI handles).
#pragma once

#include <algorithm>
#include <string>
#include <vector>

#include "rkmf_internal.cuh"

namespace rkmf_b200 {
// a sketch as its consumer reads it: `groups` partial d-vectors summed in order
struct SketchSum {
  const double* part = nullptr;
  int groups = 0;
};
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* ensure(size_t bytes) {
    if (bytes <= cap && p) return p;
    if (p) RKMF_CUDA(cudaFree(p));
    p = nullptr;
    cap = 0;
    RKMF_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
    cap = std::max<size_t>(bytes, 256);
    return p;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// a DevBuf freed when it leaves scope (setup-time temporaries)
struct ScopedBuf : DevBuf {
  ScopedBuf() = default;
  ScopedBuf(const ScopedBuf&) = delete;
  ScopedBuf& operator=(const ScopedBuf&) = delete;
  ~ScopedBuf() { release(); }
};

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

}  // namespace rkmf_b200

namespace rkmf_b200 {
// Collectives of the row-partitioned solve, on device buffers and the
// context stream. NcclTransport (comm.cu) is the product path, one process
// per GPU over NVLink/NVSwitch; HostTransport stages through pinned host
// memory into caller callbacks (rkmf_host_comm: MPI, gloo, tests).
struct Transport {
  virtual ~Transport() {}
  virtual int kind() const = 0;       // 1 NCCL, 2 host callbacks
  virtual int comm_size() const = 0;  // ranks of the communicator (ncclCommCount for NCCL)
  // in-place elementwise sum (or max) of count doubles over all ranks
  virtual void allreduce(double* dev, size_t count, bool max, cudaStream_t st) = 0;
  // personalised exchange of 8-byte elements: segment q of the send buffer
  // (scnt[q] elements at soff[q]) goes to rank q; what rank q sends here lands
  // at roff[q] (rcnt[q] elements). Counts are agreed beforehand; the own-rank
  // segment is not moved.
  virtual void alltoallv(const void* send, const std::vector<int64_t>& soff,
                         const std::vector<int64_t>& scnt, void* recv,
                         const std::vector<int64_t>& roff, const std::vector<int64_t>& rcnt,
                         bool is_double, cudaStream_t st) = 0;
};
}  // namespace rkmf_b200

using namespace rkmf_b200;

struct rkmf_context {
  int device = 0;
  // multi-GPU: one rank per process/GPU (rkmf_context_init_comm / _host_comm)
  Transport* comm = nullptr;
  int nranks = 1, rank = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::string last_error;
  int64_t launches = 0;
  SolveState* st_dev = nullptr;
  SolveState* st_host = nullptr;  // pinned
  DevBuf z, W, U, Rbar, Racc, ws, u, g, fhat, ref, partial, qshift, qweight, qpi,
      qemx, scratch, gram, cl, diag;
  // the adaptive InvSqrt quadrature's two node sets (engine.cu QuadSet)
  struct QuadBufs {
    DevBuf shift, weight, pi, emx, partial, g;
    void release() {
      for (DevBuf* b : {&shift, &weight, &pi, &emx, &partial, &g}) b->release();
    }
  } isq[2];
  rkmf_cycle_observer observer = nullptr;  // test-only CycleObserver (restart.hpp:53)
  void* observer_user = nullptr;
  int64_t racc_ld = 0;   // leading dimension of the last solve's R_accum
  int64_t racc_cap = 0;  // allocated leading dimension of Racc (kept across solves)
  std::vector<double> last_R;
  int64_t last_M = 0;
  // deterministic-reduction scratch (detred.cuh): block partials (shared:
  // one producer at a time on the stream), then the group partials and
  // tickets of the step sketch (K2 -> K3), of the start sketch (-> start_init)
  // and of the (||y||^2, err^2) pair of K5
  DevBuf redbuf, pfin_sk, pfin_st;  // pfin: summed sketches of a partitioned solve
  SketchSum start_sum;               // the start sketch as start_init reads it
  int64_t red_cap_d = 0;
  DetRed red_sk, red_st, red_up;
  void ensure_red(int64_t d) {
    d = std::max<int64_t>(d, 2);
    if (d <= red_cap_d && redbuf.p) return;
    int sms = 0;
    RKMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int kb = 24 * std::max(sms, 1);  // K2: <= 16 blocks/SM; K5: 24 blocks/SM
    const int gk = det_groups(kb) + 1;     // enough for any grid <= kb
    const size_t nd = size_t(kb) * size_t(d) + 2 * size_t(gk) * size_t(d) + size_t(gk) * 2;
    const size_t bytes = sizeof(double) * nd + sizeof(unsigned) * size_t(3 * (gk + 1));
    redbuf.ensure(bytes);
    RKMF_CUDA(cudaMemsetAsync(redbuf.p, 0, bytes, stream));  // tickets start at zero
    double* p = redbuf.as<double>();
    unsigned* tk = reinterpret_cast<unsigned*>(p + nd);
    DetRed* rs[3] = {&red_sk, &red_st, &red_up};
    double* gp = p + size_t(kb) * size_t(d);
    for (int i = 0; i < 3; ++i) {
      rs[i]->part = p;
      rs[i]->gpart = gp;
      gp += size_t(gk) * size_t(i < 2 ? d : 2);
      rs[i]->tick = tk + i * (gk + 1);
      rs[i]->max_blocks = kb;
      rs[i]->max_len = int(i < 2 ? d : 2);
      rs[i]->max_groups = gk;
      rs[i]->groups = 0;
    }
    red_cap_d = d;
  }
  // the classical builder's k+1 dots: one reduction slice per column, up to
  // 8 blocks per SM each (classical.cu grid_rows)
  DevBuf redcl;
  int64_t red_cl_slices = 0;
  DetRed red_cl;
  const DetRed& red_classical(int64_t slices) {
    if (slices > red_cl_slices || !redcl.p) {
      int sms = 0;
      RKMF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      const int64_t nb = 8 * std::max(sms, 1), ng = det_groups(int(nb)) + 1;
      const size_t nd = size_t(slices) * size_t(nb + ng);
      const size_t bytes = sizeof(double) * nd + sizeof(unsigned) * size_t(slices * (ng + 1));
      redcl.ensure(bytes);
      RKMF_CUDA(cudaMemsetAsync(redcl.p, 0, bytes, stream));
      double* p = redcl.as<double>();
      red_cl.part = p;
      red_cl.gpart = p + size_t(slices) * size_t(nb);
      red_cl.tick = reinterpret_cast<unsigned*>(p + nd);
      red_cl.max_blocks = int(slices * nb);
      red_cl.max_len = 1;
      red_cl.max_groups = int(slices * (ng + 1));
      red_cl_slices = slices;
    }
    return red_cl;
  }
  DetRed& red_sketch(int64_t d) {
    ensure_red(d);
    return red_sk;
  }
  DetRed& red_start(int64_t d) {
    ensure_red(d);
    return red_st;
  }
  const DetRed& red_update() {
    ensure_red(2);
    return red_up;
  }
  std::vector<cudaEvent_t> events;
  cudaEvent_t event(size_t i) {
    while (events.size() <= i) {
      cudaEvent_t e;
      RKMF_CUDA(cudaEventCreate(&e));
      events.push_back(e);
    }
    return events[i];
  }
  void sync_state() {
    RKMF_CUDA(cudaMemcpyAsync(st_host, st_dev, sizeof(SolveState), cudaMemcpyDeviceToHost, stream));
    RKMF_CUDA(cudaStreamSynchronize(stream));
  }
  // ---- optional per-kernel-class timing (rkmf_context_kernel_timing) ----
  bool ktime = false;
  bool fused_cycle = true;  // small matrices: a cycle's steps in one kernel (cycle_small.cu)
  std::vector<cudaEvent_t> kpool;
  std::vector<std::pair<int, size_t>> kpend;  // (class, index of the start event)
  double kms[RKMF_KCLASS_COUNT] = {0};
  int64_t kcnt[RKMF_KCLASS_COUNT] = {0};
  template <class F>
  void timed(int cls, F&& launch) {
    if (!ktime) { launch(); return; }
    const size_t i = 2 * kpend.size();
    while (kpool.size() < i + 2) {
      cudaEvent_t e;
      RKMF_CUDA(cudaEventCreate(&e));
      kpool.push_back(e);
    }
    RKMF_CUDA(cudaEventRecord(kpool[i], stream));
    launch();
    RKMF_CUDA(cudaEventRecord(kpool[i + 1], stream));
    kpend.push_back({cls, i});
  }
  void collect_ktimes() {  // call after a stream synchronize
    for (auto& p : kpend) {
      float ms = 0.f;
      RKMF_CUDA(cudaEventElapsedTime(&ms, kpool[p.second], kpool[p.second + 1]));
      kms[p.first] += ms;
      kcnt[p.first] += 1;
    }
    kpend.clear();
  }
};

// Row-block partition of a matrix over the ranks of a context's communicator
// (partition.cpp builds the plan; comm.cu moves the data).
struct HaloPlan {
  int64_t n_global = 0, row_begin = 0, n_local = 0, n_halo = 0;
  std::vector<int64_t> send_cnt, send_off, recv_cnt, recv_off;  // per rank
  int32_t* send_idx = nullptr;  // device: local row of each value sent
  double* sendbuf = nullptr;    // device
  int64_t send_total = 0;
};

struct rkmf_matrix {
  rkmf_context* ctx = nullptr;
  int device = 0;
  CsrView view{};
  void* rp = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
  double norm1 = 0.0;
  double* dia_val = nullptr;  // optional diagonal copy (dia.cu)
  int32_t* dia_off = nullptr;  // its sorted diagonal offsets
  uint8_t* dia_tid = nullptr;  // optional row dictionary of the copy: tuple ids
  double* dia_dict = nullptr;  // and the distinct row tuples
  std::vector<double> dia_dict_host;  // host copy (K2 passes small ones as kernel parameters)
  uint8_t* rd_tid = nullptr;  // optional CSR row dictionary (rowdict.cu): form ids
  int32_t* rd_cnt = nullptr;  // per form: nonzero count, offsets, values
  int32_t* rd_off = nullptr;
  double* rd_val = nullptr;
  bool partitioned = false;
  HaloPlan halo;
  int64_t n_rows_global() const { return partitioned ? halo.n_global : view.n_rows; }
};

struct rkmf_sketch {
  rkmf_context* ctx = nullptr;
  int device = 0;
  int64_t d = 0, n = 0, zeta = 0;
  int64_t n_global = 0, col_begin = 0;  // columns [col_begin, col_begin+n) of a d x n_global S
  uint64_t seed = 0;
  double scale = 1.0;
  uint16_t* rows = nullptr;
  int8_t* signs = nullptr;
  uint16_t* tile_off = nullptr;  // one allocation: header, then entries
  uint8_t* tile_ent = nullptr;
  int64_t ent_stride = 0;  // entry bytes per tile (sketch_tiles_stride)
  size_t layout_bytes = 0;
  SketchView view() const {
    SketchView v;
    v.d = d;
    v.n = n;
    v.zeta = zeta;
    v.tile_off = tile_off;
    v.tile_ent = tile_ent;
    v.ent_stride = ent_stride;
    v.scale = scale;
    return v;
  }
};


namespace rkmf_b200 {
// dia.cu
void build_dia(rkmf_matrix* M);
void drop_dia(rkmf_matrix* M);
void build_dia_dict(rkmf_matrix* M);
void drop_dia_dict(rkmf_matrix* M);
// rowdict.cu
void build_csr_dict(rkmf_matrix* M);
void drop_csr_dict(rkmf_matrix* M);
bool dia_enabled_by_env();
// comm.cu
void comm_allreduce_sum(rkmf_context* ctx, double* buf, size_t count);
void comm_halo_exchange(rkmf_context* ctx, const rkmf_matrix* A, double* x);
}  // namespace rkmf_b200

namespace rkmf_b200 {
// engine.cu: host CSR -> device matrix (validated; require_sorted=false for
// partition-local matrices whose halo columns are renumbered past the owned ones)
rkmf_matrix* create_matrix_host(rkmf_context* ctx, int64_t n_rows, int64_t n_cols,
                                const int64_t* h_rp, const int32_t* h_ci, const double* h_v,
                                bool require_sorted);
// device CSR (int64 row pointers) -> validated matrix; with copy_colval false
// the matrix takes ownership of col/val (allocated with kNnzPad padding)
rkmf_matrix* create_from_device_rp64(rkmf_context* ctx, int64_t n_rows, int64_t n_cols,
                                     int64_t nnz, const int64_t* rp64_dev,
                                     const int32_t* col_dev, const double* val_dev,
                                     bool copy_colval, bool require_sorted);
// gen.cu: rows [rb, re) of the Q1 matrix on N^3 nodes, local numbering
// [owned | lower halo (nlo) | upper halo (nhi)] (whole matrix: 0, N^3, 0, 0)
rkmf_matrix* gen_q1_rows(rkmf_context* ctx, int64_t N, int lognormal, uint64_t coef_seed,
                         int dirichlet, int64_t rb, int64_t re, int64_t nlo, int64_t nhi);
}  // namespace rkmf_b200
