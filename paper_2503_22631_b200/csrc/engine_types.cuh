// Private definitions shared by engine.cu and comm.cu (context, matrix and
// sketch objects behind the opaque C-ABI handles).
#pragma once

#include <algorithm>
#include <string>
#include <vector>

#include "rkmf_internal.cuh"

namespace rkmf_b200 {
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

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

}  // namespace rkmf_b200

namespace rkmf_b200 {
// Collectives of the row-partitioned solve, on device buffers and the
// context stream. NcclTransport (comm.cu) is the product path, one process
// per GPU over NVLink/NVSwitch; HostTransport stages through pinned host
// memory into caller callbacks (rkmf_host_comm: MPI, gloo, tests).
struct Transport {
  virtual ~Transport() {}
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
  DevBuf z, pacc, sacc, W, U, Rbar, Racc, ws, u, g, fhat, ref, partial, qshift, qweight, qpi,
      qemx, scratch, gram, cl, diag;
  int64_t racc_ld = 0;   // leading dimension of the last solve's R_accum
  int64_t racc_cap = 0;  // allocated leading dimension of Racc (kept across solves)
  std::vector<double> last_R;
  int64_t last_M = 0;
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
  size_t layout_bytes = 0;
  uint8_t* rbin = nullptr;  // row-major copy for the row-sketch K2 (+ sbit), or null
  uint8_t* sbit = nullptr;
  uint8_t* wslow = nullptr;
  SketchView view() const {
    SketchView v;
    v.d = d;
    v.n = n;
    v.zeta = zeta;
    v.tile_off = tile_off;
    v.tile_ent = tile_ent;
    v.scale = scale;
    v.rbin = rbin;
    v.sbit = sbit;
    v.wslow = wslow;
    return v;
  }
};


namespace rkmf_b200 {
// dia.cu
void build_dia(rkmf_matrix* M);
void drop_dia(rkmf_matrix* M);
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
}  // namespace rkmf_b200
