// Diagonal (DIA) copy of a CSR matrix for the fused SpMV + sketch (K2).
//
// The SpMV half of K2 streams 12 bytes per nonzero plus row pointers from HBM
// (a CSR value and its int32 column). When every nonzero of the matrix lies on
// one of a few diagonals (col - row in a small set — the stencil matrices of
// the BASELINE configs: 5/7/27-point Laplacians, Q1, convection-diffusion),
// the same matrix is stored here as [tile][diag][128 rows] fp64 values with
// the sorted offsets on the side: 8 bytes per stored slot and no indices, and
// the x reads at row + offset are coalesced across a warp instead of gathers
// (and issued a tile ahead: they do not depend on the streamed values).
// Slots where the CSR row has no entry hold 0.0, and each row's entries keep
// the CSR's column order, so z = A x is bit-identical to the CSR kernel (a
// padding term adds exactly 0.0).
//
// Eligibility (checked on device, one pass over the nonzeros): at most
// kMaxDiag = 8 distinct offsets (27-point stencils stay on the CSR kernel,
// which splits their rows over two threads and measured faster), columns strictly increasing within each row, and
// the padded DIA stream smaller than 0.85x the CSR stream. Otherwise the matrix
// keeps the CSR path only. RKMF_DIA=0 disables the copy at creation;
// rkmf_matrix_dia() drops or (re)builds it.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <vector>

#include "engine_types.cuh"
#include "rkmf_internal.cuh"

namespace rkmf_b200 {

namespace {

constexpr int kSetSlots = 32;      // per-block offset set (shared memory)
constexpr int kGlobalSlots = 256;  // merged set (global memory)
constexpr int32_t kEmpty = INT_MIN;

__device__ __forceinline__ uint32_t hash_off(int32_t v) {
  return (uint32_t(v) * 2654435761u) >> 8;
}

// Insert v into an open-addressed set of `slots` int32 keys; returns false
// when the set is full.
__device__ bool set_insert(int32_t* set, int slots, int32_t v) {
  uint32_t h = hash_off(v) & uint32_t(slots - 1);
  for (int probe = 0; probe < slots; ++probe) {
    const int32_t cur = set[h];
    if (cur == v) return true;
    if (cur == kEmpty) {
      const int32_t old = atomicCAS(set + h, kEmpty, v);
      if (old == kEmpty || old == v) return true;
    }
    h = (h + 1) & uint32_t(slots - 1);
  }
  return false;
}

// flags[0]: a row's columns are not strictly increasing; flags[1]: more
// distinct offsets than the sets hold. gset: the merged offsets.
template <typename RP>
__global__ void dia_offsets_kernel(int64_t n, const RP* __restrict__ rp,
                                   const int32_t* __restrict__ ci, int32_t* gset, int32_t* flags) {
  __shared__ int32_t set[kSetSlots];
  __shared__ int bad;
  for (int i = threadIdx.x; i < kSetSlots; i += blockDim.x) set[i] = kEmpty;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n;
       row += int64_t(gridDim.x) * blockDim.x) {
    if (bad) break;  // racy read is fine: only an early exit
    const int64_t lo = int64_t(rp[row]), hi = int64_t(rp[row + 1]);
    int32_t prev = -1;
    for (int64_t e = lo; e < hi; ++e) {
      const int32_t c = ci[e];
      if (c <= prev) {
        atomicExch(flags + 0, 1);
        bad = 1;
        break;
      }
      prev = c;
      if (!set_insert(set, kSetSlots, int32_t(int64_t(c) - row))) {
        atomicExch(flags + 1, 1);
        bad = 1;
        break;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSetSlots; i += blockDim.x)
    if (set[i] != kEmpty && !set_insert(gset, kGlobalSlots, set[i])) atomicExch(flags + 1, 1);
}

// dval[(tile * ndiag + q) * 128 + r] = A(row, row + doff[q]) (0.0 where absent)
template <typename RP>
__global__ void dia_fill_kernel(int64_t n, const RP* __restrict__ rp,
                                const int32_t* __restrict__ ci, const double* __restrict__ val,
                                const int32_t* __restrict__ doff, int ndiag, double* dval) {
  __shared__ int32_t offs[kMaxDiag];
  for (int q = threadIdx.x; q < ndiag; q += blockDim.x) offs[q] = doff[q];
  __syncthreads();
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n;
       row += int64_t(gridDim.x) * blockDim.x) {
    const int64_t tile = row / kTileRows, r = row % kTileRows;
    double* base = dval + tile * int64_t(ndiag) * kTileRows + r;
    const int64_t lo = int64_t(rp[row]), hi = int64_t(rp[row + 1]);
    int q = 0;
    for (int64_t e = lo; e < hi; ++e) {  // columns increase, so offsets do too
      const int32_t o = int32_t(int64_t(ci[e]) - row);
      while (offs[q] != o) ++q;
      base[int64_t(q) * kTileRows] = val[e];
    }
  }
}

template <typename RP>
void launch_offsets(const CsrView& v, int32_t* gset, int32_t* flags, cudaStream_t st) {
  dia_offsets_kernel<RP><<<1184, 256, 0, st>>>(v.n_rows, static_cast<const RP*>(v.row_ptr), v.col,
                                               gset, flags);
}
template <typename RP>
void launch_fill(const CsrView& v, const int32_t* doff, int ndiag, double* dval, cudaStream_t st) {
  dia_fill_kernel<RP><<<1184, 256, 0, st>>>(v.n_rows, static_cast<const RP*>(v.row_ptr), v.col,
                                            v.val, doff, ndiag, dval);
}

}  // namespace

void drop_dia(rkmf_matrix* M) {
  if (M->dia_val) cudaFree(M->dia_val);
  if (M->dia_off) cudaFree(M->dia_off);
  M->dia_val = nullptr;
  M->dia_off = nullptr;
  M->view.dval = nullptr;
  M->view.doff = nullptr;
  M->view.ndiag = 0;
}

// Builds the diagonal copy when the matrix qualifies; leaves the CSR-only
// matrix untouched otherwise (also when the copy does not fit in memory).
void build_dia(rkmf_matrix* M) {
  drop_dia(M);
  const CsrView& v = M->view;
  if (v.n_rows == 0 || v.nnz == 0 || !v.row_ptr) return;
  rkmf_context* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  char* scr = static_cast<char*>(ctx->scratch.ensure(sizeof(int32_t) * (kGlobalSlots + 4)));
  int32_t* gset = reinterpret_cast<int32_t*>(scr);
  int32_t* flags = gset + kGlobalSlots;
  std::vector<int32_t> init(kGlobalSlots + 4, kEmpty);
  init[kGlobalSlots] = init[kGlobalSlots + 1] = 0;
  RKMF_CUDA(cudaMemcpyAsync(gset, init.data(), sizeof(int32_t) * init.size(),
                            cudaMemcpyHostToDevice, st));
  if (v.rp64) launch_offsets<int64_t>(v, gset, flags, st);
  else launch_offsets<int32_t>(v, gset, flags, st);
  RKMF_CUDA(cudaGetLastError());
  ctx->launches++;
  std::vector<int32_t> h(kGlobalSlots + 4);
  RKMF_CUDA(cudaMemcpyAsync(h.data(), gset, sizeof(int32_t) * h.size(), cudaMemcpyDeviceToHost,
                            st));
  RKMF_CUDA(cudaStreamSynchronize(st));
  if (h[kGlobalSlots] || h[kGlobalSlots + 1]) return;
  std::vector<int32_t> offs;
  for (int i = 0; i < kGlobalSlots; ++i)
    if (h[i] != kEmpty) offs.push_back(h[i]);
  if (offs.empty() || int(offs.size()) > kMaxDiag) return;
  std::sort(offs.begin(), offs.end());
  const int ndiag = int(offs.size());
  const int64_t tiles = (v.n_rows + kTileRows - 1) / kTileRows;
  const double dia_bytes = 8.0 * double(ndiag) * double(tiles * kTileRows);
  const double csr_bytes = 12.0 * double(v.nnz) + (v.rp64 ? 8.0 : 4.0) * double(v.n_rows);
  if (dia_bytes > 0.85 * csr_bytes) return;
  size_t free_b = 0, total_b = 0;
  RKMF_CUDA(cudaMemGetInfo(&free_b, &total_b));
  if (dia_bytes > 0.25 * double(free_b)) return;  // leave room for the basis
  const size_t nval = size_t(ndiag) * size_t(tiles) * kTileRows;
  if (cudaMalloc(&M->dia_val, sizeof(double) * nval) != cudaSuccess) {
    cudaGetLastError();
    M->dia_val = nullptr;
    return;
  }
  RKMF_CUDA(cudaMalloc(&M->dia_off, sizeof(int32_t) * size_t(ndiag)));
  RKMF_CUDA(cudaMemcpyAsync(M->dia_off, offs.data(), sizeof(int32_t) * size_t(ndiag),
                            cudaMemcpyHostToDevice, st));
  RKMF_CUDA(cudaMemsetAsync(M->dia_val, 0, sizeof(double) * nval, st));
  if (v.rp64) launch_fill<int64_t>(v, M->dia_off, ndiag, M->dia_val, st);
  else launch_fill<int32_t>(v, M->dia_off, ndiag, M->dia_val, st);
  RKMF_CUDA(cudaGetLastError());
  ctx->launches++;
  RKMF_CUDA(cudaStreamSynchronize(st));
  M->view.dval = M->dia_val;
  M->view.doff = M->dia_off;
  M->view.ndiag = ndiag;
}

bool dia_enabled_by_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RKMF_DIA");
    v = e ? (atoi(e) != 0) : 1;
  }
  return v != 0;
}

}  // namespace rkmf_b200
