// K2: CSR SpMV with the sparse-sign sketch fused into its epilogue.
//
// Replaces spmv (proj/src/sparse.cpp:83-95) followed by sketch_apply
// (proj/src/sketch.cpp:51-63) in the per-step loop of randomized_arnoldi
// (proj/src/basis.cpp:120-121). HBM-bound (~0.2 flop/byte): the design goal is
// to stream values/columns exactly once, coalesced, and never re-read z.
//
//  * Persistent grid (SM count x resident blocks). Block b walks tiles
//    b, b+G, ... of 128 consecutive rows, so the sketch partial of a block
//    accumulates in shared memory across all its tiles.
//  * CSR-stream: the tile's nonzero range [rp[r0], rp[r0+128]) is read with
//    fully coalesced loads into shared memory as products val*x[col] (chunks
//    of `cap` products for long rows), then thread t reduces row t from shared
//    memory in column order — the reference's row-sequential order.
//  * Sketch epilogue: z_t*scale goes to shared memory; each thread owns a
//    length-balanced set of sketch rows ("bins") and gathers the tile's
//    contributions from the per-tile transposed layout (sketch_tile_gather,
//    sketch.cu). No atomics except one
//    fp64 RED per bin per block at kernel end.
#include <cuda_runtime.h>

#include <cstdlib>

#include "rkmf_internal.cuh"

namespace rkmf_b200 {

namespace {

template <typename RP, int MODE>
__global__ void __launch_bounds__(kBlock)
    spmv_sketch_kernel(int64_t n, const RP* __restrict__ rp, const int32_t* __restrict__ ci,
                       const double* __restrict__ val, const double* __restrict__ x,
                       const double* xscale, double* __restrict__ z, int64_t num_tiles, int cap,
                       int d, int ent_stride, int64_t off_stride, const uint16_t* __restrict__ toff,
                       const uint8_t* __restrict__ tent, double sscale,
                       const int32_t* stop, int step, DetRed red) {
  if (stop != nullptr && *stop <= step) return;  // breakdown earlier in this cycle
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr bool kSpmv = MODE <= 1;
  constexpr bool kSketch = MODE >= 1;
  double* acc = reinterpret_cast<double*>(smem_raw);       // [d rounded up to even]
  double* zs = acc + (kSketch ? (d + 1) / 2 * 2 : 0);      // [2*128] (+z, -z), 16-byte aligned
  double* prod = zs + (kSketch ? 2 * kTileRows : 0);       // [cap]
  uint16_t* off = reinterpret_cast<uint16_t*>(prod + (kSpmv ? cap : 0));  // [off_stride]
  uint8_t* ent = reinterpret_cast<uint8_t*>(off + (kSketch ? off_stride : 0));  // [tile_ent_stride]

  const int t = threadIdx.x;
  const double xs = xscale ? *xscale : 1.0;
  if (kSketch)
    for (int b = t; b < d; b += kBlock) acc[b] = 0.0;

  for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
    const int64_t r0 = tile * kTileRows;
    const int64_t row = r0 + t;
    const bool live = row < n;
    double zrow = 0.0;
    if (kSpmv) {
      const int64_t r1 = min(n, r0 + kTileRows);
      const int64_t rs = int64_t(rp[r0]), re = int64_t(rp[r1]);
      const int64_t my_lo = live ? int64_t(rp[row]) : 0, my_hi = live ? int64_t(rp[row + 1]) : 0;
      double sum = 0.0;
      for (int64_t c0 = rs; c0 < re; c0 += cap) {
        const int64_t c1 = min(re, c0 + cap);
        const int cnt = int(c1 - c0);
        // coalesced stream of values and column indices; 4 loads in flight
        int e = t;
        for (; e + 3 * kBlock < cnt; e += 4 * kBlock) {
          double v[4];
          int c[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            v[q] = __ldcs(val + c0 + e + q * kBlock);
            c[q] = __ldcs(ci + c0 + e + q * kBlock);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) prod[e + q * kBlock] = v[q] * __ldg(x + c[q]);
        }
        for (; e < cnt; e += kBlock) prod[e] = __ldcs(val + c0 + e) * __ldg(x + __ldcs(ci + c0 + e));
        __syncthreads();
        const int64_t lo = max(my_lo, c0), hi = min(my_hi, c1);
        for (int64_t q = lo; q < hi; ++q) sum += prod[q - c0];
        __syncthreads();
      }
      zrow = sum * xs;
      if (live) z[row] = zrow;
    } else {
      zrow = live ? x[row] * xs : 0.0;
    }
    if (kSketch) {
      zs[t] = live ? zrow * sscale : 0.0;
      zs[kTileRows + t] = -zs[t];
      const uint16_t* go = toff + tile * off_stride;
      for (int q = t; q < off_stride; q += kBlock) off[q] = go[q];
      const int64_t es = ent_stride;
      const uint4* ge = reinterpret_cast<const uint4*>(tent + tile * es);
      uint4* se = reinterpret_cast<uint4*>(ent);
      for (int q = t; q < es / 16; q += kBlock) se[q] = __ldcs(ge + q);
      __syncthreads();
      sketch_tile_gather(t, d, off, ent, zs, acc);
      __syncthreads();
    }
  }
  if (kSketch) {  // block partials -> group partials in a fixed order (detred.cuh)
    __shared__ int rflag;
    __syncthreads();
    det_group_reduce<kBlock, 0>(red, d, acc, t, &rflag);
  }
}

size_t smem_bytes(int mode, int cap, int64_t d, int64_t ent_stride, int64_t off_stride) {
  size_t s = 0;
  if (mode >= 1) s += sizeof(double) * size_t((d + 1) / 2 * 2 + 2 * kTileRows);
  if (mode <= 1) s += sizeof(double) * size_t(cap);
  if (mode >= 1) s += sizeof(uint16_t) * size_t(off_stride) + size_t(ent_stride) + 16;
  return (s + 15) / 16 * 16;
}

template <typename RP, int MODE>
void* kernel_ptr() {
  return reinterpret_cast<void*>(&spmv_sketch_kernel<RP, MODE>);
}

void* pick(bool rp64, int mode) {
  if (rp64) {
    if (mode == 0) return kernel_ptr<int64_t, 0>();
    if (mode == 1) return kernel_ptr<int64_t, 1>();
    return kernel_ptr<int64_t, 2>();
  }
  if (mode == 0) return kernel_ptr<int32_t, 0>();
  if (mode == 1) return kernel_ptr<int32_t, 1>();
  return kernel_ptr<int32_t, 2>();
}

// RKMF_SPMV_PIPE=0 selects the plain CSR-stream kernel (A/B comparisons).
bool use_pipe() {
  static int v = -1;
  if (v < 0) {
    const char* e = knob_env("RKMF_SPMV_PIPE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

}  // namespace

int spmv_sketch_grid(const CsrView* A, const SketchView* S, int mode) {
  const int64_t n = A ? A->n_rows : S->n;
  const int64_t tiles = (n + kTileRows - 1) / kTileRows;
  const int cap = A ? A->cap : 0;
  const int64_t d = S ? S->d : 0, es = S ? S->ent_stride : 0;
  const int64_t off_stride = S ? tile_off_stride(d) : 0;
  const size_t smem = smem_bytes(mode, cap, d, es, off_stride);
  void* fn = pick(A ? A->rp64 : false, mode);
  if (smem > 48 * 1024)
    RKMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per_sm = 0;
  RKMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, smem));
  if (per_sm < 1) per_sm = 1;
  const int64_t g = int64_t(per_sm) * num_sms();
  return int(std::max<int64_t>(1, std::min<int64_t>(g, tiles)));
}

void launch_spmv_sketch(const CsrView* A, const SketchView* S, int mode, const double* x,
                        const double* xscale_dev, double* z, const int32_t* stop_flag,
                        int step, int grid, DetRed& red, cudaStream_t st) {
  const int64_t n = A ? A->n_rows : S->n;
  const int64_t tiles = (n + kTileRows - 1) / kTileRows;
  const int cap = A ? A->cap : 0;
  const int d = S ? int(S->d) : 0, es = S ? int(S->ent_stride) : 0;
  const int64_t off_stride = S ? tile_off_stride(S->d) : 0;
  const size_t smem = smem_bytes(mode, cap, d, es, off_stride);
  if (mode == 1 && A && S && use_pipe() &&
      launch_spmv_sketch_pipe(A, S, x, xscale_dev, z, stop_flag, step, red, st))
    return;
  if (mode == 2 && S && !stop_flag && use_pipe() &&
      launch_sketch_only_pipe(S, x, xscale_dev, red, st))
    return;
  if (grid <= 0) grid = spmv_sketch_grid(A, S, mode);
  if (S && (grid > red.max_blocks || S->d > red.max_len))
    param_error("internal: sketch reduction scratch too small");
  red.groups = S ? det_groups(grid) : 0;
  const uint16_t* toff = S ? S->tile_off : nullptr;
  const uint8_t* tent = S ? S->tile_ent : nullptr;
  const double sscale = S ? S->scale : 1.0;
  const bool rp64 = A ? A->rp64 : false;
#define RKMF_LAUNCH_SPMV(RP, MODE)                                                             \
  spmv_sketch_kernel<RP, MODE><<<grid, kBlock, smem, st>>>(                                    \
      n, A ? static_cast<const RP*>(A->row_ptr) : nullptr, A ? A->col : nullptr,               \
      A ? A->val : nullptr, x, xscale_dev, z, tiles, cap, d, es, off_stride, toff, tent,     \
      sscale, stop_flag, step, red)
  if (smem > 48 * 1024)
    RKMF_CUDA(cudaFuncSetAttribute(pick(rp64, mode), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
  if (rp64) {
    if (mode == 0) RKMF_LAUNCH_SPMV(int64_t, 0);
    else if (mode == 1) RKMF_LAUNCH_SPMV(int64_t, 1);
    else RKMF_LAUNCH_SPMV(int64_t, 2);
  } else {
    if (mode == 0) RKMF_LAUNCH_SPMV(int32_t, 0);
    else if (mode == 1) RKMF_LAUNCH_SPMV(int32_t, 1);
    else RKMF_LAUNCH_SPMV(int32_t, 2);
  }
#undef RKMF_LAUNCH_SPMV
  RKMF_CUDA(cudaGetLastError());
}

namespace {
__global__ void det_finish_kernel(const double* __restrict__ gpart, int ng, int64_t L,
                                  double* out) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < L;
       j += int64_t(gridDim.x) * blockDim.x)
    out[j] = det_group_sum(gpart, ng, L, j);
}
}  // namespace

void launch_det_finish(const DetRed& red, int64_t L, double* out, cudaStream_t st) {
  if (L <= 0) return;
  det_finish_kernel<<<unsigned((L + 127) / 128), 128, 0, st>>>(red.gpart, red.groups, L, out);
  RKMF_CUDA(cudaGetLastError());
}

// ---- setup kernels: norm1 (sparse.cpp:97-102) and validate (sparse.cpp:61-81) ----
namespace {

// Column abs-sums for norm1 in fixed point, so that the result does not
// depend on the order in which threads add (bitwise reproducible solves; the
// breakdown threshold 1e-14 ||A||_1 and the fixed-node InvSqrt interval read
// it). With 2^E > max |a_ij| every |a_ij| 2^-E in [0, 1) is split into two
// 40-bit integer words (bits 2^-1..2^-40 and 2^-41..2^-80) added with
// integer atomics: exact and order-free for columns of < 2^24 entries; bits
// below 2^-80 max|a_ij| are dropped. The reference sums each column in row
// order (sparse.cpp:97-102); the two agree to about one rounding.
__global__ void absmax_bits_kernel(int64_t nnz, const double* __restrict__ val,
                                   unsigned long long* out) {
  double m = 0.0;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x)
    m = fmax(m, fabs(val[k]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0)  // non-negative doubles order like their bit patterns
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__device__ __forceinline__ int fx_exponent(const unsigned long long* vmax_bits) {
  const double vm = __longlong_as_double((long long)*vmax_bits);
  return vm > 0.0 ? ilogb(vm) + 1 : 0;  // 2^E > vmax
}

__global__ void fx_colsum_kernel(int64_t nnz, const int32_t* __restrict__ ci,
                                 const double* __restrict__ val,
                                 const unsigned long long* vmax_bits, unsigned long long* hi,
                                 unsigned long long* lo) {
  const int E = fx_exponent(vmax_bits);
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz;
       k += int64_t(gridDim.x) * blockDim.x) {
    const double a = ldexp(fabs(val[k]), 40 - E);  // < 2^40
    const double h = floor(a);
    const double l = floor((a - h) * 1099511627776.0);  // 2^40
    const int32_t c = ci[k];
    if (h != 0.0) atomicAdd(hi + c, (unsigned long long)h);
    if (l != 0.0) atomicAdd(lo + c, (unsigned long long)l);
  }
}

__global__ void fx_colmax_kernel(int64_t n, const unsigned long long* __restrict__ hi,
                                 const unsigned long long* __restrict__ lo,
                                 const unsigned long long* vmax_bits, double* out) {
  const int E = fx_exponent(vmax_bits);
  double m = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    m = fmax(m, ldexp(double(hi[i]), E - 40) + ldexp(double(lo[i]), E - 80));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(m));
}

__global__ void fx_scatter_add_kernel(int64_t cnt, const int32_t* __restrict__ idx,
                                      const unsigned long long* __restrict__ v,
                                      unsigned long long* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
       i += int64_t(gridDim.x) * blockDim.x)
    if (v[i]) atomicAdd(out + idx[i], v[i]);
}

// flags[0]: shape violation, flags[1]: non-finite value
template <typename RP>
__global__ void check_kernel(int64_t n_rows, int64_t n_cols, const RP* __restrict__ rp,
                             const int32_t* __restrict__ ci, const double* __restrict__ val,
                             int32_t* flags, int sorted) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t lo = rp[r], hi = rp[r + 1];
    if (hi < lo) { flags[0] = 1; continue; }
    for (int64_t k = lo; k < hi; ++k) {
      const int64_t c = ci[k];
      if (c < 0 || c >= n_cols || (sorted && k > lo && c <= ci[k - 1])) flags[0] = 1;
      if (!isfinite(val[k])) flags[1] = 1;
    }
  }
}

}  // namespace

void launch_abs_max_bits(int64_t nnz, const double* val, unsigned long long* vmax_bits,
                         cudaStream_t st) {
  RKMF_CUDA(cudaMemsetAsync(vmax_bits, 0, sizeof(unsigned long long), st));
  if (nnz > 0) absmax_bits_kernel<<<4 * num_sms(), 256, 0, st>>>(nnz, val, vmax_bits);
  RKMF_CUDA(cudaGetLastError());
}

void launch_fx_colsum(int64_t nnz, const int32_t* col, const double* val,
                      const unsigned long long* vmax_bits, int64_t ncols, unsigned long long* hi,
                      unsigned long long* lo, cudaStream_t st) {
  RKMF_CUDA(cudaMemsetAsync(hi, 0, sizeof(unsigned long long) * size_t(ncols), st));
  RKMF_CUDA(cudaMemsetAsync(lo, 0, sizeof(unsigned long long) * size_t(ncols), st));
  if (nnz > 0) fx_colsum_kernel<<<4 * num_sms(), 256, 0, st>>>(nnz, col, val, vmax_bits, hi, lo);
  RKMF_CUDA(cudaGetLastError());
}

void launch_fx_scatter_add(int64_t cnt, const int32_t* idx, const unsigned long long* v,
                           unsigned long long* out, cudaStream_t st) {
  if (cnt > 0) fx_scatter_add_kernel<<<4 * num_sms(), 256, 0, st>>>(cnt, idx, v, out);
  RKMF_CUDA(cudaGetLastError());
}

void launch_fx_colmax(int64_t n, const unsigned long long* hi, const unsigned long long* lo,
                      const unsigned long long* vmax_bits, double* out, cudaStream_t st) {
  RKMF_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
  if (n > 0) fx_colmax_kernel<<<4 * num_sms(), 256, 0, st>>>(n, hi, lo, vmax_bits, out);
  RKMF_CUDA(cudaGetLastError());
}

// colsum: scratch of 2 * n_cols + 1 words (hi, lo, the max |a_ij| bits)
void launch_matrix_norm1(const CsrView* A, double* colsum, double* out, cudaStream_t st) {
  auto* w = reinterpret_cast<unsigned long long*>(colsum);
  unsigned long long *hi = w, *lo = w + A->n_cols, *vmax = w + 2 * A->n_cols;
  launch_abs_max_bits(A->nnz, A->val, vmax, st);
  launch_fx_colsum(A->nnz, A->col, A->val, vmax, A->n_cols, hi, lo, st);
  launch_fx_colmax(A->n_cols, hi, lo, vmax, out, st);
}

void launch_matrix_check(const CsrView* A, int32_t* flags, bool require_sorted, cudaStream_t st) {
  RKMF_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int32_t), st));
  const int g = 4 * num_sms();
  if (A->n_rows == 0) return;
  if (A->rp64)
    check_kernel<int64_t><<<g, 256, 0, st>>>(A->n_rows, A->n_cols,
                                             static_cast<const int64_t*>(A->row_ptr), A->col,
                                             A->val, flags, require_sorted ? 1 : 0);
  else
    check_kernel<int32_t><<<g, 256, 0, st>>>(A->n_rows, A->n_cols,
                                             static_cast<const int32_t*>(A->row_ptr), A->col,
                                             A->val, flags, require_sorted ? 1 : 0);
  RKMF_CUDA(cudaGetLastError());
}

}  // namespace rkmf_b200
