// Classical restarted Arnoldi on the device (S == nullptr; SURVEY.md §8(f)
// rank 3): the builder of basis.cpp:34-77 under the same restart loop
// (restart.cpp:53-55), so the paper's restart vs restart-rand comparison runs
// on B200 with identical SpMV, dense-f and restart-update kernels.
//
// basis.cpp orthogonalises z = A w_k by modified Gram-Schmidt over n-vectors
// (k+1 sequential dot + axpy pairs). On the GPU every n-length dot is a grid
// reduction, so the sweep is done as classical Gram-Schmidt applied twice
// (CGS2: h1 = W^T z, z -= W h1, h2 = W^T z, z -= W h2, H(:,k) = h1 + h2), which
// reads W four times per step instead of 2(k+1) dependent passes and is
// orthogonal to working precision like MGS (rounding-level differences only).
// Column 0 of W holds the unscaled start; sigma = 1/||start|| is folded into
// every coefficient of column 0, as in the randomized path.
#include <cuda_runtime.h>

#include "rkmf_internal.cuh"

namespace rkmf_b200 {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxCols = 1024;

__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double block_sum_d(double v, double* buf) {
  v = warp_sum_d(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) buf[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int q = 0; q < int(blockDim.x >> 5); ++q) s += buf[q];
  __syncthreads();
  return s;  // valid in thread 0
}

// block sum (valid in thread 0) -> *out in a fixed block order (detred.cuh)
__device__ __forceinline__ void det_scalar(double s, const DetRed& red, double* out) {
  __shared__ double mine[1];
  __shared__ int flag;
  if (threadIdx.x == 0) mine[0] = s;
  __syncthreads();
  det_reduce<kThreads, 0>(red, 1, mine, out, int(threadIdx.x), &flag);
}

// *out = ||x||^2
__global__ void norm2_kernel(int64_t n, const double* __restrict__ x, double* out, DetRed red) {
  __shared__ double buf[kThreads / 32];
  double s = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kThreads + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kThreads)
    s += x[i] * x[i];
  s = block_sum_d(s, buf);
  det_scalar(s, red, out);
}

// beta = ||start|| (basis.cpp:38-40); the same state fields as start_init
__global__ void cl_start_kernel(double* nrm2, SolveState* st, int first, int m_eff) {
  const double alpha = sqrt(*nrm2);
  *nrm2 = 0.0;
  st->alpha_k = alpha;
  st->sigma = 1.0 / alpha;
  if (first) st->alpha1 = alpha;
  st->zero_start = alpha == 0.0;
  st->stopped = m_eff;
  st->breakdown = 0;
  st->nonfinite = 0;
  st->yn2 = 0.0;
  st->err2 = 0.0;
}

// h[i] = <W[:,i], z> for i <= k; blockIdx.y = column (one reduction slice
// each), grid-stride over rows
__global__ void multidot_kernel(int64_t n, int k, int64_t ldw, const double* __restrict__ W,
                                const double* __restrict__ z, double* h, const SolveState* st,
                                DetRed red) {
  if (st->stopped <= k) return;
  __shared__ double buf[kThreads / 32];
  const int i = blockIdx.y;
  const double* w = W + int64_t(i) * ldw;
  const int64_t n2 = n / 2;
  double s = 0.0;
  for (int64_t r = int64_t(blockIdx.x) * kThreads + threadIdx.x; r < n2;
       r += int64_t(gridDim.x) * kThreads) {
    const double2 a = __ldcs(reinterpret_cast<const double2*>(w) + r);
    const double2 b = reinterpret_cast<const double2*>(z)[r];
    s += a.x * b.x + a.y * b.y;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) s += w[n - 1] * z[n - 1];
  s = block_sum_d(s, buf);
  det_scalar(i == 0 ? s * st->sigma : s, red, h + i);
}

// z -= W[:,0..k] h (store != 0), and *nrm2 = ||z - W h||^2 when nrm2 != null
__global__ void cgs_update_kernel(int64_t n, int k, int64_t ldw, const double* __restrict__ W,
                                  double* z, const double* __restrict__ h, double* nrm2,
                                  int store, const SolveState* st, DetRed red) {
  if (st->stopped <= k) return;
  __shared__ double coef[kMaxCols];
  __shared__ double buf[kThreads / 32];
  for (int c = threadIdx.x; c <= k; c += kThreads) coef[c] = h[c] * (c == 0 ? st->sigma : 1.0);
  __syncthreads();
  const int64_t n2 = n / 2;
  double ss = 0.0;
  for (int64_t r = int64_t(blockIdx.x) * kThreads + threadIdx.x; r < n2;
       r += int64_t(gridDim.x) * kThreads) {
    double a0 = 0.0, a1 = 0.0;
    int c = 0;
    for (; c + 3 <= k; c += 4) {
      double2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        v[q] = __ldcs(reinterpret_cast<const double2*>(W + int64_t(c + q) * ldw) + r);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a0 += v[q].x * coef[c + q];
        a1 += v[q].y * coef[c + q];
      }
    }
    for (; c <= k; ++c) {
      const double2 v = __ldcs(reinterpret_cast<const double2*>(W + int64_t(c) * ldw) + r);
      a0 += v.x * coef[c];
      a1 += v.y * coef[c];
    }
    double2 zz = reinterpret_cast<const double2*>(z)[r];
    zz.x -= a0;
    zz.y -= a1;
    if (store) reinterpret_cast<double2*>(z)[r] = zz;
    ss += zz.x * zz.x + zz.y * zz.y;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double a = 0.0;
    for (int c = 0; c <= k; ++c) a += W[int64_t(c) * ldw + n - 1] * coef[c];
    const double v = z[n - 1] - a;
    if (store) z[n - 1] = v;
    ss += v * v;
  }
  if (nrm2) {
    ss = block_sum_d(ss, buf);
    det_scalar(ss, red, nrm2);
  }
}

// H(0..k, k) = h1 + h2, H(k+1, k) = beta = ||z||, breakdown test
// (basis.cpp:57-69); the last step also writes (h2, beta) into rlast's column
// k for the fused final update. Re-zeroes the accumulators.
__global__ void cl_decide_kernel(int k, int64_t ldr, int64_t n_global, double tol, double* h1,
                                 double* h2, double* nrm2, double* Rbar, double* rlast,
                                 SolveState* st) {
  if (st->stopped <= k) return;
  const double beta = sqrt(*nrm2);
  for (int i = threadIdx.x; i <= k; i += blockDim.x) {
    Rbar[int64_t(k) * ldr + i] = h1[i] + h2[i];
    if (rlast) rlast[int64_t(k) * ldr + i] = h2[i];
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= k; i += blockDim.x) h1[i] = h2[i] = 0.0;
  if (threadIdx.x == 0) {
    *nrm2 = 0.0;
    if (beta <= tol || int64_t(k) + 1 == n_global) {
      st->stopped = k + 1;
      st->breakdown = k + 1;
    } else {
      Rbar[int64_t(k) * ldr + k + 1] = beta;
      if (rlast) rlast[int64_t(k) * ldr + k + 1] = beta;
    }
  }
}

// W[:,k+1] = z / H(k+1, k)
__global__ void cl_scale_kernel(int64_t n, int k, int64_t ldw, double* W, const double* z,
                                const double* Rbar, int64_t ldr, const SolveState* st) {
  if (st->stopped <= k) return;
  const double inv = 1.0 / Rbar[int64_t(k) * ldr + k + 1];
  double* out = W + int64_t(k + 1) * ldw;
  for (int64_t i = int64_t(blockIdx.x) * kThreads + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kThreads)
    out[i] = z[i] * inv;
}

int grid_rows(int64_t n) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return int(std::max<int64_t>(1, std::min<int64_t>((n / 2 + kThreads - 1) / kThreads, 8 * sms)));
}

}  // namespace

void check_red(const DetRed& red, int64_t blocks, int64_t slices) {
  if (blocks * slices > red.max_blocks || red.max_len < 1 ||
      (det_groups(int(blocks)) + 1) * slices > red.max_groups)
    param_error("internal: classical reduction scratch too small");
}

void launch_cl_start(int64_t n, const double* start, double* nrm2_scratch, SolveState* st_dev,
                     bool first, int m_eff, bool norm_only, const DetRed& red, cudaStream_t st) {
  if (norm_only) {
    const int g = grid_rows(2 * n);
    check_red(red, g, 1);
    norm2_kernel<<<g, kThreads, 0, st>>>(n, start, nrm2_scratch, red);
  } else {
    cl_start_kernel<<<1, 1, 0, st>>>(nrm2_scratch, st_dev, first ? 1 : 0, m_eff);
  }
  RKMF_CUDA(cudaGetLastError());
}

void launch_cl_multidot(int64_t n, int k, int64_t ldw, const double* W, const double* z,
                        double* h, const SolveState* st_dev, const DetRed& red, cudaStream_t st) {
  if (k + 1 > kMaxCols) param_error("arnoldi: m > 1024 is not supported on device");
  const int gx = std::max(1, grid_rows(n) / std::max(1, (k + 1) / 4 + 1));
  check_red(red, gx, k + 1);
  multidot_kernel<<<dim3(unsigned(gx), unsigned(k + 1)), kThreads, 0, st>>>(n, k, ldw, W, z, h,
                                                                             st_dev, red);
  RKMF_CUDA(cudaGetLastError());
}

void launch_cl_update(int64_t n, int k, int64_t ldw, const double* W, double* z, const double* h,
                      double* nrm2, bool store, const SolveState* st_dev, const DetRed& red,
                      cudaStream_t st) {
  const int g = grid_rows(n);
  if (nrm2) check_red(red, g, 1);
  cgs_update_kernel<<<g, kThreads, 0, st>>>(n, k, ldw, W, z, h, nrm2, store ? 1 : 0, st_dev, red);
  RKMF_CUDA(cudaGetLastError());
}

void launch_cl_decide(int k, int64_t ldr, int64_t n_global, double tol, double* h1, double* h2,
                      double* nrm2, double* Rbar, double* rlast, SolveState* st_dev,
                      cudaStream_t st) {
  cl_decide_kernel<<<1, 128, 0, st>>>(k, ldr, n_global, tol, h1, h2, nrm2, Rbar, rlast, st_dev);
  RKMF_CUDA(cudaGetLastError());
}

void launch_cl_scale(int64_t n, int k, int64_t ldw, double* W, const double* z,
                     const double* Rbar, int64_t ldr, const SolveState* st_dev, cudaStream_t st) {
  cl_scale_kernel<<<grid_rows(2 * n), kThreads, 0, st>>>(n, k, ldw, W, z, Rbar, ldr, st_dev);
  RKMF_CUDA(cudaGetLastError());
}

}  // namespace rkmf_b200
