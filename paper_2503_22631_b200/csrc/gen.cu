// On-device generators of the BASELINE matrices.
//
// cfg5 (Q1 hexahedral stiffness on 512^3 nodes, 3.6e9 nonzeros, int64 row
// pointers) is too large to build on the host and push over PCIe, so the
// matrix is written straight into HBM: the row pointers in closed form, then
// one thread per row fills its stencil in increasing column order. The
// entries are the same formulas as the host generators in problems.cpp
// (Q1: A_ij = h Khat(D) sum of the shared element coefficients; Laplacian:
// 5/7-point with h^-2 scaling), so a device-generated matrix equals the host
// one (bit-identical for the constant-coefficient and Laplacian cases; the
// lognormal coefficients go through the device exp/log/cos and agree to an
// ulp or so). The result is an ordinary rkmf_matrix (validated, norm1 cached).
#include <cuda_runtime.h>

#include <cmath>

#include "engine_types.cuh"

namespace rkmf_b200 {

// 5/7-point stencil values per axis (lower / upper neighbour) and diagonal;
// the Laplacian's are -1/h^2 and 2 dim/h^2
struct StencilVals {
  double lower[3], upper[3], diag;
};

namespace {

__device__ __forceinline__ uint64_t g_next(uint64_t& s) {  // rng.hpp:21-26
  uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double g_unit(uint64_t& s) {
  return double(g_next(s) >> 11) * 0x1.0p-53;
}
__device__ double g_gaussian(uint64_t seed, uint64_t i) {  // rng.hpp:47-59
  uint64_t s = seed ^ (0xA0761D6478BD642FULL + i * 0xE7037ED1A0B428DBULL);
  s = g_next(s);
  double u1 = g_unit(s);
  while (u1 <= 0.0) u1 = g_unit(s);
  const double u2 = g_unit(s);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

// prefix of the per-coordinate stencil span (2 at the ends, 3 inside)
__device__ __forceinline__ int64_t span_prefix(int64_t k, int64_t N) {
  return k == 0 ? 0 : 2 + 3 * (k - 1) - (k == N ? 1 : 0);
}
__device__ __forceinline__ int64_t span1(int64_t k, int64_t N) {
  return int64_t(k > 0) + 1 + int64_t(k < N - 1);
}

// rp[r] for the 27-point pattern on N^3 nodes, closed form:
// rp(x,y,z) = A(x) T^2 + s(x) (A(y) T + s(y) A(z)), T = 3N - 2
__device__ __forceinline__ int64_t q1_rp(int64_t r, int64_t N) {
  const int64_t n = N * N * N, T = 3 * N - 2;
  if (r == n) return T * T * T;
  const int64_t x = r / (N * N), y = (r / N) % N, z = r % N;
  return span_prefix(x, N) * T * T +
         span1(x, N) * (span_prefix(y, N) * T + span1(y, N) * span_prefix(z, N));
}
// local row pointers of rows [rb, re): rp[i] = rp(rb + i) - rp(rb)
__global__ void q1_rowptr_kernel(int64_t N, int64_t rb, int64_t re, int64_t* rp) {
  const int64_t base = q1_rp(rb, N);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= re - rb;
       i += int64_t(gridDim.x) * blockDim.x)
    rp[i] = q1_rp(rb + i, N) - base;
}

__global__ void kappa_kernel(int64_t E3, uint64_t seed, double* kappa) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < E3;
       e += int64_t(gridDim.x) * blockDim.x)
    kappa[e] = exp(g_gaussian(seed, uint64_t(e)));
}

// problems.cpp rkmf_gen_q1_hex, one thread per row, rows [rb, re). Columns
// are stored in the local numbering of a row block (comm.cu): owned c -> c -
// rb, the lower halo [rb - nlo, rb) -> n_local + (c - rb + nlo), the upper
// halo [re, ...) -> n_local + nlo + (c - re); rb = 0, re = n, nlo = 0 is the
// whole matrix in global numbering.
__global__ void q1_fill_kernel(int64_t N, const double* __restrict__ kappa, int dirichlet,
                               int64_t rb, int64_t re, int64_t nlo,
                               const int64_t* __restrict__ rp, int32_t* __restrict__ ci,
                               double* __restrict__ v) {
  const int64_t E = N - 1, n_local = re - rb;
  const double h = 1.0 / double(N - 1);
  const double khat[4] = {1.0 / 3.0, 0.0, -1.0 / 12.0, -1.0 / 12.0};
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_local;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = rb + i;
    const int64_t x = r / (N * N), y = (r / N) % N, z = r % N;
    auto bnd = [&](int64_t X, int64_t Y, int64_t Z) {
      return X == 0 || Y == 0 || Z == 0 || X == N - 1 || Y == N - 1 || Z == N - 1;
    };
    const bool brow = dirichlet && bnd(x, y, z);
    int64_t k = rp[i];
    for (int dx = -1; dx <= 1; ++dx) {
      const int64_t X = x + dx;
      if (X < 0 || X >= N) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int64_t Y = y + dy;
        if (Y < 0 || Y >= N) continue;
        for (int dz = -1; dz <= 1; ++dz) {
          const int64_t Z = z + dz;
          if (Z < 0 || Z >= N) continue;
          const int64_t c = (X * N + Y) * N + Z;
          double val;
          if (dirichlet && (brow || bnd(X, Y, Z))) {
            val = (c == r) ? 1.0 : 0.0;
          } else {
            const int D = (dx != 0) + (dy != 0) + (dz != 0);
            double ksum = 0.0;
            const int64_t ox0 = dx ? min(x, X) : x - 1, ox1 = dx ? min(x, X) : x;
            const int64_t oy0 = dy ? min(y, Y) : y - 1, oy1 = dy ? min(y, Y) : y;
            const int64_t oz0 = dz ? min(z, Z) : z - 1, oz1 = dz ? min(z, Z) : z;
            for (int64_t ox = (ox0 > 0 ? ox0 : int64_t(0)); ox <= min(E - 1, ox1); ++ox)
              for (int64_t oy = (oy0 > 0 ? oy0 : int64_t(0)); oy <= min(E - 1, oy1); ++oy)
                for (int64_t oz = (oz0 > 0 ? oz0 : int64_t(0)); oz <= min(E - 1, oz1); ++oz)
                  ksum += kappa ? kappa[(ox * E + oy) * E + oz] : 1.0;
            val = h * khat[D] * ksum;
          }
          const int64_t cl = c < rb ? n_local + (c - rb + nlo)
                                    : (c < re ? c - rb : n_local + nlo + (c - re));
          ci[k] = int32_t(cl);
          v[k++] = val;
        }
      }
    }
  }
}

// problems.cpp rkmf_gen_laplacian: row lengths, then entries
__global__ void lap_len_kernel(int dim, int64_t N, int64_t* len) {
  const int64_t n = dim == 2 ? N * N : N * N * N;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    int64_t c[3];
    if (dim == 2) { c[0] = r / N; c[1] = r % N; c[2] = 0; }
    else { c[0] = r / (N * N); c[1] = (r / N) % N; c[2] = r % N; }
    int64_t l = 1;
    for (int a = 0; a < dim; ++a) l += (c[a] > 0) + (c[a] < N - 1);
    len[r] = l;
  }
}

__global__ void lap_fill_kernel(int dim, int64_t N, const int64_t* __restrict__ rp,
                                int32_t* __restrict__ ci, double* __restrict__ v,
                                StencilVals sv) {
  const int64_t n = dim == 2 ? N * N : N * N * N;
  const int64_t stride[3] = {dim == 2 ? N : N * N, dim == 2 ? 1 : N, 1};
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    int64_t c[3];
    if (dim == 2) { c[0] = r / N; c[1] = r % N; c[2] = 0; }
    else { c[0] = r / (N * N); c[1] = (r / N) % N; c[2] = r % N; }
    int64_t k = rp[r];
    for (int a = 0; a < dim; ++a)
      if (c[a] > 0) { ci[k] = int32_t(r - stride[a]); v[k++] = sv.lower[a]; }
    ci[k] = int32_t(r);
    v[k++] = sv.diag;
    for (int a = dim - 1; a >= 0; --a)
      if (c[a] < N - 1) { ci[k] = int32_t(r + stride[a]); v[k++] = sv.upper[a]; }
  }
}

// inclusive scan of len into rp[1..n] (rp[0] = 0): one block per chunk of
// rows, sequential inside the chunk, then the chunk offsets (small)
__global__ void chunk_sum_kernel(int64_t n, int64_t chunk, const int64_t* len, int64_t* sums) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t lo = c * chunk, hi = min(n, lo + chunk);
  if (lo >= n) return;
  int64_t s = 0;
  for (int64_t r = lo; r < hi; ++r) s += len[r];
  sums[c] = s;
}
__global__ void chunk_write_kernel(int64_t n, int64_t chunk, const int64_t* len,
                                   const int64_t* offs, int64_t* rp) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t lo = c * chunk, hi = min(n, lo + chunk);
  if (lo >= n) return;
  int64_t s = offs[c];
  for (int64_t r = lo; r < hi; ++r) { s += len[r]; rp[r + 1] = s; }
  if (c == 0) rp[0] = 0;
}

__global__ void gaussian_kernel(uint64_t seed, int64_t i0, int64_t n, double* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = g_gaussian(seed, uint64_t(i0 + i));
}

int grid_for(int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32)));
}

template <class F>
int guarded_g(rkmf_context* ctx, F&& fn) {
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

// col/val allocations owned by the matrix afterwards (with the TMA padding)
struct GenArrays {
  int64_t* rp = nullptr;
  int32_t* ci = nullptr;
  double* v = nullptr;
  void alloc(int64_t n, int64_t nnz, cudaStream_t st) {
    rp_only(n);
    colval(nnz, st);
  }
  void rp_only(int64_t n) { RKMF_CUDA(cudaMalloc(&rp, sizeof(int64_t) * size_t(n + 1))); }
  void colval(int64_t nnz, cudaStream_t st) {
    RKMF_CUDA(cudaMalloc(&ci, sizeof(int32_t) * size_t(nnz + kNnzPad)));
    RKMF_CUDA(cudaMalloc(&v, sizeof(double) * size_t(nnz + kNnzPad)));
    RKMF_CUDA(cudaMemsetAsync(ci + nnz, 0, sizeof(int32_t) * kNnzPad, st));
    RKMF_CUDA(cudaMemsetAsync(v + nnz, 0, sizeof(double) * kNnzPad, st));
  }
  void release_all() {
    if (rp) cudaFree(rp);
    if (ci) cudaFree(ci);
    if (v) cudaFree(v);
    rp = nullptr;
    ci = nullptr;
    v = nullptr;
  }
};

rkmf_matrix* adopt(rkmf_context* ctx, int64_t n, int64_t n_cols, int64_t nnz, GenArrays& g,
                   bool sorted = true) {
  rkmf_matrix* M = nullptr;
  try {
    M = create_from_device_rp64(ctx, n, n_cols, nnz, g.rp, g.ci, g.v, false, sorted);
  } catch (...) {
    g.release_all();
    throw;
  }
  RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
  RKMF_CUDA(cudaFree(g.rp));  // the matrix keeps its own (possibly narrowed) copy
  return M;
}

// The 5/7-point pattern (problems.cpp rkmf_gen_laplacian order: -x, -y, -z,
// self, +z, +y, +x) with the values sv (null: the h^-2 Laplacian)
rkmf_matrix* gen_stencil7(rkmf_context* ctx, int dim, int64_t N, int64_t nnz,
                          const StencilVals* svp) {
  const int64_t n = dim == 2 ? N * N : N * N * N;
  StencilVals sv;
  if (svp) {
    sv = *svp;
  } else {
    const double h = 1.0 / double(N + 1), s = 1.0 / (h * h);
    for (int a = 0; a < 3; ++a) sv.lower[a] = sv.upper[a] = -s;
    sv.diag = 2.0 * dim * s;
  }
  cudaStream_t st = ctx->stream;
  GenArrays g;
  int64_t *len = nullptr, *sums = nullptr;
  try {
    g.alloc(n, nnz, st);
    RKMF_CUDA(cudaMallocAsync(&len, sizeof(int64_t) * size_t(n), st));
    lap_len_kernel<<<grid_for(n), 256, 0, st>>>(dim, N, len);
    const int64_t chunk = 1024, nch = (n + chunk - 1) / chunk;
    RKMF_CUDA(cudaMallocAsync(&sums, sizeof(int64_t) * size_t(nch), st));
    chunk_sum_kernel<<<unsigned((nch + 255) / 256), 256, 0, st>>>(n, chunk, len, sums);
    std::vector<int64_t> hs(static_cast<size_t>(nch));
    RKMF_CUDA(cudaMemcpyAsync(hs.data(), sums, sizeof(int64_t) * size_t(nch),
                              cudaMemcpyDeviceToHost, st));
    RKMF_CUDA(cudaStreamSynchronize(st));
    int64_t acc = 0;
    for (auto& x : hs) { const int64_t v = x; x = acc; acc += v; }
    if (acc != nnz) throw Error(RKMF_INTERNAL_ERROR, "gen_stencil7: nnz mismatch");
    RKMF_CUDA(cudaMemcpyAsync(sums, hs.data(), sizeof(int64_t) * size_t(nch),
                              cudaMemcpyHostToDevice, st));
    chunk_write_kernel<<<unsigned((nch + 255) / 256), 256, 0, st>>>(n, chunk, len, sums, g.rp);
    lap_fill_kernel<<<grid_for(n), 256, 0, st>>>(dim, N, g.rp, g.ci, g.v, sv);
    RKMF_CUDA(cudaGetLastError());
    RKMF_CUDA(cudaFreeAsync(len, st));
    RKMF_CUDA(cudaFreeAsync(sums, st));
    RKMF_CUDA(cudaStreamSynchronize(st));  // hs is a host staging buffer
    len = sums = nullptr;
    ctx->launches += 4;
  } catch (...) {
    if (len) cudaFree(len);
    if (sums) cudaFree(sums);
    g.release_all();
    throw;
  }
  return adopt(ctx, n, n, nnz, g);
}

}  // namespace

// Rows [rb, re) of the Q1 matrix on N^3 nodes in the local numbering of
// q1_fill_kernel (nlo / nhi: lower / upper halo sizes; the whole matrix is
// rb = 0, re = N^3, nlo = nhi = 0).
rkmf_matrix* gen_q1_rows(rkmf_context* ctx, int64_t N, int lognormal, uint64_t coef_seed,
                         int dirichlet, int64_t rb, int64_t re, int64_t nlo, int64_t nhi) {
  const int64_t n = N * N * N, n_local = re - rb;
  if (n >= (int64_t(1) << 31)) param_error("gen_q1_hex: n must fit int32 column indices");
  cudaStream_t st = ctx->stream;
  GenArrays g;
  double* kappa = nullptr;
  int64_t nnz = 0;
  try {
    g.rp_only(n_local);
    q1_rowptr_kernel<<<grid_for(n_local + 1), 256, 0, st>>>(N, rb, re, g.rp);
    RKMF_CUDA(cudaGetLastError());
    RKMF_CUDA(cudaMemcpyAsync(&nnz, g.rp + n_local, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RKMF_CUDA(cudaStreamSynchronize(st));
    g.colval(nnz, st);
    if (lognormal) {
      const int64_t E3 = (N - 1) * (N - 1) * (N - 1);
      RKMF_CUDA(cudaMallocAsync(&kappa, sizeof(double) * size_t(E3), st));
      kappa_kernel<<<grid_for(E3), 256, 0, st>>>(E3, coef_seed, kappa);
    }
    q1_fill_kernel<<<grid_for(n_local), 256, 0, st>>>(N, kappa, dirichlet, rb, re, nlo, g.rp, g.ci,
                                                       g.v);
    RKMF_CUDA(cudaGetLastError());
    if (kappa) RKMF_CUDA(cudaFreeAsync(kappa, st));
    kappa = nullptr;
    ctx->launches += lognormal ? 3 : 2;
  } catch (...) {
    if (kappa) cudaFree(kappa);
    g.release_all();
    throw;
  }
  // a lower halo renumbers columns past the owned ones: rows not monotone
  return adopt(ctx, n_local, n_local + nlo + nhi, nnz, g, nlo == 0);
}

}  // namespace rkmf_b200

using namespace rkmf_b200;

extern "C" {

int rkmf_matrix_gen_q1_hex(rkmf_context* ctx, int64_t N, int32_t lognormal, uint64_t coef_seed,
                           int32_t dirichlet, rkmf_matrix** out) {
  return guarded_g(ctx, [&] {
    RKMF_CUDA(cudaSetDevice(ctx->device));
    if (N < 2) param_error("gen_q1_hex: N must be >= 2");
    *out = gen_q1_rows(ctx, N, lognormal, coef_seed, dirichlet, 0, N * N * N, 0, 0);
  });
}

// 3D upwind convection-diffusion (problems.cpp rkmf_gen_convdiff_upwind) in
// HBM: the same entries bit-for-bit (the stencil values are formed on the
// host by the same expressions and passed in)
int rkmf_matrix_gen_convdiff(rkmf_context* ctx, int64_t N, double peclet, double vx, double vy,
                             double vz, rkmf_matrix** out) {
  return guarded_g(ctx, [&] {
    RKMF_CUDA(cudaSetDevice(ctx->device));
    if (N < 1 || !(peclet > 0.0)) param_error("gen_convdiff: N >= 1 and peclet > 0");
    const int64_t n = N * N * N, nnz = 7 * N * N * N - 6 * N * N;
    if (n >= (int64_t(1) << 31)) param_error("gen_convdiff: n must fit int32 column indices");
    const double h = 1.0 / double(N + 1);
    const double vel[3] = {vx, vy, vz};
    const double vmax = std::max(std::fabs(vx), std::max(std::fabs(vy), std::fabs(vz)));
    const double eps = vmax * h / (2.0 * peclet);
    const double dif = eps / (h * h);
    StencilVals sv;
    sv.diag = 6.0 * dif;
    for (int a = 0; a < 3; ++a) sv.diag += std::fabs(vel[a]) / h;
    for (int a = 0; a < 3; ++a) {
      sv.lower[a] = -dif - (vel[a] > 0 ? vel[a] / h : 0.0);
      sv.upper[a] = -dif + (vel[a] < 0 ? vel[a] / h : 0.0);
    }
    *out = gen_stencil7(ctx, 3, N, nnz, &sv);
  });
}

int rkmf_matrix_gen_laplacian(rkmf_context* ctx, int32_t dim, int64_t N, rkmf_matrix** out) {
  return guarded_g(ctx, [&] {
    RKMF_CUDA(cudaSetDevice(ctx->device));
    if ((dim != 2 && dim != 3) || N < 1) param_error("gen_laplacian: dim 2|3, N >= 1");
    const int64_t n = dim == 2 ? N * N : N * N * N;
    const int64_t nnz = dim == 2 ? 5 * N * N - 4 * N : 7 * N * N * N - 6 * N * N;
    if (n >= (int64_t(1) << 31)) param_error("gen_laplacian: n must fit int32 column indices");
    *out = gen_stencil7(ctx, dim, N, nnz, nullptr);
  });
}

}  // extern "C"

extern "C" int rkmf_gen_gaussian_device(rkmf_context* ctx, uint64_t seed, int64_t i0, int64_t n,
                                        double* d_out) {
  return guarded_g(ctx, [&] {
    RKMF_CUDA(cudaSetDevice(ctx->device));
    if (i0 < 0 || n < 0) param_error("gen_gaussian_device: bad range");
    if (n == 0) return;
    gaussian_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(seed, i0, n, d_out);
    RKMF_CUDA(cudaGetLastError());
    RKMF_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->launches++;
  });
}
