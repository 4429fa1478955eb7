// The K3 unit lower-triangular solve (warp 0, c in registers, r_i broadcast
// by shuffle) in isolation, timed with clock64.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void solve(int kk, const double* G, double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* Gs = sm;
  double* cs = Gs + kk * (kk - 1) / 2 + 2;
  for (int q = threadIdx.x; q < kk * (kk - 1) / 2; q += blockDim.x) Gs[q] = G[q];
  for (int q = threadIdx.x; q < kk; q += blockDim.x) cs[q] = 1.0 + q;
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  long long t0 = clock64();
  if (w == 0) {
    const int m0 = l, m1 = l + 32;
    const long long g0 = (long long)m0 * (m0 - 1) / 2, g1 = (long long)m1 * (m1 - 1) / 2;
    double c0 = m0 < kk ? cs[m0] : 0.0, c1 = m1 < kk ? cs[m1] : 0.0;
    for (int i = 0; i < kk; ++i) {
      const double a0 = (m0 > i && m0 < kk) ? Gs[g0 + i] : 0.0;
      const double a1 = (m1 > i && m1 < kk) ? Gs[g1 + i] : 0.0;
      const double ri = __shfl_sync(0xffffffffu, i < 32 ? c0 : c1, i & 31);
      if (m0 > i) c0 -= a0 * ri;
      if (m1 > i) c1 -= a1 * ri;
    }
    if (m0 < kk) cs[m0] = c0;
    if (m1 < kk) cs[m1] = c1;
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    out[0] = cs[kk - 1];
  }
}

int main() {
  const int kk = 50;
  double* G;
  double* out;
  long long* cyc;
  cudaMallocManaged(&G, sizeof(double) * kk * kk);
  cudaMallocManaged(&out, 8);
  cudaMallocManaged(&cyc, 8);
  for (int i = 0; i < kk * kk; ++i) G[i] = 1e-9 * (i % 7);
  for (int rep = 0; rep < 3; ++rep) {
    solve<<<1, 256, 48 * 1024>>>(kk, G, out, cyc);
    cudaDeviceSynchronize();
    printf("kk=%d: %lld cycles (%.1f per step)  %s\n", kk, cyc[0], double(cyc[0]) / kk,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
