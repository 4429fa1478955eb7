// Dependent-chain latencies on one warp (clock64): DFMA, SHFL.IDX of a
// double, and the K3 solve's shuffle + DFMA step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_lat_bench tools/lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, int iters, double a, double b) {
  const int l = threadIdx.x;
  double x = a + l;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  double y = x;
  for (int i = 0; i < iters; ++i) y = __shfl_sync(0xffffffffu, y, (l + 1) & 31);
  long long t2 = clock64();
  double c = x;
  for (int i = 0; i < iters; ++i) {
    const double ri = __shfl_sync(0xffffffffu, c, i & 31);
    if (l > (i & 31)) c -= b * ri;
  }
  long long t3 = clock64();
  float f = float(x);
  for (int i = 0; i < iters; ++i) f = fmaf(f, float(b), float(a));
  long long t4 = clock64();
  out[l] = x + y + c + f;
  if (l == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMallocManaged(&cyc, 4 * 8);
  const int iters = 4096;
  lat<<<1, 32>>>(out, cyc, iters, 1e-9, 0.999999);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(out, cyc, iters, 1e-9, 0.999999);
  cudaDeviceSynchronize();
  printf("cycles per dependent op: DFMA %.1f  SHFL(f64) %.1f  shfl+DFMA step %.1f  FFMA %.1f\n",
         double(cyc[0]) / iters, double(cyc[1]) / iters, double(cyc[2]) / iters,
         double(cyc[3]) / iters);
  return 0;
}
