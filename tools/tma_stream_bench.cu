// Microbenchmark: how fast can a ring of cp.async.bulk copies stream HBM into
// shared memory, as a function of bytes per stage, copies per stage, stages
// and resident blocks? (The K2 pipeline's producer/consumer skeleton with the
// consumer doing nothing but releasing the stage.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_tma_stream_bench tools/tma_stream_bench.cu
//   tools/_tma_stream_bench
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT;\n}\n" ::"r"(su32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LAB_SPIN:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_SPIN;\n}\n" ::"r"(su32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

constexpr int kMaxStages = 16;

__global__ void stream_kernel(const unsigned char* src, int64_t tiles, uint32_t tile_bytes,
                              int copies, int stages, double* sink, int mode) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mode == 8 ? 128 : (mode >= 9 ? 4 : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t piece = tile_bytes / copies;
  // mode 4/5: P producer threads (lane 0 of warps 2..), producer p owns
  // stages s with s % P == p and no consumer (reuse after landing)
  if (mode >= 8) {  // one producer (t == 0), 4 consumer warps (t in [32, 160))
    if (t == 0) {
      int s = 0, it = 0;
      uint32_t eph = 0;
      for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
        if (it >= stages) mbar_wait(&empty[s], eph);
        unsigned char* st = smem + size_t(s) * tile_bytes;
        mbar_expect_tx(&full[s], tile_bytes);
        bulk_g2s(st, src + tile * int64_t(tile_bytes), tile_bytes, &full[s]);
        if (++s == stages) {
          s = 0;
          if (it >= stages) eph ^= 1u;
        }
      }
      return;
    }
    if (t < 32 || t >= 160) return;
    const int l = t & 31;
    int s = 0;
    uint32_t ph = 0;
    double acc = 0.0;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      if (mode == 10) {
        if (l == 0) mbar_wait(&full[s], ph);
        __syncwarp();
      } else {
        mbar_wait(&full[s], ph);
      }
      acc += reinterpret_cast<const double*>(smem + size_t(s) * tile_bytes)[t - 32];
      if (mode == 8) {
        mbar_arrive(&empty[s]);
      } else {
        __syncwarp();
        if (l == 0) mbar_arrive(&empty[s]);
      }
      if (++s == stages) {
        s = 0;
        ph ^= 1u;
      }
    }
    if (acc == 12345.0) *sink = acc;
    return;
  }
  if (mode >= 4) {
    const int P = mode == 5 ? 4 : 2;
    // mode 4/5: lane 0 of warps 2.. ; mode 6: lanes 0..1 of warp 2 ; mode 7:
    // lanes 0 and 16 of warp 2
    int w;
    if (mode <= 5) {
      w = t / 32 - 2;
      if ((t & 31) || w < 0 || w >= P) return;
    } else {
      if (t / 32 != 2) return;
      const int l = t & 31;
      if (mode == 6 && l >= 2) return;
      if (mode == 7 && l != 0 && l != 16) return;
      w = mode == 6 ? l : l / 16;
    }
    int it = 0;
    for (int64_t tile = blockIdx.x + int64_t(w) * gridDim.x; tile < tiles;
         tile += int64_t(P) * gridDim.x, ++it) {
      const int k = it % (stages / P), s = w + P * k;
      if (it >= stages / P) mbar_wait(&full[s], uint32_t((it / (stages / P) - 1) & 1));
      unsigned char* st = smem + size_t(s) * tile_bytes;
      mbar_expect_tx(&full[s], tile_bytes);
      bulk_g2s(st, src + tile * int64_t(tile_bytes), tile_bytes, &full[s]);
    }
    return;
  }
  if (t == 0) {  // producer
    int s = 0, it = 0;
    uint32_t eph = 0;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
      if (it >= stages) {
        if (mode == 1) mbar_wait(&full[s], eph);        // no consumer: reuse after landing
        else if (mode == 3) mbar_spin(&empty[s], eph);  // spin with test_wait
        else mbar_wait(&empty[s], eph);
      }
      unsigned char* st = smem + size_t(s) * tile_bytes;
      mbar_expect_tx(&full[s], tile_bytes);
      const unsigned char* g = src + tile * int64_t(tile_bytes);
      for (int c = 0; c < copies; ++c) bulk_g2s(st + c * piece, g + c * piece, piece, &full[s]);
      if (++s == stages) {
        s = 0;
        if (it >= stages) eph ^= 1u;
      }
    }
  } else if (t == 32 && mode != 1) {  // consumer: wait, touch one word, release
    int s = 0;
    uint32_t ph = 0;
    double acc = 0.0;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      if (mode >= 2) mbar_spin(&full[s], ph);
      else mbar_wait(&full[s], ph);
      acc += reinterpret_cast<const double*>(smem + size_t(s) * tile_bytes)[0];
      mbar_arrive(&empty[s]);
      if (++s == stages) {
        s = 0;
        ph ^= 1u;
      }
    }
    if (acc == 12345.0) *sink = acc;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = size_t(1) << 30;
  unsigned char* src = nullptr;
  double* sink = nullptr;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 1, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const uint32_t sizes[] = {2048, 8192};
  const int stages_l[] = {4, 8};
  printf("mode tile_bytes stages blocks/SM  GB/s\n");
  for (int mode = 0; mode < 11; mode += (mode == 0 ? 8 : 1))
    for (uint32_t tb : sizes)
      for (int ns : stages_l)
        for (int per = 1; per <= 2; ++per) {
          const size_t smem = size_t(ns) * tb;
          if (smem * per > 220 * 1024) continue;
          const int64_t tiles = int64_t(total / tb);
          const int grid = per * sms;
          stream_kernel<<<grid, 192, smem>>>(src, tiles, tb, 1, ns, sink, mode);  // warm
          cudaEventRecord(a);
          const int reps = 5;
          for (int r = 0; r < reps; ++r)
            stream_kernel<<<grid, 192, smem>>>(src, tiles, tb, 1, ns, sink, mode);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms = 0;
          cudaEventElapsedTime(&ms, a, b);
          const cudaError_t e = cudaGetLastError();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          printf("%d %6u %2d %2d  %7.0f  (%.0f ns/tile/block)\n", mode, tb, ns, per,
                 double(total) * reps / (ms * 1e6), ms * 1e6 / reps / (double(tiles) / grid));
        }
  return 0;
}
