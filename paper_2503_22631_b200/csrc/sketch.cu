// K1: sparse-sign sketch generation on device (setup, integer only).
//
// Restates make_sketch (proj/src/sketch.cpp:13-49) with SplitMix64
// (proj/include/rkmf/rng.hpp:17-63): column j draws from the stream
// derive(seed, j); Floyd's sampling picks zeta distinct rows of d, which are
// sorted ascending; zeta Rademacher signs follow in sorted order. The output is
// bit-identical to the reference definition (checked against the CPU oracle).
//
// Two device layouts are produced:
//   rows/signs  [n][zeta]  uint16 / int8   the operator itself (export, tests)
//   tile layout            per 128-column tile, the d x 128 block of S in CSR
//                          by sketch row ("bin"), bins renumbered into slots by
//                          length: tile_off[tile][tile_off_stride(d)] uint16 =
//                          slot offsets [d+1] + slot bins [d], and
//                          tile_ent[tile][128*zeta] uint8 entries (local column |
//                          sign << 7), entries of a bin sorted by local column.
//                          This is what the fused SpMV epilogue reads: each
//                          thread owns slots and gathers their ~zeta*128/d
//                          contributions from shared memory, so the scatter-add of
//                          sketch.cpp:55-61 becomes a deterministic gather with no
//                          shared-memory atomics (fp64 smem atomics are CAS loops
//                          on sm_100a).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rkmf_internal.cuh"

namespace rkmf_b200 {

namespace {

constexpr int kMaxZeta = 64;

__device__ __forceinline__ uint64_t sm64_next(uint64_t& s) {  // rng.hpp:21-26
  uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t sm64_derive(uint64_t seed, uint64_t tag) {  // rng.hpp:56-59
  uint64_t s = seed ^ (0xA0761D6478BD642FULL + tag * 0xE7037ED1A0B428DBULL);
  return sm64_next(s);
}

// limits[i - (d - zeta)] = bound * (UINT64_MAX / bound) for bound = i + 1
// (rng.hpp:35), precomputed on the host: the 64-bit division runs once per
// distinct bound instead of once per draw.
__global__ void sketch_generate_kernel(int64_t d, int64_t n, int64_t j0, int zeta, uint64_t seed,
                                       const uint64_t* __restrict__ limits,
                                       uint16_t* __restrict__ rows, int8_t* __restrict__ signs) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  uint64_t s = sm64_derive(seed, uint64_t(j0 + j));  // global column j0 + j
  uint16_t chosen[kMaxZeta];
  int cnt = 0;
  for (int64_t i = d - zeta; i < d; ++i) {  // Floyd: sketch.cpp:33-40
    const uint64_t bound = uint64_t(i) + 1;
    const uint64_t limit = limits[i - (d - zeta)];
    uint64_t v;
    do { v = sm64_next(s); } while (v >= limit);  // next_below, rng.hpp:34-41
    const uint16_t t = uint16_t(v % bound);
    bool seen = false;
    for (int q = 0; q < cnt; ++q) seen |= (chosen[q] == t);
    chosen[cnt++] = seen ? uint16_t(i) : t;
  }
  for (int a = 1; a < zeta; ++a) {  // ascending sort, sketch.cpp:41
    const uint16_t key = chosen[a];
    int b = a - 1;
    while (b >= 0 && chosen[b] > key) { chosen[b + 1] = chosen[b]; --b; }
    chosen[b + 1] = key;
  }
  const int64_t base = j * zeta;
  for (int k = 0; k < zeta; ++k) {  // signs in sorted order, sketch.cpp:43-46
    rows[base + k] = chosen[k];
    signs[base + k] = (sm64_next(s) & 1ULL) ? int8_t(1) : int8_t(-1);
  }
}

// One block per 128-column tile: counting sort of the tile's n_tile*zeta
// entries by sketch row ("bin"), a per-bin insertion sort by local column so
// the layout (and hence every sketch sum) is deterministic, then the bins are
// renumbered into "slots" ordered by entry count (descending, ties by bin id).
// Consumers hand slots to threads in snake order (sketch_tile_gather), so the
// 32 bins a warp walks have near-equal lengths and the gather loop does not
// diverge. Output per tile (see tile_off_stride): off[slot 0..d] uint16
// offsets, bin[slot 0..d-1] uint16 sketch rows, and the entries in slot order.
__global__ void sketch_tiles_kernel(int64_t d, int64_t n, int zeta, int64_t off_stride,
                                    const uint16_t* __restrict__ rows,
                                    const int8_t* __restrict__ signs,
                                    uint16_t* __restrict__ tile_off,
                                    uint8_t* __restrict__ tile_ent) {
  extern __shared__ int sh[];
  int* cnt = sh;                   // d + 1: bin offsets
  int* cur = sh + (d + 1);         // d: insertion cursors, then slot of each bin
  int* soff = cur + d;             // d + 1: slot offsets
  uint8_t* ent = reinterpret_cast<uint8_t*>(soff + d + 1);  // kTileRows * zeta
  __shared__ int chunk_sum[kBlock];
  const int64_t tile = blockIdx.x;
  const int t = threadIdx.x;
  const int64_t col = tile * kTileRows + t;
  const bool live = col < n;
  for (int64_t b = t; b <= d; b += blockDim.x) cnt[b] = 0;
  __syncthreads();
  if (live)
    for (int k = 0; k < zeta; ++k) atomicAdd(&cnt[rows[col * zeta + k]], 1);
  __syncthreads();
  // exclusive scan of cnt[0..d) -> cnt (block scan over contiguous chunks)
  const int64_t per = (d + blockDim.x - 1) / blockDim.x;
  const int64_t lo = min(d, int64_t(t) * per), hi = min(d, lo + per);
  int s = 0;
  for (int64_t b = lo; b < hi; ++b) s += cnt[b];
  chunk_sum[t] = s;
  __syncthreads();
  if (t == 0) {
    int acc = 0;
    for (int q = 0; q < blockDim.x; ++q) { const int v = chunk_sum[q]; chunk_sum[q] = acc; acc += v; }
  }
  __syncthreads();
  int run = chunk_sum[t];
  for (int64_t b = lo; b < hi; ++b) { const int v = cnt[b]; cnt[b] = run; cur[b] = run; run += v; }
  if (t == blockDim.x - 1) cnt[d] = run;  // == n_tile * zeta
  __syncthreads();
  if (live)
    for (int k = 0; k < zeta; ++k) {
      const int r = rows[col * zeta + k];
      const int pos = atomicAdd(&cur[r], 1);
      ent[pos] = uint8_t(t | (signs[col * zeta + k] < 0 ? 0x80 : 0));
    }
  __syncthreads();
  for (int64_t b = t; b < d; b += blockDim.x) {  // deterministic order inside a bin
    const int b0 = cnt[b], b1 = cnt[b + 1];
    for (int a = b0 + 1; a < b1; ++a) {
      const uint8_t key = ent[a];
      int q = a - 1;
      while (q >= b0 && (ent[q] & 0x7f) > (key & 0x7f)) { ent[q + 1] = ent[q]; --q; }
      ent[q + 1] = key;
    }
  }
  // slot of bin b = #bins that are longer, or as long with a smaller id
  for (int64_t b = t; b < d; b += blockDim.x) {
    const int cb = cnt[b + 1] - cnt[b];
    int rank = 0;
    for (int64_t q = 0; q < d; ++q) {
      const int cq = cnt[q + 1] - cnt[q];
      rank += (cq > cb) || (cq == cb && q < b);
    }
    cur[b] = rank;
  }
  __syncthreads();
  uint16_t* toff = tile_off + tile * off_stride;
  for (int64_t b = t; b < d; b += blockDim.x) {
    soff[cur[b] + 1] = cnt[b + 1] - cnt[b];
    toff[d + 1 + cur[b]] = uint16_t(b);
  }
  __syncthreads();
  if (t == 0) {
    soff[0] = 0;
    for (int64_t q = 1; q <= d; ++q) soff[q] += soff[q - 1];
  }
  __syncthreads();
  for (int64_t q = t; q <= d; q += blockDim.x) toff[q] = uint16_t(soff[q]);
  for (int64_t q = 2 * d + 1 + t; q < off_stride; q += blockDim.x) toff[q] = 0;
  uint8_t* tent = tile_ent + tile * int64_t(kTileRows) * zeta;
  const int total = cnt[d];
  __syncthreads();  // slot bins (toff) visible to the whole block
  // Entry order inside each slot, bank-aware: the 32 slots of a group are
  // walked by one warp in lockstep (sketch_tile_gather: group = slot / 32), and
  // at position q every lane loads zs2[entry]; the double at index u sits in
  // bank pair (u mod 16) = (row mod 16). Greedily give each lane, position by
  // position, its remaining entry in the least-used bank pair, so the warp's
  // loads spread over the 16 pairs (~2 wavefronts instead of ~4-5). Only the
  // summation order inside a bin changes; the layout stays deterministic.
  const int ngroups = int((d + 31) / 32);
  for (int g = t; g < ngroups; g += blockDim.x) {
    const int s0 = 32 * g, s1 = int(min(d, int64_t(s0) + 32));
    int maxc = 0;
    for (int sl = s0; sl < s1; ++sl) maxc = max(maxc, soff[sl + 1] - soff[sl]);
    if (maxc > 64) {  // unusually long bins: keep the column order
      for (int sl = s0; sl < s1; ++sl) {
        const int b = toff[d + 1 + sl], src = cnt[b], c = soff[sl + 1] - soff[sl];
        for (int e = 0; e < c; ++e) tent[soff[sl] + e] = ent[src + e];
      }
      continue;
    }
    uint64_t used[32];
    for (int l = 0; l < 32; ++l) used[l] = 0;
    for (int q = 0; q < maxc; ++q) {
      int load[16];
      for (int k = 0; k < 16; ++k) load[k] = 0;
      for (int sl = s0; sl < s1; ++sl) {
        const int c = soff[sl + 1] - soff[sl];
        if (q >= c) continue;
        const int src = cnt[toff[d + 1 + sl]];
        int best = -1, bl = 1 << 30;
        for (int e = 0; e < c; ++e) {
          if ((used[sl - s0] >> e) & 1ull) continue;
          const int bank = ent[src + e] & 15;
          if (load[bank] < bl) { bl = load[bank]; best = e; }
        }
        used[sl - s0] |= 1ull << best;
        load[ent[src + best] & 15]++;
        tent[soff[sl] + q] = ent[src + best];
      }
    }
  }
  for (int e = total + t; e < kTileRows * zeta; e += blockDim.x) tent[e] = 0;
}

__global__ void sketch_export_kernel(int64_t count, const uint16_t* __restrict__ rows,
                                     int64_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) out[i] = rows[i];
}

}  // namespace

void launch_sketch_generate(int64_t d, int64_t n, int64_t j0, int64_t zeta, uint64_t seed,
                            uint16_t* rows,
                            int8_t* signs, cudaStream_t st) {
  if (zeta > kMaxZeta) param_error("sketch: zeta > 64 is not supported on device");
  if (d > 65535) param_error("sketch: d > 65535 is not supported on device");
  std::vector<uint64_t> lim(static_cast<size_t>(zeta));
  for (int64_t i = d - zeta; i < d; ++i) {
    const uint64_t bound = uint64_t(i) + 1;
    lim[size_t(i - (d - zeta))] = bound * (UINT64_MAX / bound);
  }
  uint64_t* dl = nullptr;
  RKMF_CUDA(cudaMallocAsync(&dl, sizeof(uint64_t) * size_t(zeta), st));
  RKMF_CUDA(cudaMemcpyAsync(dl, lim.data(), sizeof(uint64_t) * size_t(zeta),
                            cudaMemcpyHostToDevice, st));
  const int threads = 128;
  const int64_t blocks = (n + threads - 1) / threads;
  sketch_generate_kernel<<<unsigned(blocks), threads, 0, st>>>(d, n, j0, int(zeta), seed, dl, rows,
                                                               signs);
  RKMF_CUDA(cudaGetLastError());
  RKMF_CUDA(cudaFreeAsync(dl, st));
}

void launch_sketch_tiles(int64_t d, int64_t n, int64_t zeta, const uint16_t* rows,
                         const int8_t* signs, uint16_t* tile_off, uint8_t* tile_ent,
                         cudaStream_t st) {
  const int64_t tiles = (n + kTileRows - 1) / kTileRows;
  const int64_t off_stride = tile_off_stride(d);
  const size_t smem = sizeof(int) * size_t(3 * d + 2) + size_t(kTileRows * zeta) + 16;
  if (smem > 200 * 1024) param_error("sketch: d too large for the device tile layout");
  if (smem > 48 * 1024)
    RKMF_CUDA(cudaFuncSetAttribute(sketch_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
  sketch_tiles_kernel<<<unsigned(tiles), kBlock, smem, st>>>(d, n, int(zeta), off_stride, rows,
                                                              signs, tile_off, tile_ent);
  RKMF_CUDA(cudaGetLastError());
}

void launch_sketch_export(int64_t count, const uint16_t* rows, const int8_t* /*signs*/,
                          int64_t* rows64, cudaStream_t st) {
  if (count == 0) return;
  sketch_export_kernel<<<unsigned((count + 255) / 256), 256, 0, st>>>(count, rows, rows64);
  RKMF_CUDA(cudaGetLastError());
}

}  // namespace rkmf_b200
