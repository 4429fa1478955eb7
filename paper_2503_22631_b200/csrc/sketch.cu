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
                                    uint8_t* __restrict__ tile_ent, int64_t ent_stride,
                                    unsigned long long* __restrict__ size_max) {
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
      ent[pos] = uint8_t(t | (signs && signs[col * zeta + k] < 0 ? 0x80 : 0));
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
  // slot -> bin
  for (int64_t b = t; b < d; b += blockDim.x) soff[cur[b]] = b;
  __syncthreads();
  // group g = 4 j + w holds the slots of warp w in pass j (sketch_tile_gather)
  auto slot_of = [&](int64_t g, int l) -> int64_t {
    const int64_t j = g / 4, u = 32 * (g % 4) + l;
    return (j & 1) ? kSketchNT * j + kSketchNT - 1 - u : kSketchNT * j + u;
  };
  auto slot_len = [&](int64_t sl) { return sl < d ? cnt[soff[sl] + 1] - cnt[soff[sl]] : 0; };
  const int64_t ng = tile_groups(d);
  if (size_max) {  // sizing pass: this tile's entry bytes
    if (t == 0) {
      unsigned long long tot = 0;
      for (int64_t g = 0; g < ng; ++g) {
        int mx = 0;
        for (int l = 0; l < 32; ++l) mx = max(mx, slot_len(slot_of(g, l)));
        tot += 128ull * unsigned((mx + 3) / 4);
      }
      atomicMax(size_max, tot);
    }
    return;
  }
  // header: slot lengths (uint8), slot bins, group entry offsets
  uint16_t* toff = tile_off + tile * off_stride;
  uint8_t* hlen = reinterpret_cast<uint8_t*>(toff);
  uint16_t* hbin = toff + tile_hdr_bin(d);
  uint16_t* hgb = toff + tile_hdr_gbase(d);
  for (int64_t sl = t; sl < d; sl += blockDim.x) {
    hlen[sl] = uint8_t(slot_len(sl));
    hbin[sl] = uint16_t(soff[sl]);
  }
  for (int64_t q = d + t; q < 2 * tile_hdr_bin(d); q += blockDim.x) hlen[q] = 0;
  if (t == 0) {
    int base = 0;
    for (int64_t g = 0; g < ng; ++g) {
      hgb[g] = uint16_t(base);
      int mx = 0;
      for (int l = 0; l < 32; ++l) mx = max(mx, slot_len(slot_of(g, l)));
      base += 128 * ((mx + 3) / 4);
    }
    for (int64_t q = tile_hdr_gbase(d) + ng; q < off_stride; ++q) toff[q] = 0;
  }
  uint8_t* tent = tile_ent + tile * ent_stride;
  for (int64_t e = t; e < ent_stride; e += blockDim.x) tent[e] = 0;
  __syncthreads();
  // Entry order inside each slot, bank-aware. Round p of a group is one
  // shared load of zs2 per lane with len > p; a 64-bit load is served per
  // half-warp, and the double at index u sits in bank pair u mod 16 = row mod
  // 16. Round by round, every active lane takes its remaining entry whose
  // bank pair is least used so far in its half-warp. Only the summation order
  // inside a bin changes; the layout stays deterministic.
  for (int64_t g = t; g < ng; g += blockDim.x) {
    int len[32], src[32];
    uint32_t taken[32][4];
    int mx = 0;
    for (int l = 0; l < 32; ++l) {
      const int64_t sl = slot_of(g, l);
      len[l] = slot_len(sl);
      src[l] = sl < d ? cnt[soff[sl]] : 0;
      mx = max(mx, len[l]);
      for (int w = 0; w < 4; ++w) taken[l][w] = 0u;
    }
    uint8_t* ge = tent + hgb[g];
    for (int p = 0; p < mx; ++p) {
      int load[2][16];
      for (int h = 0; h < 2; ++h)
        for (int q = 0; q < 16; ++q) load[h][q] = 0;
      for (int l = 0; l < 32; ++l) {
        if (p >= len[l]) continue;
        int* ld = load[l >> 4];
        int best = -1, bl = 1 << 30;
        for (int e = 0; e < len[l]; ++e) {
          if ((taken[l][e >> 5] >> (e & 31)) & 1u) continue;
          const int bank = ent[src[l] + e] & 15;
          if (ld[bank] < bl) { bl = ld[bank]; best = e; }
        }
        taken[l][best >> 5] |= 1u << (best & 31);
        ld[ent[src[l] + best] & 15]++;
        ge[4 * (32 * (p >> 2) + l) + (p & 3)] = ent[src[l] + best];
      }
    }
  }
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

namespace {
size_t tiles_smem(int64_t d, int64_t zeta) {
  const size_t smem = sizeof(int) * size_t(3 * d + 2) + size_t(kTileRows * zeta) + 16;
  if (smem > 200 * 1024) param_error("sketch: d too large for the device tile layout");
  if (smem > 48 * 1024)
    RKMF_CUDA(cudaFuncSetAttribute(sketch_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
  return smem;
}
}  // namespace

int64_t sketch_tiles_stride(int64_t d, int64_t n, int64_t zeta, const uint16_t* rows,
                            cudaStream_t st) {
  const int64_t tiles = (n + kTileRows - 1) / kTileRows;
  if (tiles == 0) return 128;
  const size_t smem = tiles_smem(d, zeta);
  unsigned long long* dm = nullptr;
  RKMF_CUDA(cudaMallocAsync(&dm, sizeof(unsigned long long), st));
  RKMF_CUDA(cudaMemsetAsync(dm, 0, sizeof(unsigned long long), st));
  sketch_tiles_kernel<<<unsigned(tiles), kBlock, smem, st>>>(d, n, int(zeta), tile_off_stride(d),
                                                              rows, nullptr, nullptr, nullptr, 0,
                                                              dm);
  RKMF_CUDA(cudaGetLastError());
  unsigned long long hm = 0;
  RKMF_CUDA(cudaMemcpyAsync(&hm, dm, sizeof(hm), cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaStreamSynchronize(st));
  RKMF_CUDA(cudaFree(dm));
  if (hm > 65535) param_error("sketch: a tile's entry layout exceeds 64 KB (zeta too large)");
  return std::max<int64_t>(128, int64_t(hm));
}

void launch_sketch_tiles(int64_t d, int64_t n, int64_t zeta, const uint16_t* rows,
                         const int8_t* signs, uint16_t* tile_off, uint8_t* tile_ent,
                         int64_t ent_stride, cudaStream_t st) {
  const int64_t tiles = (n + kTileRows - 1) / kTileRows;
  if (tiles == 0) return;
  const size_t smem = tiles_smem(d, zeta);
  sketch_tiles_kernel<<<unsigned(tiles), kBlock, smem, st>>>(d, n, int(zeta), tile_off_stride(d),
                                                              rows, signs, tile_off, tile_ent,
                                                              ent_stride, nullptr);
  RKMF_CUDA(cudaGetLastError());
}

void launch_sketch_export(int64_t count, const uint16_t* rows, const int8_t* /*signs*/,
                          int64_t* rows64, cudaStream_t st) {
  if (count == 0) return;
  sketch_export_kernel<<<unsigned((count + 255) / 256), 256, 0, st>>>(count, rows, rows64);
  RKMF_CUDA(cudaGetLastError());
}

}  // namespace rkmf_b200
