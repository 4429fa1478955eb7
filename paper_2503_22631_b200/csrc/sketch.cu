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

// Row-major layout for the fused K2 with the sketch in the SpMV threads
// (spmv_rowsketch.cu; zeta == 8, d <= 255): for column j, slot q in 0..7
// holds one of its 8 (row, sign) entries: rbin[j][q] = row (uint8), bit q of
// sbit[j] set when the sign is negative. 9 bytes per column.
//
// The slot order is an 8-edge-colouring of each warp tile (32 consecutive
// columns, i.e. the 32 lanes of one SpMV warp): within a warp tile no two
// columns put the same row in the same slot, so when the 32 lanes add slot q
// into their warp's accumulator they touch 32 distinct bins, and a plain
// shared-memory read-add-write is race-free (no fp64 CAS atomics). The
// bipartite graph columns x rows has column degree 8, so 8 colours suffice
// whenever no row occurs more than 8 times among the 32 columns (Koenig);
// colours are assigned greedily with Kempe-chain (alternating path) swaps.
// A warp tile that cannot be coloured (a row hit > 8 times) keeps the sorted
// order and is flagged in wslow[], where the kernel falls back to atomics.
__global__ void sketch_rowbins_kernel(int64_t n, int d, const uint16_t* __restrict__ rows,
                                      const int8_t* __restrict__ signs, uint8_t* __restrict__ rbin,
                                      uint8_t* __restrict__ sbit, uint8_t* __restrict__ wslow) {
  const int64_t nwt = (n + 31) / 32;
  for (int64_t wt = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; wt < nwt;
       wt += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j0 = wt * 32;
    const int nc = int(min(int64_t(32), n - j0));
    uint8_t col[32][8];     // col[c][q] = row (bin) in slot q of column c, 255 = free
    int8_t sgn[32][8];
    int8_t binc[256][8];    // binc[b][q] = column using bin b in slot q, -1 = free
    // hw[h][q][r]: entries of half-warp h in slot q whose bin is r mod 16. A
    // half-warp's 64-bit shared accesses are conflict-free when its 16 bins
    // differ mod 16, so among the colours free at both ends the least loaded
    // residue is taken (fewer bank conflicts in the kernel's read-add-write).
    uint8_t hw[2][8][16];
    for (int h = 0; h < 2; ++h)
      for (int q = 0; q < 8; ++q)
        for (int r = 0; r < 16; ++r) hw[h][q][r] = 0;
    for (int b = 0; b < 256; ++b)
      for (int q = 0; q < 8; ++q) binc[b][q] = -1;
    for (int c = 0; c < 32; ++c)
      for (int q = 0; q < 8; ++q) col[c][q] = 255;
    bool ok = true;
    for (int c = 0; c < nc && ok; ++c) {
      for (int k = 0; k < 8 && ok; ++k) {
        const int b = rows[(j0 + c) * 8 + k];
        const int8_t sg = signs[(j0 + c) * 8 + k];
        int a = -1, e = -1;  // a: free at column c, e: free at bin b
        for (int q = 0; q < 8; ++q) {
          if (a < 0 && col[c][q] == 255) a = q;
          if (e < 0 && binc[b][q] < 0) e = q;
        }
        if (a < 0 || e < 0) { ok = false; break; }
        int use = -1, best = 1 << 20;
        for (int q = 0; q < 8; ++q)
          if (col[c][q] == 255 && binc[b][q] < 0 && hw[c >> 4][q][b & 15] < best) {
            best = hw[c >> 4][q][b & 15];
            use = q;
          }
        if (use < 0) {
          {
            // swap colours a and e along the alternating path that starts at
            // bin b with colour a: b -a- c1 -e- b1 -a- c2 ... (it cannot reach
            // column c, which has a free and e used; bipartite argument)
            int cur_b = b, cc = binc[b][a];
            while (cc >= 0) {
              const int nb = col[cc][e];  // next bin along colour e (255: end)
              // residue counts: edge (cc, cur_b) moves a -> e, edge (cc, nb) e -> a
              --hw[cc >> 4][a][cur_b & 15];
              ++hw[cc >> 4][e][cur_b & 15];
              if (nb != 255) {
                --hw[cc >> 4][e][nb & 15];
                ++hw[cc >> 4][a][nb & 15];
              }
              // swap at column cc: its a-edge (to cur_b) becomes e, its e-edge becomes a
              col[cc][e] = uint8_t(cur_b);
              const int8_t sa = sgn[cc][a];
              if (nb != 255) {
                col[cc][a] = uint8_t(nb);
                sgn[cc][a] = sgn[cc][e];
              } else {
                col[cc][a] = 255;
              }
              sgn[cc][e] = sa;
              binc[cur_b][e] = int8_t(cc);
              if (binc[cur_b][a] == cc) binc[cur_b][a] = -1;
              if (nb == 255) break;
              // bin nb: its e-edge (to cc) becomes a; continue along its old a-edge
              const int nxt = binc[nb][a];
              binc[nb][a] = int8_t(cc);
              if (binc[nb][e] == cc) binc[nb][e] = -1;
              cur_b = nb;
              cc = nxt;
            }
            use = a;
          }
        }
        col[c][use] = uint8_t(b);
        sgn[c][use] = sg;
        binc[b][use] = int8_t(c);
        ++hw[c >> 4][use][b & 15];
      }
    }
    // local search: swap two slots of one column when both bins stay unique
    // in their new slots and the half-warp's residue counts get flatter
    // (sum of squares), i.e. fewer bank conflicts in the kernel
    for (int pass = 0; pass < 4 && ok; ++pass) {
      bool moved = false;
      for (int c = 0; c < nc; ++c) {
        const int h = c >> 4;
        for (int q1 = 0; q1 < 8; ++q1)
          for (int q2 = q1 + 1; q2 < 8; ++q2) {
            const int b1 = col[c][q1], b2 = col[c][q2];
            if (binc[b1][q2] >= 0 || binc[b2][q1] >= 0) continue;
            const int r1 = b1 & 15, r2 = b2 & 15;
            if (r1 == r2) continue;
            const int a11 = hw[h][q1][r1], a21 = hw[h][q2][r1];
            const int a12 = hw[h][q1][r2], a22 = hw[h][q2][r2];
            // r1 moves q1 -> q2, r2 moves q2 -> q1
            const int delta = ((a11 - 1) * (a11 - 1) - a11 * a11) + ((a21 + 1) * (a21 + 1) - a21 * a21) +
                              ((a22 - 1) * (a22 - 1) - a22 * a22) + ((a12 + 1) * (a12 + 1) - a12 * a12);
            if (delta >= 0) continue;
            --hw[h][q1][r1]; ++hw[h][q2][r1]; --hw[h][q2][r2]; ++hw[h][q1][r2];
            binc[b1][q1] = -1; binc[b2][q2] = -1;
            binc[b1][q2] = int8_t(c); binc[b2][q1] = int8_t(c);
            col[c][q1] = uint8_t(b2); col[c][q2] = uint8_t(b1);
            const int8_t t = sgn[c][q1];
            sgn[c][q1] = sgn[c][q2];
            sgn[c][q2] = t;
            moved = true;
          }
      }
      if (!moved) break;
    }
    // self-check of the colouring before it is trusted: every slot holds
    // distinct bins across the warp tile, and every column holds exactly its
    // own 8 (row, sign) entries
    for (int q = 0; q < 8 && ok; ++q) {
      uint32_t seen[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int c = 0; c < nc; ++c) {
        const int b = col[c][q];
        if (b == 255 && d <= 255) { ok = false; break; }
        if (seen[b >> 5] & (1u << (b & 31))) { ok = false; break; }
        seen[b >> 5] |= 1u << (b & 31);
      }
    }
    for (int c = 0; c < nc && ok; ++c) {
      const int64_t j = j0 + c;
      for (int k = 0; k < 8 && ok; ++k) {
        bool found = false;
        for (int q = 0; q < 8; ++q)
          found |= col[c][q] == rows[j * 8 + k] && sgn[c][q] == signs[j * 8 + k];
        ok = found;
      }
    }
    for (int c = 0; c < nc; ++c) {
      const int64_t j = j0 + c;
      uint32_t bits = 0;
      for (int q = 0; q < 8; ++q) {
        const int b = ok ? col[c][q] : rows[j * 8 + q];
        const int8_t sg = ok ? sgn[c][q] : signs[j * 8 + q];
        rbin[j * 8 + q] = uint8_t(b);
        bits |= (sg < 0 ? 1u : 0u) << q;
      }
      sbit[j] = uint8_t(bits);
    }
    wslow[wt] = ok ? 0 : 1;
  }
}

void launch_sketch_rowbins(int64_t n, int d, const uint16_t* rows, const int8_t* signs,
                           uint8_t* rbin, uint8_t* sbit, uint8_t* wslow, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t nwt = (n + 31) / 32;
  const int64_t blocks = std::min<int64_t>((nwt + 63) / 64, 148 * 32);
  sketch_rowbins_kernel<<<int(blocks), 64, 0, st>>>(n, d, rows, signs, rbin, sbit, wslow);
  RKMF_CUDA(cudaGetLastError());
  if (getenv("RKMF_PIPE_VERBOSE")) {
    std::vector<uint8_t> h(static_cast<size_t>(nwt), uint8_t(0));
    RKMF_CUDA(cudaMemcpyAsync(h.data(), wslow, size_t(nwt), cudaMemcpyDeviceToHost, st));
    RKMF_CUDA(cudaStreamSynchronize(st));
    int64_t bad = 0;
    for (uint8_t v : h) bad += v;
    fprintf(stderr, "[rkmf] sketch row layout: %lld of %lld warp tiles without a colouring\n",
            (long long)bad, (long long)nwt);
  }
}

}  // namespace rkmf_b200
