// Diagonal (DIA) copy of a CSR matrix for the fused SpMV + sketch (K2).
//
// The SpMV half of K2 streams 12 bytes per nonzero plus row pointers from HBM
// (a CSR value and its int32 column). When every nonzero of the matrix lies on
// one of a few diagonals (col - row in a small set — the stencil matrices of
// the BASELINE configs: 5/7/27-point Laplacians, Q1, convection-diffusion),
// the same matrix is stored here as [tile][diag][128 rows] fp64 values with
// each tile's sorted offsets on the side ([tile][8] int32; the offsets may
// differ per tile, e.g. the halo columns of a row-partitioned slab sit on
// their own diagonal): 8 bytes per stored slot and no indices, and
// the x reads at row + offset are coalesced across a warp instead of gathers
// (and issued a tile ahead: they do not depend on the streamed values).
// Slots where the CSR row has no entry hold 0.0, and each row's entries keep
// the CSR's column order, so z = A x is bit-identical to the CSR kernel (a
// padding term adds exactly 0.0). The one exception: a row-partitioned rank's
// local columns (partition.cpp) put the halo of a lower rank past the owned
// columns (local index n_local + pos), so that entry comes first in the CSR
// row and last among the sorted offsets; those boundary rows then sum in a
// different order than the CSR kernel (rounding-level differences only).
//
// Eligibility (checked on device, one pass over the nonzeros): at most
// kMaxDiag = 8 distinct offsets per 128-row tile (27-point stencils stay on the CSR kernel,
// which splits their rows over two threads and measured faster), no repeated column
// within a row (validated matrices have strictly increasing columns; partition-local ones
// may not be monotone, see above), and
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

constexpr int32_t kEmpty = INT_MIN;

// One block (128 threads = the tile's rows) per tile: the distinct column
// offsets of the tile's rows, sorted, into toff[tile][kMaxDiag] (slots past
// the tile's count repeat its largest offset: a duplicate slot keeps 0.0
// values and adds an exact zero). flags[0]: a row repeats a column; flags[1]: a tile has more than kMaxDiag offsets; flags[2]: the
// largest per-tile count.
template <typename RP>
__global__ void dia_tile_offsets_kernel(int64_t n, const RP* __restrict__ rp,
                                        const int32_t* __restrict__ ci, int32_t* toff,
                                        int32_t* flags) {
  __shared__ int32_t set[kMaxDiag];
  __shared__ int over;
  const int64_t tile = blockIdx.x;
  const int64_t row = tile * kTileRows + threadIdx.x;
  if (threadIdx.x < kMaxDiag) set[threadIdx.x] = kEmpty;
  if (threadIdx.x == 0) over = 0;
  __syncthreads();
  if (row < n) {
    const int64_t lo = int64_t(rp[row]), hi = int64_t(rp[row + 1]);
    int32_t prev = -1;
    for (int64_t e = lo; e < hi; ++e) {
      const int32_t c = ci[e];
      if (c <= prev)  // not monotone (a partition-local row): look for a repeat
        for (int64_t f = lo; f < e; ++f)
          if (ci[f] == c) atomicExch(flags + 0, 1);
      prev = c;
      const int32_t o = int32_t(int64_t(c) - row);
      bool done = false;
      for (int q = 0; q < kMaxDiag && !done; ++q) {
        const int32_t cur = set[q];
        if (cur == o) {
          done = true;
        } else if (cur == kEmpty) {
          const int32_t old = atomicCAS(set + q, kEmpty, o);
          done = old == kEmpty || old == o;
        }
      }
      if (!done) over = 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (over) atomicExch(flags + 1, 1);
    int32_t v[kMaxDiag];
    int cnt = 0;
    for (int q = 0; q < kMaxDiag; ++q)
      if (set[q] != kEmpty) v[cnt++] = set[q];
    for (int a = 1; a < cnt; ++a) {  // insertion sort
      const int32_t key = v[a];
      int b = a - 1;
      while (b >= 0 && v[b] > key) { v[b + 1] = v[b]; --b; }
      v[b + 1] = key;
    }
    for (int q = 0; q < kMaxDiag; ++q) toff[tile * kMaxDiag + q] = cnt ? v[min(q, cnt - 1)] : 0;
    atomicMax(flags + 2, cnt);
  }
}

// dval[(tile * nd + q) * 128 + r] = A(row, row + toff[tile][q]) (0.0 where absent)
template <typename RP>
__global__ void dia_fill_kernel(int64_t n, const RP* __restrict__ rp,
                                const int32_t* __restrict__ ci, const double* __restrict__ val,
                                const int32_t* __restrict__ toff, int64_t stride, int nd,
                                double* dval) {
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n;
       row += int64_t(gridDim.x) * blockDim.x) {
    const int64_t tile = row / kTileRows, r = row % kTileRows;
    const int32_t* offs = toff + tile * stride;
    double* base = dval + tile * int64_t(nd) * kTileRows + r;
    const int64_t lo = int64_t(rp[row]), hi = int64_t(rp[row + 1]);
    for (int64_t e = lo; e < hi; ++e) {
      const int32_t o = int32_t(int64_t(ci[e]) - row);
      int q = 0;
      while (offs[q] != o) ++q;  // present: the offsets kernel collected it
      base[int64_t(q) * kTileRows] = val[e];
    }
  }
}

template <typename RP>
void launch_offsets(const CsrView& v, int32_t* toff, int32_t* flags, cudaStream_t st) {
  const int64_t tiles = (v.n_rows + kTileRows - 1) / kTileRows;
  dia_tile_offsets_kernel<RP><<<unsigned(tiles), kTileRows, 0, st>>>(
      v.n_rows, static_cast<const RP*>(v.row_ptr), v.col, toff, flags);
}
template <typename RP>
void launch_fill(const CsrView& v, const int32_t* toff, int64_t stride, int nd, double* dval,
                 cudaStream_t st) {
  dia_fill_kernel<RP><<<1184, 256, 0, st>>>(v.n_rows, static_cast<const RP*>(v.row_ptr), v.col,
                                            v.val, toff, stride, nd, dval);
}


// ---- row dictionary of the diagonal copy ----
// Stencil matrices with constant coefficients (cfg1, cfg2, cfg4, cfg5) have
// few distinct rows: in the diagonal layout a row is the tuple of its nd
// values, and only boundary faces, edges and corners change it (27 tuples on
// a 3D 7-point grid). Then K2 streams one byte per row (the tuple id) instead
// of 8 nd, and looks the values up in a shared-memory dictionary: the same
// values in the same order, so z stays bit-identical. Built on device: each
// row's tuple is hashed (64-bit) into an open-addressing table; the host
// orders the occupied slots by their smallest row (deterministic ids) and a
// last pass assigns each row its id and compares its values with the
// dictionary's bit for bit (a hash collision fails the build, it never
// corrupts a row). More than kMaxTuples distinct rows: no dictionary.
constexpr int kTupTable = 4096;

__device__ __forceinline__ uint64_t tup_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t row_hash(const double* __restrict__ dval, int64_t row, int nd) {
  const int64_t tile = row / kTileRows, r = row % kTileRows;
  uint64_t h = 0x9E3779B97F4A7C15ULL * uint64_t(nd + 1);
  for (int q = 0; q < nd; ++q)
    h = tup_mix(h ^ uint64_t(__double_as_longlong(dval[(tile * nd + q) * kTileRows + r])));
  return h | 1ULL;  // 0 marks an empty slot
}

// flags[0]: more than kMaxTuples distinct rows (or the table filled)
__global__ void tup_insert_kernel(int64_t n, int nd, const double* __restrict__ dval,
                                  unsigned long long* keys, unsigned long long* rep,
                                  unsigned long long* rowhash, int32_t* count, int32_t* flags) {
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n;
       row += int64_t(gridDim.x) * blockDim.x) {
    if (*(volatile int32_t*)flags) return;
    const unsigned long long h = row_hash(dval, row, nd);
    rowhash[row] = h;
    int slot = int(h & (kTupTable - 1));
    bool found = false;
    for (int i = 0; i < kTupTable; ++i) {
      const unsigned long long k = keys[slot];
      if (k == h) { found = true; break; }
      if (k == 0ULL) {
        const unsigned long long old = atomicCAS(keys + slot, 0ULL, h);
        if (old == 0ULL) {
          if (atomicAdd(count, 1) >= kMaxTuples) flags[0] = 1;
          found = true;
          break;
        }
        if (old == h) { found = true; break; }
      }
      slot = (slot + 1) & (kTupTable - 1);
    }
    if (!found) { flags[0] = 1; return; }
    atomicMin(rep + slot, (unsigned long long)row);
  }
}

__global__ void tup_gather_kernel(int ntup, int nd, const double* __restrict__ dval,
                                  const long long* __restrict__ rep_rows, double* dict) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntup * nd) return;
  const int id = i / nd, q = i % nd;
  const int64_t row = rep_rows[id], tile = row / kTileRows, r = row % kTileRows;
  dict[i] = dval[(tile * nd + q) * kTileRows + r];
}

// flags[1]: a row differs from its dictionary tuple (hash collision)
__global__ void tup_assign_kernel(int64_t n, int nd, const double* __restrict__ dval,
                                  const unsigned long long* __restrict__ keys,
                                  const int16_t* __restrict__ slot_id,
                                  const unsigned long long* __restrict__ rowhash,
                                  const double* __restrict__ dict, uint8_t* tid, int32_t* flags) {
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n;
       row += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long h = rowhash[row];
    int slot = int(h & (kTupTable - 1));
    while (keys[slot] != h) slot = (slot + 1) & (kTupTable - 1);  // inserted above
    const int id = slot_id[slot];
    const int64_t tile = row / kTileRows, r = row % kTileRows;
    for (int q = 0; q < nd; ++q)
      if (__double_as_longlong(dval[(tile * nd + q) * kTileRows + r]) !=
          __double_as_longlong(dict[id * nd + q]))
        flags[1] = 1;
    tid[row] = uint8_t(id);
  }
}

}  // namespace

void drop_dia_dict(rkmf_matrix* M) {
  if (M->dia_tid) cudaFree(M->dia_tid);
  if (M->dia_dict) cudaFree(M->dia_dict);
  M->dia_tid = nullptr;
  M->dia_dict = nullptr;
  M->dia_dict_host.clear();
  M->view.dtid = nullptr;
  M->view.ddict = nullptr;
  M->view.ddict_host = nullptr;
  M->view.ntup = 0;
}

// Builds the row dictionary of an existing diagonal copy when the matrix has
// at most kMaxTuples distinct rows (leaves it absent otherwise).
void build_dia_dict(rkmf_matrix* M) {
  drop_dia_dict(M);
  const CsrView& v = M->view;
  if (!v.dval || v.ndiag < 1 || v.n_rows < 1) return;
  rkmf_context* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  const int nd = v.ndiag;
  const int64_t n = v.n_rows, tiles = (n + kTileRows - 1) / kTileRows;
  ScopedBuf keys, rep, rowhash, slot_id, rrows, misc;
  keys.ensure(sizeof(unsigned long long) * kTupTable);
  rep.ensure(sizeof(unsigned long long) * kTupTable);
  rowhash.ensure(sizeof(unsigned long long) * size_t(n));
  misc.ensure(sizeof(int32_t) * 4);
  int32_t* cnt = misc.as<int32_t>();
  int32_t* flags = cnt + 1;
  RKMF_CUDA(cudaMemsetAsync(keys.p, 0, sizeof(unsigned long long) * kTupTable, st));
  RKMF_CUDA(cudaMemsetAsync(rep.p, 0xFF, sizeof(unsigned long long) * kTupTable, st));
  RKMF_CUDA(cudaMemsetAsync(misc.p, 0, sizeof(int32_t) * 4, st));
  const int grid = 4 * 148;
  tup_insert_kernel<<<grid, 256, 0, st>>>(n, nd, v.dval, static_cast<unsigned long long*>(keys.p),
                                          static_cast<unsigned long long*>(rep.p),
                                          static_cast<unsigned long long*>(rowhash.p), cnt, flags);
  RKMF_CUDA(cudaGetLastError());
  ctx->launches++;
  std::vector<unsigned long long> hk(kTupTable), hr(kTupTable);
  int32_t hf[4];
  RKMF_CUDA(cudaMemcpyAsync(hf, misc.p, sizeof(hf), cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaMemcpyAsync(hk.data(), keys.p, sizeof(unsigned long long) * kTupTable,
                            cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaMemcpyAsync(hr.data(), rep.p, sizeof(unsigned long long) * kTupTable,
                            cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaStreamSynchronize(st));
  if (hf[1] || hf[0] > kMaxTuples) return;
  // ids in order of each tuple's first row (deterministic)
  std::vector<std::pair<unsigned long long, int>> occ;
  for (int i = 0; i < kTupTable; ++i)
    if (hk[size_t(i)]) occ.push_back({hr[size_t(i)], i});
  std::sort(occ.begin(), occ.end());
  const int ntup = int(occ.size());
  if (ntup < 1 || ntup > kMaxTuples) return;
  std::vector<int16_t> sid(kTupTable, int16_t(-1));
  std::vector<long long> rows(static_cast<size_t>(ntup));
  for (int id = 0; id < ntup; ++id) {
    sid[size_t(occ[size_t(id)].second)] = int16_t(id);
    rows[size_t(id)] = (long long)occ[size_t(id)].first;
  }
  slot_id.ensure(sizeof(int16_t) * kTupTable);
  rrows.ensure(sizeof(long long) * size_t(ntup));
  RKMF_CUDA(cudaMemcpyAsync(slot_id.p, sid.data(), sizeof(int16_t) * kTupTable,
                            cudaMemcpyHostToDevice, st));
  RKMF_CUDA(cudaMemcpyAsync(rrows.p, rows.data(), sizeof(long long) * size_t(ntup),
                            cudaMemcpyHostToDevice, st));
  if (cudaMalloc(&M->dia_dict, sizeof(double) * size_t(ntup) * size_t(nd)) != cudaSuccess ||
      cudaMalloc(&M->dia_tid, size_t(tiles) * kTileRows + 16) != cudaSuccess) {
    cudaGetLastError();
    return drop_dia_dict(M);
  }
  RKMF_CUDA(cudaMemsetAsync(M->dia_tid, 0, size_t(tiles) * kTileRows + 16, st));
  tup_gather_kernel<<<(ntup * nd + 127) / 128, 128, 0, st>>>(
      ntup, nd, v.dval, static_cast<const long long*>(rrows.p), M->dia_dict);
  tup_assign_kernel<<<grid, 256, 0, st>>>(
      n, nd, v.dval, static_cast<const unsigned long long*>(keys.p),
      static_cast<const int16_t*>(slot_id.p), static_cast<const unsigned long long*>(rowhash.p),
      M->dia_dict, M->dia_tid, flags);
  RKMF_CUDA(cudaGetLastError());
  ctx->launches += 2;
  RKMF_CUDA(cudaMemcpyAsync(hf, misc.p, sizeof(hf), cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaStreamSynchronize(st));
  if (hf[1]) return drop_dia_dict(M);
  M->dia_dict_host.assign(size_t(ntup) * size_t(nd), 0.0);
  RKMF_CUDA(cudaMemcpy(M->dia_dict_host.data(), M->dia_dict, sizeof(double) * size_t(ntup) * size_t(nd),
                       cudaMemcpyDeviceToHost));
  M->view.dtid = M->dia_tid;
  M->view.ddict = M->dia_dict;
  M->view.ddict_host = M->dia_dict_host.data();
  M->view.ntup = ntup;
}

void drop_dia(rkmf_matrix* M) {
  drop_dia_dict(M);
  if (M->dia_val) cudaFree(M->dia_val);
  if (M->dia_off) cudaFree(M->dia_off);
  M->dia_val = nullptr;
  M->dia_off = nullptr;
  M->view.dval = nullptr;
  M->view.doff = nullptr;
  M->view.ndiag = 0;
  M->view.dstride = 0;
}

// Builds the diagonal copy when the matrix qualifies; leaves the CSR-only
// matrix untouched otherwise (also when the copy does not fit in memory).
void build_dia(rkmf_matrix* M) {
  drop_dia(M);
  const CsrView& v = M->view;
  if (v.n_rows == 0 || v.nnz == 0 || !v.row_ptr) return;
  if (v.n_rows >= (int64_t(1) << 31) - kTileRows) return;
  rkmf_context* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t tiles = (v.n_rows + kTileRows - 1) / kTileRows;
  // per-tile offsets first (small): [tiles][kMaxDiag]
  if (cudaMalloc(&M->dia_off, sizeof(int32_t) * size_t(tiles) * kMaxDiag) != cudaSuccess) {
    cudaGetLastError();
    M->dia_off = nullptr;
    return;
  }
  int32_t* flags = static_cast<int32_t*>(ctx->scratch.ensure(sizeof(int32_t) * 4));
  RKMF_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t) * 4, st));
  if (v.rp64) launch_offsets<int64_t>(v, M->dia_off, flags, st);
  else launch_offsets<int32_t>(v, M->dia_off, flags, st);
  RKMF_CUDA(cudaGetLastError());
  ctx->launches++;
  int32_t h[4];
  RKMF_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaStreamSynchronize(st));
  int nd = h[2];
  auto fail = [&] { drop_dia(M); };
  if (h[0] || h[1] || nd < 1 || nd > kMaxDiag) return fail();
  // Usually every tile draws from one set of <= 8 offsets (a single-domain
  // stencil): then store that union once (stride 0; the kernel keeps it in
  // shared memory). Otherwise (the halo diagonals of a row slab) keep the
  // per-tile lists (stride 8; read per tile, one tile ahead).
  int64_t stride = kMaxDiag;
  {
    std::vector<int32_t> ht(size_t(tiles) * kMaxDiag);
    RKMF_CUDA(cudaMemcpy(ht.data(), M->dia_off, sizeof(int32_t) * ht.size(),
                         cudaMemcpyDeviceToHost));
    std::vector<int32_t> uni(ht);
    std::sort(uni.begin(), uni.end());
    uni.erase(std::unique(uni.begin(), uni.end()), uni.end());
    if (int(uni.size()) <= kMaxDiag) {
      nd = int(uni.size());
      std::vector<int32_t> u8(kMaxDiag, uni.back());
      std::copy(uni.begin(), uni.end(), u8.begin());
      RKMF_CUDA(cudaMemcpy(M->dia_off, u8.data(), sizeof(int32_t) * kMaxDiag,
                           cudaMemcpyHostToDevice));
      stride = 0;
    }
  }
  const double dia_bytes = 8.0 * double(nd) * double(tiles * kTileRows);
  const double csr_bytes = 12.0 * double(v.nnz) + (v.rp64 ? 8.0 : 4.0) * double(v.n_rows);
  if (dia_bytes > 0.85 * csr_bytes) return fail();
  size_t free_b = 0, total_b = 0;
  RKMF_CUDA(cudaMemGetInfo(&free_b, &total_b));
  if (dia_bytes > 0.25 * double(free_b)) return fail();  // leave room for the basis
  const size_t nval = size_t(nd) * size_t(tiles) * kTileRows;
  if (cudaMalloc(&M->dia_val, sizeof(double) * nval) != cudaSuccess) {
    cudaGetLastError();
    M->dia_val = nullptr;
    return fail();
  }
  RKMF_CUDA(cudaMemsetAsync(M->dia_val, 0, sizeof(double) * nval, st));
  if (v.rp64) launch_fill<int64_t>(v, M->dia_off, stride, nd, M->dia_val, st);
  else launch_fill<int32_t>(v, M->dia_off, stride, nd, M->dia_val, st);
  RKMF_CUDA(cudaGetLastError());
  ctx->launches++;
  RKMF_CUDA(cudaStreamSynchronize(st));
  M->view.dval = M->dia_val;
  M->view.doff = M->dia_off;
  M->view.ndiag = nd;
  M->view.dstride = int(stride);
  build_dia_dict(M);
}

bool dia_enabled_by_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = knob_env("RKMF_DIA");
    v = e ? (atoi(e) != 0) : 1;
  }
  return v != 0;
}

}  // namespace rkmf_b200
