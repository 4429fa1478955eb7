// CSR row dictionary: matrices without a diagonal copy (more than 8
// diagonals: the 27-point Q1 matrices of cfg3/cfg5) whose rows, up to
// translation, take at most kMaxTuples distinct forms. A row's form is its
// nonzero count, its column offsets col - row and its values, in column
// order; a constant-coefficient stencil has one form per boundary class (27
// on a 3D grid), and a row slab of the partitioned solve a few more for the
// rows that reach its halo (the halo columns sit in natural order after the
// owned rows, so those offsets are constant per class too). K2 then streams
// one byte per row (the form id) instead of 12 bytes per nonzero and takes
// offsets and values from a shared-memory dictionary, in column order (one
// thread per row: z agrees with the CSR kernel's two-lane rows to rounding).
//
// Built on device like the diagonal copy's dictionary (dia.cu): a 64-bit hash
// per row into an open-addressing table, ids in the order of each form's
// first row (deterministic), and a last pass that checks every row against its
// form bit for bit (a hash collision fails the build, it never corrupts a row).
#include <algorithm>
#include <cstdio>
#include <vector>

#include "rkmf_internal.cuh"
#include "engine_types.cuh"

namespace rkmf_b200 {

namespace {

constexpr int kRdTable = 4096;

__device__ __forceinline__ uint64_t rd_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// flags[0]: too many forms / table full / a row longer than kRdMaxNnz;
// flags[1]: a row differs from its form (collision); flags[2]: an offset
// outside int32
template <typename RP>
__global__ void rd_insert_kernel(int64_t n, const RP* __restrict__ rp,
                                 const int32_t* __restrict__ col, const double* __restrict__ val,
                                 unsigned long long* keys, unsigned long long* rep,
                                 unsigned long long* rowhash, int32_t* count, int32_t* flags) {
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n;
       row += int64_t(gridDim.x) * blockDim.x) {
    if (*(volatile int32_t*)flags) return;
    const int64_t e0 = int64_t(rp[row]), e1 = int64_t(rp[row + 1]);
    if (e1 - e0 > kRdMaxNnz) {
      flags[0] = 1;
      return;
    }
    uint64_t h = rd_mix(0x9E3779B97F4A7C15ULL * uint64_t(e1 - e0 + 1));
    for (int64_t e = e0; e < e1; ++e) {
      const int64_t off = int64_t(col[e]) - row;
      if (off < INT32_MIN || off > INT32_MAX) flags[2] = 1;
      h = rd_mix(h ^ uint64_t(off));
      h = rd_mix(h ^ uint64_t(__double_as_longlong(val[e])));
    }
    h |= 1ULL;  // 0 marks an empty slot
    rowhash[row] = h;
    int slot = int(h & (kRdTable - 1));
    bool found = false;
    for (int i = 0; i < kRdTable; ++i) {
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
      slot = (slot + 1) & (kRdTable - 1);
    }
    if (!found) { flags[0] = 1; return; }
    atomicMin(rep + slot, (unsigned long long)row);
  }
}

// one block per form: its count, offsets and values from its first row
template <typename RP>
__global__ void rd_gather_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ col,
                                 const double* __restrict__ val,
                                 const long long* __restrict__ rep_rows, int32_t* cnt,
                                 int32_t* off, double* dval) {
  const int id = blockIdx.x;
  const int64_t row = rep_rows[id];
  const int64_t e0 = int64_t(rp[row]), c = int64_t(rp[row + 1]) - e0;
  if (threadIdx.x == 0) cnt[id] = int32_t(c);
  for (int q = threadIdx.x; q < kRdMaxNnz; q += blockDim.x) {
    off[id * kRdMaxNnz + q] = q < c ? int32_t(int64_t(col[e0 + q]) - row) : 0;
    dval[id * kRdMaxNnz + q] = q < c ? val[e0 + q] : 0.0;
  }
}

template <typename RP>
__global__ void rd_assign_kernel(int64_t n, const RP* __restrict__ rp,
                                 const int32_t* __restrict__ col, const double* __restrict__ val,
                                 const unsigned long long* __restrict__ keys,
                                 const int16_t* __restrict__ slot_id,
                                 const unsigned long long* __restrict__ rowhash,
                                 const int32_t* __restrict__ cnt, const int32_t* __restrict__ off,
                                 const double* __restrict__ dval, uint8_t* tid, int32_t* flags) {
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < n;
       row += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long h = rowhash[row];
    int slot = int(h & (kRdTable - 1));
    while (keys[slot] != h) slot = (slot + 1) & (kRdTable - 1);  // inserted above
    const int id = slot_id[slot];
    const int64_t e0 = int64_t(rp[row]), c = int64_t(rp[row + 1]) - e0;
    bool same = c == cnt[id];
    for (int64_t q = 0; same && q < c; ++q)
      same = int64_t(col[e0 + q]) - row == int64_t(off[id * kRdMaxNnz + q]) &&
             __double_as_longlong(val[e0 + q]) == __double_as_longlong(dval[id * kRdMaxNnz + q]);
    if (!same) flags[1] = 1;
    tid[row] = uint8_t(id);
  }
}

}  // namespace

void drop_csr_dict(rkmf_matrix* M) {
  if (M->rd_tid) cudaFree(M->rd_tid);
  if (M->rd_cnt) cudaFree(M->rd_cnt);
  if (M->rd_off) cudaFree(M->rd_off);
  if (M->rd_val) cudaFree(M->rd_val);
  M->rd_tid = nullptr;
  M->rd_cnt = nullptr;
  M->rd_off = nullptr;
  M->rd_val = nullptr;
  M->view.rtid = nullptr;
  M->view.rcnt = nullptr;
  M->view.roff = nullptr;
  M->view.rval = nullptr;
  M->view.rntup = 0;
  M->view.rkd = 0;
}

void build_csr_dict(rkmf_matrix* M) {
  drop_csr_dict(M);
  const CsrView& v = M->view;
  if (v.ndiag > 0 || v.n_rows < 1 || v.nnz < 1 || !v.row_ptr || !v.col || !v.val) return;
  if (v.n_rows >= (int64_t(1) << 31) - kTileRows) return;
  rkmf_context* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = v.n_rows, tiles = (n + kTileRows - 1) / kTileRows;
  ScopedBuf keys, rep, rowhash, slot_id, rrows, misc;
  keys.ensure(sizeof(unsigned long long) * kRdTable);
  rep.ensure(sizeof(unsigned long long) * kRdTable);
  if (cudaMalloc(&rowhash.p, sizeof(unsigned long long) * size_t(n)) != cudaSuccess) {
    cudaGetLastError();
    rowhash.p = nullptr;
    return;
  }
  rowhash.cap = sizeof(unsigned long long) * size_t(n);
  misc.ensure(sizeof(int32_t) * 4);
  int32_t* count = misc.as<int32_t>();
  int32_t* flags = count + 1;
  RKMF_CUDA(cudaMemsetAsync(keys.p, 0, sizeof(unsigned long long) * kRdTable, st));
  RKMF_CUDA(cudaMemsetAsync(rep.p, 0xFF, sizeof(unsigned long long) * kRdTable, st));
  RKMF_CUDA(cudaMemsetAsync(misc.p, 0, sizeof(int32_t) * 4, st));
  const int grid = 4 * 148;
  auto insert = [&](auto* rpp) {
    rd_insert_kernel<<<grid, 256, 0, st>>>(n, rpp, v.col, v.val,
                                           static_cast<unsigned long long*>(keys.p),
                                           static_cast<unsigned long long*>(rep.p),
                                           static_cast<unsigned long long*>(rowhash.p), count,
                                           flags);
  };
  if (v.rp64) insert(static_cast<const int64_t*>(v.row_ptr));
  else insert(static_cast<const int32_t*>(v.row_ptr));
  RKMF_CUDA(cudaGetLastError());
  ctx->launches++;
  std::vector<unsigned long long> hk(kRdTable), hr(kRdTable);
  int32_t hf[4];
  RKMF_CUDA(cudaMemcpyAsync(hf, misc.p, sizeof(hf), cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaMemcpyAsync(hk.data(), keys.p, sizeof(unsigned long long) * kRdTable,
                            cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaMemcpyAsync(hr.data(), rep.p, sizeof(unsigned long long) * kRdTable,
                            cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaStreamSynchronize(st));
  if (hf[1] || hf[3] || hf[0] > kMaxTuples) return;  // hf: count, flags[0..2]
  std::vector<std::pair<unsigned long long, int>> occ;
  for (int i = 0; i < kRdTable; ++i)
    if (hk[size_t(i)]) occ.push_back({hr[size_t(i)], i});
  std::sort(occ.begin(), occ.end());
  const int ntup = int(occ.size());
  if (ntup < 1 || ntup > kMaxTuples) return;
  std::vector<int16_t> sid(kRdTable, int16_t(-1));
  std::vector<long long> rows(static_cast<size_t>(ntup));
  for (int id = 0; id < ntup; ++id) {
    sid[size_t(occ[size_t(id)].second)] = int16_t(id);
    rows[size_t(id)] = (long long)occ[size_t(id)].first;
  }
  slot_id.ensure(sizeof(int16_t) * kRdTable);
  rrows.ensure(sizeof(long long) * size_t(ntup));
  RKMF_CUDA(cudaMemcpyAsync(slot_id.p, sid.data(), sizeof(int16_t) * kRdTable,
                            cudaMemcpyHostToDevice, st));
  RKMF_CUDA(cudaMemcpyAsync(rrows.p, rows.data(), sizeof(long long) * size_t(ntup),
                            cudaMemcpyHostToDevice, st));
  const size_t tid_bytes = size_t(tiles) * kTileRows + 16;
  if (cudaMalloc(&M->rd_cnt, sizeof(int32_t) * size_t(ntup)) != cudaSuccess ||
      cudaMalloc(&M->rd_off, sizeof(int32_t) * size_t(ntup) * kRdMaxNnz) != cudaSuccess ||
      cudaMalloc(&M->rd_val, sizeof(double) * size_t(ntup) * kRdMaxNnz) != cudaSuccess ||
      cudaMalloc(&M->rd_tid, tid_bytes) != cudaSuccess) {
    cudaGetLastError();
    return drop_csr_dict(M);
  }
  RKMF_CUDA(cudaMemsetAsync(M->rd_tid, 0, tid_bytes, st));
  auto finish = [&](auto* rpp) {
    rd_gather_kernel<<<ntup, 32, 0, st>>>(rpp, v.col, v.val,
                                          static_cast<const long long*>(rrows.p), M->rd_cnt,
                                          M->rd_off, M->rd_val);
    rd_assign_kernel<<<grid, 256, 0, st>>>(
        n, rpp, v.col, v.val, static_cast<const unsigned long long*>(keys.p),
        static_cast<const int16_t*>(slot_id.p), static_cast<const unsigned long long*>(rowhash.p),
        M->rd_cnt, M->rd_off, M->rd_val, M->rd_tid, flags);
  };
  if (v.rp64) finish(static_cast<const int64_t*>(v.row_ptr));
  else finish(static_cast<const int32_t*>(v.row_ptr));
  RKMF_CUDA(cudaGetLastError());
  ctx->launches += 2;
  std::vector<int32_t> hc(static_cast<size_t>(ntup));
  RKMF_CUDA(cudaMemcpyAsync(hf, misc.p, sizeof(hf), cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaMemcpyAsync(hc.data(), M->rd_cnt, sizeof(int32_t) * hc.size(),
                            cudaMemcpyDeviceToHost, st));
  RKMF_CUDA(cudaStreamSynchronize(st));
  if (hf[2]) return drop_csr_dict(M);
  M->view.rtid = M->rd_tid;
  M->view.rcnt = M->rd_cnt;
  M->view.roff = M->rd_off;
  M->view.rval = M->rd_val;
  M->view.rntup = ntup;
  M->view.rkd = *std::max_element(hc.begin(), hc.end());
}

}  // namespace rkmf_b200
