// Row-block partition and halo plan for the multi-GPU path (host only).
//
// The reference is single-process; this is the B200
// build's domain decomposition: contiguous row blocks balanced by nonzeros,
// W / z / f sharded identically, and for every rank the list of off-rank
// columns ("halo") its rows reference. Per Krylov step the owners send those x
// entries (NCCL send/recv in the device path), the local SpMV runs on the
// extended vector [owned | halo], the d-long sketch partials are summed with
// an allreduce and the sketch-space Gram-Schmidt is replicated.
//
// Everything here is plain host C++ so the plan can be tested without a GPU
// (tests/test_partition_gloo.py drives it from two gloo ranks).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "rkmf_b200.h"

extern "C" {

// row_starts[0..nranks]: contiguous blocks whose nonzero counts are as equal
// as the row granularity allows (boundary r is the first row whose prefix
// nnz reaches floor(r * nnz / nranks)).
int rkmf_partition_rows(int64_t n, const int64_t* row_ptr, int32_t nranks, int64_t* row_starts) {
  if (nranks < 1 || n < 0) return RKMF_PARAMETER_ERROR;
  const int64_t nnz = row_ptr[n];
  row_starts[0] = 0;
  for (int32_t r = 1; r < nranks; ++r) {
    const int64_t target = int64_t((__int128)nnz * r / nranks);
    const int64_t* it = std::lower_bound(row_ptr, row_ptr + n + 1, target);
    int64_t row = int64_t(it - row_ptr);
    row = std::max(row, row_starts[r - 1]);
    row = std::min(row, n);
    row_starts[r] = row;
  }
  row_starts[nranks] = n;
  return RKMF_OK;
}

// Halo plan of `rank`. Inputs: the rank's rows [row_starts[rank],
// row_starts[rank+1]) as CSR with local row pointers (row_ptr_local[0] == 0)
// and GLOBAL column indices. Outputs (pass NULL arrays first to get *n_halo;
// each non-NULL array is filled):
//   halo_global[n_halo]  sorted distinct off-rank columns (grouped by owner)
//   recv_counts[nranks]  how many halo entries each rank owns
//   col_local[nnz]       owned column c -> c - row_begin; halo column -> n_local + position
int rkmf_partition_halo(int32_t nranks, int32_t rank, const int64_t* row_starts,
                        const int64_t* row_ptr_local, const int32_t* col_global,
                        int64_t* n_halo, int64_t* halo_global, int64_t* recv_counts,
                        int32_t* col_local) {
  if (rank < 0 || rank >= nranks) return RKMF_PARAMETER_ERROR;
  const int64_t rb = row_starts[rank], re = row_starts[rank + 1];
  const int64_t n_local = re - rb;
  const int64_t nnz = row_ptr_local[n_local];
  std::vector<int64_t> halo;
  for (int64_t k = 0; k < nnz; ++k) {
    const int64_t c = col_global[k];
    if (c < rb || c >= re) halo.push_back(c);
  }
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  *n_halo = int64_t(halo.size());
  // each output is filled when its pointer is given (an empty halo may come
  // with a null halo_global)
  if (halo_global) std::copy(halo.begin(), halo.end(), halo_global);
  if (recv_counts) {
    for (int32_t q = 0; q < nranks; ++q) recv_counts[q] = 0;
    int32_t owner = 0;
    for (int64_t c : halo) {  // halo is sorted and blocks are contiguous
      while (c >= row_starts[owner + 1]) ++owner;
      ++recv_counts[owner];
    }
  }
  if (col_local) {
    for (int64_t k = 0; k < nnz; ++k) {
      const int64_t c = col_global[k];
      if (c >= rb && c < re) {
        col_local[k] = int32_t(c - rb);
      } else {
        const int64_t pos = int64_t(std::lower_bound(halo.begin(), halo.end(), c) - halo.begin());
        col_local[k] = int32_t(n_local + pos);
      }
    }
  }
  return RKMF_OK;
}

}  // extern "C"
