// Deterministic grid reductions of per-block partial vectors.
//
// The reference is bitwise reproducible run to run (rng.hpp:13-16,
// test_restart.cpp:405-443); a grid that adds its block partials with fp64
// atomics is not (the arrival order changes the rounding). Here block b
// writes its L partials to part[b][0..L); blocks form groups of gsz
// consecutive indices; the last block of a group to arrive (a ticket counter)
// sums the group's partials in block order into gpart[g][0..L). Which block
// does the work depends on timing, the order of every addition does not.
//
// Two ways to finish:
//   * det_group_reduce (K2, every Krylov step): stop at the ng group
//     partials; the consumer (K3, start_init) sums them in group order while
//     it reads them anyway (det_group_sum), so K2's tail grows by one store,
//     one ticket round trip and one sqrt(grid)-long read, not by a second
//     level;
//   * det_reduce (K5, once per cycle): a second ticket level sums the group
//     partials into out[0..L).
// A 2D grid reduces gridDim.y independent slices (blockIdx.y), each with its
// own partials, groups and tickets (the classical builder's k+1 dots).
// Tickets are reset by the block that consumed them, so consecutive launches
// on one stream reuse the scratch without a memset. The release/acquire
// pattern is the one of cooperative-groups grid sync: bar.sync, then one
// thread fences and takes the ticket.
#pragma once

#include <cstdint>

namespace rkmf_b200 {

struct DetRed {
  double* part = nullptr;      // [blocks][L]
  double* gpart = nullptr;     // [groups][L]
  unsigned* tick = nullptr;    // [groups + 1], zero between launches
  int max_blocks = 0;          // capacity of part (blocks)
  int max_len = 0;             // capacity per block (L)
  int max_groups = 0;          // capacity of gpart (groups, over all slices) and tick (+slices)
  int groups = 0;              // host side: group partials the last launch wrote
};

// groups of ceil(sqrt(blocks)) consecutive blocks
__host__ __device__ inline int det_group_size(int blocks) {
  int g = 1;
  while (g * g < blocks) ++g;
  return g;
}
__host__ __device__ inline int det_groups(int blocks) {
  const int g = det_group_size(blocks);
  return (blocks + g - 1) / g;
}

template <int NT, int BAR>
__device__ __forceinline__ void det_bar() {
  asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
}

// sum_{q in [q0, q1)} a[q * L + j] in q order, W loads in flight (one L2
// round trip per W terms)
template <int W = 8>
__device__ __forceinline__ double det_ordered_sum(const double* a, int64_t L, int q0, int q1,
                                                  int64_t j) {
  double s = 0.0;
  for (int q = q0; q < q1; q += W) {
    double v[W];
#pragma unroll
    for (int i = 0; i < W; ++i) v[i] = q + i < q1 ? __ldcg(a + int64_t(q + i) * L + j) : 0.0;
#pragma unroll
    for (int i = 0; i < W; ++i)
      if (q + i < q1) s += v[i];
  }
  return s;
}

// Value j of the reduced vector from the ng group partials (the consumer side
// of det_group_reduce; call after the producing grid completed).
template <int W = 32>
__device__ __forceinline__ double det_group_sum(const double* gpart, int ng, int64_t L,
                                                int64_t j) {
  return det_ordered_sum<W>(gpart, L, 0, ng, j);
}

// Level 1, called by the NT threads u = 0..NT-1 of every block that take
// part (synchronised on named barrier BAR) once `mine` (shared memory, L
// values) holds the block's partials. Returns true in the block that wrote
// its group's partial. flag: a __shared__ int of the caller.
template <int NT, int BAR, int W = 8>
__device__ __forceinline__ bool det_group_reduce(const DetRed& r, int L, const double* mine,
                                                 int u, int* flag) {
  const int nb = int(gridDim.x), b = int(blockIdx.x);
  const int gsz = det_group_size(nb), ng = (nb + gsz - 1) / gsz;
  const int g = b / gsz, b0 = g * gsz, b1 = min(nb, b0 + gsz);
  const int64_t sl = blockIdx.y;
  double* part = r.part + sl * nb * L;
  double* gpart = r.gpart + sl * ng * L;
  unsigned* tick = r.tick + sl * (ng + 1);
  for (int j = u; j < L; j += NT) part[int64_t(b) * L + j] = mine[j];
  det_bar<NT, BAR>();
  if (u == 0) {
    __threadfence();  // release the block's stores (ordered after the barrier)
    *flag = atomicAdd(tick + g, 1u) == unsigned(b1 - b0 - 1);
    if (*flag) __threadfence();  // acquire the group's partials
  }
  det_bar<NT, BAR>();
  if (!*flag) return false;
  for (int j = u; j < L; j += NT)
    gpart[int64_t(g) * L + j] = det_ordered_sum<W>(part, L, b0, b1, j);
  if (u == 0) tick[g] = 0u;
  return true;
}

// Both levels: writes out[0..L) once per launch, in the last group to finish.
template <int NT, int BAR>
__device__ __forceinline__ void det_reduce(const DetRed& r, int L, const double* mine,
                                           double* out, int u, int* flag) {
  if (!det_group_reduce<NT, BAR>(r, L, mine, u, flag)) return;
  const int ng = det_groups(int(gridDim.x));
  const int64_t sl = blockIdx.y;
  const double* gpart = r.gpart + sl * ng * L;
  unsigned* tick = r.tick + sl * (ng + 1);
  det_bar<NT, BAR>();
  if (u == 0) {
    __threadfence();
    *flag = atomicAdd(tick + ng, 1u) == unsigned(ng - 1);
    if (*flag) __threadfence();
  }
  det_bar<NT, BAR>();
  if (!*flag) return;
  for (int j = u; j < L; j += NT) out[j] = det_ordered_sum(gpart, L, 0, ng, j);
  if (u == 0) tick[ng] = 0u;
}

}  // namespace rkmf_b200
