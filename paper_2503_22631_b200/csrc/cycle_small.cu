// K-cycle: the m steps of one randomized-Arnoldi cycle (basis.cpp:119-139) in
// ONE cooperative kernel, for matrices small enough to live in L2 (cfg1:
// 65K rows). There each step of the three-kernel chain (K2 SpMV + sketch, K3
// sketched Gram-Schmidt, K4 basis update) is a few microseconds of work
// behind ~10 us of launch, PDL hand-off and grid-drain latency; here a step is
// three phases separated by two grid barriers:
//   A  every block: SpMV of its tiles' rows (CSR, column order: the same z as
//      K2) and the sketch gather of those tiles (the K2 tile layout, read
//      from L2), block partials -> fixed-order group partials (detred.cuh);
//   -- grid barrier --
//   B  every block, redundantly and identically: the sketch p from the group
//      partials, the Gram-form Gram-Schmidt of K3 (c = U^T p, the new Gram
//      row, the unit-triangular solve, p -= U r, r_kk), the breakdown test.
//      Block 0 alone writes U[:,k+1], Rbar and the Gram row; every block takes
//      the same decision from the same bytes;
//   C  every block: w_{k+1} = (z - W[:,0..k] r) / r_kk for its rows (K4's
//      arithmetic, same order);
//   -- grid barrier -- (not after the last step, or after C is skipped)
// The per-cycle work around it (start sketch, dense f, K5) is unchanged.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "rkmf_internal.cuh"
#include "detred.cuh"

namespace cg = cooperative_groups;

namespace rkmf_b200 {

namespace {

constexpr int kCyGroups = 4;                      // tiles in flight per block
constexpr int kCyThreads = kCyGroups * kTileRows;  // 512
constexpr int kCyMaxKK = 64;                      // k + 1 <= 64: register triangular solve
#ifndef RKMF_CY_TWO_LEVEL
#define RKMF_CY_TWO_LEVEL 1
#endif

__device__ __forceinline__ double cy_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename RP>
__global__ void __launch_bounds__(kCyThreads)
    cycle_small_kernel(int64_t n, const RP* __restrict__ rp, const int32_t* __restrict__ ci,
                       const double* __restrict__ val, int d, int64_t off_stride,
                       const uint16_t* __restrict__ toff, const uint8_t* __restrict__ tent,
                       int64_t ent_stride, double sscale, int m_eff, int fuse_last, double* W,
                       int64_t ldw, double* z, double* U, double* Rbar, int64_t ldr, double* G,
                       double tol, int64_t n_global, SolveState* st, DetRed red, int stage_cap) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  const int t = threadIdx.x, grp = t / kTileRows, u = t % kTileRows;
  const int w = t >> 5, l = t & 31;
  constexpr int kW = kCyThreads / 32;
  const int dd = (d + 1) / 2 * 2;
  double* zs2 = sm;                                 // [kCyGroups][256]
  double* acc = zs2 + kCyGroups * 2 * kTileRows;    // [kCyGroups][dd]
  double* ps = acc + kCyGroups * dd;                // [dd]
  double* cs = ps + dd;                             // [kCyMaxKK]
  double* Gs = cs + kCyMaxKK;                       // packed Gram rows 1..k: [kCyMaxKK^2 / 2]
  // U[:,0..m] resident in every block: column 0 from start_init, column k+1
  // computed by every block from the same bytes (block 0 also stores it)
  double* Us = Gs + kCyMaxKK * kCyMaxKK / 2;        // [m_eff + 1][d]
  double* tmp = Us + int64_t(m_eff + 1) * d;        // [kCyThreads]: reduction chunks
  // stage_cap > 0: every group has one tile (one round), and its CSR rows and
  // sketch layout (constant over the cycle) are staged in shared memory once:
  // per group [stage_cap] values, [stage_cap] columns, [129] row offsets, the
  // header and the entry block
  const int64_t hb = int64_t(off_stride) * 2;
  const int64_t gstage = stage_cap > 0 ? int64_t(stage_cap) * 12 + 129 * 4 + hb + ent_stride : 0;
  unsigned char* stg = reinterpret_cast<unsigned char*>(tmp + kCyThreads) + grp * ((gstage + 15) & ~15);
  double* sval = reinterpret_cast<double*>(stg);
  int32_t* scol = reinterpret_cast<int32_t*>(stg + int64_t(stage_cap) * 8);
  int32_t* srp = scol + stage_cap;
  uint16_t* shdr = reinterpret_cast<uint16_t*>(srp + 129);
  uint8_t* sent = reinterpret_cast<uint8_t*>(shdr) + hb;
  __shared__ double red_s[kW];
  const int64_t tiles = (n + kTileRows - 1) / kTileRows;
  const int32_t n32 = int32_t(n);
  const double sigma = st->sigma;
  for (int j = t; j < d; j += kCyThreads) Us[j] = __ldcg(U + j);
  const int64_t mytile = int64_t(blockIdx.x) * kCyGroups + grp;
  if (stage_cap > 0 && mytile < tiles) {
    const int64_t r0 = mytile * kTileRows, r1 = min(n, r0 + kTileRows);
    const int64_t e0 = int64_t(rp[r0]), ecnt = int64_t(rp[r1]) - e0;
    for (int64_t e = u; e < ecnt; e += kTileRows) {
      sval[e] = val[e0 + e];
      scol[e] = ci[e0 + e];
    }
    for (int64_t r = u; r <= r1 - r0; r += kTileRows) srp[r] = int32_t(int64_t(rp[r0 + r]) - e0);
    const uint16_t* gh = toff + mytile * off_stride;
    for (int64_t q = u; q < off_stride; q += kTileRows) shdr[q] = gh[q];
    const uint32_t* ge = reinterpret_cast<const uint32_t*>(tent + mytile * ent_stride);
    uint32_t* se = reinterpret_cast<uint32_t*>(sent);
    for (int64_t q = u; q < ent_stride / 4; q += kTileRows) se[q] = ge[q];
  }
  __syncthreads();
  for (int k = 0; k < m_eff; ++k) {
    const bool last = fuse_last && k == m_eff - 1;
    // ---- A: SpMV + sketch of this block's tiles ----
    for (int j = t; j < kCyGroups * dd; j += kCyThreads) acc[j] = 0.0;
    __syncthreads();
    const double* x = W + int64_t(k) * ldw;
    const double xs = k == 0 ? sigma : 1.0;
    double* zsg = zs2 + grp * 2 * kTileRows;
    double* accg = acc + grp * dd;
    for (int64_t tile = int64_t(blockIdx.x) * kCyGroups + grp; tile < tiles;
         tile += int64_t(gridDim.x) * kCyGroups) {
      const int32_t row = int32_t(tile) * kTileRows + u;
      const bool live = row < n32;
      double sum = 0.0;
      if (live) {
        if (stage_cap > 0) {
          const int e1 = srp[u + 1];
          for (int e = srp[u]; e < e1; ++e) sum += sval[e] * __ldcg(x + scol[e]);
        } else {
          const int64_t e1 = int64_t(rp[row + 1]);
          for (int64_t e = int64_t(rp[row]); e < e1; ++e) sum += val[e] * __ldcg(x + ci[e]);
        }
        sum *= xs;
        z[row] = sum;
      }
      const double zt = live ? sum * sscale : 0.0;
      zsg[u] = zt;
      zsg[kTileRows + u] = -zt;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(kTileRows) : "memory");
      if (stage_cap > 0)
        sketch_tile_gather(u, d, shdr, sent, zsg, accg);
      else
        sketch_tile_gather(u, d, toff + tile * off_stride, tent + tile * ent_stride, zsg, accg);
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(kTileRows) : "memory");
    }
    __syncthreads();
    for (int j = t; j < d; j += kCyThreads) {  // the groups in a fixed order
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kCyGroups; ++q) s += acc[q * dd + j];
      red.part[int64_t(blockIdx.x) * d + j] = s;
    }
    grid.sync();
    // ---- B: sketched Gram-Schmidt (K3's Gram form), every block ----
#if RKMF_CY_TWO_LEVEL
    // p: one warp per bin sums the blocks' partials (lane l takes blocks l,
    // l + 32, ... in order, then a fixed butterfly) into red.gpart, a second
    // barrier, and every block reads the d values
    {
      const int nb = int(gridDim.x);
      for (int j = int(blockIdx.x) * kW + w; j < d; j += nb * kW) {
        double v = 0.0;
        for (int b = l; b < nb; b += 32) v += __ldcg(red.part + int64_t(b) * d + j);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (l == 0) red.gpart[j] = v;
      }
      grid.sync();
      for (int jj = t; jj < d; jj += kCyThreads) ps[jj] = __ldcg(red.gpart + jj);
    }
#else
    // p = sum over the blocks' partials in a fixed order: nch chunks of
    // consecutive blocks per bin (independent loads in flight), then the
    // chunks in order
    {
      const int nb = int(gridDim.x);
      const int nch = d >= kCyThreads ? 1 : min(kCyThreads / d, nb);
      for (int q = t; q < nch * d; q += kCyThreads) {
        const int j = q % d, c = q / d;
        const int b0 = int(int64_t(c) * nb / nch), b1 = int(int64_t(c + 1) * nb / nch);
        tmp[q] = det_ordered_sum<8>(red.part, d, b0, b1, j);
      }
      __syncthreads();
      for (int j = t; j < d; j += kCyThreads) {
        double s = 0.0;
        for (int c = 0; c < nch; ++c) s += tmp[c * d + j];
        ps[j] = s;
      }
    }
#endif
    const int kk = k + 1;
    const int64_t g0 = int64_t(k) * (k - 1) / 2;  // packed row k starts here
    __syncthreads();
    const double* uk = Us + int64_t(k) * d;
    const int ntask = 2 * k + 1;  // c_q = <u_q, p> (q < kk), G_kj = <u_k, u_j> (j < k)
    for (int q = w; q < ntask; q += kW) {
      const double* a = q < kk ? Us + int64_t(q) * d : Us + int64_t(q - kk) * d;
      const double* bv = q < kk ? ps : uk;
      double s = 0.0;
      for (int j = l; j < d; j += 32) s += a[j] * bv[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (l == 0) {
        if (q < kk) {
          cs[q] = s;
        } else {
          Gs[g0 + (q - kk)] = s;
          if (blockIdx.x == 0) G[g0 + (q - kk)] = s;
        }
      }
    }
    __syncthreads();
    if (w == 0) {  // unit lower-triangular solve (I + L) r = c (kk <= 64)
      const int m0 = l, m1 = l + 32;
      const int64_t q0 = int64_t(m0) * (m0 - 1) / 2, q1 = int64_t(m1) * (m1 - 1) / 2;
      double c0 = m0 < kk ? cs[m0] : 0.0, c1 = m1 < kk ? cs[m1] : 0.0;
      for (int i = 0; i < kk; ++i) {
        const double a0 = (m0 > i && m0 < kk) ? Gs[q0 + i] : 0.0;
        const double a1 = (m1 > i && m1 < kk) ? Gs[q1 + i] : 0.0;
        const double ri = __shfl_sync(0xffffffffu, i < 32 ? c0 : c1, i & 31);
        if (m0 > i) c0 -= a0 * ri;
        if (m1 > i) c1 -= a1 * ri;
      }
      if (m0 < kk) cs[m0] = c0;
      if (m1 < kk) cs[m1] = c1;
    }
    __syncthreads();
    double ss = 0.0;
    for (int j = t; j < d; j += kCyThreads) {
      double v = ps[j];
      for (int i = 0; i < kk; ++i) v -= cs[i] * Us[int64_t(i) * d + j];
      ps[j] = v;
      ss += v * v;
    }
    ss = cy_warp_sum(ss);
    if (l == 0) red_s[w] = ss;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int q = 0; q < kW; ++q) tot += red_s[q];
    const double rkk = sqrt(tot);
    const bool brk = rkk <= tol || int64_t(k) + 1 == n_global;  // basis.cpp:131-134
    if (!brk)
      for (int j = t; j < d; j += kCyThreads) {
        const double v = ps[j] / rkk;
        Us[int64_t(k + 1) * d + j] = v;
        if (blockIdx.x == 0) U[int64_t(k + 1) * d + j] = v;
      }
    if (blockIdx.x == 0) {
      for (int i = t; i <= k; i += kCyThreads) Rbar[int64_t(k) * ldr + i] = cs[i];
      if (t == 0) {
        if (brk) {
          st->stopped = k + 1;
          st->breakdown = k + 1;
        } else {
          Rbar[int64_t(k) * ldr + k + 1] = rkk;
        }
      }
    }
    if (brk || last) break;  // the same decision in every block
    // ---- C: w_{k+1} = (z - W[:,0..k] r) / r_kk, this block's rows ----
    if (t <= k) cs[t] *= (t == 0 ? sigma : 1.0);  // column 0 holds the unscaled start
    __syncthreads();
    double* out = W + int64_t(k + 1) * ldw;
    for (int64_t tile = int64_t(blockIdx.x) * kCyGroups + grp; tile < tiles;
         tile += int64_t(gridDim.x) * kCyGroups) {
      const int32_t row = int32_t(tile) * kTileRows + u;
      if (row >= n32) continue;
      double a = 0.0;
      int c = 0;
      for (; c + 7 <= k; c += 8) {  // eight independent loads in flight
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = __ldcg(W + int64_t(c + q) * ldw + row);
#pragma unroll
        for (int q = 0; q < 8; ++q) a += v[q] * cs[c + q];
      }
      for (; c <= k; ++c) a += __ldcg(W + int64_t(c) * ldw + row) * cs[c];
      out[row] = (__ldcg(z + row) - a) / rkk;
    }
    grid.sync();
  }
}

template <typename RP>
size_t cycle_small_smem(int d, int m_eff, int64_t gstage) {
  const int dd = (d + 1) / 2 * 2;
  return sizeof(double) *
             size_t(kCyGroups * 2 * kTileRows + kCyGroups * dd + dd + kCyMaxKK +
                    kCyMaxKK * kCyMaxKK / 2 + (m_eff + 1) * d + kCyThreads + 2) +
         size_t(kCyGroups) * size_t((gstage + 15) & ~15);
}

int sms_count() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

}  // namespace

bool cycle_small_applicable(const CsrView* A, const SketchView* S, int64_t m_eff) {
  if (!A || !S || A->rp64 || A->n_rows != A->n_cols) return false;
  if (A->n_rows > kCycleSmallMaxRows || m_eff + 1 > kCyMaxKK || S->d > 1024) return false;
  return true;
}

bool launch_cycle_small(const CsrView* A, const SketchView* S, int m_eff, bool fuse_last,
                        double* W, int64_t ldw, double* z, double* U, double* Rbar, int64_t ldr,
                        double* G, double tol, int64_t n_global, SolveState* st_dev,
                        DetRed& red, cudaStream_t st) {
  auto fn = cycle_small_kernel<int32_t>;
  // one tile per group (a single round) -> stage its rows and layout once
  const int64_t tiles0 = (A->n_rows + kTileRows - 1) / kTileRows;
  int stage_cap = int(std::min<int64_t>(A->max_tile_nnz, int64_t(1) << 20));
  const int64_t gstage = int64_t(stage_cap) * 12 + 129 * 4 + 2 * tile_off_stride(S->d) + S->ent_stride;
  size_t smem = cycle_small_smem<int32_t>(int(S->d), m_eff, gstage);
  if (tiles0 > int64_t(kCyGroups) * sms_count() || smem > 200 * 1024) {
    stage_cap = 0;
    smem = cycle_small_smem<int32_t>(int(S->d), m_eff, 0);
  }
  if (smem > 200 * 1024) return false;
  if (smem > 48 * 1024)
    RKMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int per = 0;
  RKMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kCyThreads, smem));
  if (per < 1) return false;
  const int64_t tiles = (A->n_rows + kTileRows - 1) / kTileRows;
  const int64_t units = (tiles + kCyGroups - 1) / kCyGroups;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(units, int64_t(per) * sms_count())));
  if (grid > red.max_blocks || S->d > red.max_len) return false;
  red.groups = det_groups(grid);
  int64_t n = A->n_rows;
  const int32_t* rp = static_cast<const int32_t*>(A->row_ptr);
  const int32_t* ci = A->col;
  const double* val = A->val;
  int d = int(S->d);
  int64_t off_stride = tile_off_stride(S->d);
  const uint16_t* toff = S->tile_off;
  const uint8_t* tent = S->tile_ent;
  int64_t es = S->ent_stride;
  double sscale = S->scale;
  int fl = fuse_last ? 1 : 0;
  void* args[] = {&n,  &rp, &ci,   &val, &d,    &off_stride, &toff, &tent,     &es,
                  &sscale, &m_eff, &fl, &W, &ldw, &z, &U, &Rbar, &ldr, &G, &tol, &n_global,
                  &st_dev, &red, &stage_cap};
  RKMF_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), dim3(grid),
                                        dim3(kCyThreads), args, smem, st));
  return true;
}

}  // namespace rkmf_b200
