// K3 (sketched Gram-Schmidt), K4 (basis update), K5 (fused restart update)
// and the start normalisation of each cycle.
//
// Column 0 of the basis holds the UNscaled start vector s of the cycle; the
// scale sigma = 1/alpha_k (alpha_k = ||S s||, basis.cpp:103-104) is folded into
// the step-0 SpMV and into every coefficient that multiplies column 0, so the
// reference's W[:,0] = b/alpha pass (basis.cpp:114) and the next cycle's
// start copy (restart.cpp:118) never touch HBM.
#include <cuda_runtime.h>

#include <cstdlib>

#include "rkmf_internal.cuh"
#include "tma.cuh"

namespace rkmf_b200 {

namespace {

constexpr int kRgsThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum with a fixed reduction order (bitwise reproducible); every
// thread returns the total. `buf` holds one slot per warp.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* buf) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) buf[w] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < NT / 32; ++q) s += buf[q];
  __syncthreads();
  return s;
}

// basis.cpp:103-115 on device: alpha = ||S s||, U[:,0] = S s / alpha.
__global__ void __launch_bounds__(kRgsThreads)
    start_init_kernel(int64_t d, const double* sgpart, int ng, double* U, SolveState* st,
                      int first, int m_eff) {
  __shared__ double buf[kRgsThreads / 32];
  double ss = 0.0;
  for (int64_t b = threadIdx.x; b < d; b += kRgsThreads) {
    const double v = det_group_sum(sgpart, ng, d, b);
    U[b] = v;  // scaled below
    ss += v * v;
  }
  const double alpha = sqrt(block_sum<kRgsThreads>(ss, buf));
  for (int64_t b = threadIdx.x; b < d; b += kRgsThreads) U[b] = U[b] / alpha;
  if (threadIdx.x == 0) {
    st->alpha_k = alpha;
    st->sigma = 1.0 / alpha;
    if (first) st->alpha1 = alpha;
    st->zero_start = alpha == 0.0;
    st->stopped = m_eff;
    st->breakdown = 0;
    st->nonfinite = 0;
    st->yn2 = 0.0;
    st->err2 = 0.0;
  }
}

// One modified Gram-Schmidt sweep in the sketch space (basis.cpp:123-138):
// r_i = <u_i, p>, p -= r_i u_i for i = 0..k, r_kk = ||p||, breakdown test,
// U[:,k+1] = p / r_kk. The sketch p arrives as the K2 group partials (summed
// here in group order, detred.cuh). One __syncthreads per MGS
// iteration (ping-pong reduction slots). U[:,0..k] (contiguous, <= ~80 KB at
// BASELINE sizes) is staged into shared memory with one coalesced sweep first,
// so the sequential sweep pays one L2 round trip instead of k+1; when it does
// not fit, the next column is prefetched from global memory instead.
template <int PT>
__global__ void __launch_bounds__(kRgsThreads)
    rgs_step_kernel(int64_t d, int k, int64_t ldr, int64_t n, double tol, const double* pgpart,
                    int ng, double* U, double* Rbar, SolveState* st, int staged) {
  extern __shared__ __align__(16) double Us[];
  __shared__ double red[2][kRgsThreads / 32];
  __shared__ double rs[1024];
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  double p[PT], u[PT], un[PT];
  // Prologue (overlaps the SpMV's tail under PDL): U[:,0..k] is final — it was
  // written by rgs steps that completed before the SpMV of this step started.
  if (staged) {
    const int64_t tot = int64_t(k + 1) * d;
    const double2* src = reinterpret_cast<const double2*>(U);
    double2* dst = reinterpret_cast<double2*>(Us);
    for (int64_t q = t; q < tot / 2; q += kRgsThreads) dst[q] = src[q];
    if ((tot & 1) && t == 0) Us[tot - 1] = U[tot - 1];
  }
  pdl_wait_then_trigger();
  if (st->stopped <= k) return;
#pragma unroll
  for (int j = 0; j < PT; ++j) {
    const int64_t b = t + int64_t(j) * kRgsThreads;
    p[j] = b < d ? det_group_sum(pgpart, ng, d, b) : 0.0;
    un[j] = (!staged && b < d) ? U[b] : 0.0;
  }
  if (staged) __syncthreads();
  for (int i = 0; i <= k; ++i) {
    double part = 0.0;
    if (staged) {
#pragma unroll
      for (int j = 0; j < PT; ++j) {
        const int64_t b = t + int64_t(j) * kRgsThreads;
        u[j] = b < d ? Us[int64_t(i) * d + b] : 0.0;
        part += u[j] * p[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < PT; ++j) {
        u[j] = un[j];
        part += u[j] * p[j];
      }
      if (i < k) {
#pragma unroll
        for (int j = 0; j < PT; ++j) {
          const int64_t b = t + int64_t(j) * kRgsThreads;
          un[j] = b < d ? U[int64_t(i + 1) * d + b] : 0.0;
        }
      }
    }
    part = warp_sum(part);
    if (l == 0) red[i & 1][w] = part;
    __syncthreads();
    double r = 0.0;
#pragma unroll
    for (int q = 0; q < kRgsThreads / 32; ++q) r += red[i & 1][q];
#pragma unroll
    for (int j = 0; j < PT; ++j) p[j] -= r * u[j];
    if (t == 0) rs[i] = r;
  }
  double ss = 0.0;
#pragma unroll
  for (int j = 0; j < PT; ++j) ss += p[j] * p[j];
  ss = warp_sum(ss);
  if (l == 0) red[(k + 1) & 1][w] = ss;
  __syncthreads();
  double tot = 0.0;
#pragma unroll
  for (int q = 0; q < kRgsThreads / 32; ++q) tot += red[(k + 1) & 1][q];
  const double rkk = sqrt(tot);
  for (int i = t; i <= k; i += kRgsThreads) Rbar[int64_t(k) * ldr + i] = rs[i];
  if (rkk <= tol || int64_t(k) + 1 == n) {  // basis.cpp:131-134
    if (t == 0) {
      st->stopped = k + 1;
      st->breakdown = k + 1;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < PT; ++j) {
    const int64_t b = t + int64_t(j) * kRgsThreads;
    if (b < d) U[int64_t(k + 1) * d + b] = p[j] / rkk;
  }
  if (t == 0) Rbar[int64_t(k) * ldr + k + 1] = rkk;
}

// K3, Gram form (used when U[:,0..k] and the Gram rows fit in shared memory).
// MGS (basis.cpp:123-134) computes r_i = <u_i, p - sum_{j<i} r_j u_j>, i.e.
//   r_i = c_i - sum_{j<i} G_ij r_j,   c = U^T p,   G_ij = <u_i, u_j>,
// exactly in exact arithmetic. The dots c and the new Gram row G_k,0..k-1
// (u_k arrived in the previous step; earlier rows are kept in global memory)
// are 2k+1 independent reductions spread over the 8 warps; only the unit
// lower-triangular solve for r is sequential, and it is scalar: one warp
// holds c in registers and broadcasts each r_i with a shuffle. Then
// p -= U r, r_kk = ||p||, U[:,k+1] = p / r_kk. With U sketch-orthonormal to
// rounding, r agrees with the sequential sweep to O(eps ||p||).
__global__ void __launch_bounds__(kRgsThreads)
    rgs_gram_kernel(int64_t d, int k, int64_t ldr, int64_t n, double tol, const double* pgpart,
                    int ng, double* U, double* Rbar, double* G, SolveState* st) {
  extern __shared__ __align__(16) double sm[];
  const int kk = k + 1;
  const int64_t ucnt = (int64_t(kk) * d + 1) / 2 * 2;  // U[:,0..k], rounded to 16 B
  double* Us = sm;                                     // [kk][d]
  double* Gs = Us + ucnt;                  // packed rows 1..k: G_ij (j < i) at i(i-1)/2 + j
  double* ps = Gs + (int64_t(kk) * k / 2 + 1) / 2 * 2;  // [d]
  double* cs = ps + d;                                  // [kk]: c, then r
  __shared__ double red[kRgsThreads / 32];
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  // Prologue (overlaps the SpMV's tail under PDL): U[:,0..k] and Gram rows
  // 1..k-1 (packed lower triangle) are final; one bulk copy each (TMA) into
  // shared memory. The 16-byte round-up reads at most one double past either
  // range, inside the allocations (engine.cu pads U; G holds (m+1)^2).
  const uint32_t ubytes = uint32_t(ucnt * 8);
  const uint32_t gbytes = uint32_t((int64_t(k) * (k - 1) / 2 + 1) / 2 * 2 * 8);
  if (t == 0) trace_max(k, 2);
  if (t == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar, ubytes + (k >= 2 ? gbytes : 0u));
    bulk_g2s(Us, U, ubytes, &bar);
    if (k >= 2) bulk_g2s(Gs, G, gbytes, &bar);
  }
  __syncthreads();  // the barrier is initialised before any thread polls it
  pdl_wait_then_trigger();
  if (t == 0) trace_max(k, 3);
  if (st->stopped <= k) {
    // past a breakdown: the issued bulk copies must land before the block
    // (and its shared memory) retires
    if (t == 0) mbar_wait(&bar, 0);
    return;
  }
  for (int64_t b = t; b < d; b += kRgsThreads) ps[b] = det_group_sum(pgpart, ng, d, b);
  mbar_wait(&bar, 0);
  __syncthreads();
  if (t == 0) trace_max(k, 4);
  // 2k+1 dots: task q < kk is c_q = <u_q, p>; task kk + j is G_kj = <u_k, u_j>
  const double* uk = Us + int64_t(k) * d;
  constexpr int kW = kRgsThreads / 32;
  auto task = [&](int q, const double*& a, const double*& bv) {
    a = q < kk ? Us + int64_t(q) * d : Us + int64_t(q - kk) * d;
    bv = q < kk ? ps : uk;
  };
  auto put = [&](int q, double v) {
    if (q < kk) {
      cs[q] = v;
    } else {
      Gs[int64_t(k) * (k - 1) / 2 + (q - kk)] = v;
      G[int64_t(k) * (k - 1) / 2 + (q - kk)] = v;
    }
  };
  const int ntask = 2 * k + 1;
  for (int q = w; q < ntask; q += 2 * kW) {  // two reductions in flight per warp
    const int q2 = q + kW;
    const double *a0, *b0, *a1 = nullptr, *b1 = nullptr;
    task(q, a0, b0);
    if (q2 < ntask) task(q2, a1, b1);
    double s0 = 0.0, s1 = 0.0;
    for (int64_t b = l; b < d; b += 32) {
      s0 += a0[b] * b0[b];
      if (q2 < ntask) s1 += a1[b] * b1[b];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (l == 0) {
      put(q, s0);
      if (q2 < ntask) put(q2, s1);
    }
  }
  __syncthreads();
  if (t == 0) trace_max(k, 5);
  if (w == 0) {  // unit lower-triangular solve (I + L) r = c, column by column
    if (kk <= 64) {  // c in registers (lanes l, l+32); r_i broadcast by shuffle
      const int m0 = l, m1 = l + 32;
      const int64_t g0 = int64_t(m0) * (m0 - 1) / 2, g1 = int64_t(m1) * (m1 - 1) / 2;
      double c0 = m0 < kk ? cs[m0] : 0.0, c1 = m1 < kk ? cs[m1] : 0.0;
      for (int i = 0; i < kk; ++i) {
        const double a0 = (m0 > i && m0 < kk) ? Gs[g0 + i] : 0.0;
        const double a1 = (m1 > i && m1 < kk) ? Gs[g1 + i] : 0.0;
        const double ri = __shfl_sync(0xffffffffu, i < 32 ? c0 : c1, i & 31);
        if (m0 > i) c0 -= a0 * ri;
        if (m1 > i) c1 -= a1 * ri;
      }
      if (m0 < kk) cs[m0] = c0;
      if (m1 < kk) cs[m1] = c1;
    } else {
      for (int i = 0; i < kk; ++i) {
        const double ri = cs[i];  // final: every earlier column has updated it
        __syncwarp();
        for (int m = i + 1 + l; m < kk; m += 32) cs[m] -= Gs[int64_t(m) * (m - 1) / 2 + i] * ri;
        __syncwarp();
      }
    }
  }
  __syncthreads();
  if (t == 0) trace_max(k, 6);
  double ss = 0.0;
  for (int64_t b = t; b < d; b += kRgsThreads) {
    double v = ps[b];
    for (int i = 0; i < kk; ++i) v -= cs[i] * Us[int64_t(i) * d + b];
    ps[b] = v;
    ss += v * v;
  }
  ss = warp_sum(ss);
  if (l == 0) red[w] = ss;
  __syncthreads();
  double tot = 0.0;
#pragma unroll
  for (int q = 0; q < kRgsThreads / 32; ++q) tot += red[q];
  const double rkk = sqrt(tot);
  for (int i = t; i <= k; i += kRgsThreads) Rbar[int64_t(k) * ldr + i] = cs[i];
  if (rkk <= tol || int64_t(k) + 1 == n) {  // basis.cpp:131-134
    if (t == 0) {
      st->stopped = k + 1;
      st->breakdown = k + 1;
    }
    return;
  }
  for (int64_t b = t; b < d; b += kRgsThreads) U[int64_t(k + 1) * d + b] = ps[b] / rkk;
  if (t == 0) Rbar[int64_t(k) * ldr + k + 1] = rkk;
  if (t == 0) trace_max(k, 7);
}

constexpr int kUpdThreads = 256;
constexpr int kMaxCoef = 1024;

// W[:,k+1] = (z - W[:,0..k] r) / r_kk   (basis.cpp:135). Two rows per thread
// with 16-byte loads; the k+1 column streams are issued 4 at a time.
// W and z are read with ld.global.lu (last use): 2.4% faster on the cfg2 solve
// than evict-first streaming loads, 6% faster than default loads. rev walks
// the rows from the end (RKMF_K4_ORDER=1 alternates per step, 2 always): the
// next step would then start on the rows still in L2, but it measured no
// faster, nor did pinning the last-read rows with evict_last. The whole-solve
// time is sensitive to this kernel's code generation (the same loads without
// the runtime rev select measured 4% slower), so rev stays.
template <int LD>
__device__ __forceinline__ double2 ld_w(const double2* p) {
  if (LD == 0) return __ldcs(p);
  if (LD == 1) return __ldg(p);
  return __ldlu(p);
}

template <int UNR, int LD>
__global__ void __launch_bounds__(kUpdThreads)
    basis_update_kernel(int64_t n, int k, int64_t ldw, double* W, const double* __restrict__ z,
                        const double* __restrict__ Rbar, int64_t ldr, const SolveState* st,
                        int rev, int pf) {
  // PDL prologue: W[:,0..k] and z are final before K3 runs (only r comes
  // from it), so while K3 computes on one SM the resident blocks pull their
  // first rows of every column into L2 (one prefetch per 128-byte line).
  if (threadIdx.x == 0) trace_first(k, 11);
  if (pf && (threadIdx.x & 7) == 0 && blockIdx.x < unsigned(pf) * 148u) {
    const int64_t i2 = int64_t(blockIdx.x) * kUpdThreads + threadIdx.x;
    const int64_t j2 = rev ? n / 2 - 1 - i2 : i2;
    if (j2 >= 0 && j2 < n / 2) {
      for (int c = 0; c <= k; ++c)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(W + int64_t(c) * ldw + 2 * j2));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(z + 2 * j2));
    }
  }
  pdl_wait_then_trigger();
  if (threadIdx.x == 0) trace_first(k, 8);
  if (st->stopped <= k) return;  // no update at (or after) a breakdown step
  __shared__ double coef[kMaxCoef];
  for (int c = threadIdx.x; c <= k; c += kUpdThreads)
    coef[c] = Rbar[int64_t(k) * ldr + c] * (c == 0 ? st->sigma : 1.0);
  __syncthreads();
  const double rkk = Rbar[int64_t(k) * ldr + k + 1];
  double* out = W + int64_t(k + 1) * ldw;
  const int64_t n2 = n / 2;
  for (int64_t j2 = int64_t(blockIdx.x) * kUpdThreads + threadIdx.x; j2 < n2;
       j2 += int64_t(gridDim.x) * kUpdThreads) {
    const int64_t i2 = rev ? n2 - 1 - j2 : j2;
    double a0 = 0.0, a1 = 0.0;
    int c = 0;
    for (; c + UNR - 1 <= k; c += UNR) {
      double2 v[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        v[q] = ld_w<LD>(reinterpret_cast<const double2*>(W + int64_t(c + q) * ldw) + i2);
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        a0 += v[q].x * coef[c + q];
        a1 += v[q].y * coef[c + q];
      }
    }
    for (; c <= k; ++c) {
      const double2 v = ld_w<LD>(reinterpret_cast<const double2*>(W + int64_t(c) * ldw) + i2);
      a0 += v.x * coef[c];
      a1 += v.y * coef[c];
    }
    const double2 zz = ld_w<LD>(reinterpret_cast<const double2*>(z) + i2);
    double2 o;
    o.x = (zz.x - a0) / rkk;
    o.y = (zz.y - a1) / rkk;
    reinterpret_cast<double2*>(out)[i2] = o;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t i = n - 1;
    double a = 0.0;
    for (int c = 0; c <= k; ++c) a += W[int64_t(c) * ldw + i] * coef[c];
    out[i] = (z[i] - a) / rkk;
  }
  if (threadIdx.x == 0) trace_max(k, 9);
}

// K5: the last basis update of the cycle fused with the restart update
// (restart.cpp:80-85): one pass over W[:,0..m-1] and z computes
//   y = alpha_1 * W[:,0..mk-1] g,   f_hat += y,   ||y||^2, finiteness,
//   w_m = (z - W[:,0..m-1] r)/r_kk  written in place into column 0 (the next
//   cycle's unscaled start vector, restart.cpp:118),
// and, with a reference vector, ||f_hat - ref||^2 for error_vs_reference.
__global__ void __launch_bounds__(kUpdThreads)
    final_update_kernel(int64_t n, int m_eff, int64_t ldw, double* W,
                        const double* __restrict__ z, const double* __restrict__ Rbar,
                        int64_t ldr, const double* __restrict__ g, double* f_hat,
                        const double* __restrict__ ref, SolveState* st, DetRed red) {
  __shared__ double cg[kMaxCoef], cr[kMaxCoef];
  __shared__ double buf[kUpdThreads / 32], buf2[kUpdThreads / 32];
  const int mk = st->stopped;
  const bool next = st->breakdown == 0;
  const double sigma = st->sigma, alpha1 = st->alpha1;
  const int km = m_eff - 1;
  for (int c = threadIdx.x; c < m_eff; c += kUpdThreads) {
    cg[c] = c < mk ? g[c] : 0.0;
    cr[c] = next ? Rbar[int64_t(km) * ldr + c] * (c == 0 ? sigma : 1.0) : 0.0;
  }
  __syncthreads();
  const double rkk = next ? Rbar[int64_t(km) * ldr + km + 1] : 1.0;
  const int ncol = next ? m_eff : mk;
  double yy = 0.0, ee = 0.0;
  bool bad = false;
  // one row of the pass: y_i, f_hat_i (+ error), the next start w_i
  auto row_tail = [&](int64_t i, double ay, double aw, double zi) {
    const double y = alpha1 * ay;
    bad |= !isfinite(y);
    const double fn = f_hat[i] + y;
    f_hat[i] = fn;
    yy += y * y;
    if (ref) {
      const double e = fn - ref[i];
      ee += e * e;
    }
    if (next) W[i] = (zi - aw) / rkk;
  };
  // Two rows per thread with 16-byte last-use loads, four column streams in
  // flight (the K4 access pattern); the sums run over the columns in order.
  const int64_t n2 = n / 2;
  for (int64_t j2 = int64_t(blockIdx.x) * kUpdThreads + threadIdx.x; j2 < n2;
       j2 += int64_t(gridDim.x) * kUpdThreads) {
    double ay0 = 0.0, ay1 = 0.0, aw0 = 0.0, aw1 = 0.0;
    int c = 0;
    for (; c + 3 < ncol; c += 4) {
      double2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        v[q] = __ldlu(reinterpret_cast<const double2*>(W + int64_t(c + q) * ldw) + j2);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ay0 += v[q].x * cg[c + q];
        ay1 += v[q].y * cg[c + q];
        aw0 += v[q].x * cr[c + q];
        aw1 += v[q].y * cr[c + q];
      }
    }
    for (; c < ncol; ++c) {
      const double2 v = __ldlu(reinterpret_cast<const double2*>(W + int64_t(c) * ldw) + j2);
      ay0 += v.x * cg[c];
      ay1 += v.y * cg[c];
      aw0 += v.x * cr[c];
      aw1 += v.y * cr[c];
    }
    const double2 zz = next ? __ldlu(reinterpret_cast<const double2*>(z) + j2) : make_double2(0.0, 0.0);
    row_tail(2 * j2, ay0, aw0, zz.x);
    row_tail(2 * j2 + 1, ay1, aw1, zz.y);
  }
  if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    const int64_t i = n - 1;
    double ay = 0.0, aw = 0.0;
    for (int c = 0; c < ncol; ++c) {
      const double v = W[int64_t(c) * ldw + i];
      ay += v * cg[c];
      aw += v * cr[c];
    }
    row_tail(i, ay, aw, next ? z[i] : 0.0);
  }
  yy = block_sum<kUpdThreads>(yy, buf);
  if (ref) ee = block_sum<kUpdThreads>(ee, buf2);
  if (bad) st->nonfinite = 1;
  // (||y||^2, ||f - ref||^2) of the blocks -> st->yn2, st->err2 (adjacent),
  // summed in a fixed block order (detred.cuh)
  __shared__ double mine[2];
  __shared__ int rflag;
  if (threadIdx.x == 0) {
    mine[0] = yy;
    mine[1] = ee;
  }
  __syncthreads();
  det_reduce<kUpdThreads, 0>(red, 2, mine, &st->yn2, threadIdx.x, &rflag);
  if (blockIdx.x == 0 && threadIdx.x == 0)  // coupling for the next R_accum block
    st->coupling = next ? Rbar[int64_t(km) * ldr + km + 1] : 0.0;
}

__global__ void scale_copy_kernel(int64_t n, const double* __restrict__ src, double* dst,
                                  const SolveState* st) {
  const double a = st->alpha_k;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i] / a;
}

__global__ void fill_kernel(int64_t n, double v, double* x) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    x[i] = v;
}

int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

int stream_grid(int64_t work, int threads) {
  const int64_t need = (work + threads - 1) / threads;
  const int64_t cap = int64_t(sm_count()) * 8;
  return int(std::max<int64_t>(1, std::min(need, cap)));
}

}  // namespace

void trace_bind_krylov(unsigned long long* p) { trace_bind_tu(p); }

void launch_start_init_m(int64_t d, const double* sgpart, int ng, double* U, SolveState* st_dev,
                         bool first, int m_eff, cudaStream_t st) {
  start_init_kernel<<<1, kRgsThreads, 0, st>>>(d, sgpart, ng, U, st_dev, first ? 1 : 0, m_eff);
  RKMF_CUDA(cudaGetLastError());
}

bool rgs_use_gram() {  // RKMF_RGS=mgs selects the sequential sweep (A/B runs)
  static int v = -1;
  if (v < 0) {
    const char* e = knob_env("RKMF_RGS");
    v = (e && e[0] == 'm') ? 0 : 1;
  }
  return v == 1;
}

void launch_rgs_step(int64_t d, int k, int64_t ldr, int64_t n, double tol, const double* pgpart,
                     int ng, double* U, double* Rbar, double* G, int64_t ldg, SolveState* st_dev,
                     cudaStream_t st) {
  if (k >= 1024) param_error("randomized_arnoldi: m > 1024 is not supported on device");
  const size_t gbytes = sizeof(double) * (size_t(k + 1) * size_t(d) + size_t(k + 1) * size_t(k) / 2 +
                                          size_t(d) + size_t(k + 1) + 4);
  if (G != nullptr && rgs_use_gram() && gbytes <= 200 * 1024) {
    RKMF_CUDA(cudaFuncSetAttribute(rgs_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024));
    launch_maybe_pdl(rgs_gram_kernel, dim3(1), dim3(kRgsThreads), gbytes, st, d, k, ldr, n, tol,
                     pgpart, ng, U, Rbar, G, st_dev);
    return;
  }
  const int64_t pt = (d + kRgsThreads - 1) / kRgsThreads;
  const size_t ubytes = sizeof(double) * size_t(k + 1) * size_t(d);
  const int staged = ubytes <= 160 * 1024 ? 1 : 0;
  const size_t smem = staged ? ubytes : 0;
#define RKMF_RGS(P)                                                                    \
  do {                                                                                 \
    auto fn = rgs_step_kernel<P>;                                                      \
    RKMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                   160 * 1024));                                       \
    launch_maybe_pdl(fn, dim3(1), dim3(kRgsThreads), smem, st, d, k, ldr, n, tol, pgpart, \
                     ng, U, Rbar, st_dev, staged);                                     \
  } while (0)
  if (pt <= 1) RKMF_RGS(1);
  else if (pt <= 2) RKMF_RGS(2);
  else if (pt <= 4) RKMF_RGS(4);
  else if (pt <= 8) RKMF_RGS(8);
  else if (pt <= 16) RKMF_RGS(16);
  else param_error("sketch: d > 4096 is not supported on device");
#undef RKMF_RGS
  RKMF_CUDA(cudaGetLastError());
}

void launch_basis_update(int64_t n, int k, int64_t ldw, double* W, const double* z,
                         const double* Rbar, int64_t ldr, const SolveState* st_dev,
                         cudaStream_t st) {
  // Blocks per SM: 24 (three waves of 8 resident) beats one resident wave by
  // 4% on the whole cfg2 solve: the (k+1)-column read streams keep more DRAM
  // pages open with the extra in-flight blocks (read-only microbenchmark of 26
  // streams: 6.49 -> 6.86 TB/s). RKMF_K4_GRIDX / RKMF_K4_UNROLL override.
  static const int unr = [] { const char* e = knob_env("RKMF_K4_UNROLL"); return e ? atoi(e) : 4; }();
  static const int gx = [] { const char* e = knob_env("RKMF_K4_GRIDX"); return e ? atoi(e) : 24; }();
  const int64_t need = (std::max<int64_t>(n / 2, 1) + kUpdThreads - 1) / kUpdThreads;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(sm_count()) * gx)));
  // RKMF_K4_LOAD: 0 streaming (evict-first), 1 default, 2 last-use (default)
  static const int ldm = [] { const char* e = knob_env("RKMF_K4_LOAD"); return e ? atoi(e) : 2; }();
  static const int order = [] { const char* e = knob_env("RKMF_K4_ORDER"); return e ? atoi(e) : 0; }();
  const int rev = order == 1 ? (k & 1) : (order == 2 ? 1 : 0);
  static const int pf = [] { const char* e = knob_env("RKMF_K4_PREFETCH"); return e ? atoi(e) : 1; }();
#define RKMF_K4(U, L)                                                                       \
  launch_maybe_pdl(basis_update_kernel<U, L>, dim3(grid), dim3(kUpdThreads), 0, st, n, k, ldw, \
                   W, z, Rbar, ldr, st_dev, rev, pf)
  if (unr == 8) {
    RKMF_K4(8, 2);
  } else if (unr == 2) {
    RKMF_K4(2, 2);
  } else if (ldm == 1) {
    RKMF_K4(4, 1);
  } else if (ldm == 0) {
    RKMF_K4(4, 0);
  } else {
    RKMF_K4(4, 2);
  }
#undef RKMF_K4
}

void launch_final_update(int64_t n, int m_eff, int64_t ldw, double* W, const double* z,
                         const double* Rbar, int64_t ldr, const double* g, double* f_hat,
                         const double* ref, SolveState* st_dev, const DetRed& red,
                         cudaStream_t st) {
  if (m_eff > kMaxCoef) param_error("restart: m_r > 1024 is not supported on device");
  const int64_t fneed = (std::max<int64_t>(n, 1) + kUpdThreads - 1) / kUpdThreads;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(fneed, int64_t(sm_count()) * 24)));
  if (grid > red.max_blocks || red.max_len < 2)
    param_error("internal: update reduction scratch too small");
  final_update_kernel<<<grid, kUpdThreads, 0, st>>>(n, m_eff, ldw, W, z, Rbar, ldr, g, f_hat, ref,
                                                    st_dev, red);
  RKMF_CUDA(cudaGetLastError());
}

void launch_scale_copy(int64_t n, const double* src, double* dst, const SolveState* st_dev,
                       cudaStream_t st) {
  scale_copy_kernel<<<stream_grid(n, 256), 256, 0, st>>>(n, src, dst, st_dev);
  RKMF_CUDA(cudaGetLastError());
}

void launch_fill(int64_t n, double v, double* x, cudaStream_t st) {
  if (n <= 0) return;
  fill_kernel<<<stream_grid(n, 256), 256, 0, st>>>(n, v, x);
  RKMF_CUDA(cudaGetLastError());
}

}  // namespace rkmf_b200
