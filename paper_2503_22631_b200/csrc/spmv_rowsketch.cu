// K2 (row-sketch form): fused SpMV over the diagonal copy + sparse-sign
// sketch, with the sketch done by the SpMV threads themselves.
//
// The warp-specialised K2 (spmv_pipe.cu) hands each tile's z to 128
// dedicated sketch threads, which gather the tile's bins from a bin-sorted
// entry list: per slot a header lookup, per entry a byte load and a signed-z
// load. That costs more issue slots than the SpMV itself. Here the thread
// that computes z_r adds its zeta = 8 signed contributions (sketch.cpp:55-61,
// column r of S) straight into its warp's private accumulator in shared
// memory, one slot at a time: the slots of each 32-column warp tile are
// edge-coloured at setup so that the 32 lanes of a slot hit distinct bins, and
// the add is a plain read-add-write (fp64 shared atomics are CAS loops on
// sm_100a: 69 vs 40 us per launch when used here). There is no hand-off, no
// signed-z table and no slot header: the per-tile sketch stream is 9 bytes
// per row (rbin: 8 row indices as uint8, sbit: 8 sign bits; sketch.cu
// launch_sketch_rowbins), and a block is 128 + 32 threads, so more blocks fit
// per SM. Requires zeta == 8 and d <= 255 (else spmv_pipe.cu).
//
// The per-warp accumulators are summed in warp order at the end and added to
// the global partials with one atomic per bin (as in spmv_pipe.cu): the sum
// within a block is deterministic, across blocks it follows the atomics.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "rkmf_internal.cuh"
#include "tma.cuh"

namespace rkmf_b200 {

namespace {

constexpr int kRsStages = 8;
constexpr int kRsThreads = kTileRows + 32;  // one SpMV thread per row + producer warp

struct RsLayout {
  uint32_t val, bin, sgn, stride;
};
__host__ __device__ inline RsLayout rs_layout(int nd) {
  RsLayout L;
  L.val = 0;
  L.bin = uint32_t(nd) * kTileRows * 8u;
  L.sgn = L.bin + kTileRows * 8u;
  L.stride = (L.sgn + kTileRows + 127u) & ~127u;
  return L;
}

// ND diagonals (val == nullptr: the identity, i.e. the sketch of x alone).
template <int ND>
__global__ void __launch_bounds__(kRsThreads)
    spmv_rowsketch_kernel(int64_t n, const double* __restrict__ val, const double* __restrict__ x,
                          const double* xscale, double* __restrict__ z, int64_t num_tiles, int d,
                          const uint8_t* __restrict__ rbin, const uint8_t* __restrict__ sbit,
                          const uint8_t* __restrict__ wslow,
                          double sscale, double* pacc, const int32_t* stop, int step, int nstages,
                          const int32_t* __restrict__ doff, int64_t ncols, int dstride,
                          int l2_hints) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kRsStages], empty[kRsStages];
  __shared__ int32_t doff_s[kMaxDiag];
  const RsLayout L = rs_layout(val ? ND : 0);
  const int dpad = (d + 2) / 2 * 2;  // bins 0..d-1 and the trash bin d
  double* acc = reinterpret_cast<double*>(smem + nstages * L.stride);  // [4 warps][dpad]
  const int t = threadIdx.x;
  if (t < kMaxDiag) doff_s[t] = doff ? doff[t] : 0;
  if (t == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTileRows / 32);  // one arrival per SpMV warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int b = t; b < 4 * dpad; b += kRsThreads) acc[b] = 0.0;
  __syncthreads();
  const bool producer = t == kTileRows;
  if (!producer) {
    if (t > kTileRows) return;  // idle lanes of the producer warp
    pdl_wait_then_trigger();
    if (stop != nullptr && *stop <= step) return;  // breakdown earlier in this cycle
  }

  if (producer) {  // ---------------- producer: one lane ----------------
    bool waited = false;
    auto wait_prev = [&](int issued) {  // as in spmv_pipe.cu: constant streams go first
      waited = true;
      asm volatile("griddepcontrol.wait;" ::: "memory");
      if (stop != nullptr && *stop <= step) {
        for (int i = 0; i < issued; ++i) mbar_wait(&full[i], 0u);
        return true;
      }
      return false;
    };
    const uint64_t pol = l2_policy(l2_hints >= 1 ? 1 : 0);
    const uint64_t mpol = l2_policy(l2_hints);
    const uint32_t vbytes = val ? uint32_t(ND) * kTileRows * 8u : 0u;
    int s = 0, it = 0;
    uint32_t eph = 0;
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      if (it == nstages && !waited && wait_prev(it)) return;
      if (it >= nstages) mbar_wait(&empty[s], eph);
      unsigned char* st = smem + s * L.stride;
      mbar_expect_tx(&full[s], vbytes + kTileRows * 9u);
      if (val) bulk_g2s(st + L.val, val + tile * int64_t(ND) * kTileRows, vbytes, &full[s], pol);
      bulk_g2s(st + L.bin, rbin + tile * int64_t(kTileRows) * 8, kTileRows * 8u, &full[s], mpol);
      bulk_g2s(st + L.sgn, sbit + tile * int64_t(kTileRows), kTileRows, &full[s], mpol);
      if (++s == nstages) {
        s = 0;
        if (it >= nstages) eph ^= 1u;
      }
    }
    if (!waited) wait_prev(it);
    return;
  }

  // ---------------- SpMV + sketch threads: row rl of each tile ----------------
  const int rl = t, w = t >> 5, lane = t & 31;
  double* accw = acc + w * dpad;
  const double xs = xscale ? *xscale : 1.0;
  auto load_x = [&](int64_t tl, double* dst) {  // spmv_pipe.cu FMT 2
    int doffr[ND];
    if (dstride == 0) {
#pragma unroll
      for (int q = 0; q < ND; ++q) doffr[q] = doff_s[q];
    } else {
      const int4* p = reinterpret_cast<const int4*>(doff + tl * kMaxDiag);
      const int4 a = __ldg(p), b = __ldg(p + 1);
      const int all[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int q = 0; q < ND; ++q) doffr[q] = all[q];
    }
    const int64_t r0 = tl * kTileRows, row = r0 + rl;
    if (r0 + doffr[0] >= 0 && r0 + kTileRows - 1 + doffr[ND - 1] < ncols && r0 + kTileRows <= n) {
      const double* xr = x + row;
#pragma unroll
      for (int q = 0; q < ND; ++q) dst[q] = __ldg(xr + doffr[q]);
    } else {
#pragma unroll
      for (int q = 0; q < ND; ++q) {
        const int64_t c = row + doffr[q];
        dst[q] = (row < n && c >= 0 && c < ncols) ? __ldg(x + c) : 0.0;
      }
    }
  };
  int s = 0;
  uint32_t ph = 0;
  auto step_tile = [&](int64_t tile, const double* xc, double* xn) {
    const int64_t nt = tile + gridDim.x;
    if (nt < num_tiles) load_x(nt, xn);
    const bool slow = __ldg(wslow + tile * (kTileRows / 32) + w) != 0;
    mbar_wait(&full[s], ph);
    const unsigned char* st = smem + s * L.stride;
    const int64_t row = tile * kTileRows + rl;
    const bool live = row < n;
    double sum = 0.0;
    if (val) {
      const double* vt = reinterpret_cast<const double*>(st + L.val) + rl;
#pragma unroll
      for (int q = 0; q < ND; ++q) sum += vt[q * kTileRows] * xc[q];
    } else {
      sum = xc[0];
    }
    sum *= xs;
    if (live && z) z[row] = sum;
    const double zt = live ? sum * sscale : 0.0;
    const uint2 bb = *reinterpret_cast<const uint2*>(st + L.bin + rl * 8);
    const uint32_t sg = st[L.sgn + rl];
    if (!slow) {
      // slot q: the warp's live lanes hit distinct bins (sketch.cu colours
      // the slots), so a plain read-add-write is race-free; rows past n add
      // to the trash bin d. Adding a zero z changes no bin (the reference
      // skips zero entries, sketch.cpp:53-54).
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t b = live ? ((q < 4 ? bb.x : bb.y) >> (8 * (q & 3))) & 0xffu : uint32_t(d);
        accw[b] += ((sg >> q) & 1u) ? -zt : zt;
        __syncwarp();  // slot q's stores land before slot q+1's loads
      }
    } else if (zt != 0.0) {  // warp tile without a colouring: CAS atomics
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t b = ((q < 4 ? bb.x : bb.y) >> (8 * (q & 3))) & 0xffu;
        atomicAdd(accw + b, ((sg >> q) & 1u) ? -zt : zt);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == nstages) {
      s = 0;
      ph ^= 1u;
    }
  };
  double xa[ND], xb[ND];
  int64_t tile = blockIdx.x;
  if (tile < num_tiles) load_x(tile, xa);
  for (; tile < num_tiles; tile += 2 * int64_t(gridDim.x)) {
    step_tile(tile, xa, xb);
    const int64_t t2 = tile + gridDim.x;
    if (t2 < num_tiles) step_tile(t2, xb, xa);
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kTileRows) : "memory");  // all warps' atomics done
  for (int b = t; b < d; b += kTileRows) {
    const double v = acc[b] + acc[dpad + b] + acc[2 * dpad + b] + acc[3 * dpad + b];
    atomicAdd(pacc + b, v);
  }
}

size_t rs_smem(int nd, int d, int stages) {
  return size_t(stages) * rs_layout(nd).stride + sizeof(double) * 4 * size_t((d + 2) / 2 * 2);
}

int sms_rs() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

template <int ND>
bool launch_rs_t(const CsrView* A, const SketchView* S, const double* x, const double* xscale_dev,
                 double* z, double* pacc, const int32_t* stop, int step, cudaStream_t st) {
  auto fn = spmv_rowsketch_kernel<ND>;
  const int nd = A->dval ? ND : 0;
  // the most resident blocks, then the most stages with >= 3 (cached per shape)
  static thread_local int64_t keys[4] = {-1, -1, -1, -1};
  static thread_local int bests[4][2];
  static thread_local int next_slot = 0;
  const int64_t key = (int64_t(nd) << 32) ^ S->d;
  int slot = -1;
  for (int i = 0; i < 4; ++i)
    if (keys[i] == key) slot = i;
  if (slot < 0) {
    int best_s = 0, best_per = 0;
    static const int env_s = [] { const char* e = getenv("RKMF_RS_STAGES"); return e ? atoi(e) : 0; }();
    for (int s = 3; s <= kRsStages; ++s) {
      if (env_s && s != env_s) continue;
      const size_t sm = rs_smem(nd, int(S->d), s);
      if (sm > 200 * 1024) continue;
      RKMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      int per = 0;
      RKMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kRsThreads, sm));
      if (per > best_per || (per == best_per && per > 0)) {
        best_per = per;
        best_s = s;
      }
    }
    if (getenv("RKMF_PIPE_VERBOSE"))
      fprintf(stderr, "[rkmf] K2 row-sketch ND=%d: stages=%d blocks/SM=%d stride=%u\n", nd, best_s,
              best_per, rs_layout(nd).stride);
    slot = next_slot;
    next_slot = (next_slot + 1) & 3;
    keys[slot] = key;
    bests[slot][0] = best_s;
    bests[slot][1] = best_per;
  }
  const int stages = bests[slot][0], per_sm = bests[slot][1];
  if (stages == 0 || per_sm == 0) return false;
  const size_t smem = rs_smem(nd, int(S->d), stages);
  RKMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t tiles = (A->n_rows + kTileRows - 1) / kTileRows;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(per_sm) * sms_rs())));
  launch_maybe_pdl(fn, dim3(grid), dim3(kRsThreads), smem, st, A->n_rows, A->dval, x, xscale_dev,
                   z, tiles, int(S->d), S->rbin, S->sbit, S->wslow, S->scale, pacc, stop, step,
                   stages,
                   A->doff, A->n_cols, A->dstride, 1);
  return true;
}

}  // namespace

// Diagonal-copy matrices (A->dval, <= 8 diagonals) or A->dval == nullptr with
// ndiag 1 (the identity: the sketch of x alone), and a sketch with the
// row-major copy. Returns false when not applicable.
bool launch_spmv_rowsketch(const CsrView* A, const SketchView* S, const double* x,
                           const double* xscale_dev, double* z, double* pacc,
                           const int32_t* stop_flag, int step, cudaStream_t st) {
  if (!S || !S->rbin || !S->sbit || !S->wslow || S->zeta != 8 || S->d > 255) return false;
  if (A->ndiag < 1 || A->ndiag > kMaxDiag) return false;
#define RKMF_RS(NDV) \
  case NDV: return launch_rs_t<NDV>(A, S, x, xscale_dev, z, pacc, stop_flag, step, st)
  switch (A->ndiag) {
    RKMF_RS(1); RKMF_RS(2); RKMF_RS(3); RKMF_RS(4);
    RKMF_RS(5); RKMF_RS(6); RKMF_RS(7); RKMF_RS(8);
    default: break;
  }
#undef RKMF_RS
  return false;
}

}  // namespace rkmf_b200
