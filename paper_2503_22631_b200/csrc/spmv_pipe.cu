// K2 (pipelined): fused CSR SpMV + sparse-sign sketch, warp-specialised and
// fed by TMA bulk copies through an S-stage shared-memory ring.
//
// Why: the plain CSR-stream kernel (spmv.cu) is latency-bound on B200 — ncu
// shows long-scoreboard stalls dominating at ~26% of HBM bandwidth, because
// every 128-row tile pays row_ptr -> (val, col) -> x dependent round trips
// in sequence. Here one producer lane per block streams each tile's row
// pointers, values, column indices and sketch metadata with
// cp.async.bulk (TMA, UBLKCP in SASS) into stage s, arriving on an mbarrier
// with the transaction byte count, S tiles ahead of the consumers. The four
// consumer warps only gather x (L2-resident) and reduce rows in the
// reference's column order, then run the same deterministic bin gather for the
// sketch as spmv.cu. Stages are released through a second mbarrier.
//
// Alignment: bulk copies need 16-byte aligned addresses and sizes, so each
// copy starts at the aligned address at or below the tile's first nonzero and
// the consumers index with the recorded shift. Arrays are allocated with
// >= 16 bytes of tail padding (engine.cu) so the rounded-up copies stay in
// bounds.
#include <cuda_runtime.h>

#include <cstdlib>

#include "rkmf_internal.cuh"
#include "tma.cuh"

namespace rkmf_b200 {

namespace {

constexpr int kConsumers = 128;  // = kTileRows, one row per consumer thread
constexpr int kPipeThreads = kConsumers + 32;
constexpr int kStages = 4;
__device__ __forceinline__ void named_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

struct StageLayout {
  uint32_t rp, val, col, off, ent, zs, meta, stride;
};

__host__ __device__ inline StageLayout stage_layout(int rp_bytes, int cap, int off_stride,
                                                    int zeta) {
  auto r16 = [](uint32_t x) { return (x + 15u) & ~15u; };
  StageLayout L;
  uint32_t o = 0;
  L.rp = o;
  o += r16(uint32_t(rp_bytes) * 136u);
  L.val = o;
  o += r16(uint32_t(cap + 2) * 8u);
  L.col = o;
  o += r16(uint32_t(cap + 4) * 4u);
  L.off = o;
  o += r16(uint32_t(off_stride) * 2u);
  L.ent = o;
  o += r16(uint32_t(kTileRows * zeta));
  L.zs = o;  // zs2: +z then -z of the tile's rows (sketch_tile_gather)
  o += 2 * kTileRows * 8u;
  L.meta = o;
  o += 16u;
  L.stride = (o + 127u) & ~127u;
  return L;
}

struct TileMeta {
  long long rs;
  int vshift, cshift;
};

template <typename RP>
__global__ void __launch_bounds__(kPipeThreads)
    spmv_sketch_pipe_kernel(int64_t n, const RP* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ val, const double* __restrict__ x,
                            const double* xscale, double* __restrict__ z, int64_t num_tiles,
                            int cap, int d, int zeta, int off_stride,
                            const uint16_t* __restrict__ toff, const uint8_t* __restrict__ tent,
                            double sscale, double* pacc, const int32_t* stop, int step,
                            int nstages, int l2_hints, int debug) {
  extern __shared__ __align__(128) unsigned char smem[];
  const StageLayout L = stage_layout(int(sizeof(RP)), cap, off_stride, zeta);
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  double* acc = reinterpret_cast<double*>(smem + nstages * L.stride);  // [d]
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int b = t; b < d; b += kPipeThreads) acc[b] = 0.0;
  __syncthreads();
  pdl_wait_then_trigger();  // x, pacc and the stop flag come from earlier kernels
  if (stop != nullptr && *stop <= step) return;  // breakdown earlier in this cycle

  if (t >= kConsumers) {  // ---------------- producer warp ----------------
    if (t != kConsumers) return;
    const uint64_t pol = l2_policy(l2_hints >= 1 ? 1 : 0);
    // the sketch tile layout is re-read every step: ask L2 to keep it
    const uint64_t mpol = l2_policy(l2_hints);
    int it = 0;
    // row-pointer pair of the next tile, prefetched one iteration ahead so the
    // bulk copies of a tile are issued without a dependent global round trip
    long long nrs = 0, nre = 0;
    if (blockIdx.x < num_tiles) {
      const int64_t r0 = int64_t(blockIdx.x) * kTileRows;
      nrs = (long long)rp[r0];
      nre = (long long)rp[min(n, r0 + kTileRows)];
    }
    int s = 0;
    uint32_t eph = 0;  // parity of the empty barrier round being waited for
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const long long rs = nrs, re = nre;
      const int64_t nt = tile + gridDim.x;
      if (nt < num_tiles) {
        nrs = (long long)rp[nt * kTileRows];
        nre = (long long)rp[min(n, nt * kTileRows + kTileRows)];
      }
      if (it >= nstages) mbar_wait(&empty[s], eph);
      unsigned char* st = smem + s * L.stride;
      const int64_t r0 = tile * kTileRows;
      const long long vs0 = rs & ~1LL, cs0 = rs & ~3LL;
      const uint32_t vbytes = uint32_t(((re - vs0) * 8 + 15) & ~15LL);
      const uint32_t cbytes = uint32_t(((re - cs0) * 4 + 15) & ~15LL);
      const uint32_t rbytes = sizeof(RP) == 4 ? 528u : 1040u;
      const uint32_t obytes = uint32_t(off_stride) * 2u;
      const uint32_t ebytes = uint32_t(kTileRows * zeta);
      TileMeta* meta = reinterpret_cast<TileMeta*>(st + L.meta);
      meta->rs = rs;
      meta->vshift = int(rs - vs0);
      meta->cshift = int(rs - cs0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&full[s], rbytes + (re > rs ? vbytes + cbytes : 0u) + obytes + ebytes);
      bulk_g2s(st + L.rp, rp + r0, rbytes, &full[s], pol);
      if (re > rs) {
        bulk_g2s(st + L.val, val + vs0, vbytes, &full[s], pol);
        bulk_g2s(st + L.col, ci + cs0, cbytes, &full[s], pol);
      }
      bulk_g2s(st + L.off, toff + tile * off_stride, obytes, &full[s], mpol);
      bulk_g2s(st + L.ent, tent + tile * int64_t(kTileRows) * zeta, ebytes, &full[s], mpol);
      if (++s == nstages) {
        s = 0;
        if (it >= nstages) eph ^= 1u;  // rounds 1, 2, ... of each stage
      }
    }
    return;
  }

  // ---------------- consumer warps: one row per thread ----------------
  // Software-pipelined by one tile: the x gathers of tile i are issued, then
  // the sketch gather of tile i-1 runs from shared memory while they are in
  // flight, then tile i's row sums finish. The consumers therefore hold two
  // stages (i-1 until its sketch is gathered, and i).
  const double xs = xscale ? *xscale : 1.0;
  int s = 0, ps = -1;  // current stage; stage of the tile whose sketch is pending
  uint32_t fph = 0;    // parity of the full barrier round being waited for
  auto gather_prev = [&] {
    if (ps < 0) return;
    unsigned char* pst = smem + ps * L.stride;
    if (!(debug & 1))
      sketch_tile_gather(t, d, reinterpret_cast<const uint16_t*>(pst + L.off), pst + L.ent,
                         reinterpret_cast<const double*>(pst + L.zs), acc);
    mbar_arrive(&empty[ps]);
  };
  for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
    mbar_wait(&full[s], fph);
    unsigned char* st = smem + s * L.stride;
    if (debug & 4) {  // ablation: stream only
      mbar_arrive(&empty[s]);
      if (++s == nstages) { s = 0; fph ^= 1u; }
      continue;
    }
    const RP* rps = reinterpret_cast<const RP*>(st + L.rp);
    double* zs = reinterpret_cast<double*>(st + L.zs);
    const TileMeta meta = *reinterpret_cast<const TileMeta*>(st + L.meta);
    const double* vals = reinterpret_cast<const double*>(st + L.val) + meta.vshift;
    const int32_t* cols = reinterpret_cast<const int32_t*>(st + L.col) + meta.cshift;
    const int64_t row = tile * kTileRows + t;
    const bool live = row < n;
    int lo = 0, hi = 0;
    if (live) {
      lo = int((long long)rps[t] - meta.rs);
      hi = int((long long)rps[t + 1] - meta.rs);
    }
    // first 8 nonzeros: gathers in flight across the previous tile's sketch.
    // Lanes past the row end re-read the row's last column (a valid index the
    // row already uses) and contribute a zero product.
    double v[8], xv[8];
    if (lo < hi) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int ee = min(lo + q, hi - 1);
        v[q] = vals[ee];
        xv[q] = (debug & 2) ? double(cols[ee]) : __ldg(x + cols[ee]);
      }
    }
    gather_prev();
    double sum = 0.0;
    if (lo < hi) {
#pragma unroll
      for (int q = 0; q < 8; ++q) sum += (lo + q < hi ? v[q] : 0.0) * xv[q];
      for (int e = lo + 8; e < hi; e += 8) {  // long rows (27-point stencils)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int ee = min(e + q, hi - 1);
          v[q] = vals[ee];
          xv[q] = (debug & 2) ? double(cols[ee]) : __ldg(x + cols[ee]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) sum += (e + q < hi ? v[q] : 0.0) * xv[q];
      }
    }
    sum *= xs;
    if (live) z[row] = sum;
    const double zt = live ? sum * sscale : 0.0;
    zs[t] = zt;
    zs[kConsumers + t] = -zt;
    named_sync();  // zs2 of this tile complete; orders acc updates across threads
    ps = s;
    if (++s == nstages) {
      s = 0;
      fph ^= 1u;
    }
  }
  gather_prev();
  named_sync();  // acc[b] may have been written by another consumer thread
  for (int b = t; b < d; b += kConsumers) atomicAdd(pacc + b, acc[b]);
}

template <typename RP>
size_t pipe_smem(int cap, int d, int off_stride, int zeta, int stages) {
  const StageLayout L = stage_layout(int(sizeof(RP)), cap, off_stride, zeta);
  return size_t(stages) * L.stride + sizeof(double) * size_t((d + 1) / 2 * 2);
}

// RKMF_L2_HINTS: 0 no L2 hints, 1 evict_first on the matrix and sketch
// streams, 2 (default) evict_first on the matrix and evict_last on the sketch
// tile layout, which every step re-reads.
int env_l2_hints() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RKMF_L2_HINTS");
    v = e ? atoi(e) : 2;
    if (v < 0 || v > 2) v = 2;
  }
  return v;
}

int env_debug() {  // RKMF_PIPE_DEBUG: ablation bits (1 no sketch, 2 no x gather, 4 stream only)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RKMF_PIPE_DEBUG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

int env_stages() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RKMF_PIPE_STAGES");
    v = e ? atoi(e) : 0;
    if (v < 0 || v > kStages) v = 0;
  }
  return v;
}

int sms() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

template <typename RP>
bool launch_pipe_t(const CsrView* A, const SketchView* S, const double* x,
                   const double* xscale_dev, double* z, double* pacc, const int32_t* stop,
                   int step, cudaStream_t st) {
  const int off_stride = int(tile_off_stride(S->d));
  auto fn = spmv_sketch_pipe_kernel<RP>;
  // Pick the stage count that maximises consumer warps per SM while keeping
  // at least one tile in flight ahead of the consumers (cached per shape).
  static thread_local int64_t key_c = -1;
  static thread_local int best_s = 0, best_per = 0;
  const int64_t key = (int64_t(A->cap) << 40) ^ (S->d << 20) ^ (S->zeta << 8) ^ sizeof(RP);
  if (key != key_c) {
    best_s = 0;
    best_per = 0;
    for (int s = 3; s <= kStages; ++s) {  // consumers hold 2 stages (pipelined)
      if (env_stages() && s != env_stages()) continue;
      const size_t sm = pipe_smem<RP>(A->cap, int(S->d), off_stride, int(S->zeta), s);
      if (sm > 220 * 1024) continue;
      RKMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      int per = 0;
      RKMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kPipeThreads, sm));
      // prefer more resident blocks; on a tie, more stages
      if (per > 0 && (per > best_per || (per == best_per && s > best_s))) {
        best_per = per;
        best_s = s;
      }
    }
    key_c = key;
  }
  if (best_s == 0) return false;
  const int stages = best_s, per_sm = best_per;
  const size_t smem = pipe_smem<RP>(A->cap, int(S->d), off_stride, int(S->zeta), stages);
  RKMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t tiles = (A->n_rows + kTileRows - 1) / kTileRows;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(per_sm) * sms())));
  launch_maybe_pdl(fn, dim3(grid), dim3(kPipeThreads), smem, st, A->n_rows,
                   static_cast<const RP*>(A->row_ptr), A->col, A->val, x, xscale_dev, z, tiles,
                   A->cap, int(S->d), int(S->zeta), off_stride, S->tile_off, S->tile_ent,
                   S->scale, pacc, stop, step, stages, env_l2_hints(), env_debug());
  return true;
}

}  // namespace

bool launch_spmv_sketch_pipe(const CsrView* A, const SketchView* S, const double* x,
                             const double* xscale_dev, double* z, double* pacc,
                             const int32_t* stop_flag, int step, cudaStream_t st) {
  if (!A->padded || A->max_tile_nnz > A->cap || A->cap > 4096) return false;
  return A->rp64 ? launch_pipe_t<int64_t>(A, S, x, xscale_dev, z, pacc, stop_flag, step, st)
                 : launch_pipe_t<int32_t>(A, S, x, xscale_dev, z, pacc, stop_flag, step, st);
}

}  // namespace rkmf_b200
