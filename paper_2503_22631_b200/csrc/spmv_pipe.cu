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

#include <cstdio>
#include <cstdlib>

#include "rkmf_internal.cuh"
#include "detred.cuh"
#include "tma.cuh"

namespace rkmf_b200 {

namespace {


constexpr int kStages = 8;
// diagonal kernels: block b takes chunks of RKMF_K2_CHUNK consecutive tiles,
// chunk b, b + grid, ... (1 = plain round robin)
#ifndef RKMF_K2_CHUNK
#define RKMF_K2_CHUNK 1
#endif
// doubles per row-dictionary tuple in shared memory (ND rounded up to even)
template <int ND>
constexpr int kDictStride = (ND + 1) / 2 * 2;
// A row dictionary of at most kDictParam doubles travels in the kernel's
// parameter space (__grid_constant__: read through the constant cache, one
// access per warp when its rows share a tuple) instead of shared memory,
// whose 16-byte loads cost the load/store pipe about 13% of its wavefronts.
constexpr int kDictParam = 224;
struct DictParam {
  double v[kDictParam];
};


struct StageLayout {
  uint32_t rp, val, col, off, ent, zs, meta, stride;
};

// FMT 0 (CSR): row pointers, up to cap values and columns (+ alignment slack);
// FMT 2 (DIA): cap = ndiag * 128 values, no row pointers or columns.
__host__ __device__ inline StageLayout stage_layout(int rp_bytes, int cap, int off_stride,
                                                    int ent_bytes, int fmt) {
  auto r16 = [](uint32_t x) { return (x + 15u) & ~15u; };
  StageLayout L;
  uint32_t o = 0;
  L.rp = o;
  o += fmt ? 0u : r16(uint32_t(rp_bytes) * 136u);
  L.val = o;
  o += fmt ? uint32_t(cap) * 8u : r16(uint32_t(cap + 2) * 8u);
  L.col = o;
  o += fmt ? 0u : r16(uint32_t(cap + 4) * 4u);
  L.off = o;
  o += r16(uint32_t(off_stride) * 2u);
  L.ent = o;
  o += r16(uint32_t(ent_bytes));
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

// Thread roles of one block (warp-specialised):
//   [0, G*128*TPR)        SpMV threads: G groups, group g takes the block's
//                         tiles it = g, g+G, ...; TPR threads per row
//   next kSketchThreads   sketch threads: every tile in order, from shared memory
//   last warp             producer: one elected lane issues the bulk copies
// Per stage s (ring of NS >= G + 2): full[s] (producer tx bytes) -> the SpMV
// group writes z and the signed z table into the stage and arrives on zsr[s]
// -> the sketch threads gather the tile's bins and arrive on empty[s] -> the
// producer refills. The SpMV groups never wait for the sketch, so G tiles'
// x gathers are in flight per block while the sketch of an older tile runs.
constexpr int kSketchThreads = 128;

template <int TPR, int G>
constexpr int spmv_threads() { return G * kTileRows * TPR; }
template <int TPR, int G>
constexpr int block_threads() { return spmv_threads<TPR, G>() + kSketchThreads + 32; }

// FMT 2 streams a diagonal (DIA) copy of the matrix instead of the CSR arrays
// (build_dia, dia.cu): val = [tile][diag][128] values, doff = [tile][8] sorted
// column offsets (ndiag <= 8 used); x is read at row + off (coalesced)
// one tile ahead of the stage it multiplies. (FMT 1 was the same without the
// x prefetch; at 27 diagonals either DIA variant loses to the CSR kernel with
// two threads per row, 875 vs 465 us on cfg3, so the copy is limited to 8.)
// (a 4-blocks-per-SM register cap, 56 registers with spills, measured slower)
#define RKMF_PIPE_PARAMS                                                                       \
  int64_t n, const RP *__restrict__ rp, const int32_t *__restrict__ ci,                        \
      const double *__restrict__ val, const double *__restrict__ x, const double *xscale,      \
      double *__restrict__ z, int64_t num_tiles, int cap, int d, int ent_stride, int off_stride,     \
      const uint16_t *__restrict__ toff, const uint8_t *__restrict__ tent, double sscale,      \
      const int32_t *stop, int step, int nstages, int l2_hints_arg, int debug_arg,        \
      const int32_t *__restrict__ doff, int ndiag, int64_t ncols, int sync_mode_arg, int dstride,   \
      const double *__restrict__ ddict, int ntup, const int32_t *__restrict__ rcnt,              \
      const int32_t *__restrict__ roff, const double *__restrict__ rval, int rntup, DetRed red
#define RKMF_PIPE_ARGS                                                                       \
  n, rp, ci, val, x, xscale, z, num_tiles, cap, d, ent_stride, off_stride, toff, tent, sscale, \
      stop, step, nstages, l2_hints_arg, debug_arg, doff, ndiag, ncols, sync_mode_arg, dstride, ddict, \
      ntup, rcnt, roff, rval, rntup, red

// The ablation knobs (RKMF_PIPE_DEBUG / _SYNC / RKMF_L2_HINTS) reach the
// kernel only in the experiments build; the product build folds them to
// their defaults at compile time (fewer instructions in an issue-bound kernel).
#ifdef RKMF_EXPERIMENTS
#define RKMF_KNOB(arg, def) (arg)
#else
#define RKMF_KNOB(arg, def) (def)
#endif

template <typename RP, int TPR, int G, int FMT, int ND>
__device__ __forceinline__ void pipe_body(RKMF_PIPE_PARAMS, const DictParam& dpar) {
  const int debug = RKMF_KNOB(debug_arg, 0);
  const int sync_mode = RKMF_KNOB(sync_mode_arg, 1);
  const int l2_hints = RKMF_KNOB(l2_hints_arg, 1);
  constexpr int kSpmv = spmv_threads<TPR, G>();
  constexpr int kGroup = kTileRows * TPR;
  extern __shared__ __align__(128) unsigned char smem[];
  const int ent_bytes = ent_stride;
  const StageLayout L = stage_layout(int(sizeof(RP)), cap, off_stride, ent_bytes, FMT);
  __shared__ __align__(8) uint64_t full[kStages], zsr[kStages], empty[kStages];
  // shared-space addresses, converted once (not per barrier call)
  const uint32_t full_u = su32(full), zsr_u = su32(zsr), empty_u = su32(empty);
  const uint32_t smem_u = su32(smem);
  __shared__ int32_t doff_s[kMaxDiag];  // FMT 2 with one offset list (dstride 0)
  if (FMT && threadIdx.x < kMaxDiag) doff_s[threadIdx.x] = doff ? doff[threadIdx.x] : 0;
  double* acc = reinterpret_cast<double*>(smem + nstages * L.stride);  // [d], sketch threads
  // FMT 3: the row dictionary [ntup][ND] after acc (constant: loaded before
  // the PDL wait)
  double* dict_s = acc + (d + 1) / 2 * 2;
  const int t = threadIdx.x;
  const bool dict_par = ntup * ND <= kDictParam;
  // FMT 4: the CSR row dictionary [rntup][kRdMaxNnz] values, then offsets and
  // counts, after acc (constant: loaded before the PDL wait)
  double* rd_val_s = dict_s;
  int32_t* rd_off_s = reinterpret_cast<int32_t*>(rd_val_s + rntup * kRdMaxNnz);
  int32_t* rd_cnt_s = rd_off_s + rntup * kRdMaxNnz;
  if constexpr (FMT == 4) {
    for (int i = t; i < rntup * kRdMaxNnz; i += block_threads<TPR, G>()) {
      rd_val_s[i] = rval[i];
      rd_off_s[i] = roff[i];
    }
    for (int i = t; i < rntup; i += block_threads<TPR, G>()) rd_cnt_s[i] = rcnt[i];
  }
  // this block's k-th tile and tile count (chunks of CH consecutive tiles)
  constexpr int64_t CH = FMT ? RKMF_K2_CHUNK : 1;
  auto tile_of = [&](int64_t k) -> int64_t {
    return (int64_t(blockIdx.x) + (k / CH) * int64_t(gridDim.x)) * CH + k % CH;
  };
  int64_t tcount;
  {
    const int64_t nsup = (num_tiles + CH - 1) / CH, b = blockIdx.x;
    const int64_t ns = nsup > b ? (nsup - b + gridDim.x - 1) / gridDim.x : 0;
    tcount = ns * CH;
    if (ns > 0) tcount -= max(int64_t(0), (b + (ns - 1) * int64_t(gridDim.x)) * CH + CH - num_tiles);
  }
  if constexpr (FMT == 3)
    if (!dict_par)
    for (int i = t; i < ntup * kDictStride<ND>; i += block_threads<TPR, G>()) {
      const int tup = i / kDictStride<ND>, q = i % kDictStride<ND>;
      dict_s[i] = q < ND ? ddict[tup * ND + q] : 0.0;
    }
  if (t == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&zsr[s], kGroup);
      mbar_init(&empty[s], (sync_mode & 1) ? 1 : kSketchThreads);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int b = t; b < d; b += block_threads<TPR, G>()) acc[b] = 0.0;
  __syncthreads();
  // The matrix and the sketch layout are constant, so the producer fills the
  // first nstages stages before waiting on the previous kernel (PDL: that
  // overlaps the basis update's tail); x and the stop flag come from
  // earlier kernels, so every other thread waits first.
  const bool producer = t == kSpmv + kSketchThreads;
  if (t == 0 && stop) trace_first(step, 10);
  if (!producer) {
    pdl_wait_then_trigger();
    if (t == 0 && stop) trace_first(step, 0);
    if (stop != nullptr && *stop <= step) return;  // breakdown earlier in this cycle
  }

  if (t >= kSpmv + kSketchThreads) {  // ---------------- producer warp ----------------
    if (!producer) return;
    bool waited = false;
    // after the early stages: wait for the previous kernel; if this step is
    // past a breakdown, let the issued copies land (the block's shared
    // memory must not be released under them) and leave
    auto wait_prev = [&](int issued) {
      waited = true;
      asm volatile("griddepcontrol.wait;" ::: "memory");
      if (stop != nullptr && *stop <= step) {
        for (int i = 0; i < issued; ++i) mbar_wait_u(full_u + 8u * (i), 0u);
        return true;
      }
      return false;
    };
    if ((debug & 16) && wait_prev(0)) return;  // ablation: no early stage fill
    const uint64_t pol = l2_policy(l2_hints >= 1 ? 1 : 0);
    // the sketch tile layout's policy (RKMF_L2_HINTS, env_l2_hints)
    const uint64_t mpol = l2_policy(l2_hints);
    // row-pointer pair of the next tile, prefetched one iteration ahead so the
    // bulk copies of a tile are issued without a dependent global round trip
    long long nrs = 0, nre = 0;
    if (!FMT && blockIdx.x < num_tiles) {
      const int64_t r0 = int64_t(blockIdx.x) * kTileRows;
      nrs = (long long)rp[r0];
      nre = (long long)rp[min(n, r0 + kTileRows)];
    }
    int s = 0, it = 0;
    uint32_t eph = 0;  // parity of the empty barrier round being waited for
    for (; it < tcount; ++it) {
      const int64_t tile = tile_of(it);
      const long long rs = nrs, re = nre;
      const int64_t nt = tile + gridDim.x;
      if (!FMT && nt < num_tiles) {
        nrs = (long long)rp[nt * kTileRows];
        nre = (long long)rp[min(n, nt * kTileRows + kTileRows)];
      }
      if (it == nstages && !waited && wait_prev(it)) return;
      if (it >= nstages) mbar_wait_u(empty_u + 8u * (s), eph);
      unsigned char* st = smem + s * L.stride;
      const uint32_t st_u = smem_u + uint32_t(s) * L.stride;
      const int64_t r0 = tile * kTileRows;
      const long long vs0 = rs & ~1LL, cs0 = rs & ~3LL;
      const uint32_t vbytes = uint32_t(((re - vs0) * 8 + 15) & ~15LL);
      const uint32_t cbytes = uint32_t(((re - cs0) * 4 + 15) & ~15LL);
      const uint32_t rbytes = sizeof(RP) == 4 ? 528u : 1040u;
      const uint32_t obytes = uint32_t(off_stride) * 2u;
      const uint32_t ebytes = uint32_t(ent_bytes);
      if (FMT) {  // one contiguous block of ndiag x 128 values
        const uint32_t dbytes = val ? uint32_t(cap) * 8u : 0u;
        mbar_expect_tx_u(full_u + 8u * s, dbytes + obytes + ebytes);
        if (val) bulk_g2s_u(st_u + L.val, val + tile * int64_t(cap), dbytes, full_u + 8u * s, pol);
        bulk_g2s_u(st_u + L.off, toff + tile * off_stride, obytes, full_u + 8u * s, mpol);
        bulk_g2s_u(st_u + L.ent, tent + tile * int64_t(ent_bytes), ebytes, full_u + 8u * s, mpol);
        if (++s == nstages) {
          s = 0;
          if (it >= nstages) eph ^= 1u;
        }
        continue;
      }
      TileMeta* meta = reinterpret_cast<TileMeta*>(st + L.meta);
      meta->rs = rs;
      meta->vshift = int(rs - vs0);
      meta->cshift = int(rs - cs0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx_u(full_u + 8u * s, rbytes + (re > rs ? vbytes + cbytes : 0u) + obytes + ebytes);
      bulk_g2s_u(st_u + L.rp, rp + r0, rbytes, full_u + 8u * s, pol);
      if (re > rs) {
        bulk_g2s_u(st_u + L.val, val + vs0, vbytes, full_u + 8u * s, pol);
        bulk_g2s_u(st_u + L.col, ci + cs0, cbytes, full_u + 8u * s, pol);
      }
      bulk_g2s_u(st_u + L.off, toff + tile * off_stride, obytes, full_u + 8u * s, mpol);
      bulk_g2s_u(st_u + L.ent, tent + tile * int64_t(ent_bytes), ebytes, full_u + 8u * s, mpol);
      if (++s == nstages) {
        s = 0;
        if (it >= nstages) eph ^= 1u;  // rounds 1, 2, ... of each stage
      }
    }
    if (!waited) wait_prev(it);
    return;
  }

  if (t >= kSpmv) {  // ---------------- sketch threads ----------------
    const int u = t - kSpmv;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t k = 0; k < tcount; ++k) {
      if (sync_mode & 1) {
        // named barrier 8 + s (the SpMV group bar.arrives on it): a hardware
        // barrier, so the waiting sketch warps take no issue slots
        asm volatile("bar.sync %0, %1;" ::"r"(8 + s), "n"(kGroup + kSketchThreads) : "memory");
      } else {
        mbar_wait_u(zsr_u + 8u * (s), ph);
        mbar_wait_u(full_u + 8u * (s), ph);  // completed already (the SpMV group waited on it)
      }
      unsigned char* st = smem + s * L.stride;
      if (!(debug & 1))
        sketch_tile_gather(u, d, reinterpret_cast<const uint16_t*>(st + L.off),
                                           st + L.ent,
                                           reinterpret_cast<const double*>(st + L.zs), acc);
      // orders this tile's acc updates before the next tile's (slot -> bin
      // ownership changes per tile)
      asm volatile("bar.sync 2, %0;" ::"n"(kSketchThreads) : "memory");
      if (!(sync_mode & 1) || u == 0) mbar_arrive_u(empty_u + 8u * (s));
      if (++s == nstages) {
        s = 0;
        ph ^= 1u;
      }
    }
    // the block's d partials -> its group's partial, summed in a fixed block
    // order (detred.cuh; K3 sums the groups). The last tile's bar.sync 2
    // above completed acc.
    __shared__ int rflag;
    if (!(debug & 8)) det_group_reduce<kSketchThreads, 2, 16>(red, d, acc, u, &rflag);
    if (u == 0 && stop) trace_max(step, 1);
    return;
  }

  // ---------------- SpMV threads: group g, TPR threads per row ----------------
  // Adjacent lanes of a row take its nonzeros round-robin and combine their
  // partial sums with a fixed butterfly (deterministic). 8 gathers per thread
  // are in flight before the first FMA; lanes past the row end re-read the
  // row's last column (a valid index the row already uses) and contribute a
  // zero product.
  const double xs = xscale ? *xscale : 1.0;
  const int g = t / kGroup, gt = t % kGroup;
  const int rl = gt / TPR, part = gt % TPR;
  // stage s and its full-barrier parity advance incrementally (G < nstages)
  int s = g;
  uint32_t ph = 0;
  auto advance = [&] {
    s += G;
    if (s >= nstages) {
      s -= nstages;
      ph ^= 1u;
    }
  };
  auto handoff = [&] {  // z table of stage s complete -> the sketch threads
    if (sync_mode & 1)
      asm volatile("bar.arrive %0, %1;" ::"r"(8 + s), "n"(kGroup + kSketchThreads) : "memory");
    else
      mbar_arrive_u(zsr_u + 8u * (s));
  };
  if constexpr (FMT == 2 || FMT == 3) {
    // Diagonal copy, ND diagonals: x is read at row + offset. Those reads do
    // not depend on the staged values, so each thread loads the next tile's x
    // (into the other register buffer) before waiting for this tile's stage.
    // Row indices fit in 32 bits (build_dia), so the addressing is 32-bit;
    // with one offset list for all tiles (dstride 0) the offsets sit in
    // registers and the tiles whose reads are all in range (every tile but
    // the first and last few) are one index interval, tested per tile with
    // two compares.
    const int32_t n32 = int32_t(n), nc32 = int32_t(ncols), nt32 = int32_t(num_tiles);
    const bool single = dstride == 0;
    int offs[ND];
    int32_t tlo = 0, thi = 0;  // interior tiles [tlo, thi) (single list)
    if (single) {
#pragma unroll
      for (int q = 0; q < ND; ++q) offs[q] = doff ? doff_s[q] : 0;
      // tile t is interior when 128 t + offs[0] >= 0, 128 t + 127 + offs[ND-1] < ncols
      // and 128 t + 128 <= n
      tlo = offs[0] >= 0 ? 0 : (-offs[0] + kTileRows - 1) / kTileRows;
      const int64_t lim = min(int64_t(nc32) - kTileRows - int64_t(offs[ND - 1]),
                              int64_t(n32) - kTileRows);
      thi = lim < 0 ? 0 : int32_t(lim / kTileRows) + 1;
      thi = max(tlo, min(thi, nt32));
    }
    uint64_t zpol;  // z with an L2 evict_last hint: K4 reads it next
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(zpol));
    auto load_x = [&](int32_t tl, double* dst) {
      const int32_t row = tl * kTileRows + rl;
      if (single && tl >= tlo && tl < thi) {
        // row + offs[q] >= 0 here: one 32-bit add and one wide multiply-add
#pragma unroll
        for (int q = 0; q < ND; ++q) dst[q] = __ldg(x + uint32_t(row + offs[q]));
        return;
      }
      int o[ND];
      if (single) {
#pragma unroll
        for (int q = 0; q < ND; ++q) o[q] = offs[q];
      } else if (doff) {  // the tile's own sorted offsets ([tile][kMaxDiag])
        const int4* p = reinterpret_cast<const int4*>(doff + int64_t(tl) * kMaxDiag);
        const int4 a = __ldg(p), b = __ldg(p + 1);
        const int all[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int q = 0; q < ND; ++q) o[q] = all[q];
      } else {
#pragma unroll
        for (int q = 0; q < ND; ++q) o[q] = 0;
      }
#pragma unroll
      for (int q = 0; q < ND; ++q) {
        const int32_t c = row + o[q];
        dst[q] = (row < n32 && c >= 0 && c < nc32) ? __ldg(x + uint32_t(c)) : 0.0;
      }
    };
    // One register buffer: a tile's x is loaded right after the previous
    // tile's products consumed the buffer, so the loads are in flight while
    // the thread waits for the tile's stage (the same overlap as a double
    // buffer, half the registers: no spills at four blocks per SM).
    static_assert(G == 1 || RKMF_K2_CHUNK == 1, "chunked tile runs take one SpMV group");
    double xc[ND];
    int64_t kk = g;
    int32_t tile = kk < tcount ? int32_t(tile_of(kk)) : nt32;
    if (kk < tcount) load_x(tile, xc);
    for (; kk < tcount; kk += G, tile = kk < tcount ? int32_t(tile_of(kk)) : nt32) {
      mbar_wait_u(full_u + 8u * (s), ph);
      const unsigned char* st = smem + s * L.stride;
      if (!(debug & 4)) {
        const int32_t row = tile * kTileRows + rl;
        const bool live = row < n32;
        double sum = 0.0;
        if constexpr (FMT == 3) {
          // the row's tuple id (one streamed byte) -> its ND values in the
          // shared dictionary: the same values in the same order as FMT 2
          const int tid = int(st[L.val + rl]);
          if (dict_par) {
            const double* dv = dpar.v + tid * ND;
#pragma unroll
            for (int q = 0; q < ND; ++q) sum += dv[q] * xc[q];
          } else {
            // (tuples padded to an even count of doubles: 16-byte loads)
            const double2* dv = reinterpret_cast<const double2*>(dict_s + tid * kDictStride<ND>);
#pragma unroll
            for (int q = 0; q < ND; q += 2) {
              const double2 v = dv[q / 2];
              sum += v.x * xc[q];
              if (q + 1 < ND) sum += v.y * xc[q + 1];
            }
          }
        } else if (val) {
          const double* vt = reinterpret_cast<const double*>(st + L.val) + rl;
#pragma unroll
          for (int q = 0; q < ND; ++q) sum += vt[q * kTileRows] * xc[q];
        } else {  // identity: z = x
          sum = xc[0];
        }
        sum *= xs;
        if (live && z)
          asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(z + uint32_t(row)),
                       "d"(sum), "l"(zpol)
                       : "memory");
        const double zt = live ? sum * sscale : 0.0;
        double* zs = reinterpret_cast<double*>(const_cast<unsigned char*>(st) + L.zs);
        zs[rl] = zt;
        zs[kTileRows + rl] = -zt;
      }
      handoff();
      advance();
      if (kk + G < tcount) load_x(int32_t(tile_of(kk + G)), xc);
    }
    return;
  } else if constexpr (FMT == 4) {
  // CSR row dictionary: the row's form id (one streamed byte) -> its count,
  // offsets and values in shared memory (one broadcast per warp when its rows
  // share the form), walked as the CSR branch below walks the row's
  // nonzeros (column order; with TPR 1 sequentially).
  for (int64_t tile = blockIdx.x + int64_t(g) * gridDim.x; tile < num_tiles;
       tile += int64_t(G) * gridDim.x) {
    mbar_wait_u(full_u + 8u * (s), ph);
    unsigned char* st = smem + s * L.stride;
    if (!(debug & 4)) {
      double* zs = reinterpret_cast<double*>(st + L.zs);
      const int64_t row = tile * kTileRows + rl;
      const bool live = row < n;
      const int f = live ? int(st[L.val + rl]) : 0;
      const int hi = live ? rd_cnt_s[f] : 0;
      const double* vals = rd_val_s + f * kRdMaxNnz;
      const int32_t* offs = rd_off_s + f * kRdMaxNnz;
      const int32_t row32 = int32_t(row);
      double sum = 0.0;
      int e = part;
      for (; e + TPR * 7 < hi; e += 8 * TPR) {  // full batches: no clamps
        double v[8], xv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          v[q] = vals[e + TPR * q];
          xv[q] = __ldg(x + uint32_t(row32 + offs[e + TPR * q]));
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) sum += v[q] * xv[q];
      }
      if (e < hi) {  // the last partial batch
        double v[8], xv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int ee = min(e + TPR * q, hi - 1);
          v[q] = vals[ee];
          xv[q] = __ldg(x + uint32_t(row32 + offs[ee]));
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) sum += (e + TPR * q < hi ? v[q] : 0.0) * xv[q];
      }
#pragma unroll
      for (int o = 1; o < TPR; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      sum *= xs;
      if (part == 0) {
        if (live && z) z[row] = sum;
        const double zt = live ? sum * sscale : 0.0;
        zs[rl] = zt;
        zs[kTileRows + rl] = -zt;
      }
    }
    handoff();
    advance();
  }
  } else {
  // CSR: adjacent lanes of a row take its nonzeros round-robin and combine
  // their partial sums with a fixed butterfly (deterministic). 8 gathers per
  // thread are in flight before the first FMA; lanes past the row end re-read
  // the row's last column (a valid index the row already uses) and contribute
  // a zero product.
  for (int64_t tile = blockIdx.x + int64_t(g) * gridDim.x; tile < num_tiles;
       tile += int64_t(G) * gridDim.x) {
    mbar_wait_u(full_u + 8u * (s), ph);
    unsigned char* st = smem + s * L.stride;
    if (!(debug & 4)) {
      const RP* rps = reinterpret_cast<const RP*>(st + L.rp);
      double* zs = reinterpret_cast<double*>(st + L.zs);
      const TileMeta meta = *reinterpret_cast<const TileMeta*>(st + L.meta);
      const double* vals = reinterpret_cast<const double*>(st + L.val) + meta.vshift;
      const int32_t* cols = reinterpret_cast<const int32_t*>(st + L.col) + meta.cshift;
      const int64_t row = tile * kTileRows + rl;
      const bool live = row < n;
      int lo = 0, hi = 0;
      if (live) {
        lo = int((long long)rps[rl] - meta.rs);
        hi = int((long long)rps[rl + 1] - meta.rs);
      }
      double sum = 0.0;
      int e = lo + part;
      for (; e + TPR * 7 < hi; e += 8 * TPR) {  // full batches: no clamps
        double v[8], xv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          v[q] = vals[e + TPR * q];
          xv[q] = (debug & 2) ? double(cols[e + TPR * q]) : __ldg(x + cols[e + TPR * q]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) sum += v[q] * xv[q];
      }
      if (e < hi) {  // the last partial batch
        double v[8], xv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int ee = min(e + TPR * q, hi - 1);
          v[q] = vals[ee];
          xv[q] = (debug & 2) ? double(cols[ee]) : __ldg(x + cols[ee]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) sum += (e + TPR * q < hi ? v[q] : 0.0) * xv[q];
      }
#pragma unroll
      for (int o = 1; o < TPR; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      sum *= xs;
      if (part == 0) {
        if (live && z) z[row] = sum;  // (an evict_last hint here: cfg3 same, cfg5 3% slower)
        const double zt = live ? sum * sscale : 0.0;
        zs[rl] = zt;
        zs[kTileRows + rl] = -zt;
      }
    }
    handoff();
    advance();
  }
  }
}

// The diagonal kernel runs three or four 288-thread blocks per SM and is left
// to ptxas's register heuristics (it is sensitive to code generation). The CSR
// kernel runs one 544-672-thread block per SM (its stages fill shared
// memory): its own bounds (min one block) let it keep a thread's eight x
// gathers in flight; left to the heuristics, ptxas squeezed it to 40
// registers for a second block that never fits and interleaved the gathers
// with the FMA chain (cfg3 K2 502 vs 462 us).
// four resident blocks per SM (56 registers, no spills): cfg4 K2 246 vs 316 us
// at three blocks (70 registers), cfg2 41.5 vs 49.0 us (profiles/r02e_variants.txt)
#ifndef RKMF_K2_DIA_MINB
#define RKMF_K2_DIA_MINB 4
#endif
// SpMV groups of the diagonal-dictionary kernel (FMT 3)
#ifndef RKMF_K2_DICT_G
#define RKMF_K2_DICT_G 1
#endif
template <typename RP, int TPR, int G, int FMT, int ND = 1>
__global__ void __launch_bounds__(block_threads<TPR, G>(), RKMF_K2_DIA_MINB)
    spmv_sketch_pipe_kernel(RKMF_PIPE_PARAMS, const __grid_constant__ DictParam dpar) {
  pipe_body<RP, TPR, G, FMT, ND>(RKMF_PIPE_ARGS, dpar);
}
// The CSR row-dictionary kernel (FMT 4) is bound by its x gathers (27 per row
// on the Q1 matrices), so it runs one thread per row, two SpMV groups and two
// resident blocks per SM (70 registers): cfg5 K2 4.50 ms, vs 5.69 ms with the
// CSR kernel's two threads per row and one block, 5.28 ms with three groups
// and one block, 5.09 ms at three blocks of 48 registers
// (profiles/r02zg_rd_tuning.txt).
#ifndef RKMF_K2_RD_MINB
#define RKMF_K2_RD_MINB 2
#endif
#ifndef RKMF_K2_RD_TPR
#define RKMF_K2_RD_TPR 1
#endif
#ifndef RKMF_K2_RD_G
#define RKMF_K2_RD_G 2
#endif
template <typename RP, int TPR, int G, int FMT, int ND = 1>
__global__ void __launch_bounds__(block_threads<TPR, G>(), (FMT == 4 ? RKMF_K2_RD_MINB : 1))
    spmv_sketch_pipe_csr_kernel(RKMF_PIPE_PARAMS) {
  pipe_body<RP, TPR, G, FMT, ND>(RKMF_PIPE_ARGS, DictParam{});
}

template <typename RP>
size_t pipe_smem(int cap, int d, int off_stride, int ent_bytes, int stages, int fmt, int dict_len = 0) {
  const StageLayout L = stage_layout(int(sizeof(RP)), cap, off_stride, ent_bytes, fmt);
  return size_t(stages) * L.stride + sizeof(double) * size_t((d + 1) / 2 * 2 + dict_len);
}

// RKMF_L2_HINTS: 0 no L2 hints, 1 (default) evict_first on the matrix and
// sketch streams, 2 evict_first on the matrix and evict_last on the sketch
// tile layout (re-read every step). Keeping the layout in L2 helps K2 less than
// the L2 it takes from K4's streams costs: cfg2 solve 8590 vs 8540 vec/s
// (five alternating runs each) with 1.
int env_l2_hints() {
  static int v = -1;
  if (v < 0) {
    const char* e = knob_env("RKMF_L2_HINTS");
    v = e ? atoi(e) : 1;
    if (v < 0 || v > 2) v = 1;
  }
  return v;
}

int env_debug() {  // RKMF_PIPE_DEBUG: ablation bits (1 no sketch, 2 no x gather, 4 no SpMV, 8 no sketch flush, 16 producer waits before filling)
  static int v = -1;
  if (v < 0) {
    const char* e = knob_env("RKMF_PIPE_DEBUG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

// RKMF_PIPE_SYNC bits: 1 (default) the SpMV -> sketch handoff on named
// barriers 8 + s (bar.arrive / bar.sync: the sketch warps wait in hardware
// instead of polling an mbarrier, which takes issue slots in this
// issue-bound kernel) and one empty arrival per tile; 0 = mbarriers;
// 2 = also one warp per SpMV group polls the TMA barrier (slower)
int env_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = knob_env("RKMF_PIPE_SYNC");
    v = e ? atoi(e) : 1;
  }
  return v;
}

int env_stages() {
  static int v = -1;
  if (v < 0) {
    const char* e = knob_env("RKMF_PIPE_STAGES");
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

template <typename RP, int TPR, int G, int FMT = 0, int ND = 1>
bool launch_pipe_t(const CsrView* A, const SketchView* S, const double* x,
                   const double* xscale_dev, double* z, const int32_t* stop,
                   int step, DetRed& red, cudaStream_t st) {
  constexpr int kThreads = block_threads<TPR, G>();
  const int off_stride = int(tile_off_stride(S->d));
  auto fn = [] {
    if constexpr (FMT == 2 || FMT == 3) return spmv_sketch_pipe_kernel<RP, TPR, G, FMT, ND>;
    else return spmv_sketch_pipe_csr_kernel<RP, TPR, G, FMT, ND>;
  }();
  // FMT 3/4 stream one id byte per row: 128 bytes = 16 "values" per tile
  const int cap = FMT >= 3 ? kTileRows / 8 : FMT ? A->ndiag * kTileRows : A->cap;
  const bool dict_par = FMT == 3 && A->ntup * ND <= kDictParam;
  // after acc: the FMT 3 row dictionary (unless a kernel parameter), or the
  // FMT 4 CSR row dictionary (values, then int32 offsets and counts)
  const int dict_len =
      FMT == 3 ? (dict_par ? 0 : A->ntup * kDictStride<ND>)
               : FMT == 4 ? A->rntup * kRdMaxNnz + (A->rntup * kRdMaxNnz + A->rntup + 1) / 2 : 0;
  // Pick the stage count. G stages feed the SpMV groups and one the sketch,
  // so (stages - G - 1) x resident blocks x stage bytes are in flight ahead
  // of them: take the configuration that keeps >= 64 KB per SM ahead (HBM
  // latency x per-SM bandwidth), then the one with more resident blocks, then
  // more stages. Cached per shape.
  // (a few shapes per thread: the step SpMV and the start sketch alternate)
  static thread_local int64_t keys[4] = {-1, -1, -1, -1};
  static thread_local int bests[4][2];
  static thread_local int next_slot = 0;
  const int64_t key = (int64_t(cap) << 40) ^ (S->d << 20) ^ (S->ent_stride << 8) ^ sizeof(RP) ^
                      (FMT << 4) ^ (int64_t(ND) << 32) ^ (int64_t(dict_len) << 48);
  int slot = -1;
  for (int i = 0; i < 4; ++i)
    if (keys[i] == key) slot = i;
  int best_s = slot >= 0 ? bests[slot][0] : 0, best_per = slot >= 0 ? bests[slot][1] : 0;
  if (slot < 0) {
    best_s = 0;
    best_per = 0;
    int64_t best_ahead = -1;
    const int64_t stride = int64_t(stage_layout(int(sizeof(RP)), cap, off_stride,
                                                int(S->ent_stride), FMT).stride);
    for (int s = G + 2; s <= kStages; ++s) {
      if (env_stages() && s != env_stages()) continue;
      const size_t sm = pipe_smem<RP>(cap, int(S->d), off_stride, int(S->ent_stride), s, FMT, dict_len);
      if (sm > 220 * 1024) continue;
      RKMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      int per = 0;
      RKMF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kThreads, sm));
      if (per <= 0) continue;
      const int64_t ahead = std::min<int64_t>(int64_t(per) * (s - G - 1) * stride, 64 * 1024);
      if (ahead > best_ahead || (ahead == best_ahead && per > best_per) ||
          (ahead == best_ahead && per == best_per && s > best_s)) {
        best_ahead = ahead;
        best_per = per;
        best_s = s;
      }
    }
    if (knob_env("RKMF_PIPE_VERBOSE"))
      fprintf(stderr, "[rkmf] K2 pipe RP=%d TPR=%d G=%d FMT=%d ND=%d: stages=%d blocks/SM=%d stride=%lld\n",
              int(sizeof(RP)), TPR, G, FMT, ND, best_s, best_per, (long long)stride);
    slot = next_slot;
    next_slot = (next_slot + 1) & 3;
    keys[slot] = key;
    bests[slot][0] = best_s;
    bests[slot][1] = best_per;
  }
  if (best_s == 0) return false;
  const int stages = best_s, per_sm = best_per;
  const size_t smem = pipe_smem<RP>(cap, int(S->d), off_stride, int(S->ent_stride), stages, FMT, dict_len);
  RKMF_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int64_t tiles = (A->n_rows + kTileRows - 1) / kTileRows;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t(per_sm) * sms())));
  if (grid > red.max_blocks || S->d > red.max_len)
    param_error("internal: sketch reduction scratch too small");
  red.groups = det_groups(grid);
#define RKMF_PIPE_LAUNCH_ARGS                                                                  \
  A->n_rows, static_cast<const RP*>(A->row_ptr), A->col,                                       \
      FMT == 4   ? reinterpret_cast<const double*>(A->rtid)                                    \
      : FMT == 3 ? reinterpret_cast<const double*>(A->dtid)                                    \
      : FMT      ? A->dval                                                                     \
                 : A->val,                                                                     \
      x, xscale_dev, z, tiles, cap, int(S->d), int(S->ent_stride), off_stride, S->tile_off,    \
      S->tile_ent, S->scale, stop, step, stages, env_l2_hints(), env_debug(), A->doff,         \
      A->ndiag, A->n_cols, env_sync(), A->dstride, A->ddict, A->ntup, A->rcnt, A->roff,        \
      A->rval, A->rntup, red
  if constexpr (FMT == 2 || FMT == 3) {
    DictParam dp{};
    if (dict_par && A->ddict_host)
      for (int i = 0; i < A->ntup * ND; ++i) dp.v[i] = A->ddict_host[i];
    launch_maybe_pdl(fn, dim3(grid), dim3(kThreads), smem, st, RKMF_PIPE_LAUNCH_ARGS, dp);
  } else {
    launch_maybe_pdl(fn, dim3(grid), dim3(kThreads), smem, st, RKMF_PIPE_LAUNCH_ARGS);
  }
#undef RKMF_PIPE_LAUNCH_ARGS
  return true;
}

// Threads per row: enough that each thread's first 8 gathers cover an average
// row (RKMF_PIPE_TPR=1|2|4 overrides).
int pick_tpr(const CsrView* A) {
  static int env = -1;
  if (env < 0) {
    const char* e = knob_env("RKMF_PIPE_TPR");
    env = e ? atoi(e) : 0;
  }
  if (env == 1 || env == 2 || env == 4) return env;
  const double avg = A->n_rows ? double(A->nnz) / double(A->n_rows) : 0.0;
  return avg <= 10.0 ? 1 : (avg <= 40.0 ? 2 : 4);
}

// SpMV groups per block: one for short rows (its tiles are small, several
// blocks fit per SM), two for long rows (one block per SM; two tiles' gathers
// in flight). RKMF_PIPE_GROUPS=1|2|3 overrides.
int pick_groups(const CsrView* A) {
  static int env = -1;
  if (env < 0) {
    const char* e = knob_env("RKMF_PIPE_GROUPS");
    env = e ? atoi(e) : 0;
  }
  if (env >= 1 && env <= 3) return env;
  const double avg = A->n_rows ? double(A->nnz) / double(A->n_rows) : 0.0;
  return avg <= 10.0 ? 1 : 2;
}

template <typename RP, int TPR, int FMT = 0>
bool launch_pipe_g(const CsrView* A, const SketchView* S, const double* x,
                   const double* xscale_dev, double* z, const int32_t* stop,
                   int step, DetRed& red, cudaStream_t st) {
  // at most 1024 threads per block: TPR 4 runs one group, TPR 2 up to three
  int g = pick_groups(A);
  while (g > 1 && g * kTileRows * TPR + kSketchThreads + 32 > 1024) --g;
  if (g >= 3 && TPR <= 2)
    return launch_pipe_t<RP, TPR, (TPR <= 2 ? 3 : 1), FMT>(A, S, x, xscale_dev, z, stop, step,
                                                          red, st);
  if (g == 2 && TPR <= 2)
    return launch_pipe_t<RP, TPR, (TPR <= 2 ? 2 : 1), FMT>(A, S, x, xscale_dev, z, stop, step,
                                                          red, st);
  return launch_pipe_t<RP, TPR, 1, FMT>(A, S, x, xscale_dev, z, stop, step, red, st);
}

template <typename RP, int FMT = 0>
bool launch_pipe_rp(const CsrView* A, const SketchView* S, const double* x,
                    const double* xscale_dev, double* z, const int32_t* stop,
                    int step, DetRed& red, cudaStream_t st) {
  switch (pick_tpr(A)) {
    case 4: return launch_pipe_g<RP, 4, FMT>(A, S, x, xscale_dev, z, stop, step, red, st);
    case 2: return launch_pipe_g<RP, 2, FMT>(A, S, x, xscale_dev, z, stop, step, red, st);
    default: return launch_pipe_g<RP, 1, FMT>(A, S, x, xscale_dev, z, stop, step, red, st);
  }
}

}  // namespace

void trace_bind_spmv_pipe(unsigned long long* p) { trace_bind_tu(p); }

// sketch of x alone through the same pipeline (no matrix stream): the start
// vector's S*start (basis.cpp:103-104), mode 2 of launch_spmv_sketch
bool launch_sketch_only_pipe(const SketchView* S, const double* x, const double* xscale_dev,
                             DetRed& red, cudaStream_t st) {
  // the diagonal path with one diagonal of ones: x staged by the same
  // prefetching SpMV threads, no matrix stream
  CsrView v{};
  v.n_rows = S->n;
  v.n_cols = S->n;
  v.ndiag = 1;
  return launch_pipe_t<int32_t, 1, 1, 2, 1>(&v, S, x, xscale_dev, nullptr, nullptr, 0, red, st);
}

bool launch_spmv_sketch_pipe(const CsrView* A, const SketchView* S, const double* x,
                             const double* xscale_dev, double* z,
                             const int32_t* stop_flag, int step, DetRed& red, cudaStream_t st) {
  if (A->ndiag > 0 && A->dtid && A->ntup > 0) {  // row dictionary of the diagonal copy
#define RKMF_DIT(NDV) \
  case NDV: return launch_pipe_t<int32_t, 1, RKMF_K2_DICT_G, 3, NDV>(A, S, x, xscale_dev, z, stop_flag, step, red, st)
    switch (A->ndiag) {
      RKMF_DIT(1); RKMF_DIT(2); RKMF_DIT(3); RKMF_DIT(4);
      RKMF_DIT(5); RKMF_DIT(6); RKMF_DIT(7); RKMF_DIT(8);
      default: break;
    }
#undef RKMF_DIT
  }
  if (A->ndiag > 0 && A->dval) {  // diagonal copy (at most 8 diagonals), x prefetched
#define RKMF_DIA(NDV) \
  case NDV: return launch_pipe_t<int32_t, 1, 1, 2, NDV>(A, S, x, xscale_dev, z, stop_flag, step, red, st)
    switch (A->ndiag) {
      RKMF_DIA(1); RKMF_DIA(2); RKMF_DIA(3); RKMF_DIA(4);
      RKMF_DIA(5); RKMF_DIA(6); RKMF_DIA(7); RKMF_DIA(8);
      default: break;
    }
#undef RKMF_DIA
  }
  if (A->rtid && A->rntup > 0 && A->rkd <= kRdMaxNnz) {  // CSR row dictionary
    return launch_pipe_t<int32_t, RKMF_K2_RD_TPR, RKMF_K2_RD_G, 4>(A, S, x, xscale_dev, z,
                                                                   stop_flag, step, red, st);
  }
  if (!A->padded || A->max_tile_nnz > A->cap || A->cap > 4096) return false;
  return A->rp64 ? launch_pipe_rp<int64_t>(A, S, x, xscale_dev, z, stop_flag, step, red, st)
                 : launch_pipe_rp<int32_t>(A, S, x, xscale_dev, z, stop_flag, step, red, st);
}

}  // namespace rkmf_b200
