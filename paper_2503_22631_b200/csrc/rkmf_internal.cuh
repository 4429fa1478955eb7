// Internal declarations of the rkmf_b200 CUDA library (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "detred.cuh"
#include "rkmf_b200.h"

namespace rkmf_b200 {

// ---- error plumbing: C++ exceptions inside, status codes at the C ABI ----
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void param_error(const std::string& m) { throw Error(RKMF_PARAMETER_ERROR, m); }
[[noreturn]] inline void shape_error(const std::string& m) { throw Error(RKMF_SHAPE_ERROR, m); }
[[noreturn]] inline void numerical_error(const std::string& m) {
  throw Error(RKMF_NUMERICAL_ERROR, m);
}

#define RKMF_CUDA(call)                                                                  \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::rkmf_b200::Error(RKMF_DEVICE_ERROR, std::string("CUDA error: ") +          \
                                                      cudaGetErrorString(e_) + " at " + \
                                                      __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// ---- ablation knobs: environment variables are read only in
// the experiments build (`make experiments` -> _lib/librkmf_b200_exp.so,
// -DRKMF_EXPERIMENTS); the product library always runs the defaults. ----
inline const char* knob_env(const char* name) {
#ifdef RKMF_EXPERIMENTS
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// ---- programmatic dependent launch (PDL) between the per-step kernels ----
// Each step kernel runs its dependency-free prologue, then waits for the
// previous kernel in the stream (griddepcontrol.wait: full completion and
// memory visibility), then lets the next kernel launch. Triggering only after
// the wait keeps the chain strictly ordered (kernel i+1 never overlaps i-1).
// Without the launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_wait_then_trigger() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();  // RKMF_PDL=0 disables (engine.cu)

template <typename... KArgs, typename... Args>
void launch_maybe_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (e != cudaSuccess)
    throw Error(RKMF_DEVICE_ERROR, std::string("cudaLaunchKernelEx: ") + cudaGetErrorString(e));
}

// ---- optional device timeline of the step kernels (tools/trace_steps.py) ----
// Per step k, kTraceSlots globaltimer stamps (ns), merged with atomicMax, so
// a buffer armed before a solve holds its last cycle; "first" stamps are
// taken by block 0 only. Off (null pointer) unless rkmf_debug_trace armed it;
// the pointer is per translation unit (trace_bind_*).
constexpr int kTraceSlots = 16;
static __device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Compiled in only with -DRKMF_TRACE (make trace: _lib/librkmf_b200_trace.so):
// the product kernels carry no stamps (K2 and K4 are sensitive to code
// generation; the stamps cost ~1.5% of the cfg2 solve).
__device__ __forceinline__ void trace_max(int k, int slot) {
#ifdef RKMF_TRACE
  if (g_trace) atomicMax(g_trace + k * kTraceSlots + slot, gtime());
#endif
}
__device__ __forceinline__ void trace_first(int k, int slot) {
#ifdef RKMF_TRACE
  if (g_trace && blockIdx.x == 0) atomicMax(g_trace + k * kTraceSlots + slot, gtime());
#endif
}
static inline void trace_bind_tu(unsigned long long* p) {
  cudaMemcpyToSymbol(g_trace, &p, sizeof(p));
}
void trace_bind_krylov(unsigned long long* p);
void trace_bind_spmv_pipe(unsigned long long* p);

// Tile geometry shared by the SpMV, sketch and update kernels: one tile is
// kTileRows consecutive rows handled by one 128-thread block iteration.
constexpr int kTileRows = 128;
constexpr int kBlock = 128;

// Per-solve device state: scalars that the kernels communicate through, read
// back by the host once or twice per cycle (pinned mirror in the context).
struct SolveState {
  int32_t stopped;     // number of valid steps this cycle (m_eff unless breakdown)
  int32_t breakdown;   // 1-based breakdown step, 0 = none
  int32_t zero_start;  // start vector sketched to zero
  int32_t nonfinite;   // y had a NaN/Inf
  double alpha_k;      // this cycle's start norm ||S start||
  double sigma;        // 1 / alpha_k (folded into column 0)
  double alpha1;       // cycle-1 start norm (global scale)
  double coupling;     // previous cycle's subdiagonal r_{m+1,m}
  double yn2;          // ||y_k||^2 accumulator        } adjacent: one allreduce
  double err2;         // ||f_hat - reference||^2      }   of 2 doubles (multi-GPU)
  double rnorm1;       // ||R_accum||_1 (full dense-f path)
};

// ---- kernels (definitions in *.cu) ----
// sketch.cu
// columns [j0, j0 + n) of the global operator (j0 = 0 for a whole sketch)
void launch_sketch_generate(int64_t d, int64_t n, int64_t j0, int64_t zeta, uint64_t seed,
                            uint16_t* rows, int8_t* signs, cudaStream_t st);
// bytes per tile the entry layout needs (the largest tile's), then the layout
int64_t sketch_tiles_stride(int64_t d, int64_t n, int64_t zeta, const uint16_t* rows,
                            cudaStream_t st);
void launch_sketch_tiles(int64_t d, int64_t n, int64_t zeta, const uint16_t* rows,
                         const int8_t* signs, uint16_t* tile_off, uint8_t* tile_ent,
                         int64_t ent_stride, cudaStream_t st);
void launch_sketch_export(int64_t count, const uint16_t* rows, const int8_t* signs,
                          int64_t* rows64, cudaStream_t st);

// spmv.cu
struct CsrView {
  int64_t n_rows, n_cols, nnz;
  const void* row_ptr;  // int32 or int64
  bool rp64;
  const int32_t* col;
  const double* val;
  int cap;  // products staged per chunk (shared memory)
  int64_t max_tile_nnz;  // largest nonzero count of a 128-row tile
  bool padded;           // arrays carry the tail padding the TMA path needs
  // optional diagonal copy (dia.cu): [tile][diag][128] values at the sorted
  // column offsets doff; ndiag == 0 when the matrix has none
  const double* dval;
  const int32_t* doff;  // offsets: [8] for every tile (dstride 0) or [tile][8] (dstride 8)
  int ndiag;
  int dstride;
  // optional row dictionary of the diagonal copy (dia.cu): every row's ndiag
  // values are one of ntup distinct tuples; dtid[tile * 128 + r] = the row's
  // tuple id, ddict[id * ndiag + q] its values. ntup == 0 when absent.
  const uint8_t* dtid;
  const double* ddict;
  const double* ddict_host;  // host copy of ddict
  int ntup;
  // optional CSR row dictionary (rowdict.cu; matrices without a diagonal
  // copy): rtid[tile * 128 + r] = the row's form id; form f has rcnt[f]
  // nonzeros at column offsets roff[f * kRdMaxNnz + q] (col - row) with values
  // rval[f * kRdMaxNnz + q], q in column order. rntup == 0 when absent; rkd =
  // the largest rcnt.
  const uint8_t* rtid;
  const int32_t* rcnt;
  const int32_t* roff;
  const double* rval;
  int rntup;
  int rkd;
};
constexpr int kRdMaxNnz = 32;
constexpr int kMaxDiag = 8;
constexpr int kMaxTuples = 256;
// Row-pointer tail padding (entries) and value/column padding (elements)
// allocated by the engine so 16-byte-rounded bulk copies stay in bounds.
constexpr int64_t kRpPad = 136;
constexpr int64_t kNnzPad = 8;
struct SketchView {
  int64_t d, n, zeta;
  const uint16_t* tile_off;  // [num_tiles][tile_off_stride(d)]: the tile header (below)
  const uint8_t* tile_ent;   // [num_tiles][ent_stride]: entries, local row | sign<<7
  int64_t ent_stride;        // bytes per tile of tile_ent (a multiple of 128)
  double scale;
};
// Sketch tile layout (built by sketch_tiles_kernel, read by sketch_tile_gather).
// The d sketch rows ("bins") of a 128-column tile are renumbered into slots by
// entry count, descending; the 128 sketch threads walk the slots in snake
// order, warp w of pass j taking slots [128 j + 32 w, +32) (j even) or
// [128 j + 96 - 32 w, +32) (j odd, lane order reversed): a "group" of 32
// slots of near-equal length per warp. Header (uint16 units):
//   len[d]  uint8  slot lengths                 (bytes 0 .. d-1)
//   bin[d]  uint16 the sketch row of each slot  (from tile_hdr_bin(d))
//   gb[ng]  uint16 byte offset of group g's entries (from tile_hdr_gbase(d))
// Entries of a group: ceil(L/4) rounds of one 32-bit word per lane, L the
// group's longest slot (word k of lane l at gb + 4 (32 k + l)); byte c of the
// word is the lane's entry 4k + c, which feeds its chain c (the sums are those
// of a slot-contiguous layout with the same entry order). Each round is one
// conflict-free shared load per warp; bytes past a lane's length are padding.
// A tile's groups take sum over groups of 128 ceil(L/4) bytes; every tile has
// the sketch's largest such size (ent_stride, measured when it is built).
constexpr int kSketchNT = 128;  // sketch threads per tile (fixed by the layout)
__host__ __device__ inline int64_t tile_groups(int64_t d) {
  return 4 * ((d + kSketchNT - 1) / kSketchNT);
}
__host__ __device__ inline int64_t tile_hdr_bin(int64_t d) { return (d + 1) / 2; }
__host__ __device__ inline int64_t tile_hdr_gbase(int64_t d) { return (d + 1) / 2 + d; }
__host__ __device__ inline int64_t tile_off_stride(int64_t d) {
  return (tile_hdr_gbase(d) + tile_groups(d) + 7) / 8 * 8;
}

// Sketch epilogue of one 128-row tile (sketch.cpp:51-63 as a gather): thread t
// sums the tile's contributions to the slots it owns and adds them to
// acc[bin]. zs2 holds the scaled z of the tile's rows twice, zs2[r] = +z_r and
// zs2[128 + r] = -z_r, so an entry byte (local row | sign << 7) indexes its
// signed value directly. The warp runs the group's rounds in lockstep (trip
// count = the group's longest slot), a lane's padding bytes predicated off.
// Entry bytes are extracted with a byte permute (PRMT) so each entry's table
// address is two instructions (PRMT, IMAD) rather than shift, mask and add.
// Every lane of the warp executes this (slots past d have length 0).
__device__ __forceinline__ void sketch_tile_gather(int t, int d, const uint16_t* hdr,
                                                   const uint8_t* ent, const double* zs2,
                                                   double* acc) {
  constexpr int NT = kSketchNT;
  const uint8_t* lens = reinterpret_cast<const uint8_t*>(hdr);
  const uint16_t* bins = hdr + tile_hdr_bin(d);
  const uint16_t* gbase = hdr + tile_hdr_gbase(d);
  const int lane = t & 31, w = t >> 5;
  for (int j = 0; NT * j < d; ++j) {
    const int s = (j & 1) ? NT * j + NT - 1 - t : NT * j + t;
    const int len = s < d ? int(lens[s]) : 0;
    const int mx = int(__reduce_max_sync(0xffffffffu, unsigned(len)));
    const uint32_t* gw = reinterpret_cast<const uint32_t*>(ent + gbase[4 * j + w]) + lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int p = 0;
#pragma unroll 1
    for (; p + 4 < mx; p += 8, gw += 64) {  // two rounds per iteration
      const uint32_t e = gw[0], f = gw[32];
      if (p < len) a0 += zs2[__byte_perm(e, 0, 0x4440)];
      if (p + 1 < len) a1 += zs2[__byte_perm(e, 0, 0x4441)];
      if (p + 2 < len) a2 += zs2[__byte_perm(e, 0, 0x4442)];
      if (p + 3 < len) a3 += zs2[__byte_perm(e, 0, 0x4443)];
      if (p + 4 < len) a0 += zs2[__byte_perm(f, 0, 0x4440)];
      if (p + 5 < len) a1 += zs2[__byte_perm(f, 0, 0x4441)];
      if (p + 6 < len) a2 += zs2[__byte_perm(f, 0, 0x4442)];
      if (p + 7 < len) a3 += zs2[__byte_perm(f, 0, 0x4443)];
    }
    if (p < mx) {
      const uint32_t e = gw[0];
      if (p < len) a0 += zs2[__byte_perm(e, 0, 0x4440)];
      if (p + 1 < len) a1 += zs2[__byte_perm(e, 0, 0x4441)];
      if (p + 2 < len) a2 += zs2[__byte_perm(e, 0, 0x4442)];
      if (p + 3 < len) a3 += zs2[__byte_perm(e, 0, 0x4443)];
    }
    if (s < d) acc[bins[s]] += (a0 + a1) + (a2 + a3);
  }
}

// mode: 0 = z = xscale*A x ; 1 = also sketch z ; 2 = sketch x only. The
// sketch comes out as red.groups group partials in red.gpart (detred.cuh:
// a fixed-order, reproducible reduction); consumers sum them in group order
// (det_group_sum), launch_det_finish writes the plain d-vector.
void launch_spmv_sketch(const CsrView* A, const SketchView* S, int mode, const double* x,
                        const double* xscale_dev, double* z, const int32_t* stop_flag,
                        int step, int grid, DetRed& red, cudaStream_t st);
void launch_det_finish(const DetRed& red, int64_t L, double* out, cudaStream_t st);
int spmv_sketch_grid(const CsrView* A, const SketchView* S, int mode);
// the same pipeline for the sketch of x alone (mode 2)
bool launch_sketch_only_pipe(const SketchView* S, const double* x, const double* xscale_dev,
                             DetRed& red, cudaStream_t st);
// TMA-pipelined mode-1 kernel (spmv_pipe.cu); returns false when not applicable.
bool launch_spmv_sketch_pipe(const CsrView* A, const SketchView* S, const double* x,
                             const double* xscale_dev, double* z,
                             const int32_t* stop_flag, int step, DetRed& red, cudaStream_t st);
// colsum: scratch of 2 * n_cols + 1 doubles (fixed-point words, spmv.cu)
void launch_matrix_norm1(const CsrView* A, double* colsum, double* out, cudaStream_t st);
// the fixed-point column abs-sums behind norm1 (order-independent; spmv.cu)
void launch_abs_max_bits(int64_t nnz, const double* val, unsigned long long* vmax_bits,
                         cudaStream_t st);
void launch_fx_colsum(int64_t nnz, const int32_t* col, const double* val,
                      const unsigned long long* vmax_bits, int64_t ncols, unsigned long long* hi,
                      unsigned long long* lo, cudaStream_t st);
void launch_fx_scatter_add(int64_t cnt, const int32_t* idx, const unsigned long long* v,
                           unsigned long long* out, cudaStream_t st);
void launch_fx_colmax(int64_t n, const unsigned long long* hi, const unsigned long long* lo,
                      const unsigned long long* vmax_bits, double* out, cudaStream_t st);
void launch_matrix_check(const CsrView* A, int32_t* flags, bool require_sorted, cudaStream_t st);

// cycle_small.cu: a whole cycle's steps in one cooperative kernel (small n)
constexpr int64_t kCycleSmallMaxRows = 131072;
bool cycle_small_applicable(const CsrView* A, const SketchView* S, int64_t m_eff);
bool launch_cycle_small(const CsrView* A, const SketchView* S, int m_eff, bool fuse_last,
                        double* W, int64_t ldw, double* z, double* U, double* Rbar, int64_t ldr,
                        double* G, double tol, int64_t n_global, SolveState* st_dev,
                        DetRed& red, cudaStream_t st);

// krylov.cu
// the start sketch arrives as ng group partials (detred.cuh)
void launch_start_init_m(int64_t d, const double* sgpart, int ng, double* U, SolveState* st_dev,
                         bool first, int m_eff, cudaStream_t st);
// G: (m+1) x (m+1) scratch for the Gram rows of U (row i at i*ldg), or null
// for the sequential MGS sweep.
// p = S A w_k arrives as ng group partials pgpart[ng][d] (detred.cuh)
void launch_rgs_step(int64_t d, int k, int64_t m, int64_t n, double tol, const double* pgpart,
                     int ng, double* U, double* Rbar, double* G, int64_t ldg, SolveState* st_dev,
                     cudaStream_t st);
void launch_basis_update(int64_t n, int k, int64_t ldw, double* W, const double* z,
                         const double* Rbar, int64_t ldr, const SolveState* st_dev,
                         cudaStream_t st);
void launch_final_update(int64_t n, int m_eff, int64_t ldw, double* W, const double* z,
                         const double* Rbar, int64_t ldr, const double* g, double* f_hat,
                         const double* ref, SolveState* st_dev, const DetRed& red,
                         cudaStream_t st);
void launch_scale_copy(int64_t n, const double* src, double* dst, const SolveState* st_dev,
                       cudaStream_t st);
void launch_fill(int64_t n, double v, double* x, cudaStream_t st);

// classical.cu: the classical builder (S == nullptr) via CGS2
// the grid reductions (norms, the k+1 dots as reduction slices) are the
// fixed-order ones of detred.cuh
void launch_cl_start(int64_t n, const double* start, double* nrm2_scratch, SolveState* st_dev,
                     bool first, int m_eff, bool norm_only, const DetRed& red, cudaStream_t st);
void launch_cl_multidot(int64_t n, int k, int64_t ldw, const double* W, const double* z,
                        double* h, const SolveState* st_dev, const DetRed& red, cudaStream_t st);
void launch_cl_update(int64_t n, int k, int64_t ldw, const double* W, double* z, const double* h,
                      double* nrm2, bool store, const SolveState* st_dev, const DetRed& red,
                      cudaStream_t st);
void launch_cl_decide(int k, int64_t ldr, int64_t n_global, double tol, double* h1, double* h2,
                      double* nrm2, double* Rbar, double* rlast, SolveState* st_dev,
                      cudaStream_t st);
void launch_cl_scale(int64_t n, int k, int64_t ldw, double* W, const double* z,
                     const double* Rbar, int64_t ldr, const SolveState* st_dev, cudaStream_t st);

// diag.cu: per-cycle kappa_W and leftmost Ritz value (opt-in)
size_t gram_scratch_doubles(int64_t n, int m);
bool launch_gram(int64_t n, int m, int64_t ldw, const double* W, const SolveState* st_dev,
                 double* G, cudaStream_t st);
double kappa_from_gram(const std::vector<double>& G, int m);
double leftmost_ritz(const std::vector<double>& Rbar, int64_t ldr, int m);
void ritz_values(const std::vector<double>& Rbar, int64_t ldr, int m, std::vector<double>& wr,
                 std::vector<double>& wi);

// densef.cu
void launch_raccum_append(double* R, int64_t ldr_acc, int64_t M, const double* Rbar,
                          int64_t ldr, SolveState* st_dev, cudaStream_t st);
void launch_dense_norm1(const double* R, int64_t ld, int64_t N, double* out, cudaStream_t st);
// Full exp(-t R) e1 by Taylor-19 Paterson-Stockmeyer scaling and squaring.
// Writes u = exp(-tR) e1 (length N) into u_out. ws must hold 6*N*N doubles.
void dense_expneg_e1(const double* R, int64_t ldr, int64_t N, double t, int s, double* ws,
                     double* u_out, cudaStream_t st, int64_t* launches);
// g[j] = alpha1 * u[M + j] (j < mk), g[0] *= sigma
void launch_make_g(const double* u, int64_t M, int mk, double* g, const SolveState* st_dev,
                   cudaStream_t st);
// InvSqrt restart quadrature: see densef.cu for the recursion.
struct QuadState {
  int nq;
  double* log_w;   // per node scalar state (double), size nq
  double* pi;      // running products, size nq
  double* emx;     // e_m^T x of the current block, size nq
  double* shift;   // sigma_q, size nq
  double* weight;  // w_q, size nq
};
// mk_replay >= 0: replay a past cycle (its R_accum block and coupling) into
// the node states of a new node set; no output
void launch_quad_invsqrt_cycle(const double* Rbar, int64_t ldr, int mk, int64_t cycle,
                               QuadState* q, double* g, const SolveState* st_dev,
                               double* partial, cudaStream_t st, int mk_replay = -1,
                               double coupling_replay = 0.0);
// the InvSqrt node set from the extremes of the Ritz values seen (densef.cu)
struct InvSqrtDesign {
  double u0 = 0, h = 0.25, lmin = 0, lmax = 0, thmax = 0;
  int nq = 0;
  bool covers(double lmin_seen, double lmax_seen, double thmax_seen) const;
  InvSqrtDesign doubled() const;  // same interval, half the step
};
InvSqrtDesign design_invsqrt(double lmin, double lmax, double thmax);
void invsqrt_nodes(const InvSqrtDesign& d, std::vector<double>& shift, std::vector<double>& weight);
// ExpNeg quadrature (complex nodes, see densef.cu): shift/weight/pi/emx hold
// nq complex values (interleaved re, im)
// mk_replay >= 0: replay a past cycle (its R_accum block, its coupling) to
// rebuild the node states after a contour change; no output
void launch_quad_expneg_cycle(const double* Rbar, int64_t ldr, int mk, int64_t cycle,
                              QuadState* q, double* g, const SolveState* st_dev,
                              double* partial, cudaStream_t st, int mk_replay = -1,
                              double coupling_replay = 0.0);
// the contour for exp(-t z) from the t-scaled Ritz values of the first cycle
struct ExpContour {
  double x0 = 0, p = 1, q = 10, h = 0.05, lmin = 0;
  int K = 0;
  bool inside(double re, double im) const;  // with the design margins
};
ExpContour design_exp_contour(const std::vector<double>& wr, const std::vector<double>& wi);
// host node arrays: shift (sigma = -zeta / t) and weight, complex interleaved
void exp_contour_nodes(const ExpContour& c, double t, std::vector<double>& shift,
                       std::vector<double>& weight);

}  // namespace rkmf_b200
