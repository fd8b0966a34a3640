// internal.h -- host-side declarations shared by the API and the kernel files.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace h2d {

// launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its predecessor's last CTAs run; kernels call pdl_wait()
// before any global access.  HOM2D_NO_PDL=1: ordinary launches (A/B).
bool pdl_enabled();
void pdl_refresh();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_if(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  return launch_pdl_if(true, kernel, grid, block, smem, s, args...);
}

// Opt a kernel into more than 48 KB of dynamic shared memory once per device
// (the attribute is per device; `done` holds one bit per device ordinal).
// Thread-safe: a race only repeats the idempotent call.  Returns its error.
template <typename... KArgs>
cudaError_t smem_optin(void (*kernel)(KArgs...), int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
  return e;
}

// One RK stage (or a bare residual):  out = a0*q0 + a1*q + bcoef*dt*R(q)
// (SSP-RK3 of P:868 in Shu-Osher form; residual mode: a0 = a1 = 0, bcoef = 1,
// dt == nullptr).  Arrays are the local strip in the canonical SoA layout.
struct StageArgs {
  const double* q;        // stage input (neighbours read from here)
  const double* q0;       // q^n (pointwise only); may alias out; nullptr if a0 == 0
  double* out;
  int nx, nrows;          // local strip: nx element columns, nrows element rows
  long long cs;           // component stride of q, q0, out (values)
  // y-neighbour rows beyond the strip (full element/cell rows, canonical layout
  // with component stride gcs).  nullptr = physical transmissive boundary.
  const double* ghost_lo; // rows -G..-1  (G = 1 HO, 2 FV)
  const double* ghost_hi; // rows nrows..nrows+G-1
  long long gcs;
  int bcx;                // x boundary: 0 periodic, 1 transmissive
  double rdx2, rdy2;      // HO: 2/dx, 2/dy (metric of the affine map); FV: 1/dx, 1/dy
  double a0, a1, bcoef;
  const double* dt;       // device scalar; nullptr -> 1.0; a stage with *dt == 0 is skipped
  double gamma;
  unsigned long long* lam; // optional: atomicMax of max(|u|,|v|)+c of `out` (bits of a double >= 0)
  unsigned long long* bad; // optional: atomicMin of the first non-physical point index
  long long* dec;          // optional: decision counters [8]
  long long* dmap;         // optional (FV, with dec, one rank): per-cell minmod outcomes [nx*nrows]
  int count_bot;           // this strip owns the domain's bottom face row (decision counting)
  double* qbar;            // optional (HO limiter runs): element averages of `out`, [4][nx*nrows]
                           // (Alg. 9: 1/4 sum_ab w_a w_b q_ab), fused into the stage epilogue
  int fv_unlimited;        // FV: unlimited kappa-scheme (hom2d_config.fv_unlimited)
  int no_pdl;              // launch without programmatic serialization (after a cross-stream
                           // event wait: griddepcontrol.wait only covers the previous kernel)
  int row_lo, row_hi;      // this launch updates strip rows [row_lo, row_hi) (row_hi == 0: all rows);
                          // it may read rows row_lo-G .. row_hi+G-1 (ghost rows outside the strip)
  int rows;                // marching kernels: element rows per CTA (set by the launcher)
  int row_lo2, row_hi2;    // optional second row band (row_hi2 > row_lo2): the strip's two boundary
                           // bands of the multi-GPU path in one launch
  int nb1;                 // row blocks of the first band (set by the launcher)
  double* laml;            // optional (limiter runs, stage 3): per element line, the largest
  unsigned long long* badl;  // max(|u|,|v|)+c of `out` and its first non-physical point (LamFuse)
  // dt of the step without a k_dt launch (dtrole 1: stage 1 computes dt = cflh / lam from the
  // clock and the wave speed, thread (0,0,0) publishes it to clk[1]; dtrole 2: stage 2 reads it
  // and thread (0,0,0) commits the clock {t += dt, steps++, stepped} and recycles lam)
  int dtrole;
  double* clk;
  unsigned long long* lamdt;
  double cflh;
};

// ring-stage stride of the marching HO kernels (doubles): the 128-B-swizzled P3
// rows need 1024-B aligned stages; the 1-D bulk-copy paths (P1, P2, P4) only
// 16-B alignment (H2D_STGA_1K=1: the round-1 1024-B stride everywhere)
#ifndef H2D_STGA_1K
#define H2D_STGA_1K 0
#endif
#define H2D_STGA(STG) ((SWZ || H2D_STGA_1K) ? (((STG) + 127) & ~127) : (((STG) + 1) & ~1))

// normalise the launch's row range; returns its row count
inline int row_range(StageArgs& a) {
  if (a.row_hi <= 0) { a.row_lo = 0; a.row_hi = a.nrows; }
  if (a.row_hi2 < a.row_lo2) a.row_hi2 = a.row_lo2;
  return (a.row_hi - a.row_lo) + (a.row_hi2 - a.row_lo2);
}
// grid rows of a marching launch over the band(s) at `rows` rows per CTA (sets a.nb1)
inline int band_blocks(StageArgs& a) {
  a.nb1 = (a.row_hi - a.row_lo + a.rows - 1) / a.rows;
  return a.nb1 + (a.row_hi2 - a.row_lo2 + a.rows - 1) / a.rows;
}

// rows per CTA for a marching kernel: enough CTAs to fill the GPU (ctas_per_sm
// resident per SM), at most rb_max (each march re-reads 1-2 prologue rows: long
// marches on big grids, short ones -- down to 1 row -- on the latency-bound
// small grids)
int march_rows(int nrows, int strips, int rb_max, int ctas_per_sm = 4);

// host: 3-D TMA tensor map {16 points, nelem elements, 4 components} (fp64,
// box {16, box_e, box_c}, 128-B swizzle) over an element-row array; base == nullptr
// gives an unused zero map (transmissive boundary)
bool make_map(CUtensorMap* m, const double* base, long long nelem, long long cs, int box_e, int box_c = 1);

int launch_gl_stage(int method, int k, const StageArgs& a, cudaStream_t s);   // DG, SD (marching)
int launch_gll_stage(int method, int k, const StageArgs& a, cudaStream_t s);  // CPR, NDG
int launch_fv_stage(int k, const StageArgs& a, cudaStream_t s);
int launch_dgoi_stage(int k, const StageArgs& a, cudaStream_t s);
// P1 element-per-lane kernel (CPR, NDG, DG, SD); -1 if it does not apply (layout, variant)
int launch_p1_stage(int method, const StageArgs& a, cudaStream_t s);
int march_rows_waves(int nrows, int strips, int rb_max, int ctas_per_sm);  // DG, (k+2)-point over-integration (f3)

// peer-memory halo (peer.cu): signal "my X is complete" into the neighbours'
// flags; pull the neighbours' G boundary rows of X (their memory, mapped) into
// the local ghost buffers once both have signalled exchange `seq`
struct PeerPull {
  const unsigned long long *flag_lo, *flag_hi;  // own flags, written by the lo / hi neighbour
  unsigned long long seq;
  const double *src_lo, *src_hi;  // neighbour rows (mapped); nullptr = no neighbour on that side
  long long src_cs;               // their component stride
  double *dst_lo, *dst_hi;        // ghost buffers [4][cnt]
  long long cnt;                  // values per component (G rows)
  int vec;                        // every run 16-B aligned and cnt even: 16-B copies
};
int launch_peer_signal(unsigned long long* to_lo, unsigned long long* to_hi, unsigned long long seq,
                       cudaStream_t s);
int launch_peer_pull(const PeerPull& p, cudaStream_t s);

struct AuxArgs {
  int method, k, nx, nrows, row0, ny_global;
  double xmin, xmax, ymin, ymax, gamma;
  long long cs;
  const double* dt;  // optional: skip the pass when *dt == 0 (clipped-out step)
};

// max(|u|,|v|)+c over the state -> atomicMax into lam (bits); optional bad-point check
void launch_lambda(const AuxArgs& a, const double* q, unsigned long long* lam, unsigned long long* bad,
                   cudaStream_t s);
// dt bookkeeping: see aux.cu
// clock = {t, dt, steps, stepped, t_end} (device): one step's dt, clipped to t_end - t
void launch_dt(double* clock, unsigned long long* lam_acc, double cfl, double hmin, cudaStream_t s);
void launch_init_case(const AuxArgs& a, int case_id, double* q, cudaStream_t s);
// per-block partial sums {sum w|d|, sum w d^2, max|d|} -> part[3*nblocks]; returns nblocks
int launch_error_partials(const AuxArgs& a, const double* q, int var, const double* clock, double* part,
                          int max_blocks, cudaStream_t s);
void launch_error_final(const double* part, int nblocks, double* out3, cudaStream_t s);
// FV reconstructed-solution error partials (hom2d_config.fv_error_recon);
// glo / ghi: 2 ghost rows each side (component stride gcs), nullptr = transmissive
int launch_error_fv_recon(const AuxArgs& a, const double* q, const double* glo, const double* ghi, long long gcs,
                          int bcx, int unlimited, int var, const double* clock, double* part, int max_blocks,
                          cudaStream_t s);
// averages Qbar[4][nx*nrows] and the detect+limit pass (HO)
void launch_averages(const AuxArgs& a, const double* q, double* qbar, cudaStream_t s);
// LamFuse (limiter runs, after stage 3): the dt wave speed and the non-physical
// check of the LIMITED state without another pass over it -- unmarked elements
// keep their stage-3 output, whose per-line speeds / first bad points the stage
// kernel wrote (laml / badl, N entries per element); marked elements are
// evaluated by k_limit at their rebuilt points.  lam_out == nullptr: off.
struct LamFuse {
  const double* laml = nullptr;
  const unsigned long long* badl = nullptr;
  unsigned long long* lam_out = nullptr;
  unsigned long long* bad_out = nullptr;
};
void launch_limit(const AuxArgs& a, double* q, const double* qbar, const double* qbar_lo, const double* qbar_hi,
                  long long qbar_gcs, int bcx, double eps, int all_vars, int charact, long long* dec,
                  long long* emap, cudaStream_t s,
                  const LamFuse& lf = LamFuse());

}  // namespace h2d
