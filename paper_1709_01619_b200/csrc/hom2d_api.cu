// hom2d_api.cu -- the C ABI of include/hom2d.h: handle, workspace carve-up,
// strip partition, halo exchange (NCCL over NVLink when nranks > 1), and the
// SSP-RK3 driver loop that keeps t and dt on the device.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/hom2d.h"
#include "internal.h"

using namespace h2d;

struct hom2d {
  hom2d_config cfg;
  int rank = 0, nranks = 1, device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t xstream = nullptr;          // nranks > 1: halo exchange stream (highest priority)
  bool self_x = false;                     // HOM2D_SELF_EXCHANGE test mode (see self_exchange_env)
  bool self_nccl = false;                  // HOM2D_SELF_EXCHANGE=2: the same through a 1-rank NCCL communicator
  // peer-memory halo (hom2d_peer_connect; HOM2D_SELF_EXCHANGE=3: with itself as both neighbours)
  char* ws = nullptr;                      // the caller's workspace (same carve on every rank)
  bool peer = false;
  char *pws_lo = nullptr, *pws_hi = nullptr;  // the neighbours' workspaces, mapped
  void* ipc_mapped[2] = {nullptr, nullptr};   // IPC mappings to close
  unsigned long long peer_seq = 0;         // exchanges so far (the same count on every rank)
  unsigned long long* pflag = nullptr;     // [2]: last exchange signalled by the lo / hi neighbour
  cudaEvent_t ev_in = nullptr, ev_halo = nullptr;
  // CUDA graphs of 2^i steps (single GPU, untimed): launch-bound small grids
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev_a = nullptr, gev_b = nullptr;
  cudaGraphExec_t gexec[7] = {};
  long long glaunch[7] = {};
  bool graph_off = false;
  long long eager_steps = 0;
  bool dtfuse = true;                      // dt computed by stage 1 / committed by stage 2 (no k_dt)
  int dtrole = 0;                          // role of the next run_stage (StageArgs::dtrole)
  long long graph_after = 2048;            // eager steps before batches run as graphs (their capture sits
                                           // in the device timeline: ~2 ms, repaid after ~2-4k steps;
                                           // profiles/round2_small_grids.md)
  int graph_min_batch = 64;                // smallest batch run as a graph
  ncclComm_t comm = nullptr;
  int row0 = 0, nrows = 0, np = 1, G = 1;  // G ghost rows (HO 1, FV 2)
  long long nloc = 0;                      // values per component of the local strip
  double *Qn = nullptr, *Q1 = nullptr, *Q2 = nullptr;
  double* clock = nullptr;                 // [t, dt, steps, stepped]
  unsigned long long* lam = nullptr;       // [acc, cur]
  unsigned long long* bad = nullptr;
  long long* dec = nullptr;
  long long* dmap = nullptr;               // record_decisions, one rank: per-element decision map [nx*nrows]
  double* part = nullptr;                  // error partials
  int max_part = 0;
  double* err3 = nullptr;
  double* qbar = nullptr;                  // HO limiter averages [4][nx*nrows]
  double* laml = nullptr;                 // limiter runs: stage-3 per-line wave speeds (LamFuse)
  unsigned long long* badl = nullptr;
  double *glo = nullptr, *ghi = nullptr;   // received ghost rows [4][G*nx*np]
  double *qblo = nullptr, *qbhi = nullptr; // received ghost average rows [4][nx]
  double* t_host = nullptr;               // pinned: [0..3] clock, [5] t_end, [6..7] bad flags
  bool ovr_active = false;                 // hom2d_residual_strip ghost override
  const double *ovr_lo = nullptr, *ovr_hi = nullptr;
  bool poisoned = false;
  long long launches = 0;
  std::vector<cudaEvent_t> ev;             // stage-kernel timing: pairs (start, stop)
  int ev_used = 0;
  char msg[512] = {0};
};

// NVTX ranges (host timeline: hom2d_step / stage / exchange / limiter / error
// query; visible to nsys / ncu --nvtx, no cost without a tool attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

namespace {

hom2d_status fail(hom2d* h, hom2d_status st, const char* fmt, ...) {
  if (h) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(h->msg, sizeof(h->msg), fmt, ap);
    va_end(ap);
    if (st == HOM2D_ERR_CUDA || st == HOM2D_ERR_NCCL) h->poisoned = true;
  }
  return st;
}

#define CU(h, x)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) return fail(h, HOM2D_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)
#define NC(h, x)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (x);                                                              \
    if (r_ != ncclSuccess) return fail(h, HOM2D_ERR_NCCL, "%s: %s", #x, ncclGetErrorString(r_)); \
  } while (0)
// every entry point: valid, unpoisoned handle, its device current (handles of
// several devices may live in one process)
#define GUARD(h)                                                     \
  do {                                                               \
    if (!(h)) return HOM2D_ERR_ARG;                                  \
    if ((h)->poisoned) return HOM2D_ERR_STATE;                       \
    CU(h, cudaSetDevice((h)->device));                               \
  } while (0)

int points_per_elem(const hom2d_config& c) { return c.method == HOM2D_FV ? 1 : (c.k + 1) * (c.k + 1); }

// Test modes (one rank, periodic): the overlapped multi-GPU stage path --
// exchange stream, events, interior / boundary launches, ghost buffers -- on one
// GPU, bitwise against the plain path.  HOM2D_SELF_EXCHANGE=1: the NCCL send/recv
// replaced by device copies of the strip's own wrap rows; =2: the real NCCL data
// plane on a 1-rank communicator (ncclCommInitRank, the grouped ncclSend/ncclRecv
// of exchange() with rank 0 as both strip neighbours, every ncclAllReduce); =3:
// the peer-memory halo (peer.cu) with the handle's own workspace as both
// neighbours' (signal + flag-gated pull kernels; no IPC mapping).
int self_exchange_env(const hom2d_config& c, int nranks) {
  const char* v = getenv("HOM2D_SELF_EXCHANGE");
  if (nranks != 1 || c.bc != HOM2D_PERIODIC || !v) return 0;
  return v[0] == '1' ? 1 : v[0] == '2' ? 2 : v[0] == '3' ? 3 : 0;
}

hom2d_status check_cfg(const hom2d_config* c, int nranks) {
  if (!c) return HOM2D_ERR_ARG;
  if (c->method < 0 || c->method > 4 || (c->bc != 0 && c->bc != 1)) return HOM2D_ERR_ARG;
  if (c->method == HOM2D_FV ? (c->k < 1 || c->k > 2) : (c->k < 1 || c->k > 4)) return HOM2D_ERR_ORDER;
  if (c->nx < 2 || c->ny < 2 || !(c->xmax > c->xmin) || !(c->ymax > c->ymin)) return HOM2D_ERR_MESH;
  if (nranks < 1 || c->ny % nranks != 0) return HOM2D_ERR_MESH;
  const int G = c->method == HOM2D_FV ? 2 : 1;
  if (c->ny / nranks < G) return HOM2D_ERR_MESH;
  if (!(c->gamma > 1.0) || !(c->cfl > 0.0)) return HOM2D_ERR_ARG;
  if ((unsigned)c->limiter_per_step > 1u || (unsigned)c->limiter_all_vars > 1u || (unsigned)c->fv_unlimited > 1u ||
      (unsigned)c->limiter_characteristic > 1u || (unsigned)c->fv_error_recon > 1u ||
      (unsigned)c->dg_overintegrate > 1u)
    return HOM2D_ERR_ARG;
  return HOM2D_OK;
}

struct Carve {
  char* base;
  size_t off = 256;  // guard: bulk copies may read up to 8 B outside an array
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

// lay out the workspace; base == nullptr only measures
size_t carve(hom2d* h, const hom2d_config& c, int nranks, char* base) {
  Carve cv{base};
  const int np = points_per_elem(c);
  const int G = c.method == HOM2D_FV ? 2 : 1;
  const long long nrows = c.ny / nranks;
  const long long nloc = (long long)c.nx * nrows * np;
  const int max_part = 148 * 16;
  double* Qn = cv.take<double>(4 * nloc);
  double* Q1 = cv.take<double>(4 * nloc);
  double* Q2 = cv.take<double>(4 * nloc);
  double* clk = cv.take<double>(8);
  auto* lam = cv.take<unsigned long long>(4);
  auto* bad = cv.take<unsigned long long>(2);
  auto* dec = cv.take<long long>(8);
  double* part = cv.take<double>(3 * max_part);
  double* err3 = cv.take<double>(4);
  double* qbar = (c.method != HOM2D_FV) ? cv.take<double>(4 * (size_t)c.nx * nrows) : nullptr;
  // limiter runs: per element line, the stage-3 wave speed / first bad point (LamFuse)
  const bool lim = c.limiter && c.method != HOM2D_FV;
  const size_t nl = lim ? (size_t)c.nx * nrows * (c.k + 1) : 0;
  double* laml = lim ? cv.take<double>(nl) : nullptr;
  auto* badl = lim ? cv.take<unsigned long long>(nl) : nullptr;
  long long* dmap = (c.record_decisions && nranks == 1) ? cv.take<long long>((size_t)c.nx * nrows) : nullptr;
  double *glo = nullptr, *ghi = nullptr, *qblo = nullptr, *qbhi = nullptr;
  unsigned long long* pflag = nullptr;
  if (nranks > 1 || self_exchange_env(c, nranks)) {
    pflag = cv.take<unsigned long long>(2);  // (same offset on every rank: peer-memory halo flags)
    glo = cv.take<double>(4 * (size_t)G * c.nx * np);
    ghi = cv.take<double>(4 * (size_t)G * c.nx * np);
    if (c.method != HOM2D_FV) {
      qblo = cv.take<double>(4 * (size_t)c.nx);
      qbhi = cv.take<double>(4 * (size_t)c.nx);
    }
  }
  if (h && base) {
    h->Qn = Qn; h->Q1 = Q1; h->Q2 = Q2; h->clock = clk; h->lam = lam; h->bad = bad; h->dec = dec;
    h->part = part; h->max_part = max_part; h->err3 = err3; h->qbar = qbar; h->dmap = dmap;
    h->laml = laml; h->badl = badl;
    h->glo = glo; h->ghi = ghi; h->qblo = qblo; h->qbhi = qbhi; h->pflag = pflag;
  }
  return cv.off + 512;  // trailing guard
}

AuxArgs aux(const hom2d* h) {
  AuxArgs a;
  a.method = h->cfg.method; a.k = h->cfg.k; a.nx = h->cfg.nx; a.nrows = h->nrows; a.row0 = h->row0;
  a.ny_global = h->cfg.ny; a.xmin = h->cfg.xmin; a.xmax = h->cfg.xmax; a.ymin = h->cfg.ymin;
  a.ymax = h->cfg.ymax; a.gamma = h->cfg.gamma; a.cs = h->nloc; a.dt = nullptr;
  return a;
}

hom2d_strip_plan_t plan_of(const hom2d_config& c, int rank, int R) {
  hom2d_strip_plan_t p;
  p.nrows = c.ny / R;
  p.row0 = rank * p.nrows;
  p.ghost_rows = c.method == HOM2D_FV ? 2 : 1;
  p.peer_lo = (rank + R - 1) % R;
  p.peer_hi = (rank + 1) % R;
  p.has_lo = (c.bc == HOM2D_PERIODIC || rank > 0) ? 1 : 0;
  p.has_hi = (c.bc == HOM2D_PERIODIC || rank < R - 1) ? 1 : 0;
  p.row_values = (int64_t)c.nx * points_per_elem(c);
  return p;
}

// Exchange G boundary rows of the stage input X with the strip neighbours and
// return the ghost pointers the stage kernel reads (y-strip partition).
// Message order per peer: "last rows -> peer_hi" before "first rows -> peer_lo"
// and "recv lo" before "recv hi", so that with 2 periodic ranks (peer_lo ==
// peer_hi) NCCL's in-order matching pairs last->lo and first->hi.
hom2d_status exchange(hom2d* h, const double* X, long long comp_stride, long long row_vals, const double** lo,
                      const double** hi, long long* gcs, double* rlo, double* rhi, int G, cudaStream_t xs) {
  const int R = h->nranks;
  if (h->ovr_active) {  // hom2d_residual_strip: caller-supplied ghost rows
    *gcs = (long long)G * row_vals;
    *lo = h->ovr_lo;
    *hi = h->ovr_hi;
    return HOM2D_OK;
  }
  if (h->peer) {  // peer-memory halo (peer.cu): signal my X, pull the neighbours' rows of theirs
    NvtxRange nv("hom2d halo exchange (peer memory)");
    const hom2d_strip_plan_t P = plan_of(h->cfg, h->rank, R);
    const unsigned long long seq = ++h->peer_seq;
    const long long off = (const char*)X - h->ws, pf = (const char*)h->pflag - h->ws;
    // my lo neighbour's flag [1] ("from hi") and my hi neighbour's flag [0] ("from lo")
    unsigned long long* to_lo = P.has_lo ? reinterpret_cast<unsigned long long*>(h->pws_lo + pf) + 1 : nullptr;
    unsigned long long* to_hi = P.has_hi ? reinterpret_cast<unsigned long long*>(h->pws_hi + pf) + 0 : nullptr;
    int e = launch_peer_signal(to_lo, to_hi, seq, h->stream);  // after the kernels that produced X
    if (e) return fail(h, HOM2D_ERR_CUDA, "peer signal: %s", cudaGetErrorString((cudaError_t)e));
    h->launches++;
    PeerPull pp;
    pp.flag_lo = h->pflag + 0;
    pp.flag_hi = h->pflag + 1;
    pp.seq = seq;
    pp.src_lo = P.has_lo ? reinterpret_cast<const double*>(h->pws_lo + off) + (long long)(h->nrows - G) * row_vals
                         : nullptr;
    pp.src_hi = P.has_hi ? reinterpret_cast<const double*>(h->pws_hi + off) : nullptr;
    pp.src_cs = comp_stride;
    pp.dst_lo = rlo;
    pp.dst_hi = rhi;
    pp.cnt = (long long)G * row_vals;
    pp.vec = ((off | (long long)(h->nrows - G) * row_vals * 8 | comp_stride * 8 | pp.cnt * 8 |
               (long long)(uintptr_t)rlo | (long long)(uintptr_t)rhi) & 15) == 0;
    e = launch_peer_pull(pp, xs);
    if (e) return fail(h, HOM2D_ERR_CUDA, "peer pull: %s", cudaGetErrorString((cudaError_t)e));
    h->launches++;
    *gcs = pp.cnt;
    *lo = P.has_lo ? rlo : nullptr;
    *hi = P.has_hi ? rhi : nullptr;
    return HOM2D_OK;
  }
  if (R == 1 && h->self_x && !h->comm) {  // test mode: the periodic wrap rows through the ghost buffers, on xs
    const long long cnt = (long long)G * row_vals;
    for (int c = 0; c < 4; ++c) {
      CU(h, cudaMemcpyAsync(rlo + c * cnt, X + c * comp_stride + (long long)(h->nrows - G) * row_vals,
                            cnt * sizeof(double), cudaMemcpyDeviceToDevice, xs));
      CU(h, cudaMemcpyAsync(rhi + c * cnt, X + c * comp_stride, cnt * sizeof(double), cudaMemcpyDeviceToDevice, xs));
    }
    *gcs = cnt;
    *lo = rlo;
    *hi = rhi;
    return HOM2D_OK;
  }
  if (R == 1 && !h->comm) {
    *gcs = comp_stride;
    *lo = (h->cfg.bc == HOM2D_PERIODIC) ? X + (long long)(h->nrows - G) * row_vals : nullptr;
    *hi = (h->cfg.bc == HOM2D_PERIODIC) ? X : nullptr;
    return HOM2D_OK;
  }
  if (!h->comm) return fail(h, HOM2D_ERR_STATE, "strip-only handle (created without an NCCL id)");
  NvtxRange nv("hom2d halo exchange");
  const hom2d_strip_plan_t P = plan_of(h->cfg, h->rank, R);
  const long long cnt = (long long)G * row_vals;
  NC(h, ncclGroupStart());
  for (int c = 0; c < 4; ++c) {
    const double* first = X + c * comp_stride;
    const double* last = X + c * comp_stride + (long long)(h->nrows - G) * row_vals;
    if (P.has_hi) NC(h, ncclSend(last, cnt, ncclDouble, P.peer_hi, h->comm, xs));
    if (P.has_lo) NC(h, ncclSend(first, cnt, ncclDouble, P.peer_lo, h->comm, xs));
    if (P.has_lo) NC(h, ncclRecv(rlo + c * cnt, cnt, ncclDouble, P.peer_lo, h->comm, xs));
    if (P.has_hi) NC(h, ncclRecv(rhi + c * cnt, cnt, ncclDouble, P.peer_hi, h->comm, xs));
  }
  NC(h, ncclGroupEnd());
  const bool lo_ok = P.has_lo, hi_ok = P.has_hi;
  *gcs = cnt;
  *lo = lo_ok ? rlo : nullptr;
  *hi = hi_ok ? rhi : nullptr;
  return HOM2D_OK;
}

int launch_stage(hom2d* h, const StageArgs& s) {
  if (h->cfg.method == HOM2D_FV) return launch_fv_stage(h->cfg.k, s, h->stream);
  int method = h->cfg.method;
  if (method == HOM2D_DG && h->cfg.dg_overintegrate) return launch_dgoi_stage(h->cfg.k, s, h->stream);
  if (method == HOM2D_CPR && !h->cfg.cpr_chain_rule) method = HOM2D_NDG;  // flux-differentiation CPR == NDG
  return (method == HOM2D_CPR || method == HOM2D_NDG) ? launch_gll_stage(method, h->cfg.k, s, h->stream)
                                                      : launch_gl_stage(method, h->cfg.k, s, h->stream);
}

// One RK stage.  nranks == 1: one launch over the strip.  nranks > 1 (SURVEY
// 8(e) overlap): the G boundary rows of the stage input go to the neighbours on
// the exchange stream while the compute stream updates the interior rows
// [G, nrows-G) (which read no ghost row); the two boundary bands follow once the
// ghost rows have arrived.  Per-element arithmetic does not depend on the
// launch split, so the result is bitwise the single-launch one.
hom2d_status run_stage(hom2d* h, const double* q, const double* q0, double* out, double a0, double a1, double b,
                       const double* dt, unsigned long long* lam, unsigned long long* bad, double* qbar = nullptr,
                       bool lamfuse = false) {
  NvtxRange nv("hom2d stage");
  StageArgs s{};
  const long long row_vals = (long long)h->cfg.nx * h->np;
  const int G = h->G;
  const bool split = (h->nranks > 1 || h->self_x) && h->nrows > 2 * G;
  const bool async = split && (h->comm || h->self_x) && !h->ovr_active;
  const bool timed = 2 * (h->ev_used + 1) <= (int)h->ev.size();
  if (timed) cudaEventRecord(h->ev[2 * h->ev_used], h->stream);
  if (async) {  // the exchange stream may read q only once its producer has finished
    CU(h, cudaEventRecord(h->ev_in, h->stream));
    CU(h, cudaStreamWaitEvent(h->xstream, h->ev_in, 0));
  }
  hom2d_status st = exchange(h, q, h->nloc, row_vals, &s.ghost_lo, &s.ghost_hi, &s.gcs, h->glo, h->ghi, G,
                             async ? h->xstream : h->stream);
  if (st) return st;
  if (async) CU(h, cudaEventRecord(h->ev_halo, h->xstream));
  s.q = q; s.q0 = q0; s.out = out; s.nx = h->cfg.nx; s.nrows = h->nrows; s.cs = h->nloc;
  s.bcx = h->cfg.bc;
  const double dx = (h->cfg.xmax - h->cfg.xmin) / h->cfg.nx, dy = (h->cfg.ymax - h->cfg.ymin) / h->cfg.ny;
  if (h->cfg.method == HOM2D_FV) { s.rdx2 = 1.0 / dx; s.rdy2 = 1.0 / dy; }
  else { s.rdx2 = 2.0 / dx; s.rdy2 = 2.0 / dy; }
  s.a0 = a0; s.a1 = a1; s.bcoef = b; s.dt = dt; s.gamma = h->cfg.gamma;
  s.lam = lam; s.bad = bad;
  s.dec = h->cfg.record_decisions ? h->dec : nullptr;
  s.dmap = h->cfg.record_decisions ? h->dmap : nullptr;
  s.count_bot = (h->rank == 0);
  s.qbar = qbar;
  s.laml = lamfuse ? h->laml : nullptr;
  s.badl = lamfuse ? h->badl : nullptr;
  s.dtrole = dt ? h->dtrole : 0;
  s.clk = h->clock;
  s.lamdt = h->lam;
  s.cflh = h->cfg.cfl * fmin((h->cfg.xmax - h->cfg.xmin) / h->cfg.nx, (h->cfg.ymax - h->cfg.ymin) / h->cfg.ny);
  s.fv_unlimited = h->cfg.fv_unlimited;
  int e = 0;
  if (!split) {
    s.row_lo = 0; s.row_hi = h->nrows;
    e = launch_stage(h, s);
    h->launches++;
  } else {
    StageArgs in = s;  // interior rows: never read the ghost rows
    in.row_lo = G; in.row_hi = h->nrows - G;
    e = launch_stage(h, in);
    if (!e && async) e = (int)cudaStreamWaitEvent(h->stream, h->ev_halo, 0);
    // both boundary bands [0, G) and [nrows-G, nrows) in ONE launch (the second
    // band's CTAs follow the first's in the grid): one launch latency per stage
    StageArgs bd = s;
    bd.row_lo = 0; bd.row_hi = G;
    bd.row_lo2 = h->nrows - G; bd.row_hi2 = h->nrows;
    bd.no_pdl = async ? 1 : 0;  // it follows the wait on the exchange stream's event
    if (bd.dtrole == 2) bd.dtrole = 0;  // the clock is committed once (by the interior launch)
    if (!e) e = launch_stage(h, bd);
    h->launches += 2;
  }
  if (timed) cudaEventRecord(h->ev[2 * h->ev_used++ + 1], h->stream);
  if (e) return fail(h, HOM2D_ERR_CUDA, "stage kernel launch: %s", cudaGetErrorString((cudaError_t)e));
  return HOM2D_OK;
}

// HO limiter on X in place: averages (unless the stage kernel that produced X
// already wrote them, avg_done), (exchange average rows), detect + limit.
// dt != nullptr: skipped on the device when the step was clipped out (*dt == 0).
hom2d_status run_limiter(hom2d* h, double* X, const double* dt = nullptr, bool avg_done = false,
                         bool lamfuse = false) {
  NvtxRange nv("hom2d limiter");
  AuxArgs A = aux(h);
  A.dt = dt;
  if (!avg_done) {
    launch_averages(A, X, h->qbar, h->stream);
    h->launches++;
  }
  const long long ne = (long long)h->cfg.nx * h->nrows;
  const double *lo, *hi;
  long long gcs;
  hom2d_status st = exchange(h, h->qbar, ne, h->cfg.nx, &lo, &hi, &gcs, h->qblo, h->qbhi, 1, h->stream);
  if (st) return st;
  launch_limit(A, X, h->qbar, lo, hi, gcs, h->cfg.bc, h->cfg.limiter_eps, h->cfg.limiter_all_vars,
               h->cfg.limiter_characteristic, h->cfg.record_decisions ? h->dec : nullptr,
               h->cfg.record_decisions ? h->dmap : nullptr, h->stream,
               lamfuse ? LamFuse{h->laml, h->badl, h->lam, h->bad} : LamFuse());
  h->launches++;
  CU(h, cudaPeekAtLastError());
  return HOM2D_OK;
}

hom2d_status allreduce_max_lam(hom2d* h) {
  if (h->comm) NC(h, ncclAllReduce(h->lam, h->lam, 1, ncclUint64, ncclMax, h->comm, h->stream));
  return HOM2D_OK;
}

// wave-speed max of the current state -> lam[0]; mark it "fresh" for k_dt
hom2d_status refresh_lambda(hom2d* h) {
  CU(h, cudaMemsetAsync(h->lam, 0, sizeof(unsigned long long), h->stream));
  launch_lambda(aux(h), h->Qn, h->lam, nullptr, h->stream);
  h->launches++;
  CU(h, cudaPeekAtLastError());
  hom2d_status st = allreduce_max_lam(h);
  if (st) return st;
  const double one = 1.0;
  CU(h, cudaMemcpyAsync(h->clock + 3, &one, sizeof(double), cudaMemcpyHostToDevice, h->stream));
  return HOM2D_OK;
}

hom2d_status reset_clock(hom2d* h, double t0) {
  double c[4] = {t0, 0.0, 0.0, 0.0};
  CU(h, cudaMemcpyAsync(h->clock, c, sizeof(c), cudaMemcpyHostToDevice, h->stream));
  CU(h, cudaMemsetAsync(h->dec, 0, 8 * sizeof(long long), h->stream));
  if (h->dmap) CU(h, cudaMemsetAsync(h->dmap, 0, (size_t)h->cfg.nx * h->nrows * sizeof(long long), h->stream));
  CU(h, cudaMemsetAsync(h->bad, 0xff, sizeof(unsigned long long), h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  return HOM2D_OK;
}

}  // namespace

extern "C" {

hom2d_status hom2d_strip_plan(const hom2d_config* cfg, int32_t rank, int32_t nranks, hom2d_strip_plan_t* out) {
  hom2d_status st = check_cfg(cfg, nranks);
  if (st) return st;
  if (!out || rank < 0 || rank >= nranks) return HOM2D_ERR_ARG;
  *out = plan_of(*cfg, rank, nranks);
  return HOM2D_OK;
}

hom2d_status hom2d_workspace_bytes(const hom2d_config* cfg, const hom2d_dist* dist, size_t* bytes) {
  const int R = dist ? dist->nranks : 1;
  hom2d_status st = check_cfg(cfg, R);
  if (st) return st;
  if (!bytes) return HOM2D_ERR_ARG;
  *bytes = carve(nullptr, *cfg, R, nullptr);
  return HOM2D_OK;
}

hom2d_status hom2d_nccl_unique_id(void* out128) {
  if (!out128) return HOM2D_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return HOM2D_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, 128);
  return HOM2D_OK;
}

namespace {
// the allocation holding p (CUDA IPC exports whole allocations)
bool alloc_base(const void* p, char** base) {
  typedef CUresult (*fn_t)(CUdeviceptr*, size_t*, CUdeviceptr);
  static fn_t fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<fn_t>(f);
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (CUdeviceptr)(uintptr_t)p) != CUDA_SUCCESS) return false;
  *base = reinterpret_cast<char*>((uintptr_t)b);
  return true;
}
hom2d_status own_peer_id(hom2d* h, hom2d_peer_id_t* out) {
  memset(out, 0, sizeof(*out));
  char* base = nullptr;
  if (!alloc_base(h->ws, &base)) return fail(h, HOM2D_ERR_CUDA, "peer id: cuMemGetAddressRange failed");
  cudaIpcMemHandle_t mh;
  static_assert(sizeof(mh) == sizeof(out->ipc), "cudaIpcMemHandle_t size");
  CU(h, cudaIpcGetMemHandle(&mh, base));
  memcpy(out->ipc, &mh, sizeof(mh));
  out->offset = (uint64_t)(h->ws - base);
  out->rank = h->rank;
  out->device = h->device;
  return HOM2D_OK;
}
}  // namespace

hom2d_status hom2d_peer_id(hom2d* h, hom2d_peer_id_t* out) {
  GUARD(h);
  if (!out) return fail(h, HOM2D_ERR_ARG, "peer id: null pointer");
  if (!h->pflag) return fail(h, HOM2D_ERR_STATE, "peer id: a handle with nranks > 1 is needed");
  return own_peer_id(h, out);
}

hom2d_status hom2d_peer_connect(hom2d* h, const hom2d_peer_id_t* lo, const hom2d_peer_id_t* hi) {
  GUARD(h);
  if (!lo || !hi) return fail(h, HOM2D_ERR_ARG, "peer connect: null id");
  if (!h->pflag || !h->glo) return fail(h, HOM2D_ERR_STATE, "peer connect: a handle with nranks > 1 is needed");
  if (h->peer) return fail(h, HOM2D_ERR_STATE, "peer connect: already connected");
  if (h->nranks > 1 && !h->comm) return fail(h, HOM2D_ERR_STATE, "peer connect: strip-only handle (no NCCL id)");
  hom2d_peer_id_t me;
  hom2d_status st = own_peer_id(h, &me);
  if (st) return st;
  const hom2d_peer_id_t* ids[2] = {lo, hi};
  char* mapped[2] = {nullptr, nullptr};
  for (int side = 0; side < 2; ++side) {
    const hom2d_peer_id_t* id = ids[side];
    if (!memcmp(id->ipc, me.ipc, sizeof(me.ipc))) {  // this process's own allocation (self / test)
      mapped[side] = h->ws - me.offset;
    } else if (side == 1 && !memcmp(ids[0]->ipc, id->ipc, sizeof(id->ipc)) && mapped[0]) {
      mapped[1] = mapped[0];  // two ranks: both neighbours are the same peer (one mapping)
    } else {
      cudaIpcMemHandle_t mh;
      memcpy(&mh, id->ipc, sizeof(mh));
      void* p = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        for (void*& m : h->ipc_mapped)
          if (m) { cudaIpcCloseMemHandle(m); m = nullptr; }
        return fail(h, HOM2D_ERR_CUDA, "peer connect: cudaIpcOpenMemHandle (rank %d): %s", id->rank,
                    cudaGetErrorString(e));
      }
      h->ipc_mapped[side] = p;
      mapped[side] = (char*)p;
    }
  }
  h->pws_lo = mapped[0] + lo->offset;
  h->pws_hi = mapped[1] + hi->offset;
  h->peer = true;
  return HOM2D_OK;
}

hom2d_status hom2d_create(const hom2d_config* cfg, const hom2d_dist* dist, void* workspace, size_t ws_bytes,
                          hom2d** out) {
  if (!out) return HOM2D_ERR_ARG;
  *out = nullptr;
  const int R = dist ? dist->nranks : 1;
  hom2d_status st = check_cfg(cfg, R);
  if (st) return st;
  if (dist && (dist->rank < 0 || dist->rank >= R)) return HOM2D_ERR_ARG;
  if (!workspace || ((uintptr_t)workspace & 255)) return HOM2D_ERR_ARG;
  if (ws_bytes < carve(nullptr, *cfg, R, nullptr)) return HOM2D_ERR_NOMEM;
  hom2d* h = new (std::nothrow) hom2d();
  if (!h) return HOM2D_ERR_NOMEM;
  h->cfg = *cfg;
  h->rank = dist ? dist->rank : 0;
  h->nranks = R;
  if (dist) h->device = dist->device; else cudaGetDevice(&h->device);
  h->stream = dist ? (cudaStream_t)dist->cuda_stream : nullptr;
  h->np = points_per_elem(*cfg);
  h->G = cfg->method == HOM2D_FV ? 2 : 1;
  h->nrows = cfg->ny / R;
  h->row0 = h->rank * h->nrows;
  h->nloc = (long long)cfg->nx * h->nrows * h->np;
  {
    const char* ng = getenv("HOM2D_NO_GRAPH");  // A/B: eager launches instead of CUDA graphs
    h->graph_off = ng && ng[0] == '1';
    const char* nd = getenv("HOM2D_NO_DTFUSE");  // A/B: k_dt launch instead of the fused dt
    h->dtfuse = !(nd && nd[0] == '1');
    const char* gm = getenv("HOM2D_GRAPH_AFTER");  // A/B: eager steps before graph batches (default 2048)
    if (gm && *gm) h->graph_after = atoll(gm);
    const char* gb = getenv("HOM2D_GRAPH_MIN_BATCH");  // A/B: smallest graphed batch (default 64)
    if (gb && *gb) h->graph_min_batch = atoi(gb);
    pdl_refresh();
  }
  cudaError_t ce = cudaSetDevice(h->device);
  if (ce != cudaSuccess) { delete h; return HOM2D_ERR_CUDA; }
  carve(h, *cfg, R, (char*)workspace);
  if (cudaMallocHost(&h->t_host, 8 * sizeof(double)) != cudaSuccess) { delete h; return HOM2D_ERR_CUDA; }
  const int sxm = self_exchange_env(*cfg, R);
  h->self_x = sxm != 0;
  h->self_nccl = sxm == 2;
  h->ws = (char*)workspace;
  if (h->pflag && cudaMemset(h->pflag, 0, 2 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaFreeHost(h->t_host);
    delete h;
    return HOM2D_ERR_CUDA;
  }
  if (sxm == 3) {  // peer-memory halo with itself as both neighbours
    h->peer = true;
    h->pws_lo = h->pws_hi = h->ws;
  }
  if ((R > 1 && dist->nccl_id) || h->self_x) {  // (no id: strip-only handle, see hom2d_residual_strip)
    if (R > 1 || h->self_nccl) {
      ncclUniqueId id;
      if (R > 1) memcpy(&id, dist->nccl_id, sizeof(id));
      if ((R == 1 && ncclGetUniqueId(&id) != ncclSuccess) || ncclCommInitRank(&h->comm, R, id, h->rank) != ncclSuccess) {
        cudaFreeHost(h->t_host);
        delete h;
        return HOM2D_ERR_NCCL;
      }
    }
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (cudaStreamCreateWithPriority(&h->xstream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming) != cudaSuccess) {
      hom2d_destroy(h);
      return HOM2D_ERR_CUDA;
    }
  }
  cudaMemsetAsync(h->lam, 0, 4 * sizeof(unsigned long long), h->stream);
  if (reset_clock(h, 0.0)) { hom2d_destroy(h); return HOM2D_ERR_CUDA; }
  *out = h;
  return HOM2D_OK;
}

hom2d_status hom2d_local_extent(const hom2d* h, int32_t* row0, int32_t* nrows, int64_t* n_values) {
  if (!h) return HOM2D_ERR_ARG;
  if (row0) *row0 = h->row0;
  if (nrows) *nrows = h->nrows;
  if (n_values) *n_values = 4 * h->nloc;
  return HOM2D_OK;
}

hom2d_status hom2d_set_state(hom2d* h, const double* q, int64_t n_values, int32_t on_device, double t0) {
  GUARD(h);
  if (!q || n_values != 4 * h->nloc) return fail(h, HOM2D_ERR_ARG, "set_state: expected %lld values", 4 * h->nloc);
  CU(h, cudaMemcpyAsync(h->Qn, q, n_values * sizeof(double), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                        h->stream));
  hom2d_status st = reset_clock(h, t0);
  if (st) return st;
  st = refresh_lambda(h);
  if (st) return st;
  CU(h, cudaStreamSynchronize(h->stream));
  return HOM2D_OK;
}

hom2d_status hom2d_get_state(hom2d* h, double* q, int64_t n_values, int32_t on_device) {
  GUARD(h);
  if (!q || n_values != 4 * h->nloc) return fail(h, HOM2D_ERR_ARG, "get_state: expected %lld values", 4 * h->nloc);
  CU(h, cudaMemcpyAsync(q, h->Qn, n_values * sizeof(double), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                        h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  return HOM2D_OK;
}

hom2d_status hom2d_init_case(hom2d* h, int32_t case_id) {
  GUARD(h);
  if (case_id != HOM2D_CASE_VORTEX && case_id != HOM2D_CASE_SHOCK) return fail(h, HOM2D_ERR_ARG, "unknown case %d", case_id);
  launch_init_case(aux(h), case_id, h->Qn, h->stream);
  h->launches++;
  CU(h, cudaPeekAtLastError());
  if (h->cfg.limiter && h->cfg.method != HOM2D_FV) {
    hom2d_status st = run_limiter(h, h->Qn);
    if (st) return st;
  }
  hom2d_status st = reset_clock(h, 0.0);
  if (st) return st;
  st = refresh_lambda(h);
  if (st) return st;
  CU(h, cudaStreamSynchronize(h->stream));
  return HOM2D_OK;
}

hom2d_status hom2d_residual(hom2d* h, const double* q_dev, double* r_dev) {
  GUARD(h);
  if (!q_dev || !r_dev) return fail(h, HOM2D_ERR_ARG, "residual: null pointer");
  // stage kernels stream from the handle's own (guarded, aligned) arrays
  CU(h, cudaMemcpyAsync(h->Q1, q_dev, 4 * h->nloc * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  hom2d_status st = run_stage(h, h->Q1, nullptr, h->Q2, 0.0, 0.0, 1.0, nullptr, nullptr, nullptr);
  if (st) return st;
  CU(h, cudaMemcpyAsync(r_dev, h->Q2, 4 * h->nloc * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  if (st) return st;
  CU(h, cudaStreamSynchronize(h->stream));
  return HOM2D_OK;
}

hom2d_status hom2d_residual_strip(hom2d* h, const double* q_dev, const double* ghost_lo_dev,
                                  const double* ghost_hi_dev, double* r_dev) {
  GUARD(h);
  if (!q_dev || !r_dev) return fail(h, HOM2D_ERR_ARG, "residual_strip: null pointer");
  const long long gvals = 4LL * h->G * h->cfg.nx * h->np;
  if (!h->glo || !h->ghi) return fail(h, HOM2D_ERR_STATE, "residual_strip needs a handle with nranks > 1");
  CU(h, cudaMemcpyAsync(h->Q1, q_dev, 4 * h->nloc * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  if (ghost_lo_dev)
    CU(h, cudaMemcpyAsync(h->glo, ghost_lo_dev, gvals * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  if (ghost_hi_dev)
    CU(h, cudaMemcpyAsync(h->ghi, ghost_hi_dev, gvals * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  h->ovr_active = true;
  h->ovr_lo = ghost_lo_dev ? h->glo : nullptr;
  h->ovr_hi = ghost_hi_dev ? h->ghi : nullptr;
  hom2d_status st = run_stage(h, h->Q1, nullptr, h->Q2, 0.0, 0.0, 1.0, nullptr, nullptr, nullptr);
  h->ovr_active = false;
  if (st) return st;
  CU(h, cudaMemcpyAsync(r_dev, h->Q2, 4 * h->nloc * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  return HOM2D_OK;
}

hom2d_status hom2d_limit(hom2d* h) {
  GUARD(h);
  if (h->cfg.method == HOM2D_FV) return fail(h, HOM2D_ERR_ARG, "limit: HO methods only");
  hom2d_status st = run_limiter(h, h->Qn);
  if (st) return st;
  st = refresh_lambda(h);
  if (st) return st;
  CU(h, cudaStreamSynchronize(h->stream));
  return HOM2D_OK;
}

hom2d_status hom2d_compute_dt(hom2d* h, double* dt) {
  GUARD(h);
  if (!dt) return HOM2D_ERR_ARG;
  hom2d_status st = refresh_lambda(h);
  if (st) return st;
  unsigned long long bits;
  CU(h, cudaMemcpyAsync(&bits, h->lam, sizeof(bits), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  double l;
  memcpy(&l, &bits, 8);
  if (!(l > 0.0 && l < HUGE_VAL))  // NaN / inf wave speed: a non-physical state (the reduction keeps NaN)
    return fail(h, HOM2D_ERR_NONPHYSICAL, "compute_dt: max wave speed %g", l);
  const double dx = (h->cfg.xmax - h->cfg.xmin) / h->cfg.nx, dy = (h->cfg.ymax - h->cfg.ymin) / h->cfg.ny;
  *dt = h->cfg.cfl * fmin(dx, dy) / l;
  return HOM2D_OK;
}

}  // extern "C"

namespace {

// one SSP-RK3 step on h->stream: dt (device), three stages, the
// limiter (if on) and the lambda allreduce (nranks > 1)
hom2d_status enqueue_step(hom2d* h) {
  const double dx = (h->cfg.xmax - h->cfg.xmin) / h->cfg.nx, dy = (h->cfg.ymax - h->cfg.ymin) / h->cfg.ny;
  const bool lim = h->cfg.limiter && h->cfg.method != HOM2D_FV;
  hom2d_status st;
  // dt of the step: computed by every CTA of stage 1 and committed by stage 2
  // (StageArgs::dtrole; no k_dt launch in the chain), or by k_dt (HOM2D_NO_DTFUSE=1)
  if (!h->dtfuse) {
    launch_dt(h->clock, h->lam, h->cfg.cfl, fmin(dx, dy), h->stream);
    h->launches++;
  }
  const double* dt = h->clock + 1;
  // limiter runs: the stage kernels also write the element averages of their output;
  // limiter_per_step (f3): only after stage 3
  const bool lim12 = lim && !h->cfg.limiter_per_step;
  double* qb = lim ? h->qbar : nullptr;
  double* qb12 = lim12 ? h->qbar : nullptr;
  h->dtrole = h->dtfuse ? 1 : 0;
  if ((st = run_stage(h, h->Qn, nullptr, h->Q1, 0.0, 1.0, 1.0, dt, nullptr, nullptr, qb12))) return st;
  h->dtrole = h->dtfuse ? 2 : 0;
  if (lim12 && (st = run_limiter(h, h->Q1, dt, true))) return st;
  if ((st = run_stage(h, h->Q1, h->Qn, h->Q2, 0.75, 0.25, 0.25, dt, nullptr, nullptr, qb12))) return st;
  h->dtrole = 0;
  if (lim12 && (st = run_limiter(h, h->Q2, dt, true))) return st;
  if (!lim) {
    if ((st = run_stage(h, h->Q2, h->Qn, h->Qn, 1.0 / 3.0, 2.0 / 3.0, 2.0 / 3.0, dt, h->lam, h->bad))) return st;
  } else {
    // the dt wave speed / non-physical check of the LIMITED state: unmarked elements
    // from the stage-3 epilogue (per line), rebuilt elements in k_limit -- no pass
    if ((st = run_stage(h, h->Q2, h->Qn, h->Qn, 1.0 / 3.0, 2.0 / 3.0, 2.0 / 3.0, dt, nullptr, nullptr, qb, true)))
      return st;
    if ((st = run_limiter(h, h->Qn, dt, true, true))) return st;
  }
  return allreduce_max_lam(h);
}

// n steps through cached CUDA graphs of 2^i steps (binary decomposition of n)
hom2d_status graph_steps(hom2d* h, int n) {
  if (!h->gstream) {
    CU(h, cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking));
    CU(h, cudaEventCreateWithFlags(&h->gev_a, cudaEventDisableTiming));
    CU(h, cudaEventCreateWithFlags(&h->gev_b, cudaEventDisableTiming));
  }
  CU(h, cudaEventRecord(h->gev_a, h->stream));
  CU(h, cudaStreamWaitEvent(h->gstream, h->gev_a, 0));
  for (int i = 6; i >= 0; --i) {
    if (!(n & (1 << i))) continue;
    if (!h->gexec[i]) {  // capture 2^i steps once
      cudaStream_t user = h->stream;
      const long long l0 = h->launches;
      h->stream = h->gstream;
      CU(h, cudaStreamBeginCapture(h->gstream, cudaStreamCaptureModeThreadLocal));
      hom2d_status st = HOM2D_OK;
      for (int k = 0; k < (1 << i) && !st; ++k) st = enqueue_step(h);
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(h->gstream, &g);
      h->stream = user;
      h->glaunch[i] = h->launches - l0;
      h->launches = l0;
      if (st) { if (g) cudaGraphDestroy(g); return st; }
      CU(h, ce);
      const cudaError_t ie = cudaGraphInstantiate(&h->gexec[i], g, 0);
      cudaGraphDestroy(g);
      CU(h, ie);
    }
    CU(h, cudaGraphLaunch(h->gexec[i], h->gstream));
    h->launches += h->glaunch[i];
  }
  CU(h, cudaEventRecord(h->gev_b, h->gstream));
  CU(h, cudaStreamWaitEvent(h->stream, h->gev_b, 0));
  return HOM2D_OK;
}

}  // namespace

extern "C" hom2d_status hom2d_step(hom2d* h, int32_t max_steps, double t_end, double* t_out, int64_t* steps_out) {
  GUARD(h);
  NvtxRange nv("hom2d_step");
  if (max_steps < 0) return fail(h, HOM2D_ERR_ARG, "max_steps < 0");
  // graphs: single GPU (NCCL calls stay eagerly enqueued), no per-stage timing events
  const bool graphs = !h->graph_off && !h->comm && !h->self_x && h->ev.empty();
  h->t_host[5] = t_end;
  CU(h, cudaMemcpyAsync(h->clock + 4, h->t_host + 5, sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CU(h, cudaMemcpyAsync(h->t_host, h->clock, 4 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  const double steps0 = h->t_host[2];
  int done = 0;
  hom2d_status st = HOM2D_OK;
  while (done < max_steps) {
    int batch = (max_steps - done) < 64 ? (max_steps - done) : 64;
    // near t_end: no more steps than the clock needs (+1; clipped-out steps are no-ops)
    if (std::isfinite(t_end) && h->t_host[1] > 0.0) {
      const double est = std::ceil((t_end - h->t_host[0]) / h->t_host[1]) + 1.0;
      if (est < batch) batch = est < 1.0 ? 1 : (int)est;
    } else if (std::isfinite(t_end)) {
      // no dt yet (fresh handle): one step first, so the next batch can be sized
      // from it -- otherwise a short run to t_end launches up to 63 clipped-out
      // (no-op) steps, ~10 us each on the paper's grids
      batch = 1;
    }
    // graphs pay for their capture only on long runs: 64-step batches once the
    // handle has marched graph_after steps eagerly
    if (graphs && batch >= h->graph_min_batch && h->eager_steps >= h->graph_after) {
      if ((st = graph_steps(h, batch))) return st;
    } else {
      for (int s = 0; s < batch; ++s)
        if ((st = enqueue_step(h))) return st;
      h->eager_steps += batch;
    }
    done += batch;
    CU(h, cudaPeekAtLastError());
    // every rank leaves the loop in the same batch: the flag is min-reduced over
    // the ranks (bad[1]) before the host looks at it; the local point (bad[0])
    // names the element when this rank found it
    if (h->comm)
      NC(h, ncclAllReduce(h->bad, h->bad + 1, 1, ncclUint64, ncclMin, h->comm, h->stream));
    else
      CU(h, cudaMemcpyAsync(h->bad + 1, h->bad, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, h->stream));
    CU(h, cudaMemcpyAsync(h->t_host, h->clock, 4 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaMemcpyAsync(h->t_host + 6, h->bad, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    unsigned long long badv, bad_any;
    memcpy(&badv, h->t_host + 6, 8);
    memcpy(&bad_any, h->t_host + 7, 8);
    if (bad_any != ~0ull) {
      if (t_out) *t_out = h->t_host[0];
      if (steps_out) *steps_out = (int64_t)(h->t_host[2] - steps0);
      if (badv == ~0ull)
        return fail(h, HOM2D_ERR_NONPHYSICAL, "non-physical state on another rank, t=%.17g", h->t_host[0]);
      const long long m = (long long)(badv / h->np);
      return fail(h, HOM2D_ERR_NONPHYSICAL,
                  "non-physical state at element (i=%lld, j=%lld), point %lld, rank %d, t=%.17g", m % h->cfg.nx,
                  m / h->cfg.nx + h->row0, (long long)(badv % h->np), h->rank, h->t_host[0]);
    }
    if (!(h->t_host[0] < t_end)) break;
  }
  if (t_out) *t_out = h->t_host[0];
  if (steps_out) *steps_out = (int64_t)(h->t_host[2] - steps0);
  return HOM2D_OK;
}

extern "C" {

hom2d_status hom2d_error(hom2d* h, int32_t case_id, int32_t var, double* l1, double* l2, double* linf) {
  GUARD(h);
  NvtxRange nv("hom2d_error");
  if (case_id != HOM2D_CASE_VORTEX) return fail(h, HOM2D_ERR_ARG, "error: exact solution only for the vortex");
  if (var < 0 || var > 3) return fail(h, HOM2D_ERR_ARG, "error: var must be 0..3");
  int nb;
  if (h->cfg.method == HOM2D_FV && h->cfg.fv_error_recon) {
    // the reconstruction reads one cell row beyond the strip: the FV ghost rows
    const double *lo, *hi;
    long long gcs;
    hom2d_status st = exchange(h, h->Qn, h->nloc, h->cfg.nx, &lo, &hi, &gcs, h->glo, h->ghi, 2, h->stream);
    if (st) return st;
    nb = launch_error_fv_recon(aux(h), h->Qn, lo, hi, gcs, h->cfg.bc, h->cfg.fv_unlimited, var, h->clock, h->part,
                               h->max_part, h->stream);
  } else {
    nb = launch_error_partials(aux(h), h->Qn, var, h->clock, h->part, h->max_part, h->stream);
  }
  launch_error_final(h->part, nb, h->err3, h->stream);
  h->launches += 2;
  CU(h, cudaPeekAtLastError());
  if (h->comm) {
    NC(h, ncclAllReduce(h->err3, h->err3, 2, ncclDouble, ncclSum, h->comm, h->stream));
    NC(h, ncclAllReduce(h->err3 + 2, h->err3 + 2, 1, ncclDouble, ncclMax, h->comm, h->stream));
  }
  double r[3];
  CU(h, cudaMemcpyAsync(r, h->err3, sizeof(r), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  const double ne = (double)h->cfg.nx * h->cfg.ny;
  if (l1) *l1 = r[0] / ne;
  if (l2) *l2 = sqrt(r[1] / ne);
  if (linf) *linf = r[2];
  return HOM2D_OK;
}

hom2d_status hom2d_time(const hom2d* h, double* t) {
  if (!h || !t) return HOM2D_ERR_ARG;
  if (h->poisoned) return HOM2D_ERR_STATE;
  if (cudaMemcpyAsync(h->t_host, h->clock, sizeof(double), cudaMemcpyDeviceToHost, h->stream) != cudaSuccess)
    return HOM2D_ERR_CUDA;
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return HOM2D_ERR_CUDA;
  *t = h->t_host[0];
  return HOM2D_OK;
}

hom2d_status hom2d_decisions(hom2d* h, int64_t* counts8) {
  GUARD(h);
  if (!counts8) return HOM2D_ERR_ARG;
  CU(h, cudaMemcpyAsync(counts8, h->dec, 8 * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  if (h->comm) {  // sum over ranks through the device scratch
    NC(h, ncclAllReduce(h->dec, h->part, 8, ncclInt64, ncclSum, h->comm, h->stream));
    CU(h, cudaMemcpyAsync(counts8, h->part, 8 * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
  }
  return HOM2D_OK;
}

hom2d_status hom2d_decision_map(hom2d* h, int64_t* out, int64_t n) {
  GUARD(h);
  if (!out) return HOM2D_ERR_ARG;
  if (!h->dmap) return fail(h, HOM2D_ERR_STATE, "decision_map needs record_decisions = 1 and one rank");
  if (n != (int64_t)h->cfg.nx * h->nrows) return fail(h, HOM2D_ERR_ARG, "decision_map: expected %lld entries",
                                                     (long long)h->cfg.nx * h->nrows);
  CU(h, cudaMemcpyAsync(out, h->dmap, n * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  return HOM2D_OK;
}

int64_t hom2d_launch_count(const hom2d* h) { return h ? h->launches : 0; }

hom2d_status hom2d_stage_timing(hom2d* h, int32_t max_launches) {
  GUARD(h);
  if (max_launches < 0) return HOM2D_ERR_ARG;
  CU(h, cudaStreamSynchronize(h->stream));
  for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
  h->ev.clear();
  h->ev_used = 0;
  for (int i = 0; i < 2 * max_launches; ++i) {
    cudaEvent_t e;
    CU(h, cudaEventCreate(&e));
    h->ev.push_back(e);
  }
  return HOM2D_OK;
}

hom2d_status hom2d_stage_time(hom2d* h, double* total_ms, int64_t* n_launches) {
  GUARD(h);
  CU(h, cudaStreamSynchronize(h->stream));
  double tot = 0.0;
  for (int i = 0; i < h->ev_used; ++i) {
    float ms = 0.f;
    CU(h, cudaEventElapsedTime(&ms, h->ev[2 * i], h->ev[2 * i + 1]));
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (n_launches) *n_launches = h->ev_used;
  h->ev_used = 0;
  return HOM2D_OK;
}

const char* hom2d_last_error(const hom2d* h) { return h ? h->msg : "null handle"; }

void hom2d_destroy(hom2d* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream); else cudaDeviceSynchronize();
  if (h->xstream) cudaStreamSynchronize(h->xstream);
  for (void*& m : h->ipc_mapped)
    if (m) { cudaIpcCloseMemHandle(m); m = nullptr; }
  for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
  if (h->xstream) cudaStreamSynchronize(h->xstream);
  if (h->gstream) cudaStreamSynchronize(h->gstream);
  for (cudaGraphExec_t& g : h->gexec)
    if (g) cudaGraphExecDestroy(g);
  if (h->gev_a) cudaEventDestroy(h->gev_a);
  if (h->gev_b) cudaEventDestroy(h->gev_b);
  if (h->gstream) cudaStreamDestroy(h->gstream);
  if (h->comm) ncclCommDestroy(h->comm);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_halo) cudaEventDestroy(h->ev_halo);
  if (h->xstream) cudaStreamDestroy(h->xstream);
  if (h->t_host) cudaFreeHost(h->t_host);
  delete h;
}

}  // extern "C"
