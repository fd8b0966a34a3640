/*
 * hom2d.h -- C ABI of libhom2d.so, the B200 (sm_100a) implementation of the
 * data-parallel hot path of Zimmerman, Regele & Wie, "A Comparative Study of 2D
 * Numerical Methods with GPU Computing" (arXiv 1709.01619): one explicit SSP-RK3
 * step of the 2-D Euler semi-discretisation on a uniform quadrilateral grid, for
 * CPR, DG, NDG, SD and MUSCL-FV.  "P:<line>" cites PAPER.md.
 *
 * The calls follow the paper's statement of the problem: a mesh and
 * an initial state go in, then the method, order and CFL are fixed, the solution
 * is marched and the error is queried.
 *
 * DATA LAYOUT (every array argument, host or device): canonical SoA fp64,
 *   Q[c*(Ne*np) + m*np + p],  c in {0: rho, 1: rho u, 2: rho v, 3: e}  (Eq. (3))
 *   element m = j*nx + i (row-major; i = x index, j = y index, local strip rows),
 *   point   p = b*n + a   (a = xi index fastest), n = k+1, np = n*n; FV: np = 1.
 * Solution points: GLL (CPR, NDG) or Gauss-Legendre (DG, SD) nodes mapped
 * affinely to each element (Fig. 1).  "SoA" follows P:399-406.
 *
 * STREAM / ERRORS: every call is ordered on the stream given at create time
 * (NULL = legacy default stream).  Every call returns a status; none aborts.
 * After HOM2D_ERR_CUDA or HOM2D_ERR_NCCL the handle is poisoned and later calls
 * return HOM2D_ERR_STATE.  hom2d_last_error() gives a message.
 *
 * OWNERSHIP: the caller owns the config structs (copied at create), every host
 * array, and the device workspace (must outlive the handle).  The handle owns
 * the sub-allocation of that workspace and, when nranks > 1, the NCCL
 * communicator it creates from the caller's unique id.  It never frees caller
 * memory.
 *
 * MULTI-GPU (SPMD): with nranks > 1 the grid is partitioned into contiguous
 * y-strips (rank r owns element rows [r*ny/G, (r+1)*ny/G)); every rank calls
 * every function with the same arguments; arrays passed to set/get_state are
 * the LOCAL strip in the layout above.  Boundary element rows are exchanged with
 * ncclSend/ncclRecv once per RK stage (or pulled from the neighbours' memory
 * after hom2d_peer_connect); the dt wave-speed max and the error sums are
 * ncclAllReduce'd.  ny % nranks == 0 is required.
 */
#ifndef HOM2D_H
#define HOM2D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hom2d hom2d; /* opaque handle */

typedef enum {
  HOM2D_OK = 0,
  HOM2D_ERR_ARG = 1,          /* bad pointer / enum / size */
  HOM2D_ERR_MESH = 2,         /* nx, ny < 2, empty box, ny % nranks != 0 */
  HOM2D_ERR_ORDER = 3,        /* HO k outside [1,4]; FV k outside [1,2] */
  HOM2D_ERR_NONPHYSICAL = 4,  /* rho <= 0, p <= 0 or non-finite after a step */
  HOM2D_ERR_CUDA = 5,
  HOM2D_ERR_NCCL = 6,
  HOM2D_ERR_NOMEM = 7,        /* workspace too small */
  HOM2D_ERR_STATE = 8         /* poisoned handle */
} hom2d_status;

enum { HOM2D_FV = 0, HOM2D_CPR = 1, HOM2D_DG = 2, HOM2D_NDG = 3, HOM2D_SD = 4 };
enum { HOM2D_PERIODIC = 0, HOM2D_TRANSMISSIVE = 1 };
enum { HOM2D_CASE_VORTEX = 0, HOM2D_CASE_SHOCK = 1 };

typedef struct {
  int32_t nx, ny;             /* GLOBAL element (FV: cell) counts, >= 2 */
  double xmin, xmax, ymin, ymax;
  int32_t bc;                 /* HOM2D_PERIODIC | HOM2D_TRANSMISSIVE (all four sides) */
  int32_t method;             /* HOM2D_FV .. HOM2D_SD */
  int32_t k;                  /* HO: degree 1..4 (P^k); FV: 1 = MUSCL-2, 2 = MUSCL-3 */
  double gamma;               /* ratio of specific heats (paper silent; 1.4) */
  double cfl;                 /* Eq. (36): dt = cfl*min(dx,dy)/max(max(|u|,|v|)+c) */
  int32_t limiter;            /* HO: 1 = minmod detect + slope-limit after every stage */
  double limiter_eps;         /* detection threshold, P:357 (1e-3) */
  int32_t cpr_chain_rule;     /* CPR: 1 = chain-rule divergence; 0 = flux differentiation */
  int32_t record_decisions;   /* 1 = count branch decisions (minmod outcomes, marks); slower */
  /* Method variants where the paper is silent (0 = the DESIGN.md reading):   */
  int32_t limiter_per_step;   /* HO: 1 = limit once per SSP-RK3 step (after stage 3) instead of after
                                 every stage ("The updated solution is interpolated..."; Q13) */
  int32_t limiter_all_vars;   /* HO: 1 = trouble detection on all four conserved components instead of
                                 density only (Alg. 10 P:802-836 names no variable; Q12) */
  int32_t fv_unlimited;       /* FV: 1 = unlimited kappa-scheme (kappa = 0 for k = 1, 1/3 for k = 2),
                                 i.e. MUSCL without the minmod of P:346-351 (Q10) */
  int32_t limiter_characteristic; /* HO: 1 = the Eq. (35) slopes limited per characteristic
                                 field of the element average (Cockburn-Shu) instead of per
                                 conserved component (Q12) */
  int32_t fv_error_recon;     /* FV: 1 = hom2d_error measures the reconstructed solution ("For P^2 FV,
                                 the error was computed by reconstructing the solution along element
                                 faces, and then using a quadrature rule"; DESIGN R22): per
                                 cell the quadratic through the scheme's MUSCL face states with the cell
                                 mean, per direction, summed, against the exact solution at the 3x3
                                 Gauss-Legendre points; 0 = cell value vs exact cell average */
  int32_t dg_overintegrate;   /* DG: 1 = the volume and surface integrals of the weak form (Eq. (19),
                                 P:240-254) by (k+2)-point Gauss-Legendre over-integration (SPEC's
                                 alternative; DESIGN f3) instead of the n-point collocation of Eq. (20)
                                 (the default); a separate, slower stage kernel */
} hom2d_config;

typedef struct {
  int32_t rank, nranks;       /* 0, 1 for a single GPU */
  int32_t device;             /* CUDA device ordinal of this rank */
  const void* nccl_id;        /* nranks > 1: 128-byte ncclUniqueId from hom2d_nccl_unique_id on rank 0 */
  void* cuda_stream;          /* cudaStream_t, borrowed; NULL = default stream */
} hom2d_dist;

/* Host-only (no CUDA): the y-strip partition of rank `rank` of `nranks` and its
 * per-stage halo exchange plan.  Rows are element (FV: cell) rows.  The ghost
 * rows below the strip come from `peer_lo` (its last `ghost_rows` rows), the
 * ghost rows above from `peer_hi` (its first `ghost_rows` rows); has_lo/has_hi
 * = 0 at a physical transmissive boundary (no exchange).  row_values = values
 * of one row of one component (nx * points per element). */
typedef struct {
  int32_t row0, nrows, ghost_rows;
  int32_t peer_lo, peer_hi, has_lo, has_hi;
  int64_t row_values;
} hom2d_strip_plan_t;
hom2d_status hom2d_strip_plan(const hom2d_config* cfg, int32_t rank, int32_t nranks, hom2d_strip_plan_t* out);

/* Bytes of device workspace hom2d_create needs for this config/partition. */
hom2d_status hom2d_workspace_bytes(const hom2d_config* cfg, const hom2d_dist* dist, size_t* bytes);

/* Fill out[128] with a fresh ncclUniqueId (call on rank 0, broadcast the bytes). */
hom2d_status hom2d_nccl_unique_id(void* out128);

/* Peer-memory halo (SURVEY 8(e) "Stretch" / 8(f) f4: the strip halo by device
 * loads from the neighbours' memory over NVLink instead of NCCL send/recv; the
 * per-stage exchange of P:866-874's explicit scheme is the same data).  Every
 * rank exports its workspace allocation (CUDA IPC handle + the workspace's
 * offset in it) with hom2d_peer_id, the ids are exchanged by the caller (e.g.
 * torch.distributed all_gather), and each rank calls hom2d_peer_connect with
 * the ids of its strip neighbours (hom2d_strip_plan peer_lo / peer_hi; an id of
 * this process's own allocation is used without a mapping).  From then on every
 * halo exchange is: a signal kernel that publishes a sequence number into each
 * neighbour's flag after the kernels that produced the exchanged array, and a
 * pull kernel on the exchange stream that waits for both neighbours' numbers and
 * copies their boundary rows into the local ghost buffers (traps after 60 s if a
 * neighbour never signals).  NCCL still carries the allreduces (dt, errors).
 * Both: handles with nranks > 1 created with an NCCL id, the same config on
 * every rank; HOM2D_ERR_STATE otherwise, HOM2D_ERR_CUDA if a mapping fails.
 * The id is plain bytes (copyable between processes of one node).  A
 * neighbour may read this rank's rows until it returns from its own last
 * hom2d_step / hom2d_limit / hom2d_error: every rank must have returned from
 * those (e.g. a host barrier) before any rank destroys its handle and frees its
 * workspace (the Python binding's close() does the barrier). */
typedef struct {
  uint8_t ipc[64];            /* cudaIpcMemHandle_t of the allocation holding the workspace */
  uint64_t offset;            /* workspace start within that allocation (bytes) */
  int32_t rank, device;       /* informational */
} hom2d_peer_id_t;
hom2d_status hom2d_peer_id(hom2d* h, hom2d_peer_id_t* out);
hom2d_status hom2d_peer_connect(hom2d* h, const hom2d_peer_id_t* lo, const hom2d_peer_id_t* hi);

/* Create a solver.  dist == NULL means one GPU (current device, default stream).
 * workspace: caller-owned device memory of >= hom2d_workspace_bytes, 256-B aligned. */
hom2d_status hom2d_create(const hom2d_config* cfg, const hom2d_dist* dist, void* workspace,
                          size_t ws_bytes, hom2d** out);

/* Local strip: first global element row, row count, and number of fp64 values of
 * the local state array (4 * nx * nrows * np). */
hom2d_status hom2d_local_extent(const hom2d* h, int32_t* row0, int32_t* nrows, int64_t* n_values);

/* Copy a state in (canonical layout, local strip).  on_device = 1: q is a device
 * pointer; 0: host pointer (synchronous copy).  Resets t to t0. */
hom2d_status hom2d_set_state(hom2d* h, const double* q, int64_t n_values, int32_t on_device, double t0);
hom2d_status hom2d_get_state(hom2d* h, double* q, int64_t n_values, int32_t on_device);

/* Closed-form initial data at t = 0 (P:897-913 vortex; P:1043-1047 shock tube):
 * HO pointwise at the solution points; FV 8x8 Gauss-Legendre cell averages.
 * With the limiter on (HO) the limiter is applied once to the initial data. */
hom2d_status hom2d_init_case(hom2d* h, int32_t case_id);

/* r = R(q), the spatial residual dq/dt of one RK stage (tests; device pointers). */
hom2d_status hom2d_residual(hom2d* h, const double* q_dev, double* r_dev);

/* Residual of the local strip with caller-supplied neighbour rows (device
 * pointers, layout [4][ghost_rows][nx * np], NULL = physical transmissive
 * boundary): exactly the kernel path a multi-GPU stage takes after its halo
 * exchange.  Needs nranks > 1; such a handle may be created WITHOUT an NCCL id
 * ("strip-only": collectives are then skipped), which lets one GPU check the
 * strip decomposition against the whole-grid residual. */
hom2d_status hom2d_residual_strip(hom2d* h, const double* q_dev, const double* ghost_lo_dev,
                                  const double* ghost_hi_dev, double* r_dev);

/* Apply the HO limiter (Eq. (35), Algs. 9-11) in place to the current state. */
hom2d_status hom2d_limit(hom2d* h);

/* Global dt of Eq. (36) for the current state (not clipped). */
hom2d_status hom2d_compute_dt(hom2d* h, double* dt);

/* March with SSP-RK3 until *steps_out == max_steps or t == t_end (last dt
 * clipped).  dt is recomputed from the state every step.  Syncs the host once
 * per batch of up to 64 steps.  Returns HOM2D_ERR_NONPHYSICAL if a bad state
 * appeared.  Single GPU, long runs (after 256 eager steps on the handle): full
 * 64-step batches replay a cached CUDA graph (captured once on an internal
 * stream, fenced to the handle's stream by events; environment HOM2D_NO_GRAPH=1
 * or per-stage timing keep eager launches). */
hom2d_status hom2d_step(hom2d* h, int32_t max_steps, double t_end, double* t_out, int64_t* steps_out);

/* Error of component var (0..3) against the exact vortex at the current t
 * (P:878-879): HO: quadrature-weighted pointwise error at the solution
 * points, L2 = sqrt(sum_m sum_ab w_a w_b/4 d^2 / Ne) (reproduces Tables 2-3);
 * FV: cell value vs exact 8x8-GL cell average.  Global (allreduced) values. */
hom2d_status hom2d_error(hom2d* h, int32_t case_id, int32_t var, double* l1, double* l2, double* linf);

hom2d_status hom2d_time(const hom2d* h, double* t);

/* Branch-decision counters accumulated since create/set_state (record_decisions
 * = 1), counts8[8]: [0] limiter marks (element-stage), [1] minmod -> 0,
 * [2] minmod -> first argument, [3] minmod -> second argument (MUSCL, per face
 * side and component, each face once), [4] minmod ties (an argument or their
 * difference within 1e-12 of the switch point; not counted in 1-3), [5-7] 0. */
hom2d_status hom2d_decisions(hom2d* h, int64_t* counts8);

/* Per-element decision map accumulated since create/set_state/init_case
 * (record_decisions = 1, nranks == 1; SURVEY C12 "per-element dumps"): host
 * array out[n], n = nx * ny, element m = j*nx + i.
 *   HO limiter runs: out[m] = number of limiter passes (Alg. 10-11)
 *     that marked element m.
 *   FV (MUSCL + minmod): the outcomes of the minmods that limit cell
 *     m's own slopes (both directions, all components, each face side once, as
 *     in counts8[1..4]), packed as  sum over outcomes of 1 << (16 * slot),
 *     slot 0 -> 0, 1 -> first argument, 2 -> second argument, 3 -> tie.  A
 *     reconstruction of a ghost cell counts for the cell it copies (periodic
 *     wrap / transmissive clamp).
 * HOM2D_ERR_STATE without record_decisions or with nranks > 1. */
hom2d_status hom2d_decision_map(hom2d* h, int64_t* out, int64_t n);

/* Kernel launches issued by this handle since create (bench accounting). */
int64_t hom2d_launch_count(const hom2d* h);

/* Per-launch CUDA-event timing of the RK-stage kernels on the handle's stream
 * (bench accounting).  max_launches > 0 enables it and preallocates that many
 * event pairs (later launches are not timed); 0 disables it. */
hom2d_status hom2d_stage_timing(hom2d* h, int32_t max_launches);
/* Synchronises the stream, returns the summed duration (ms) and the number of
 * timed stage launches since the last call, and resets the accumulator. */
hom2d_status hom2d_stage_time(hom2d* h, double* total_ms, int64_t* n_launches);

const char* hom2d_last_error(const hom2d* h);
void hom2d_destroy(hom2d* h);

#ifdef __cplusplus
}
#endif
#endif /* HOM2D_H */
