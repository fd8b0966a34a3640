// gll_stage.cu -- fused RK-stage kernel of the methods whose solution points are
// Gauss-Lobatto nodes coinciding with the flux points: CPR (chain rule,
// Radau/g_DG correction, Algs. 7-8 P:684-767) and NDG (D[F] + lift,
// Eqs. (24)-(29) P:300-318).  "The operations to compute the flux derivative are
// contained in one GPU kernel" -- here together with the SSP-RK3
// combination and the dt wave-speed reduction.
//
// B200 design (not the paper's thread-per-point Algs. 7-8):
//  * a CTA owns a strip of TX elements and MARCHES up RB element rows of it;
//  * element rows (strip + W/E halo element) stream HBM -> shared memory by TMA
//    in an NSTG-deep mbarrier ring, issued two rows ahead, so HBM traffic is
//    continuous and each state value is read from HBM once.  For P3 (one
//    element row of one component = 128 B) a 3-D tensor map moves the whole
//    row (4 components x 34 elements) in ONE cp.async.bulk.tensor with the
//    128-byte swizzle, which makes the column reads below bank-conflict free;
//    other orders use 1-D bulk copies (their odd element strides are
//    conflict-free by themselves, P1 2-way);
//  * one thread per element LINE (the n points of row b of one element): the
//    xi-direction work (derivative, both x-faces, correction) is register
//    resident; the eta operands are broadcast reads of the element's columns;
//  * each face point's Rusanov flux is computed once: x-faces by the element to
//    their right, the N faces of row j by line n-1 of row j, whose jump for the
//    element above is carried to the next marching step (S faces are free);
//  * results leave by coalesced stores straight from registers (out = a0 q0 +
//    a1 q + bcoef dt R), with the wave-speed max for the next dt.
#include <cudaTypedefs.h>

#include <cstring>

#include "common.cuh"
#include "ops_tables.h"
#include "tma.cuh"

namespace h2d {

namespace {

template <int K> struct GTile;
// CTAs per SM (register cap 64K / (MINB x threads)) and strip widths, A/B-timed on
// 4096^2 / 8192^2 (round 1): P1 MINB 4 (+9 % over 2), P2 MINB 4 (+41 % over 2),
// P4 12-element strips (60 threads) at 4 CTAs/SM (+18-23 % over 16 at 2, +25 % over 32 at 1)
#ifndef H2D_P1V2
#define H2D_P1V2 1  // CPR P1 1-D path: 16-B pair loads of lines and element rows (+2 %, shock +4.7 %)
#endif
#ifndef H2D_MINB1
#define H2D_MINB1 4
#endif
#ifndef H2D_MINB2
#define H2D_MINB2 4
#endif
#ifndef H2D_TX4
#define H2D_TX4 12
#endif
#ifndef H2D_MINB4
#define H2D_MINB4 4
#endif
template <> struct GTile<1> { static constexpr int TX = 64, RB = 64, MINB = H2D_MINB1; };  // 128 threads
template <> struct GTile<2> { static constexpr int TX = 32, RB = 64, MINB = H2D_MINB2; };  //  96 threads
#ifndef H2D_MINB3
#define H2D_MINB3 4
#endif
#ifndef H2D_NDG_TX3
#define H2D_NDG_TX3 14  // A/B: +8.5 % over 16 (3 -> 4 CTAs/SM)
#endif
#ifndef H2D_TX3
#define H2D_TX3 16  // 64 threads: 4 CTAs/SM interleave their barrier phases (A/B: +2.5 % over 32)
#endif
template <> struct GTile<3> { static constexpr int TX = H2D_TX3, RB = 64, MINB = H2D_MINB3; };  // 128 threads
template <> struct GTile<4> { static constexpr int TX = H2D_TX4, RB = 64, MINB = H2D_MINB4; };  // 5 TX threads

enum { GM_CPR = 1, GM_NDG = 3 };
// NDG strip widths (its g buffer makes its shared memory larger than CPR's)
#ifndef H2D_NDG_TX1
#define H2D_NDG_TX1 64
#endif
#ifndef H2D_NDG_TX2
#define H2D_NDG_TX2 32
#endif
#ifndef H2D_NDG_TX4
#define H2D_NDG_TX4 H2D_TX4
#endif
constexpr int NSTG = 3;  // ring depth (rows): current, N neighbour, one in flight
#ifndef H2D_SWZ_CONTIG
#define H2D_SWZ_CONTIG 1
#endif
#ifndef H2D_Q0TMA
#define H2D_Q0TMA 1
#endif
// NDG: y work by column (as gl_stage.cu's H2D_GL_COLY): the thread of line b
// also owns column b of its element for the y direction -- g at the column's
// points, D g, its S / N jumps (the S one carried in registers from the row
// below) and their lift -- and hands the N points' y residual to the line
// owners (0: the round-2 layout, A/B; A/B on 4096^2 NDG P2 / P3 / P4: 63.3 /
// 60.7 / 59.6 -> 67.2 / 69.7 / 60.8 % of HBM).  CPR keeps the line layout: its
// column owner would need the column points' primitives for B(q) (one more
// reciprocal chain per point) and the larger buffer costs it a CTA per SM
// (CPR P2 / P3 / P4: 71 / 68 / 63 -> 63 / 63 / 56 %)
#ifndef H2D_GLL_COLY
#define H2D_GLL_COLY 1
#endif

struct GMaps {   // P3: 3-D tensor maps {16 points, TX+2 elements, 4 components}
  CUtensorMap q, lo, hi;
  CUtensorMap q0;  // (Q0T) q^n, box {16, TX, 4}
};

template <int M, int K>
struct G {
  static constexpr int N = K + 1, NP = N * N;
  // NDG P3 keeps g of every point in smem: 14-element strips (16-slot TMA rows)
  // keep it at 4 CTAs/SM
  static constexpr int TX = (M == GM_NDG) ? (K == 1 ? H2D_NDG_TX1 : K == 2 ? H2D_NDG_TX2 : K == 3 ? H2D_NDG_TX3
                                                                                     : H2D_NDG_TX4)
                                          : GTile<K>::TX,
                       RB = GTile<K>::RB, NT = TX * N;
  static constexpr bool SWZ = (NP == 16);           // element row of one component == 128 B
  static constexpr int NSL = TX + 2;                 // W halo, TX elements, E halo
  // 1-D path: W piece | main piece | E piece per component (aligned supersets)
  static constexpr int CW = (NP + 1 + 1) & ~1;
  static constexpr int CM = ((TX * NP + 1) + 1) & ~1;
  static constexpr int CREG = CW + CM + CW;
  // per stage (doubles): SWZ: 4 components x RSW rows of 16, each component at a
  // 1024-B boundary so the swizzle phase of a slot is (slot & 7) for every
  // component (+ 8 unswizzled fix-up rows); else 4 * CREG
  // CONTIG (NDG): the 4 components of a row as ONE 3-D box {16, NSL, 4} (rows of
  // 16 doubles contiguous over components, no padding to whole 1024-B blocks;
  // the swizzle phase of row r = c NSL + e of the box is r & 7).  A/B (round
  // 2b): NDG P3 +1 %, CPR P3 -1 % (it keeps four per-component boxes)
  // Q0T (P3): q^n of a row by TMA into a 2-row swizzled ring, issued two rows
  // ahead (instead of one row ahead by per-thread cp.async); the contiguous
  // box below pays for its shared memory
  static constexpr bool Q0T = H2D_Q0TMA && SWZ;
  static constexpr bool CONTIG = H2D_SWZ_CONTIG && (M == GM_NDG || Q0T);
  static constexpr int RSW = CONTIG ? NSL : (NSL + 7) & ~7;
  static constexpr int FIXO = 4 * RSW * 16;
  static constexpr int STG = SWZ ? FIXO + 8 * 16 : 4 * CREG;
  static constexpr int STGA = H2D_STGA(STG);          // stage stride (see H2D_STGA)
  static constexpr int OR_ = 0;
  static constexpr int QSTG = 4 * TX * 16;            // (Q0T) one q^n row: [4 x TX rows of 16], 1024-B multiple
  static constexpr int OQT = OR_ + NSTG * STGA;       // (Q0T) q^n ring [2][QSTG]
  static constexpr int OFW = OQT + (Q0T ? 2 * QSTG : 0);  // W-face fluxes [TX+1][N][4]
  static constexpr bool CY = H2D_GLL_COLY && M == GM_NDG;  // y work by column (NDG)
  static constexpr int OJN = OFW + (TX + 1) * N * 4;  // N jumps of the current row [TX][N][4]
  static constexpr int OJS = OJN + (CY ? 0 : TX * N * 4);      // S jumps, double-buffered [2][TX][N][4]
  static constexpr int OG = OJS + (CY ? 0 : 2 * TX * N * 4);   // NDG (!CY): g at every point [TX][NP][4]
  static constexpr int GS = NP * 4 + 2;  // padded element stride (conflict-free column reads)
  // CY: y part of the residual of every point (written by the point's column
  // owner): element lx, point (row a, column x) at lx * RES + x * RCS + a * 4
  // (strides as gl_stage.cu: conflict-free column writes, 2-way line reads)
  // (odd N: no element padding -- the lane groups of an element do not align
  // with quarter warps anyway, and it keeps NDG P2 / P4 at 4 CTAs/SM)
  static constexpr int RCS = N * 4 + 2, RES = N % 2 ? N * RCS : N * RCS + ((8 - (N * RCS) % 16) + 16) % 16;
  static constexpr int ORY = OG + (M == GM_NDG && !CY ? TX * GS : 0);
  static constexpr int OT = ORY + (CY ? TX * RES : 0);
  static constexpr int ORD = OT + ((N * N + 3 * N + 1) & ~1);
  static constexpr int OB = ORD + 32;                 // mbarriers (as doubles)
  static constexpr int LP = (N + 1) & ~1;             // q^n line slot (16-B multiple)
  static constexpr int OQ0 = OB + ((NSTG + 2 + 1) & ~1);  // q^n prefetch [4][N][NT], thread-private (!Q0T)
  static constexpr int TOTAL = OQ0 + (Q0T ? 0 : 4 * N * NT);
  static_assert(!Q0T || (QSTG % 128 == 0 && OQT % 128 == 0), "1024-B aligned q^n stages");
  static_assert(OQ0 % 2 == 0, "16-B cp.async slots");
  static constexpr size_t SMEM = TOTAL * sizeof(double);
};

// cp.async (LDGSTS) of this thread's q^n line (4 components x N doubles) into its
// private smem slots, one row ahead of its use
template <int N, int NT, int LP>
__device__ __forceinline__ void q0_prefetch(double* sq0, const double* q0, long long cs, long long base, int tid,
                                            bool vec) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double* s = q0 + c * cs + base;
    if (N % 2 == 0 && vec) {  // 16-B pieces, layout [c][x/2][thread] of double2
#pragma unroll
      for (int x = 0; x < N; x += 2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sq0 + (c * N + x) * NT + 2 * tid)),
                     "l"(s + x)
                     : "memory");
    } else {
#pragma unroll
      for (int x = 0; x < N; ++x)  // layout [c][x][thread]: conflict-free read-back
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sq0 + (c * N + x) * NT + tid)),
                     "l"(s + x)
                     : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

struct GTab {
  double v[25 + 10 + 5];  // D [N][N], g'_L, g'_R, GLL weights
};

template <int K>
GTab make_gtab() {
  using O = Ops<K>;
  constexpr int N = K + 1;
  GTab t{};
  for (int a = 0; a < N; ++a) {
    for (int l = 0; l < N; ++l) t.v[a * N + l] = O::D_gll[a][l];
    t.v[N * N + a] = O::gLp_gll[a];
    t.v[N * N + N + a] = O::gRp_gll[a];
    t.v[N * N + 2 * N + a] = O::w_gll[a];
  }
  return t;
}

__device__ __forceinline__ void st4(double* p, const double v[4]) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
}
__device__ __forceinline__ void ld4(const double* p, double v[4]) {
  const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

#ifndef H2D_Q0LATE
#define H2D_Q0LATE 1
#endif
#ifndef H2D_VIEWCARRY
#define H2D_VIEWCARRY 1  // a row's view of the ring (source, piece offsets) computed once, carried to the next row
#endif
#ifndef H2D_WSQRT
#define H2D_WSQRT fsqrt_ws  // Rusanov dissipation speed (common.cuh; A/B: fsqrt)
#endif
// node evaluation: the DIR flux and the DIR normal wave speed |u_n| + c
template <int DIR>
__device__ __forceinline__ void node_eval(const double q[4], double gm1, double gam, double f[4], double& s) {
  const Prim w = prims(q, gm1);
  flux<DIR>(q, w, f);
  s = fabs(DIR == 0 ? w.u : w.v) + H2D_WSQRT(gam * w.p * w.ri);  // Rusanov dissipation speed only
}

__device__ __forceinline__ void rus(const double qL[4], const double fL[4], double sL, const double qR[4],
                                    const double fR[4], double sR, double F[4]) {
  const double lam = fmax(sL, sR);
#pragma unroll
  for (int c = 0; c < 4; ++c) F[c] = 0.5 * (fL[c] + fR[c]) - 0.5 * lam * (qR[c] - qL[c]);
}

// row jr (local strip row; -1 / nrows are the ghost rows) of the stage input:
// base pointer and component stride; nullptr = physical transmissive boundary
__device__ __forceinline__ const double* row_src(const StageArgs& a, int jr, int np, long long& cs) {
  if (jr < 0) { cs = a.gcs; return a.ghost_lo; }
  if (jr >= a.nrows) { cs = a.gcs; return a.ghost_hi; }
  cs = a.cs;
  return a.q + (long long)jr * a.nx * np;
}

// 1-D path: aligned-superset copy of [src, src+n) doubles; offset (0 or 1
// double) of src inside the destination
__device__ __forceinline__ int piece_off(const double* src) {
  return (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
}
__device__ __forceinline__ uint32_t piece_bytes(const double* src, int n) {
  const uintptr_t s0 = reinterpret_cast<uintptr_t>(src);
  return (uint32_t)(((s0 + (uintptr_t)n * 8 + 15) & ~uintptr_t(15)) - (s0 & ~uintptr_t(15)));
}
__device__ __forceinline__ const void* piece_src(const double* src) {
  return reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15));
}

}  // namespace

// V (stage variant, compile time): bit 0 q^n read (RK stages 2, 3), bit 1 the
// dt wave speed / non-physical epilogue (stage 3), bit 2 fused element
// averages (limiter runs): each launch runs only the code its stage needs
template <int M, int K, int V>
__global__ void __launch_bounds__(G<M, K>::NT, GTile<K>::MINB)
    gll_stage_kernel(const StageArgs a, const GTab tab, const __grid_constant__ GMaps maps) {
  // V == 8: any other combination, decided at run time from the pointers
  const bool HQ0 = V == 8 ? a.q0 != nullptr : (V & 1), HLAM = V == 8 ? (a.lam || a.bad) : (V & 2) != 0,
             HAVG = V == 8 ? a.qbar != nullptr : (V & 4) != 0;
  using H = G<M, K>;
  constexpr int N = H::N, NP = H::NP, TX = H::TX, NT = H::NT, NSL = H::NSL;
  constexpr int CW = H::CW, CM = H::CM, CREG = H::CREG, STGA = H::STGA;
  extern __shared__ __align__(1024) double4 smem4[];  // no static smem: the window base is 1024-B aligned
  double* sm = reinterpret_cast<double*>(smem4);
  double* ring = sm + H::OR_;
  double* sFW = sm + H::OFW;
  double* sRY = sm + H::ORY;
  double* sJN = sm + H::OJN;
  double* sJS = sm + H::OJS;
  double* sG = sm + H::OG;
  double* sT = sm + H::OT;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + H::OB);
  double* sQ0 = sm + H::OQ0;
  double* sQT = sm + H::OQT;                  // (Q0T) q^n ring
  uint64_t* qbar = bar + NSTG;                // (Q0T) its mbarriers

  const int tid = threadIdx.x;
  int bhi;
  const int i0 = blockIdx.x * TX, jb = band_start(a, bhi);
  const int TXv = min(TX, a.nx - i0), RBv = min(a.rows, bhi - jb);
  const double gam = a.gamma, gm1 = a.gamma - 1.0;
  const int lx = tid / N, b = tid - lx * N;
  const bool own = lx < TXv;
  // vector global access: every line start 32-B (P3) / 16-B aligned in out and q^n
  const unsigned long long amask = N == 4 ? 31ull : 15ull;
  const bool vec = ((((unsigned long long)a.out | (unsigned long long)a.q0 |
                      (unsigned long long)(a.cs * 8)) & amask) == 0);
  const bool mirW = (i0 == 0 && a.bcx), mirE = (i0 + TXv == a.nx && a.bcx);
  const bool wrapW = (i0 == 0 && !a.bcx), wrapE = (i0 + TXv == a.nx && !a.bcx);
  const int iw = i0 > 0 ? i0 - 1 : a.nx - 1;      // W halo element (periodic wrap)
  const int ie = i0 + TXv < a.nx ? i0 + TXv : 0;  // E halo element
  const int nload = RBv + 2;                      // rows jb-1 .. jb+RBv

  for (int i = tid; i < N * N + 3 * N; i += NT) sT[i] = tab.v[i];
  if (tid == 0) {
    for (int s = 0; s < NSTG + (H::Q0T ? 2 : 0); ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();  // everything above touched only shared memory and kernel parameters
  pdl_launch();
  // (read after pdl_wait; stage 1 / 2 of a fused-dt step publish / commit the clock)
  const double dtv = stage_dt(a);
  if (dtv == 0.0) return;  // clipped-out step (t == t_end): uniform across the grid

  // ---- streaming: thread 0 moves row L (L = 0 -> row jb-1) into stage L % NSTG ----
  auto issue_row = [&](int L) {
    if (tid != 0) return;
    const int jr = jb - 1 + L;
    long long cs;
    const double* rb = row_src(a, jr, NP, cs);
    uint64_t* br = &bar[L % NSTG];
    double* st = ring + (L % NSTG) * STGA;
    if (!rb) { mbar_arrive_expect_tx(br, 0); return; }
    if constexpr (H::SWZ) {
      const CUtensorMap* mp = jr < 0 ? &maps.lo : (jr >= a.nrows ? &maps.hi : &maps.q);
      const int y0 = (jr < 0 || jr >= a.nrows ? 0 : jr * a.nx) + i0 - 1;
      uint32_t tx = 4u * NSL * 128u;
      if (wrapW) tx += 4u * 128u;
      if (wrapE) tx += 4u * 128u;
      mbar_arrive_expect_tx(br, tx);
      if (H::CONTIG) tma_load_3d(st, mp, 0, y0, 0, br);
      else
        for (int c = 0; c < 4; ++c) tma_load_3d(st + c * H::RSW * 16, mp, 0, y0, c, br);
      double* fix = st + H::FIXO;
      for (int c = 0; c < 4; ++c) {
        if (wrapW) tma_load_1d(fix + (0 * 4 + c) * 16, rb + c * cs + (long long)iw * NP, NP * 8, br);
        if (wrapE) tma_load_1d(fix + (1 * 4 + c) * 16, rb + c * cs + (long long)ie * NP, NP * 8, br);
      }
    } else {
      uint32_t tx = 0;
      for (int c = 0; c < 4; ++c) {
        const double* comp = rb + c * cs;
        tx += piece_bytes(comp + (long long)i0 * NP, TXv * NP);
        if (!mirW) tx += piece_bytes(comp + (long long)iw * NP, NP);
        if (!mirE) tx += piece_bytes(comp + (long long)ie * NP, NP);
      }
      mbar_arrive_expect_tx(br, tx);
      for (int c = 0; c < 4; ++c) {
        const double* comp = rb + c * cs;
        double* dst = st + c * CREG;
        const double* s1 = comp + (long long)i0 * NP;
        tma_load_1d(dst + CW, piece_src(s1), piece_bytes(s1, TXv * NP), br);
        if (!mirW) {
          const double* s0 = comp + (long long)iw * NP;
          tma_load_1d(dst, piece_src(s0), piece_bytes(s0, NP), br);
        }
        if (!mirE) {
          const double* s2 = comp + (long long)ie * NP;
          tma_load_1d(dst + CW + CM, piece_src(s2), piece_bytes(s2, NP), br);
        }
      }
    }
  };

  // ---- addressing of stage data: element slot e (0 W halo, 1..TXv own, TXv+1 E halo) ----
  struct RowView {
    const double* st;
    int dW, dM, dE;  // 1-D path offsets of component 0 (odd component strides flip them)
    int csodd;
    bool have;
    bool v2;  // 1-D path: every component's own piece 16-B aligned (P1 pairs load as double2)
  };
  const bool has_glo = a.ghost_lo != nullptr, has_ghi = a.ghost_hi != nullptr;
  auto view = [&](int L) {
    RowView v;
    v.st = ring + (L % NSTG) * STGA;
    v.dW = v.dM = v.dE = 0;
    v.csodd = 0;
    v.v2 = false;
    if constexpr (H::SWZ) {  // (the 128-B rows need no piece offsets: only whether the row exists)
      const int jr = jb - 1 + L;
      v.have = jr < 0 ? has_glo : (jr >= a.nrows ? has_ghi : true);
      return v;
    }
    long long cs;
    const double* rb = row_src(a, jb - 1 + L, NP, cs);
    v.have = rb != nullptr;
    v.csodd = (int)(cs & 1);
    if (!H::SWZ && rb) {
      v.dM = piece_off(rb + (long long)i0 * NP);
      v.dW = piece_off(rb + (long long)iw * NP);
      v.dE = piece_off(rb + (long long)ie * NP);
    }
    v.v2 = H2D_P1V2 && M == GM_CPR && N == 2 && !H::SWZ && (((v.dM | v.csodd) & 1) == 0);  // NDG: -0.8 %
    return v;
  };
  // address of (c, p) of own element slot e on the 1-D path (N == 2 pair loads)
  auto own_ptr = [&](const RowView& v, int c, int e, int p) -> const double* {
    return v.st + c * CREG + CW + (v.dM ^ (c & v.csodd)) + (e - 1) * NP + p;
  };
  // value (c, p) of own element slot e = lx + 1 (hot path: no branches)
  auto own_at = [&](const RowView& v, int c, int e, int p) -> double {
    if constexpr (H::SWZ) {  // 128-B swizzle: 16-B chunk (p >> 1) of row e sits at chunk (p >> 1) ^ (e & 7)
      const int r = c * H::RSW + e;
      return v.st[r * 16 + ((((p >> 1) ^ ((H::CONTIG ? r : e) & 7)) << 1) | (p & 1))];
    } else {
      return v.st[c * CREG + CW + (v.dM ^ (c & v.csodd)) + (e - 1) * NP + p];
    }
  };
  // value (c, p) of any slot e (0 W halo, TXv+1 E halo): the index is selected,
  // not branched on (no divergent regions in the face work)
  auto any_at = [&](const RowView& v, int c, int e, int p) -> double {
    if constexpr (H::SWZ) {
      const bool fw = (e == 0 && wrapW), fe = (e == TXv + 1 && wrapE);
      const int r = c * H::RSW + e;
      const int iS = r * 16 + ((((p >> 1) ^ ((H::CONTIG ? r : e) & 7)) << 1) | (p & 1));
      const int iF = H::FIXO + ((fe ? 4 : 0) + c) * 16 + p;
      return v.st[(fw || fe) ? iF : iS];
    } else {
      const int iW = c * CREG + (v.dW ^ (c & v.csodd)) + p;
      const int iE = c * CREG + CW + CM + (v.dE ^ (c & v.csodd)) + p;
      const int iM = c * CREG + CW + (v.dM ^ (c & v.csodd)) + (e - 1) * NP + p;
      return v.st[e == 0 ? iW : (e == TXv + 1 ? iE : iM)];
    }
  };

  for (int L = 0; L < NSTG && L < nload; ++L) issue_row(L);
  // (Q0T) q^n of own row jb + m into ring slot m & 1, by one TMA box
  auto issue_q0 = [&](int m) {
    if (tid != 0) return;
    uint64_t* bq = &qbar[m & 1];
    mbar_arrive_expect_tx(bq, 4u * TX * 128u);
    tma_load_3d(sQT + (m & 1) * H::QSTG, &maps.q0, 0, (jb + m) * a.nx + i0, 0, bq);
  };
  if (H::Q0T) {
    if (HQ0) {  // the first two own rows
      issue_q0(0);
      if (RBv > 1) issue_q0(1);
    }
  } else if (HQ0 && own) {  // q^n of the first own row (step L = 1)
    q0_prefetch<N, NT, H::LP>(sQ0, a.q0, a.cs, ((long long)jb * a.nx + i0 + lx) * NP + b * N, tid, vec);
  }

  [[maybe_unused]] const double* D = sT;
  [[maybe_unused]] const double gLb = sT[N * N + b], gRb = sT[N * N + N + b];
  double lam = 0.0;
  const double bdt = a.bcoef * dtv;
  const double cx = -bdt * a.rdx2, cy = -bdt * a.rdy2;

  double JSr[4] = {0.0, 0.0, 0.0, 0.0};  // CY: S jump of this thread's column (from the row below's N face)
  RowView vcar = view(0);  // (H2D_VIEWCARRY) the next row's view, carried
  for (int L = 0; L <= RBv; ++L) {
    mbar_wait(&bar[L % NSTG], (L / NSTG) & 1);
    mbar_wait(&bar[(L + 1) % NSTG], ((L + 1) / NSTG) & 1);
    const RowView vc = H2D_VIEWCARRY ? vcar : view(L), vn = view(L + 1);
    vcar = vn;
    double* jSc = sJS + (L & 1) * TX * N * 4;        // S jumps of row L (written in step L-1)
    double* jSn = sJS + ((L + 1) & 1) * TX * N * 4;  // S jumps of row L+1 (written now)
    const long long jr = jb - 1 + L;                 // local strip row of this step

    double q[4][N], fW[4], fE[4], jW[4];
    double fxl[4][N];  // NDG: x fluxes of the line
    double lpart[4] = {0.0, 0.0, 0.0, 0.0};  // limiter runs: the line's share of the element average
    Prim pW, pE;
    // Face work of the row, straight-line so that the independent node
    // evaluations (reciprocal / square-root chains) interleave: the W face of
    // each line (computed by the element on its right), the N face of column b
    // of each element (spread over the lines: no divergence; its jump for the
    // element above is carried to the next step); transmissive ends by selects.
    if (own) {
      double qd[4], qu[4];  // column b: own top point, next row's bottom point
      double colv[4][N];  // CY: column b of the element (the prologue row's slot may hold no row: then unused)
      if constexpr (H::CY) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int l = 0; l < N; ++l) colv[c][l] = own_at(vc, c, lx + 1, l * N + b);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double d = H::CY ? colv[c][N - 1] : own_at(vc, c, lx + 1, (N - 1) * N + b),
                     u = own_at(vn, c, lx + 1, b);
        qd[c] = vc.have ? d : u;
        qu[c] = vn.have ? u : d;
      }
      if (L > 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int x = 0; x < N; ++x) {
            if constexpr (H::SWZ) {  // 16-B chunks: points (4b + 2h, 4b + 2h + 1)
              if ((x & 1) == 0) {
                const double2 u = *reinterpret_cast<const double2*>(
                    vc.st + (c * H::RSW + lx + 1) * 16 +
                    (((2 * b + (x >> 1)) ^ ((H::CONTIG ? c * H::RSW + lx + 1 : lx + 1) & 7)) << 1));
                q[c][x] = u.x;
                q[c][x + 1] = u.y;
              }
            } else if (N == 2 && vc.v2) {  // P1: the line's two points as one 16-B load
              if (x == 0) {
                const double2 u = *reinterpret_cast<const double2*>(own_ptr(vc, c, lx + 1, b * N));
                q[c][0] = u.x;
                q[c][1 % N] = u.y;
              }
            } else {
              q[c][x] = own_at(vc, c, lx + 1, b * N + x);
            }
          }
        double qw[4] = {q[0][0], q[1][0], q[2][0], q[3][0]}, sw;
        double qe[4] = {q[0][N - 1], q[1][N - 1], q[2][N - 1], q[3][N - 1]}, se;
        double ql[4];  // E point of the W neighbour's line (the domain's W end mirrors)
        const bool mw = (lx == 0 && mirW);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double v = any_at(vc, c, lx, b * N + N - 1);
          ql[c] = mw ? qw[c] : v;
        }
        pW = prims(qw, gm1);  // kept for the chain rule at points 0 and n-1
        pE = prims(qe, gm1);
        flux<0>(qw, pW, fW);
        flux<0>(qe, pE, fE);
        sw = fabs(pW.u) + H2D_WSQRT(gam * pW.p * pW.ri);
        se = fabs(pE.u) + H2D_WSQRT(gam * pE.p * pE.ri);
        double fl[4], sl, gd[4], sd, gu[4], su;
        node_eval<0>(ql, gm1, gam, fl, sl);
        node_eval<1>(qd, gm1, gam, gd, sd);
        node_eval<1>(qu, gm1, gam, gu, su);
        double F[4], Gf[4], j[4];
        rus(ql, fl, sl, qw, fW, sw, F);
        rus(qd, gd, sd, qu, gu, su, Gf);
        st4(sFW + (lx * N + b) * 4, F);
#pragma unroll
        for (int c = 0; c < 4; ++c) jW[c] = F[c] - fW[c];
#pragma unroll
        for (int c = 0; c < 4; ++c) j[c] = Gf[c] - gd[c];
        if constexpr (H::CY) {  // y part of the residual at the points (a, b) of column b, to their line owners
          double gc[N][4];  // g at the column's points
#pragma unroll
          for (int l = 0; l < N; ++l) {
            double v[4] = {colv[0][l], colv[1][l], colv[2][l], colv[3][l]};
            flux<1>(v, prims(v, gm1), gc[l]);
          }
#pragma unroll
          for (int aa = 0; aa < N; ++aa) {  // D g + the lift of the S / N jumps at (a, b)
            const double gLa = tab.v[N * N + aa], gRa = tab.v[N * N + N + aa];
            double gy[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              double sv = tab.v[aa * N] * gc[0][c];
#pragma unroll
              for (int l = 1; l < N; ++l) sv = fma(tab.v[aa * N + l], gc[l][c], sv);
              gy[c] = sv + gLa * JSr[c] + gRa * j[c];
            }
            st4(sRY + lx * H::RES + b * H::RCS + aa * 4, gy);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) JSr[c] = Gf[c] - gu[c];
        } else {
          st4(sJN + (lx * N + b) * 4, j);
#pragma unroll
          for (int c = 0; c < 4; ++c) j[c] = Gf[c] - gu[c];
          st4(jSn + (lx * N + b) * 4, j);
        }
        if (lx == TXv - 1) {  // the strip's last E face
          if (mirE) {
            rus(qe, fE, se, qe, fE, se, F);
          } else {
            double qr[4], fr[4], sr;
#pragma unroll
            for (int c = 0; c < 4; ++c) qr[c] = any_at(vc, c, TXv + 1, b * N);
            node_eval<0>(qr, gm1, gam, fr, sr);
            rus(qe, fE, se, qr, fr, sr, F);
          }
          st4(sFW + (TXv * N + b) * 4, F);
        }
        if (M == GM_NDG) {  // eta operands: g at the points of the line (smem); f kept in registers
#pragma unroll
          for (int x = 0; x < N; ++x) {
            double v[4] = {q[0][x], q[1][x], q[2][x], q[3][x]}, f[4];
            const Prim w = (x == 0) ? pW : (x == N - 1) ? pE : prims(v, gm1);
            flux<0>(v, w, f);
#pragma unroll
            for (int c = 0; c < 4; ++c) fxl[c][x] = f[c];
            if constexpr (!H::CY) {
              double g[4];
              flux<1>(v, w, g);
              st4(sG + lx * H::GS + (b * N + x) * 4, g);
            }
          }
        }
      } else {  // prologue row (below the march): only its N face, as the first row's S face
        double gd[4], sd, gu[4], su, Gf[4], j[4];
        node_eval<1>(qd, gm1, gam, gd, sd);
        node_eval<1>(qu, gm1, gam, gu, su);
        rus(qd, gd, sd, qu, gu, su, Gf);
#pragma unroll
        for (int c = 0; c < 4; ++c) j[c] = Gf[c] - gu[c];
        if constexpr (H::CY) {
#pragma unroll
          for (int c = 0; c < 4; ++c) JSr[c] = j[c];
        } else {
          st4(jSn + (lx * N + b) * 4, j);
        }
      }
    }
    __syncthreads();

    if (L > 0 && own) {
      const long long base = (jr * a.nx + i0 + lx) * NP + b * N;
      // q^n of the line: prefetched by cp.async one row ahead into thread-private smem
      if (HQ0) {
        if (H::Q0T) mbar_wait(&qbar[(L - 1) & 1], ((L - 1) >> 1) & 1);
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      const double* q0s = sQT + ((L - 1) & 1) * H::QSTG;  // (Q0T) this row's q^n slot
#define Q0V(c, x)                                                                                           \
  (H::Q0T ? q0s[((c) * TX + lx) * 16 +                                                                      \
                ((((2 * b + ((x) >> 1)) ^ (((c) * TX + lx) & 7)) << 1) | ((x) & 1))]                        \
   : (N % 2 == 0 && vec ? sQ0[((c) * N + ((x) & ~1)) * NT + 2 * tid + ((x) & 1)]                             \
                        : sQ0[((c) * N + (x)) * NT + tid]))
      double F[4], jE[4];
      ld4(sFW + ((lx + 1) * N + b) * 4, F);
#pragma unroll
      for (int c = 0; c < 4; ++c) jE[c] = F[c] - fE[c];
      // CPR P3: eta-derivatives of all points of the line at once, two points per
      // 16-B swizzled chunk (half the shared-memory loads of a per-point loop)
      double dyall[N][4];
      if constexpr (M == GM_CPR && H::SWZ && !H::CY) {
        // (sums start from their first product: no zero-initialised accumulators)
#pragma unroll
        for (int l = 0; l < N; ++l) {
          const double db = D[b * N + l];
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int h = 0; h < N / 2; ++h) {
              const double2 u = *reinterpret_cast<const double2*>(
                  vc.st + (c * H::RSW + lx + 1) * 16 +
                  (((2 * l + h) ^ ((H::CONTIG ? c * H::RSW + lx + 1 : lx + 1) & 7)) << 1));
              if (l == 0) {
                dyall[2 * h][c] = db * u.x;
                dyall[2 * h + 1][c] = db * u.y;
              } else {
                dyall[2 * h][c] = fma(db, u.x, dyall[2 * h][c]);
                dyall[2 * h + 1][c] = fma(db, u.y, dyall[2 * h + 1][c]);
              }
            }
        }
      }
      // CPR P1 (1-D path, aligned): eta-derivatives of both points of the line
      // from the element's rows as 16-B pairs (same operation order as below)
      double dy2[N][4];
      if constexpr (M == GM_CPR && N == 2 && !H::SWZ && !H::CY) {
        if (vc.v2) {
#pragma unroll
          for (int l = 0; l < N; ++l) {
            const double db = D[b * N + l];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const double2 u = *reinterpret_cast<const double2*>(own_ptr(vc, c, lx + 1, l * N));
              dy2[0][c] = l == 0 ? db * u.x : fma(db, u.x, dy2[0][c]);
              dy2[1 % N][c] = l == 0 ? db * u.y : fma(db, u.y, dy2[1 % N][c]);
            }
          }
        }
      }
      double ov[4][N], q0v[4][N];  // q^n of the line (0 in stage 1: a0 = 0)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int x = 0; x < N; ++x) q0v[c][x] = HQ0 ? Q0V(c, x) : 0.0;
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double v[4] = {q[0][x], q[1][x], q[2][x], q[3][x]};
        if constexpr (H::CY) {  // NDG: D[F] + the y part from the owner of column x
          double gy[4];
          ld4(sRY + lx * H::RES + x * H::RCS + b * 4, gy);
          const double gLa = tab.v[N * N + x], gRa = tab.v[N * N + N + x];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double sv = tab.v[x * N] * fxl[c][0];
#pragma unroll
            for (int l = 1; l < N; ++l) sv = fma(tab.v[x * N + l], fxl[c][l], sv);
            const double fx = sv + gLa * jW[c] + gRa * jE[c];
            // out = a0 q^n + a1 q + bdt R,  R = -(2/dx) fx - (2/dy) gy  (metric folded into cx, cy)
            const double rk = fma(a.a1, v[c], fma(cx, fx, cy * gy[c]));
            ov[c][x] = HQ0 ? fma(a.a0, q0v[c][x], rk) : rk;
          }
        } else {
        double Fx[4], Gy[4], dy[4];
#pragma unroll
        for (int l = 0; l < N; ++l) {  // column x of the element (broadcast over its lines)
          const double db = D[b * N + l];
          if (M == GM_CPR && H::SWZ) {
            if (l == 0) {
#pragma unroll
              for (int c = 0; c < 4; ++c) dy[c] = dyall[x][c];
            }
          } else if (M == GM_CPR && N == 2 && vc.v2) {
            if (l == 0) {
#pragma unroll
              for (int c = 0; c < 4; ++c) dy[c] = dy2[x][c];
            }
          } else if (M == GM_CPR) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const double u = own_at(vc, c, lx + 1, l * N + x);
              dy[c] = l == 0 ? db * u : fma(db, u, dy[c]);
            }
          } else {
            double u[4];
            ld4(sG + lx * H::GS + (l * N + x) * 4, u);
#pragma unroll
            for (int c = 0; c < 4; ++c) dy[c] = l == 0 ? db * u[c] : fma(db, u[c], dy[c]);
          }
        }
        if (M == GM_CPR) {  // chain rule: A(q) dq/dxi + B(q) dq/deta
          double dx[4];
#pragma unroll
          for (int l = 0; l < N; ++l) {
            const double da = tab.v[x * N + l];  // compile-time index: constant-bank operand
#pragma unroll
            for (int c = 0; c < 4; ++c) dx[c] = l == 0 ? da * q[c][l] : fma(da, q[c][l], dx[c]);
          }
          const Prim w = (x == 0) ? pW : (x == N - 1) ? pE : prims(v, gm1);
          jac_pair(v, w, gm1, dx, dy, Fx, Gy);
        } else {            // NDG: D[F]
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double s = tab.v[x * N] * fxl[c][0];
#pragma unroll
            for (int l = 1; l < N; ++l) s = fma(tab.v[x * N + l], fxl[c][l], s);
            Fx[c] = s;
            Gy[c] = dy[c];
          }
        }
        double jS[4], jN[4];
        ld4(jSc + (lx * N + x) * 4, jS);
        ld4(sJN + (lx * N + x) * 4, jN);
        const double gLa = tab.v[N * N + x], gRa = tab.v[N * N + N + x];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double fx = Fx[c] + gLa * jW[c] + gRa * jE[c];
          const double gy = Gy[c] + gLb * jS[c] + gRb * jN[c];
          // out = a0 q^n + a1 q + bdt R,  R = -(2/dx) fx - (2/dy) gy  (metric folded into cx, cy)
          const double rk = fma(a.a1, v[c], fma(cx, fx, cy * gy));
          ov[c][x] = HQ0 ? fma(a.a0, q0v[c][x], rk) : rk;
        }
        }
      }
      if (HLAM) {  // dt wave speed and non-physical check share one reciprocal (straight-line)
        unsigned long long bidx = ~0ull;
#pragma unroll
        for (int x = 0; x < N; ++x) {
          const double o[4] = {ov[0][x], ov[1][x], ov[2][x], ov[3][x]};
          const Prim w = prims(o, gm1);
          lam = nanmax(lam, fmax(fabs(w.u), fabs(w.v)) + fsqrt(gam * w.p * w.ri));
          if (!admissible(o[0], w.p)) bidx = min(bidx, (unsigned long long)(base + x));
        }
        if (a.bad && bidx != ~0ull) atomicMin(a.bad, bidx);
      }
      if (HAVG && a.laml) {  // limiter runs: this line's wave speed / first bad point for k_limit (LamFuse)
        unsigned long long bidx = ~0ull;
        double ll = 0.0;
#pragma unroll
        for (int x = 0; x < N; ++x) {
          const double o[4] = {ov[0][x], ov[1][x], ov[2][x], ov[3][x]};
          const Prim w = prims(o, gm1);
          ll = nanmax(ll, fmax(fabs(w.u), fabs(w.v)) + fsqrt(gam * w.p * w.ri));
          if (!admissible(o[0], w.p)) bidx = min(bidx, (unsigned long long)(base + x));
        }
        const long long li = (jr * a.nx + i0 + lx) * N + b;
        a.laml[li] = ll;
        a.badl[li] = bidx;
      }
      // a thread's line of one component is N contiguous doubles: one 32-B (P3) or
      // 16-B (P1) store per component when aligned
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double* o = a.out + c * a.cs + base;
        if (N == 4 && vec) {
          asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o), "d"(ov[c][0]), "d"(ov[c][1 % N]),
                       "d"(ov[c][2 % N]), "d"(ov[c][3 % N])
                       : "memory");
        } else if (N == 2 && vec) {
          asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(o), "d"(ov[c][0]), "d"(ov[c][1 % N]) : "memory");
        } else {
#pragma unroll
          for (int x = 0; x < N; ++x) o[x] = ov[c][x];
        }
      }
      if (!H::Q0T && HQ0 && L < RBv && !H2D_Q0LATE)  // q^n of the next row into the (now consumed) private slots
        q0_prefetch<N, NT, H::LP>(sQ0, a.q0, a.cs, base + (long long)a.nx * NP, tid, vec);
      if (HAVG) {  // this line's share of the element average: w_b sum_x w_x q
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double sx = 0.0;
#pragma unroll
          for (int x = 0; x < N; ++x) sx += tab.v[N * N + 2 * N + x] * ov[c][x];
          lpart[c] = sT[N * N + 2 * N + b] * sx;
        }
      }
    }
    if (HAVG && (N == 2 || N == 4)) {  // element averages: the element's N lines are N aligned lanes
      // lanes of this warp that exist (NT need not be a multiple of 32; element lane groups are whole)
      const unsigned wmask = (NT % 32 == 0 || (tid >> 5) < NT / 32) ? 0xffffffffu : ((1u << (NT % 32)) - 1u);
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int o = 1; o < N; o <<= 1) lpart[c] += __shfl_xor_sync(wmask, lpart[c], o);
      if (L > 0 && own && b == 0) {
        const long long m = jr * a.nx + i0 + lx, ne = (long long)a.nx * a.nrows;
#pragma unroll
        for (int c = 0; c < 4; ++c) a.qbar[c * ne + m] = 0.25 * lpart[c];
      }
    } else if (HAVG) {  // element averages (N = 3, 5: through the W-face buffer)
      __syncthreads();
      if (L > 0 && own) st4(sFW + (lx * N + b) * 4, lpart);
      __syncthreads();
      if (L > 0 && own) {
        const long long m = jr * a.nx + i0 + lx, ne = (long long)a.nx * a.nrows;
        for (int c = b; c < 4; c += N) {
          double s = 0.0;
#pragma unroll
          for (int bb = 0; bb < N; ++bb) s += sFW[(lx * N + bb) * 4 + c];
          a.qbar[c * ne + m] = 0.25 * s;
        }
      }
    }
    __syncthreads();  // stage L % NSTG and the face buffers are free again
    if (L + NSTG < nload) {
      if (tid == 0) fence_proxy_async_smem();
      issue_row(L + NSTG);
    }
    // q^n of the next row into the consumed private slots -- after the proxy
    // fence of the TMA issue: the fence waits for this thread's in-flight
    // cp.async writes, so a prefetch issued before it stalled warp 0 for a
    // global-memory round trip every row (H2D_Q0LATE=0: the round-2 order)
    if (!H::Q0T && H2D_Q0LATE && HQ0 && own && L > 0 && L < RBv)
      q0_prefetch<N, NT, H::LP>(sQ0, a.q0, a.cs, ((long long)(jb + L) * a.nx + i0 + lx) * NP + b * N, tid, vec);
    if (H::Q0T && HQ0 && L > 0 && L + 1 < RBv) {  // q^n two rows ahead into the slot this row consumed
      if (tid == 0) fence_proxy_async_smem();
      issue_q0(L + 1);
    }
  }
  if (HLAM && a.lam) block_max_to(lam, a.lam, sm + H::ORD);
}

// ---- host: tensor maps (P3 path) ------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
}  // namespace

// {16 points, nelem elements, 4 components} fp64, box {16, box_e, box_c}, 128-byte swizzle
bool make_map(CUtensorMap* m, const double* base, long long nelem, long long cs, int box_e, int box_c) {
  memset(m, 0, sizeof(*m));
  if (!base) return true;  // transmissive boundary: never used
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {16, (cuuint64_t)nelem, 4};
  cuuint64_t strides[2] = {16 * sizeof(double), (cuuint64_t)cs * sizeof(double)};
  cuuint32_t box[3] = {16, (cuuint32_t)box_e, (cuuint32_t)box_c};  // one component or all four per copy
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int M, int K, int V>
static cudaError_t launch_v(dim3 grid, const StageArgs& b, const GTab& tab, const GMaps& maps, cudaStream_t s) {
  using H = G<M, K>;
  static std::atomic<unsigned long long> attr{0};
  const cudaError_t e = smem_optin(gll_stage_kernel<M, K, V>, (int)H::SMEM, attr);
  if (e != cudaSuccess) return e;
  return launch_pdl_if(!b.no_pdl, gll_stage_kernel<M, K, V>, grid, dim3(H::NT), H::SMEM, s, b, tab, maps);
}

template <int M, int K>
static int launch_g(const StageArgs& a, cudaStream_t s) {
  using H = G<M, K>;
  static const GTab tab = make_gtab<K>();
  GMaps maps;
  memset(&maps, 0, sizeof(maps));
  if (H::SWZ) {
    const long long nel = (long long)a.nx * a.nrows;
    const int bc = H::CONTIG ? 4 : 1;
    if (!make_map(&maps.q, a.q, nel, a.cs, H::NSL, bc) || !make_map(&maps.lo, a.ghost_lo, a.nx, a.gcs, H::NSL, bc) ||
        !make_map(&maps.hi, a.ghost_hi, a.nx, a.gcs, H::NSL, bc) ||
        (H::Q0T && !make_map(&maps.q0, a.q0, nel, a.cs, H::TX, 4)))
      return (int)cudaErrorInvalidValue;
  }
  StageArgs b = a;
  const int strips = (a.nx + H::TX - 1) / H::TX;
  const int nr = row_range(b);
  if (nr <= 0) return 0;
  b.rows = march_rows(nr, strips, H::RB);
  dim3 grid(strips, band_blocks(b));
  const int v = (a.q0 ? 1 : 0) | ((a.lam || a.bad) ? 2 : 0) | (a.qbar ? 4 : 0);
  cudaError_t e = cudaSuccess;
  switch (v) {
    case 0: e = launch_v<M, K, 0>(grid, b, tab, maps, s); break;
    case 1: e = launch_v<M, K, 1>(grid, b, tab, maps, s); break;
    case 3: e = launch_v<M, K, 3>(grid, b, tab, maps, s); break;
    case 4: e = launch_v<M, K, 4>(grid, b, tab, maps, s); break;
    case 5: e = launch_v<M, K, 5>(grid, b, tab, maps, s); break;
    default: e = launch_v<M, K, 8>(grid, b, tab, maps, s); break;
  }
  return e != cudaSuccess ? (int)e : (int)cudaPeekAtLastError();
}

int launch_gll_stage(int method, int k, const StageArgs& a, cudaStream_t s) {
  if (k == 1) {  // P1: the element-per-lane warp kernel where it applies (p1_stage.cu)
    const int e = launch_p1_stage(method, a, s);
    if (e >= 0) return e;
  }
  if (method == GM_CPR) {
    switch (k) {
      case 1: return launch_g<GM_CPR, 1>(a, s);
      case 2: return launch_g<GM_CPR, 2>(a, s);
      case 3: return launch_g<GM_CPR, 3>(a, s);
      case 4: return launch_g<GM_CPR, 4>(a, s);
    }
  } else if (method == GM_NDG) {
    switch (k) {
      case 1: return launch_g<GM_NDG, 1>(a, s);
      case 2: return launch_g<GM_NDG, 2>(a, s);
      case 3: return launch_g<GM_NDG, 3>(a, s);
      case 4: return launch_g<GM_NDG, 4>(a, s);
    }
  }
  return (int)cudaErrorInvalidValue;
}

}  // namespace h2d
