// gl_stage.cu -- fused RK-stage kernels of the methods with Gauss-Legendre
// solution points: DG (weak form on GL points, Eqs. (18)-(21), Algs. 2-4,
// P:240-267) and SD (GL solution points, Chebyshev-Gauss-Lobatto flux
// points, Eqs. (30)-(34), Algs. 5-6).
//
// Same B200 design as gll_stage.cu (marching strips, TMA row ring, one thread
// per element line); what the GL point sets add:
//  * traces are interpolated (DG: Alg. 2; SD: flux points 0 and n of a line),
//    the W neighbour's E trace is interpolated by the thread on its right from
//    the ring, the N/S traces from the element's columns;
//  * DG is evaluated in the weak form of Eq. (19) with n-point GL collocation
//    (SURVEY C6), sum-factorised and divided by the diagonal mass w_a w_b:
//    R = (2/dx)[sum_l (w_l/w_a) l'_a(xi_l) f_l - (l_a(1) F^E - l_a(-1) F^W)/w_a]
//      + (2/dy)[... g, F^N, F^S ...]  -- only the Rusanov face fluxes enter, no
//    interpolated edge flux and no jump pass (one barrier per row fewer than
//    the equivalent strong form with the g_DG correction, SBP identity P7);
//  * SD interpolates each line and each column to its n+1 flux points, evaluates
//    the interior flux points and differentiates the flux polynomial at the
//    solution points; the end flux points carry the Rusanov fluxes;
//  * the N face flux of row j is carried to row j+1 as its S face flux.
#include <cstring>

#include "common.cuh"
#include "ops_tables.h"
#include "tma.cuh"

namespace h2d {

namespace {

// strip width (elements) per method and order: DG keeps g of every point in
// smem, so narrower strips keep 2+ CTAs per SM (A/B on 4096^2: DG 16 > 32 by
// 37 % at P3, 3-6 % at P2/P4; SD 32 > 16 by 10 % at P3, 16 > 32 by 13 % at P4)
#ifndef H2D_DG_TX
#define H2D_DG_TX (K == 3 ? 14 : 12)  // P3: 14-element strips = 16-slot TMA rows, 4 CTAs/SM (+7.5 % over 16);
                                     // P4: 12 (60 threads) at 4 CTAs/SM since the by-column layout and the
                                     // 5-entry table copy shrank shared memory (+3.3 % over 11)
#endif
#ifndef H2D_SD_TX
#define H2D_SD_TX (K == 3 ? 14 : 12)  // A/B: P3 14 +2.5 % over 32; P4 12 (4 CTAs/SM, +4.2 % over 11)
#endif
#ifndef H2D_LMINB
#define H2D_LMINB 1
#endif
// A/B on 8192^2 / 4096^2 (round 1): P1 at 4 CTAs/SM (<= 128 registers; SD +7 %),
// P2 32-element strips at 4 CTAs/SM (DG +20 %, SD +36 % over 16 at 1)
#ifndef H2D_LMINB4
#define H2D_LMINB4 H2D_LMINB
#endif
#ifndef H2D_LMINB1
#define H2D_LMINB1 4
#endif
#ifndef H2D_LTX2
#define H2D_LTX2 32
#endif
#ifndef H2D_LMINB2
#define H2D_LMINB2 4
#endif
#ifndef H2D_DG_TX2
#define H2D_DG_TX2 30  // DG P2: 90 threads, 4 CTAs/SM (its g buffer: 32 fits 3; +2.7 %)
#endif
enum { LM_DG = 2, LM_SD = 4 };
#ifndef H2D_Q0LATE
#define H2D_Q0LATE 1
#endif
#ifndef H2D_VIEWCARRY
#define H2D_VIEWCARRY 1  // a row's view of the ring (source, piece offsets) computed once, carried to the next row
#endif
#ifndef H2D_Q0TMA
#define H2D_Q0TMA 1
#endif
#ifndef H2D_WSQRT
#define H2D_WSQRT fsqrt_ws  // Rusanov dissipation speed (common.cuh; A/B: fsqrt)
#endif
// y work by column: the thread of line b also owns column b of its element for
// the y direction (the column's fluxes, its S / N face fluxes -- the S one
// carried in registers from the row below -- and the y derivative at the
// column's points) and hands the y part of the residual to the line owners
// through shared memory: N points per thread cross shared memory instead of
// the N^2 column fluxes (DG g, SD interior flux points) and the 2N face fluxes
// every line thread read (0: the round-2 layout, A/B)
#ifndef H2D_GL_COLY
#define H2D_GL_COLY 1
#endif
#ifndef H2D_GL_RESPAD
#define H2D_GL_RESPAD 0
#endif
template <int M, int K> struct LTile {
  static constexpr int TX = K == 1 ? 64 : K == 2 ? (M == LM_DG ? H2D_DG_TX2 : H2D_LTX2) : (M == LM_DG ? H2D_DG_TX : H2D_SD_TX),
                       RB = 64;
  static constexpr int MINB = K == 1 ? H2D_LMINB1 : K == 2 ? H2D_LMINB2 : K == 3 ? H2D_LMINB : H2D_LMINB4;
};

constexpr int NSTG = 3;

struct LMaps {
  CUtensorMap q, lo, hi;
  CUtensorMap q0;  // (Q0T) q^n, box {16, TX, 4}
};

// operator table (kernel parameter: compile-time indices become constant-bank operands)
template <int K>
struct LOps {
  static constexpr int N = K + 1;
  static constexpr int EL = 0;                 // l_l(-1)
  static constexpr int ER = EL + N;            // l_l(+1)
  static constexpr int SI = ER + N;            // sd_I[N+1][N]
  static constexpr int SD = SI + (N + 1) * N;  // sd_D[N][N+1]
  static constexpr int DV = SD + N * (N + 1);  // DG volume operator (w_l / w_a) l'_a(xi_l)  [N][N]
  static constexpr int SR = DV + N * N;        // DG surface weights l_a(+1) / w_a
  static constexpr int SL = SR + N;            // DG surface weights l_a(-1) / w_a
  static constexpr int W = SL + N;             // GL weights (element averages, Alg. 9)
  static constexpr int TOT = W + N;
};
struct LTab {
  double v[10 + 30 + 30 + 25 + 10 + 5];
};
template <int K>
LTab make_ltab() {
  using O = Ops<K>;
  using T = LOps<K>;
  constexpr int N = K + 1;
  LTab t{};
  for (int a = 0; a < N; ++a) {
    t.v[T::EL + a] = O::eL_gl[a];
    t.v[T::ER + a] = O::eR_gl[a];
    for (int r = 0; r <= N; ++r) {
      t.v[T::SI + r * N + a] = O::sd_I[r][a];
      t.v[T::SD + a * (N + 1) + r] = O::sd_D[a][r];
    }
    for (int l = 0; l < N; ++l) t.v[T::DV + a * N + l] = O::dg_vol[a][l];
    t.v[T::SR + a] = O::dg_sR[a];
    t.v[T::SL + a] = O::dg_sL[a];
    t.v[T::W + a] = O::w_gl[a];
  }
  return t;
}

template <int M, int K>
struct L {
  static constexpr int N = K + 1, NP = N * N;
  static constexpr int TX = LTile<M, K>::TX, RB = LTile<M, K>::RB, NT = TX * N;
  static constexpr bool SWZ = (NP == 16);
  static constexpr int NSL = TX + 2;
  static constexpr int CW = (NP + 1 + 1) & ~1;
  static constexpr int CM = ((TX * NP + 1) + 1) & ~1;
  static constexpr int CREG = CW + CM + CW;
  static constexpr int RSW = (NSL + 7) & ~7;
  static constexpr int FIXO = 4 * RSW * 16;
  static constexpr int STG = SWZ ? FIXO + 8 * 16 : 4 * CREG;
  static constexpr int STGA = H2D_STGA(STG);  // stage stride (see H2D_STGA)
  static constexpr int OR_ = 0;
  // Q0T (P3): q^n of a row by TMA into a 2-row swizzled ring two rows ahead (as gll_stage.cu)
  static constexpr bool Q0T = H2D_Q0TMA && SWZ;
  static constexpr int QSTG = 4 * TX * 16;                  // one q^n row: [4 x TX rows of 16]
  static constexpr int OQT = OR_ + NSTG * STGA;             // (Q0T) q^n ring [2][QSTG]
  static constexpr int OFW = OQT + (Q0T ? 2 * QSTG : 0);    // W-face fluxes [TX+1][N][4]
#if H2D_GL_COLY
  // y part of the residual of every point, written by the thread that owns the
  // point's column, read by the one that owns its line: element lx, point
  // (row a, column x) at lx * RES + x * RCS + a * 4.  The column stride is 2 mod
  // 4 doubles (a column's writes by the N column threads fall into different
  // 16-B bank groups) and RES is 8 mod 16 doubles (the two elements of a
  // quarter warp 64 B apart; odd N: no element padding -- the lane groups of
  // an element do not align with quarter warps anyway)
  static constexpr int RCS = N * 4 + 2,
                       RES = (N % 2 && !H2D_GL_RESPAD) ? N * RCS : N * RCS + ((8 - (N * RCS) % 16) + 16) % 16;
  static constexpr int ORY = OFW + (TX + 1) * N * 4;
  static constexpr int OT = ORY + TX * RES;
#else
  static constexpr int OFN = OFW + (TX + 1) * N * 4;       // N-face fluxes, double-buffered [2][TX][N][4]
  static constexpr int OG = OFN + 2 * TX * N * 4;          // DG: g at points [TX][NP][4]
  // per-element strides padded to 2 mod 4 doubles: the column reads of 8
  // elements of a warp then fall into 8 different 16-B bank groups
  static constexpr int GS = NP * 4 + 2, PYS = N * (N - 1) * 4 + 2;
  static constexpr int OPY = OG + (M == LM_DG ? TX * GS : 0);        // SD: column interior fluxes [TX][N][N-1][4]
  static constexpr int OT = OPY + (M == LM_SD ? TX * PYS : 0);
#endif
  // operator table copy for run-time (line-dependent) indices: by column only
  // the weights of the element averages are indexed by the line
  static constexpr int TOFF = H2D_GL_COLY ? LOps<K>::W : 0, TSZ = H2D_GL_COLY ? N : LOps<K>::TOT;
  static constexpr int ORD = OT + ((TSZ + 1) & ~1);
  static constexpr int OB = ORD + 32;
  static constexpr int OQ0 = OB + ((NSTG + 2 + 1) & ~1);  // q^n prefetch [4][N][NT], thread-private (!Q0T)
  static constexpr int TOTAL = OQ0 + (Q0T ? 0 : 4 * N * NT);
  static_assert(!Q0T || (QSTG % 128 == 0 && OQT % 128 == 0), "1024-B aligned q^n stages");
  static constexpr size_t SMEM = TOTAL * sizeof(double);
};

// cp.async of this thread's q^n line into its private smem slots, one row ahead
// (even N and 16-B aligned lines: 16-B pieces, layout [c][x/2][thread] of double2;
// else 8-B pieces, layout [c][x][thread])
template <int N, int NT>
__device__ __forceinline__ void q0_prefetch(double* sq0, const double* q0, long long cs, long long base, int tid,
                                            bool vec) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double* s = q0 + c * cs + base;
    if (N % 2 == 0 && vec) {
#pragma unroll
      for (int x = 0; x < N; x += 2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sq0 + (c * N + x) * NT + 2 * tid)),
                     "l"(s + x)
                     : "memory");
    } else {
#pragma unroll
      for (int x = 0; x < N; ++x)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sq0 + (c * N + x) * NT + tid)),
                     "l"(s + x)
                     : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void st4(double* p, const double v[4]) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
}
__device__ __forceinline__ void ld4(const double* p, double v[4]) {
  const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
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
__device__ __forceinline__ const double* row_src(const StageArgs& a, int jr, int np, long long& cs) {
  if (jr < 0) { cs = a.gcs; return a.ghost_lo; }
  if (jr >= a.nrows) { cs = a.gcs; return a.ghost_hi; }
  cs = a.cs;
  return a.q + (long long)jr * a.nx * np;
}
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

// V (stage variant, compile time): bit 0 q^n read, bit 1 dt / non-physical
// epilogue, bit 2 fused element averages (as gll_stage_kernel)
template <int M, int K, int V>
__global__ void __launch_bounds__(L<M, K>::NT, LTile<M, K>::MINB) gl_stage_kernel(const StageArgs a, const LTab tab,
                                                               const __grid_constant__ LMaps maps) {
  // V == 8: any other combination, decided at run time from the pointers
  const bool HQ0 = V == 8 ? a.q0 != nullptr : (V & 1), HLAM = V == 8 ? (a.lam || a.bad) : (V & 2) != 0,
             HAVG = V == 8 ? a.qbar != nullptr : (V & 4) != 0;
  using H = L<M, K>;
  using T = LOps<K>;
  constexpr int N = H::N, NP = H::NP, TX = H::TX, NT = H::NT, NSL = H::NSL;
  constexpr int CW = H::CW, CM = H::CM, CREG = H::CREG, STGA = H::STGA;
  extern __shared__ __align__(1024) double4 smem4[];
  double* sm = reinterpret_cast<double*>(smem4);
  double* ring = sm + H::OR_;
  double* sFW = sm + H::OFW;
#if H2D_GL_COLY
  double* sRY = sm + H::ORY;
#else
  double* sFN = sm + H::OFN;
  double* sG = sm + H::OG;
  double* sPY = sm + H::OPY;
#endif
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
  // vector global access: every line start 32-B (P3) / 16-B (P1) aligned in out and q^n
  const unsigned long long amask = N == 4 ? 31ull : 15ull;
  const bool vec = ((((unsigned long long)a.out | (unsigned long long)a.q0 |
                      (unsigned long long)(a.cs * 8)) & amask) == 0);
  const bool mirW = (i0 == 0 && a.bcx), mirE = (i0 + TXv == a.nx && a.bcx);
  const bool wrapW = (i0 == 0 && !a.bcx), wrapE = (i0 + TXv == a.nx && !a.bcx);
  const int iw = i0 > 0 ? i0 - 1 : a.nx - 1;
  const int ie = i0 + TXv < a.nx ? i0 + TXv : 0;
  const int nload = RBv + 2;

  for (int i = tid; i < H::TSZ; i += NT) sT[i] = tab.v[H::TOFF + i];
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

  auto issue_row = [&](int Lr) {
    if (tid != 0) return;
    const int jr = jb - 1 + Lr;
    long long cs;
    const double* rb = row_src(a, jr, NP, cs);
    uint64_t* br = &bar[Lr % NSTG];
    double* st = ring + (Lr % NSTG) * STGA;
    if (!rb) { mbar_arrive_expect_tx(br, 0); return; }
    if constexpr (H::SWZ) {
      const CUtensorMap* mp = jr < 0 ? &maps.lo : (jr >= a.nrows ? &maps.hi : &maps.q);
      const int y0 = (jr < 0 || jr >= a.nrows ? 0 : jr * a.nx) + i0 - 1;
      uint32_t tx = 4u * NSL * 128u;
      if (wrapW) tx += 4u * 128u;
      if (wrapE) tx += 4u * 128u;
      mbar_arrive_expect_tx(br, tx);
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
  struct RowView {
    const double* st;
    int dW, dM, dE, csodd;
    bool have;
  };
  const bool has_glo = a.ghost_lo != nullptr, has_ghi = a.ghost_hi != nullptr;
  auto view = [&](int Lr) {
    RowView v;
    v.st = ring + (Lr % NSTG) * STGA;
    v.dW = v.dM = v.dE = 0;
    v.csodd = 0;
    if constexpr (H::SWZ) {  // (the 128-B rows need no piece offsets: only whether the row exists)
      const int jr = jb - 1 + Lr;
      v.have = jr < 0 ? has_glo : (jr >= a.nrows ? has_ghi : true);
      return v;
    }
    long long cs;
    const double* rb = row_src(a, jb - 1 + Lr, NP, cs);
    v.have = rb != nullptr;
    v.csodd = (int)(cs & 1);
    if (!H::SWZ && rb) {
      v.dM = piece_off(rb + (long long)i0 * NP);
      v.dW = piece_off(rb + (long long)iw * NP);
      v.dE = piece_off(rb + (long long)ie * NP);
    }
    return v;
  };
  auto own_at = [&](const RowView& v, int c, int e, int p) -> double {
    if constexpr (H::SWZ) {
      return v.st[(c * H::RSW + e) * 16 + ((((p >> 1) ^ (e & 7)) << 1) | (p & 1))];
    } else {
      return v.st[c * CREG + CW + (v.dM ^ (c & v.csodd)) + (e - 1) * NP + p];
    }
  };
  // value (c, p) of any slot e (0 W halo, TXv+1 E halo): the index is selected,
  // not branched on (no divergent regions in the face work)
  auto any_at = [&](const RowView& v, int c, int e, int p) -> double {
    if constexpr (H::SWZ) {
      const bool fw = (e == 0 && wrapW), fe = (e == TXv + 1 && wrapE);
      const int iS = (c * H::RSW + e) * 16 + ((((p >> 1) ^ (e & 7)) << 1) | (p & 1));
      const int iF = H::FIXO + ((fe ? 4 : 0) + c) * 16 + p;
      return v.st[(fw || fe) ? iF : iS];
    } else {
      const int iW = c * CREG + (v.dW ^ (c & v.csodd)) + p;
      const int iE = c * CREG + CW + CM + (v.dE ^ (c & v.csodd)) + p;
      const int iM = c * CREG + CW + (v.dM ^ (c & v.csodd)) + (e - 1) * NP + p;
      return v.st[e == 0 ? iW : (e == TXv + 1 ? iE : iM)];
    }
  };
  // interpolation of a line (dir 0: row bb of slot e) or column (dir 1: column bb)
  // of the element in slot e with the weights w[l]
  auto interp = [&](const RowView& v, int e, int dir, int bb, const double* w, double out[4], bool anyslot) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double s;  // (sums start from their first product: no zero-initialised accumulators)
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const int p = dir == 0 ? bb * N + l : l * N + bb;
        const double val = anyslot ? any_at(v, c, e, p) : own_at(v, c, e, p);
        s = l == 0 ? w[l] * val : fma(w[l], val, s);
      }
      out[c] = s;
    }
  };

  for (int Lr = 0; Lr < NSTG && Lr < nload; ++Lr) issue_row(Lr);
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
  } else if (HQ0 && own) {  // q^n of the first own row
    q0_prefetch<N, NT>(sQ0, a.q0, a.cs, ((long long)jb * a.nx + i0 + lx) * NP + b * N, tid, vec);
  }

  double lam = 0.0;
  const double bdt = a.bcoef * dtv;
  const double cx = bdt * a.rdx2, cy = bdt * a.rdy2;  // metric x dt folded (R below is bdt R)
  const double* EL = tab.v + T::EL;
  const double* ER = tab.v + T::ER;
  const double* SI0 = tab.v + T::SI;               // flux point 0 row of sd_I (== eL)
  const double* SIN = tab.v + T::SI + N * N;       // flux point n row (== eR)

#if H2D_GL_COLY
  double FSr[4] = {0.0, 0.0, 0.0, 0.0};  // S-face flux of this thread's column (the row below's N face)
#endif
  RowView vcar = view(0);  // (H2D_VIEWCARRY) the next row's view, carried
  for (int Lr = 0; Lr <= RBv; ++Lr) {
    mbar_wait(&bar[Lr % NSTG], (Lr / NSTG) & 1);
    mbar_wait(&bar[(Lr + 1) % NSTG], ((Lr + 1) / NSTG) & 1);
    const RowView vc = H2D_VIEWCARRY ? vcar : view(Lr), vn = view(Lr + 1);
    vcar = vn;
#if !H2D_GL_COLY
    double* FNc = sFN + (Lr & 1) * TX * N * 4;        // N-face fluxes of this row (written now)
    double* FSc = sFN + ((Lr + 1) & 1) * TX * N * 4;  // S-face fluxes of this row (written in step Lr-1)
#endif
    const long long jr = jb - 1 + Lr;

    double q[4][N];
    double phi[N + 1][4];           // SD: x flux-point fluxes (interior; [0] = F^W)
    double fl[4][N];                // DG: x fluxes of the line
    double lpart[4] = {0.0, 0.0, 0.0, 0.0};  // limiter runs: the line's share of the element average
    // Face work of the row, straight-line so that the independent node
    // evaluations interleave: the W face of each line (its W neighbour's E trace
    // interpolated here), the N face of column b of each element (own N trace vs
    // the next row's S trace; carried as that row's S face); transmissive ends
    // by selects.
    if (own) {
      const double* wl = (M == LM_DG) ? EL : SI0;
      const double* wr = (M == LM_DG) ? ER : SIN;
      double qd[4], qu[4];
#if H2D_GL_COLY
      // column b of the element, read once: its N trace here, its fluxes below
      // (the prologue row's slot may hold no row: its values are then unused)
      double colv[4][N];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int l = 0; l < N; ++l) colv[c][l] = own_at(vc, c, lx + 1, l * N + b);
      {
        double u[4];
        interp(vn, lx + 1, 1, b, wl, u, false);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double s = wr[0] * colv[c][0];
#pragma unroll
          for (int l = 1; l < N; ++l) s = fma(wr[l], colv[c][l], s);
          qd[c] = vc.have ? s : u[c];
          qu[c] = vn.have ? u[c] : s;
        }
      }
#else
      {
        double d[4], u[4];
        interp(vc, lx + 1, 1, b, wr, d, false);
        interp(vn, lx + 1, 1, b, wl, u, false);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          qd[c] = vc.have ? d[c] : u[c];
          qu[c] = vn.have ? u[c] : d[c];
        }
      }
#endif
      if (Lr > 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int x = 0; x < N; ++x) {
            if constexpr (H::SWZ) {  // 16-B chunks: points (4b + 2h, 4b + 2h + 1)
              if ((x & 1) == 0) {
                const double2 u = *reinterpret_cast<const double2*>(
                    vc.st + (c * H::RSW + lx + 1) * 16 + (((2 * b + (x >> 1)) ^ ((lx + 1) & 7)) << 1));
                q[c][x] = u.x;
                q[c][x + 1] = u.y;
              }
            } else {
              q[c][x] = own_at(vc, c, lx + 1, b * N + x);
            }
          }
        double qw[4], qe[4], ql[4], sw, se, sl, fW[4], fE[4], flf[4], gd[4], sd, gu[4], su;
        {
          double v[4];
          if constexpr (H::SWZ) {  // E trace of the W neighbour's line: its row b as two 16-B chunks
            const bool fw = (lx == 0 && wrapW);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              double row[N];
#pragma unroll
              for (int h = 0; h < N / 2; ++h) {
                const int iS = (c * H::RSW + lx) * 16 + (((2 * b + h) ^ (lx & 7)) << 1);
                const int iF = H::FIXO + c * 16 + N * b + 2 * h;
                const double2 u2 = *reinterpret_cast<const double2*>(vc.st + (fw ? iF : iS));
                row[2 * h] = u2.x;
                row[2 * h + 1] = u2.y;
              }
              double sv = wr[0] * row[0];
#pragma unroll
              for (int l = 1; l < N; ++l) sv = fma(wr[l], row[l], sv);
              v[c] = sv;
            }
          } else {
            interp(vc, lx, 0, b, wr, v, true);  // E trace of the W neighbour's line
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double s0 = wl[0] * q[c][0], s1 = wr[0] * q[c][0];
#pragma unroll
            for (int l = 1; l < N; ++l) { s0 = fma(wl[l], q[c][l], s0); s1 = fma(wr[l], q[c][l], s1); }
            qw[c] = s0;
            qe[c] = s1;
          }
          const bool mw = (lx == 0 && mirW);
#pragma unroll
          for (int c = 0; c < 4; ++c) ql[c] = mw ? qw[c] : v[c];
        }
        node_eval<0>(qw, gm1, gam, fW, sw);
        node_eval<0>(qe, gm1, gam, fE, se);
        node_eval<0>(ql, gm1, gam, flf, sl);
        node_eval<1>(qd, gm1, gam, gd, sd);
        node_eval<1>(qu, gm1, gam, gu, su);
        if (M == LM_DG) {
#if H2D_GL_COLY  // f at every point of the line (registers); g at the column's points below
#pragma unroll
          for (int x = 0; x < N; ++x) {
            double v[4] = {q[0][x], q[1][x], q[2][x], q[3][x]}, f[4];
            flux<0>(v, prims(v, gm1), f);
#pragma unroll
            for (int c = 0; c < 4; ++c) fl[c][x] = f[c];
          }
#else  // f (registers) and g (smem, for the columns) at every point of the line
#pragma unroll
          for (int x = 0; x < N; ++x) {
            double v[4] = {q[0][x], q[1][x], q[2][x], q[3][x]}, f[4], g[4];
            const Prim w = prims(v, gm1);
            flux<0>(v, w, f);
            flux<1>(v, w, g);
#pragma unroll
            for (int c = 0; c < 4; ++c) fl[c][x] = f[c];
            st4(sG + lx * H::GS + (b * N + x) * 4, g);
          }
#endif
        } else {  // SD: interior x flux points of the line, interior y flux points of column b
#pragma unroll
          for (int r = 1; r < N; ++r) {
            double v[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              double s = tab.v[T::SI + r * N] * q[c][0];
#pragma unroll
              for (int l = 1; l < N; ++l) s = fma(tab.v[T::SI + r * N + l], q[c][l], s);
              v[c] = s;
            }
            flux<0>(v, prims(v, gm1), phi[r]);
          }
#if !H2D_GL_COLY
          // column b of the element, read once for its N-1 interior flux points
          double colv[4][N];
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int l = 0; l < N; ++l) colv[c][l] = own_at(vc, c, lx + 1, l * N + b);
#pragma unroll
          for (int r = 1; r < N; ++r) {
            double v[4], g[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              double sv = tab.v[T::SI + r * N] * colv[c][0];
#pragma unroll
              for (int l = 1; l < N; ++l) sv = fma(tab.v[T::SI + r * N + l], colv[c][l], sv);
              v[c] = sv;
            }
            flux<1>(v, prims(v, gm1), g);
            st4(sPY + lx * H::PYS + (b * (N - 1) + (r - 1)) * 4, g);
          }
#endif
        }
        double F[4], G[4];
        rus(ql, flf, sl, qw, fW, sw, F);
        rus(qd, gd, sd, qu, gu, su, G);
        st4(sFW + (lx * N + b) * 4, F);
#if H2D_GL_COLY
        {  // y part of the residual at the points (a, b) of column b, to their line owners
          double gc[N + 1][4];  // DG: g at the column's points; SD: g at its interior flux points 1..N-1
          if (M == LM_DG) {
#pragma unroll
            for (int l = 0; l < N; ++l) {
              double v[4] = {colv[0][l], colv[1][l], colv[2][l], colv[3][l]};
              flux<1>(v, prims(v, gm1), gc[l]);
            }
          } else {
#pragma unroll
            for (int r = 1; r < N; ++r) {
              double v[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                double sv = tab.v[T::SI + r * N] * colv[c][0];
#pragma unroll
                for (int l = 1; l < N; ++l) sv = fma(tab.v[T::SI + r * N + l], colv[c][l], sv);
                v[c] = sv;
              }
              flux<1>(v, prims(v, gm1), gc[r]);
            }
          }
#pragma unroll
          for (int aa = 0; aa < N; ++aa) {
            double gy[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              if (M == LM_DG) {  // sum_l (w_l/w_a) l'_a(eta_l) g_l + (l_a(-1) F^S - l_a(1) F^N) / w_a
                double s = tab.v[T::DV + aa * N] * gc[0][c];
#pragma unroll
                for (int l = 1; l < N; ++l) s = fma(tab.v[T::DV + aa * N + l], gc[l][c], s);
                gy[c] = s + tab.v[T::SL + aa] * FSr[c] - tab.v[T::SR + aa] * G[c];
              } else {  // sum_r D_ar g_r over the flux points, the end ones the face fluxes
                double s = tab.v[T::SD + aa * (N + 1)] * FSr[c] + tab.v[T::SD + aa * (N + 1) + N] * G[c];
#pragma unroll
                for (int r = 1; r < N; ++r) s += tab.v[T::SD + aa * (N + 1) + r] * gc[r][c];
                gy[c] = s;
              }
            }
            st4(sRY + lx * H::RES + b * H::RCS + aa * 4, gy);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) FSr[c] = G[c];
        }
#else
        st4(FNc + (lx * N + b) * 4, G);
#endif
#pragma unroll
        for (int c = 0; c < 4; ++c) phi[0][c] = F[c];
        if (lx == TXv - 1) {  // the strip's last E face
          if (mirE) {
            rus(qe, fE, se, qe, fE, se, G);
          } else {
            double qr[4], fr[4], sr;
            interp(vc, TXv + 1, 0, b, wl, qr, true);
            node_eval<0>(qr, gm1, gam, fr, sr);
            rus(qe, fE, se, qr, fr, sr, G);
          }
          st4(sFW + (TXv * N + b) * 4, G);
        }
      } else {  // prologue row (below the march): only its N face, as the first row's S face
        double gd[4], sd, gu[4], su, G[4];
        node_eval<1>(qd, gm1, gam, gd, sd);
        node_eval<1>(qu, gm1, gam, gu, su);
        rus(qd, gd, sd, qu, gu, su, G);
#if H2D_GL_COLY
#pragma unroll
        for (int c = 0; c < 4; ++c) FSr[c] = G[c];
#else
        st4(FNc + (lx * N + b) * 4, G);
#endif
      }
    }
    __syncthreads();

    if (Lr > 0 && own) {
      const long long base = (jr * a.nx + i0 + lx) * NP + b * N;
      if (HQ0) {
        if (H::Q0T) mbar_wait(&qbar[(Lr - 1) & 1], ((Lr - 1) >> 1) & 1);
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      const double* q0s = sQT + ((Lr - 1) & 1) * H::QSTG;  // (Q0T) this row's q^n slot
#define Q0V(c, x)                                                                                           \
  (H::Q0T ? q0s[((c) * TX + lx) * 16 +                                                                      \
                ((((2 * b + ((x) >> 1)) ^ (((c) * TX + lx) & 7)) << 1) | ((x) & 1))]                        \
   : (N % 2 == 0 && vec ? sQ0[((c) * N + ((x) & ~1)) * NT + 2 * tid + ((x) & 1)]                             \
                        : sQ0[((c) * N + (x)) * NT + tid]))
      double FW[4], FE[4];
      ld4(sFW + (lx * N + b) * 4, FW);
      ld4(sFW + ((lx + 1) * N + b) * 4, FE);
      if (M == LM_SD) {
#pragma unroll
        for (int c = 0; c < 4; ++c) phi[N][c] = FE[c];
      }
      double ov[4][N], q0v[4][N];  // q^n of the line (0 in stage 1: a0 = 0)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int x = 0; x < N; ++x) q0v[c][x] = HQ0 ? Q0V(c, x) : 0.0;
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double v[4] = {q[0][x], q[1][x], q[2][x], q[3][x]};
        double R[4];
#if H2D_GL_COLY
        double gy[4];  // y part of the residual at (b, x), from the owner of column x
        ld4(sRY + lx * H::RES + x * H::RCS + b * 4, gy);
        if (M == LM_DG) {
          const double sRa = tab.v[T::SR + x], sLa = tab.v[T::SL + x];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double fx = tab.v[T::DV + x * N] * fl[c][0];
#pragma unroll
            for (int l = 1; l < N; ++l) fx = fma(tab.v[T::DV + x * N + l], fl[c][l], fx);
            fx += sLa * FW[c] - sRa * FE[c];
            R[c] = fma(cx, fx, cy * gy[c]);  // bdt R, R = (2/dx) fx + (2/dy) gy (weak form signs)
          }
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double fx = tab.v[T::SD + x * (N + 1)] * phi[0][c];
#pragma unroll
            for (int r = 1; r <= N; ++r) fx = fma(tab.v[T::SD + x * (N + 1) + r], phi[r][c], fx);
            R[c] = fma(-cx, fx, -cy * gy[c]);  // bdt R, R = -(2/dx) fx - (2/dy) gy
          }
        }
#else
        double FS[4], FN[4];
        ld4(FSc + (lx * N + x) * 4, FS);
        ld4(FNc + (lx * N + x) * 4, FN);
        if (M == LM_DG) {
          // weak form, Eq. (19) / SURVEY C6 divided by w_a:
          // (2/dx) [sum_l (w_l/w_a) l'_a(xi_l) f_l - (l_a(1) F^E - l_a(-1) F^W) / w_a] + (y likewise)
          double gy[4];
#pragma unroll
          for (int l = 0; l < N; ++l) {  // column x of the element: g of its points (16-B smem reads)
            double g[4];
            ld4(sG + lx * H::GS + (l * N + x) * 4, g);
            const double dv = sT[T::DV + b * N + l];
#pragma unroll
            for (int c = 0; c < 4; ++c) gy[c] = l == 0 ? dv * g[c] : fma(dv, g[c], gy[c]);
          }
          const double sRa = tab.v[T::SR + x], sLa = tab.v[T::SL + x];
          const double sRb = sT[T::SR + b], sLb = sT[T::SL + b];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double fx = tab.v[T::DV + x * N] * fl[c][0];
#pragma unroll
            for (int l = 1; l < N; ++l) fx = fma(tab.v[T::DV + x * N + l], fl[c][l], fx);
            fx += sLa * FW[c] - sRa * FE[c];
            const double g2 = gy[c] + sLb * FS[c] - sRb * FN[c];
            R[c] = fma(cx, fx, cy * g2);  // bdt R, R = (2/dx) fx + (2/dy) g2 (weak form signs)
          }
        } else {  // SD
          double gy[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) gy[c] = sT[T::SD + b * (N + 1) + 0] * FS[c] + sT[T::SD + b * (N + 1) + N] * FN[c];
#pragma unroll
          for (int r = 1; r < N; ++r) {  // interior y flux points of column x (16-B smem reads)
            double pv[4];
            ld4(sPY + lx * H::PYS + (x * (N - 1) + (r - 1)) * 4, pv);
            const double dr = sT[T::SD + b * (N + 1) + r];
#pragma unroll
            for (int c = 0; c < 4; ++c) gy[c] += dr * pv[c];
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double fx = tab.v[T::SD + x * (N + 1)] * phi[0][c];
#pragma unroll
            for (int r = 1; r <= N; ++r) fx = fma(tab.v[T::SD + x * (N + 1) + r], phi[r][c], fx);
            R[c] = fma(-cx, fx, -cy * gy[c]);  // bdt R, R = -(2/dx) fx - (2/dy) gy
          }
        }
#endif
#pragma unroll
        for (int c = 0; c < 4; ++c) ov[c][x] = HQ0 ? fma(a.a0, q0v[c][x], fma(a.a1, v[c], R[c])) : fma(a.a1, v[c], R[c]);
      }
      if (HLAM) {  // dt wave speed and non-physical check (straight-line)
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
#undef Q0V
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
      if (!H::Q0T && HQ0 && Lr < RBv && !H2D_Q0LATE)  // q^n of the next row into the consumed private slots
        q0_prefetch<N, NT>(sQ0, a.q0, a.cs, base + (long long)a.nx * NP, tid, vec);
      if (HAVG) {  // this line's share of the element average: w_b sum_x w_x q
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double sx = 0.0;
#pragma unroll
          for (int x = 0; x < N; ++x) sx += tab.v[T::W + x] * ov[c][x];
          lpart[c] = sT[T::W - H::TOFF + b] * sx;
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
      if (Lr > 0 && own && b == 0) {
        const long long m = jr * a.nx + i0 + lx, ne = (long long)a.nx * a.nrows;
#pragma unroll
        for (int c = 0; c < 4; ++c) a.qbar[c * ne + m] = 0.25 * lpart[c];
      }
    } else if (HAVG) {  // element averages (N = 3, 5: through the W-face buffer)
      __syncthreads();
      if (Lr > 0 && own) st4(sFW + (lx * N + b) * 4, lpart);
      __syncthreads();
      if (Lr > 0 && own) {
        const long long m = jr * a.nx + i0 + lx, ne = (long long)a.nx * a.nrows;
        for (int c = b; c < 4; c += N) {
          double s = 0.0;
#pragma unroll
          for (int bb = 0; bb < N; ++bb) s += sFW[(lx * N + bb) * 4 + c];
          a.qbar[c * ne + m] = 0.25 * s;
        }
      }
    }
    __syncthreads();
    if (Lr + NSTG < nload) {
      if (tid == 0) fence_proxy_async_smem();
      issue_row(Lr + NSTG);
    }
    // q^n of the next row into the consumed private slots -- after the proxy
    // fence of the TMA issue: the fence waits for this thread's in-flight
    // cp.async writes, so a prefetch issued before it stalled warp 0 for a
    // global-memory round trip every row (H2D_Q0LATE=0: the round-2 order)
    if (!H::Q0T && H2D_Q0LATE && HQ0 && own && Lr > 0 && Lr < RBv)
      q0_prefetch<N, NT>(sQ0, a.q0, a.cs, ((long long)(jb + Lr) * a.nx + i0 + lx) * NP + b * N, tid, vec);
    if (H::Q0T && HQ0 && Lr > 0 && Lr + 1 < RBv) {  // q^n two rows ahead into the slot this row consumed
      if (tid == 0) fence_proxy_async_smem();
      issue_q0(Lr + 1);
    }
  }
  if (HLAM && a.lam) block_max_to(lam, a.lam, sm + H::ORD);
}

template <int M, int K, int V>
static cudaError_t launch_lv(dim3 grid, const StageArgs& b, const LTab& tab, const LMaps& maps, cudaStream_t s) {
  using H = L<M, K>;
  static std::atomic<unsigned long long> attr{0};
  const cudaError_t e = smem_optin(gl_stage_kernel<M, K, V>, (int)H::SMEM, attr);
  if (e != cudaSuccess) return e;
  return launch_pdl_if(!b.no_pdl, gl_stage_kernel<M, K, V>, grid, dim3(H::NT), H::SMEM, s, b, tab, maps);
}

template <int M, int K>
static int launch_l(const StageArgs& a, cudaStream_t s) {
  using H = L<M, K>;
  static const LTab tab = make_ltab<K>();
  LMaps maps;
  memset(&maps, 0, sizeof(maps));
  if (H::SWZ) {
    const long long nel = (long long)a.nx * a.nrows;
    if (!make_map(&maps.q, a.q, nel, a.cs, H::NSL) || !make_map(&maps.lo, a.ghost_lo, a.nx, a.gcs, H::NSL) ||
        !make_map(&maps.hi, a.ghost_hi, a.nx, a.gcs, H::NSL) ||
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
    case 0: e = launch_lv<M, K, 0>(grid, b, tab, maps, s); break;
    case 1: e = launch_lv<M, K, 1>(grid, b, tab, maps, s); break;
    case 3: e = launch_lv<M, K, 3>(grid, b, tab, maps, s); break;
    case 4: e = launch_lv<M, K, 4>(grid, b, tab, maps, s); break;
    case 5: e = launch_lv<M, K, 5>(grid, b, tab, maps, s); break;
    default: e = launch_lv<M, K, 8>(grid, b, tab, maps, s); break;
  }
  return e != cudaSuccess ? (int)e : (int)cudaPeekAtLastError();
}

int launch_gl_stage(int method, int k, const StageArgs& a, cudaStream_t s) {
  if (k == 1) {  // P1: the element-per-lane warp kernel where it applies (p1_stage.cu)
    const int e = launch_p1_stage(method, a, s);
    if (e >= 0) return e;
  }
  if (method == LM_DG) {
    switch (k) {
      case 1: return launch_l<LM_DG, 1>(a, s);
      case 2: return launch_l<LM_DG, 2>(a, s);
      case 3: return launch_l<LM_DG, 3>(a, s);
      case 4: return launch_l<LM_DG, 4>(a, s);
    }
  } else if (method == LM_SD) {
    switch (k) {
      case 1: return launch_l<LM_SD, 1>(a, s);
      case 2: return launch_l<LM_SD, 2>(a, s);
      case 3: return launch_l<LM_SD, 3>(a, s);
      case 4: return launch_l<LM_SD, 4>(a, s);
    }
  }
  return (int)cudaErrorInvalidValue;
}

}  // namespace h2d
