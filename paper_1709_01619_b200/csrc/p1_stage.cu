// p1_stage.cu -- fused RK-stage kernel of the high-order methods at P1 (k = 1,
// 2 x 2 solution points per element): CPR (chain rule + Radau g_DG correction,
// P:226-238, Algs. 7-8), NDG (D[F] + lift, Eqs. (24)-(29)), DG (weak form on
// Gauss-Legendre points, Eqs. (18)-(21)) and SD (GL solution points, Chebyshev-
// Lobatto flux points {-1, 0, 1}, Eqs. (30)-(34)).  P1 is the order every table
// of the paper is printed at (Tables 1-4).
//
// The warp-strip design of the FV kernel (fv_stage.cu) with one ELEMENT per lane:
//  * every warp marches its own strip of 31 elements up the element rows (lane
//    31 works on the E halo element), no CTA barrier in the march;
//  * a lane holds its element's 4 points x 4 components in registers: all the
//    x AND y work of the element is lane-local (the line kernels exchange the
//    eta operands through shared memory);
//  * W face: the W neighbour's E trace from the shared-memory ring, the Rusanov
//    flux once per face point; E face: the right lane's W-face flux by a
//    shuffle; N face: with the element above (next ring row), carried to the
//    next row as its S face;
//  * rows stream into a per-warp ring by predicated cp.async, q^n through its own
//    ring one row ahead; SSP-RK combination, dt wave speed, non-physical check and
//    element averages fused in the epilogue; one 32-B store per component.
// Arithmetic per face point / solution point is that of the line kernels' (same
// helpers: prims, flux, jac_pair, Rusanov), so the residual matches the oracle
// to rounding.
#include "common.cuh"
#include "ops_tables.h"
#include "tma.cuh"

namespace h2d {

namespace {
enum { PM_CPR = 1, PM_DG = 2, PM_NDG = 3, PM_SD = 4 };
constexpr int PWPC = 2;                 // warps per CTA (independent strips)
constexpr int PWS = 31;                 // elements per warp strip (lane 31: the E halo element)
constexpr int PSL = 33;                 // ring slots per row: W halo element + 32 lanes
#ifndef H2D_P1W_DEPTH
#define H2D_P1W_DEPTH 1
#endif
constexpr int PWD = H2D_P1W_DEPTH, PWNS = 2 + PWD, PQS = PWD + 1;
constexpr int PRING = PWNS * 4 * PSL * 4, PQR = PQS * 4 * 32 * 4;  // doubles per warp
constexpr size_t p1_smem(bool hq0) { return sizeof(double) * ((size_t)PWPC * (PRING + (hq0 ? PQR : 0)) + PWPC); }

// Rusanov along DIR from two states with their physical fluxes and normal speeds
__device__ __forceinline__ void rus1(const double qL[4], const double fL[4], double sL, const double qR[4],
                                     const double fR[4], double sR, double F[4]) {
  const double lam = fmax(sL, sR);
#pragma unroll
  for (int c = 0; c < 4; ++c) F[c] = 0.5 * (fL[c] + fR[c]) - 0.5 * lam * (qR[c] - qL[c]);
}

// flux along DIR and normal speed |u_n| + c of a state (Rusanov dissipation speed)
template <int DIR>
__device__ __forceinline__ void feval(const double q[4], double gm1, double gam, double f[4], double& s) {
  const Prim w = prims(q, gm1);
  flux<DIR>(q, w, f);
  s = fabs(DIR == 0 ? w.u : w.v) + fsqrt_ws(gam * w.p * w.ri);
}
}  // namespace

// the P1 operator tables as device constants (literal indices into the generated
// constexpr tables are constant expressions)
struct P1Ops {
  double Dl[2][2], gL[2], gR[2], eL[2], eR[2], dv[2][2], sR[2], sL[2], sI1[2], sD[2][3], wl[2], wg[2];
};
constexpr P1Ops p1ops() {
  using O = Ops<1>;
  return P1Ops{{{O::D_gll[0][0], O::D_gll[0][1]}, {O::D_gll[1][0], O::D_gll[1][1]}},
               {O::gLp_gll[0], O::gLp_gll[1]},
               {O::gRp_gll[0], O::gRp_gll[1]},
               {O::eL_gl[0], O::eL_gl[1]},
               {O::eR_gl[0], O::eR_gl[1]},
               {{O::dg_vol[0][0], O::dg_vol[0][1]}, {O::dg_vol[1][0], O::dg_vol[1][1]}},
               {O::dg_sR[0], O::dg_sR[1]},
               {O::dg_sL[0], O::dg_sL[1]},
               {O::sd_I[1][0], O::sd_I[1][1]},
               {{O::sd_D[0][0], O::sd_D[0][1], O::sd_D[0][2]}, {O::sd_D[1][0], O::sd_D[1][1], O::sd_D[1][2]}},
               {O::w_gll[0], O::w_gll[1]},
               {O::w_gl[0], O::w_gl[1]}};
}

#ifndef H2D_P1W_MINB
#define H2D_P1W_MINB 4
#endif
template <int M, int V>
__global__ void __launch_bounds__(PWPC * 32, H2D_P1W_MINB) p1_warp_kernel(const StageArgs a) {
  constexpr P1Ops O = p1ops();
  constexpr bool GLL = (M == PM_CPR || M == PM_NDG);
  const bool HQ0 = (V & 1) != 0, HLAM = (V & 2) != 0, HAVG = (V & 4) != 0;
  extern __shared__ __align__(16) double p1_smem_[];
  double(*const ring)[PWNS][4][PSL * 4] = reinterpret_cast<double(*)[PWNS][4][PSL * 4]>(p1_smem_);
  double(*const qring)[PQS][4][32 * 4] = reinterpret_cast<double(*)[PQS][4][32 * 4]>(p1_smem_ + PWPC * PRING);
  double* const sred = p1_smem_ + PWPC * PRING + (HQ0 ? PWPC * PQR : 0);
  pdl_wait();
  pdl_launch();
  const double dtv = stage_dt(a);  // (stage 1 / 2 of a fused-dt step: publishes / commits the clock)
  if (dtv == 0.0) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i0 = (blockIdx.x * PWPC + wid) * PWS;
  int bhi;
  const int jb = band_start(a, bhi);
  const double gam = a.gamma, gm1 = a.gamma - 1.0;
  double lam = 0.0;
  if (i0 < a.nx) {  // warp-uniform
    const int TXv = min(PWS, a.nx - i0), RBv = min(a.rows, bhi - jb);
    const bool own = lane < TXv;
    const bool halo = lane == TXv;                                  // the E halo element
    const bool mirW = lane == 0 && i0 == 0 && a.bcx != 0;           // transmissive W end
    const bool mirE = halo && i0 + TXv == a.nx && a.bcx != 0;       // transmissive E end
    double(*const rw)[4][PSL * 4] = ring[wid];
    double(*const qw)[4][32 * 4] = qring[HQ0 ? wid : 0];
    // the lane's element (own, or the wrapped E halo) and lane 0's W neighbour
    int ie = i0 + lane;
    if (ie >= a.nx) ie = a.bcx == 0 ? ie - a.nx : a.nx - 1;
    const int iw = i0 > 0 ? i0 - 1 : (a.bcx == 0 ? a.nx - 1 : 0);
    const int pe = (own || (halo && !mirE)) ? 1 : 0, pw = (lane == 0 && !mirW) ? 1 : 0;
    auto row_ptr = [&](int jr, long long& cs) -> const double* {  // element row jr; nullptr: transmissive
      cs = a.cs;
      if (jr < 0) { cs = a.gcs; return a.ghost_lo; }
      if (jr >= a.nrows) { cs = a.gcs; return a.ghost_hi; }
      return a.q + (long long)jr * a.nx * 4;
    };
    auto cp16 = [](double* d, const double* g, int p) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p cp.async.cg.shared.global [%0], [%1], 16;\n\t}" ::"r"(
              smem_u32(d)),
          "l"(g), "r"(p)
          : "memory");
    };
    auto issue_row = [&](int jr, int slot) {
      long long cs;
      const double* rb = row_ptr(jr, cs);
      if (!rb) return;  // physical boundary: mirrored traces, nothing to load
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double* g = rb + c * cs;
        cp16(&rw[slot][c][(1 + lane) * 4], g + (long long)ie * 4, pe);
        cp16(&rw[slot][c][(1 + lane) * 4 + 2], g + (long long)ie * 4 + 2, pe);
        cp16(&rw[slot][c][0], g + (long long)iw * 4, pw);
        cp16(&rw[slot][c][2], g + (long long)iw * 4 + 2, pw);
      }
    };
    auto issue_q0 = [&](int jr, int slot) {
      const double* g0 = a.q0 + ((long long)jr * a.nx + (own ? i0 + lane : i0)) * 4;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        cp16(&qw[slot][c][lane * 4], g0 + c * a.cs, own ? 1 : 0);
        cp16(&qw[slot][c][lane * 4 + 2], g0 + c * a.cs + 2, own ? 1 : 0);
      }
    };
    auto commit = [] { asm volatile("cp.async.commit_group;" ::: "memory"); };
    auto has_row = [&](int jr) { return (jr >= 0 && jr < a.nrows) || (jr < 0 ? a.ghost_lo : a.ghost_hi) != nullptr; };
    // own element of ring slot s (4 points x 4 components, p = b*2 + a)
    auto ld_elem = [&](int s, int slotidx, double q[4][4]) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double2 u = *reinterpret_cast<const double2*>(&rw[s][c][slotidx * 4]);
        const double2 v = *reinterpret_cast<const double2*>(&rw[s][c][slotidx * 4 + 2]);
        q[c][0] = u.x; q[c][1] = u.y; q[c][2] = v.x; q[c][3] = v.y;
      }
    };
    // traces of an element (GLL: the edge points; GL: interpolated along the lines)
    // side: 0 W (rows b), 1 E, 2 S (columns a), 3 N; t = line index
    auto trace = [&](const double q[4][4], int side, int t, double o[4]) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (GLL) {
          o[c] = side == 0 ? q[c][t * 2] : side == 1 ? q[c][t * 2 + 1] : side == 2 ? q[c][t] : q[c][2 + t];
        } else {
          const double* e = (side == 0 || side == 2) ? O.eL : O.eR;
          o[c] = side <= 1 ? fma(e[1], q[c][t * 2 + 1], e[0] * q[c][t * 2])
                           : fma(e[1], q[c][2 + t], e[0] * q[c][t]);
        }
      }
    };

    // prologue: element rows jb-1 (ring slot 0) and jb (slot 1), q^n rows jb ..
    // jb+WD-1; the S face of row jb; then rows jb+1 .. jb+WD (one group each)
    issue_row(jb - 1, 0);
    issue_row(jb, 1);
    if (HQ0)
      for (int r = 0; r < PWD && r < RBv; ++r) issue_q0(jb + r, r);
    commit();
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    double FS[2][4];  // S-face fluxes of the current row (the N faces of the row below)
    {
      double qb[4][4], qo[4][4];
      ld_elem(0, 1 + lane, qb);
      ld_elem(1, 1 + lane, qo);
      const bool mS = !has_row(jb - 1);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        double ql[4], qr[4], fl[4], fr[4], sl, sr;
        trace(qo, 2, t, qr);
        trace(qb, 3, t, ql);
        if (mS) {
#pragma unroll
          for (int c = 0; c < 4; ++c) ql[c] = qr[c];
        }
        feval<1>(ql, gm1, gam, fl, sl);
        feval<1>(qr, gm1, gam, fr, sr);
        rus1(ql, fl, sl, qr, fr, sr, FS[t]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int k = 1; k <= PWD; ++k) {
      if (k <= RBv) issue_row(jb + k, (k + 1) % PWNS);
      commit();
    }

    const double bdt = a.bcoef * dtv;
    const double cx = -bdt * a.rdx2, cy = -bdt * a.rdy2;
    int S0 = 1 % PWNS, S1 = 2 % PWNS, SI = 0, Q0 = 0, QI = PWD % PQS;
    auto adv = [](int& x, int n) { x = (x + 1 == n) ? 0 : x + 1; };
#pragma unroll 1
    for (int r = 0; r < RBv; ++r) {
      asm volatile("cp.async.wait_group %0;" ::"n"(PWD - 1) : "memory");
      __syncwarp();
      if (r + 1 + PWD <= RBv) issue_row(jb + r + 1 + PWD, SI);
      if (HQ0 && r + PWD < RBv) issue_q0(jb + r + PWD, QI);
      commit();
      const int jr = jb + r;
      double q[4][4], qn[4][4];
      ld_elem(S0, 1 + lane, q);
      ld_elem(S1, 1 + lane, qn);
      // GLL (CPR, NDG): the element's own points are its traces -- primitives and
      // sound speed once per point, fluxes formed where needed
      Prim wp[4];
      double cp[4] = {0.0, 0.0, 0.0, 0.0};
      if constexpr (GLL) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const double v[4] = {q[0][p], q[1][p], q[2][p], q[3][p]};
          wp[p] = prims(v, gm1);
          cp[p] = fsqrt_ws(gam * wp[p].p * wp[p].ri);
        }
      }
      auto own_trace = [&](int side, int t, double o4[4], double f4[4], double& s) {  // GLL point flux
        const int p = side == 0 ? t * 2 : side == 1 ? t * 2 + 1 : side == 2 ? t : 2 + t;
        const double v[4] = {q[0][p], q[1][p], q[2][p], q[3][p]};
#pragma unroll
        for (int c = 0; c < 4; ++c) o4[c] = v[c];
        if (side <= 1) {
          flux<0>(v, wp[p], f4);
          s = fabs(wp[p].u) + cp[p];
        } else {
          flux<1>(v, wp[p], f4);
          s = fabs(wp[p].v) + cp[p];
        }
      };
      // ---- W face (per row b): W neighbour's E trace | own W trace ----
      double FW[2][4], FE[2][4], FN[2][4];
      double fWt[2][4], gNt[2][4];  // own W / N trace fluxes (CPR/NDG corrections)
      {
        double qwn[4][4];
        ld_elem(S0, lane, qwn);  // slot lane = the element on the left (lane 0: the W halo)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          double ql[4], qr[4], fl[4], fr[4], sl, sr;
          if constexpr (GLL) own_trace(0, t, qr, fr, sr);
          else {
            trace(q, 0, t, qr);
            feval<0>(qr, gm1, gam, fr, sr);
          }
          trace(qwn, 1, t, ql);
          if (mirW) {  // transmissive W end: the ghost trace is the own one
#pragma unroll
            for (int c = 0; c < 4; ++c) ql[c] = qr[c];
          }
          feval<0>(ql, gm1, gam, fl, sl);
#pragma unroll
          for (int c = 0; c < 4; ++c) fWt[t][c] = fr[c];
          if (mirE) {  // the halo lane at a transmissive E end: the ghost trace is the last element's
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              qr[c] = ql[c];
              fr[c] = fl[c];
            }
            sr = sl;
          }
          rus1(ql, fl, sl, qr, fr, sr, FW[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int c = 0; c < 4; ++c) FE[t][c] = __shfl_down_sync(0xffffffffu, FW[t][c], 1);
      // ---- N face (per column a): own N trace | the element above's S trace ----
      {
        const bool mN = !has_row(jr + 1);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          double ql[4], qr[4], fl[4], fr[4], sl, sr;
          if constexpr (GLL) own_trace(3, t, ql, fl, sl);
          else {
            trace(q, 3, t, ql);
            feval<1>(ql, gm1, gam, fl, sl);
          }
          trace(qn, 2, t, qr);
          feval<1>(qr, gm1, gam, fr, sr);
          if (mN) {  // transmissive top: the ghost trace is the own one
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              qr[c] = ql[c];
              fr[c] = fl[c];
            }
            sr = sl;
          }
          rus1(ql, fl, sl, qr, fr, sr, FN[t]);
#pragma unroll
          for (int c = 0; c < 4; ++c) gNt[t][c] = fl[c];
        }
      }
      // ---- element residual and the stage combination ----
      double o[4][4];  // [c][p]
      if constexpr (GLL) {
        // E / S trace fluxes of the own points (the corrections' f(own trace))
        double fEt[2][4], gSt[2][4];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          double dq[4], ds;
          own_trace(1, t, dq, fEt[t], ds);
          own_trace(2, t, dq, gSt[t], ds);
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int ax = p & 1, by = p >> 1;
          double v[4], Fx[4], Gy[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) v[c] = q[c][p];
          if constexpr (M == PM_CPR) {  // chain rule: A(q) dq/dxi + B(q) dq/deta
            double dx[4], dy[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              dx[c] = fma(O.Dl[ax][1], q[c][by * 2 + 1], O.Dl[ax][0] * q[c][by * 2]);
              dy[c] = fma(O.Dl[by][1], q[c][2 + ax], O.Dl[by][0] * q[c][ax]);
            }
            jac_pair(v, wp[p], gm1, dx, dy, Fx, Gy);
          } else {  // NDG: D[f], D[g] from the point fluxes (own traces)
            // f at (0,b) is fWt[b], at (1,b) fEt[b]; g at (a,0) gSt[a], at (a,1) gNt[a]
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              Fx[c] = fma(O.Dl[ax][1], fEt[by][c], O.Dl[ax][0] * fWt[by][c]);
              Gy[c] = fma(O.Dl[by][1], gNt[ax][c], O.Dl[by][0] * gSt[ax][c]);
            }
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double jW = FW[by][c] - fWt[by][c], jE = FE[by][c] - fEt[by][c];
            const double jS = FS[ax][c] - gSt[ax][c], jN = FN[ax][c] - gNt[ax][c];
            const double fx = Fx[c] + O.gL[ax] * jW + O.gR[ax] * jE;
            const double gy = Gy[c] + O.gL[by] * jS + O.gR[by] * jN;
            o[c][p] = fma(a.a1, v[c], fma(cx, fx, cy * gy));
          }
        }
      } else if constexpr (M == PM_DG) {
        // weak form (Eq. (19)): (2/dx) [sum_l (w_l/w_a) l'_a(xi_l) f_lb - (l_a(1) F^E - l_a(-1) F^W) / w_a] + y
        double f[4][4], g[4][4];  // [p][c]
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          double v[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) v[c] = q[c][p];
          const Prim w = prims(v, gm1);
          flux<0>(v, w, f[p]);
          flux<1>(v, w, g[p]);
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int ax = p & 1, by = p >> 1;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double vx = fma(O.dv[ax][1], f[by * 2 + 1][c], O.dv[ax][0] * f[by * 2][c]);
            const double vy = fma(O.dv[by][1], g[2 + ax][c], O.dv[by][0] * g[ax][c]);
            const double rx = vx - (O.sR[ax] * FE[by][c] - O.sL[ax] * FW[by][c]);
            const double ry = vy - (O.sR[by] * FN[ax][c] - O.sL[by] * FS[ax][c]);
            // R = rdx2 rx + rdy2 ry;  out = a1 q + bdt R  (cx = -bdt rdx2)
            o[c][p] = fma(a.a1, q[c][p], -fma(cx, rx, cy * ry));
          }
        }
      } else {  // SD: flux polynomial through {-1, 0, 1} per line, differentiated at the GL points
        double fm[2][4], gm[2][4];  // interior flux point (xi = 0) of row b / column a
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          double qr[4], qc[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            qr[c] = fma(O.sI1[1], q[c][t * 2 + 1], O.sI1[0] * q[c][t * 2]);
            qc[c] = fma(O.sI1[1], q[c][2 + t], O.sI1[0] * q[c][t]);
          }
          const Prim wr = prims(qr, gm1), wc = prims(qc, gm1);
          flux<0>(qr, wr, fm[t]);
          flux<1>(qc, wc, gm[t]);
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int ax = p & 1, by = p >> 1;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double fx = fma(O.sD[ax][2], FE[by][c], fma(O.sD[ax][1], fm[by][c], O.sD[ax][0] * FW[by][c]));
            const double gy = fma(O.sD[by][2], FN[ax][c], fma(O.sD[by][1], gm[ax][c], O.sD[by][0] * FS[ax][c]));
            o[c][p] = fma(a.a1, q[c][p], fma(cx, fx, cy * gy));
          }
        }
      }
      // ---- q^n, store, wave speed / non-physical check, element averages ----
      const long long m = (long long)jr * a.nx + i0 + lane;
      if (HQ0) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int p = 0; p < 4; ++p) o[c][p] = fma(a.a0, qw[Q0][c][lane * 4 + p], o[c][p]);
      }
      if (own) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(a.out + c * a.cs + m * 4), "d"(o[c][0]),
                       "d"(o[c][1]), "d"(o[c][2]), "d"(o[c][3])
                       : "memory");
      }
      if (HLAM) {
        unsigned long long bidx = ~0ull;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const double v[4] = {o[0][p], o[1][p], o[2][p], o[3][p]};
          const Prim w = prims(v, gm1);
          const double sp = fmax(fabs(w.u), fabs(w.v)) + fsqrt(gam * w.p * w.ri);
          lam = own ? nanmax(lam, sp) : lam;
          if (own && !admissible(v[0], w.p)) bidx = min(bidx, (unsigned long long)(m * 4 + p));
        }
        if (a.bad && bidx != ~0ull) atomicMin(a.bad, bidx);
      }
      if (HAVG && own && a.laml) {  // limiter runs: the element's wave speed / first bad point (LamFuse)
        unsigned long long bidx = ~0ull;
        double ll = 0.0;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const double v[4] = {o[0][p], o[1][p], o[2][p], o[3][p]};
          const Prim w = prims(v, gm1);
          ll = nanmax(ll, fmax(fabs(w.u), fabs(w.v)) + fsqrt(gam * w.p * w.ri));
          if (!admissible(v[0], w.p)) bidx = min(bidx, (unsigned long long)(m * 4 + p));
        }
        a.laml[m * 2] = ll;
        a.laml[m * 2 + 1] = 0.0;
        a.badl[m * 2] = bidx;
        a.badl[m * 2 + 1] = ~0ull;
      }
      if (HAVG && own) {  // Alg. 9: 1/4 sum_ab w_a w_b q_ab (GLL and GL P1 weights are 1)
        const long long ne = (long long)a.nx * a.nrows;
        const double* wq = GLL ? O.wl : O.wg;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double s = 0.0;
#pragma unroll
          for (int p = 0; p < 4; ++p) s += wq[p & 1] * wq[p >> 1] * o[c][p];
          a.qbar[c * ne + m] = 0.25 * s;
        }
      }
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int c = 0; c < 4; ++c) FS[t][c] = FN[t][c];
      adv(S0, PWNS); adv(S1, PWNS); adv(SI, PWNS); adv(Q0, PQS); adv(QI, PQS);
    }
  }
  if (HLAM && a.lam) block_max_to(lam, a.lam, sred);
}

namespace {
template <int M, int V>
cudaError_t p1_launch_v(dim3 grid, const StageArgs& a, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  const size_t sm = p1_smem((V & 1) != 0);
  const cudaError_t e = smem_optin(p1_warp_kernel<M, V>, (int)p1_smem(true), attr);
  if (e != cudaSuccess) return e;
  return launch_pdl_if(!a.no_pdl, p1_warp_kernel<M, V>, grid, dim3(PWPC * 32), sm, s, a);
}
template <int M>
cudaError_t p1_launch_m(int v, dim3 grid, const StageArgs& a, cudaStream_t s) {
  switch (v) {
    case 0: return p1_launch_v<M, 0>(grid, a, s);
    case 1: return p1_launch_v<M, 1>(grid, a, s);
    case 3: return p1_launch_v<M, 3>(grid, a, s);
    case 4: return p1_launch_v<M, 4>(grid, a, s);
    case 5: return p1_launch_v<M, 5>(grid, a, s);
    case 7: return p1_launch_v<M, 7>(grid, a, s);
    default: return cudaErrorNotSupported;
  }
}
bool al32(const void* p) { return ((uintptr_t)p & 31u) == 0; }
}  // namespace

#ifndef H2D_P1W
#define H2D_P1W 1  // the element-per-lane P1 kernel (0: the line kernels at P1 too)
#endif

// returns -1 when the P1 warp kernel does not apply (then the line kernels run)
int launch_p1_stage(int method, const StageArgs& a0, cudaStream_t s) {
  StageArgs a = a0;
  const int v = (a.q0 ? 1 : 0) | ((a.lam || a.bad) ? 2 : 0) | (a.qbar ? 4 : 0);
  // 32-B element stores and 16-B copies: every array and component stride aligned
  if (!H2D_P1W || !al32(a.q) || !al32(a.q0) || !al32(a.out) || !al32(a.ghost_lo) || !al32(a.ghost_hi) ||
      (a.cs % 4) || (a.gcs % 4) || (v != 0 && v != 1 && v != 3 && v != 4 && v != 5 && v != 7))
    return -1;
  const int nr = row_range(a);
  if (nr <= 0) return 0;
  const int strips = ((a.nx + PWS - 1) / PWS + PWPC - 1) / PWPC;
  a.rows = march_rows_waves(nr, strips, 64, H2D_P1W_MINB);
  const dim3 grid(strips, band_blocks(a));
  cudaError_t e;
  switch (method) {
    case PM_CPR: e = p1_launch_m<PM_CPR>(v, grid, a, s); break;
    case PM_NDG: e = p1_launch_m<PM_NDG>(v, grid, a, s); break;
    case PM_DG: e = p1_launch_m<PM_DG>(v, grid, a, s); break;
    case PM_SD: e = p1_launch_m<PM_SD>(v, grid, a, s); break;
    default: return -1;
  }
  return (int)e;
}

}  // namespace h2d
