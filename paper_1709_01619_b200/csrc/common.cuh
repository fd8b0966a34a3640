// common.cuh -- device-side physics of the 2-D Euler equations (Eqs. (1)-(5),
// P:120-146) and the Rusanov flux for the sm_100a kernels.
// Own implementation; shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace h2d {

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may become resident while its
// predecessor in the stream drains; it must not touch global memory before
// pdl_wait() (full completion and visibility of the predecessor).  pdl_launch()
// lets the successor start launching once every CTA of this grid has run it.
// Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// first row and row bound of this CTA's march: row blocks past the first band's
// (a.nb1) march the optional second band
__device__ __forceinline__ int band_start(const StageArgs& a, int& hi) {
  const int by = blockIdx.y;
  if (a.row_hi2 > a.row_lo2 && by >= a.nb1) {
    hi = a.row_hi2;
    return a.row_lo2 + (by - a.nb1) * a.rows;
  }
  hi = a.row_hi;
  return a.row_lo + by * a.rows;
}

// the stage's dt (Eq. (36) via the step's clock; see StageArgs::dtrole).  The
// same arithmetic as k_dt: lam of the last completed step (lam[0] if that step
// advanced, else lam[1]), dt = cfl*h / lam clipped to t_end - t.
__device__ __forceinline__ double stage_dt(const StageArgs& a) {
  if (!a.dt) return 1.0;
  const bool lead = blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
  if (a.dtrole == 1) {
    const double* c = a.clk;
    // five independent loads (one L2 round trip, not a dependent chain)
    const unsigned long long l0 = a.lamdt[0], l1 = a.lamdt[1];
    const double c0 = c[0], c3 = c[3], c4 = c[4];
    const unsigned long long lb = c3 != 0.0 ? l0 : l1;
    double dt = a.cflh / __longlong_as_double((long long)lb);
    const double rem = c4 - c0;
    if (!(rem > 0.0)) dt = 0.0;
    else if (dt > rem) dt = rem;
    if (lead) a.clk[1] = dt;
    return dt;
  }
  const double dt = *a.dt;
  if (a.dtrole == 2 && lead) {
    double* c = a.clk;
    if (c[3] != 0.0) a.lamdt[1] = a.lamdt[0];
    a.lamdt[0] = 0ull;
    if (dt != 0.0) {
      c[0] = c[0] + dt;
      c[2] += 1.0;
      c[3] = 1.0;
    } else {
      c[3] = 0.0;
    }
  }
  return dt;
}

struct Prim {
  double ri, u, v, p;  // 1/rho, velocities, pressure
};

// fp64 reciprocal: MUFU seed + two Newton steps (faithful to ~1 ulp, no slow
// path; non-finite / zero inputs propagate as inf / NaN and are flagged later)
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// fp64 square root: MUFU rsqrt seed (relative error e0 <= ~2^-21: the seed sees
// the high word only), one Newton step (e1 ~ 1.5 e0^2 ~ 2^-41), then s = x y and
// one Markstein correction s + y (x - s^2) / 2 (error ~ 1.5 e1^2 + final rounding),
// i.e. as accurate as two Newton steps + correction, 4 fp64 operations fewer
__device__ __forceinline__ double fsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, e, y);
  const double s = x * y;
  return fma(0.5 * y, fma(-s, s, x), s);
}

// square root for the Rusanov dissipation speed only (|u_n| + c in lam (q_R - q_L),
// P:869-870): the MUFU seed and one Newton step, s = x y (relative error
// ~1.5 e0^2 <= ~2^-41).  lam multiplies a state jump, so its error enters the
// flux at <= 2^-41 |q_R - q_L| / |f| -- far below the rounding of the flux
// itself on smooth data and below the parity bar on any data -- and 3 fp64
// operations per call are saved.  Not used where c decides dt (Eq. (36)).
__device__ __forceinline__ double fsqrt_ws(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0);
  y = fma(0.5 * y, e, y);
  return x * y;
}

// one reciprocal per point (the only fp64 division of a flux evaluation)
__device__ __forceinline__ Prim prims(const double q[4], double gm1) {
  Prim w;
  w.ri = frcp(q[0]);
  w.u = q[1] * w.ri;
  w.v = q[2] * w.ri;
  w.p = gm1 * (q[3] - 0.5 * (q[1] * w.u + q[2] * w.v));
  return w;
}

// Eq. (4): f (DIR 0) or g (DIR 1)
template <int DIR>
__device__ __forceinline__ void flux(const double q[4], const Prim& w, double f[4]) {
  if (DIR == 0) {
    f[0] = q[1];
    f[1] = q[1] * w.u + w.p;
    f[2] = q[1] * w.v;
    f[3] = w.u * (q[3] + w.p);
  } else {
    f[0] = q[2];
    f[1] = q[2] * w.u;
    f[2] = q[2] * w.v + w.p;
    f[3] = w.v * (q[3] + w.p);
  }
}

// Rusanov flux along axis DIR for (west|south, east|north) states; also returns
// the two physical fluxes (the CPR/NDG correction needs F^ - f(own trace)).
template <int DIR>
__device__ __forceinline__ void rusanov(const double qL[4], const double qR[4], double gm1, double gam,
                                        double F[4], double fL[4], double fR[4]) {
  Prim wl = prims(qL, gm1), wr = prims(qR, gm1);
  flux<DIR>(qL, wl, fL);
  flux<DIR>(qR, wr, fR);
  double sl = fabs(DIR == 0 ? wl.u : wl.v) + fsqrt(gam * wl.p * wl.ri);
  double sr = fabs(DIR == 0 ? wr.u : wr.v) + fsqrt(gam * wr.p * wr.ri);
  double lam = fmax(sl, sr);
#pragma unroll
  for (int c = 0; c < 4; ++c) F[c] = 0.5 * (fL[c] + fR[c]) - 0.5 * lam * (qR[c] - qL[c]);
}

// Flux-Jacobian action A(q).d (DIR 0) or B(q).d (DIR 1): the chain rule of the
// CPR divergence.
template <int DIR>
__device__ __forceinline__ void jac(const double q[4], const Prim& w, double gm1, double gam, const double d[4],
                                    double o[4]) {
  const double u = w.u, v = w.v;
  const double phi = 0.5 * gm1 * (u * u + v * v);
  const double H = (q[3] + w.p) * w.ri;
  if (DIR == 0) {
    o[0] = d[1];
    o[1] = (phi - u * u) * d[0] + (3.0 - gam) * u * d[1] - gm1 * v * d[2] + gm1 * d[3];
    o[2] = -u * v * d[0] + v * d[1] + u * d[2];
    o[3] = u * (phi - H) * d[0] + (H - gm1 * u * u) * d[1] - gm1 * u * v * d[2] + gam * u * d[3];
  } else {
    o[0] = d[2];
    o[1] = -u * v * d[0] + v * d[1] + u * d[2];
    o[2] = (phi - v * v) * d[0] - gm1 * u * d[1] + (3.0 - gam) * v * d[2] + gm1 * d[3];
    o[3] = v * (phi - H) * d[0] - gm1 * u * v * d[1] + (H - gm1 * v * v) * d[2] + gam * v * d[3];
  }
}

// The same Jacobian actions through the primitive-variable differentials
// (A(q).d = d f along d): du = (d1 - u d0)/rho, dv = (d2 - v d0)/rho,
// dp = (gamma-1)(d3 - u d1 - v d2 + (u^2+v^2)/2 d0), then
// d f = (d1, d1 u + rho u du + dp, d1 v + rho u dv, du (e+p) + u (d3 + dp)) and
// d g = (d2, d2 u + rho v du, d2 v + rho v dv + dp, dv (e+p) + v (d3 + dp)).
// Algebraically identical to jac<0> + jac<1> (tests compare them to the
// oracle's matrix form); ~30 % fewer fp64 operations for the pair.
__device__ __forceinline__ void jac_pair(const double q[4], const Prim& w, double gm1, const double dx[4],
                                         const double dy[4], double fx[4], double gy[4]) {
  const double u = w.u, v = w.v, k = 0.5 * (u * u + v * v), ep = q[3] + w.p;
  {
    const double du = w.ri * fma(-u, dx[0], dx[1]), dv = w.ri * fma(-v, dx[0], dx[2]);
    const double dp = gm1 * fma(k, dx[0], fma(-v, dx[2], fma(-u, dx[1], dx[3])));
    fx[0] = dx[1];
    fx[1] = fma(dx[1], u, fma(q[1], du, dp));
    fx[2] = fma(dx[1], v, q[1] * dv);
    fx[3] = fma(du, ep, u * (dx[3] + dp));
  }
  {
    const double du = w.ri * fma(-u, dy[0], dy[1]), dv = w.ri * fma(-v, dy[0], dy[2]);
    const double dp = gm1 * fma(k, dy[0], fma(-v, dy[2], fma(-u, dy[1], dy[3])));
    gy[0] = dy[2];
    gy[1] = fma(dy[2], u, q[2] * du);
    gy[2] = fma(dy[2], v, fma(q[2], dv, dp));
    gy[3] = fma(dv, ep, v * (dy[3] + dp));
  }
}

// max(|u|,|v|) + c  (2-D reading of Eq. (36))
__device__ __forceinline__ double wave_speed(const double q[4], double gm1, double gam) {
  Prim w = prims(q, gm1);
  return fmax(fabs(w.u), fabs(w.v)) + fsqrt(gam * w.p * w.ri);
}

// Non-physical state (rho <= 0, p <= 0 or any component non-finite),
// decided from rho and p = (gamma-1)(e - (rho u u + rho v v)/2) alone: given
// 0 < rho < inf, a non-finite rho u or rho v makes the kinetic term +inf or NaN
// (p = -inf or NaN), a non-finite e makes p = +-inf or NaN, and finite inputs
// give p <= (gamma-1) e < inf (the kinetic term is >= 0). So
// "0 < rho < inf and 0 < p < inf" is exactly "all finite, rho > 0, p > 0".
__device__ __forceinline__ bool admissible(double rho, double p) {
  return rho > 0.0 && rho < HUGE_VAL && p > 0.0 && p < HUGE_VAL;
}

__device__ __forceinline__ bool nonphysical(const double q[4], double gm1) {
  Prim w = prims(q, gm1);
  return !admissible(q[0], w.p);
}

// NaN-propagating max (fmax would drop a NaN): a non-finite wave speed must
// reach the dt of Eq. (36) rather than vanish in the reduction
__device__ __forceinline__ double nanmax(double v, double o) { return (o > v || o != o) ? o : v; }

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// block-wide max of a non-negative value -> one atomicMax on the bit pattern
// (IEEE order of non-negative doubles == unsigned order of their bits; NaN wins)
__device__ __forceinline__ void block_max_to(double v, unsigned long long* dst, double* s_red) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    double x = lane < nw ? s_red[lane] : 0.0;
    x = warp_max(x);
    if (lane == 0) atomicMax(dst, (unsigned long long)__double_as_longlong(x));
  }
}

__device__ __forceinline__ void count_dec(long long* dec, int which, int w = 1) {
  if (dec && w) atomicAdd((unsigned long long*)&dec[which], (unsigned long long)w);
}

// minmod of two arguments (ties return the first argument, zero if the
// signs differ or either is zero), optionally recording the branch taken.  A
// decision within DEC_TIE of its switch point (a = 0, b = 0 or a = b) is counted
// as a tie (slot 4), not by outcome: its branch may legitimately differ between
// two fp64 evaluation orders.
#define DEC_TIE 1e-12
// |a| <= |b| (minmod's magnitude test); H2D_ICMP: on the integer pipe (sign-masked
// bit patterns compare like magnitudes for non-NaN values) instead of a DSETP
#ifndef H2D_ICMP
#define H2D_ICMP 0
#endif
__device__ __forceinline__ bool mag_le(double a, double b) {
#if H2D_ICMP
  const unsigned long long m = 0x7fffffffffffffffull;
  return ((unsigned long long)__double_as_longlong(a) & m) <= ((unsigned long long)__double_as_longlong(b) & m);
#else
  return fabs(a) <= fabs(b);
#endif
}
// (w: how many of the paper's face evaluations this one call stands for; mp:
// optional per-cell decision-map entry, the outcome added as w << 16*(slot),
// slot 0 -> 0, 1 -> first argument, 2 -> second, 3 tie -- hom2d_decision_map)
__device__ __forceinline__ double minmod2(double a, double b, long long* dec, int w = 1, long long* mp = nullptr) {
  // value without branches: the argument of smaller magnitude when both have the
  // same strict sign (equal magnitudes: equal values), else 0.  Equal sign BITS
  // suffice: a zero argument has the smaller magnitude, so m is then +-0 anyway.
  const double m = mag_le(a, b) ? a : b;
  const double r = (__double2hiint(a) ^ __double2hiint(b)) >= 0 ? m : 0.0;
  if (dec) {
    int which = 1;
    if ((a > 0.0 && b > 0.0) || (a < 0.0 && b < 0.0)) which = (fabs(a) <= fabs(b)) ? 2 : 3;
    if (fabs(a) <= DEC_TIE || fabs(b) <= DEC_TIE || fabs(a - b) <= DEC_TIE) which = 4;
    count_dec(dec, which, w);
    if (mp && w) atomicAdd((unsigned long long*)mp, (unsigned long long)w << (16 * (which - 1)));
  }
  return r;
}

// FV MUSCL reconstruction, shared by the FV stage kernel
// and the reconstructed-solution error.
// the two reconstructed face values of cell i (stencil i-1, i, i+1): lo at its
// i-1/2 face, hi at its i+1/2 face (the face states of P:346-351; SURVEY C8 with
// the same arithmetic as the per-face form, so values are bitwise those of
// reconstructing at each face).  w = how many face evaluations of the paper's
// form this one reconstruction stands for (decision counting only).
template <int ORDER>
__device__ __forceinline__ void cell_faces(double qm, double q0, double qp, double& lo, double& hi, long long* dec,
                                           int w, long long* mp = nullptr) {
  // explicit rounding (no contraction freedom): a face state is bitwise the same
  // wherever it is evaluated (prologue or carried), so results do not depend on
  // how the rows are split over CTAs / launches / ranks
  if (ORDER == 3) {  // unlimited kappa = 0 (f3 variant of MUSCL-2)
    const double d = (q0 - qm) + (qp - q0);
    hi = __fma_rn(0.25, d, q0);
    lo = __fma_rn(-0.25, d, q0);
  } else if (ORDER == 4) {  // unlimited kappa = 1/3 (f3 variant of MUSCL-3)
    constexpr double kap = 1.0 / 3.0;
    const double dm = q0 - qm, dp = qp - q0;
    constexpr double c1 = 0.25 * (1.0 - kap), c2 = 0.25 * (1.0 + kap);
    hi = __fma_rn(c1, dm, __fma_rn(c2, dp, q0));
    lo = __fma_rn(-c1, dp, __fma_rn(-c2, dm, q0));
  } else if (ORDER == 1) {
    const double s = minmod2(q0 - qm, qp - q0, dec, w, mp);
    hi = __fma_rn(0.5, s, q0);
    lo = __fma_rn(-0.5, s, q0);
  } else {  // kappa = 1/3, beta = (3 - kappa)/(1 - kappa) = 4
    constexpr double kap = 1.0 / 3.0, beta = (3.0 - kap) / (1.0 - kap);
    const double dm = q0 - qm, dp = qp - q0;
    double A, B;
    if (dec) {
      A = minmod2(dm, beta * dp, dec, w, mp);
      B = minmod2(dp, beta * dm, dec, w, mp);
    } else {  // both minmods share the sign test (beta > 0): one sign-bit comparison
      const double bdp = beta * dp, bdm = beta * dm;
      const bool same = (__double2hiint(dm) ^ __double2hiint(dp)) >= 0;
      const double ma = mag_le(dm, bdp) ? dm : bdp, mb = mag_le(dp, bdm) ? dp : bdm;
      A = same ? ma : 0.0;
      B = same ? mb : 0.0;
    }
    // q0 +- ((1 - kappa) X + (1 + kappa) Y) / 4 with the quarter folded into the weights
    constexpr double c1 = 0.25 * (1.0 - kap), c2 = 0.25 * (1.0 + kap);
    hi = __fma_rn(c1, A, __fma_rn(c2, B, q0));
    lo = __fma_rn(-c1, B, __fma_rn(-c2, A, q0));
  }
}

}  // namespace h2d
