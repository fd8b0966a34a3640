// aux.cu -- the non-stage kernels of the hot path: wave-speed max and dt
// bookkeeping (Eq. (36)), closed-form initial data (vortex P:897-913,
// radial shock tube P:1043-1047), error reductions, and the
// high-order limiter (Average Alg. 9; Limit Algs. 10-11 P:802-864;
// Eq. (35)).
#include <cstdlib>

#include "common.cuh"
#include "ops_tables.h"

// k_limit: 8 CTAs/SM (<= 64 registers) for P1/P2 -- the per-element limit branch
// is rare, its spills are cheap, detection wants the occupancy (+11 % on the
// shock-tube steps); P3/P4 at 4 (their limit branch spills heavily at 8)
#ifndef H2D_LIMIT_MINB
#define H2D_LIMIT_MINB (N <= 3 ? 8 : 4)
#endif

namespace h2d {

namespace {
struct Nodes {
  int n;
  double xi[5], w[5], eL[5], eR[5];
};

template <int K>
Nodes nodes_k(bool gll) {
  using O = Ops<K>;
  Nodes r{};
  r.n = K + 1;
  for (int a = 0; a <= K; ++a) {
    r.xi[a] = gll ? O::xi_gll[a] : O::xi_gl[a];
    r.w[a] = gll ? O::w_gll[a] : O::w_gl[a];
    r.eL[a] = gll ? (a == 0 ? 1.0 : 0.0) : O::eL_gl[a];
    r.eR[a] = gll ? (a == K ? 1.0 : 0.0) : O::eR_gl[a];
  }
  return r;
}

Nodes nodes_for(int method, int k) {
  const bool gll = (method == 1 || method == 3);
  switch (k) {
    case 1: return nodes_k<1>(gll);
    case 2: return nodes_k<2>(gll);
    case 3: return nodes_k<3>(gll);
    default: return nodes_k<4>(gll);
  }
}

struct GL8v {
  double x[8], w[8];
};
GL8v gl8() {
  GL8v g;
  for (int i = 0; i < 8; ++i) { g.x[i] = GL8::x[i]; g.w[i] = GL8::w[i]; }
  return g;
}

}  // namespace

static int g_pdl_on = 1;
// (re)read HOM2D_NO_PDL; called at every hom2d_create
void pdl_refresh() {
  const char* v = getenv("HOM2D_NO_PDL");
  g_pdl_on = (v && v[0] == '1') ? 0 : 1;
}
bool pdl_enabled() { return g_pdl_on == 1; }

namespace {
int grid_for(long long n, int bs) {
  long long b = (n + bs - 1) / bs;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

__device__ __forceinline__ double wrapc(double s, double lo, double hi) {
  const double L = hi - lo;
  return s - L * floor((s - lo) / L);
}

// conserved state of the isentropic vortex (eps = 5, mean (1,1,0,1)) at (x,y,t):
// the initial field advected by (t, 0), single periodic image
__device__ void vortex(const AuxArgs& A, double x, double y, double t, double q[4]) {
  const double eps = 5.0, PI = 3.141592653589793;
  const double g = A.gamma;
  const double xs = wrapc(x - t, A.xmin, A.xmax), ys = wrapc(y, A.ymin, A.ymax);
  const double r2 = xs * xs + ys * ys;
  const double e1 = exp(0.5 * (1.0 - r2));
  const double du = -(eps / (2.0 * PI)) * e1 * ys, dv = (eps / (2.0 * PI)) * e1 * xs;
  const double T = 1.0 - (g - 1.0) * eps * eps / (8.0 * g * PI * PI) * e1 * e1;
  const double rho = pow(T, 1.0 / (g - 1.0));
  const double p = rho * T, u = 1.0 + du, v = dv;
  q[0] = rho;
  q[1] = rho * u;
  q[2] = rho * v;
  q[3] = p / (g - 1.0) + 0.5 * rho * (u * u + v * v);
}

__device__ void shock(const AuxArgs& A, double x, double y, double q[4]) {
  const bool in = x * x + y * y < 0.16;
  q[0] = in ? 1.0 : 0.125;
  q[1] = 0.0;
  q[2] = 0.0;
  q[3] = (in ? 1.0 : 0.1) / (A.gamma - 1.0);
}

__device__ void case_state(const AuxArgs& A, int cid, double x, double y, double t, double q[4]) {
  if (cid == 0) vortex(A, x, y, t, q); else shock(A, x, y, q);
}

__global__ void k_lambda(const AuxArgs A, const double* __restrict__ q, long long npts, unsigned long long* lam,
                         unsigned long long* bad) {
  __shared__ double sred[32];
  pdl_wait();
  pdl_launch();
  const double gm1 = A.gamma - 1.0;
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npts; i += (long long)gridDim.x * blockDim.x) {
    double v[4] = {q[i], q[A.cs + i], q[2 * A.cs + i], q[3 * A.cs + i]};
    const double s = wave_speed(v, gm1, A.gamma);
    m = (s <= m) ? m : s;  // NaN propagates
    if (bad && nonphysical(v, gm1)) atomicMin(bad, (unsigned long long)i);
  }
  block_max_to(m, lam, sred);
}

// clock: [0] t, [1] dt, [2] steps, [3] stepped flag;  lam: [0] accumulator, [1] current
// clk = {t, dt, steps, stepped, t_end}: t_end comes from device memory so that a
// captured CUDA graph of steps does not depend on it
__global__ void k_dt(double* clk, unsigned long long* lam, double cfl, double hmin) {
  pdl_wait();
  pdl_launch();
  if (clk[3] != 0.0) lam[1] = lam[0];
  lam[0] = 0ull;
  const double l = __longlong_as_double((long long)lam[1]);
  double dt = cfl * hmin / l;
  const double rem = clk[4] - clk[0];
  if (!(rem > 0.0)) dt = 0.0;
  else if (dt > rem) dt = rem;
  clk[1] = dt;
  if (dt != 0.0) {
    clk[0] = clk[0] + dt;
    clk[2] += 1.0;
    clk[3] = 1.0;
  } else {
    clk[3] = 0.0;
  }
}

__global__ void k_init(const AuxArgs A, Nodes nd, GL8v g8, int cid, double* q) {
  const int n = nd.n, np = (A.method == 0) ? 1 : n * n;
  const long long npts = (long long)A.nx * A.nrows * np;
  const double dx = (A.xmax - A.xmin) / A.nx, dy = (A.ymax - A.ymin) / A.ny_global;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < npts; t += (long long)gridDim.x * blockDim.x) {
    const long long m = t / np;
    const int p = (int)(t % np);
    const int i = (int)(m % A.nx), j = (int)(m / A.nx) + A.row0;
    const double xc = A.xmin + (i + 0.5) * dx, yc = A.ymin + (j + 0.5) * dy;
    double qq[4];
    if (A.method == 0) {
      double acc[4] = {0, 0, 0, 0};
      for (int b = 0; b < 8; ++b)
        for (int a = 0; a < 8; ++a) {
          double v[4];
          case_state(A, cid, xc + 0.5 * dx * g8.x[a], yc + 0.5 * dy * g8.x[b], 0.0, v);
          const double w = 0.25 * g8.w[a] * g8.w[b];
          for (int c = 0; c < 4; ++c) acc[c] += w * v[c];
        }
      for (int c = 0; c < 4; ++c) qq[c] = acc[c];
    } else {
      case_state(A, cid, xc + 0.5 * dx * nd.xi[p % n], yc + 0.5 * dy * nd.xi[p / n], 0.0, qq);
    }
    for (int c = 0; c < 4; ++c) q[c * A.cs + t] = qq[c];
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic per-block partials: {sum w|d|, sum w d^2, max |d|}
__global__ void k_err(const AuxArgs A, Nodes nd, GL8v g8, const double* __restrict__ q, int var,
                      const double* clk, double* part) {
  __shared__ double s1[32], s2[32], s3[32];
  const int n = nd.n, np = (A.method == 0) ? 1 : n * n;
  const long long npts = (long long)A.nx * A.nrows * np;
  const double dx = (A.xmax - A.xmin) / A.nx, dy = (A.ymax - A.ymin) / A.ny_global;
  const double t = clk[0];
  double a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (long long tt = blockIdx.x * (long long)blockDim.x + threadIdx.x; tt < npts; tt += (long long)gridDim.x * blockDim.x) {
    const long long m = tt / np;
    const int p = (int)(tt % np);
    const int i = (int)(m % A.nx), j = (int)(m / A.nx) + A.row0;
    const double xc = A.xmin + (i + 0.5) * dx, yc = A.ymin + (j + 0.5) * dy;
    double ex, w;
    if (A.method == 0) {
      double acc = 0.0;
      for (int b = 0; b < 8; ++b)
        for (int a = 0; a < 8; ++a) {
          double v[4];
          vortex(A, xc + 0.5 * dx * g8.x[a], yc + 0.5 * dy * g8.x[b], t, v);
          acc += 0.25 * g8.w[a] * g8.w[b] * v[var];
        }
      ex = acc;
      w = 1.0;
    } else {
      double v[4];
      vortex(A, xc + 0.5 * dx * nd.xi[p % n], yc + 0.5 * dy * nd.xi[p / n], t, v);
      ex = v[var];
      w = 0.25 * nd.w[p % n] * nd.w[p / n];
    }
    const double d = q[var * A.cs + tt] - ex;
    a1 += w * fabs(d);
    a2 += w * d * d;
    a3 = fmax(a3, fabs(d));
  }
  a1 = warp_sum(a1);
  a2 = warp_sum(a2);
  a3 = warp_max(a3);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { s1[wid] = a1; s2[wid] = a2; s3[wid] = a3; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b1 = 0, b2 = 0, b3 = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { b1 += s1[w]; b2 += s2[w]; b3 = fmax(b3, s3[w]); }
    part[3 * blockIdx.x] = b1;
    part[3 * blockIdx.x + 1] = b2;
    part[3 * blockIdx.x + 2] = b3;
  }
}

// FV reconstructed-solution error (reading R22): per cell, the MUSCL
// face states of the scheme (cell_faces, the stage kernel's reconstruction) and
// the cell value fix one quadratic per direction,
//   q_d(s) = qbar + (hi - lo)/2 s + (hi + lo - 2 qbar)/4 (3 s^2 - 1),
// the cell's solution is q_x(xi) + q_y(eta) - qbar, compared pointwise with the
// exact vortex at the 3x3 Gauss-Legendre points (weights w_a w_b / 4), like the
// HO convention R8.  One thread per cell; y-neighbours beyond the strip from the
// ghost rows (2 rows, component stride gcs), or clamped (transmissive).
template <int REC>
__global__ void k_err_fvr(const AuxArgs A, Nodes g3, const double* __restrict__ q, const double* glo,
                          const double* ghi, long long gcs, int bcx, int var, const double* clk, double* part) {
  __shared__ double s1[32], s2[32], s3[32];
  const long long ne = (long long)A.nx * A.nrows;
  const double dx = (A.xmax - A.xmin) / A.nx, dy = (A.ymax - A.ymin) / A.ny_global;
  const double t = clk[0];
  const double* qv = q + var * A.cs;
  double a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < ne; m += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(m % A.nx), jl = (int)(m / A.nx), j = jl + A.row0;
    int iw = i - 1, ie = i + 1;
    if (bcx == 0) { iw = iw < 0 ? iw + A.nx : iw; ie = ie >= A.nx ? ie - A.nx : ie; }
    else { iw = iw < 0 ? 0 : iw; ie = ie >= A.nx ? A.nx - 1 : ie; }
    const double qb = qv[m];
    const double qw = qv[(long long)jl * A.nx + iw], qe = qv[(long long)jl * A.nx + ie];
    const double qs = jl > 0 ? qv[m - A.nx] : (glo ? glo[var * gcs + (long long)A.nx + i] : qb);
    const double qn = jl + 1 < A.nrows ? qv[m + A.nx] : (ghi ? ghi[var * gcs + i] : qb);
    double lx, hx, ly, hy;
    cell_faces<REC>(qw, qb, qe, lx, hx, nullptr, 0);
    cell_faces<REC>(qs, qb, qn, ly, hy, nullptr, 0);
    const double xc = A.xmin + (i + 0.5) * dx, yc = A.ymin + (j + 0.5) * dy;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double sy = g3.xi[b];
      const double qy = qb + 0.5 * (hy - ly) * sy + 0.25 * (hy + ly - 2.0 * qb) * (3.0 * sy * sy - 1.0);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double sx = g3.xi[a];
        const double qx = qb + 0.5 * (hx - lx) * sx + 0.25 * (hx + lx - 2.0 * qb) * (3.0 * sx * sx - 1.0);
        double v[4];
        vortex(A, xc + 0.5 * dx * sx, yc + 0.5 * dy * sy, t, v);
        const double d = (qx + qy - qb) - v[var];
        const double w = 0.25 * g3.w[a] * g3.w[b];
        a1 += w * fabs(d);
        a2 += w * d * d;
        a3 = nanmax(a3, fabs(d));
      }
    }
  }
  a1 = warp_sum(a1);
  a2 = warp_sum(a2);
  a3 = warp_max(a3);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { s1[wid] = a1; s2[wid] = a2; s3[wid] = a3; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b1 = 0, b2 = 0, b3 = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { b1 += s1[w]; b2 += s2[w]; b3 = nanmax(b3, s3[w]); }
    part[3 * blockIdx.x] = b1;
    part[3 * blockIdx.x + 1] = b2;
    part[3 * blockIdx.x + 2] = b3;
  }
}

__global__ void k_err_final(const double* part, int nb, double* out3) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double b1 = 0, b2 = 0, b3 = 0;
  for (int i = 0; i < nb; ++i) { b1 += part[3 * i]; b2 += part[3 * i + 1]; b3 = fmax(b3, part[3 * i + 2]); }
  out3[0] = b1;
  out3[1] = b2;
  out3[2] = b3;
}

__global__ void k_avg(const AuxArgs A, Nodes nd, const double* __restrict__ q, double* qbar) {
  pdl_wait();
  pdl_launch();
  if (A.dt && *A.dt == 0.0) return;
  const int n = nd.n, np = n * n;
  const long long ne = (long long)A.nx * A.nrows;
  for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < ne; m += (long long)gridDim.x * blockDim.x) {
    for (int c = 0; c < 4; ++c) {
      double s = 0.0;
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) s += nd.w[a] * nd.w[b] * q[c * A.cs + m * np + b * n + a];
      qbar[c * ne + m] = 0.25 * s;
    }
  }
}

// one thread per element (2-D grid: x = element column, y = element row, no
// index division): detect on density at every edge point (Alg. 10: all 4N edge
// values evaluated, straight-line), limit all four components if marked (Alg. 11,
// Eq. (35) in 2-D)
// Characteristic limiting (Cockburn-Shu): eigenvectors of the Euler flux
// Jacobian along axis DIR at the element average qb -- right columns
// (1, u -/+ c n, H -/+ c u_n) acoustic, (1, u, |u|^2/2) entropy, (0, t, u_t) shear;
// left rows in closed form (b1 = (gamma-1)/c^2, b2 = b1 |u|^2/2) -- the slope of
// each field is minmod(L dp, L dm) and s = R (field slopes).
template <int DIR>
__device__ __forceinline__ void char_slopes(const double qb[4], const double dp[4], const double dm[4], double gam,
                                            double s[4]) {
  const double ri = 1.0 / qb[0], u = qb[1] * ri, v = qb[2] * ri;
  const double q2 = 0.5 * (u * u + v * v), p = (gam - 1.0) * (qb[3] - qb[0] * q2);
  const double H = (qb[3] + p) * ri, c = sqrt(gam * p * ri), rc = 1.0 / c;
  const double nx = DIR == 0 ? 1.0 : 0.0, ny = 1.0 - nx;
  const double un = DIR == 0 ? u : v, ut = DIR == 0 ? v : -u;
  const double b1 = (gam - 1.0) * rc * rc, b2 = b1 * q2;
  const double Lm[4][4] = {{0.5 * (b2 + un * rc), -0.5 * (b1 * u + nx * rc), -0.5 * (b1 * v + ny * rc), 0.5 * b1},
                           {1.0 - b2, b1 * u, b1 * v, -b1},
                           {-ut, -ny, nx, 0.0},
                           {0.5 * (b2 - un * rc), -0.5 * (b1 * u - nx * rc), -0.5 * (b1 * v - ny * rc), 0.5 * b1}};
  double w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int c2 = 0; c2 < 4; ++c2) {
      a += Lm[k][c2] * dp[c2];
      b += Lm[k][c2] * dm[c2];
    }
    w[k] = minmod2(a, b, nullptr);
  }
  s[0] = w[0] + w[1] + w[3];
  s[1] = (u - c * nx) * w[0] + u * w[1] - ny * w[2] + (u + c * nx) * w[3];
  s[2] = (v - c * ny) * w[0] + v * w[1] + nx * w[2] + (v + c * ny) * w[3];
  s[3] = (H - c * un) * w[0] + q2 * w[1] + ut * w[2] + (H + c * un) * w[3];
}

// neighbour averages of component c of element (i, j) (own average at a transmissive boundary)
struct Nbr {
  const AuxArgs& A;
  const double* __restrict__ qbar;
  const double *qbar_lo, *qbar_hi;
  long long gcs, ne, m;
  int i, j, iw, ie;
  bool hw, he;
  __device__ Nbr(const AuxArgs& A_, const double* __restrict__ qb, const double* lo, const double* hi, long long g,
                 int bcx, int i_, int j_)
      : A(A_), qbar(qb), qbar_lo(lo), qbar_hi(hi), gcs(g), ne((long long)A_.nx * A_.nrows),
        m((long long)j_ * A_.nx + i_), i(i_), j(j_), iw(i_ - 1), ie(i_ + 1), hw(true), he(true) {
    if (iw < 0) { if (bcx) hw = false; else iw += A.nx; }
    if (ie >= A.nx) { if (bcx) he = false; else ie -= A.nx; }
  }
  __device__ void operator()(int c, double own, double& W, double& E, double& S, double& Nn) const {
    W = hw ? qbar[c * ne + (long long)j * A.nx + iw] : own;
    E = he ? qbar[c * ne + (long long)j * A.nx + ie] : own;
    if (j > 0) S = qbar[c * ne + m - A.nx];
    else S = qbar_lo ? qbar_lo[c * gcs + i] : own;
    if (j < A.nrows - 1) Nn = qbar[c * ne + m + A.nx];
    else Nn = qbar_hi ? qbar_hi[c * gcs + i] : own;
  }
};

// minmod3(a, b, c) with (b, c) fixed: minmod3 = min(a, b, c) if all
// three are > 0, max(a, b, c) if all are < 0, else 0 (the oracle's form); here
// the pair (b, c) is reduced once per element and direction.  Same value as the
// three-way form whenever every argument is nonzero (the smallest magnitude of
// the three when all signs agree, else 0); with a zero argument both give a
// signed zero (and qbar -+ 0 is qbar), so the detector's decisions are identical.  Sign tests on the high
// words (integer pipe), one fp64 magnitude compare per edge point.
struct MM3 {
  double B;  // the smaller-magnitude of b, c (its sign is the pair's common sign)
  bool same;
  __device__ __forceinline__ MM3(double b, double c) {
    const int hb = __double2hiint(b), hc = __double2hiint(c);
    same = (hb ^ hc) >= 0;
    B = fabs(b) <= fabs(c) ? b : c;
  }
  __device__ __forceinline__ double operator()(double a) const {
    const bool ok = same && (__double2hiint(a) ^ __double2hiint(B)) >= 0;
    const double m = fabs(a) <= fabs(B) ? a : B;
    // 0 by masking the bits (the compiler would branch on a select here)
    return __longlong_as_double(__double_as_longlong(m) & -(long long)ok);
  }
};

// Alg. 10: does element (i, j) trip the detector?  (loads only: the detections of
// several elements of one thread overlap their memory latency)
template <int N, bool GLLP, bool ALL>
__device__ __forceinline__ bool detect_element(const AuxArgs& A, const Nodes& nd, const double* __restrict__ q,
                                               const Nbr& nbr, double eps) {
  constexpr int NP = N * N;
  const long long ne = nbr.ne, m = nbr.m;
  const double* __restrict__ qbar = nbr.qbar;
  const double qb = qbar[m];
  double rW, rE, rS, rN;
  nbr(0, qb, rW, rE, rS, rN);
  bool trip = false;
#pragma unroll
  for (int c = 0; c < (ALL ? 4 : 1); ++c) {  // density (Q12); ALL: every conserved component (f3)
    double cb = qb, cW = rW, cE = rE, cS = rS, cN = rN;
    if (c > 0) {
      cb = qbar[c * ne + m];
      nbr(c, cb, cW, cE, cS, cN);
    }
    // the neighbour-difference arguments of minmod3 are the element's, shared by
    // its 2N edge points along each axis: reduce them once
    const MM3 mx(cE - cb, cb - cW), my(cN - cb, cb - cS);
    double r[NP];
    const double* Qc = q + c * A.cs + m * NP;
    if constexpr (NP % 4 == 0) {  // P1, P3: the element's values as 32-B vectors (32-B aligned: cs, NP % 4 == 0)
#pragma unroll
      for (int p = 0; p < NP; p += 4)
        asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(r[p]), "=d"(r[p + 1]), "=d"(r[p + 2]), "=d"(r[p + 3])
                     : "l"(Qc + p));
    } else {
#pragma unroll
      for (int p = 0; p < NP; ++p) r[p] = Qc[p];
    }
#pragma unroll
    for (int t = 0; t < N; ++t) {
      double qw, qe_, qs, qn;
      if (GLLP) {  // GLL edge nodes are solution points
        qw = r[t * N];
        qe_ = r[t * N + N - 1];
        qs = r[t];
        qn = r[(N - 1) * N + t];
      } else {     // GL: interpolated traces of row t / column t
        qw = qe_ = qs = qn = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) {
          qw += nd.eL[l] * r[t * N + l];
          qe_ += nd.eR[l] * r[t * N + l];
          qs += nd.eL[l] * r[l * N + t];
          qn += nd.eR[l] * r[l * N + t];
        }
      }
      // right/top side: q_e = qbar + mm(q_l - qbar, ...); left/bottom: qbar - mm(qbar - q_l, ...)
      const double ew = cb - mx(cb - qw);
      const double ee = cb + mx(qe_ - cb);
      const double es = cb - my(cb - qs);
      const double en = cb + my(qn - cb);
      trip |= (fabs(qw - ew) > eps) | (fabs(qe_ - ee) > eps) | (fabs(qs - es) > eps) | (fabs(qn - en) > eps);
    }
  }
  return trip;
}

// Alg. 11 / Eq. (35) on a marked element: minmod slopes of the neighbour-average
// differences, per component or (CHAR, f3 variant of Q12) per characteristic
// field of the average; all four components rebuilt
template <int N, bool CHAR>
__device__ __forceinline__ void rebuild_element(const AuxArgs& A, const Nodes& nd, double* __restrict__ q,
                                             const Nbr& nbr, double dx, double dy, long long* dec, long long* emap,
                                             bool wantlam = false, double* lam = nullptr,
                                             unsigned long long* bad = nullptr) {
  constexpr int NP = N * N;
  const long long ne = nbr.ne, m = nbr.m;
  const double* __restrict__ qbar = nbr.qbar;
  if (dec) atomicAdd((unsigned long long*)&dec[0], 1ull);
  if (emap) emap[m] += 1;  // one thread per element
  double qv[4], dE[4], dW[4], dN[4], dS[4], sx[4], sy[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double qc = qbar[c * ne + m];
    double W, E, S, Nn;
    nbr(c, qc, W, E, S, Nn);
    qv[c] = qc;
    dE[c] = (E - qc) / dx;
    dW[c] = (qc - W) / dx;
    dN[c] = (Nn - qc) / dy;
    dS[c] = (qc - S) / dy;
  }
  if (CHAR) {
    char_slopes<0>(qv, dE, dW, A.gamma, sx);
    char_slopes<1>(qv, dN, dS, A.gamma, sy);
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      sx[c] = minmod2(dE[c], dW[c], nullptr);
      sy[c] = minmod2(dN[c], dS[c], nullptr);
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double* Qc = q + c * A.cs + m * NP;
#pragma unroll
    for (int b = 0; b < N; ++b)
#pragma unroll
      for (int a = 0; a < N; ++a)
        Qc[b * N + a] = qv[c] + (0.5 * dx) * nd.xi[a] * sx[c] + (0.5 * dy) * nd.xi[b] * sy[c];
  }
  if (wantlam) {  // the dt wave speed and non-physical check of the rebuilt points (same values)
    const double gm1 = A.gamma - 1.0;
    for (int b = 0; b < N; ++b)
      for (int a = 0; a < N; ++a) {
        double v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = qv[c] + (0.5 * dx) * nd.xi[a] * sx[c] + (0.5 * dy) * nd.xi[b] * sy[c];
        const Prim w = prims(v, gm1);
        *lam = nanmax(*lam, fmax(fabs(w.u), fabs(w.v)) + fsqrt(A.gamma * w.p * w.ri));
        if (!admissible(v[0], w.p)) *bad = min(*bad, (unsigned long long)(m * NP + b * N + a));
      }
  }
}

// rows of elements per thread: the detections of a thread's LROWS elements issue
// their loads back to back (and with the dt flag's), one memory round trip for all
// A/B: 4 vs 2 +0.8 % (CPR P1 shock tube); at the 64-register cap 4 rows double the
// spills of the characteristic variants and spill the P2 GL one, so 4 only for
// the default P1 variants
#ifndef H2D_LROWS
#define H2D_LROWS(N, CHAR) ((N) == 2 && !(CHAR) ? 4 : ((N) <= 3 ? 2 : 1))
#endif

// LamFuse (limiter runs, after stage 3): the dt wave speed and the non-physical
// check of the LIMITED state without another pass over it -- unmarked elements
// keep their stage-3 output, whose per-line speeds / first bad points the stage
// kernel wrote (laml / badl, N entries per element); marked elements are
// evaluated here at their rebuilt points; block max -> atomicMax(lam_out)


template <int N, bool GLLP, bool ALL, bool CHAR>
__global__ void __launch_bounds__(128, H2D_LIMIT_MINB) k_limit(const AuxArgs A, Nodes nd, double* __restrict__ q,
                                                               const double* __restrict__ qbar,
                                                               const double* qbar_lo, const double* qbar_hi,
                                                               long long gcs, int bcx, double eps, double dx,
                                                               double dy, long long* dec, long long* emap,
                                                               const LamFuse lf) {
  constexpr int R = H2D_LROWS(N, CHAR);
  __shared__ double sred[32];
  pdl_wait();
  pdl_launch();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < A.nx, fuse = lf.lam_out != nullptr;
  const bool done = A.dt && *A.dt == 0.0;  // past t_end (graph replay): no writes (uniform)
  double lam = 0.0;
  unsigned long long bad = ~0ull;
  if (active) {
    for (int j0 = blockIdx.y * R; j0 < A.nrows; j0 += gridDim.y * R) {
      bool trip[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        trip[r] = j0 + r < A.nrows &&
                  detect_element<N, GLLP, ALL>(A, nd, q, Nbr(A, qbar, qbar_lo, qbar_hi, gcs, bcx, i, j0 + r), eps);
      if (done) return;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (trip[r]) {
          rebuild_element<N, CHAR>(A, nd, q, Nbr(A, qbar, qbar_lo, qbar_hi, gcs, bcx, i, j0 + r), dx, dy, dec, emap,
                                   fuse, &lam, &bad);
        } else if (fuse && j0 + r < A.nrows) {
          const long long li = ((long long)(j0 + r) * A.nx + i) * N;
#pragma unroll
          for (int b = 0; b < N; ++b) {
            lam = nanmax(lam, lf.laml[li + b]);
            bad = min(bad, lf.badl[li + b]);
          }
        }
      }
    }
  }
  if (done || !fuse) return;  // (uniform)
  if (lf.bad_out && bad != ~0ull) atomicMin(lf.bad_out, bad);
  block_max_to(lam, lf.lam_out, sred);
}
}  // namespace

void launch_lambda(const AuxArgs& a, const double* q, unsigned long long* lam, unsigned long long* bad,
                   cudaStream_t s) {
  const long long npts = a.cs;
  launch_pdl(k_lambda, dim3(grid_for(npts, 256)), dim3(256), 0, s, a, q, npts, lam, bad);
}

void launch_dt(double* clock, unsigned long long* lam, double cfl, double hmin, cudaStream_t s) {
  launch_pdl(k_dt, dim3(1), dim3(1), 0, s, clock, lam, cfl, hmin);
}

void launch_init_case(const AuxArgs& a, int case_id, double* q, cudaStream_t s) {
  k_init<<<grid_for(a.cs, 256), 256, 0, s>>>(a, nodes_for(a.method, a.k), gl8(), case_id, q);
}

int launch_error_partials(const AuxArgs& a, const double* q, int var, const double* clock, double* part,
                          int max_blocks, cudaStream_t s) {
  int nb = grid_for(a.cs, 256);
  if (nb > max_blocks) nb = max_blocks;
  k_err<<<nb, 256, 0, s>>>(a, nodes_for(a.method, a.k), gl8(), q, var, clock, part);
  return nb;
}

int launch_error_fv_recon(const AuxArgs& a, const double* q, const double* glo, const double* ghi, long long gcs,
                          int bcx, int unlimited, int var, const double* clock, double* part, int max_blocks,
                          cudaStream_t s) {
  int nb = grid_for((long long)a.nx * a.nrows, 256);
  if (nb > max_blocks) nb = max_blocks;
  const Nodes g3 = nodes_for(2 /* Gauss-Legendre */, 2);
  switch (a.k + (unlimited ? 2 : 0)) {
    case 1: k_err_fvr<1><<<nb, 256, 0, s>>>(a, g3, q, glo, ghi, gcs, bcx, var, clock, part); break;
    case 2: k_err_fvr<2><<<nb, 256, 0, s>>>(a, g3, q, glo, ghi, gcs, bcx, var, clock, part); break;
    case 3: k_err_fvr<3><<<nb, 256, 0, s>>>(a, g3, q, glo, ghi, gcs, bcx, var, clock, part); break;
    default: k_err_fvr<4><<<nb, 256, 0, s>>>(a, g3, q, glo, ghi, gcs, bcx, var, clock, part); break;
  }
  return nb;
}

void launch_error_final(const double* part, int nb, double* out3, cudaStream_t s) {
  k_err_final<<<1, 32, 0, s>>>(part, nb, out3);
}

void launch_averages(const AuxArgs& a, const double* q, double* qbar, cudaStream_t s) {
  const long long ne = (long long)a.nx * a.nrows;
  launch_pdl(k_avg, dim3(grid_for(ne, 128)), dim3(128), 0, s, a, nodes_for(a.method, a.k), q, qbar);
}

template <int N, bool GLLP, bool ALL, bool CHAR>
void launch_limit_t(const AuxArgs& a, double* q, const double* qbar, const double* qbar_lo, const double* qbar_hi,
                    long long qbar_gcs, int bcx, double eps, long long* dec, long long* emap, const LamFuse& lf,
                    cudaStream_t s) {
  const int ry = (a.nrows + H2D_LROWS(N, CHAR) - 1) / H2D_LROWS(N, CHAR);
  dim3 grid((a.nx + 127) / 128, ry < 65535 ? ry : 65535);
  // element widths (Eq. (35)) in host IEEE double: bitwise the device's quotient
  const double dx = (a.xmax - a.xmin) / a.nx, dy = (a.ymax - a.ymin) / a.ny_global;
  launch_pdl(k_limit<N, GLLP, ALL, CHAR>, grid, dim3(128), 0, s, a, nodes_for(a.method, a.k), q, qbar, qbar_lo,
             qbar_hi, qbar_gcs, bcx, eps, dx, dy, dec, emap, lf);
}

template <int N, bool GLLP>
void launch_limit_g(const AuxArgs& a, double* q, const double* qbar, const double* qbar_lo, const double* qbar_hi,
                    long long qbar_gcs, int bcx, double eps, int all_vars, int charact, long long* dec,
                    long long* emap, const LamFuse& lf, cudaStream_t s) {
  if (all_vars && charact) launch_limit_t<N, GLLP, true, true>(a, q, qbar, qbar_lo, qbar_hi, qbar_gcs, bcx, eps, dec, emap, lf, s);
  else if (all_vars) launch_limit_t<N, GLLP, true, false>(a, q, qbar, qbar_lo, qbar_hi, qbar_gcs, bcx, eps, dec, emap, lf, s);
  else if (charact) launch_limit_t<N, GLLP, false, true>(a, q, qbar, qbar_lo, qbar_hi, qbar_gcs, bcx, eps, dec, emap, lf, s);
  else launch_limit_t<N, GLLP, false, false>(a, q, qbar, qbar_lo, qbar_hi, qbar_gcs, bcx, eps, dec, emap, lf, s);
}

template <int N>
void launch_limit_n(const AuxArgs& a, double* q, const double* qbar, const double* qbar_lo, const double* qbar_hi,
                    long long qbar_gcs, int bcx, double eps, int all_vars, int charact, long long* dec,
                    long long* emap, const LamFuse& lf, cudaStream_t s) {
  if (a.method == 1 || a.method == 3)
    launch_limit_g<N, true>(a, q, qbar, qbar_lo, qbar_hi, qbar_gcs, bcx, eps, all_vars, charact, dec, emap, lf, s);
  else
    launch_limit_g<N, false>(a, q, qbar, qbar_lo, qbar_hi, qbar_gcs, bcx, eps, all_vars, charact, dec, emap, lf, s);
}

void launch_limit(const AuxArgs& a, double* q, const double* qbar, const double* qbar_lo, const double* qbar_hi,
                  long long qbar_gcs, int bcx, double eps, int all_vars, int charact, long long* dec,
                  long long* emap, cudaStream_t s, const LamFuse& lf) {
  switch (a.k) {
    case 1: return launch_limit_n<2>(a, q, qbar, qbar_lo, qbar_hi, qbar_gcs, bcx, eps, all_vars, charact, dec, emap, lf, s);
    case 2: return launch_limit_n<3>(a, q, qbar, qbar_lo, qbar_hi, qbar_gcs, bcx, eps, all_vars, charact, dec, emap, lf, s);
    case 3: return launch_limit_n<4>(a, q, qbar, qbar_lo, qbar_hi, qbar_gcs, bcx, eps, all_vars, charact, dec, emap, lf, s);
    default: return launch_limit_n<5>(a, q, qbar, qbar_lo, qbar_hi, qbar_gcs, bcx, eps, all_vars, charact, dec, emap, lf, s);
  }
}

}  // namespace h2d
