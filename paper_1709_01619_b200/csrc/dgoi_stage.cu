// dgoi_stage.cu -- RK-stage kernel of DG with (k+2)-point Gauss-Legendre
// over-integration (hom2d_config.dg_overintegrate): the weak
// form of Eq. (19) with its volume and surface integrals evaluated
// by the (k+2)-point rule instead of the n-point collocation of Eq. (20)
// (the default DG path in gl_stage.cu).
//
//   R_ab = (2/dx) [ sum_rs W_r W_s f(q_h(z_r, z_s)) l'_a(z_r) l_b(z_s)
//                 - sum_t W_t (l_a(1) F^E(z_t) - l_a(-1) F^W(z_t)) l_b(z_t) ] / (w_a w_b)
//        + (2/dy) [ same with g, l_a <-> l_b, F^N, F^S ]
//
// q_h is the GL nodal polynomial of the element; F^E/W/N/S are Rusanov fluxes
// between the two traces at the k+2 Gauss points of the face.  A
// method variant, not the hot path: one thread per element, the element's
// values and its residual in shared memory (thread-interleaved, conflict-free),
// the integrals sum-factorised row by row of quadrature points, neighbour traces
// read from global memory (each element row is L2-resident while its
// neighbours run).  The stage epilogue (SSP-RK combination, wave speed,
// non-physical check, element averages for the limiter) is the fused one of the
// other stage kernels.
#include "common.cuh"
#include "ops_tables.h"

namespace h2d {

namespace {
constexpr int OI_NT = 64;  // threads (elements) per CTA

template <int K>
struct OiTab {
  double L[K + 2][K + 1], dL[K + 2][K + 1], W[K + 2], w[K + 1], eL[K + 1], eR[K + 1];
};

template <int K>
OiTab<K> make_oitab() {
  using O = Ops<K>;
  OiTab<K> t;
  for (int r = 0; r < K + 2; ++r) {
    t.W[r] = O::oi_W[r];
    for (int a = 0; a < K + 1; ++a) {
      t.L[r][a] = O::oi_L[r][a];
      t.dL[r][a] = O::oi_dL[r][a];
    }
  }
  for (int a = 0; a < K + 1; ++a) {
    t.w[a] = O::w_gl[a];
    t.eL[a] = O::eL_gl[a];
    t.eR[a] = O::eR_gl[a];
  }
  return t;
}
}  // namespace

template <int K>
__global__ void __launch_bounds__(OI_NT) dgoi_stage_kernel(const StageArgs a, const OiTab<K> T) {
  constexpr int n = K + 1, nq = K + 2, np = n * n;
  extern __shared__ __align__(16) double oi_smem[];
  double* const sq = oi_smem;                    // [4*np][OI_NT] element values
  double* const sR = oi_smem + 4 * np * OI_NT;   // [4*np][OI_NT] residual accumulator
  double* const sred = oi_smem + 8 * np * OI_NT;
  pdl_wait();
  pdl_launch();
  const double dtv = stage_dt(a);  // (stage 1 / 2 of a fused-dt step: publishes / commits the clock)
  if (dtv == 0.0) return;
  const int tid = threadIdx.x;
  const long long n1 = (long long)a.nx * (a.row_hi - a.row_lo);
  const long long nel = n1 + (long long)a.nx * (a.row_hi2 > a.row_lo2 ? a.row_hi2 - a.row_lo2 : 0);
  const long long e = (long long)blockIdx.x * OI_NT + tid;
  const double gm1 = a.gamma - 1.0, gam = a.gamma;
  double lam = 0.0;
  if (e < nel) {
    const int i = (int)(e % a.nx);
    const int jr = e < n1 ? a.row_lo + (int)(e / a.nx) : a.row_lo2 + (int)((e - n1) / a.nx);
    const long long m = (long long)jr * a.nx + i;
#define SQ(c, p) sq[((c) * np + (p)) * OI_NT + tid]
#define SR(c, p) sR[((c) * np + (p)) * OI_NT + tid]
    for (int c = 0; c < 4; ++c)
      for (int p = 0; p < np; ++p) {
        SQ(c, p) = a.q[c * a.cs + m * np + p];
        SR(c, p) = 0.0;
      }
    // ---- volume integrals, one row z_s of quadrature points at a time ----
#pragma unroll 1
    for (int s = 0; s < nq; ++s) {
      double qy[4][n];  // q_h(xi_a, z_s) along the GL x-nodes
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int aa = 0; aa < n; ++aa) {
          double v = 0.0;
#pragma unroll
          for (int b = 0; b < n; ++b) v = fma(T.L[s][b], SQ(c, b * n + aa), v);
          qy[c][aa] = v;
        }
      double tx[4][n], ty[4][n];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int aa = 0; aa < n; ++aa) tx[c][aa] = ty[c][aa] = 0.0;
#pragma unroll
      for (int r = 0; r < nq; ++r) {
        double qq[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double v = 0.0;
#pragma unroll
          for (int aa = 0; aa < n; ++aa) v = fma(T.L[r][aa], qy[c][aa], v);
          qq[c] = v;
        }
        const Prim w = prims(qq, gm1);
        double f[4], g[4];
        flux<0>(qq, w, f);
        flux<1>(qq, w, g);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int aa = 0; aa < n; ++aa) {
            tx[c][aa] = fma(T.W[r] * T.dL[r][aa], f[c], tx[c][aa]);
            ty[c][aa] = fma(T.W[r] * T.L[r][aa], g[c], ty[c][aa]);
          }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int b = 0; b < n; ++b) {
          const double cx = a.rdx2 * T.W[s] * T.L[s][b], cy = a.rdy2 * T.W[s] * T.dL[s][b];
#pragma unroll
          for (int aa = 0; aa < n; ++aa) SR(c, b * n + aa) = fma(cx, tx[c][aa], fma(cy, ty[c][aa], SR(c, b * n + aa)));
        }
    }
    // ---- surface integrals ----
    // trace line of element values V (row-major [b][a]) on side sd: x sides give a
    // line over b (contract a with e), y sides a line over a (contract b with e)
    int iw = i - 1, ie = i + 1;
    bool hw = true, he = true;
    if (a.bcx == 0) {
      iw = iw < 0 ? iw + a.nx : iw;
      ie = ie >= a.nx ? ie - a.nx : ie;
    } else {
      hw = iw >= 0;
      he = ie < a.nx;
    }
    // neighbour element base pointers and component strides (nullptr: transmissive)
    const double* pW = hw ? a.q + ((long long)jr * a.nx + iw) * np : nullptr;
    const double* pE = he ? a.q + ((long long)jr * a.nx + ie) * np : nullptr;
    long long csS = a.cs, csN = a.cs;
    const double* pS = nullptr;
    const double* pN = nullptr;
    if (jr > 0) pS = a.q + (m - a.nx) * np;
    else if (a.ghost_lo) { pS = a.ghost_lo + (long long)i * np; csS = a.gcs; }
    if (jr + 1 < a.nrows) pN = a.q + (m + a.nx) * np;
    else if (a.ghost_hi) { pN = a.ghost_hi + (long long)i * np; csN = a.gcs; }
    // one side at a time: sd 0 W, 1 E, 2 S, 3 N
#pragma unroll 1
    for (int sd = 0; sd < 4; ++sd) {
      const int dir = sd >> 1;
      const bool hiside = sd & 1;
      const double* pn = sd == 0 ? pW : sd == 1 ? pE : sd == 2 ? pS : pN;  // neighbour across the side
      const long long cn = sd == 2 ? csS : sd == 3 ? csN : a.cs;
      // own trace line on this side (e = eR on the hi side, eL on the lo side) and
      // the neighbour's trace on its facing side (the opposite e)
      double ol[4][n], nl[4][n];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int t = 0; t < n; ++t) {
          double vo = 0.0, vn = 0.0;
#pragma unroll
          for (int l = 0; l < n; ++l) {
            const int p = dir == 0 ? t * n + l : l * n + t;  // x: line t over l = a; y: column t over l = b
            const double eo = hiside ? T.eR[l] : T.eL[l], en = hiside ? T.eL[l] : T.eR[l];
            vo = fma(eo, SQ(c, p), vo);
            if (pn) vn = fma(en, pn[c * cn + p], vn);
          }
          ol[c][t] = vo;
          nl[c][t] = pn ? vn : vo;  // transmissive: ghost = own trace
        }
      double sacc[4][n];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int t = 0; t < n; ++t) sacc[c][t] = 0.0;
#pragma unroll 1
      for (int z = 0; z < nq; ++z) {
        double qo[4], qn[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double v0 = 0.0, v1 = 0.0;
#pragma unroll
          for (int t = 0; t < n; ++t) {
            v0 = fma(T.L[z][t], ol[c][t], v0);
            v1 = fma(T.L[z][t], nl[c][t], v1);
          }
          qo[c] = v0;
          qn[c] = v1;
        }
        // (west|south, east|north) order: the lo side's neighbour is on the left
        double F[4], f1[4], f2[4];
        if (dir == 0) {
          if (hiside) rusanov<0>(qo, qn, gm1, gam, F, f1, f2);
          else rusanov<0>(qn, qo, gm1, gam, F, f1, f2);
        } else {
          if (hiside) rusanov<1>(qo, qn, gm1, gam, F, f1, f2);
          else rusanov<1>(qn, qo, gm1, gam, F, f1, f2);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int t = 0; t < n; ++t) sacc[c][t] = fma(T.W[z] * T.L[z][t], F[c], sacc[c][t]);
      }
      // x: S^x_ab = eR_a sacc^E_b - eL_a sacc^W_b ; y: S^y_ab = eR_b sacc^N_a - eL_b sacc^S_a
      const double rd = (dir == 0 ? a.rdx2 : a.rdy2) * (hiside ? -1.0 : 1.0);
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int b = 0; b < n; ++b)
#pragma unroll
          for (int aa = 0; aa < n; ++aa) {
            const double S = dir == 0 ? (hiside ? T.eR[aa] : T.eL[aa]) * sacc[c][b]
                                      : (hiside ? T.eR[b] : T.eL[b]) * sacc[c][aa];
            SR(c, b * n + aa) = fma(rd, S, SR(c, b * n + aa));
          }
    }
    // ---- epilogue: mass matrix, RK combination, wave speed, averages ----
    const double bdt = a.bcoef * dtv;
    double avg[4] = {0, 0, 0, 0};
    unsigned long long bidx = ~0ull;
    for (int p = 0; p < np; ++p) {
      const double wab = T.w[p % n] * T.w[p / n];
      double o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double R = SR(c, p) / wab;
        double v = fma(a.a1, SQ(c, p), bdt * R);
        if (a.q0) v = fma(a.a0, a.q0[c * a.cs + m * np + p], v);
        o[c] = v;
        a.out[c * a.cs + m * np + p] = v;
        avg[c] = fma(0.25 * wab, v, avg[c]);
      }
      if (a.lam || a.bad) {
        const Prim w = prims(o, gm1);
        lam = nanmax(lam, fmax(fabs(w.u), fabs(w.v)) + fsqrt(gam * w.p * w.ri));
        if (!admissible(o[0], w.p)) bidx = min(bidx, (unsigned long long)(m * np + p));
      }
    }
    if (a.qbar) {
      const long long ne = (long long)a.nx * a.nrows;
#pragma unroll
      for (int c = 0; c < 4; ++c) a.qbar[c * ne + m] = avg[c];
    }
    if (a.qbar && a.laml) {  // limiter runs: the element's wave speed / first bad point (LamFuse)
      unsigned long long bl = ~0ull;
      double ll = 0.0;
      for (int p = 0; p < np; ++p) {
        double v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = a.out[c * a.cs + m * np + p];
        const Prim w = prims(v, gm1);
        ll = nanmax(ll, fmax(fabs(w.u), fabs(w.v)) + fsqrt(gam * w.p * w.ri));
        if (!admissible(v[0], w.p)) bl = min(bl, (unsigned long long)(m * np + p));
      }
      for (int b = 0; b < n; ++b) {
        a.laml[m * n + b] = b == 0 ? ll : 0.0;
        a.badl[m * n + b] = b == 0 ? bl : ~0ull;
      }
    }
    if (a.bad && bidx != ~0ull) atomicMin(a.bad, bidx);
#undef SQ
#undef SR
  }
  if (a.lam) block_max_to(lam, a.lam, sred);
}

template <int K>
static int launch_k(const StageArgs& a, int nr, cudaStream_t s) {
  static const OiTab<K> tab = make_oitab<K>();
  static std::atomic<unsigned long long> attr{0};
  constexpr int np = (K + 1) * (K + 1);
  const size_t smem = sizeof(double) * (8 * (size_t)np * OI_NT + 32);
  cudaError_t e = smem_optin(dgoi_stage_kernel<K>, (int)smem, attr);
  if (e != cudaSuccess) return (int)e;
  const long long nel = (long long)a.nx * nr;
  const dim3 grid((unsigned)((nel + OI_NT - 1) / OI_NT));
  e = launch_pdl_if(!a.no_pdl, dgoi_stage_kernel<K>, grid, dim3(OI_NT), smem, s, a, tab);
  return (int)e;
}

int launch_dgoi_stage(int k, const StageArgs& a0, cudaStream_t s) {
  StageArgs a = a0;
  const int nr = row_range(a);
  if (nr <= 0) return 0;
  switch (k) {
    case 1: return launch_k<1>(a, nr, s);
    case 2: return launch_k<2>(a, nr, s);
    case 3: return launch_k<3>(a, nr, s);
    default: return launch_k<4>(a, nr, s);
  }
}

}  // namespace h2d
