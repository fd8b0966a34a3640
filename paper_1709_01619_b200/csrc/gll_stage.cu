// gll_stage.cu -- fused RK-stage kernel of the methods whose solution points are
// Gauss-Lobatto nodes that coincide with the flux points: CPR (chain rule,
// Radau/g_DG correction, Algs. 7-8 P:684-767) and NDG (D[F] + lift,
// Eqs. (24)-(29) P:300-318).  "All computations of the flux derivative are
// contained in one GPU kernel" -- here together with the SSP-RK3
// combination and the dt wave-speed reduction.
//
// One thread per solution point, a TX x TY element tile per CTA.
//   phase 0  own point: 4 coalesced fp64 loads; primitives (one reciprocal), f, g,
//            |u|+c, |v|+c -> smem.  Halo edge nodes of the 4 neighbour
//            element strips are loaded and evaluated the same way (GLL: the
//            neighbour's trace IS its edge node; no interpolation).
//   phase 1  one Rusanov flux per tile face point from the precomputed q, f, s
//            of both sides (no division, no sqrt); the jumps F^ - f(own) of both
//            neighbouring elements -> smem.
//   phase 2  own point: d/dxi, d/deta along the element lines from smem, chain
//            rule (CPR) or D[F] (NDG), + the four correction terms, RK
//            combination, one coalesced store per component.
#include "common.cuh"
#include "ops_tables.h"

namespace h2d {

namespace {

template <int K> struct GTile;
template <> struct GTile<1> { static constexpr int TX = 8, TY = 8, MINB = 3; };   // 256 threads
template <> struct GTile<2> { static constexpr int TX = 8, TY = 4, MINB = 2; };   // 288 threads
template <> struct GTile<3> { static constexpr int TX = 4, TY = 4, MINB = 3; };   // 256 threads
template <> struct GTile<4> { static constexpr int TX = 4, TY = 3, MINB = 2; };   // 300 threads

enum { GM_CPR = 1, GM_NDG = 3 };

template <int M, int K>
struct G {
  static constexpr int N = K + 1, NP = N * N;
  static constexpr int TX = GTile<K>::TX, TY = GTile<K>::TY, MINB = GTile<K>::MINB;
  static constexpr int NE = TX * TY, NT = NE * NP;
  static constexpr int SX = TX + 2, SY = TY + 2, NS = SX * SY;    // element slots incl. halo
  static constexpr int NH = 2 * TY * N + 2 * TX * N;              // halo edge nodes
  static constexpr int NFX = (TX + 1) * TY * N, NFY = TX * (TY + 1) * N;
  // shared memory (doubles)
  static constexpr int OQ = 0;                       // q  [slot][p][4]
  static constexpr int OF = OQ + NS * NP * 4;        // f  [slot][p][4]
  static constexpr int OG = OF + NS * NP * 4;        // g  [slot][p][4]
  static constexpr int OS = OG + NS * NP * 4;        // (|u|+c, |v|+c) [slot][p][2]
  static constexpr int OJ = OS + NS * NP * 2;        // jumps [el][side W,E,S,N][t][4]
  static constexpr int OT = OJ + NE * 4 * N * 4;     // operator tables: D[N][N], gL[N], gR[N]
  static constexpr int OR = OT + N * N + 2 * N;      // reduction scratch [32]
  static constexpr int TOTAL = OR + 32;
  static constexpr size_t SMEM = TOTAL * sizeof(double);
};

struct GTab {
  double v[25 + 10];
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

// evaluate a point: primitives, both fluxes and both normal wave speeds -> smem
__device__ __forceinline__ void eval_point(const double q[4], double gm1, double gam, double* sf, double* sg, double* ss,
                                           Prim& w) {
  w = prims(q, gm1);
  double f[4], g[4];
  flux<0>(q, w, f);
  flux<1>(q, w, g);
  const double c = sqrt(gam * w.p * w.ri);
  st4(sf, f);
  st4(sg, g);
  reinterpret_cast<double2*>(ss)[0] = make_double2(fabs(w.u) + c, fabs(w.v) + c);
}

}  // namespace

template <int M, int K>
__global__ void __launch_bounds__(G<M, K>::NT, G<M, K>::MINB) gll_stage_kernel(const StageArgs a, const GTab tab) {
  using H = G<M, K>;
  constexpr int N = H::N, NP = H::NP, TX = H::TX, TY = H::TY, SX = H::SX, NT = H::NT;
  extern __shared__ double4 smem4[];
  double* sm = reinterpret_cast<double*>(smem4);
  double* sQ = sm + H::OQ;
  double* sF = sm + H::OF;
  double* sG = sm + H::OG;
  double* sS = sm + H::OS;
  double* sJ = sm + H::OJ;
  double* sT = sm + H::OT;

  double dtv = 1.0;
  if (a.dt) {
    dtv = *a.dt;
    if (dtv == 0.0) return;  // clipped-out step (t == t_end): uniform across the grid
  }
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int TXv = min(TX, a.nx - i0), TYv = min(TY, a.nrows - j0);
  const double gam = a.gamma, gm1 = a.gamma - 1.0;
  for (int i = tid; i < N * N + 2 * N; i += NT) sT[i] = tab.v[i];

  // ---- phase 0: own point -------------------------------------------------------
  const int el = tid / NP, p = tid - el * NP;
  const int lx = el % TX, ly = el / TX;
  const int ai = p % N, bi = p / N;
  const bool own = (lx < TXv) && (ly < TYv);
  const int slot = (ly + 1) * SX + (lx + 1);
  const long long gidx = ((long long)(j0 + ly) * a.nx + (i0 + lx)) * NP + p;
  double q[4];
  Prim w;
  if (own) {
#pragma unroll
    for (int c = 0; c < 4; ++c) q[c] = __ldg(a.q + c * a.cs + gidx);
    st4(sQ + (slot * NP + p) * 4, q);
    eval_point(q, gm1, gam, sF + (slot * NP + p) * 4, sG + (slot * NP + p) * 4, sS + (slot * NP + p) * 2, w);
  }
  // halo edge nodes: W column, E column, S row, N row of the neighbour elements
  for (int h = tid; h < H::NH; h += NT) {
    int hs, hx, hy, hp;   // slot x/y, node
    int gi, gj;
    bool ok = true;
    if (h < 2 * TY * N) {           // W / E
      const int side = h / (TY * N), r = h % (TY * N), yy = r / N, t = r % N;
      if (yy >= TYv) ok = false;
      hy = yy + 1;
      if (side == 0) { hx = 0; gi = i0 - 1; hp = t * N + (N - 1); }
      else { hx = TXv + 1; gi = i0 + TXv; hp = t * N; }
      gj = j0 + yy;
    } else {                        // S / N
      const int r0 = h - 2 * TY * N, side = r0 / (TX * N), r = r0 % (TX * N), xx = r / N, t = r % N;
      if (xx >= TXv) ok = false;
      hx = xx + 1;
      if (side == 0) { hy = 0; gj = j0 - 1; hp = (N - 1) * N + t; }
      else { hy = TYv + 1; gj = j0 + TYv; hp = t; }
      gi = i0 + xx;
    }
    if (!ok) continue;
    if (gi < 0) { if (a.bcx) continue; gi += a.nx; }
    else if (gi >= a.nx) { if (a.bcx) continue; gi -= a.nx; }
    const double* base;
    long long cs;
    if (gj < 0) { if (!a.ghost_lo) continue; base = a.ghost_lo; cs = a.gcs; gj = 0; }
    else if (gj >= a.nrows) { if (!a.ghost_hi) continue; base = a.ghost_hi; cs = a.gcs; gj -= a.nrows; }
    else { base = a.q; cs = a.cs; }
    hs = hy * SX + hx;
    const long long gx = ((long long)gj * a.nx + gi) * NP + hp;
    double hq[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) hq[c] = __ldg(base + c * cs + gx);
    Prim hw;
    st4(sQ + (hs * NP + hp) * 4, hq);
    eval_point(hq, gm1, gam, sF + (hs * NP + hp) * 4, sG + (hs * NP + hp) * 4, sS + (hs * NP + hp) * 2, hw);
  }
  __syncthreads();

  // ---- phase 1: Rusanov at every tile face point ----------------------
  for (int t = tid; t < H::NFX + H::NFY; t += NT) {
    int sL, pL, sR, pR, elL, elR, sideL, sideR, ln, dir;
    bool hasL, hasR, mirL, mirR, ok;
    if (t < H::NFX) {
      dir = 0;
      ln = t % N;
      const int r = t / N, fx = r % (TX + 1), yy = r / (TX + 1);
      ok = (yy < TYv) && (fx <= TXv);
      sL = (yy + 1) * SX + fx; pL = ln * N + (N - 1);
      sR = (yy + 1) * SX + fx + 1; pR = ln * N;
      hasL = fx > 0; hasR = fx < TXv;
      elL = yy * TX + fx - 1; elR = yy * TX + fx;
      sideL = 1; sideR = 0;
      mirL = (fx == 0 && i0 == 0 && a.bcx); mirR = (fx == TXv && i0 + TXv == a.nx && a.bcx);
    } else {
      dir = 1;
      const int u = t - H::NFX;
      ln = u % N;
      const int r = u / N, xx = r % TX, fy = r / TX;
      ok = (xx < TXv) && (fy <= TYv);
      sL = fy * SX + xx + 1; pL = (N - 1) * N + ln;
      sR = (fy + 1) * SX + xx + 1; pR = ln;
      hasL = fy > 0; hasR = fy < TYv;
      elL = (fy - 1) * TX + xx; elR = fy * TX + xx;
      sideL = 3; sideR = 2;
      mirL = (fy == 0 && j0 == 0 && !a.ghost_lo); mirR = (fy == TYv && j0 + TYv == a.nrows && !a.ghost_hi);
    }
    if (!ok) continue;
    if (mirL) { sL = sR; pL = pR; }
    if (mirR) { sR = sL; pR = pL; }
    const double* sFl = dir == 0 ? sF : sG;
    double qL[4], qR[4], fL[4], fR[4];
    ld4(sQ + (sL * NP + pL) * 4, qL);
    ld4(sQ + (sR * NP + pR) * 4, qR);
    ld4(sFl + (sL * NP + pL) * 4, fL);
    ld4(sFl + (sR * NP + pR) * 4, fR);
    const double lam = fmax(sS[(sL * NP + pL) * 2 + dir], sS[(sR * NP + pR) * 2 + dir]);
    double jL[4], jR[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double F = 0.5 * (fL[c] + fR[c]) - 0.5 * lam * (qR[c] - qL[c]);
      jL[c] = F - fL[c];
      jR[c] = F - fR[c];
    }
    if (hasL) st4(sJ + ((elL * 4 + sideL) * N + ln) * 4, jL);
    if (hasR) st4(sJ + ((elR * 4 + sideR) * N + ln) * 4, jR);
  }
  __syncthreads();

  // ---- phase 2: residual at the own point + SSP-RK3 combination ---------------------
  double lam = 0.0;
  if (own) {
    double Fx[4], Gy[4];
    const double* D = sT;
    if (M == GM_CPR) {  // chain rule: A(q) dq/dxi + B(q) dq/deta
      double dx[4] = {0, 0, 0, 0}, dy[4] = {0, 0, 0, 0};
#pragma unroll
      for (int l = 0; l < N; ++l) {
        double v[4], u[4];
        ld4(sQ + (slot * NP + bi * N + l) * 4, v);
        ld4(sQ + (slot * NP + l * N + ai) * 4, u);
        const double da = D[ai * N + l], db = D[bi * N + l];
#pragma unroll
        for (int c = 0; c < 4; ++c) { dx[c] += da * v[c]; dy[c] += db * u[c]; }
      }
      jac<0>(q, w, gm1, gam, dx, Fx);
      jac<1>(q, w, gm1, gam, dy, Gy);
    } else {            // NDG: D[F]
#pragma unroll
      for (int c = 0; c < 4; ++c) { Fx[c] = 0.0; Gy[c] = 0.0; }
#pragma unroll
      for (int l = 0; l < N; ++l) {
        double v[4], u[4];
        ld4(sF + (slot * NP + bi * N + l) * 4, v);
        ld4(sG + (slot * NP + l * N + ai) * 4, u);
        const double da = D[ai * N + l], db = D[bi * N + l];
#pragma unroll
        for (int c = 0; c < 4; ++c) { Fx[c] += da * v[c]; Gy[c] += db * u[c]; }
      }
    }
    // correction (CPR, Radau g_DG) == lift (NDG): 2 updates per direction (Alg. 8)
    const double gLa = sT[N * N + ai], gRa = sT[N * N + N + ai], gLb = sT[N * N + bi], gRb = sT[N * N + N + bi];
    double jW[4], jE[4], jS[4], jN[4];
    ld4(sJ + ((el * 4 + 0) * N + bi) * 4, jW);
    ld4(sJ + ((el * 4 + 1) * N + bi) * 4, jE);
    ld4(sJ + ((el * 4 + 2) * N + ai) * 4, jS);
    ld4(sJ + ((el * 4 + 3) * N + ai) * 4, jN);
    const double bdt = a.bcoef * dtv;
    double o[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double fx = Fx[c] + gLa * jW[c] + gRa * jE[c];
      const double gy = Gy[c] + gLb * jS[c] + gRb * jN[c];
      const double R = -a.rdx2 * fx - a.rdy2 * gy;
      double v = a.a1 * q[c] + bdt * R;
      if (a.q0) v += a.a0 * a.q0[c * a.cs + gidx];
      o[c] = v;
      a.out[c * a.cs + gidx] = v;
    }
    if (a.lam) lam = wave_speed(o, gm1, gam);
    if (a.bad && nonphysical(o, gm1)) atomicMin(a.bad, (unsigned long long)gidx);
  }
  if (a.lam) block_max_to(lam, a.lam, sm + H::OR);
}

template <int M, int K>
static int launch_g(const StageArgs& a, cudaStream_t s) {
  using H = G<M, K>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gll_stage_kernel<M, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H::SMEM);
    attr = true;
  }
  static const GTab tab = make_gtab<K>();
  dim3 grid((a.nx + H::TX - 1) / H::TX, (a.nrows + H::TY - 1) / H::TY);
  gll_stage_kernel<M, K><<<grid, H::NT, H::SMEM, s>>>(a, tab);
  return (int)cudaPeekAtLastError();
}

int launch_gll_stage(int method, int k, const StageArgs& a, cudaStream_t s) {
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
