// gll_stage.cu -- fused RK-stage kernel of the methods whose solution points are
// Gauss-Lobatto nodes coinciding with the flux points: CPR (chain rule,
// Radau/g_DG correction, Algs. 7-8 P:684-767) and NDG (D[F] + lift,
// Eqs. (24)-(29) P:300-318).  "The operations to compute the flux derivative are
// contained in one GPU kernel" -- here together with the SSP-RK3
// combination and the dt wave-speed reduction.
//
// Mapping (B200 design, not the paper's thread-per-point Alg. 7-8): ONE THREAD
// PER ELEMENT LINE (the n points of row b of one element), a TX x TY element
// tile per CTA.  The xi-direction work of a line (derivative, both x-faces'
// jumps, correction) stays in registers; only the eta-derivative operands
// (the element's q, or g for NDG) and the face records cross threads through
// shared memory, mostly as broadcasts (all n lines of an element read the same
// column values).  Loads/stores: a line is n contiguous doubles of the
// canonical layout, consecutive lanes hold consecutive lines -> fully coalesced.
//
//   phase 0  load the line; eta-operands -> smem; E-node record (q, f, |u|+c)
//            for the E neighbour; line n-1: N-row records (q, g, |v|+c);
//            halo threads: W-halo E-node records, S-halo N-row records.
//   phase 1  each line: its W face Rusanov flux (one per face); line 0: the S
//            faces; halo threads: the tile's E and N boundary faces.
//   phase 2  jE from the right neighbour's W-face flux; line n-1: the N jumps.
//   phase 3  per point: derivatives, chain rule (CPR) / D[F] (NDG), the four
//            correction terms, RK combination, coalesced store, dt epilogue.
#include "common.cuh"
#include "ops_tables.h"

namespace h2d {

namespace {

template <int K> struct GTile;
// tiles sized so that two CTAs fit the 228 KB of shared memory of an SM
template <> struct GTile<1> { static constexpr int TX = 16, TY = 8, MINB = 2; };  // 256 threads,  95 KB
template <> struct GTile<2> { static constexpr int TX = 8, TY = 8, MINB = 2; };   // 192 threads,  79 KB
template <> struct GTile<3> { static constexpr int TX = 8, TY = 6, MINB = 2; };   // 192 threads,  86 KB
template <> struct GTile<4> { static constexpr int TX = 8, TY = 4, MINB = 2; };   // 160 threads,  78 KB

enum { GM_CPR = 1, GM_NDG = 3 };
constexpr int RS = 10;  // record: q[4], flux[4], speed, pad

template <int M, int K>
struct G {
  static constexpr int N = K + 1, NP = N * N;
  static constexpr int TX = GTile<K>::TX, TY = GTile<K>::TY, MINB = GTile<K>::MINB;
  static constexpr int NE = TX * TY, NT = NE * N;
  // shared memory (doubles)
  static constexpr int OQ = 0;                              // eta operands [el][p][4] (q or g)
  static constexpr int ORE = OQ + NE * NP * 4;              // E-node records [ry][sx 0..TX][b][RS]
  static constexpr int ORN = ORE + TY * (TX + 1) * N * RS;  // N-row records [sy 0..TY][lx][a][RS]
  static constexpr int OFW = ORN + (TY + 1) * TX * N * RS;  // W-face fluxes [ry][fx 0..TX][b][4]
  static constexpr int OFS = OFW + TY * (TX + 1) * N * 4;   // S-face fluxes [fy 0..TY][lx][a][4]
  static constexpr int OJ = OFS + (TY + 1) * TX * N * 4;    // y jumps [el][S,N][a][4]
  static constexpr int OT = OJ + NE * 2 * N * 4;            // D[N][N], gL[N], gR[N]
  static constexpr int OR = OT + ((N * N + 2 * N + 1) & ~1);
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

// node record: q, the DIR flux, the DIR normal wave speed |u_n| + c
template <int DIR>
__device__ __forceinline__ void make_rec(const double q[4], double gm1, double gam, double f[4], double& s) {
  const Prim w = prims(q, gm1);
  flux<DIR>(q, w, f);
  s = fabs(DIR == 0 ? w.u : w.v) + sqrt(gam * w.p * w.ri);
}
__device__ __forceinline__ void put_rec(double* r, const double q[4], const double f[4], double s) {
  st4(r, q);
  st4(r + 4, f);
  r[8] = s;
}
__device__ __forceinline__ void get_rec(const double* r, double q[4], double f[4], double& s) {
  ld4(r, q);
  ld4(r + 4, f);
  s = r[8];
}

// Rusanov flux from two precomputed records (no division, no sqrt)
__device__ __forceinline__ void rus(const double qL[4], const double fL[4], double sL, const double qR[4],
                                    const double fR[4], double sR, double F[4]) {
  const double lam = fmax(sL, sR);
#pragma unroll
  for (int c = 0; c < 4; ++c) F[c] = 0.5 * (fL[c] + fR[c]) - 0.5 * lam * (qR[c] - qL[c]);
}

// start of element row gj (values) and its component stride; nullptr at a
// physical transmissive boundary (rows -1 / nrows come from the ghost rows)
__device__ __forceinline__ const double* row_base(const StageArgs& a, int gj, int np, long long& cs) {
  if (gj < 0) { cs = a.gcs; return a.ghost_lo; }
  if (gj >= a.nrows) { cs = a.gcs; return a.ghost_hi ? a.ghost_hi + (long long)(gj - a.nrows) * a.nx * np : nullptr; }
  cs = a.cs;
  return a.q + (long long)gj * a.nx * np;
}

}  // namespace

template <int M, int K>
__global__ void __launch_bounds__(G<M, K>::NT, G<M, K>::MINB) gll_stage_kernel(const StageArgs a, const GTab tab) {
  using H = G<M, K>;
  constexpr int N = H::N, NP = H::NP, TX = H::TX, TY = H::TY, NT = H::NT;
  extern __shared__ double4 smem4[];
  double* sm = reinterpret_cast<double*>(smem4);
  double* sQ = sm + H::OQ;
  double* sRE = sm + H::ORE;
  double* sRN = sm + H::ORN;
  double* sFW = sm + H::OFW;
  double* sFS = sm + H::OFS;
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

  const int el = tid / N, b = tid - el * N;
  const int lx = el % TX, ly = el / TX;
  const bool own = (lx < TXv) && (ly < TYv);
  const bool mirW = (i0 == 0 && a.bcx), mirE = (i0 + TXv == a.nx && a.bcx);
  const bool mirS = (j0 == 0 && !a.ghost_lo), mirN = (j0 + TYv == a.nrows && !a.ghost_hi);
  auto RE = [&](int ry, int sx, int bb) { return sRE + ((ry * (TX + 1) + sx) * N + bb) * RS; };
  auto RN = [&](int sy, int xx, int aa) { return sRN + ((sy * TX + xx) * N + aa) * RS; };
  auto FW = [&](int ry, int fx, int bb) { return sFW + ((ry * (TX + 1) + fx) * N + bb) * 4; };
  auto FS = [&](int fy, int xx, int aa) { return sFS + ((fy * TX + xx) * N + aa) * 4; };

  // ---- phase 0 ------------------------------------------------------------------
  const long long gel = (long long)(j0 + ly) * a.nx + (i0 + lx);  // global element
  double q[4][N];   // q[c][a] of the own line
  double fW[4], fE[4], sW = 0.0;
  if (own) {
    const long long base = gel * NP + b * N;
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int x = 0; x < N; ++x) q[c][x] = __ldg(a.q + c * a.cs + base + x);
    // eta operands: q (CPR) or g(q) (NDG) at every point of the line
#pragma unroll
    for (int x = 0; x < N; ++x) {
      double v[4] = {q[0][x], q[1][x], q[2][x], q[3][x]};
      if (M == GM_NDG) {
        double g[4];
        flux<1>(v, prims(v, gm1), g);
        st4(sQ + (el * NP + b * N + x) * 4, g);
      } else {
        st4(sQ + (el * NP + b * N + x) * 4, v);
      }
    }
    double qw[4] = {q[0][0], q[1][0], q[2][0], q[3][0]};
    double qe[4] = {q[0][N - 1], q[1][N - 1], q[2][N - 1], q[3][N - 1]};
    double se;
    make_rec<0>(qw, gm1, gam, fW, sW);
    make_rec<0>(qe, gm1, gam, fE, se);
    put_rec(RE(ly, lx + 1, b), qe, fE, se);
    if (lx == 0 && mirW) put_rec(RE(ly, 0, b), qw, fW, sW);  // transmissive: ghost = own trace
    if (b == N - 1) {  // N-row records for the element above
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double v[4] = {q[0][x], q[1][x], q[2][x], q[3][x]}, g[4], s;
        make_rec<1>(v, gm1, gam, g, s);
        put_rec(RN(ly + 1, lx, x), v, g, s);
      }
    }
  }
  // halo: W neighbour E-node records (TY*N), S neighbour N-row records (TX*N)
  for (int h = tid; h < TY * N + TX * N; h += NT) {
    if (h < TY * N) {
      const int ry = h / N, bb = h % N;
      if (ry >= TYv || mirW) continue;
      int gi = i0 - 1;
      if (gi < 0) gi += a.nx;
      const long long gx = ((long long)(j0 + ry) * a.nx + gi) * NP + bb * N + (N - 1);
      double v[4], f[4], s;
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = __ldg(a.q + c * a.cs + gx);
      make_rec<0>(v, gm1, gam, f, s);
      put_rec(RE(ry, 0, bb), v, f, s);
    } else {
      const int u = h - TY * N, xx = u / N, aa = u % N;
      if (xx >= TXv) continue;
      long long cs;
      const double* rb = row_base(a, j0 - 1, NP, cs);
      double v[4], f[4], s;
      if (rb) {
        const long long gx = (long long)(i0 + xx) * NP + (N - 1) * N + aa;
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = __ldg(rb + c * cs + gx);
      } else {  // transmissive: ghost = own S-row node
        const long long gx = ((long long)j0 * a.nx + i0 + xx) * NP + aa;
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = __ldg(a.q + c * a.cs + gx);
      }
      make_rec<1>(v, gm1, gam, f, s);
      put_rec(RN(0, xx, aa), v, f, s);
    }
  }
  __syncthreads();

  // ---- phase 1: one Rusanov flux per face point ------------------------
  double jW[4];
  if (own) {
    double qw[4] = {q[0][0], q[1][0], q[2][0], q[3][0]}, ql[4], fl[4], sl, F[4];
    get_rec(RE(ly, lx, b), ql, fl, sl);
    rus(ql, fl, sl, qw, fW, sW, F);
    st4(FW(ly, lx, b), F);
#pragma unroll
    for (int c = 0; c < 4; ++c) jW[c] = F[c] - fW[c];
    if (b == 0) {  // S faces of the element
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double v[4] = {q[0][x], q[1][x], q[2][x], q[3][x]}, g[4], s, qb[4], gb[4], sb, G[4], j[4];
        make_rec<1>(v, gm1, gam, g, s);
        get_rec(RN(ly, lx, x), qb, gb, sb);
        rus(qb, gb, sb, v, g, s, G);
        st4(FS(ly, lx, x), G);
#pragma unroll
        for (int c = 0; c < 4; ++c) j[c] = G[c] - g[c];
        st4(sJ + ((el * 2 + 0) * N + x) * 4, j);
      }
    }
  }
  // halo: the tile's E boundary faces (TY*N) and N boundary faces (TX*N)
  for (int h = tid; h < TY * N + TX * N; h += NT) {
    if (h < TY * N) {
      const int ry = h / N, bb = h % N;
      if (ry >= TYv) continue;
      double ql[4], fl[4], sl, v[4], f[4], s, F[4];
      get_rec(RE(ry, TXv, bb), ql, fl, sl);
      if (mirE) {
        rus(ql, fl, sl, ql, fl, sl, F);
      } else {
        int gi = i0 + TXv;
        if (gi >= a.nx) gi -= a.nx;
        const long long gx = ((long long)(j0 + ry) * a.nx + gi) * NP + bb * N;
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = __ldg(a.q + c * a.cs + gx);
        make_rec<0>(v, gm1, gam, f, s);
        rus(ql, fl, sl, v, f, s, F);
      }
      st4(FW(ry, TXv, bb), F);
    } else {
      const int u = h - TY * N, xx = u / N, aa = u % N;
      if (xx >= TXv) continue;
      double qb[4], gb[4], sb, v[4], g[4], s, G[4];
      get_rec(RN(TYv, xx, aa), qb, gb, sb);
      long long cs;
      const double* rb = row_base(a, j0 + TYv, NP, cs);
      if (mirN || !rb) {
        rus(qb, gb, sb, qb, gb, sb, G);
      } else {
        const long long gx = (long long)(i0 + xx) * NP + aa;
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = __ldg(rb + c * cs + gx);
        make_rec<1>(v, gm1, gam, g, s);
        rus(qb, gb, sb, v, g, s, G);
      }
      st4(FS(TYv, xx, aa), G);
    }
  }
  __syncthreads();

  // ---- phase 2: jumps on the E face (each line) and the N faces (line n-1) ----------
  double jE[4];
  if (own) {
    double F[4];
    ld4(FW(ly, lx + 1, b), F);
#pragma unroll
    for (int c = 0; c < 4; ++c) jE[c] = F[c] - fE[c];
    if (b == N - 1) {
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double G[4], qn[4], gn[4], sn, j[4];
        ld4(FS(ly + 1, lx, x), G);
        get_rec(RN(ly + 1, lx, x), qn, gn, sn);
#pragma unroll
        for (int c = 0; c < 4; ++c) j[c] = G[c] - gn[c];
        st4(sJ + ((el * 2 + 1) * N + x) * 4, j);
      }
    }
  }
  __syncthreads();

  // ---- phase 3: residual at the points of the line + SSP-RK3 --------------------------
  double lam = 0.0;
  if (own) {
    const double* D = sT;
    const double gLb = sT[N * N + b], gRb = sT[N * N + N + b];
    double fx_line[4][N];
    if (M == GM_NDG) {  // x-fluxes of the whole line for D[F]
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double v[4] = {q[0][x], q[1][x], q[2][x], q[3][x]}, f[4];
        flux<0>(v, prims(v, gm1), f);
#pragma unroll
        for (int c = 0; c < 4; ++c) fx_line[c][x] = f[c];
      }
    }
    const double bdt = a.bcoef * dtv;
    const long long base = gel * NP + b * N;
#pragma unroll
    for (int x = 0; x < N; ++x) {
      double v[4] = {q[0][x], q[1][x], q[2][x], q[3][x]};
      double Fx[4], Gy[4], dy[4] = {0, 0, 0, 0};
#pragma unroll
      for (int l = 0; l < N; ++l) {  // eta operands of column x from smem (broadcast over lines)
        double u[4];
        ld4(sQ + (el * NP + l * N + x) * 4, u);
        const double db = D[b * N + l];
#pragma unroll
        for (int c = 0; c < 4; ++c) dy[c] += db * u[c];
      }
      if (M == GM_CPR) {  // chain rule: A(q) dq/dxi + B(q) dq/deta
        double dx[4] = {0, 0, 0, 0};
#pragma unroll
        for (int l = 0; l < N; ++l) {
          const double da = D[x * N + l];
#pragma unroll
          for (int c = 0; c < 4; ++c) dx[c] += da * q[c][l];
        }
        const Prim w = prims(v, gm1);
        jac<0>(v, w, gm1, gam, dx, Fx);
        jac<1>(v, w, gm1, gam, dy, Gy);
      } else {            // NDG: D[F]
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double s = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) s += D[x * N + l] * fx_line[c][l];
          Fx[c] = s;
          Gy[c] = dy[c];
        }
      }
      double jS[4], jN[4];
      ld4(sJ + ((el * 2 + 0) * N + x) * 4, jS);
      ld4(sJ + ((el * 2 + 1) * N + x) * 4, jN);
      const double gLa = sT[N * N + x], gRa = sT[N * N + N + x];
      double o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double fx = Fx[c] + gLa * jW[c] + gRa * jE[c];
        const double gy = Gy[c] + gLb * jS[c] + gRb * jN[c];
        const double R = -a.rdx2 * fx - a.rdy2 * gy;
        double val = a.a1 * v[c] + bdt * R;
        if (a.q0) val += a.a0 * a.q0[c * a.cs + base + x];
        o[c] = val;
        a.out[c * a.cs + base + x] = val;
      }
      if (a.lam) lam = fmax(lam, wave_speed(o, gm1, gam));
      if (a.bad && nonphysical(o, gm1)) atomicMin(a.bad, (unsigned long long)(base + x));
    }
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
