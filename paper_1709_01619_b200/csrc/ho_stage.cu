// ho_stage.cu -- fused RK-stage kernels of the high-order methods (CPR, NDG, DG,
// SD) for sm_100a.  One launch = one full RK stage over the local strip:
//   state tile + neighbour halo -> shared memory            (P:399-406 SoA reads)
//   traces / interpolation to flux points  (DG: Alg. 2; SD: Alg. 5)
//   Rusanov flux at every tile face point  (Alg. 3; Alg. 8)
//   element-local derivative + correction  (CPR/NDG: Algs. 7-8 P:684-767;
//      DG: Alg. 4 P:537-570 sum-factorised; SD: Alg. 6)
//   SSP-RK3 combination, non-physical check and the wave-speed max of the
//   new state for the next dt (Eq. (36)) in the epilogue.
// The paper's 1-3 kernels per stage plus RK update become one kernel; face
// fluxes, traces and flux-point values never touch HBM.
#include <cstdio>

#include "common.cuh"
#include "ops_tables.h"

namespace h2d {

enum { M_FV = 0, M_CPR = 1, M_DG = 2, M_NDG = 3, M_SD = 4 };

// element tile per CTA (TX x TY elements, one thread per solution point)
template <int K> struct Tile;
template <> struct Tile<1> { static constexpr int TX = 16, TY = 4; };  // 256 threads
template <> struct Tile<2> { static constexpr int TX = 8, TY = 4; };   // 288
template <> struct Tile<3> { static constexpr int TX = 8, TY = 2; };   // 256
template <> struct Tile<4> { static constexpr int TX = 4, TY = 3; };   // 300

template <int M, int K>
struct HO {
  static constexpr int N = K + 1, NP = N * N;
  static constexpr int TX = Tile<K>::TX, TY = Tile<K>::TY;
  static constexpr int NE = TX * TY, NT = NE * NP;
  static constexpr int SX = TX + 2, SY = TY + 2;
  static constexpr bool GLL = (M == M_CPR || M == M_NDG);
  // shared-memory carve-up (doubles)
  static constexpr int OPS = 0;                                   // operator tables
  static constexpr int OPS_SZ = 96;
  static constexpr int RED = OPS + OPS_SZ;                        // reduction scratch
  static constexpr int RED_SZ = 32;
  static constexpr int QS = RED + RED_SZ;                         // state tile + halo
  static constexpr int QS_SZ = 4 * SY * SX * NP;
  static constexpr int JS = QS + QS_SZ;                           // face arrays [4 sides][NE][N][4]
  static constexpr int JS_SZ = (M == M_SD) ? 0 : 4 * NE * N * 4;
  static constexpr int FS = JS + JS_SZ;                           // point fluxes f,g [2][4][NE][NP]
  static constexpr int FS_SZ = (M == M_NDG || M == M_DG) ? 2 * 4 * NE * NP : 0;
  static constexpr int PS = FS + FS_SZ;                           // SD flux-point fluxes [2][NE][N][N+1][4]
  static constexpr int PS_SZ = (M == M_SD) ? 2 * NE * N * (N + 1) * 4 : 0;
  static constexpr int TOTAL = PS + PS_SZ;
  static constexpr size_t SMEM = TOTAL * sizeof(double);
};

// operator tables, filled on the host from the generated constexpr Ops<K> and
// passed by value as a kernel parameter (constant bank), then copied to smem
enum { O_D = 0, O_I = 32, O_V1 = 64, O_V2 = 72, O_EL = 80, O_ER = 88, O_N = 96 };
struct OpTab {
  double v[O_N];
};

template <int M, int K>
static OpTab make_tab() {
  using O = Ops<K>;
  constexpr int N = K + 1;
  OpTab t{};
  for (int a = 0; a < N; ++a) {
    for (int l = 0; l < N; ++l) {
      if (M == M_CPR || M == M_NDG) t.v[O_D + a * N + l] = O::D_gll[a][l];
      if (M == M_DG) t.v[O_D + a * N + l] = O::dg_vol[a][l];
    }
    if (M == M_CPR || M == M_NDG) { t.v[O_V1 + a] = O::gLp_gll[a]; t.v[O_V2 + a] = O::gRp_gll[a]; }
    if (M == M_DG) {
      t.v[O_V1 + a] = O::dg_sL[a]; t.v[O_V2 + a] = O::dg_sR[a];
      t.v[O_EL + a] = O::eL_gl[a]; t.v[O_ER + a] = O::eR_gl[a];
    }
    if (M == M_SD)
      for (int r = 0; r <= N; ++r) { t.v[O_D + a * (N + 1) + r] = O::sd_D[a][r]; t.v[O_I + r * N + a] = O::sd_I[r][a]; }
  }
  return t;
}

template <int M, int K>
__global__ void __launch_bounds__(HO<M, K>::NT) ho_stage_kernel(const StageArgs a, const OpTab tab) {
  using H = HO<M, K>;
  constexpr int N = H::N, NP = H::NP, TX = H::TX, TY = H::TY, SX = H::SX, SY = H::SY, NT = H::NT, NE = H::NE;
  extern __shared__ double smem[];
  double* so = smem + H::OPS;
  double* sred = smem + H::RED;
  double* sq = smem + H::QS;
  double* sj = smem + H::JS;   // [side W,E,S,N][el][line][c]
  double* sf = smem + H::FS;   // [dir][c][el][p]
  double* sp = smem + H::PS;   // [dir][el][line][r][c]

  double dtv = 1.0;
  if (a.dt) {
    dtv = *a.dt;
    if (dtv == 0.0) return;  // clipped-out step (t == t_end): uniform across the grid
  }
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int TXv = min(TX, a.nx - i0), TYv = min(TY, a.nrows - j0);
  const double gam = a.gamma, gm1 = a.gamma - 1.0;

  for (int i = tid; i < O_N; i += NT) so[i] = tab.v[i];

  // ---- 1. state tile + halo -> smem (GLL: only the halo edge nodes) ----------
  auto SQ = [&](int c, int sy, int sx, int p) -> double& { return sq[((c * SY + sy) * SX + sx) * NP + p]; };
  for (int t = tid; t < 4 * SY * SX * NP; t += NT) {
    const int p = t % NP;
    int r = t / NP;
    const int sx = r % SX;
    r /= SX;
    const int sy = r % SY;
    const int c = r / SY;
    if (sx > TXv + 1 || sy > TYv + 1) continue;
    const bool hx = (sx == 0 || sx == TXv + 1), hy = (sy == 0 || sy == TYv + 1);
    if (hx && hy) continue;
    if (H::GLL && (hx || hy)) {
      const int pa = p % N, pb = p / N;
      if ((sx == 0 && pa != N - 1) || (sx == TXv + 1 && pa != 0) || (sy == 0 && pb != N - 1) ||
          (sy == TYv + 1 && pb != 0))
        continue;
    }
    int i = i0 - 1 + sx, j = j0 - 1 + sy;
    if (i < 0) { if (a.bcx) continue; i += a.nx; }
    else if (i >= a.nx) { if (a.bcx) continue; i -= a.nx; }
    const double* base;
    long long cs;
    if (j < 0) { if (!a.ghost_lo) continue; base = a.ghost_lo; cs = a.gcs; j = 0; }
    else if (j >= a.nrows) { if (!a.ghost_hi) continue; base = a.ghost_hi; cs = a.gcs; j -= a.nrows; }
    else { base = a.q; cs = a.cs; }
    SQ(c, sy, sx, p) = __ldg(base + c * cs + ((long long)j * a.nx + i) * NP + p);
  }
  __syncthreads();

  // traces of the element in slot (sy,sx) on line t: GLL edge node or GL interpolation
  auto trace = [&](int side, int sy, int sx, int t, double q[4]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (H::GLL) {
        const int p = side == 0 ? t * N : side == 1 ? t * N + N - 1 : side == 2 ? t : (N - 1) * N + t;
        q[c] = SQ(c, sy, sx, p);
      } else if (M == M_DG) {
        const double* e = (side == 0 || side == 2) ? so + O_EL : so + O_ER;
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) s += e[l] * SQ(c, sy, sx, side <= 1 ? t * N + l : l * N + t);
        q[c] = s;
      } else {  // SD: flux point 0 / N of the line (== GL edge interpolation)
        const double* I = so + O_I + ((side == 0 || side == 2) ? 0 : N * N);
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) s += I[l] * SQ(c, sy, sx, side <= 1 ? t * N + l : l * N + t);
        q[c] = s;
      }
    }
  };
  auto SJ = [&](int side, int el, int t, int c) -> double& { return sj[((side * NE + el) * N + t) * 4 + c]; };
  auto SP = [&](int dir, int el, int t, int r, int c) -> double& {
    return sp[(((dir * NE + el) * N + t) * (N + 1) + r) * 4 + c];
  };

  // ---- 2. point fluxes (NDG: D[F]; DG: volume integral) -----------------------
  if (M == M_NDG || M == M_DG) {
    if (tid < NT) {
      const int el = tid / NP, p = tid % NP, lx = el % TX, ly = el / TX;
      if (lx < TXv && ly < TYv) {
        double q[4], f[4], g[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) q[c] = SQ(c, ly + 1, lx + 1, p);
        Prim w = prims(q, gm1);
        flux<0>(q, w, f);
        flux<1>(q, w, g);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          sf[((0 * 4 + c) * NE + el) * NP + p] = f[c];
          sf[((1 * 4 + c) * NE + el) * NP + p] = g[c];
        }
      }
    }
  }
  // ---- 2b. SD interior flux points: interpolate the solution line, evaluate F --
  if (M == M_SD) {
    for (int t = tid; t < NE * N * (N - 1) * 2; t += NT) {
      const int r = 1 + t % (N - 1);
      int u = t / (N - 1);
      const int ln = u % N;
      u /= N;
      const int dir = u & 1, el = u >> 1;
      const int lx = el % TX, ly = el / TX;
      if (lx >= TXv || ly >= TYv) continue;
      double q[4], f[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) s += so[O_I + r * N + l] * SQ(c, ly + 1, lx + 1, dir == 0 ? ln * N + l : l * N + ln);
        q[c] = s;
      }
      Prim w = prims(q, gm1);
      if (dir == 0) flux<0>(q, w, f); else flux<1>(q, w, f);
#pragma unroll
      for (int c = 0; c < 4; ++c) SP(dir, el, ln, r, c) = f[c];
    }
  }

  // ---- 3. common interface fluxes (Rusanov), each tile face point once -------
  for (int t = tid; t < TY * (TX + 1) * N; t += NT) {   // x-faces
    const int ln = t % N;
    const int r = t / N;
    const int fx = r % (TX + 1), ly = r / (TX + 1);
    if (ly >= TYv || fx > TXv) continue;
    const bool mirL = (fx == 0 && i0 == 0 && a.bcx), mirR = (fx == TXv && i0 + TXv == a.nx && a.bcx);
    double qL[4], qR[4], F[4], fL[4], fR[4];
    if (!mirL) trace(1, ly + 1, fx, ln, qL);
    if (!mirR) trace(0, ly + 1, fx + 1, ln, qR);
#pragma unroll
    for (int c = 0; c < 4; ++c) { if (mirL) qL[c] = qR[c]; if (mirR) qR[c] = qL[c]; }
    rusanov<0>(qL, qR, gm1, gam, F, fL, fR);
    const int elL = ly * TX + fx - 1, elR = ly * TX + fx;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (H::GLL) {  // store F^ - f(own trace) (CPR correction / NDG lift input)
        if (fx > 0) SJ(1, elL, ln, c) = F[c] - fL[c];
        if (fx < TXv) SJ(0, elR, ln, c) = F[c] - fR[c];
      } else if (M == M_DG) {
        if (fx > 0) SJ(1, elL, ln, c) = F[c];
        if (fx < TXv) SJ(0, elR, ln, c) = F[c];
      } else {
        if (fx > 0) SP(0, elL, ln, N, c) = F[c];
        if (fx < TXv) SP(0, elR, ln, 0, c) = F[c];
      }
    }
  }
  for (int t = tid; t < (TY + 1) * TX * N; t += NT) {   // y-faces
    const int ln = t % N;
    const int r = t / N;
    const int lx = r % TX, fy = r / TX;
    if (lx >= TXv || fy > TYv) continue;
    const bool mirS = (fy == 0 && j0 == 0 && !a.ghost_lo), mirN = (fy == TYv && j0 + TYv == a.nrows && !a.ghost_hi);
    double qL[4], qR[4], F[4], fL[4], fR[4];
    if (!mirS) trace(3, fy, lx + 1, ln, qL);
    if (!mirN) trace(2, fy + 1, lx + 1, ln, qR);
#pragma unroll
    for (int c = 0; c < 4; ++c) { if (mirS) qL[c] = qR[c]; if (mirN) qR[c] = qL[c]; }
    rusanov<1>(qL, qR, gm1, gam, F, fL, fR);
    const int elL = (fy - 1) * TX + lx, elR = fy * TX + lx;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (H::GLL) {
        if (fy > 0) SJ(3, elL, ln, c) = F[c] - fL[c];
        if (fy < TYv) SJ(2, elR, ln, c) = F[c] - fR[c];
      } else if (M == M_DG) {
        if (fy > 0) SJ(3, elL, ln, c) = F[c];
        if (fy < TYv) SJ(2, elR, ln, c) = F[c];
      } else {
        if (fy > 0) SP(1, elL, ln, N, c) = F[c];
        if (fy < TYv) SP(1, elR, ln, 0, c) = F[c];
      }
    }
  }
  __syncthreads();

  // ---- 4. residual at every solution point + RK combination -------------------
  double lam = 0.0;
  if (tid < NT) {
    const int el = tid / NP, p = tid % NP, lx = el % TX, ly = el / TX;
    const int ai = p % N, bi = p / N;
    if (lx < TXv && ly < TYv) {
      double q[4], R[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) q[c] = SQ(c, ly + 1, lx + 1, p);
      if (M == M_CPR || M == M_NDG) {
        double Fx[4], Gy[4];
        if (M == M_CPR) {  // chain rule: A(q) dq/dxi + B(q) dq/deta
          double dqx[4], dqy[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double sx = 0.0, sy = 0.0;
#pragma unroll
            for (int l = 0; l < N; ++l) {
              sx += so[O_D + ai * N + l] * SQ(c, ly + 1, lx + 1, bi * N + l);
              sy += so[O_D + bi * N + l] * SQ(c, ly + 1, lx + 1, l * N + ai);
            }
            dqx[c] = sx;
            dqy[c] = sy;
          }
          Prim w = prims(q, gm1);
          jac<0>(q, w, gm1, gam, dqx, Fx);
          jac<1>(q, w, gm1, gam, dqy, Gy);
        } else {           // NDG: D[F]
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double sx = 0.0, sy = 0.0;
#pragma unroll
            for (int l = 0; l < N; ++l) {
              sx += so[O_D + ai * N + l] * sf[((0 * 4 + c) * NE + el) * NP + bi * N + l];
              sy += so[O_D + bi * N + l] * sf[((1 * 4 + c) * NE + el) * NP + l * N + ai];
            }
            Fx[c] = sx;
            Gy[c] = sy;
          }
        }
        const double gLa = so[O_V1 + ai], gRa = so[O_V2 + ai], gLb = so[O_V1 + bi], gRb = so[O_V2 + bi];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          Fx[c] += gLa * SJ(0, el, bi, c) + gRa * SJ(1, el, bi, c);
          Gy[c] += gLb * SJ(2, el, ai, c) + gRb * SJ(3, el, ai, c);
          R[c] = -a.rdx2 * Fx[c] - a.rdy2 * Gy[c];
        }
      } else if (M == M_DG) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double vx = 0.0, vy = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) {
            vx += so[O_D + ai * N + l] * sf[((0 * 4 + c) * NE + el) * NP + bi * N + l];
            vy += so[O_D + bi * N + l] * sf[((1 * 4 + c) * NE + el) * NP + l * N + ai];
          }
          vx += so[O_V1 + ai] * SJ(0, el, bi, c) - so[O_V2 + ai] * SJ(1, el, bi, c);
          vy += so[O_V1 + bi] * SJ(2, el, ai, c) - so[O_V2 + bi] * SJ(3, el, ai, c);
          R[c] = a.rdx2 * vx + a.rdy2 * vy;
        }
      } else {  // SD: differentiate the flux polynomial through the flux points
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double fx = 0.0, gy = 0.0;
#pragma unroll
          for (int r = 0; r <= N; ++r) {
            fx += so[O_D + ai * (N + 1) + r] * SP(0, el, bi, r, c);
            gy += so[O_D + bi * (N + 1) + r] * SP(1, el, ai, r, c);
          }
          R[c] = -a.rdx2 * fx - a.rdy2 * gy;
        }
      }
      // RK combination  out = a0 q0 + a1 q + bcoef dt R
      const long long gidx = ((long long)(j0 + ly) * a.nx + (i0 + lx)) * NP + p;
      double o[4];
      const double bdt = a.bcoef * dtv;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double v = a.a1 * q[c] + bdt * R[c];
        if (a.q0) v += a.a0 * a.q0[c * a.cs + gidx];
        o[c] = v;
        a.out[c * a.cs + gidx] = v;
      }
      if (a.lam) lam = wave_speed(o, gm1, gam);
      if (a.bad && nonphysical(o, gm1)) atomicMin(a.bad, (unsigned long long)gidx);
    }
  }
  if (a.lam) block_max_to(lam, a.lam, sred);
}

template <int M, int K>
static int launch_t(const StageArgs& a, cudaStream_t s) {
  using H = HO<M, K>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ho_stage_kernel<M, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H::SMEM);
    attr = true;
  }
  dim3 grid((a.nx + H::TX - 1) / H::TX, (a.nrows + H::TY - 1) / H::TY);
  static const OpTab tab = make_tab<M, K>();
  ho_stage_kernel<M, K><<<grid, H::NT, H::SMEM, s>>>(a, tab);
  return (int)cudaPeekAtLastError();
}

template <int M>
static int launch_m(int k, const StageArgs& a, cudaStream_t s) {
  switch (k) {
    case 1: return launch_t<M, 1>(a, s);
    case 2: return launch_t<M, 2>(a, s);
    case 3: return launch_t<M, 3>(a, s);
    case 4: return launch_t<M, 4>(a, s);
  }
  return (int)cudaErrorInvalidValue;
}

int launch_ho_stage(int method, int k, const StageArgs& a, cudaStream_t s) {
  switch (method) {
    case M_DG: return launch_m<M_DG>(k, a, s);
    case M_SD: return launch_m<M_SD>(k, a, s);
  }
  return (int)cudaErrorInvalidValue;
}

}  // namespace h2d
