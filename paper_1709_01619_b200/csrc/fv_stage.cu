// fv_stage.cu -- fused RK-stage kernel of the MUSCL finite-volume method
// (Eqs. (6)-(8); MUSCL + minmod; Alg. 1).
// The paper's two kernels (FV_Reconstruct writing face fluxes to global memory,
// then the flux-derivative kernel) become one: a TX x TY cell tile
// plus a 2-cell halo is staged in shared memory, every tile face is
// reconstructed and Rusanov-coupled once, the flux differences and the SSP-RK3
// combination are applied in registers, and only the new state is written.
#include "common.cuh"

namespace h2d {

namespace {
constexpr int FTX = 32, FTY = 8, FNT = FTX * FTY;
constexpr int FSX = FTX + 4, FSY = FTY + 4;

// face states from the stencil (i-1, i, i+1, i+2) for the face i+1/2
template <int ORDER>
__device__ __forceinline__ void muscl(double qm1, double q0, double q1, double q2, double& qW, double& qE,
                                      long long* dec) {
  if (ORDER == 1) {
    const double s0 = minmod2(q0 - qm1, q1 - q0, dec);
    const double s1 = minmod2(q1 - q0, q2 - q1, dec);
    qW = q0 + 0.5 * s0;
    qE = q1 - 0.5 * s1;
  } else {  // kappa = 1/3, beta = (3 - kappa)/(1 - kappa) = 4
    constexpr double kap = 1.0 / 3.0, beta = (3.0 - kap) / (1.0 - kap);
    const double dm0 = q0 - qm1, dp0 = q1 - q0, dm1 = q1 - q0, dp1 = q2 - q1;
    qW = q0 + 0.25 * ((1.0 - kap) * minmod2(dm0, beta * dp0, dec) + (1.0 + kap) * minmod2(dp0, beta * dm0, dec));
    qE = q1 - 0.25 * ((1.0 - kap) * minmod2(dp1, beta * dm1, dec) + (1.0 + kap) * minmod2(dm1, beta * dp1, dec));
  }
}
}  // namespace

template <int ORDER>
__global__ void __launch_bounds__(FNT) fv_stage_kernel(const StageArgs a) {
  __shared__ double sq[4][FSY][FSX];
  __shared__ double sF[FTY][FTX + 1][4];
  __shared__ double sG[FTY + 1][FTX][4];
  __shared__ double sred[32];
  double dtv = 1.0;
  if (a.dt) {
    dtv = *a.dt;
    if (dtv == 0.0) return;
  }
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * FTX, j0 = blockIdx.y * FTY;
  const int TXv = min(FTX, a.nx - i0), TYv = min(FTY, a.nrows - j0);
  const double gam = a.gamma, gm1 = a.gamma - 1.0;

  // cells (j0-2 .. j0+TYv+1) x (i0-2 .. i0+TXv+1), corners excluded
  for (int t = tid; t < 4 * FSY * FSX; t += FNT) {
    const int sx = t % FSX, sy = (t / FSX) % FSY, c = t / (FSX * FSY);
    if (sx >= TXv + 4 || sy >= TYv + 4) continue;
    const bool hx = (sx < 2 || sx >= TXv + 2), hy = (sy < 2 || sy >= TYv + 2);
    if (hx && hy) continue;
    int i = i0 - 2 + sx, j = j0 - 2 + sy;
    if (a.bcx == 0) i = (i % a.nx + a.nx) % a.nx;
    else i = i < 0 ? 0 : (i >= a.nx ? a.nx - 1 : i);  // ghost cells copy the boundary cell
    const double* base = a.q;
    long long cs = a.cs;
    if (j < 0) {
      if (a.ghost_lo) { base = a.ghost_lo; cs = a.gcs; j += 2; } else j = 0;
    } else if (j >= a.nrows) {
      if (a.ghost_hi) { base = a.ghost_hi; cs = a.gcs; j -= a.nrows; } else j = a.nrows - 1;
    }
    sq[c][sy][sx] = __ldg(base + c * cs + (long long)j * a.nx + i);
  }
  __syncthreads();

  for (int t = tid; t < FTY * (FTX + 1); t += FNT) {  // x-faces: between cells fx-1 and fx
    const int fx = t % (FTX + 1), ly = t / (FTX + 1);
    if (ly >= TYv || fx > TXv) continue;
    double qW[4], qE[4], F[4], fL[4], fR[4];
    // tile-edge faces are computed by both neighbouring tiles; count each face once
    long long* dec = (fx < TXv || i0 + TXv == a.nx) ? a.dec : nullptr;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      muscl<ORDER>(sq[c][ly + 2][fx], sq[c][ly + 2][fx + 1], sq[c][ly + 2][fx + 2], sq[c][ly + 2][fx + 3], qW[c],
                   qE[c], dec);
    rusanov<0>(qW, qE, gm1, gam, F, fL, fR);
#pragma unroll
    for (int c = 0; c < 4; ++c) sF[ly][fx][c] = F[c];
  }
  for (int t = tid; t < (FTY + 1) * FTX; t += FNT) {  // y-faces
    const int lx = t % FTX, fy = t / FTX;
    if (lx >= TXv || fy > TYv) continue;
    double qW[4], qE[4], F[4], fL[4], fR[4];
    long long* dec = (fy < TYv || (j0 + TYv == a.nrows && a.count_top)) ? a.dec : nullptr;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      muscl<ORDER>(sq[c][fy][lx + 2], sq[c][fy + 1][lx + 2], sq[c][fy + 2][lx + 2], sq[c][fy + 3][lx + 2], qW[c],
                   qE[c], dec);
    rusanov<1>(qW, qE, gm1, gam, F, fL, fR);
#pragma unroll
    for (int c = 0; c < 4; ++c) sG[fy][lx][c] = F[c];
  }
  __syncthreads();

  double lam = 0.0;
  const int lx = tid % FTX, ly = tid / FTX;
  if (lx < TXv && ly < TYv) {
    const long long gidx = (long long)(j0 + ly) * a.nx + (i0 + lx);
    const double bdt = a.bcoef * dtv;
    double o[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double R = -(sF[ly][lx + 1][c] - sF[ly][lx][c]) * a.rdx2 - (sG[ly + 1][lx][c] - sG[ly][lx][c]) * a.rdy2;
      double v = a.a1 * sq[c][ly + 2][lx + 2] + bdt * R;
      if (a.q0) v += a.a0 * a.q0[c * a.cs + gidx];
      o[c] = v;
      a.out[c * a.cs + gidx] = v;
    }
    if (a.lam) lam = wave_speed(o, gm1, gam);
    if (a.bad && nonphysical(o, gm1)) atomicMin(a.bad, (unsigned long long)gidx);
  }
  if (a.lam) block_max_to(lam, a.lam, sred);
}

int launch_fv_stage(int k, const StageArgs& a, cudaStream_t s) {
  dim3 grid((a.nx + FTX - 1) / FTX, (a.nrows + FTY - 1) / FTY);
  if (k == 1) fv_stage_kernel<1><<<grid, FNT, 0, s>>>(a);
  else fv_stage_kernel<2><<<grid, FNT, 0, s>>>(a);
  return (int)cudaPeekAtLastError();
}

}  // namespace h2d
