// fv_stage.cu -- fused RK-stage kernel of the MUSCL finite-volume method
// (Eqs. (6)-(8); MUSCL + minmod; Alg. 1).
//
// The paper's two kernels (FV_Reconstruct writing face fluxes to global memory,
// then the flux-derivative kernel) become one marching kernel:
//  * a CTA owns a strip of TX cells (one thread per cell column) and marches up
//    RB cell rows;
//  * a 5-row ring in shared memory holds rows j-1..j+2 (the MUSCL stencil of
//    the x faces of row j and of its N face); row j+3 is prefetched into
//    registers one step ahead (coalesced loads), so HBM latency hides behind a
//    step's arithmetic and each value is read from HBM once;
//  * x faces: one reconstruction + Rusanov per face (each thread its W face, the
//    strip's last thread also the E face), exchanged through shared memory;
//    y faces: each thread computes the N face of its column and carries it in
//    registers as the S face of the next row -- no face array ever reaches HBM;
//  * flux differences, the SSP-RK combination, the dt wave speed and the
//    non-physical check are fused; one coalesced store per component.
#include "common.cuh"
#include "tma.cuh"

namespace h2d {

namespace {
#ifndef H2D_FTX
#define H2D_FTX 128  // A/B: 64 at 8 CTAs/SM -5 %; 256 exceeds the static smem limit
#endif
#ifndef H2D_FV_DEPTH
#define H2D_FV_DEPTH 2  // ring rows in flight (cp.async); 3 is +1 % at 4 CTAs/SM but its 46 KB keep 5 out
#endif
constexpr int FTX = H2D_FTX, FRB = 64, FD = H2D_FV_DEPTH, FNS = 3 + FD;  // cells/strip, rows/march, in flight, ring rows
constexpr int FW = FTX + 4;                    // ring row width: 2 halo cells each side

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
      const double ma = fabs(dm) <= fabs(bdp) ? dm : bdp, mb = fabs(dp) <= fabs(bdm) ? dp : bdm;
      A = same ? ma : 0.0;
      B = same ? mb : 0.0;
    }
    // q0 +- ((1 - kappa) X + (1 + kappa) Y) / 4 with the quarter folded into the weights
    constexpr double c1 = 0.25 * (1.0 - kap), c2 = 0.25 * (1.0 + kap);
    hi = __fma_rn(c1, A, __fma_rn(c2, B, q0));
    lo = __fma_rn(-c1, B, __fma_rn(-c2, A, q0));
  }
}

// TWICE the Rusanov flux along DIR: fL + fR - lam (qR - qL).  The
// factor 1/2 moves into the metric of the flux difference (0.5 / dx): scaling
// by powers of two is exact, so nothing changes but 5 multiplications per face.
template <int DIR>
__device__ __forceinline__ void rusanov2(const double qL[4], const double qR[4], double gm1, double gam, double F2[4]) {
  const Prim wl = prims(qL, gm1), wr = prims(qR, gm1);
  double fL[4], fR[4];
  flux<DIR>(qL, wl, fL);
  flux<DIR>(qR, wr, fR);
  const double sl = fabs(DIR == 0 ? wl.u : wl.v) + fsqrt(gam * wl.p * wl.ri);
  const double sr = fabs(DIR == 0 ? wr.u : wr.v) + fsqrt(gam * wr.p * wr.ri);
  const double lam = fmax(sl, sr);
#pragma unroll
  for (int c = 0; c < 4; ++c) F2[c] = fma(-lam, qR[c] - qL[c], fL[c] + fR[c]);
}
}  // namespace

#ifndef H2D_FV_ASYNC
#define H2D_FV_ASYNC 1  // ring rows by cp.async, two rows in flight (0: register-staged, one row)
#endif
#ifndef H2D_FV_MINB
#define H2D_FV_MINB 5  // 96 registers, no spills, 5 x 42 KB smem (A/B: +1.5 % over 4 at depth 3; 4 was +12 % over 3)
#endif
// V (stage variant, compile time): bit 0 q^n read, bit 1 dt / non-physical epilogue
template <int ORDER, bool REC, int V>
__global__ void __launch_bounds__(FTX, H2D_FV_MINB) fv_stage_kernel(const StageArgs a) {
  // V == 8: any other combination, decided at run time from the pointers
  const bool HQ0 = V == 8 ? a.q0 != nullptr : (V & 1), HLAM = V == 8 ? (a.lam || a.bad) : (V & 2) != 0;
  __shared__ double ring[FNS][4][FW];
  __shared__ double sF[FTX + 1][4];   // W-face fluxes of the row (+ the strip's last E face)
  __shared__ double sXL[2][4][FTX + 2], sXH[2][4][FTX + 2];  // x face states lo/hi per cell, 2 rows
  __shared__ double sred[32];
  pdl_wait();
  pdl_launch();
  double dtv = 1.0;
  if (a.dt) {
    dtv = *a.dt;
    if (dtv == 0.0) return;
  }
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * FTX, jb = a.row_lo + blockIdx.y * a.rows;
  const int TXv = min(FTX, a.nx - i0), RBv = min(a.rows, a.row_hi - jb);
  const double gam = a.gamma, gm1 = a.gamma - 1.0;
  const bool own = tid < TXv;

  long long* const dec = REC ? a.dec : nullptr;  // decision counters (parity runs only)
  // this thread's halo column (threads 0..3: slots 0, 1 = cells i0-2, i0-1 and
  // TXv+2, TXv+3 = cells i0+TXv, +1): x periodic wrap or transmissive clamp, once
  int hx = tid < 2 ? i0 - 2 + tid : i0 + TXv + (tid - 2);
  if (a.bcx == 0) hx = hx < 0 ? hx + a.nx : (hx >= a.nx ? hx - a.nx : hx);
  else hx = hx < 0 ? 0 : (hx >= a.nx ? a.nx - 1 : hx);
  // start of cell row jr (y: ghost rows, or clamp at a transmissive boundary)
  auto row_ptr = [&](int jr, long long& cs) -> const double* {
    cs = a.cs;
    if (jr < 0) {
      if (a.ghost_lo) { cs = a.gcs; return a.ghost_lo + (long long)(jr + 2) * a.nx; }
      jr = 0;
    } else if (jr >= a.nrows) {
      if (a.ghost_hi) { cs = a.gcs; return a.ghost_hi + (long long)(jr - a.nrows) * a.nx; }
      jr = a.nrows - 1;
    }
    return a.q + (long long)jr * a.nx;
  };
  auto slot_of = [&](int r) { return ((r % FNS) + FNS) % FNS; };  // r = row - jb
  // decision-map entry of cell (jr, ir) (REC runs, one rank): a ghost cell's
  // reconstruction is attributed to the cell it copies (periodic wrap /
  // transmissive clamp), as the oracle's fv_idx does
  auto dmap_at = [&](int jr, int ir) -> long long* {
    if (!REC || !a.dmap) return nullptr;
    if (ir < 0) ir = a.bcx == 0 ? ir + a.nx : 0;
    if (ir >= a.nx) ir = a.bcx == 0 ? ir - a.nx : a.nx - 1;
    if (jr < 0) jr = a.ghost_lo ? jr + a.nrows : 0;
    if (jr >= a.nrows) jr = a.ghost_hi ? jr - a.nrows : a.nrows - 1;
    return a.dmap + (long long)jr * a.nx + ir;
  };
#if H2D_FV_ASYNC
  // this thread's ring column(s) of row jr (own cell: slot tid + 2; threads 0..3
  // also a halo slot) copied by cp.async straight into ring slot `slot`: no
  // register staging, so FD rows stay in flight (the ring's FNS = 3 + FD slots
  // hold rows r .. r+2+FD; rows r-2, r-1 are dead once row r starts)
  auto issue_row = [&](int jr, int slot) {
    long long cs;
    const double* rb = row_ptr(jr, cs);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (own)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&ring[slot][c][tid + 2])),
                     "l"(rb + c * cs + i0 + tid)
                     : "memory");
      if (tid < 4)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&ring[slot][c][tid < 2 ? tid : TXv + tid])),
                     "l"(rb + c * cs + hx)
                     : "memory");
    }
  };
  auto commit = [] { asm volatile("cp.async.commit_group;" ::: "memory"); };
  // prologue: rows jb-2 .. jb+1 (group 0), jb+2 (group 1); rows jb+3, jb+4 go
  // into the slots of rows jb-2, jb-1 once the prologue below has read them
  for (int r = -2; r <= 1; ++r) issue_row(jb + r, slot_of(r));
  commit();
  issue_row(jb + 2, slot_of(2));
  commit();
  asm volatile("cp.async.wait_group 1;" ::: "memory");
  __syncthreads();
#else
  // this thread's ring column(s): own cell (slot tid + 2), threads 0..3 also a halo slot
  auto load_row = [&](int jr, double v[4], double h[4]) {
    long long cs;
    const double* rb = row_ptr(jr, cs);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      v[c] = own ? __ldg(rb + c * cs + i0 + tid) : 0.0;
      h[c] = tid < 4 ? __ldg(rb + c * cs + hx) : 0.0;
    }
  };
  auto store_row = [&](int slot, const double v[4], const double h[4]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (own) ring[slot][c][tid + 2] = v[c];
      if (tid < 4) ring[slot][c][tid < 2 ? tid : TXv + tid] = h[c];
    }
  };

  // prologue: rows jb-2 .. jb+1 into the ring, jb+2 into registers
  double pv[4], ph[4];
  for (int r = -2; r <= 1; ++r) {
    load_row(jb + r, pv, ph);
    store_row((r + FNS) % FNS, pv, ph);
  }
  load_row(jb + 2, pv, ph);
  __syncthreads();
#endif

  // y reconstruction once per cell: the hi (N-side) state of the row below the
  // current one is carried in registers.  Decision weights: an own row stands
  // for its S and N face evaluations (2); the ghost row below the domain's first
  // row (bottom face, counted once: count_bot) and the one above the strip's
  // last row when that is the domain's top (1); rows of a neighbouring CTA are
  // counted by their owner (0).
  double GS[4], yHi[4];
  {
    double lo[4], hi[4], dm;
    const int wb = (jb == 0 && a.count_bot) ? 1 : 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double r0 = own ? ring[slot_of(-2)][c][tid + 2] : 1.0, r1 = own ? ring[slot_of(-1)][c][tid + 2] : 1.0;
      const double r2 = own ? ring[slot_of(0)][c][tid + 2] : 1.0, r3 = own ? ring[slot_of(1)][c][tid + 2] : 1.0;
      cell_faces<ORDER>(r0, r1, r2, dm, hi[c], own ? dec : nullptr, wb, own ? dmap_at(jb - 1, i0 + tid) : nullptr);
      cell_faces<ORDER>(r1, r2, r3, lo[c], yHi[c], own ? dec : nullptr, 2, own ? dmap_at(jb, i0 + tid) : nullptr);
    }
    if (own) rusanov2<1>(hi, lo, gm1, gam, GS);
  }

  // x reconstruction once per cell, one row ahead, into buffer buf: slot s holds
  // cell i0-1+s (own cells 1..TXv; slot 0 / TXv+1 the strip's halo cells, whose
  // hi / lo state the strip's end faces need).  Decision weights as for y: own
  // cells 2, the domain's end cells' ghosts 1, a neighbouring strip's cells 0.
  auto recon_x = [&](int rs, int buf, int jr) {
    double dm;
    if (own) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        cell_faces<ORDER>(ring[rs][c][tid + 1], ring[rs][c][tid + 2], ring[rs][c][tid + 3], sXL[buf][c][tid + 1],
                          sXH[buf][c][tid + 1], dec, 2, dmap_at(jr, i0 + tid));
    }
    if (tid == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        cell_faces<ORDER>(ring[rs][c][0], ring[rs][c][1], ring[rs][c][2], dm, sXH[buf][c][0], dec, i0 == 0 ? 1 : 0,
                          dmap_at(jr, i0 - 1));
    }
    if (tid == TXv - 1) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        cell_faces<ORDER>(ring[rs][c][TXv + 1], ring[rs][c][TXv + 2], ring[rs][c][TXv + 3], sXL[buf][c][TXv + 1], dm,
                          dec, (i0 + TXv == a.nx) ? 1 : 0, dmap_at(jr, i0 + TXv));
    }
  };
  recon_x(slot_of(0), 0, jb);  // read after the first loop barrier

  double lam = 0.0;
  const double bdt = a.bcoef * dtv;
  const double hrdx = 0.5 * a.rdx2, hrdy = 0.5 * a.rdy2;
  for (int r = 0; r < RBv; ++r) {
#if H2D_FV_ASYNC
    // row r+2 has landed (this thread's copies; the barrier publishes everyone's);
    // after the barrier row r-1's slot is dead: row r+4 goes there (at r = 0
    // also row 3, into row -2's slot)
    if (r == 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
    else asm volatile("cp.async.wait_group %0;" ::"n"(FD - 1) : "memory");
    __syncthreads();
    if (r == 0) {
#pragma unroll
      for (int k = 3; k < 2 + FD; ++k) {
        if (k <= RBv + 1) issue_row(jb + k, slot_of(k));
        commit();
      }
    }
    if (r + 2 + FD <= RBv + 1) issue_row(jb + r + 2 + FD, slot_of(r + 2 + FD));
    commit();
#else
    // the prefetched row r+2 enters the ring; prefetch row r+3
    store_row(slot_of(r + 2), pv, ph);
    if (r + 3 <= RBv + 1) load_row(jb + r + 3, pv, ph);
    __syncthreads();
#endif
    const int sc = slot_of(r);
    const long long gidx = (long long)(jb + r) * a.nx + (i0 + tid);
    double q0v[4] = {0, 0, 0, 0};
    if (HQ0 && own) {
#pragma unroll
      for (int c = 0; c < 4; ++c) q0v[c] = a.q0[c * a.cs + gidx];
    }
    // x faces (the W face of each own cell, from the face states reconstructed one
    // row earlier) and the N face of the column (carried hi state of row r, lo
    // state of row r+1 reconstructed now from rows r..r+2; its hi state is
    // carried on): straight-line, so that both Rusanov evaluations interleave
    double GN[4];
    if (own) {
      const int b = r & 1;
      const int wn = (r + 1 < RBv) ? 2 : ((jb + RBv == a.nrows) ? 1 : 0);
      double qL[4], qR[4], lo[4], hi[4], F[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        qL[c] = sXH[b][c][tid];
        qR[c] = sXL[b][c][tid + 1];
        cell_faces<ORDER>(ring[sc][c][tid + 2], ring[slot_of(r + 1)][c][tid + 2], ring[slot_of(r + 2)][c][tid + 2],
                          lo[c], hi[c], dec, wn, dmap_at(jb + r + 1, i0 + tid));
      }
      rusanov2<0>(qL, qR, gm1, gam, F);
      rusanov2<1>(yHi, lo, gm1, gam, GN);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        sF[tid][c] = F[c];
        yHi[c] = hi[c];
      }
    }
    if (own && tid == TXv - 1) {  // the strip's last E face
      const int b = r & 1;
      double qL[4], qR[4], F[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        qL[c] = sXH[b][c][tid + 1];
        qR[c] = sXL[b][c][tid + 2];
      }
      rusanov2<0>(qL, qR, gm1, gam, F);
#pragma unroll
      for (int c = 0; c < 4; ++c) sF[tid + 1][c] = F[c];
    }
    if (r + 1 < RBv) recon_x(slot_of(r + 1), (r + 1) & 1, jb + r + 1);
    __syncthreads();
    if (own) {
      double o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double R = -(sF[tid + 1][c] - sF[tid][c]) * hrdx - (GN[c] - GS[c]) * hrdy;  // fluxes are 2 F
        const double v = fma(a.a0, q0v[c], fma(a.a1, ring[sc][c][tid + 2], bdt * R));
        o[c] = v;
        a.out[c * a.cs + gidx] = v;
        GS[c] = GN[c];
      }
      if (HLAM) {
        const Prim w = prims(o, gm1);
        lam = fmax(lam, fmax(fabs(w.u), fabs(w.v)) + fsqrt(gam * w.p * w.ri));
        if (a.bad && !admissible(o[0], w.p)) atomicMin(a.bad, (unsigned long long)gidx);
      }
    }
  }
  if (HLAM && a.lam) block_max_to(lam, a.lam, sred);
}

int march_rows(int nrows, int strips, int rb_max, int ctas_per_sm) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0) nsm = 148;
  }
  const long long target = (long long)ctas_per_sm * nsm;
  long long rows = ((long long)nrows * strips + target - 1) / target;
  if (rows > rb_max) rows = rb_max;
  if (rows < 1) rows = 1;  // small grids: short marches, more CTAs (latency-bound sizes)
  return (int)rows;
}

template <int ORDER, bool REC>
static void fv_launch_v(int v, dim3 grid, const StageArgs& a, cudaStream_t s) {
  switch (v) {
    case 0: launch_pdl_if(!a.no_pdl, fv_stage_kernel<ORDER, REC, 0>, grid, dim3(FTX), 0, s, a); break;
    case 1: launch_pdl_if(!a.no_pdl, fv_stage_kernel<ORDER, REC, 1>, grid, dim3(FTX), 0, s, a); break;
    case 3: launch_pdl_if(!a.no_pdl, fv_stage_kernel<ORDER, REC, 3>, grid, dim3(FTX), 0, s, a); break;
    default: launch_pdl_if(!a.no_pdl, fv_stage_kernel<ORDER, REC, 8>, grid, dim3(FTX), 0, s, a); break;
  }
}

template <bool REC>
static void fv_launch_r(int rec, int v, dim3 grid, const StageArgs& a, cudaStream_t s) {
  switch (rec) {
    case 1: fv_launch_v<1, REC>(v, grid, a, s); break;
    case 2: fv_launch_v<2, REC>(v, grid, a, s); break;
    case 3: fv_launch_v<3, REC>(v, grid, a, s); break;
    default: fv_launch_v<4, REC>(v, grid, a, s); break;
  }
}

int launch_fv_stage(int k, const StageArgs& a0, cudaStream_t s) {
  StageArgs a = a0;
  const int strips = (a.nx + FTX - 1) / FTX;
  const int nr = row_range(a);
  if (nr <= 0) return 0;
  a.rows = march_rows(nr, strips, FRB, H2D_FV_MINB);
  dim3 grid(strips, (nr + a.rows - 1) / a.rows);
  // reconstruction: 1 MUSCL-2, 2 MUSCL-3 (minmod-limited); 3 / 4 the same
  // kappa-schemes unlimited (hom2d_config.fv_unlimited, f3)
  const int rec = k + (a.fv_unlimited ? 2 : 0);
  const int v = (a.q0 ? 1 : 0) | ((a.lam || a.bad) ? 2 : 0);
  if (a.dec) fv_launch_r<true>(rec, v, grid, a, s);
  else fv_launch_r<false>(rec, v, grid, a, s);
  return (int)cudaPeekAtLastError();
}

}  // namespace h2d
