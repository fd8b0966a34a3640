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

#ifndef H2D_FV_WSQRT
#define H2D_FV_WSQRT fsqrt_ws  // dissipation-speed square root (A/B: fsqrt)
#endif
// TWICE the Rusanov flux along DIR: fL + fR - lam (qR - qL).  The
// factor 1/2 moves into the metric of the flux difference (0.5 / dx): scaling
// by powers of two is exact, so nothing changes but 5 multiplications per face.
template <int DIR>
__device__ __forceinline__ void rusanov2(const double qL[4], const double qR[4], double gm1, double gam, double F2[4]) {
  const Prim wl = prims(qL, gm1), wr = prims(qR, gm1);
  double fL[4], fR[4];
  flux<DIR>(qL, wl, fL);
  flux<DIR>(qR, wr, fR);
  const double sl = fabs(DIR == 0 ? wl.u : wl.v) + H2D_FV_WSQRT(gam * wl.p * wl.ri);
  const double sr = fabs(DIR == 0 ? wr.u : wr.v) + H2D_FV_WSQRT(gam * wr.p * wr.ri);
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
  const double dtv = stage_dt(a);  // (stage 1 / 2 of a fused-dt step: publishes / commits the clock)
  if (dtv == 0.0) return;
  const int tid = threadIdx.x;
  int bhi;
  const int i0 = blockIdx.x * FTX, jb = band_start(a, bhi);
  const int TXv = min(FTX, a.nx - i0), RBv = min(a.rows, bhi - jb);
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

// ---------------------------------------------------------------------------
// Warp-strip kernel (the default): every warp marches its own strip of WS = 62
// cells up the rows -- two adjacent cells per lane, lane 31 on the right halo --
// with its own cp.async rings (stage input with a 2-cell halo each side, q^n)
// and no CTA barrier in the march:
//  * a lane reconstructs its two cells in x from one 16-B read of its pair and
//    its neighbours (and the hi state of the cell on its left, recomputed, not
//    shuffled); the face between its cells is lane-local, the E face of its
//    second cell is the right lane's W-face flux by a shuffle -- every x face is
//    evaluated once and no lane runs a face alone;
//  * y faces as in the CTA kernel: the N face of each column is carried to the
//    next row as its S face;
//  * q^n arrives through its own ring one row ahead (no global load latency in
//    the epilogue); the march length is chosen so the grid is a whole number of
//    waves.
// Arithmetic per face / cell is the CTA kernel's (same helpers, same order).
#ifndef H2D_FVW_DEPTH
#define H2D_FVW_DEPTH 1
#endif
#ifndef H2D_FVW_MINB
#define H2D_FVW_MINB 3
#endif
namespace {
constexpr int WPC = 4;                     // warps per CTA (independent strips)
// a warp strip is WS = 62 cells: lanes 0..30 own two cells each, lane 31 (and, in a
// ragged strip, every lane past the last cell) works on the halo cells to the
// right, so the strip's E face comes to the last owning lane by the same shuffle
// as every other E face -- no divergent face evaluation; WL = 64 pair slots
constexpr int WS = 62, WL = 64, WW = WL + 4;  // cells per warp strip; ring row width (2 halo cells each side)
constexpr int WD = H2D_FVW_DEPTH, WNS = 3 + WD;  // rows in flight; ring rows
constexpr int QS = WD + 1;                       // q^n ring rows (row x lands with ring row x+2, read at step x)
// dynamic shared memory: per warp WNS ring rows x 4 components x WW, then (stages
// with q^n) QS q-ring rows x 4 x WL, then the block-max scratch
constexpr int WRING = WNS * 4 * WW, WQ = QS * 4 * WL;
constexpr size_t fvw_smem(bool hq0) { return sizeof(double) * ((size_t)WPC * (WRING + (hq0 ? WQ : 0)) + WPC); }
}  // namespace

template <int ORDER, bool REC, int V>
__global__ void __launch_bounds__(WPC * 32, H2D_FVW_MINB) fv_warp_kernel(const StageArgs a) {
  const bool HQ0 = V == 8 ? a.q0 != nullptr : (V & 1), HLAM = V == 8 ? (a.lam || a.bad) : (V & 2) != 0;
  extern __shared__ __align__(16) double fv_smem[];
  double(*const ring)[WNS][4][WW] = reinterpret_cast<double(*)[WNS][4][WW]>(fv_smem);
  double(*const qring)[QS][4][WL] = reinterpret_cast<double(*)[QS][4][WL]>(fv_smem + WPC * WRING);
  double* const sred = fv_smem + WPC * WRING + (HQ0 ? WPC * WQ : 0);
  pdl_wait();
  pdl_launch();
  const double dtv = stage_dt(a);  // (stage 1 / 2 of a fused-dt step: publishes / commits the clock)
  if (dtv == 0.0) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int bhi;
  const int i0 = (blockIdx.x * WPC + wid) * WS, jb = band_start(a, bhi);
  const double gam = a.gamma, gm1 = a.gamma - 1.0;
  double lam = 0.0;
  if (i0 < a.nx) {  // warp-uniform
    const int TXv = min(WS, a.nx - i0), RBv = min(a.rows, bhi - jb);
    const int c0 = 2 * lane;                         // local index of the lane's first cell
    const bool own0 = c0 < TXv, own1 = c0 + 1 < TXv;
    long long* const dec = REC ? a.dec : nullptr;
    double(*const rw)[4][WW] = ring[wid];
    double(*const qw)[4][WL] = qring[HQ0 ? wid : 0];
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
    auto dmap_at = [&](int jr, int ir) -> long long* {
      if (!REC || !a.dmap) return nullptr;
      if (ir < 0) ir = a.bcx == 0 ? ir + a.nx : 0;
      if (ir >= a.nx) ir = a.bcx == 0 ? ir - a.nx : a.nx - 1;
      if (jr < 0) jr = a.ghost_lo ? jr + a.nrows : 0;
      if (jr >= a.nrows) jr = a.ghost_hi ? jr - a.nrows : a.nrows - 1;
      return a.dmap + (long long)jr * a.nx + ir;
    };
    // the lane's pair (16 B when aligned) of each component of a row into dst[c][...]
    // copies without branches (a TMA bulk-copy ring with one mbarrier per slot
    // was measured 7-13 % slower: one lane issuing 8-16 small bulk copies per
    // step): predicated cp.async -- the lane's pair as one 16-B copy (or its last
    // own cell as an 8-B copy), the halo cells by lanes 0..3; a lane past the
    // strip copies nothing (its slots are never read as data, and a zero-filling
    // copy there would race with the halo copies into slots TXv+2, TXv+3)
    // halo column of lanes 0..3: slots 0, 1 = cells i0-2, i0-1; TXv+2, TXv+3 = cells i0+TXv, +1
    int hx = lane < 2 ? i0 - 2 + lane : i0 + TXv + (lane - 2);
    if (a.bcx == 0) hx = hx < 0 ? hx + a.nx : (hx >= a.nx ? hx - a.nx : hx);
    else hx = hx < 0 ? 0 : (hx >= a.nx ? a.nx - 1 : hx);
    const int p16 = own1, p8 = own0 && !own1, ph = lane < 4;
    const int hs = ph ? (lane < 2 ? lane : TXv + lane) : 0;
    const int pc = own0 ? c0 : 0;  // a valid address for lanes past the strip
    const int hxx = ph ? hx : i0;
    auto copy_pair = [&](double* d0, int dstride, const double* g, long long cs) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p cp.async.cg.shared.global [%0], [%1], 16;\n\t}"
            ::"r"(smem_u32(d0 + c * dstride)), "l"(g + c * cs), "r"(p16)
            : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p cp.async.ca.shared.global [%0], [%1], 8;\n\t}"
            ::"r"(smem_u32(d0 + c * dstride)), "l"(g + c * cs), "r"(p8)
            : "memory");
      }
    };
    auto issue_row = [&](int jr, int slot) {
      long long cs;
      const double* rb = row_ptr(jr, cs);
      copy_pair(&rw[slot][0][c0 + 2], WW, rb + i0 + pc, cs);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p cp.async.ca.shared.global [%0], [%1], 8;\n\t}"
            ::"r"(smem_u32(&rw[slot][c][hs])), "l"(rb + c * cs + hxx), "r"(ph)
            : "memory");
    };
    auto issue_q0 = [&](int jr, int slot) {  // q^n row jr (an own row) into q-ring slot
      copy_pair(&qw[slot][0][c0], WL, a.q0 + (long long)jr * a.nx + i0 + pc, a.cs);
    };
    auto commit = [] { asm volatile("cp.async.commit_group;" ::: "memory"); };

    // prologue: rows jb-2 .. jb+1 (ring slot of row r: (r + 2) % WNS) and q^n rows
    // jb .. jb+WD-1 (q slot r); the S face of row jb and the hi y-state of row jb;
    // then rows jb+2 .. jb+1+WD, one group each (row jb+2 into row jb-2's slot)
    for (int r = -2; r <= 1; ++r) issue_row(jb + r, r + 2);
    if (HQ0)
      for (int r = 0; r < WD && r < RBv; ++r) issue_q0(jb + r, r);
    commit();
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    double GS[2][4], yHi[2][4];
    {
      const int wb = (jb == 0 && a.count_bot) ? 1 : 0;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const bool ok = k ? own1 : own0;
        double lo[4], hi[4], dm;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double r0 = rw[0][c][c0 + 2 + k], r1 = rw[1][c][c0 + 2 + k];
          const double r2 = rw[2][c][c0 + 2 + k], r3 = rw[3][c][c0 + 2 + k];
          cell_faces<ORDER>(r0, r1, r2, dm, hi[c], ok ? dec : nullptr, wb, ok ? dmap_at(jb - 1, i0 + c0 + k) : nullptr);
          cell_faces<ORDER>(r1, r2, r3, lo[c], yHi[k][c], ok ? dec : nullptr, 2, ok ? dmap_at(jb, i0 + c0 + k) : nullptr);
        }
        rusanov2<1>(hi, lo, gm1, gam, GS[k]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int k = 2; k < 2 + WD; ++k) {
      if (k <= RBv + 1) issue_row(jb + k, (k + 2) % WNS);
      commit();
    }

    const double bdt = a.bcoef * dtv;
    const double hrdx = 0.5 * a.rdx2, hrdy = 0.5 * a.rdy2;
    // ring slots of rows r, r+1, r+2 and of the row issued at step r (r+2+WD: the
    // slot of row r-1), q-ring slots of rows r (read) and r+WD (issued)
    int S0 = 2 % WNS, S1 = 3 % WNS, S2 = 4 % WNS, SI = 1 % WNS, Q0 = 0, QI = WD % QS;
    auto adv = [](int& x, int n) { x = (x + 1 == n) ? 0 : x + 1; };
#pragma unroll 1
    for (int r = 0; r < RBv; ++r) {
      asm volatile("cp.async.wait_group %0;" ::"n"(WD - 1) : "memory");
      __syncwarp();
      if (r + 2 + WD <= RBv + 1) issue_row(jb + r + 2 + WD, SI);
      if (HQ0 && r + WD < RBv) issue_q0(jb + r + WD, QI);
      commit();
      const int jr = jb + r;
      const long long gidx = (long long)jr * a.nx + (i0 + c0);
      // x: the pair, its neighbours, the face states of both cells and the hi
      // state of the cell left of the pair (recomputed, no shuffle); then the W
      // face of the first cell, the face between them and (by shuffle: the right
      // lane's W face) the E face of the second, reduced at once to the x flux
      // differences Rx.  A lane's cell past the strip's last cell is the halo
      // cell i0+TXv (first fake cell; its lo state gives the strip's E face) or
      // beyond (unused values)
      double xq[2][4], Rx[2][4];
      {
        double lo[2][4], hi[2][4], hL[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 p = *reinterpret_cast<const double2*>(&rw[S0][c][c0 + 2]);
          const double2 m2 = *reinterpret_cast<const double2*>(&rw[S0][c][c0]);
          const double xp = rw[S0][c][c0 + 4];
          xq[0][c] = p.x;
          xq[1][c] = p.y;
          double dm;
          // left cell: counted by its owner (the left lane), here only the domain's
          // W ghost of the first lane (P:346-351 face form: the bottom/left ghost face)
          cell_faces<ORDER>(m2.x, m2.y, p.x, dm, hL[c], lane == 0 ? dec : nullptr, i0 == 0 ? 1 : 0,
                            lane == 0 ? dmap_at(jr, i0 - 1) : nullptr);
          const bool h0 = !own0 && c0 == TXv, h1 = !own1 && c0 + 1 == TXv;  // the halo cell i0+TXv
          const int wh = i0 + TXv == a.nx ? 1 : 0;
          cell_faces<ORDER>(m2.y, p.x, p.y, lo[0][c], hi[0][c], (own0 || h0) ? dec : nullptr, own0 ? 2 : wh,
                            (own0 || h0) ? dmap_at(jr, i0 + c0) : nullptr);
          cell_faces<ORDER>(p.x, p.y, xp, lo[1][c], hi[1][c], (own1 || h1) ? dec : nullptr, own1 ? 2 : wh,
                            (own1 || h1) ? dmap_at(jr, i0 + c0 + 1) : nullptr);
        }
        double FW[4], FM[4], FE[4];
        rusanov2<0>(hL, lo[0], gm1, gam, FW);
        rusanov2<0>(hi[0], lo[1], gm1, gam, FM);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          FE[c] = __shfl_down_sync(0xffffffffu, FW[c], 1);
          Rx[0][c] = -(FM[c] - FW[c]) * hrdx;  // fluxes are 2 F
          Rx[1][c] = -(FE[c] - FM[c]) * hrdx;
        }
      }
      // y, per column: the lo / hi states of row r+1 (rows r .. r+2), the N face,
      // the residual, the RK combination and the store
      const int wn = (r + 1 < RBv) ? 2 : ((jb + RBv == a.nrows) ? 1 : 0);
      double o[2][4], y1[2][4], y2[2][4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double2 p1 = *reinterpret_cast<const double2*>(&rw[S1][c][c0 + 2]);
        const double2 p2 = *reinterpret_cast<const double2*>(&rw[S2][c][c0 + 2]);
        y1[0][c] = p1.x; y1[1][c] = p1.y;
        y2[0][c] = p2.x; y2[1][c] = p2.y;
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const bool ok = k ? own1 : own0;
        double ylo[4], yhn[4], GN[4];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          cell_faces<ORDER>(xq[k][c], y1[k][c], y2[k][c], ylo[c], yhn[c],
                            ok ? dec : nullptr, wn, ok ? dmap_at(jr + 1, i0 + c0 + k) : nullptr);
        rusanov2<1>(yHi[k], ylo, gm1, gam, GN);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double R = Rx[k][c] - (GN[c] - GS[k][c]) * hrdy;
          double v = fma(a.a1, xq[k][c], bdt * R);
          if (HQ0) v = fma(a.a0, qw[Q0][c][c0 + k], v);
          o[k][c] = v;
          GS[k][c] = GN[c];
          yHi[k][c] = yhn[c];
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double* g = a.out + c * a.cs + gidx;
        if (own1) *reinterpret_cast<double2*>(g) = make_double2(o[0][c], o[1][c]);
        if (own0 && !own1) g[0] = o[0][c];
      }
      if (HLAM) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const bool ok = k ? own1 : own0;
          const Prim w = prims(o[k], gm1);
          const double sp = fmax(fabs(w.u), fabs(w.v)) + fsqrt(gam * w.p * w.ri);
          lam = ok ? nanmax(lam, sp) : lam;
          if (ok && a.bad && !admissible(o[k][0], w.p)) atomicMin(a.bad, (unsigned long long)(gidx + k));
        }
      }
      adv(S0, WNS); adv(S1, WNS); adv(S2, WNS); adv(SI, WNS); adv(Q0, QS); adv(QI, QS);
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

// rows per CTA such that the grid is (close to) a whole number of waves of
// ctas_per_sm x #SM resident CTAs: the fewest waves whose marches fit rb_max
int march_rows_waves(int nrows, int strips, int rb_max, int ctas_per_sm) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm <= 0) nsm = 148;
  }
  const long long target = (long long)ctas_per_sm * nsm;
  for (long long w = 1;; ++w) {
    const long long bpc = w * target / strips;  // row blocks per strip column in w waves
    if (bpc < 1) continue;
    const long long rows = (nrows + bpc - 1) / bpc;
    if (rows <= rb_max) return (int)(rows < 1 ? 1 : rows);
  }
}

#ifndef H2D_FV_WARP
#define H2D_FV_WARP 1  // warp-strip kernel where the layout allows (0: the CTA-strip kernel always)
#endif
template <int ORDER, bool REC, int V>
static cudaError_t fvw_launch(dim3 grid, const StageArgs& a, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  const size_t sm = fvw_smem(V == 8 ? a.q0 != nullptr : (V & 1) != 0);
  const cudaError_t e = smem_optin(fv_warp_kernel<ORDER, REC, V>, (int)fvw_smem(true), attr);
  if (e != cudaSuccess) return e;
  return launch_pdl_if(!a.no_pdl, fv_warp_kernel<ORDER, REC, V>, grid, dim3(WPC * 32), sm, s, a);
}

template <int ORDER, bool REC>
static void fv_launch_v(int v, dim3 grid, const StageArgs& a, cudaStream_t s, bool warp) {
  if (warp) {
    switch (v) {
      case 0: fvw_launch<ORDER, REC, 0>(grid, a, s); break;
      case 1: fvw_launch<ORDER, REC, 1>(grid, a, s); break;
      case 3: fvw_launch<ORDER, REC, 3>(grid, a, s); break;
      default: fvw_launch<ORDER, REC, 8>(grid, a, s); break;
    }
    return;
  }
  switch (v) {
    case 0: launch_pdl_if(!a.no_pdl, fv_stage_kernel<ORDER, REC, 0>, grid, dim3(FTX), 0, s, a); break;
    case 1: launch_pdl_if(!a.no_pdl, fv_stage_kernel<ORDER, REC, 1>, grid, dim3(FTX), 0, s, a); break;
    case 3: launch_pdl_if(!a.no_pdl, fv_stage_kernel<ORDER, REC, 3>, grid, dim3(FTX), 0, s, a); break;
    default: launch_pdl_if(!a.no_pdl, fv_stage_kernel<ORDER, REC, 8>, grid, dim3(FTX), 0, s, a); break;
  }
}

template <bool REC>
static void fv_launch_r(int rec, int v, dim3 grid, const StageArgs& a, cudaStream_t s, bool warp) {
  switch (rec) {
    case 1: fv_launch_v<1, REC>(v, grid, a, s, warp); break;
    case 2: fv_launch_v<2, REC>(v, grid, a, s, warp); break;
    case 3: fv_launch_v<3, REC>(v, grid, a, s, warp); break;
    default: fv_launch_v<4, REC>(v, grid, a, s, warp); break;
  }
}

static bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

int launch_fv_stage(int k, const StageArgs& a0, cudaStream_t s) {
  StageArgs a = a0;
  const int nr = row_range(a);
  if (nr <= 0) return 0;
  // the warp kernel moves cell pairs as 16-B units: every row / component start
  // even and every array 16-B aligned (odd widths, e.g. 45 or 131 cells: the CTA kernel)
  const bool warp = H2D_FV_WARP && (a.nx % 2 == 0) && (a.cs % 2 == 0) && (a.gcs % 2 == 0) && al16(a.q) &&
                    al16(a.q0) && al16(a.out) && al16(a.ghost_lo) && al16(a.ghost_hi);
  int strips;
  if (warp) {
    strips = ((a.nx + WS - 1) / WS + WPC - 1) / WPC;  // CTAs across x
    a.rows = march_rows_waves(nr, strips, FRB, H2D_FVW_MINB);
  } else {
    strips = (a.nx + FTX - 1) / FTX;
    a.rows = march_rows(nr, strips, FRB, H2D_FV_MINB);
  }
  dim3 grid(strips, band_blocks(a));
  // reconstruction: 1 MUSCL-2, 2 MUSCL-3 (minmod-limited); 3 / 4 the same
  // kappa-schemes unlimited (hom2d_config.fv_unlimited, f3)
  const int rec = k + (a.fv_unlimited ? 2 : 0);
  const int v = (a.q0 ? 1 : 0) | ((a.lam || a.bad) ? 2 : 0);
  if (a.dec) fv_launch_r<true>(rec, v, grid, a, s, warp);
  else fv_launch_r<false>(rec, v, grid, a, s, warp);
  return (int)cudaPeekAtLastError();
}

}  // namespace h2d
