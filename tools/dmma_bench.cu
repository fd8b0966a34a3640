// dmma_bench.cu -- the north star's FP64 tensor-core question for the element
// operators (BASELINE.json north_star: "FP64 tensor cores are used only if
// applying the element-local operators at high order, cast as a batched dense
// contraction, is shown by ncu to beat CUDA-core FP64").
//
// The contraction of the P3/P4 stage kernels: for every element line (n = k+1
// solution points, 4 conserved components) y_a = sum_l D_al q_l, the n x n
// GLL/GL differentiation matrix D applied to many lines (CPR/NDG: P:684-767,
// Alg. 7-8; DG: Alg. 4; SD: Alg. 6).  Two kernels apply it
// to the same lines held in shared memory, repeated REP times so that the
// contraction (not HBM) is what is timed:
//   dfma: one thread per line, D in registers, n^2 DFMA per line and component
//         (the stage kernels' form);
//   dmma: one warp per 8 lines, mma.sync.aligned.m8n8k4.f64: A = D padded to 8
//         rows (and, at n = 5, to K = 8: two MMAs), B = 4 points x 8 lines from
//         shared memory in the fragment layout, C = 8 x 8 (n rows used).
// Both write the same y; the host checks them against each other.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o dmma_bench tools/dmma_bench.cu
//   ./dmma_bench  [then under ncu: sm__inst_executed_pipe_fp64, sm__pipe_fp64_cycles_active,
//                  smsp__inst_executed, gpu__time_duration]
// Profiling aid only (not part of the product path).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int LINES = 256;   // lines per CTA (in shared memory, [line][point] x 4 components)
constexpr int REP = 256;     // contractions per line per launch

template <int N>
__global__ void __launch_bounds__(256) k_dfma(const double* __restrict__ Dg, const double* __restrict__ q,
                                              double* __restrict__ y) {
  __shared__ double sq[4][LINES][N];
  double D[N][N];
#pragma unroll
  for (int a = 0; a < N; ++a)
#pragma unroll
    for (int l = 0; l < N; ++l) D[a][l] = Dg[a * N + l];
  const double* qb = q + (size_t)blockIdx.x * 4 * LINES * N;
  for (int i = threadIdx.x; i < 4 * LINES * N; i += blockDim.x) (&sq[0][0][0])[i] = qb[i];
  __syncthreads();
  const int line = threadIdx.x;  // blockDim == LINES
  double acc[4][N];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int a = 0; a < N; ++a) acc[c][a] = 0.0;
  for (int r = 0; r < REP; ++r) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double v[N];
#pragma unroll
      for (int l = 0; l < N; ++l) v[l] = sq[c][(line + r) & (LINES - 1)][l];  // r-dependent: no hoisting
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) s = fma(D[a][l], v[l], s);
        acc[c][a] += s;
      }
    }
  }
  double* yb = y + (size_t)blockIdx.x * 4 * LINES * N;
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int a = 0; a < N; ++a) yb[(c * LINES + line) * N + a] = acc[c][a];
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

template <int N>
__global__ void __launch_bounds__(256) k_dmma(const double* __restrict__ Dg, const double* __restrict__ q,
                                              double* __restrict__ y) {
  __shared__ double sq[4][LINES][N];
  const double* qb = q + (size_t)blockIdx.x * 4 * LINES * N;
  for (int i = threadIdx.x; i < 4 * LINES * N; i += blockDim.x) (&sq[0][0][0])[i] = qb[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;  // A: row g, col t; B: row t, col g; C: row g, cols 2t, 2t+1
  constexpr int KS = (N + 3) / 4;         // k-steps of 4
  double A[KS];
#pragma unroll
  for (int s = 0; s < KS; ++s) {
    const int l = 4 * s + t;
    A[s] = (g < N && l < N) ? Dg[g * N + l] : 0.0;
  }
  // each warp: LINES / 8 warps... 256 threads = 8 warps, 32 groups of 8 lines -> 4 groups per warp
  constexpr int GROUPS = LINES / 8 / 8;
  double acc[4][GROUPS][2];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int gr = 0; gr < GROUPS; ++gr) acc[c][gr][0] = acc[c][gr][1] = 0.0;
  for (int r = 0; r < REP; ++r) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int gr = 0; gr < GROUPS; ++gr) {
        const int l0 = (warp * GROUPS + gr) * 8;  // first line of the group
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const int k = 4 * s + t;
          const double bv = k < N ? sq[c][(l0 + g + r) & (LINES - 1)][k] : 0.0;  // B[k][n = g]: point k of line l0+g
          dmma(d0, d1, A[s], bv, d0, d1);
        }
        acc[c][gr][0] += d0;
        acc[c][gr][1] += d1;
      }
  }
  double* yb = y + (size_t)blockIdx.x * 4 * LINES * N;
  if (g < N) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int gr = 0; gr < GROUPS; ++gr) {
        const int l0 = (warp * GROUPS + gr) * 8;
        yb[(c * LINES + l0 + 2 * t) * N + g] = acc[c][gr][0];
        yb[(c * LINES + l0 + 2 * t + 1) * N + g] = acc[c][gr][1];
      }
  }
}

template <int N>
static void run(int nblk) {
  const size_t nv = (size_t)nblk * 4 * LINES * N;
  std::vector<double> hD(N * N), hq(nv);
  for (int i = 0; i < N * N; ++i) hD[i] = 0.1 * (i % 7) - 0.3;
  for (size_t i = 0; i < nv; ++i) hq[i] = 1.0 + 1e-3 * (double)(i % 101);
  double *D, *q, *y1, *y2;
  cudaMalloc(&D, N * N * 8);
  cudaMalloc(&q, nv * 8);
  cudaMalloc(&y1, nv * 8);
  cudaMalloc(&y2, nv * 8);
  cudaMemcpy(D, hD.data(), N * N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(q, hq.data(), nv * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms[2];
  for (int v = 0; v < 2; ++v) {
    for (int it = 0; it < 2; ++it) {  // warm-up, then timed
      cudaEventRecord(e0);
      if (v == 0) k_dfma<N><<<nblk, LINES>>>(D, q, y1);
      else k_dmma<N><<<nblk, LINES>>>(D, q, y2);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms[v], e0, e1);
    }
  }
  std::vector<double> a(nv), b(nv);
  cudaMemcpy(a.data(), y1, nv * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), y2, nv * 8, cudaMemcpyDeviceToHost);
  double err = 0.0;
  for (size_t i = 0; i < nv; ++i) err = fmax(err, fabs(a[i] - b[i]) / (fabs(a[i]) + 1e-300));
  const double lines = (double)nblk * LINES * 4 * REP;  // line contractions (per component)
  const double useful = lines * N * N * 2.0;             // flops
  printf("N=%d  dfma %.3f ms  %.2f TFLOP/s useful | dmma %.3f ms  %.2f TFLOP/s useful | max rel diff %.2e\n", N,
         ms[0], useful / ms[0] / 1e9, ms[1], useful / ms[1] / 1e9, err);
  cudaFree(D);
  cudaFree(q);
  cudaFree(y1);
  cudaFree(y2);
}

int main() {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int nblk = nsm * 8;
  run<4>(nblk);
  run<5>(nblk);
  return 0;
}
