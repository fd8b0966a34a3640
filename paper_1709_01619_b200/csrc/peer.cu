// peer.cu -- the peer-memory halo of the y-strip partition (SURVEY 8(e) "Stretch",
// 8(f) f4: "device-initiated peer stores via symmetric memory for halos"): instead
// of NCCL send/recv, every rank maps its strip neighbours' workspaces (CUDA IPC,
// NVLink peer access) and
//  * k_peer_signal -- after the kernels that produced a stage input X, one thread
//    publishes a sequence number into a flag of each neighbour's workspace
//    (system-scope fence, then a release store through the peer mapping): "my X
//    is complete";
//  * k_peer_pull  -- on the exchange stream, every CTA waits (acquire loads of its
//    own two flags) until both neighbours have published this exchange's number,
//    then the grid copies the neighbours' G boundary rows of X straight out of
//    their memory into the local ghost buffers (the ghost layout of exchange()).
// The stage kernels then read the ghost rows exactly as after an NCCL exchange.
//
// Why a neighbour never overwrites rows that are still being pulled: its writes
// to its boundary rows of any array happen in its boundary-band launch (and
// k_limit after it), which follows its own pull of the same exchange, which
// waits for this rank's signal of that exchange -- issued only after this rank's
// previous stage (and its pull) completed.  Every exchange is one signal + one
// pull on every rank, in the same order (SPMD), so the sequence numbers agree.
#include <cstdint>

#include "internal.h"

namespace h2d {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_peer_signal(unsigned long long* to_lo, unsigned long long* to_hi, unsigned long long seq) {
  __threadfence_system();  // the stage input written by the preceding kernels, before the flags
  if (to_lo) st_release_sys(to_lo, seq);
  if (to_hi) st_release_sys(to_hi, seq);
}

__global__ void __launch_bounds__(256) k_peer_pull(PeerPull p) {
  if (threadIdx.x == 0) {
    // both neighbours' signals of this exchange; a neighbour that never signals
    // (a dead rank) traps after 60 s instead of hanging the device
    const unsigned long long t0 = globaltimer();
    while ((p.src_lo && ld_acquire_sys(p.flag_lo) < p.seq) || (p.src_hi && ld_acquire_sys(p.flag_hi) < p.seq)) {
      __nanosleep(256);
      if (globaltimer() - t0 > 60000000000ull) __trap();
    }
  }
  __syncthreads();
  // [side][component][cnt] values; 16-B pieces when every run is 16-B aligned
  const long long n = p.cnt;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (int side = 0; side < 2; ++side) {
    const double* src = side ? p.src_hi : p.src_lo;
    double* dst = side ? p.dst_hi : p.dst_lo;
    if (!src) continue;
    for (int c = 0; c < 4; ++c) {
      const double* s = src + c * p.src_cs;
      double* d = dst + c * n;
      if (p.vec) {
        const double2* s2 = reinterpret_cast<const double2*>(s);
        double2* d2 = reinterpret_cast<double2*>(d);
        for (long long i = tid; i < n / 2; i += nth) d2[i] = __ldcg(s2 + i);
      } else {
        for (long long i = tid; i < n; i += nth) d[i] = __ldcg(s + i);
      }
    }
  }
}

}  // namespace

int launch_peer_signal(unsigned long long* to_lo, unsigned long long* to_hi, unsigned long long seq,
                       cudaStream_t s) {
  k_peer_signal<<<1, 1, 0, s>>>(to_lo, to_hi, seq);
  return (int)cudaPeekAtLastError();
}

int launch_peer_pull(const PeerPull& p, cudaStream_t s) {
  const long long per = p.vec ? p.cnt / 2 : p.cnt;
  int blocks = (int)((per + 255) / 256);
  if (blocks > 148) blocks = 148;  // a copy of a few MB: one CTA per SM at most
  if (blocks < 1) blocks = 1;
  k_peer_pull<<<blocks, 256, 0, s>>>(p);
  return (int)cudaPeekAtLastError();
}

}  // namespace h2d
