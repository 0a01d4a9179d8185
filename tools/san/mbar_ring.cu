// Decode-kernel-shaped mbarrier rings (dynamic smem, 1 KB aligned, per-warp
// rings, expect_tx + bulk copy), for compute-sanitizer synccheck triage.
#include <cstdio>
#include <cstdint>
#include "../../paper_2507_03153_b200/csrc/hgca_common.cuh"
#include "../../paper_2507_03153_b200/csrc/hgca_tc.cuh"
using namespace hgca;
#ifndef NCV
#define NCV 2
#endif
#ifndef ITERS
#define ITERS 50
#endif
#ifndef BAROFF
#define BAROFF 36416
#endif
constexpr int STAGE = 16384, S = 2, RING = 36864, NC = NCV;
template <int MODE>  // 0 plain arrive; 1 expect_tx + bulk copy; 2 = 1 + align slack
__global__ void ring(int iters, const float* src, int* out, int rtoff) {
#ifdef RTOFF
  const int baroff = rtoff;
#else
  const int baroff = BAROFF;
#endif
  #ifdef ALIGN1K
  extern __shared__ __align__(1024) unsigned char raw[];
#else
  extern __shared__ unsigned char raw[];
#endif
  unsigned char* sm = MODE == 2 ? reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023)) : raw;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < NC) {
    uint64_t* b = reinterpret_cast<uint64_t*>(sm + warp * RING + baroff);
    if (lane < S) { mbar_init(b + lane, 1); mbar_init(b + S + lane, 1); }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp >= NC) {
    unsigned char* cw = sm + (warp - NC) * RING;
    uint64_t* full = reinterpret_cast<uint64_t*>(cw + baroff);
    uint64_t* empty = full + S;
    for (int k = 0; k < iters; ++k) {
      const int s = k % S;
      if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
      if (lane == 0) {
#ifndef NOSTORE
        reinterpret_cast<int*>(cw + 36352)[s * 8] = k;
#endif
        if (MODE == 0) mbar_arrive(&full[s]);
        else { mbar_expect_tx(&full[s], 1024); bulk_g2s(cw + s * STAGE, src, 1024, &full[s]); }
      }
      __syncwarp();
    }
  } else {
    unsigned char* cw = sm + warp * RING;
    uint64_t* full = reinterpret_cast<uint64_t*>(cw + baroff);
    uint64_t* empty = full + S;
    int acc = 0;
    for (int k = 0; k < iters; ++k) {
      const int s = k % S;
      mbar_wait(&full[s], (k / S) & 1);
#ifndef NOSTORE
      acc += reinterpret_cast<int*>(cw + 36352)[s * 8];
#else
      acc += k;
#endif
#ifdef ARRIVE_FIRST
      if (lane == 0) mbar_arrive(&empty[s]);
      __syncwarp();
#else
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
#endif
    }
    if (lane == 0) out[blockIdx.x * NC + warp] = acc;
  }
}
template <int MODE> void run(const float* src, int* d) {
  const int smem = NC * RING + 1024;
  cudaFuncSetAttribute(ring<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ring<MODE><<<148, 2 * NC * 32, smem>>>(ITERS, src, d, BAROFF);
  int h[2]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("mode %d: %s acc=%d (expect %d)\n", MODE, cudaGetErrorString(cudaGetLastError()), h[0], (ITERS - 1) * ITERS / 2);
}
int main(int argc, char** argv) {
  float* src; int* d; cudaMalloc(&src, 4096); cudaMalloc(&d, 148 * NC * 4);
  const int m = argc > 1 ? atoi(argv[1]) : 0;
  if (m == 0) run<0>(src, d); else if (m == 1) run<1>(src, d); else run<2>(src, d);
  return 0;
}
