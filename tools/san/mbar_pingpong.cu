// Minimal producer/consumer mbarrier ring (the decode kernel's init pattern:
// consumer warp initialises, __syncthreads, producer waits on "empty").
// Used only to check compute-sanitizer synccheck behaviour.
#include <cstdio>
#include <cstdint>
#include "../../paper_2507_03153_b200/csrc/hgca_common.cuh"
using namespace hgca;
__global__ void pingpong(int iters, int* out) {
  __shared__ __align__(8) uint64_t full[2], empty[2];
  __shared__ int slot[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane < 2) { mbar_init(&full[lane], 1); mbar_init(&empty[lane], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 1) {
    for (int k = 0; k < iters; ++k) {
      const int s = k % 2;
      if (k >= 2) mbar_wait(&empty[s], ((k / 2) - 1) & 1);
      if (lane == 0) { slot[s] = k; mbar_arrive(&full[s]); }
      __syncwarp();
    }
  } else {
    int acc = 0;
    for (int k = 0; k < iters; ++k) {
      const int s = k % 2;
      mbar_wait(&full[s], (k / 2) & 1);
      acc += slot[s];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (lane == 0) out[blockIdx.x] = acc;
  }
}
int main() {
  int* d; cudaMalloc(&d, 148 * 4);
  pingpong<<<148, 64>>>(100, d);
  int h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("pingpong %s acc=%d (expect %d)\n", cudaGetErrorString(cudaGetLastError()), h[0], 99 * 100 / 2);
  return 0;
}
