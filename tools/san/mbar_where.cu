// Where may an mbarrier live for compute-sanitizer synccheck? Ping-pong of
// one producer and one consumer warp on barriers at byte offset OFF of
// dynamic shared memory (OFF < 0: static shared memory).
#include <cstdio>
#include <cstdint>
#include "../../paper_2507_03153_b200/csrc/hgca_common.cuh"
using namespace hgca;
__global__ void where(int off, int iters, int* out, int pairs, int own) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  __shared__ __align__(8) uint64_t st[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // pair p = (consumer warp p, producer warp pairs + p), barriers at off + 64 p
  const int p = warp % pairs;
  uint64_t* b = off < 0 ? st : reinterpret_cast<uint64_t*>(dyn + off + 64 * p);
  uint64_t *full = b, *empty = b + 2;
  if (own ? warp < pairs : warp == 0) {
    for (int q = own ? warp : 0; q < (own ? warp + 1 : pairs); ++q) {
      uint64_t* bq = reinterpret_cast<uint64_t*>(dyn + off + 64 * q);
      if (lane < 2) { mbar_init(bq + lane, 1); mbar_init(bq + 2 + lane, 1); }
    }
    fence_mbar_init();
  }
  __syncthreads();
  int acc = 0;
#ifdef SPLIT
  if (warp >= pairs) {
    for (int k = 0; k < iters; ++k) {
      const int s = k & 1;
      if (k >= 2) mbar_wait(&empty[s], ((k >> 1) - 1) & 1);
      if (lane == 0) mbar_arrive(&full[s]);
      __syncwarp();
    }
  } else {
    for (int k = 0; k < iters; ++k) {
      const int s = k & 1;
      mbar_wait(&full[s], (k >> 1) & 1);
      acc += k;
      if (lane == 0) mbar_arrive(&empty[s]);
      __syncwarp();
    }
  }
#else
  for (int k = 0; k < iters; ++k) {
    const int s = k & 1;
    if (warp >= pairs) {
      if (k >= 2) mbar_wait(&empty[s], ((k >> 1) - 1) & 1);
      if (lane == 0) mbar_arrive(&full[s]);
    } else {
      mbar_wait(&full[s], (k >> 1) & 1);
      acc += k;
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    __syncwarp();
  }
#endif
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}
int main(int argc, char** argv) {
  int* d; cudaMalloc(&d, 4 * 148);
  const int off = atoi(argv[1]), smem = atoi(argv[2]), pairs = atoi(argv[3]), own = atoi(argv[4]);
  cudaFuncSetAttribute(where, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  where<<<148, 64 * pairs, smem>>>(off, 20, d, pairs, own);
  int h; cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("off %d smem %d pairs %d own %d: %s acc=%d\n", off, smem, pairs, own, cudaGetErrorString(cudaGetLastError()), h);
}
