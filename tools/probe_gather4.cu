// Probe: TMA tile::gather4 (4 arbitrary rows per op) vs cp.async for random
// 256 B row gathers on B200. Checks correctness against direct loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/probe_gather4 tools/probe_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// each warp: lanes 0..7 issue one gather4 per sub-chunk of 32 rows; NS stages per warp
template <int NS>
__global__ void __launch_bounds__(256) g4_kernel(const __grid_constant__ CUtensorMap map, const int* __restrict__ idx,
                                                 int nrows, unsigned* sink, int check, const uint4* tab) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  unsigned char* ws = sm + warp * (NS * 8192 + 128);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ws + NS * 8192);
  if (lane < NS) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(&bar[lane])), "r"(1));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gw = blockIdx.x * nw + warp, nwt = gridDim.x * nw;
  const int nsub = nrows / 32;
  unsigned acc = 0;
  int k = 0;
  auto issue = [&](int sub, int s) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[s])), "r"(8192));
    __syncwarp();
    if (lane < 8) {
      const int* ix = idx + sub * 32 + lane * 4;
      int r0 = ix[0], r1 = ix[1], r2 = ix[2], r3 = ix[3];
      unsigned char* dst = ws + s * 8192 + lane * 1024;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
          ::"r"(s32(dst)), "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(s32(&bar[s]))
          : "memory");
    }
  };
  int mine = 0;
  for (int sub = gw; sub < nsub; sub += nwt) ++mine;
  for (int j = 0; j < NS && j < mine; ++j) issue(gw + j * nwt, j);
  for (int j = 0; j < mine; ++j) {
    const int s = j % NS;
    const uint32_t par = (j / NS) & 1;
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
                 ::"r"(s32(&bar[s])), "r"(par) : "memory");
    const uint4* rowp = reinterpret_cast<const uint4*>(ws + s * 8192 + lane * 256);
    for (int p = 0; p < 16; ++p) {
      uint4 v = rowp[(p + lane) & 15];
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
      if (check) {
        const int sub = gw + j * nwt;
        const int row = idx[sub * 32 + lane];
        uint4 w = tab[(size_t)row * 16 + ((p + lane) & 15)];
        if (w.x != v.x || w.y != v.y || w.z != v.z || w.w != v.w) atomicAdd(sink + 1, 1u);
      }
    }
    __syncwarp();
    if (j + NS < mine) issue(gw + (j + NS) * nwt, s);
  }
  if (acc == 0x12345u) sink[0] = acc;
}

__global__ void fill(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4((unsigned)i, (unsigned)(i * 7), (unsigned)(i >> 3), 0xabcd0000u ^ (unsigned)i);
}

int main() {
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
  if (!encode) { printf("no encode fn\n"); return 1; }
  const size_t bytes = 4ull << 30;
  const size_t nt = bytes / 256;
  uint4* tab;
  CK(cudaMalloc(&tab, bytes));
  fill<<<1184, 256>>>(tab, bytes / 16);
  const int nrows = 1 << 22;
  std::vector<int> h(nrows);
  std::mt19937 gen(3);
  for (auto& x : h) x = gen() % nt;
  int* didx;
  CK(cudaMalloc(&didx, nrows * 4));
  CK(cudaMemcpy(didx, h.data(), nrows * 4, cudaMemcpyHostToDevice));
  unsigned* sink;
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(sink, 0, 8));
  CUtensorMap map;
  cuuint64_t gdim[2] = {128, (cuuint64_t)nt};
  cuuint64_t gstr[1] = {256};
  cuuint32_t box[2] = {128, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, tab, gdim, gstr, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)r);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int NS = 3;
  const int smem = 8 * (NS * 8192 + 128);
  CK(cudaFuncSetAttribute(g4_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  g4_kernel<NS><<<148, 256, smem>>>(map, didx, 1 << 16, sink, 1, tab);
  CK(cudaDeviceSynchronize());
  unsigned hs[2];
  CK(cudaMemcpy(hs, sink, 8, cudaMemcpyDeviceToHost));
  printf("gather4 correctness: %u mismatching 16B pieces (of %d)\n", hs[1], (1 << 16) * 16);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    g4_kernel<NS><<<148, 256, smem>>>(map, didx, nrows, sink, 0, tab);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("gather4 NS=%d 8 warps/SM: %.1f GB/s\n", NS, (double)nrows * 256 / ms / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
