// B200 micro-probes for the hybrid decode-attention design.
//   1. pure-read HBM streaming ceiling (LDG.128, 4 GiB)
//   2. FP64 DFMA throughput (F3 puts fp64 QK on the critical path)
//   3. random 256 B / 512 B row gathers: LDGSTS (cp.async 16 B) vs TMA bulk (cp.async.bulk)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe tools/probe_b200.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void read_stream(const int4* __restrict__ p, size_t n, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    int4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
    acc.x ^= a.x ^ b.x ^ c.x ^ d.x; acc.y ^= a.y ^ b.y ^ c.y ^ d.y;
    acc.z ^= a.z ^ b.z ^ c.z ^ d.z; acc.w ^= a.w ^ b.w ^ c.w ^ d.w;
  }
  for (; i < n; i += stride) { int4 a = __ldcs(p + i); acc.x ^= a.x; }
  if (acc.x == 0x12345678 && acc.y == 7) sink[0] = acc;
}

__global__ void dfma_chain(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void ffma_chain(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  float a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float m = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; ++i) {
    a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
    a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// cvt f32->f64 throughput
__global__ void cvt_chain(double* out, const float* in, int iters) {
  float x0 = in[threadIdx.x], x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double acc0 = 0, acc1 = 0;
  for (int i = 0; i < iters; ++i) {
    acc0 += (double)x0 + (double)x1; acc1 += (double)x2 + (double)x3;
    x0 += 1.f; x1 += 1.f; x2 += 1.f; x3 += 1.f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1;
}

// ---- gather via cp.async (LDGSTS) ----
template <int ROWB, int CH>
__global__ void gather_ldgsts(const char* __restrict__ base, const int* __restrict__ idx, int nrows, int* sink) {
  extern __shared__ __align__(16) char smem[];
  constexpr int VPR = ROWB / 16;  // 16 B vectors per row
  int chunks = nrows / CH;
  unsigned acc = 0;
  for (int c = blockIdx.x; c < chunks; c += gridDim.x) {
    int buf = (c / gridDim.x) & 1;
    char* s = smem + buf * CH * ROWB;
    for (int v = threadIdx.x; v < CH * VPR; v += blockDim.x) {
      int r = v / VPR, o = v % VPR;
      const char* src = base + (size_t)idx[c * CH + r] * ROWB + o * 16;
      unsigned dst = (unsigned)__cvta_generic_to_shared(s + r * ROWB + o * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 1;");
    __syncthreads();
    acc ^= ((unsigned*)s)[threadIdx.x];
  }
  asm volatile("cp.async.wait_group 0;");
  if (acc == 0xdeadbeef) sink[0] = acc;
}

// ---- gather via TMA bulk copies (cp.async.bulk), multi-stage mbarrier ring ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}

template <int ROWB, int CH, int ST>
__global__ void gather_bulk(const char* __restrict__ base, const int* __restrict__ idx, int nrows, int* sink) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bars[ST];
  int chunks = nrows / CH;
  int my = 0;
  for (int c = blockIdx.x; c < chunks; c += gridDim.x) ++my;
  if (threadIdx.x == 0) for (int s = 0; s < ST; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  auto issue = [&](int k) {  // warp 0 issues chunk k of this CTA
    int c = blockIdx.x + k * gridDim.x;
    int s = k % ST;
    char* dst = smem + s * CH * ROWB;
    if (threadIdx.x == 0) mbar_expect_tx(&bars[s], CH * ROWB);
    __syncwarp();
    for (int r = threadIdx.x; r < CH; r += 32)
      bulk_g2s(dst + r * ROWB, base + (size_t)idx[c * CH + r] * ROWB, ROWB, &bars[s]);
  };
  if (threadIdx.x < 32) for (int k = 0; k < ST && k < my; ++k) issue(k);
  unsigned acc = 0;
  for (int k = 0; k < my; ++k) {
    int s = k % ST;
    mbar_wait(&bars[s], (k / ST) & 1);
    acc ^= ((unsigned*)(smem + s * CH * ROWB))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x < 32 && k + ST < my) issue(k + ST);
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d smem/SM %zu clock %d kHz\n", prop.name, prop.multiProcessorCount,
         prop.sharedMemPerMultiprocessor, prop.clockRate);
  int nsm = prop.multiProcessorCount;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  // 1. read stream
  size_t bytes = 4ull << 30;
  int4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  int4* sink; CK(cudaMalloc(&sink, 64));
  for (int bpsm : {2, 4, 8}) {
    for (int t : {256, 512}) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0));
        read_stream<<<nsm * bpsm, t>>>(buf, bytes / 16, sink);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1)); best = std::min(best, ms);
      }
      printf("read_stream grid=%d*%d thr=%d: %.1f GB/s\n", nsm, bpsm, t, bytes / best / 1e6);
    }
  }
  // 2. DFMA / FFMA throughput
  double* dout; CK(cudaMalloc(&dout, 1 << 26));
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 4096, blocks = nsm * 8, thr = 256;
    CK(cudaEventRecord(e0));
    dfma_chain<<<blocks, thr>>>(dout, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double n = (double)blocks * thr * iters * 8;
    printf("DFMA: %.2f TFLOP/s fp64 (%.1f DFMA/clk/SM at %d MHz)\n", 2 * n / ms / 1e9,
           n / (ms * 1e-3) / nsm / (prop.clockRate * 1e3), prop.clockRate / 1000);
    CK(cudaEventRecord(e0));
    ffma_chain<<<blocks, thr>>>((float*)dout, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("FFMA: %.2f TFLOP/s fp32\n", 2 * n / ms / 1e9);
    CK(cudaEventRecord(e0));
    cvt_chain<<<blocks, thr>>>(dout, (float*)buf, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("F2F.F64.F32: %.2f Tcvt/s (+2 DADD per 2 cvt)\n", (double)blocks * thr * iters * 4 / ms / 1e9);
  }
  // 3. gathers over a 4 GiB table of rows
  std::mt19937 gen(1);
  for (int rowb : {256, 512}) {
    int nrows_tab = (int)(bytes / rowb);
    int nrows = 1 << 21;  // 2M rows gathered
    std::vector<int> h(nrows);
    for (auto& x : h) x = gen() % nrows_tab;
    int* didx; CK(cudaMalloc(&didx, nrows * 4)); CK(cudaMemcpy(didx, h.data(), nrows * 4, cudaMemcpyHostToDevice));
    double gb = (double)nrows * rowb;
    for (int bpsm : {2, 4, 8}) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0));
        if (rowb == 256) {
          CK(cudaFuncSetAttribute(gather_ldgsts<256, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 256));
          gather_ldgsts<256, 64><<<nsm * bpsm, 128, 2 * 64 * 256>>>((char*)buf, didx, nrows, (int*)sink);
        } else {
          CK(cudaFuncSetAttribute(gather_ldgsts<512, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 512));
          gather_ldgsts<512, 64><<<nsm * bpsm, 128, 2 * 64 * 512>>>((char*)buf, didx, nrows, (int*)sink);
        }
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
      }
      printf("gather LDGSTS row=%dB blocks/SM=%d: %.1f GB/s\n", rowb, bpsm, gb / best / 1e6);
      best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0));
        if (rowb == 256) {
          CK(cudaFuncSetAttribute(gather_bulk<256, 64, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 64 * 256));
          gather_bulk<256, 64, 4><<<nsm * bpsm, 128, 4 * 64 * 256>>>((char*)buf, didx, nrows, (int*)sink);
        } else {
          CK(cudaFuncSetAttribute(gather_bulk<512, 32, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 512));
          gather_bulk<512, 32, 4><<<nsm * bpsm, 128, 4 * 32 * 512>>>((char*)buf, didx, nrows, (int*)sink);
        }
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
      }
      CK(cudaGetLastError());
      printf("gather BULK   row=%dB blocks/SM=%d: %.1f GB/s\n", rowb, bpsm, gb / best / 1e6);
    }
    CK(cudaFree(didx));
  }
  return 0;
}
