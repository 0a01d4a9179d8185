// Latency of dependent fp64 chains on B200 (decides the fp32 decode kernel's
// score-loop structure): one warp, a chain of N DFMA (s = fma(q, k, s)) with k
// converted from fp32, vs 2 and 4 interleaved chains; also the F2F.F64.F32
// conversion inside the chain. Prints cycles per chain element.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chain(const float* k, const double* q, double* out, long long* cyc, int n) {
  double s[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) s[c] = 0.0;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; i += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double qq = q[(i + u) & 127];
#pragma unroll
      for (int c = 0; c < CH; ++c) s[c] = fma(qq, (double)k[((i + u) & 127) + c * 128 + threadIdx.x * 512], s[c]);
    }
  }
  long long t1 = clock64();
  double r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r += s[c];
  out[threadIdx.x] = r;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void chain_pure(double* out, long long* cyc, int n, double a) {
  double s = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) s = fma(s, a, 1.0);
  long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* k; double *q, *out; long long* cyc;
  cudaMalloc(&k, 32 * 512 * 4 * 4); cudaMalloc(&q, 128 * 8); cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 8);
  cudaMemset(k, 0, 32 * 512 * 16); cudaMemset(q, 0, 128 * 8);
  long long h;
  const int n = 4096;
  chain_pure<<<1, 32>>>(out, cyc, n, 0.999); cudaDeviceSynchronize();
  chain_pure<<<1, 32>>>(out, cyc, n, 0.999); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("pure DFMA chain: %.2f cycles/op\n", (double)h / n);
  chain<1><<<1, 32>>>(k, q, out, cyc, n); cudaDeviceSynchronize();
  chain<1><<<1, 32>>>(k, q, out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("1 chain (ld f32 + cvt + ld q + DFMA): %.2f cycles/elem\n", (double)h / n);
  chain<2><<<1, 32>>>(k, q, out, cyc, n); cudaDeviceSynchronize();
  chain<2><<<1, 32>>>(k, q, out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("2 chains: %.2f cycles/elem-step\n", (double)h / n);
  chain<4><<<1, 32>>>(k, q, out, cyc, n); cudaDeviceSynchronize();
  chain<4><<<1, 32>>>(k, q, out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("4 chains: %.2f cycles/elem-step\n", (double)h / n);
  return 0;
}
