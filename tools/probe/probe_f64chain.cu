// Microbenchmark: the fp32-path score loop (lane = row, 128-element sequential
// fp64 chain over fp32 K converted with F2F, q in fp64 from smem) at several
// warps per SM and rows per lane (ILP), plus the bare DFMA chain latency.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP, bool CVT_INT>
__global__ void chain(const float* __restrict__ k, double* out, long long* cyc, int iters) {
  __shared__ float ks[4 * 32][65];
  __shared__ double qs[128];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128; i += blockDim.x) qs[i] = 1.0 + i * 1e-3;
  for (int r = 0; r < ILP; ++r)
    for (int c = 0; c < 128; ++c) if (w == 0) ks[r * 32 + lane][c & 63] = k[(r * 32 + lane) * 128 + c];
  __syncthreads();
  long long t0 = clock64();
  double acc[ILP];
  for (int r = 0; r < ILP; ++r) acc[r] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int c = 0; c < 128; ++c) {
      const double q = qs[c];
#pragma unroll
      for (int r = 0; r < ILP; ++r) {
        const float kf = ks[r * 32 + lane][c & 63];
        double kd;
        if (CVT_INT) {
          const unsigned x = __float_as_uint(kf);
          const unsigned hi = (x & 0x80000000u) | (((x & 0x7fffffffu) >> 3) + 0x38000000u);
          kd = __hiloint2double((int)hi, (int)(x << 29));
        } else {
          kd = (double)kf;
        }
        acc[r] = fma(q, kd, acc[r]);
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int r = 0; r < ILP; ++r) s += acc[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (lane == 0) cyc[blockIdx.x * 16 + w] = t1 - t0;
}
__global__ void dfma_lat(double* out, long long* cyc, double a, double b) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int ILP, bool CI>
void run(int warps, const float* k, double* out, long long* cyc) {
  const int iters = 4;
  chain<ILP, CI><<<148, warps * 32>>>(k, out, cyc, iters);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chain<ILP, CI><<<148, warps * 32>>>(k, out, cyc, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  long long h[148 * 16];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int b = 0; b < 148; ++b) for (int w = 0; w < warps; ++w) m += h[b * 16 + w];
  m /= 148.0 * warps;
  printf("warps/SM %2d ILP %d cvt %s: %.0f cycles per 128-element chain (per warp), %.1f cycles/element-row\n", warps, ILP,
         CI ? "int" : "F2F", m / iters, m / iters / 128 / ILP);
}
int main() {
  float* k; double* out; long long* cyc;
  cudaMalloc(&k, 128 * 128 * 4); cudaMemset(k, 0, 128 * 128 * 4);
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 148 * 16 * 8);
  dfma_lat<<<1, 32>>>(out, cyc, 1.0, 0.999);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent DFMA latency: %.1f cycles\n", c / 1024.0);
  for (int w : {1, 3, 6, 12}) { run<1, false>(w, k, out, cyc); run<2, false>(w, k, out, cyc); run<1, true>(w, k, out, cyc); run<2, true>(w, k, out, cyc); }
  run<4, false>(3, k, out, cyc); run<4, true>(3, k, out, cyc);
  return 0;
}
