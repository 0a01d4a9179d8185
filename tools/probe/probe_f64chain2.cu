// Microbenchmark 2: the fp32-path score loop as the decode kernel runs it
// (LDS.128 of 4 fp32 K elements, q as fp64 double2 broadcast, sequential fp64
// chain), conversion by F2F, by integer bit assembly, or none (K pre-widened
// to fp64, the bound), at 3/6/12/16 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>  // 0 F2F, 1 int, 2 fp64 K
__global__ void chain(double* out, long long* cyc, int iters) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* qs = reinterpret_cast<double*>(smem);              // 128 fp64
  float* ks = reinterpret_cast<float*>(smem + 1024);         // 32 rows x 128 fp32 (row stride 132 floats)
  double* kd = reinterpret_cast<double*>(smem + 1024 + 32 * 132 * 4);  // 32 x 128 fp64 (stride 130)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128; i += blockDim.x) qs[i] = 1.0 + i * 1e-3;
  for (int i = threadIdx.x; i < 32 * 132; i += blockDim.x) ks[i] = 0.5f + (i & 7);
  for (int i = threadIdx.x; i < 32 * 130; i += blockDim.x) kd[i] = 0.25 + (i & 3);
  __syncthreads();
  long long t0 = clock64();
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const float* kr = ks + lane * 132;
    const double* kdr = kd + lane * 130;
#pragma unroll 2
    for (int c0 = 0; c0 < 32; c0 += 4) {
      double k[16];
      if (MODE == 2) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double2 v = *reinterpret_cast<const double2*>(kdr + c0 * 4 + 2 * u);
          k[2 * u] = v.x; k[2 * u + 1] = v.y;
        }
      } else {
        float4 kv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) kv[u] = *reinterpret_cast<const float4*>(kr + (c0 + u) * 4);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float f[4] = {kv[u].x, kv[u].y, kv[u].z, kv[u].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (MODE == 0) {
              k[4 * u + e] = (double)f[e];
            } else {
              const unsigned x = __float_as_uint(f[e]);
              const unsigned hi = (x & 0x80000000u) | (((x & 0x7fffffffu) >> 3) + 0x38000000u);
              k[4 * u + e] = __hiloint2double((int)hi, (int)(x << 29));
            }
          }
        }
      }
      const double* qg = qs + c0 * 4;
#pragma unroll
      for (int e = 0; e < 16; e += 2) {
        const double2 qq = *reinterpret_cast<const double2*>(qg + e);
        acc = fma(qq.x, k[e], acc);
        acc = fma(qq.y, k[e + 1], acc);
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lane == 0) cyc[blockIdx.x * 32 + w] = t1 - t0;
}
template <int MODE>
void run(int warps, double* out, long long* cyc) {
  const int iters = 8, smem = 1024 + 32 * 132 * 4 + 32 * 130 * 8;
  cudaFuncSetAttribute(chain<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  chain<MODE><<<148, warps * 32, smem>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  chain<MODE><<<148, warps * 32, smem>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[148 * 32];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int b = 0; b < 148; ++b) for (int w = 0; w < warps; ++w) m += h[b * 32 + w];
  m /= 148.0 * warps;
  const double per = m / iters;
  printf("mode %-4s warps/SM %2d: %5.0f cycles per 128-element row chain per warp (%.1f/elem); SM: %.3f warp-elem/clk\n",
         MODE == 0 ? "F2F" : (MODE == 1 ? "int" : "f64"), warps, per, per / 128, warps * 128 / per);
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 148 * 32 * 8);
  for (int w : {1, 3, 6, 8, 12, 16}) { run<0>(w, out, cyc); run<1>(w, out, cyc); run<2>(w, out, cyc); }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
