// Standalone check of the tcgen05 descriptors in hgca_umma.cuh (run on a B200):
//   D[128 x N] = A[128 x K] . B  with A K-major and B either K-major ([N][K]) or
//   MN-major ([K][N]), bf16 in, fp32 out, 128-byte-swizzled shared-memory tiles
//   (the layout TMA SWIZZLE_128B boxes of 64 bf16 produce). Compared on the host
//   with an fp64 reference; for MN-major B a few (LBO, SBO) encodings are tried.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_2507_03153_b200/csrc/hgca_common.cuh"
#include "../../paper_2507_03153_b200/csrc/hgca_umma.cuh"

using namespace hgca;
constexpr int M = 128, N = 128, K = 128;

// byte offset of element (r, c) in a [rows][64-element atom] SW128 tile with
// atoms along the contiguous dimension: atom a = c / 64 at a * rows * 128
__host__ __device__ inline uint32_t sw128_off(int r, int c, int rows) {
  const int a = c / 64, cc = c % 64;
  const int chunk = (cc * 2) / 16, within = (cc * 2) % 16;
  return a * rows * 128 + (r / 8) * 1024 + (r % 8) * 128 + ((chunk ^ (r % 8)) * 16) + within;
}

// bmn: B stored MN-major ([K][N], N contiguous) -> smem [K rows][N atoms]; lbo/sbo for B's descriptor
__global__ void umma_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int bmn, uint32_t b_lbo,
                            uint32_t b_sbo, uint32_t b_katom_step) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sa = sm;              // A: [M rows][K] K-major SW128, 2 atoms
  unsigned char* sb = sm + M * K * 2;  // B
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, c = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sa + sw128_off(r, c, M)) = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    if (!bmn) {  // B[n][k]: rows n, contiguous k
      const int n = i / K, k = i % K;
      *reinterpret_cast<__nv_bfloat16*>(sb + sw128_off(n, k, N)) = B[i];
    } else {  // B[k][n]: rows k, contiguous n
      const int k = i / N, n = i % N;
      *reinterpret_cast<__nv_bfloat16*>(sb + sw128_off(k, n, K)) = B[i];
    }
  }
  umma::fence_smem_async();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) umma::tmem_alloc<128>(smem_u32(&tbase));
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t idesc = umma::idesc_bf16_f32(M, N, false, bmn != 0);
    for (int k = 0; k < K / 16; ++k) {
      // A: K-major, atom k/4, 32 bytes per k-step inside the 128-byte row
      const uint64_t ad = umma::smem_desc(smem_u32(sa) + (k / 4) * M * 128 + (k % 4) * 32, 16, 1024);
      uint64_t bd;
      if (!bmn)
        bd = umma::smem_desc(smem_u32(sb) + (k / 4) * N * 128 + (k % 4) * 32, 16, 1024);
      else  // MN-major: k-step of 16 rows = 2 swizzle atoms of 8 rows
        bd = umma::smem_desc(smem_u32(sb) + k * b_katom_step, b_lbo, b_sbo);
      umma::mma_bf16(tmem, ad, bd, idesc, k > 0);
    }
    umma::commit(smem_u32(&bar));
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  umma::fence_after_sync();
  // warp w reads rows 32w..32w+31 (TMEM lanes), 16 columns at a time
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    umma::ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
    umma::ld_wait();
    const int row = warp * 32 + (tid & 31);
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(r[j]);
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc<128>(tmem);
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  std::vector<__nv_bfloat16> hA(M * K), hBk(N * K), hBm(K * N);
  std::vector<float> fA(M * K), fB(K * N);  // fB[k][n]
  srand(1);
  for (int i = 0; i < M * K; ++i) { fA[i] = bf((rand() / (float)RAND_MAX) - 0.5f); hA[i] = __float2bfloat16(fA[i]); }
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) {
      const float v = bf((rand() / (float)RAND_MAX) - 0.5f);
      fB[k * N + n] = v;
      hBm[k * N + n] = __float2bfloat16(v);
      hBk[n * K + k] = __float2bfloat16(v);
    }
  std::vector<double> ref(M * N, 0.0);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)fA[m * K + k] * fB[k * N + n];
      ref[m * N + n] = s;
    }
  __nv_bfloat16 *dA, *dBk, *dBm;
  float* dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dBk, N * K * 2); cudaMalloc(&dBm, N * K * 2); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dBk, hBk.data(), N * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dBm, hBm.data(), N * K * 2, cudaMemcpyHostToDevice);
  const int smem = (M * K + N * K) * 2 + 1024;
  cudaFuncSetAttribute(umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  auto run = [&](const char* name, int bmn, uint32_t lbo, uint32_t sbo, uint32_t kstep) {
    cudaMemset(dD, 0, M * N * 4);
    umma_kernel<<<1, 128, smem>>>(dA, bmn ? dBm : dBk, dD, bmn, lbo, sbo, kstep);
    const cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> hD(M * N);
    cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0, mag = 0;
    for (int i = 0; i < M * N; ++i) { err = fmax(err, fabs(hD[i] - ref[i])); mag = fmax(mag, fabs(ref[i])); }
    printf("%-44s %s  max|err| %.3e (max|ref| %.2f)%s\n", name, cudaGetErrorString(e), err, mag,
           err < 1e-3 * mag ? "  MATCH" : "");
    return e == cudaSuccess;
  };
  if (!run("K-major A, K-major B", 0, 16, 1024, 0)) return 1;
  // MN-major B: smem [K rows][N atoms of 64]; one 16-row k-step = 2 8-row groups = 2048 bytes
  const uint32_t atom = K * 128;  // bytes between the two 64-wide N atoms
  const uint32_t cand[][3] = {{atom, 1024, 2048}, {1024, atom, 2048}, {atom, 2048, 2048}, {2048, atom, 2048}};
  for (auto& c : cand) {
    char name[96];
    snprintf(name, sizeof name, "MN-major B lbo=%u sbo=%u kstep=%u", c[0], c[1], c[2]);
    if (!run(name, 1, c[0], c[1], c[2])) return 1;
  }
  return 0;
}
