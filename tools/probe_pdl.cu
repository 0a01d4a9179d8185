// Floor of the decode step's launch structure on B200: per-step time of a
// chain of (persistent 1-CTA-per-SM kernel -> small merge-like kernel) pairs,
// captured into one CUDA graph, with and without programmatic dependent
// launch, vs a chain of persistent kernels alone. The kernels do no work
// beyond one dependent global write/read, so the numbers are the structural
// cost per step (launch, grid drain, memory flush, CTA rasterisation).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/probe_pdl tools/probe_pdl.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void big_kernel(int* buf, int pdl) {
  extern __shared__ unsigned char sm[];
  if (pdl) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (threadIdx.x == 0) {
    sm[0] = (unsigned char)buf[blockIdx.x];
    buf[blockIdx.x] = sm[0] + 1;
  }
}

__global__ void small_kernel(int* buf, int pdl) {
  extern __shared__ unsigned char sm[];
  if (pdl) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (threadIdx.x == 0) {
    sm[0] = (unsigned char)buf[blockIdx.x % 148];
    buf[148 + blockIdx.x] = sm[0];
  }
}

static void launch(void (*k)(int*, int), int grid, int block, int smem, cudaStream_t s, int* buf, int pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, buf, pdl);
}

static float run(int mode, int pdl, int small_grid, int steps) {
  int* buf;
  cudaMalloc(&buf, 8192 * 4);
  cudaMemset(buf, 0, 8192 * 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < steps; ++i) {
    launch(big_kernel, 148, 384, 200 * 1024, s, buf, pdl);
    if (mode == 1) launch(small_kernel, small_grid, 128, 50 * 1024, s, buf, pdl);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaFree(buf);
  cudaStreamDestroy(s);
  return ms * 1e3f / (5 * steps);
}

int main() {
  cudaFuncSetAttribute(big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  const int steps = 200;
  printf("persistent kernel alone, no PDL : %.2f us/step\n", run(0, 0, 0, steps));
  printf("persistent kernel alone, PDL    : %.2f us/step\n", run(0, 1, 0, steps));
  for (int sg : {32, 128, 512}) {
    printf("pair (merge grid %3d), no PDL   : %.2f us/step\n", sg, run(1, 0, sg, steps));
    printf("pair (merge grid %3d), PDL      : %.2f us/step\n", sg, run(1, 1, sg, steps));
  }
  return 0;
}
