// Do SHFL and LDS share a throughput limit on B200?  Per-SM issue of conflict-free LDS.32, SHFL.IDX, and
// both interleaved (32 warps per SM, dependent-free streams), in instructions per clock per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mio_probe tools/mio_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(1024) k(float *out, int iters) {
  __shared__ float s[1024 * 4];
  const int t = threadIdx.x, lane = t & 31;
  for (int i = t; i < 4096; i += 1024) s[i] = i;
  __syncthreads();
  float a0 = 0, a1 = 0, a2 = 0, a3 = 0, v = t;
  int idx = (lane * 5) & 31;
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0 || MODE == 2) {
      a0 += s[(t + i) & 4095]; a1 += s[(t + i + 1024) & 4095]; a2 += s[(t + i + 2048) & 4095]; a3 += s[(t + i + 3072) & 4095];
    }
    if (MODE == 1 || MODE == 2) {
      a0 += __shfl_sync(0xffffffffu, v + a0, idx); a1 += __shfl_sync(0xffffffffu, v + a1, idx ^ 1);
      a2 += __shfl_sync(0xffffffffu, v + a2, idx ^ 2); a3 += __shfl_sync(0xffffffffu, v + a3, idx ^ 3);
    }
  }
  out[blockIdx.x * 1024 + t] = a0 + a1 + a2 + a3;
}
int main() {
  float *out; cudaMalloc(&out, 148 * 1024 * 4);
  int sms = 148, iters = 4096;
  auto run = [&](auto kern, const char *name, int ops) {
    kern<<<sms, 1024>>>(out, 16); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); kern<<<sms, 1024>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_instr = 32.0 * iters * ops;  // per SM
    double clk = ms * 1e-3 * 1.965e9;
    printf("%-14s %.3f ms  %.2f warp-instr/clk/SM\n", name, ms, warp_instr / clk);
  };
  run(k<0>, "lds x4", 4);
  run(k<1>, "shfl x4", 4);
  run(k<2>, "lds+shfl x8", 8);
  return 0;
}
