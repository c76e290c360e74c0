// Does programmatic dependent launch overlap consecutive kernels (stream and CUDA graph)?
#include <cstdio>
#include <cuda_runtime.h>

__device__ void spin(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}
// pre: independent prologue (before griddepcontrol.wait); post: dependent work
__global__ void k(long long pre, long long post, int *sink) {
  asm volatile("griddepcontrol.launch_dependents;");
  spin(pre);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  spin(post);
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(sink, 1);
}

static void launch(bool pdl, long long pre, long long post, int *sink, cudaStream_t st, int ctas, int threads,
                   size_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, pre, post, sink);
}

int main() {
  int *sink;
  cudaMalloc(&sink, 4);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 50;
  struct Cfg { int threads; size_t smem; const char *name; } cfgs[] = {
      {512, 0, "512 thr, no smem (co-resident)"}, {512, 120 * 1024, "512 thr, 120 KB smem (exclusive)"}};
  for (auto c : cfgs)
    for (long long pre : {0LL, 4000LL})
      for (int pdl = 0; pdl < 2; ++pdl) {
        const long long post = 4000;
        for (int i = 0; i < 5; ++i) launch(pdl, pre, post, sink, st, 148, c.threads, c.smem);
        cudaEventRecord(a, st);
        for (int i = 0; i < N; ++i) launch(pdl, pre, post, sink, st, 148, c.threads, c.smem);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        // graph
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < N; ++i) launch(pdl, pre, post, sink, st, 148, c.threads, c.smem);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        cudaEventRecord(a, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float gms;
        cudaEventElapsedTime(&gms, a, b);
        printf("%-34s pre=%5lld post=%lld pdl=%d : stream %6.2f us/kernel, graph %6.2f us/kernel\n", c.name, pre, post,
               pdl, ms * 1e3 / N, gms * 1e3 / N);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
