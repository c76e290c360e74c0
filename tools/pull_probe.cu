// Isolates the fused host-I/O prologue: 148 CTAs each pull a 1/148 slice of a 36 KB host vector
// (mapped pinned memory) into device memory, optionally followed by a flag-based grid-wide arrival.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>  // 0: plain loads, 1: ld.cv loads, 2: plain + flag barrier, 3: ld.cv + barrier
__global__ void k_pull(const float4 *xh, float4 *xd, int n4, unsigned long long *flags, unsigned long long epoch) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const int per = (n4 + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per, i1 = min(n4, i0 + per);
  for (int i = i0 + lane; i < i1; i += 32) xd[i] = (MODE & 1) ? __ldcv(xh + i) : xh[i];
  if (MODE >= 2) {
    __threadfence();
    __syncwarp();
    if (lane == 0) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags + blockIdx.x), "l"(epoch) : "memory");
    bool ok;
    do {
      ok = true;
      for (unsigned b = lane; b < gridDim.x; b += 32) {
        unsigned long long f;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(flags + b) : "memory");
        ok = ok && f == epoch;
      }
    } while (!__all_sync(0xffffffffu, ok));
  }
}
__global__ void k_empty() {}

template <typename F>
double per_call_us(F f, int reps = 1000) {
  for (int i = 0; i < 20; ++i) f();
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) f();
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

int main() {
  const int n = 9216;
  float *hx, *dx;
  unsigned long long *flags;
  cudaHostAlloc(&hx, n * 4, cudaHostAllocMapped);
  cudaMalloc(&dx, n * 4);
  cudaMalloc(&flags, 4096);
  cudaMemset(flags, 0, 4096);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  unsigned long long ep = 1;
  printf("empty 148x896 + sync     %6.2f us\n", per_call_us([&] { k_empty<<<148, 896, 0, s>>>(); cudaStreamSynchronize(s); }));
  printf("pull plain  + sync       %6.2f us\n", per_call_us([&] { k_pull<0><<<148, 896, 0, s>>>((const float4 *)hx, (float4 *)dx, n / 4, flags, ++ep); cudaStreamSynchronize(s); }));
  printf("pull ld.cv  + sync       %6.2f us\n", per_call_us([&] { k_pull<1><<<148, 896, 0, s>>>((const float4 *)hx, (float4 *)dx, n / 4, flags, ++ep); cudaStreamSynchronize(s); }));
  printf("pull plain + barrier     %6.2f us\n", per_call_us([&] { k_pull<2><<<148, 896, 0, s>>>((const float4 *)hx, (float4 *)dx, n / 4, flags, ++ep); cudaStreamSynchronize(s); }));
  printf("pull ld.cv + barrier     %6.2f us\n", per_call_us([&] { k_pull<3><<<148, 896, 0, s>>>((const float4 *)hx, (float4 *)dx, n / 4, flags, ++ep); cudaStreamSynchronize(s); }));
  for (int g : {8, 16, 37, 74}) {
    printf("pull plain %3d CTAs+barr %6.2f us\n", g, per_call_us([&] { k_pull<2><<<g, 896, 0, s>>>((const float4 *)hx, (float4 *)dx, n / 4, flags, ++ep); cudaStreamSynchronize(s); }));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
