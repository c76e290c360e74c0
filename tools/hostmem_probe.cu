// Host-memory access latencies on the GPU box: copy engine vs zero-copy (mapped pinned) kernel reads/writes.
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>

__global__ void k_empty() {}
// CTA-cooperative 16 B loads of n floats from (mapped host) src into dst
__global__ void k_pull(const float4 *__restrict__ src, float4 *__restrict__ dst, int n4) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
// every CTA reads the whole vector (the mat-vec's x staging pattern) from src
__global__ void k_bcast(const float4 *__restrict__ src, float *out, int n4) {
  float acc = 0.f;
  for (int i = threadIdx.x; i < n4; i += blockDim.x) { float4 v = src[i]; acc += v.x + v.y + v.z + v.w; }
  if (acc == 12345.f) out[blockIdx.x] = acc;
}
__global__ void k_push(const float4 *__restrict__ src, float4 *__restrict__ dst, int n4) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

template <typename F>
double per_call_us(F f, int reps = 2000) {
  for (int i = 0; i < 50; ++i) f();
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) f();
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

int main() {
  const int n = 9216, m = 4096;
  float *hx, *hy, *dx, *dy, *dxh, *dyh, *scratch;
  cudaHostAlloc(&hx, n * 4, cudaHostAllocMapped);
  cudaHostAlloc(&hy, m * 4, cudaHostAllocMapped);
  cudaHostGetDevicePointer(&dxh, hx, 0);
  cudaHostGetDevicePointer(&dyh, hy, 0);
  cudaMalloc(&dx, n * 4);
  cudaMalloc(&dy, m * 4);
  cudaMalloc(&scratch, 4096);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  printf("sync only              %6.2f us\n", per_call_us([&] { cudaStreamSynchronize(s); }));
  printf("empty kernel + sync    %6.2f us\n", per_call_us([&] { k_empty<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }));
  printf("H2D 36KB memcpy + sync %6.2f us\n", per_call_us([&] { cudaMemcpyAsync(dx, hx, n * 4, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s); }));
  printf("D2H 16KB memcpy + sync %6.2f us\n", per_call_us([&] { cudaMemcpyAsync(hy, dy, m * 4, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }));
  printf("H2D+D2H memcpy + sync  %6.2f us\n", per_call_us([&] { cudaMemcpyAsync(dx, hx, n * 4, cudaMemcpyHostToDevice, s); cudaMemcpyAsync(hy, dy, m * 4, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s); }));
  for (int g : {1, 4, 16}) {
    printf("pull 36KB %2d CTAs+sync %6.2f us\n", g, per_call_us([&] { k_pull<<<g, 512, 0, s>>>((const float4 *)dxh, (float4 *)dx, n / 4); cudaStreamSynchronize(s); }));
  }
  printf("bcast 36KB 148 CTAs    %6.2f us\n", per_call_us([&] { k_bcast<<<148, 896, 0, s>>>((const float4 *)dxh, scratch, n / 4); cudaStreamSynchronize(s); }));
  for (int g : {1, 4, 16}) {
    printf("push 16KB %2d CTAs+sync %6.2f us\n", g, per_call_us([&] { k_push<<<g, 512, 0, s>>>((const float4 *)dy, (float4 *)dyh, m / 4); cudaStreamSynchronize(s); }));
  }
  printf("pull+push kernels+sync %6.2f us\n", per_call_us([&] { k_pull<<<4, 512, 0, s>>>((const float4 *)dxh, (float4 *)dx, n / 4); k_push<<<4, 512, 0, s>>>((const float4 *)dy, (float4 *)dyh, m / 4); cudaStreamSynchronize(s); }));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
