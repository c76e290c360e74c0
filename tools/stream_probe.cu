// Streaming micro-benchmark: per-warp contiguous 2 KB windows (what k_matvec's colI stream looks like).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_probe tools/stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int FLAVOR>
__device__ __forceinline__ uint4 ld(const uint4 *p) {
  uint4 r;
  if (FLAVOR == 0) {
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  } else if (FLAVOR == 1) {
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  } else if (FLAVOR == 2) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  } else {
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  }
  return r;
}

// each warp: contiguous [w*per_warp, (w+1)*per_warp) uint4s; window = 32 lanes x NV uint4; DEPTH windows in flight
template <int FLAVOR, int NV, int WORK>
__global__ void __launch_bounds__(512) stream(const uint4 *__restrict__ src, size_t per_warp, unsigned *out) {
  const int lane = threadIdx.x & 31;
  const size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const uint4 *p = src + w * per_warp;
  unsigned acc = 0;
  uint4 a[NV], b[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) a[v] = ld<FLAVOR>(p + lane * NV + v);
  for (size_t base = 0; base < per_warp; base += 64 * NV) {
#pragma unroll
    for (int v = 0; v < NV; ++v) b[v] = (base + 32 * NV < per_warp) ? ld<FLAVOR>(p + base + 32 * NV + lane * NV + v) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int v = 0; v < NV; ++v) acc ^= a[v].x + a[v].y * 3 + a[v].z * 5 + a[v].w;
    for (int i = 0; i < WORK; ++i) acc = acc * 1664525u + __shfl_xor_sync(0xffffffffu, acc, 1);
#pragma unroll
    for (int v = 0; v < NV; ++v) a[v] = (base + 64 * NV < per_warp) ? ld<FLAVOR>(p + base + 64 * NV + lane * NV + v) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int v = 0; v < NV; ++v) acc ^= b[v].x + b[v].y * 3 + b[v].z * 5 + b[v].w;
    for (int i = 0; i < WORK; ++i) acc = acc * 1664525u + __shfl_xor_sync(0xffffffffu, acc, 1);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int FLAVOR, int NV, int WORK>
void run(const char *name, uint4 *d, size_t bytes, int blocks_per_sm, int threads, unsigned *out) {
  const int sms = 148;
  const size_t warps = (size_t)sms * blocks_per_sm * threads / 32;
  const size_t per_warp = (bytes / 16 / warps) / (64 * NV) * (64 * NV);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  for (int i = 0; i < 3; ++i) stream<FLAVOR, NV, WORK><<<sms * blocks_per_sm, threads>>>(d, per_warp, out);
  cudaEventRecord(s);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) stream<FLAVOR, NV, WORK><<<sms * blocks_per_sm, threads>>>(d, per_warp, out);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  const double moved = (double)per_warp * 16 * warps;
  printf("%-28s warps/SM=%3d NV=%d work=%3d  %8.1f GB/s\n", name, blocks_per_sm * threads / 32, NV, WORK,
         moved * reps / (ms * 1e-3) / 1e9);
}

int main() {
  const size_t bytes = size_t(1) << 30;
  uint4 *d;
  unsigned *out;
  cudaMalloc(&d, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(d, 1, bytes);
  for (int bps : {1, 2, 4}) {
    run<0, 4, 0>("ld.global", d, bytes, bps, 512, out);
    run<1, 4, 0>("ld.global.nc", d, bytes, bps, 512, out);
    run<2, 4, 0>("ld.nc.noalloc.L2::256B", d, bytes, bps, 512, out);
    run<3, 4, 0>("ld.global.cs", d, bytes, bps, 512, out);
    run<2, 4, 64>("nc.noalloc+work64", d, bytes, bps, 512, out);
    run<2, 4, 256>("nc.noalloc+work256", d, bytes, bps, 512, out);
    run<2, 2, 0>("nc.noalloc NV=2", d, bytes, bps, 512, out);
    run<2, 8, 0>("nc.noalloc NV=8", d, bytes, bps, 512, out);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
