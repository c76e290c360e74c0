// L2 -> SM bandwidth probe: repeated reads of an L2-resident buffer (contiguous and random 512 B rows).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void contig(const float4 *__restrict__ src, size_t n4, int iters, float *out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      float4 v = __ldg(src + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 1234.5f) out[0] = acc;
}

// each warp gathers random rows of ROWB bytes (lanes read consecutive float4s)
template <int V>
__global__ void gather(const float *__restrict__ X, int nrows, int ldx, const int *__restrict__ idx, int nidx,
                       float *out) {
  const int lane = threadIdx.x & 31;
  const size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (size_t i = w; i < (size_t)nidx; i += nw) {
    const float *r = X + (size_t)idx[i] * ldx + lane * V;
    if (V == 4) {
      float4 v = __ldg(reinterpret_cast<const float4 *>(r));
      acc += v.x + v.y + v.z + v.w;
    } else {
      float2 v = __ldg(reinterpret_cast<const float2 *>(r));
      acc += v.x + v.y;
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  float *out;
  cudaMalloc(&out, 4);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  for (size_t mb : {16, 48, 96}) {
    const size_t bytes = mb << 20;
    float4 *buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    contig<<<148 * 8, 512>>>(buf, bytes / 16, 2, out);
    cudaEventRecord(s);
    const int iters = 20;
    contig<<<148 * 8, 512>>>(buf, bytes / 16, iters, out);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    printf("contig %3zu MB resident: %8.1f GB/s\n", mb, (double)bytes * iters / (ms * 1e-3) / 1e9);
    cudaFree(buf);
  }
  // random row gathers: X = 9216 x 64 (B=64) and 25088 x 128 (B=128)
  for (int cfg = 0; cfg < 2; ++cfg) {
    const int nrows = cfg ? 25088 : 9216, ld = cfg ? 128 : 64;
    float *X;
    cudaMalloc(&X, (size_t)nrows * ld * 4);
    cudaMemset(X, 0, (size_t)nrows * ld * 4);
    const int nidx = 4 << 20;
    int *h = new int[nidx];
    uint32_t st = 12345;
    for (int i = 0; i < nidx; ++i) { st = st * 1664525u + 1013904223u; h[i] = st % nrows; }
    int *idx;
    cudaMalloc(&idx, nidx * 4);
    cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice);
    for (int bps : {4, 8}) {
      if (cfg) gather<4><<<148 * bps, 256>>>(X, nrows, ld, idx, nidx, out);
      else gather<2><<<148 * bps, 256>>>(X, nrows, ld, idx, nidx, out);
      cudaEventRecord(s);
      for (int r = 0; r < 5; ++r) {
        if (cfg) gather<4><<<148 * bps, 256>>>(X, nrows, ld, idx, nidx, out);
        else gather<2><<<148 * bps, 256>>>(X, nrows, ld, idx, nidx, out);
      }
      cudaEventRecord(e);
      cudaEventSynchronize(e);
      float ms;
      cudaEventElapsedTime(&ms, s, e);
      printf("gather rows of %d B (X %d x %d), %d CTAs/SM: %8.1f GB/s\n", ld * 4, nrows, ld, bps * 2,
             (double)nidx * ld * 4 * 5 / (ms * 1e-3) / 1e9);
    }
    cudaFree(X);
    cudaFree(idx);
    delete[] h;
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
