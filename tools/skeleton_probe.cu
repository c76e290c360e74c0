// Attainable floor of one AlexNet-fc6-sized CER mat-vec call on this GPU (VERDICT r1 "next" #4): the
// window kernel's memory skeleton without its arithmetic, timed like tools/mv_time.py (CUDA graph of
// 16 calls over rotating cold copies, 20 replays).  Same grid as k_matvec (148 CTAs x 896 threads,
// rows split evenly over warps), same byte streams as the encoding:
//   rowPtr u32 (m+1), rowEntry u32 (m+1), colI u16 (nnz), omegaPtr u32 (segs+1), x f32 (n), y f32 (m)
// Variants:
//   0 empty        launch + retire only
//   1 stream       each warp streams its rows' colI and omegaPtr spans (16 B loads), writes y
//   2 chain        1 behind the dependent index chain rowPtr/rowEntry -> spans (as the product kernel)
//   3 chain+x      2 plus x staged into shared memory by one TMA bulk copy per CTA, waited on
//   4 x only       the TMA staging of x alone
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/skeleton_probe tools/skeleton_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <vector>

constexpr int kThreads = 896, kWarps = kThreads / 32;

__device__ __forceinline__ uint4 ld16(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

struct Args {
  const uint32_t *rp, *re, *op;
  const uint16_t *col;
  const float *x;
  float *y;
  int m, n;
};

template <int VAR>
__global__ void __launch_bounds__(kThreads, 1) k_skel(Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
  float *xs = reinterpret_cast<float *>(smem + 16);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (VAR == 0) return;
  if (VAR >= 3) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t bytes = a.n * 4;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
      for (uint32_t o = 0; o < bytes; o += 32768) {
        const uint32_t c = bytes - o < 32768 ? bytes - o : 32768;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(xs) + o),
                     "l"(reinterpret_cast<const char *>(a.x) + o), "r"(c), "r"(smem_u32(bar))
                     : "memory");
      }
    }
  }
  uint32_t acc = 0;
  if (VAR != 4) {
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kWarps, gw = static_cast<uint64_t>(blockIdx.x) * kWarps + wid;
    const uint32_t R0 = gw * a.m / nw, R1 = (gw + 1) * a.m / nw;
    uint32_t e0, e1, s0, s1;
    if (VAR == 1) {  // spans from a closed form (no dependent loads): rows of equal length
      const uint32_t per = a.n / 11;  // ~ AlexNet's 830 entries per row
      e0 = R0 * per;
      e1 = R1 * per;
      s0 = R0 * 125;
      s1 = R1 * 125;
    } else {
      s0 = __ldg(a.rp + R0);
      s1 = __ldg(a.rp + R1);
      e0 = __ldg(a.re + R0);
      e1 = __ldg(a.re + R1);
    }
    // every load of the warp's spans in flight at once (a row of ~830 u16 entries is <= 4 x 512 B per
    // warp; ~125 u32 segment bounds <= 2 x 512 B), then consumed -- the product kernel's access shape
    uint4 c[4], o[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t e = (e0 & ~7u) + lane * 8 + 256u * i;
      c[i] = e < e1 ? ld16(a.col + e) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const uint32_t s = (s0 & ~3u) + lane * 4 + 128u * i;
      o[i] = s < s1 ? ld16(a.op + s) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) acc += c[i].x ^ c[i].y ^ c[i].z ^ c[i].w;
#pragma unroll
    for (int i = 0; i < 2; ++i) acc += o[i].x + o[i].w;
    for (uint32_t e = (e0 & ~7u) + lane * 8 + 1024u; e < e1; e += 256) acc += ld16(a.col + e).x;  // longer rows
  }
  if (VAR >= 3) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok)
                   : "r"(smem_u32(bar))
                   : "memory");
    acc += __float_as_uint(xs[(lane * 97 + wid) % a.n]);
  }
  if (VAR != 4) {
    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kWarps, gw = static_cast<uint64_t>(blockIdx.x) * kWarps + wid;
    const uint32_t R0 = gw * a.m / nw;
    if (lane == 0 && R0 < static_cast<uint32_t>(a.m)) a.y[R0] = static_cast<float>(acc & 1);
  } else if (threadIdx.x == 0) {
    a.y[blockIdx.x] = xs[blockIdx.x];
  }
}

int main() {
  const int m = 4096, n = 9216;
  const size_t nnz = 3395269, segs = 514338;
  const int copies = 16;
  std::vector<uint32_t> rp(m + 1), re(m + 1);
  for (int r = 0; r <= m; ++r) {
    rp[r] = static_cast<uint32_t>(static_cast<uint64_t>(segs) * r / m);
    re[r] = static_cast<uint32_t>(static_cast<uint64_t>(nnz) * r / m);
  }
  std::vector<Args> args(copies);
  for (int c = 0; c < copies; ++c) {
    Args &a = args[c];
    uint32_t *d_rp, *d_re, *d_op;
    uint16_t *d_col;
    float *d_x, *d_y;
    cudaMalloc(&d_rp, 4 * (m + 1));
    cudaMalloc(&d_re, 4 * (m + 1));
    cudaMalloc(&d_op, 4 * (segs + 16));
    cudaMalloc(&d_col, 2 * (nnz + 16));
    cudaMalloc(&d_x, 4 * n);
    cudaMalloc(&d_y, 4 * m);
    cudaMemcpy(d_rp, rp.data(), 4 * (m + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(d_re, re.data(), 4 * (m + 1), cudaMemcpyHostToDevice);
    cudaMemset(d_op, 1, 4 * (segs + 16));
    cudaMemset(d_col, 1, 2 * (nnz + 16));
    cudaMemset(d_x, 0, 4 * n);
    a = Args{d_rp, d_re, d_op, d_col, d_x, d_y, m, n};
  }
  const size_t smem = 16 + 4 * n;
  auto run = [&](auto kern, const char *name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int c = 0; c < copies; ++c) kern<<<148, kThreads, smem, st>>>(args[c]);
    cudaStreamSynchronize(st);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int c = 0; c < copies; ++c) kern<<<148, kThreads, smem, st>>>(args[c]);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 20;
    cudaEventRecord(e0, st);
    for (int i = 0; i < reps; ++i) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / (reps * copies);
    const double bytes = 2.0 * nnz + 4.0 * (segs + 1) + 8.0 * (m + 1) + 4.0 * n + 4.0 * m;
    printf("{\"variant\": \"%s\", \"us_per_call\": %.3f, \"gbs_of_cer_bytes\": %.1f, \"err\": \"%s\"}\n", name, us,
           bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  run(k_skel<0>, "empty");
  run(k_skel<1>, "stream");
  run(k_skel<2>, "chain");
  run(k_skel<3>, "chain+x");
  run(k_skel<4>, "x only");
  return 0;
}
