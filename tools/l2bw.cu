// L2 -> SM read-bandwidth microbenchmark (the denominator of bench.py's L2 roofline, VERDICT r01
// item 2).  A table that fits in L2 (default 32 MiB of the 126 MB) is read repeatedly by a persistent
// grid after a warm-up pass, three ways:
//   stream : ld.global.cg.v4 (16 B per thread), 4 independent loads in flight per thread;
//   gather : the hot kernels' pattern - each warp copies whole 512-byte rows picked by a hash of
//            (warp, iteration) with cp.async.cg 16 B per lane into a shared-memory ring (4 rows per
//            stage, 2 stages), one commit group per stage, at 4..12 resident CTAs of 4 warps per SM.
// Prints one JSON object per mode: bytes read / CUDA-event time, best of `reps` launches, next to the
// SM-ingress figure 64 B/clk/SM x SMs x the current SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2bw tools/l2bw.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__global__ void __launch_bounds__(256) stream_rd(const uint4* __restrict__ p, int64_t n16, int passes, uint32_t* sink) {
  uint32_t x = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < passes; ++r)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += 4 * stride) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = i + u * stride;
        if (j < n16)
          asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + j));
        else
          v[u] = make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) x ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
  if (x == 0x12345678u) sink[0] = x;  // keeps the loads alive
}

__device__ __forceinline__ uint32_t hash32(uint32_t a) {
  a ^= a >> 16; a *= 0x7feb352dU; a ^= a >> 15; a *= 0x846ca68bU; a ^= a >> 16;
  return a;
}

// gather: 4 warps per CTA, each a 2-stage ring of 4 rows x 512 B
__global__ void __launch_bounds__(128) gather_rd(const char* __restrict__ p, uint32_t rows, int iters, uint32_t* sink) {
  extern __shared__ __align__(16) char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  char* ring = sm + w * 2 * 4 * 512;
  const uint32_t gw = blockIdx.x * 4 + w;
  uint32_t x = 0;
  for (int it = 0; it < iters; ++it) {
    const int s = it & 1;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t row = hash32(gw * 2654435761u + it * 4 + u) % rows;
      const char* src = p + (size_t)row * 512 + lane * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(
                       ring + s * 2048 + u * 512 + lane * 16)), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    x ^= *reinterpret_cast<const uint32_t*>(ring + (s ^ 1) * 2048 + lane * 16);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (x == 0x12345678u) sink[0] = x;
}

int main(int argc, char** argv) {
  const int64_t mib = argc > 1 ? atoll(argv[1]) : 32;
  const int passes = argc > 2 ? atoi(argv[2]) : 40;
  const int reps = 5;
  const int64_t bytes = mib << 20, n16 = bytes / 16;
  char* p;
  uint32_t* sink;
  cudaMalloc(&p, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(p, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int ok = 1;
  // stream
  {
    const int grid = sms * 8;
    stream_rd<<<grid, 256>>>((const uint4*)p, n16, 2, sink);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(a);
      stream_rd<<<grid, 256>>>((const uint4*)p, n16, passes, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const cudaError_t e = cudaGetLastError();
    ok &= e == cudaSuccess;
    printf("{\"mode\": \"stream\", \"l2_read_gbs\": %.1f, \"buffer_mib\": %lld, \"best_ms\": %.4f, \"sms\": %d, "
           "\"l2_bytes\": %d, \"gpu\": \"%s\", \"status\": \"%s\"}\n",
           (double)bytes * passes / (best * 1e-3) / 1e9, (long long)mib, best, sms, prop.l2CacheSize, prop.name,
           cudaGetErrorString(e));
  }
  // gather (the kernels' access pattern), at several resident-warp counts
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"mode\": \"sm_ingress_64B_per_clk\", \"l2_read_gbs\": %.1f, \"sm_clock_mhz\": %.0f}\n",
         64.0 * sms * clk_khz * 1e3 / 1e9, clk_khz / 1e3);
  for (int ctas = 4; ctas <= 12; ctas += 2) {
    const int grid = sms * ctas, smem = 4 * 2 * 4 * 512;
    const uint32_t rows = (uint32_t)(bytes / 512);
    const int iters = (int)((int64_t)passes * rows / 4 / ((int64_t)grid * 4)) + 1;  // passes over the table
    gather_rd<<<grid, 128, smem>>>(p, rows, 64, sink);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(a);
      gather_rd<<<grid, 128, smem>>>(p, rows, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const cudaError_t e = cudaGetLastError();
    ok &= e == cudaSuccess;
    const double moved = (double)grid * 4 * iters * 4 * 512;
    printf("{\"mode\": \"gather\", \"ctas_per_sm\": %d, \"l2_read_gbs\": %.1f, \"buffer_mib\": %lld, \"best_ms\": %.4f, "
           "\"status\": \"%s\"}\n", ctas, moved / (best * 1e-3) / 1e9, (long long)mib, best, cudaGetErrorString(e));
  }
  // sustained gather: back-to-back launches for `sustain_s` seconds (argv[3], 0 = skip), the board's power
  // limit applying (run next to an nvidia-smi trace); reported per 0.25-s window
  const double sustain_s = argc > 3 ? atof(argv[3]) : 0.0;
  if (sustain_s > 0) {
    const int ctas = 12, grid = sms * ctas, smem = 4 * 2 * 4 * 512;
    const uint32_t rows = (uint32_t)(bytes / 512);
    const int iters = (int)((int64_t)passes * rows / 4 / ((int64_t)grid * 4)) + 1;
    const double moved = (double)grid * 4 * iters * 4 * 512;
    double t = 0, wt = 0, wb = 0;
    int win = 0;
    while (t < sustain_s * 1e3) {
      cudaEventRecord(a);
      gather_rd<<<grid, 128, smem>>>(p, rows, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      t += ms;
      wt += ms;
      wb += moved;
      if (wt >= 250.0) {
        printf("{\"mode\": \"gather_sustained\", \"window\": %d, \"t_ms\": %.0f, \"l2_read_gbs\": %.1f}\n", win++, t,
               wb / (wt * 1e-3) / 1e9);
        wt = 0;
        wb = 0;
      }
    }
    ok &= cudaGetLastError() == cudaSuccess;
  }
  return ok ? 0 : 1;
}
