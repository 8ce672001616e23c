// Measured peak of the cfg2 kernel's binding resource: random 8-byte gathers
// from an L2-resident table (the NIRC hash grid: 12 x 2^15 float2 = 3 MB),
// issued the way the encoder issues them (8 independent gathers in flight
// per thread, every SM busy).  Reports useful gather bandwidth (8 B per
// gather) and gathers per SM per cycle; the same loop with 16-byte loads of
// aligned slot pairs gives the paired-gather ceiling.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          tools/l2_gather_peak.cu -o tools/l2_gather_peak
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  return x ^ (x >> 16);
}

template <bool kPair>
__global__ void __launch_bounds__(512) gather(const float2* __restrict__ table, uint32_t mask,
                                              int iters, float* out) {
  uint32_t s = mix(blockIdx.x * blockDim.x + threadIdx.x + 1);
  float acc = 0.0f;
  for (int it = 0; it < iters; ++it) {
    uint32_t h[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      s = mix(s + 0x9e3779b9u);
      h[k] = s & mask;
    }
    if (kPair) {
      float4 g[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        g[k] = __ldg(reinterpret_cast<const float4*>(table) + (h[k] >> 1));
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += g[k].x + g[k].w;
    } else {
      float2 g[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) g[k] = __ldg(table + h[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += g[k].x + g[k].y;
    }
  }
  if (acc == 12345.0f) *out = acc;
}

int main() {
  const size_t entries = 12u << 15;  // 3 MB of float2
  float2* t;
  float* o;
  cudaMalloc(&t, entries * sizeof(float2));
  cudaMalloc(&o, 4);
  cudaMemset(t, 0, entries * sizeof(float2));
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
  const uint32_t mask = (1u << 18) - 1u;  // 2^18 float2 slots (2 MB) + level offset below
  const int iters = 256;
  for (int pass = 0; pass < 2; ++pass) {
    for (int blocks_per_sm : {1, 2, 4}) {
      const int blocks = sms * blocks_per_sm, threads = 512;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 3; ++w) {
        if (pass) gather<true><<<blocks, threads>>>(t, mask, iters, o);
        else gather<false><<<blocks, threads>>>(t, mask, iters, o);
      }
      cudaEventRecord(a);
      const int reps = 10;
      for (int r = 0; r < reps; ++r) {
        if (pass) gather<true><<<blocks, threads>>>(t, mask, iters, o);
        else gather<false><<<blocks, threads>>>(t, mask, iters, o);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double gathers = (double)blocks * threads * iters * 8 * reps;
      const double s = ms * 1e-3;
      printf("{\"loads\": \"%s\", \"ctas_per_sm\": %d, \"gathers_per_s\": %.4g, "
             "\"useful_gbs\": %.1f, \"gathers_per_sm_cycle\": %.3f, \"clock_khz\": %d}\n",
             pass ? "16B slot pairs" : "8B slots", blocks_per_sm, gathers / s,
             gathers * (pass ? 16.0 : 8.0) / s / 1e9, gathers / s / sms / (clk * 1e3), clk);
    }
  }
  return 0;
}
