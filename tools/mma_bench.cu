// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128, K=16) for the
// NIRC tile shapes, A from shared memory (SS) vs from tensor memory (TS).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//          tools/mma_bench.cu -o tools/mma_bench
#include <cstdio>
#include <cstdint>
#include "../paper_2412_04634_b200/csrc/tc_common.cuh"

using namespace nirc::tc;

template <int N, bool TS>
__global__ void bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const uint32_t s0 = smem_u32(sm);
  const uint32_t a = s0, b = s0 + 128 * 64 * 2;  // A: 128 x 64 f16, B: N x 64 f16
  for (int i = threadIdx.x; i < (128 + N) * 64 / 2; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;  // 1.0h
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init_fence();
  }
  if (threadIdx.x < 32) tmem_alloc(smem_u32(&holder), 256);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = holder;
  fence_proxy_async();
  __syncthreads();
  if (threadIdx.x < 32) {
    fence_after();
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = sdesc(b + kk * 2 * N * 16, N * 16, 128);
          if (TS) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm),
                "r"(tm + 128 + kk * 8), "l"(bd), "r"(idesc), "r"(1u));
          } else {
            const uint64_t ad = sdesc(a + kk * 2 * 128 * 16, 128 * 16, 128);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
                "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
          }
        }
      }
      long long t1 = clock64();
      mma_commit(smem_u32(&bar));
      out[blockIdx.x * 2] = t1 - t0;
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    long long t2 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    fence_after();
    tmem_dealloc(tm, 256);
  }
}

template <int N, bool TS>
void run(int iters, int blocks) {
  long long* d;
  cudaMalloc(&d, 2 * blocks * sizeof(long long));
  const int smem = (128 + N) * 64 * 2 + 1024;
  cudaFuncSetAttribute(bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<N, TS><<<blocks, 128, smem>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double n = 4.0 * iters;
  printf("N=%3d %s blocks=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\n", N,
         TS ? "A:TMEM" : "A:SMEM", blocks, h[0] / n, h[1] / n, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int blocks : {1, 148}) {
    run<64, false>(256, blocks);
    run<64, true>(256, blocks);
    run<128, false>(256, blocks);
    run<256, false>(256, blocks);
    run<16, false>(256, blocks);
  }
  return 0;
}
