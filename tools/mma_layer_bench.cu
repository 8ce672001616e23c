// Microbenchmark of one NIRC layer on tcgen05: G groups in one CTA (one per
// warp, each with its own 128-column TMEM slot), each issuing a burst of 12
// kind::f16 MMAs (M128 N64 K16, A from TMEM) + commit, then waiting on its
// mbarrier.  Reports per group: issue cycles (first to last UTCHMMA) and
// issue->completion cycles, median over reps; also N=16 and SS (A in SMEM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          tools/mma_layer_bench.cu -o tools/mma_layer_bench
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>
#include "../paper_2412_04634_b200/csrc/tc_common.cuh"

using namespace nirc::tc;

template <int N, bool TS, int NMMA>
__global__ void bench(long long* out, int reps, int G) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[4];
  __shared__ uint32_t holder;
  const uint32_t s0 = smem_u32(sm);
  const uint32_t a = s0, b = s0 + 128 * 64 * 2;
  for (int i = threadIdx.x; i < (128 + 64) * 64 / 2; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int g = 0; g < 4; ++g) mbar_init(smem_u32(&bars[g]), 1);
    mbar_init_fence();
  }
  if (threadIdx.x < 32) tmem_alloc(smem_u32(&holder), 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = holder;
  fence_proxy_async();
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if (w < G) {
    fence_after();
    const uint32_t d = tm + w * 128;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint32_t phase = 0;
    for (int r = 0; r < reps; ++r) {
      long long t0 = clock64(), t1 = 0;
      if (elect_one()) {
#pragma unroll
        for (int m = 0; m < NMMA; ++m) {
          const int kk = m & 3;
          const uint64_t bd = sdesc(b + kk * 2 * N * 16, N * 16, 128);
          if (TS) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                "r"(d + 64 + kk * 8), "l"(bd), "r"(idesc), "r"(1u));
          } else {
            const uint64_t ad = sdesc(a + kk * 2 * 128 * 16, 128 * 16, 128);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
          }
        }
        t1 = clock64();
        mma_commit(smem_u32(&bars[w]));
      }
      __syncwarp();
      mbar_wait(smem_u32(&bars[w]), phase);
      phase ^= 1;
      long long t2 = clock64();
      if ((threadIdx.x & 31) == 0 && t1) {
        out[((size_t)blockIdx.x * 4 + w) * reps * 2 + 2 * r] = t1 - t0;
        out[((size_t)blockIdx.x * 4 + w) * reps * 2 + 2 * r + 1] = t2 - t0;
      }
    }
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    fence_after();
    tmem_dealloc(tm, 512);
  }
}

template <int N, bool TS, int NMMA>
void run(int G, int blocks) {
  const int reps = 64;
  long long* d;
  const size_t cnt = (size_t)blocks * 4 * reps * 2;
  cudaMalloc(&d, cnt * sizeof(long long));
  cudaMemset(d, 0, cnt * sizeof(long long));
  const int smem = (128 + 64) * 64 * 2 + 1024;
  cudaFuncSetAttribute(bench<N, TS, NMMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<N, TS, NMMA><<<blocks, 128, smem>>>(d, reps, G);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(cnt);
  cudaMemcpy(h.data(), d, cnt * sizeof(long long), cudaMemcpyDeviceToHost);
  std::vector<long long> is, co;
  for (int w = 0; w < G; ++w)
    for (int r = 8; r < reps; ++r) {
      is.push_back(h[(size_t)w * reps * 2 + 2 * r]);
      co.push_back(h[(size_t)w * reps * 2 + 2 * r + 1]);
    }
  std::sort(is.begin(), is.end());
  std::sort(co.begin(), co.end());
  printf("N=%2d %s NMMA=%2d groups=%d blocks=%3d: issue %5lld cyc, issue->done %5lld cyc"
         " (%.1f cyc/mma/group)  %s\n",
         N, TS ? "TS" : "SS", NMMA, G, blocks, is[is.size() / 2], co[co.size() / 2],
         (double)co[co.size() / 2] / NMMA, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int G : {1, 2, 4}) {
    run<64, true, 12>(G, 148);
    run<64, false, 12>(G, 148);
    run<16, true, 12>(G, 148);
    run<64, true, 4>(G, 148);
    run<64, true, 48>(G, 148);
  }
  return 0;
}
