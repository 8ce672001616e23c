// Probe: tcgen05.mma kind::f16 with MN-major (transposed) SMEM operands
// built as the transposed VIEW of K-major canonical buffers -- the operand
// forms of the training kernel's backward GEMMs:
//   dA  : D[128 x N] = dZ[128 x 64] . W     (B = W^T view of W's K-major image)
//   dW  : D[128 x N] = dZ^T[M=j] . X[r x i] (A = dZ^T view, B = X^T view, K = rows)
// Values are small integers (exact in fp16 and fp32); prints max error per
// (descriptor variant) so the right LBO/SBO meaning is established on HW.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2412_04634_b200/csrc \
//      -o tools/mma_mn_test tools/mma_mn_test.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "tc_common.cuh"

using namespace nirc::tc;

// byte offset of (r, k) in a K-major canonical no-swizzle f16 buffer with R rows
__host__ __device__ inline uint32_t kmaj(int r, int k, int R) {
  return (uint32_t)((k / 8) * (R * 16) + (r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2);
}

struct Args {
  int mode;      // 0 = dA form, 1 = dW form
  int N;         // MMA N
  int K;         // MMA K (total)
  uint32_t a_lbo, a_sbo, b_lbo, b_sbo;
  int a_mn, b_mn;  // transpose bits
};

__global__ void k_probe(Args g, const __half* Abuf, int abytes, const __half* Bbuf, int bbytes,
                        float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  // A at 0, B at 64 KB (junk reads of A land in zeroed memory)
  for (int i = tid; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  __syncthreads();
  for (int i = tid; i < abytes / 2; i += blockDim.x) reinterpret_cast<__half*>(sm)[i] = Abuf[i];
  for (int i = tid; i < bbytes / 2; i += blockDim.x)
    reinterpret_cast<__half*>(sm + 65536)[i] = Bbuf[i];
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init_fence();
  }
  if (tid < 32) tmem_alloc(smem_u32(&holder), 128);
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = holder;
  if (tid < 32) {
    if (elect_one()) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)g.a_mn << 15) | ((uint32_t)g.b_mn << 16) |
                             ((uint32_t)(g.N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 65536);
      for (int kk = 0; kk < g.K / 16; ++kk) {
        // advance 16 K-elements: K-major -> 2 chunks (2*LBO); MN-major -> 2 8-row groups
        // the transposed view's K-groups (8 rows of the stored buffer) are
        // 128 B apart: 16 K-elements = 256 B; K-major: 2 chunks = 2 * LBO
        const uint32_t aoff = g.a_mn ? kk * 256u : kk * 2 * g.a_lbo;
        const uint32_t boff = g.b_mn ? kk * 256u : kk * 2 * g.b_lbo;
        const uint64_t ad = sdesc(a0 + aoff, g.a_lbo, g.a_sbo);
        const uint64_t bd = sdesc(b0 + boff, g.b_lbo, g.b_sbo);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
            "l"(ad), "l"(bd), "r"(idesc), "r"(kk));
      }
      mma_commit(smem_u32(&bar));
    }
    __syncwarp();
  }
  mbar_wait(smem_u32(&bar), 0);
  fence_after();
  const uint32_t lane_off = (uint32_t)((tid >> 5) * 32) << 16;
  for (int c = 0; c < g.N; c += 16) {
    float v[16];
    tmem_ld16(tm + lane_off + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 16; ++j) out[tid * 64 + c + j] = v[j];
  }
  fence_before();
  __syncthreads();
  if (tid < 32) {
    fence_after();
    tmem_dealloc(tm, 128);
  }
}

static float rnd() { return (float)((rand() % 7) - 3); }

int main() {
  srand(1);
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode) {
    for (int N : {48, 64}) {
      // dA: A = dZ [128 x 64] K-major, B^T view of W image (rows j=64, K = i = N)
      // dW: A = dZ^T view of dZ [128 r x 64 j], B = X^T view of X [128 r x N i]
      const int R = 128;
      std::vector<float> dz(R * 64), w(64 * N), x(R * N);
      for (auto& v : dz) v = rnd();
      for (auto& v : w) v = rnd();
      for (auto& v : x) v = rnd();
      std::vector<__half> A, B;
      int K;
      std::vector<float> ref(128 * 64, 0.0f);
      if (mode == 0) {
        K = 64;
        A.assign(R * 64, __float2half(0.f));
        for (int r = 0; r < R; ++r)
          for (int j = 0; j < 64; ++j) A[kmaj(r, j, R) / 2] = __float2half(dz[r * 64 + j]);
        B.assign(64 * N, __float2half(0.f));  // W image: rows j (64), K = i (N)
        for (int j = 0; j < 64; ++j)
          for (int i = 0; i < N; ++i) B[kmaj(j, i, 64) / 2] = __float2half(w[j * N + i]);
        for (int r = 0; r < R; ++r)
          for (int i = 0; i < N; ++i) {
            float s = 0;
            for (int j = 0; j < 64; ++j) s += dz[r * 64 + j] * w[j * N + i];
            ref[r * 64 + i] = s;
          }
      } else {
        K = 128;
        A.assign(R * 64, __float2half(0.f));
        for (int r = 0; r < R; ++r)
          for (int j = 0; j < 64; ++j) A[kmaj(r, j, R) / 2] = __float2half(dz[r * 64 + j]);
        B.assign(R * N, __float2half(0.f));
        for (int r = 0; r < R; ++r)
          for (int i = 0; i < N; ++i) B[kmaj(r, i, R) / 2] = __float2half(x[r * N + i]);
        for (int j = 0; j < 64; ++j)
          for (int i = 0; i < N; ++i) {
            float s = 0;
            for (int r = 0; r < R; ++r) s += dz[r * 64 + j] * x[r * N + i];
            ref[j * 64 + i] = s;
          }
      }
      __half *dA, *dB;
      float* dO;
      cudaMalloc(&dA, A.size() * 2);
      cudaMalloc(&dB, B.size() * 2);
      cudaMalloc(&dO, 128 * 64 * 4);
      cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
      cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
      cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      // variants: (lbo, sbo) of the MN-major operands swapped or not
      for (int var = 0; var < 2; ++var) {
        Args g{};
        g.mode = mode;
        g.N = N;
        g.K = K;
        if (mode == 0) {
          g.a_mn = 0;
          g.a_lbo = R * 16;
          g.a_sbo = 128;
          g.b_mn = 1;
          // transposed view of the W image (R_orig = 64 rows): K-group stride 128, MN-unit stride 64*16
          g.b_lbo = var == 0 ? 128 : 64 * 16;
          g.b_sbo = var == 0 ? 64 * 16 : 128;
        } else {
          g.a_mn = 1;
          g.b_mn = 1;
          g.a_lbo = var == 0 ? 128 : R * 16;
          g.a_sbo = var == 0 ? R * 16 : 128;
          g.b_lbo = g.a_lbo;
          g.b_sbo = g.a_sbo;
        }
        cudaMemset(dO, 0, 128 * 64 * 4);
        k_probe<<<1, 128, 160 * 1024>>>(g, dA, (int)A.size() * 2, dB, (int)B.size() * 2, dO);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> o(128 * 64);
        cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        const int rows = mode == 0 ? 128 : 64;
        for (int m = 0; m < rows; ++m)
          for (int n = 0; n < N; ++n) err = fmax(err, fabs(o[m * 64 + n] - ref[m * 64 + n]));
        printf("mode %s N=%d variant %d (lbo,sbo swapped=%d): %s max_err=%g\n",
               mode == 0 ? "dA" : "dW", N, var, var, cudaGetErrorString(e), err);
        if (var == 0 && err != 0) ++fails;
      }
      cudaFree(dA);
      cudaFree(dB);
      cudaFree(dO);
    }
  }
  printf("%s\n", fails ? "FAIL (variant 0)" : "variant 0 OK");
  return 0;
}
