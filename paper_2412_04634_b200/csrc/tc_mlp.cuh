// Fully fused tiny-MLP chain on tcgen05 (fp32 accumulate in TMEM).
//
// A "group" is 4 consecutive warps (128 threads, thread tg <-> tile row tg
// <-> TMEM lane tg).  Each group owns one 128-row A tile in shared memory
// (hi + lo operand images) and 64 TMEM columns.  Per layer the group's
// thread 0 issues 3 x K/Kmma tcgen05.mma (lo*hi... hi*hi, split-precision
// products) into the TMEM accumulator and commits to the group's mbarrier;
// the 128 threads then tcgen05.ld their row in 16-column chunks, add bias,
// apply ReLU, split into hi/lo and write the next layer's A tile in place.
// Activations never leave SMEM / TMEM.  The weight hi/lo images of every
// layer are staged once per CTA by TMA bulk copy and shared by all groups.
//
// Precision policies (operand split x -> hi + lo, products hi*hi + hi*lo +
// lo*hi accumulated in fp32; ~2^-22 relative per product):
//   TF32x3 : kind::tf32, 4-byte operands, K = 8 per MMA, full fp32 range;
//   F16x2  : kind::f16 with fp16 operands, 2-byte operands, K = 16 per MMA:
//            half the SMEM and half the MMAs, values must stay below the fp16
//            range (|x| < 65504); entries below 2^-14 keep ~3e-8 absolute
//            accuracy.
//
// Reference semantics: mlp_forward (pkg/src/nirclab/mlp.py:102-122):
// z = a W^T + b, ReLU hidden layers, ReLU (NIRC/NRC) or sigmoid (NVC) output.
#pragma once
#include <cuda_fp16.h>
#include "common.cuh"
#include "tc_common.cuh"

namespace nirc {
namespace tc {

constexpr int kTileRows = 128;
constexpr int kMaxTcLayers = 6;
constexpr int kGroupThreads = 128;

struct PrecTF32x3 {
  static constexpr int kElemBytes = 4;
  static constexpr uint32_t kIdescFmt = (1u << 4) | (2u << 7) | (2u << 10);  // f32 <- tf32 x tf32
  static constexpr int kId = 0;
  __device__ static inline void split4(const float* x, uint32_t* hi, uint32_t* lo) {
    // 4 elements -> one 16-byte chunk each of hi and lo
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float h = tf32_hi(x[q]);
      hi[q] = __float_as_uint(h);
      lo[q] = __float_as_uint(x[q] - h);
    }
  }
};

struct PrecF16x2 {
  static constexpr int kElemBytes = 2;
  static constexpr uint32_t kIdescFmt = (1u << 4);  // f32 <- f16 x f16
  static constexpr int kId = 2;
  __device__ static inline void split8(const float* x, uint32_t* hi, uint32_t* lo) {
    // 8 elements -> one 16-byte chunk each of hi and lo; packed f16x2
    // conversions (one cvt per pair) keep the epilogue off the slow pipe
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const __half2 h = __floats2half2_rn(x[2 * q], x[2 * q + 1]);
      const float2 hf = __half22float2(h);
      const __half2 l = __floats2half2_rn(x[2 * q] - hf.x, x[2 * q + 1] - hf.y);
      hi[q] = *reinterpret_cast<const uint32_t*>(&h);
      lo[q] = *reinterpret_cast<const uint32_t*>(&l);
    }
  }
};

template <class P>
struct Geo {
  static constexpr int kEPC = 16 / P::kElemBytes;      // elements per 16-byte chunk
  static constexpr int kKmma = 2 * kEPC;               // K per MMA instruction (32 B)
  static constexpr uint32_t kAImageBytes = kTileRows * 64 * P::kElemBytes;
  static constexpr uint32_t kABufBytes = 2 * kAImageBytes;  // hi + lo
};

// byte offset of element (r, k) in a canonical K-major no-swizzle operand
template <class P>
__host__ __device__ inline uint32_t op_offset(int r, int k, int rows) {
  constexpr int E = Geo<P>::kEPC;
  return (uint32_t)((k / E) * (rows * 16) + (r >> 3) * 128 + (r & 7) * 16 +
                    (k % E) * P::kElemBytes);
}

struct TcNet {
  int nl, out_act, prec;
  int K[kMaxTcLayers], N[kMaxTcLayers];
  uint32_t woff[kMaxTcLayers];   // byte offset of layer l's hi image; lo follows
  uint32_t wbytes;               // total image bytes
};

// Host: geometry of the packed weight image for a spec (false if unsupported).
inline bool tc_net_for(const nirc_spec_t& sp, TcNet* net, int prec) {
  if (sp.n_layers < 2 || sp.n_layers > kMaxTcLayers) return false;
  const int eb = prec == PrecF16x2::kId ? 2 : 4;
  const int kstep = prec == PrecF16x2::kId ? 16 : 8;
  net->nl = sp.n_layers;
  net->out_act = sp.out_act;
  net->prec = prec;
  uint32_t off = 0;
  for (int l = 0; l < sp.n_layers; ++l) {
    const int din = sp.dims[l], dout = sp.dims[l + 1];
    const bool last = l == sp.n_layers - 1;
    if (!last && dout != 64) return false;
    if (last && (dout < 1 || dout > 16)) return false;
    if (din > 64) return false;
    net->K[l] = (din + kstep - 1) / kstep * kstep;
    net->N[l] = last ? 16 : 64;
    net->woff[l] = off;
    off += 2u * net->N[l] * net->K[l] * eb;
  }
  net->wbytes = off;
  return true;
}

// Writes one row (K values, K % 16 == 0) of an A tile as hi/lo images.
template <class P, int K>
__device__ __forceinline__ void write_a_row(uint32_t a_hi, uint32_t a_lo, int r, const float* x) {
  constexpr int E = Geo<P>::kEPC;
#pragma unroll
  for (int kc = 0; kc < K / E; ++kc) {
    uint32_t h[4], l[4];
    if constexpr (E == 4) P::split4(x + kc * E, h, l);
    else P::split8(x + kc * E, h, l);
    const uint32_t o = op_offset<P>(r, kc * E, kTileRows);
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a_hi + o), "r"(h[0]), "r"(h[1]),
                 "r"(h[2]), "r"(h[3])
                 : "memory");
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a_lo + o), "r"(l[0]), "r"(l[1]),
                 "r"(l[2]), "r"(l[3])
                 : "memory");
  }
}

template <class P>
__device__ __forceinline__ void mma_issue(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                          uint32_t acc) {
  if constexpr (P::kId == PrecF16x2::kId) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
  } else {
    mma_tf32(tmem_d, ad, bd, idesc, acc);
  }
}

// Issues one layer: D[128 x N] = A[128 x K] . W[N x K]^T, split precision.
template <class P>
__device__ __forceinline__ void issue_layer(const TcNet& net, int l, uint32_t w_base,
                                            uint32_t a_hi, uint32_t a_lo, uint32_t tmem_d) {
  const int K = net.K[l], N = net.N[l];
  const uint32_t idesc =
      P::kIdescFmt | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTileRows >> 4) << 24);
  const uint32_t w_hi = w_base + net.woff[l];
  const uint32_t w_lo = w_hi + (uint32_t)(N * K * P::kElemBytes);
  const uint32_t a_lbo = kTileRows * 16, w_lbo = (uint32_t)N * 16;
  uint32_t acc = 0;
  // small cross terms first, the dominant hi*hi term last
#pragma unroll
  for (int term = 0; term < 3; ++term) {
    const uint32_t A = term == 1 ? a_lo : a_hi;
    const uint32_t B = term == 0 ? w_lo : w_hi;
    for (int kk = 0; kk < K / Geo<P>::kKmma; ++kk) {
      const uint64_t ad = sdesc(A + kk * 2 * a_lbo, a_lbo, 128);
      const uint64_t bd = sdesc(B + kk * 2 * w_lbo, w_lbo, 128);
      mma_issue<P>(tmem_d, ad, bd, idesc, acc);
      acc = 1;
    }
  }
}

// Runs the whole network for the group's current tile.  Precondition: this
// thread wrote its row of layer-0 input into (a_hi, a_lo).  On return y[0..3]
// holds the activated outputs of row tg (only dims[nl] are meaningful).
// Pre-fills this thread's TMEM row of the accumulator with layer l's bias
// (N columns, multiple of 16): the layer's MMAs then all accumulate on top,
// so the epilogue needs no bias add.
__device__ __forceinline__ void prefill_bias(const TcNet& net, int l,
                                             const float* __restrict__ s_bias, uint32_t taddr) {
  const float* b = s_bias + l * 64;
  for (int q = 0; q < net.N[l] / 16; ++q) {
    float bq[16];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<float4*>(bq + 4 * j) = *reinterpret_cast<const float4*>(b + q * 16 + 4 * j);
    tmem_st16(taddr + q * 16, bq);
  }
  tmem_wait_st();
}

// Runs the whole network for the group's current tile.  Precondition: this
// thread wrote its row of layer-0 input into (a_hi, a_lo).  On return y[0..3]
// holds the activated outputs of row tg (only dims[nl] are meaningful).
template <class P>
__device__ __forceinline__ void run_chain(const TcNet& net, uint32_t w_base,
                                          const float* __restrict__ s_bias, int group, int tg,
                                          uint32_t a_hi, uint32_t a_lo, uint32_t tmem_d,
                                          uint32_t mbar, uint32_t& phase, float* y,
                                          long long* probe = nullptr) {
  const uint32_t lane_off = (uint32_t)((tg >> 5) * 32) << 16;
  fence_proxy_async();
  fence_before();
  named_bar_sync(1 + group, kGroupThreads);
  if ((tg >> 5) == 0) {  // warp 0 of the group issues; one elected lane
    fence_after();
    if (elect_one()) {
      issue_layer<P>(net, 0, w_base, a_hi, a_lo, tmem_d);
      mma_commit(mbar);
    }
    __syncwarp();
  }
  for (int l = 0; l < net.nl; ++l) {
    if (probe) probe[2 * l] = clock64();
    mbar_wait(mbar, phase);
    if (probe) probe[2 * l + 1] = clock64();
    phase ^= 1u;
    fence_after();
    if (l < net.nl - 1) {
      const float* b = s_bias + l * 64;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float h[32];
        tmem_ld32(tmem_d + lane_off + half * 32, h);
        float bq[32];
#pragma unroll
        for (int j = 0; j < 8; ++j)  // broadcast 16-byte bias loads overlap the TMEM load
          *reinterpret_cast<float4*>(bq + 4 * j) =
              *reinterpret_cast<const float4*>(b + half * 32 + 4 * j);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float z = h[j] + bq[j];
          h[j] = z > 0.0f ? z : 0.0f;
        }
        // 32 columns = 8 (tf32) or 4 (f16) operand chunks
        constexpr int E = Geo<P>::kEPC;
#pragma unroll
        for (int c = 0; c < 32 / E; ++c) {
          uint32_t hh[4], ll[4];
          if constexpr (E == 4) P::split4(h + c * E, hh, ll);
          else P::split8(h + c * E, hh, ll);
          const uint32_t o = op_offset<P>(tg, half * 32 + c * E, kTileRows);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a_hi + o), "r"(hh[0]),
                       "r"(hh[1]), "r"(hh[2]), "r"(hh[3])
                       : "memory");
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a_lo + o), "r"(ll[0]),
                       "r"(ll[1]), "r"(ll[2]), "r"(ll[3])
                       : "memory");
        }
      }
      if (probe) probe[16 + 3 * l] = clock64();
      fence_proxy_async();
      fence_before();
      if (probe) probe[17 + 3 * l] = clock64();
      named_bar_sync(1 + group, kGroupThreads);
      if (probe) probe[18 + 3 * l] = clock64();
      if ((tg >> 5) == 0) {
        fence_after();
        if (probe && tg == 0) probe[40 + 2 * l] = clock64();
        if (elect_one()) {
          issue_layer<P>(net, l + 1, w_base, a_hi, a_lo, tmem_d);
          if (probe) probe[41 + 2 * l] = clock64();
          mma_commit(mbar);
        }
        __syncwarp();
      }
    } else {
      float o[4];
      tmem_ld4(tmem_d + lane_off, o);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float z = o[j] + s_bias[l * 64 + j];
        y[j] = net.out_act == 0 ? (z > 0.0f ? z : 0.0f) : 1.0f / (1.0f + expf(-z));
      }
    }
  }
  fence_before();
}

// ---------------------------------------------------------------------
// F16x2 chain with the A operand in TENSOR memory ("TS" MMAs).  Measured on
// B200 (tools/mma_bench.cu): an M128 N64 K16 f16 MMA costs 48 cycles with A
// read from shared memory but 32 cycles with A in TMEM, and the epilogue
// writes the next layer's input with tcgen05.st instead of st.shared plus
// proxy fences.  Per group TMEM: D (64 fp32 columns) | A_hi (32) | A_lo (32);
// fp16 element (row m, k) sits at lane m, column k/2, half k%2.
constexpr uint32_t kTsColsPerGroup = 128;

// fp16 range guard of the F16x2 split: an operand must round to a finite
// fp16 hi part.  Rows holding a value at or above this bound (or a NaN) are
// flagged by the chain and recomputed by the fp32 SIMT fix-up kernels.
constexpr float kF16Max = 65000.0f;

__device__ __forceinline__ bool f16_unsafe(const float* x, int n) {
  float m = 0.0f;
  bool nan = false;
  for (int i = 0; i < n; ++i) {
    m = fmaxf(m, fabsf(x[i]));
    nan |= x[i] != x[i];
  }
  return nan || !(m < kF16Max);
}

// Writes this thread's row (K values, K % 16 == 0) into A_hi / A_lo (TMEM).
template <int K>
__device__ __forceinline__ void write_a_row_ts(uint32_t a_hi, uint32_t a_lo, const float* x) {
#pragma unroll
  for (int c = 0; c < K / 16; ++c) {  // 16 values -> 8 packed columns each of hi and lo
    uint32_t h[8], l[8];
    PrecF16x2::split8(x + 16 * c, h, l);
    PrecF16x2::split8(x + 16 * c + 8, h + 4, l + 4);
    tmem_st8u(a_hi + 8 * c, h);
    tmem_st8u(a_lo + 8 * c, l);
  }
}

// acc0 = 1: the accumulator was pre-filled (with the layer's bias).
__device__ __forceinline__ void issue_layer_ts(const TcNet& net, int l, uint32_t w_base,
                                               uint32_t a_hi, uint32_t a_lo, uint32_t tmem_d,
                                               uint32_t acc0 = 0) {
  const int K = net.K[l], N = net.N[l];
  const uint32_t idesc =
      PrecF16x2::kIdescFmt | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTileRows >> 4) << 24);
  const uint32_t w_hi = w_base + net.woff[l];
  const uint32_t w_lo = w_hi + (uint32_t)(N * K * 2);
  const uint32_t w_lbo = (uint32_t)N * 16;
  uint32_t acc = acc0;
#pragma unroll
  for (int term = 0; term < 3; ++term) {  // hi*lo, lo*hi, then hi*hi
    const uint32_t A = term == 1 ? a_lo : a_hi;
    const uint32_t B = term == 0 ? w_lo : w_hi;
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint64_t bd = sdesc(B + kk * 2 * w_lbo, w_lbo, 128);
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "setp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
          "r"(A + kk * 8), "l"(bd), "r"(idesc), "r"(acc));
      acc = 1;
    }
  }
}

// This thread's lane of a layer's accumulator <- the layer's bias (N columns,
// 16 or 64): the MMAs then accumulate on top of it, so no epilogue adds it.
__device__ __forceinline__ void prefill_bias_ts(const float* __restrict__ b, int N,
                                                uint32_t taddr) {
  for (int q = 0; q < N / 16; ++q) {
    float bq[16];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<float4*>(bq + 4 * j) = *reinterpret_cast<const float4*>(b + 16 * q + 4 * j);
    tmem_st16(taddr + 16 * q, bq);
  }
}

// Runs the network for the group's tile; precondition: this thread wrote its
// layer-0 row with write_a_row_ts.  Every layer's accumulator starts from
// its bias (prefill_bias_ts); the epilogue is ReLU + fp16 hi/lo split.
// `unsafe` accumulates the fp16 range guard over every hidden activation
// (an fp16 hi part that rounded to inf; activations are >= 0 after ReLU, so
// their fp16 bit patterns order like their values).
__device__ __forceinline__ void run_chain_ts(const TcNet& net, uint32_t w_base,
                                             const float* __restrict__ s_bias, int group, int tg,
                                             uint32_t tmem_grp, uint32_t mbar, uint32_t& phase,
                                             float* y, bool& unsafe) {
  const uint32_t lane_off = (uint32_t)((tg >> 5) * 32) << 16;
  const uint32_t tmem_d = tmem_grp, a_hi = tmem_grp + 64, a_lo = tmem_grp + 96;
  prefill_bias_ts(s_bias, net.N[0], tmem_d + lane_off);
  tmem_wait_st();
  fence_before();
  named_bar_sync(1 + group, kGroupThreads);
  if ((tg >> 5) == 0) {
    fence_after();
    if (elect_one()) {
      issue_layer_ts(net, 0, w_base, a_hi, a_lo, tmem_d, 1u);
      mma_commit(mbar);
    }
    __syncwarp();
  }
  for (int l = 0; l < net.nl; ++l) {
    mbar_wait(mbar, phase);
    phase ^= 1u;
    fence_after();
    if (l < net.nl - 1) {
      uint32_t hmax = 0u;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float h[32];
        tmem_ld32(tmem_d + lane_off + half * 32, h);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) h[j] = fmaxf(h[j], 0.0f);
        uint32_t hh[16], ll[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) PrecF16x2::split8(h + 8 * c, hh + 4 * c, ll + 4 * c);
#pragma unroll
        for (int c = 0; c < 16; ++c) hmax = __vmaxu2(hmax, hh[c]);
        tmem_st16u(a_hi + lane_off + half * 16, hh);
        tmem_st16u(a_lo + lane_off + half * 16, ll);
      }
      unsafe |= (hmax & 0xffffu) > 0x7bffu || (hmax >> 16) > 0x7bffu;
      // the accumulator was read: pre-fill it with the next layer's bias
      prefill_bias_ts(s_bias + (l + 1) * 64, net.N[l + 1], tmem_d + lane_off);
      tmem_wait_st();
      fence_before();
      named_bar_sync(1 + group, kGroupThreads);
      if ((tg >> 5) == 0) {
        fence_after();
        if (elect_one()) {
          issue_layer_ts(net, l + 1, w_base, a_hi, a_lo, tmem_d, 1u);
          mma_commit(mbar);
        }
        __syncwarp();
      }
    } else {
      float o[4];
      tmem_ld4(tmem_d + lane_off, o);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float z = o[j];
        y[j] = net.out_act == 0 ? (z > 0.0f ? z : 0.0f) : 1.0f / (1.0f + expf(-z));
      }
    }
  }
  fence_before();
}

// Shared-memory carve-up common to the tensor-core kernels.
struct TcSmem {
  uint32_t w_off, bias_off, a_off, abuf_bytes, bar_off, holder_off, total;
};
__host__ __device__ inline TcSmem tc_smem_layout(const TcNet& net, int ngroups, uint32_t extra) {
  TcSmem s;
  s.w_off = 0;
  // F16x2 keeps A in TMEM (run_chain_ts); TF32x3 keeps hi/lo A tiles in SMEM
  s.abuf_bytes = net.prec == PrecF16x2::kId ? 0u : 2u * kTileRows * 64 * 4u;
  s.bias_off = (net.wbytes + 1023u) & ~1023u;
  s.a_off = (s.bias_off + kMaxTcLayers * 64 * 4 + 1023u) & ~1023u;
  s.bar_off = s.a_off + ngroups * s.abuf_bytes + extra;
  s.holder_off = s.bar_off + 8 * (1 + ngroups);
  s.total = s.holder_off + 16;
  return s;
}

__host__ __device__ inline uint32_t tmem_cols_for(int ngroups, int prec) {
  const uint32_t need = (prec == PrecF16x2::kId ? kTsColsPerGroup : 64u) * (uint32_t)ngroups;
  uint32_t c = 32;
  while (c < need) c <<= 1;
  return c;
}

// CTA prologue: barriers, TMEM allocation, weight image by TMA bulk copy.
__device__ __forceinline__ void tc_prologue(uint8_t* smem, const TcSmem& L, const TcNet& net,
                                            int ngroups, const uint8_t* __restrict__ wimg,
                                            const float* __restrict__ bias_g,
                                            uint32_t& tmem_base) {
  const uint32_t s0 = smem_u32(smem);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + L.holder_off);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < 1 + ngroups; ++i) mbar_init(s0 + L.bar_off + 8 * i, 1);
    mbar_init_fence();
  }
  if ((tid >> 5) == 0) tmem_alloc(smem_u32(holder), tmem_cols_for(ngroups, net.prec));
  float* s_bias = reinterpret_cast<float*>(smem + L.bias_off);
  for (int i = tid; i < net.nl * 64; i += blockDim.x) s_bias[i] = bias_g[i];
  fence_before();
  __syncthreads();
  fence_after();
  tmem_base = *holder;
  if (tid == 0) {
    const uint32_t wbar = s0 + L.bar_off;
    mbar_expect_tx(wbar, net.wbytes);
    for (uint32_t off = 0; off < net.wbytes; off += 32768u) {
      const uint32_t sz = net.wbytes - off < 32768u ? net.wbytes - off : 32768u;
      bulk_g2s(s0 + L.w_off + off, wimg + off, sz, wbar);
    }
  }
  mbar_wait(s0 + L.bar_off, 0);
}

__device__ __forceinline__ void tc_epilogue(uint32_t tmem_base, int ngroups, int prec) {
  fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) {
    fence_after();
    tmem_dealloc(tmem_base, tmem_cols_for(ngroups, prec));
  }
}

}  // namespace tc

// fp32 network of one encoded row (in a[], result in a[0..dout)); W is the
// shared-memory copy of theta[grid_len:].
__device__ inline void simt_net_row(const nirc_spec_t& sp, const float* __restrict__ W, float* a,
                                    float* b) {
  for (int l = 0; l < sp.n_layers; ++l) {
    const int din = sp.dims[l], dout = sp.dims[l + 1];
    const float* w = W + (sp.w_off[l] - sp.grid_len);
    const float* bias = W + (sp.b_off[l] - sp.grid_len);
    const bool last = l == sp.n_layers - 1;
#pragma unroll 4
    for (int j = 0; j < dout; ++j) {
      float acc = 0.0f;
#pragma unroll 8
      for (int i = 0; i < din; ++i) acc = fmaf(a[i], w[j * din + i], acc);
      const float z = acc + bias[j];
      b[j] = (!last || sp.out_act == 0) ? (z > 0.0f ? z : 0.0f) : 1.0f / (1.0f + expf(-z));
    }
    for (int j = 0; j < dout; ++j) a[j] = b[j];
  }
}

// One launch's packed weight image (k_pack_weights), in a caller-owned
// stream-ordered buffer; `unsafe` = a weight outside the F16x2 range.
struct PackedNet {
  uint8_t* img;
  float* bias;
  int32_t* unsafe;
};

}  // namespace nirc
