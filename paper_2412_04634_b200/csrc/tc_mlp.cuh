// Fully fused tiny-MLP chain on tcgen05 (3xTF32, fp32 accumulate in TMEM).
//
// A "group" is 4 consecutive warps (128 threads, thread tg <-> tile row tg
// <-> TMEM lane tg).  Each group owns one 128-row A tile in shared memory
// (tf32 hi + lo images, 32 KB each) and 64 TMEM columns.  Per layer the
// group's thread 0 issues 3 x K/8 tcgen05.mma (hi*hi, hi*lo, lo*hi) into the
// TMEM accumulator and commits to the group's mbarrier; the 128 threads then
// tcgen05.ld their row, add bias, apply ReLU, split into tf32 hi/lo and
// write the next layer's A tile in place.  Activations never leave SMEM /
// TMEM.  Weights (hi/lo images of every layer) are staged once per CTA by
// TMA bulk copy and shared by all groups.
//
// Reference semantics: mlp_forward (pkg/src/nirclab/mlp.py:102-122):
// z = a W^T + b, ReLU hidden layers, ReLU (NIRC/NRC) or sigmoid (NVC) output.
#pragma once
#include "common.cuh"
#include "tc_common.cuh"

namespace nirc {
namespace tc {

constexpr int kTileRows = 128;
constexpr int kMaxTcLayers = 6;
constexpr int kGroupThreads = 128;
constexpr uint32_t kAImageBytes = kTileRows * 64 * 4;   // one of hi/lo, K <= 64
constexpr uint32_t kABufBytes = 2 * kAImageBytes;        // hi + lo

struct TcNet {
  int nl, out_act;
  int K[kMaxTcLayers], N[kMaxTcLayers];
  uint32_t woff[kMaxTcLayers];   // byte offset of layer l's hi image; lo follows
  uint32_t wbytes;               // total image bytes
};

// Host: geometry of the packed weight image for a spec (0 if unsupported).
inline bool tc_net_for(const nirc_spec_t& sp, TcNet* net) {
  if (sp.n_layers < 2 || sp.n_layers > kMaxTcLayers) return false;
  net->nl = sp.n_layers;
  net->out_act = sp.out_act;
  uint32_t off = 0;
  for (int l = 0; l < sp.n_layers; ++l) {
    const int din = sp.dims[l], dout = sp.dims[l + 1];
    const bool last = l == sp.n_layers - 1;
    if (!last && dout != 64) return false;
    if (last && (dout < 1 || dout > 16)) return false;
    if (din > 64) return false;
    net->K[l] = (din + 7) / 8 * 8;
    net->N[l] = last ? 16 : 64;
    net->woff[l] = off;
    off += 2u * net->N[l] * net->K[l] * 4u;
  }
  net->wbytes = off;
  return true;
}

// Writes one row (K values, K % 4 == 0) of an A tile as tf32 hi/lo images.
template <int K>
__device__ __forceinline__ void write_a_row(uint32_t a_hi, uint32_t a_lo, int r, const float* x) {
#pragma unroll
  for (int kc = 0; kc < K / 4; ++kc) {
    float h[4], l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      h[q] = tf32_hi(x[kc * 4 + q]);
      l[q] = x[kc * 4 + q] - h[q];
    }
    const uint32_t o = tile_offset(r, kc * 4, kTileRows);
    st_shared_v4(a_hi + o, h[0], h[1], h[2], h[3]);
    st_shared_v4(a_lo + o, l[0], l[1], l[2], l[3]);
  }
}

// Issues one layer: D[128 x N] = A[128 x K] . W[N x K]^T in 3xTF32.
__device__ __forceinline__ void issue_layer(const TcNet& net, int l, uint32_t w_base,
                                            uint32_t a_hi, uint32_t a_lo, uint32_t tmem_d) {
  const int K = net.K[l], N = net.N[l];
  const uint32_t idesc = idesc_tf32(kTileRows, N);
  const uint32_t w_hi = w_base + net.woff[l];
  const uint32_t w_lo = w_hi + (uint32_t)(N * K * 4);
  const uint32_t a_lbo = kTileRows * 16, w_lbo = (uint32_t)N * 16;
  uint32_t acc = 0;
  // small cross terms first, the dominant hi*hi term last
#pragma unroll
  for (int term = 0; term < 3; ++term) {
    const uint32_t A = term == 1 ? a_lo : a_hi;
    const uint32_t B = term == 0 ? w_lo : w_hi;
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint64_t ad = sdesc(A + kk * 2 * a_lbo, a_lbo, 128);
      const uint64_t bd = sdesc(B + kk * 2 * w_lbo, w_lbo, 128);
      mma_tf32(tmem_d, ad, bd, idesc, acc);
      acc = 1;
    }
  }
}

// Runs the whole network for the group's current tile.  Precondition: this
// thread wrote its row of layer-0 input into (a_hi, a_lo).  On return y[0..3]
// holds the activated outputs of row tg (only dims[nl] are meaningful).
__device__ __forceinline__ void run_chain(const TcNet& net, uint32_t w_base,
                                          const float* __restrict__ s_bias, int group, int tg,
                                          uint32_t a_hi, uint32_t a_lo, uint32_t tmem_d,
                                          uint32_t mbar, uint32_t& phase, float* y) {
  const uint32_t lane_off = (uint32_t)((tg >> 5) * 32) << 16;
  fence_proxy_async();
  fence_before();
  named_bar_sync(1 + group, kGroupThreads);
  if (tg == 0) {
    fence_after();
    issue_layer(net, 0, w_base, a_hi, a_lo, tmem_d);
    mma_commit(mbar);
  }
  for (int l = 0; l < net.nl; ++l) {
    mbar_wait(mbar, phase);
    phase ^= 1u;
    fence_after();
    const float* b = s_bias + l * 64;
    if (l < net.nl - 1) {
      float h[64];
#pragma unroll
      for (int q = 0; q < 4; ++q) tmem_ld16(tmem_d + lane_off + q * 16, h + q * 16);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const float z = h[j] + b[j];
        h[j] = z > 0.0f ? z : 0.0f;
      }
      write_a_row<64>(a_hi, a_lo, tg, h);
      fence_proxy_async();
      fence_before();
      named_bar_sync(1 + group, kGroupThreads);
      if (tg == 0) {
        fence_after();
        issue_layer(net, l + 1, w_base, a_hi, a_lo, tmem_d);
        mma_commit(mbar);
      }
    } else {
      float o[4];
      tmem_ld4(tmem_d + lane_off, o);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float z = o[j] + b[j];
        y[j] = net.out_act == 0 ? (z > 0.0f ? z : 0.0f) : 1.0f / (1.0f + expf(-z));
      }
    }
  }
  fence_before();
}

// Shared-memory carve-up common to the tensor-core kernels.
struct TcSmem {
  uint32_t w_off, bias_off, a_off, bar_off, holder_off, total;
};
__host__ __device__ inline TcSmem tc_smem_layout(const TcNet& net, int ngroups, uint32_t extra) {
  TcSmem s;
  s.w_off = 0;
  s.bias_off = (net.wbytes + 1023u) & ~1023u;
  s.a_off = (s.bias_off + kMaxTcLayers * 64 * 4 + 1023u) & ~1023u;
  s.bar_off = s.a_off + ngroups * kABufBytes + extra;
  s.holder_off = s.bar_off + 8 * (1 + ngroups);
  s.total = s.holder_off + 16;
  return s;
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
  if ((tid >> 5) == 0) tmem_alloc(smem_u32(holder), ngroups == 1 ? 64u : 128u);
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

__device__ __forceinline__ void tc_epilogue(uint32_t tmem_base, int ngroups) {
  fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) {
    fence_after();
    tmem_dealloc(tmem_base, ngroups == 1 ? 64u : 128u);
  }
}

}  // namespace tc
}  // namespace nirc
