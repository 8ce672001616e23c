// The online training step on tcgen05 (train_frame body,
// pkg/src/nirclab/caches.py:330-350, for the l2 / relative-L2 losses and
// the default NIRC layout): ONE kernel per optimizer step, one 512-thread
// CTA per 128-row tile of the batch (B = 16,384 -> 128 CTAs, one wave).
//
//   encode (bit-exact, encoding.py:111-157)
//   forward (mlp.py:102-122)        Z_l = A_{l-1} W_l^T + b_l   tcgen05, fp32 accumulate in TMEM
//   loss gradient (losses.py:23-42, f64, cast to f32 as caches.py:349)
//   backward (mlp.py:125-154)       dA_{l-1} = dZ_l W_l         tcgen05 (A = dZ in TMEM,
//                                                               B = W^T view of W's image)
//                                   dW_l = dZ_l^T A_{l-1}, db   tcgen05 (both operands as
//                                                               transposed views, K = rows)
//   hash-grid scatter (encoding.py:160-167)
//
// Precision.  Every operand is split x = hi + lo in fp16 and each GEMM
// accumulates hi*hi + hi*lo + lo*hi in fp32 (~2^-22 relative per product,
// the reference's fp32 class).  Gradients are tiny (dL/dy carries 1/(3B)),
// so the backward operands are power-of-two scaled before the split --
// exact, undone in the epilogue: dZ for dA is scaled PER ROW (dA is
// row-wise), dZ^T for dW PER COLUMN (dW sums over rows), each to a maximum
// of ~2^14, so every row / column keeps fp16's full relative precision.
// Forward operands are range-guarded (|x| < 65000): a tile that exceeds it
// is handed to the fp32 SIMT kernel (k_train_tile) through a fix-up list.
//
// Layouts (all canonical no-swizzle tcgen05 layouts, tc_common.cuh):
//   SMEM  W_l images (fp16 hi/lo, K-major, TMA bulk copy) -- forward B
//         operands and, read as their transposed (MN-major) view, the dA
//         B operands;  act0 = X (hi/lo, K-major [128 x 48], column 47 = 1
//         so dW_0's extra column is db_0);  act = A_{l-1} (hi/lo, K-major
//         [128 x 80], column 64 = 1 for db_l);  dZt = column-scaled dZ
//         (hi/lo, K-major [128 x 64]).  dW reads act / dZt as MN-major
//         views (LBO = 128 B, SBO = 2 KB: measured, tools/mma_mn_test.cu);
//         its M is 128 with rows >= 64 don't-care.
//   TMEM  cols [64 l, 64 l + 64): Z_l of hidden layer l (forward
//         accumulator, kept as the backward's stash) | [256, 320): A operand
//         hi/lo (forward layers >= 1, backward dZ) | [320, 384): dA
//         accumulator / forward output | [384, 464): dW accumulator.
//
// Deterministic pieces: the weight / bias gradients are per-tile partials
// summed in a fixed order (k_reduce_grad), the loss likewise; the hash-grid
// scatter uses atomics (coarse levels aggregated per CTA in shared memory
// first) unless dx_out is given, in which case the rows' grid gradients are
// written out for the deterministic scatter (train_scatter.cu).
#include <cmath>
#include "common.cuh"
#include "tc_mlp.cuh"

namespace nirc {

int sm_count();
int pack_weights(const nirc_spec_t& sp, const tc::TcNet& net, const float* theta,
                 cudaStream_t s, AsyncBuf& buf, PackedNet* out);

namespace ttc {

using namespace tc;

constexpr int kThreads = 512;
constexpr int kSplit = 4;               // threads per row (warps w, w+4, w+8, w+12 share a lane quadrant)
constexpr int kR = 128;                 // rows per tile = MMA M
constexpr uint32_t kChunk = kR * 16;    // bytes per 8-column chunk of a [128 x K] fp16 operand
constexpr uint32_t kColAop = 256;       // A operand: hi at +0 (32 cols = 64 fp16), lo at +32
constexpr uint32_t kColDA = 320;        // dA accumulator (<= 64) / forward output (16)
constexpr uint32_t kColDW = 384;        // dW accumulator (<= 80)
constexpr uint32_t kTmemCols = 512;
constexpr int kMaxNL = 5;               // <= 4 hidden layers (4 x 64 stash columns)
constexpr int kActCols = 80;            // 64 activations | ones column | pad
constexpr int kAct0Cols = 48;           // 47 inputs | ones column
constexpr int kDbgStride = 336;         // debug dump per row: X 48 | Z 4x64 | out 4 | unsafe 2 | pad | dX 24
constexpr int kStat4 = 7;               // per-record static encoding: 7 float4 (u | SH | aux, 1)

struct Plan {
  uint32_t w_off, bias_off, dzt_off, act_off, act0_off, dense_off, stage_off, total;
  uint32_t dense_bytes;  // the coarse levels' float2 entries, padded to 16 B
  DenseLevels dl;        // coarse levels: theta copy for the encode, then gradient accumulators
};

__host__ __device__ inline uint32_t al1k(uint32_t x) { return (x + 1023u) & ~1023u; }

inline Plan plan_for(const nirc_spec_t& sp, const TcNet& net) {
  Plan P{};
  P.w_off = 0;
  P.bias_off = al1k(net.wbytes);
  P.dzt_off = al1k(P.bias_off + kMaxTcLayers * 64 * 4);
  P.act_off = P.dzt_off + 2 * 8 * kChunk;               // dZt hi | lo (64 columns)
  P.act0_off = P.act_off + 2 * (kActCols / 8) * kChunk;  // act hi | lo (80 columns)
  P.dense_off = P.act0_off + 2 * (kAct0Cols / 8) * kChunk;
  const uint32_t stage_bytes = 64u * (kActCols + 1) * 4u;
  const uint32_t budget = 227u * 1024u - 6144u - stage_bytes - P.dense_off;
  P.dl = dense_levels_for(sp, budget, 4);
  P.dense_bytes = ((uint32_t)P.dl.off[P.dl.n] * 8u + 15u) & ~15u;
  P.stage_off = P.dense_off + P.dense_bytes;
  P.total = P.stage_off + stage_bytes;
  return P;
}

__host__ __device__ inline bool supported(const nirc_spec_t& sp) {
  if (!(sp.levels == 12 && sp.feats == 2 && sp.bands == 4 && sp.in_dim == 47 &&
        sp.dims[0] == 47))
    return false;
  if (sp.n_layers < 2 || sp.n_layers > kMaxNL) return false;
  for (int l = 1; l < sp.n_layers; ++l)
    if (sp.dims[l] != 64) return false;
  return sp.dims[sp.n_layers] >= 1 && sp.dims[sp.n_layers] <= 4;
}

// byte offset of (row r, 8-column chunk c) in a K-major [128 x K] operand
__device__ __forceinline__ uint32_t unit_off(int r, int c) {
  return (uint32_t)c * kChunk + (uint32_t)(r >> 3) * 128u + (uint32_t)(r & 7) * 16u;
}

__device__ __forceinline__ void st_unit(uint32_t addr, const uint32_t* v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3])
               : "memory");
}

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

__host__ __device__ constexpr uint32_t idesc_f16(int N, bool a_mn, bool b_mn) {
  return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kR >> 4) << 24);
}

// Forward layer 0 (SS): Z_0 += X W_0^T, X = act0 (K-major [128 x 48]).
__device__ __forceinline__ void issue_fwd0(const TcNet& net, uint32_t wbase, uint32_t act0,
                                           uint32_t d) {
  const int K = net.K[0], N = net.N[0];
  const uint32_t idesc = idesc_f16(N, false, false);
  const uint32_t w_hi = wbase + net.woff[0], w_lo = w_hi + (uint32_t)(N * K * 2);
  const uint32_t a_hi = act0, a_lo = act0 + (kAct0Cols / 8) * kChunk, w_lbo = (uint32_t)N * 16;
#pragma unroll
  for (int term = 0; term < 3; ++term) {
    const uint32_t A = term == 1 ? a_lo : a_hi, Bw = term == 0 ? w_lo : w_hi;
    for (int kk = 0; kk < K / 16; ++kk)
      mma_f16(d, sdesc(A + kk * 2 * kChunk, kChunk, 128), sdesc(Bw + kk * 2 * w_lbo, w_lbo, 128),
              idesc, 1u);
  }
}

// Forward layer l >= 1 (TS): Z_l += A W_l^T with A = relu(Z_{l-1}) in TMEM;
// every MMA accumulates onto the bias prefilled in Z_l.
__device__ __forceinline__ void issue_fwd_ts(const TcNet& net, int l, uint32_t wbase,
                                             uint32_t a_tmem, uint32_t d) {
  const int K = net.K[l], N = net.N[l];
  const uint32_t idesc = idesc_f16(N, false, false);
  const uint32_t w_hi = wbase + net.woff[l], w_lo = w_hi + (uint32_t)(N * K * 2);
  const uint32_t w_lbo = (uint32_t)N * 16;
#pragma unroll
  for (int term = 0; term < 3; ++term) {
    const uint32_t A = a_tmem + (term == 1 ? 32u : 0u), Bw = term == 0 ? w_lo : w_hi;
    for (int kk = 0; kk < K / 16; ++kk)
      mma_f16_ts(d, A + kk * 8, sdesc(Bw + kk * 2 * w_lbo, w_lbo, 128), idesc, 1u);
  }
}

// dA_{l-1} (or dX for l = 0) = dZ_l W_l: A = row-scaled dZ_l in TMEM (K =
// the layer's padded dout), B = W_l's K-major image read as its transposed
// (MN-major) view: SBO = the image's 8-column chunk (N_img * 16 B), LBO =
// 128 B (8 image rows).
__device__ __forceinline__ void issue_dA(const TcNet& net, int l, uint32_t wbase, uint32_t a_tmem,
                                         uint32_t d, int N) {
  const int Nimg = net.N[l], Kimg = net.K[l];
  const uint32_t idesc = idesc_f16(N, false, true);
  const uint32_t w_hi = wbase + net.woff[l], w_lo = w_hi + (uint32_t)(Nimg * Kimg * 2);
  const uint32_t sbo = (uint32_t)Nimg * 16;
  uint32_t acc = 0;
#pragma unroll
  for (int term = 0; term < 3; ++term) {
    const uint32_t A = a_tmem + (term == 1 ? 32u : 0u), Bw = term == 0 ? w_lo : w_hi;
    for (int kk = 0; kk < Nimg / 16; ++kk) {
      mma_f16_ts(d, A + kk * 8, sdesc(Bw + kk * 256, 128, sbo), idesc, acc);
      acc = 1;
    }
  }
}

// [dW_l | db_l] = dZt^T [A_{l-1} | 1]: both operands transposed views
// (SBO = 2 KB, LBO = 128 B), K = the tile's 128 rows; M = 128 with the rows
// >= dout don't-care.
__device__ __forceinline__ void issue_dW(uint32_t dzt, uint32_t act, uint32_t act_lo_off,
                                         uint32_t d, int N) {
  const uint32_t idesc = idesc_f16(N, true, true);
  const uint32_t z_hi = dzt, z_lo = dzt + 8 * kChunk;
  const uint32_t a_hi = act, a_lo = act + act_lo_off;
  uint32_t acc = 0;
#pragma unroll
  for (int term = 0; term < 3; ++term) {
    const uint32_t A = term == 1 ? z_lo : z_hi, Bx = term == 0 ? a_lo : a_hi;
    for (int kk = 0; kk < kR / 16; ++kk) {
      mma_f16(d, sdesc(A + kk * 256, 128, kChunk), sdesc(Bx + kk * 256, 128, kChunk), idesc, acc);
      acc = 1;
    }
  }
}

// 2^(14 - e(max)) and its inverse from the bit pattern of a max |value|
// (positive floats order as integers); 1 for an all-zero row / column.
__device__ __forceinline__ void pow2_scale(uint32_t maxbits, float& s, float& inv) {
  int e = (int)(maxbits >> 23);
  if (maxbits == 0u) e = 127 + 14;
  int se = 127 + 127 + 14 - e, ie = e - 14;
  se = se < 1 ? 1 : (se > 254 ? 254 : se);
  ie = ie < 1 ? 1 : (ie > 254 ? 254 : ie);
  s = __int_as_float(se << 23);
  inv = __int_as_float(ie << 23);
}

__device__ __forceinline__ float relu(float z) { return z > 0.0f ? z : 0.0f; }

// phase timestamps of CTA 0 / thread 0 (tools/kprof-style probes only)
#define TTC_PROBE(k)                                                   \
  do {                                                                 \
    if (prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0) prof[k] = clock64(); \
  } while (0)
// encode sub-phases of threads 0 (h = 0) and 128 (h = 1): slots 48.. / 56..
#define TTC_PROBE_E(k, dep)                                                              \
  do {                                                                                   \
    if (prof != nullptr && blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 128)) { \
      asm volatile("" ::"r"(__float_as_uint(dep)));                                      \
      prof[48 + (threadIdx.x == 128 ? 8 : 0) + (k)] = clock64();                        \
    }                                                                                    \
  } while (0)

// 32 fp32 values -> 4 K-major 16-byte units of hi and lo (chunks c0..c0+3)
template <int NU>
__device__ __forceinline__ void put_units(uint32_t base_hi, uint32_t lo_off, int r, int c0,
                                          const float* v) {
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    uint32_t hh[4], ll[4];
    PrecF16x2::split8(v + 8 * u, hh, ll);
    const uint32_t o = unit_off(r, c0 + u);
    st_unit(base_hi + o, hh);
    st_unit(base_hi + lo_off + o, ll);
  }
}

// One level's two hash features (4 bytes of hi and of lo fp16) into act0:
// X column 2 lvl, 2 lvl + 1 = chunk lvl / 4, slot lvl % 4.
__device__ __forceinline__ void put_level(uint32_t act0, uint32_t lo_off, int r, int lvl,
                                          float2 f) {
  const __half2 hi = __floats2half2_rn(f.x, f.y);
  const float2 hf = __half22float2(hi);
  const __half2 lo = __floats2half2_rn(f.x - hf.x, f.y - hf.y);
  const uint32_t o = unit_off(r, lvl >> 2) + 4u * (uint32_t)(lvl & 3);
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(act0 + o), "r"(*reinterpret_cast<const uint32_t*>(&hi))
               : "memory");
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(act0 + lo_off + o),
               "r"(*reinterpret_cast<const uint32_t*>(&lo))
               : "memory");
}

// Per-record, theta-independent part of the encoding (computed once per
// frame for all its optimizer steps): the normalised position u (f64
// affine + clamp, then f32, encoding.py:49-66), the SH block (f64
// recurrences -> f32, bit-identical to encode_batch) and the aux block
// (encoding.py:94-101), plus the constant 1 of dW_0's bias column.
// Layout per record (28 floats): u.xyz, 0 | SH[16] | aux[7], 1.
__global__ void k_record_static(nirc_spec_t sp, nirc_records_t rec, float4* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rec.n) return;
  float v[28];
  const double* p = rec.pos + 3 * i;
  v[0] = norm_coord(p[0], sp.bb_min[0], sp.bb_inv[0]);
  v[1] = norm_coord(p[1], sp.bb_min[1], sp.bb_inv[1]);
  v[2] = norm_coord(p[2], sp.bb_min[2], sp.bb_inv[2]);
  v[3] = 0.0f;
  const double* d = rec.dirs + 3 * i;
  sh_eval<true>(d[0], d[1], d[2], 4, sp.sh_k,
                [&](int k, double x) { v[4 + k] = __double2float_rn(x); });
  const double* nn = rec.ns + 3 * i;
  const double* al = rec.alb + 3 * i;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    v[20 + c] = __double2float_rn(dmul(dadd(nn[c], 1.0), 0.5));
    v[23 + c] = __double2float_rn(al[c]);
  }
  v[26] = __double2float_rn(rec.rough[i]);
  v[27] = 1.0f;
#pragma unroll
  for (int k = 0; k < kStat4; ++k)
    out[i * kStat4 + k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
}

// Per optimizer step (theta changes every step): the F16x2 weight images
// and biases (k_pack_weights' layout), the fp16-range flag, and a dense copy
// of the coarse hash levels -- dense[off_l + (z R + y) R + x] = table_l[
// hash(x, y, z)] (R = res + 2) -- that the tiles TMA into shared memory, so
// no tile gathers the few hot cache lines of the coarse levels from L2.
__global__ void k_train_prepare(nirc_spec_t sp, TcNet net, DenseLevels dl,
                                const float* __restrict__ theta, uint8_t* __restrict__ img,
                                float* __restrict__ bias, int32_t* __restrict__ unsafe,
                                float2* __restrict__ dense, uint32_t* __restrict__ dslot,
                                float4* __restrict__ zero_a, int64_t n_zero_a,
                                float4* __restrict__ zero_b, int64_t n_zero_b,
                                int32_t* __restrict__ zero_c, int32_t* __restrict__ zero_d) {
  // the step's zero-initialised buffers (grid gradient, fixed-point
  // accumulators, fix-up count, Adam's bad flag): no separate memsets
  {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = g; i < n_zero_a; i += stride) zero_a[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = g; i < n_zero_b; i += stride) zero_b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (g == 0) {
      if (zero_c) *zero_c = 0;
      if (zero_d) *zero_d = 0;
    }
  }
  int nw = 0;
  for (int l = 0; l < net.nl; ++l) nw += net.N[l] * net.K[l];
  const int nb = net.nl * 64, nd = dl.off[dl.n];
  const uint32_t T = 1u << sp.table_log2;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nw + nb + nd;
       t += gridDim.x * blockDim.x) {
    if (t < nw) {
      int l = 0, base = 0;
      while (t >= base + net.N[l] * net.K[l]) {
        base += net.N[l] * net.K[l];
        ++l;
      }
      const int e = t - base, nrow = e / net.K[l], k = e - nrow * net.K[l];
      const int din = sp.dims[l], dout = sp.dims[l + 1];
      const float w = (nrow < dout && k < din) ? theta[sp.w_off[l] + (int64_t)nrow * din + k] : 0.0f;
      if (!(fabsf(w) < kF16Max)) atomicExch(unsafe, 1);
      const __half hi = __float2half_rn(w);
      const __half lo = __float2half_rn(w - __half2float(hi));
      const uint32_t o = op_offset<PrecF16x2>(nrow, k, net.N[l]);
      *reinterpret_cast<__half*>(img + net.woff[l] + o) = hi;
      *reinterpret_cast<__half*>(img + net.woff[l] + net.N[l] * net.K[l] * 2 + o) = lo;
    } else if (t < nw + nb) {
      const int l = (t - nw) / 64, j = (t - nw) % 64;
      bias[t - nw] = j < sp.dims[l + 1] ? theta[sp.b_off[l] + j] : 0.0f;
    } else {
      const int i = t - nw - nb;
      int l = 0;
      while (i >= dl.off[l + 1]) ++l;
      const int R = dl.R[l], e = i - dl.off[l];
      const int x = e % R, y = (e / R) % R, z = e / (R * R);
      const uint32_t slot = hash3((uint32_t)x, (uint32_t)y, (uint32_t)z, T - 1u);
      dense[i] = reinterpret_cast<const float2*>(theta + (size_t)l * T * 2)[slot];
      dslot[i] = (uint32_t)l * T + slot;  // the scatter's flush target (level-major slot)
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_train_tc(nirc_spec_t sp, TcNet net, Plan P, const uint8_t* __restrict__ wimg,
               const float* __restrict__ bias_g, const int32_t* __restrict__ w_unsafe,
               const float2* __restrict__ dense_g, const uint32_t* __restrict__ dslot,
               const float* __restrict__ theta,
               const float4* __restrict__ rstat, nirc_records_t rec,
               const int64_t* __restrict__ idx, int64_t B, int loss_kind, double loss_eps,
               float* __restrict__ grad, float* __restrict__ partials,
               double* __restrict__ loss_part, int32_t* __restrict__ flags, int64_t tile0,
               int32_t* __restrict__ fix, float* __restrict__ dx_out,
               uint32_t* __restrict__ lvlmax, float* __restrict__ dbg,
               long long* __restrict__ prof) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t s_rmax[kSplit][kR];
  __shared__ float s_dzo[4][kR];
  __shared__ uint32_t s_cmax[2][64];
  __shared__ double s_loss[kThreads / 32];
  __shared__ __align__(8) uint64_t s_bar[3];
  __shared__ uint32_t s_tmem;
  if (flags[0] & 3) return;  // an earlier step diverged / saw a bad pdf
  // thread (row r, quarter h): warp w reaches TMEM lanes 32 (w % 4) ..; the
  // four warps of a lane quadrant split every row's columns / levels
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, q = w & 3, h = w >> 2;
  const int r = 32 * q + lane;
  const uint32_t lane_off = (uint32_t)(32 * q) << 16;
  const int64_t tile = tile0 + blockIdx.x;
  const int64_t row = tile * kR + r;
  const bool live = row < B;
  const int NL = net.nl;
  const uint32_t s0 = smem_u32(smem);
  const uint32_t wbar = smem_u32(&s_bar[0]), mbar_a = smem_u32(&s_bar[1]),
                 mbar_w = smem_u32(&s_bar[2]);
  const uint32_t w_base = s0 + P.w_off, dzt = s0 + P.dzt_off, act = s0 + P.act_off,
                 act0 = s0 + P.act0_off;
  const uint32_t act_lo = (kActCols / 8) * kChunk, act0_lo = (kAct0Cols / 8) * kChunk;
  float* s_bias = reinterpret_cast<float*>(smem + P.bias_off);
  float2* dense = reinterpret_cast<float2*>(smem + P.dense_off);
  float* stage = reinterpret_cast<float*>(smem + P.stage_off);
  constexpr int kSt = kActCols + 1;  // staging row stride (floats)
  // ---- prologue: barriers, TMEM, weights + coarse levels (TMA) -------------
  if (tid == 0) {
    mbar_init(wbar, 1);
    mbar_init(mbar_a, 1);
    mbar_init(mbar_w, 1);
    mbar_init_fence();
  }
  if (w == 0) tmem_alloc(smem_u32(&s_tmem), kTmemCols);
  for (int i = tid; i < NL * 64; i += kThreads) s_bias[i] = bias_g[i];
  if (tid < kR) {  // constant columns 64..79 of act: [1, 0, ...] (db_l), lo all zero
    const uint32_t one[4] = {0x3C00u, 0u, 0u, 0u}, zero[4] = {0u, 0u, 0u, 0u};
    st_unit(act + unit_off(tid, 8), one);
    st_unit(act + unit_off(tid, 9), zero);
    st_unit(act + act_lo + unit_off(tid, 8), zero);
    st_unit(act + act_lo + unit_off(tid, 9), zero);
    reinterpret_cast<uint32_t*>(s_cmax)[tid] = 0u;
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = s_tmem;
  TTC_PROBE(0);
  if (tid == 0) {
    mbar_expect_tx(wbar, net.wbytes + P.dense_bytes);
    for (uint32_t off = 0; off < net.wbytes; off += 32768u) {
      const uint32_t sz = net.wbytes - off < 32768u ? net.wbytes - off : 32768u;
      bulk_g2s(w_base + off, wimg + off, sz, wbar);
    }
    if (P.dense_bytes) bulk_g2s(s0 + P.dense_off, dense_g, P.dense_bytes, wbar);
  }
  // ---- encode (bit-exact X): h = 0 -> coarse levels 0-3 from the shared
  // copy + the record's static SH / aux block; h = 1, 2, 3 -> the fine
  // levels {4,5,6}, {7,8,9}, {10,11} from the L2-resident tables
  const uint32_t T = 1u << sp.table_log2;
  int64_t ri = 0;
  float ux = 0.f, uy = 0.f, uz = 0.f;
  TTC_PROBE_E(0, 0.0f);
  if (live) {
    ri = idx[row];
    TTC_PROBE_E(1, (float)ri);
    const float4 u = rstat[ri * kStat4];
    ux = u.x;
    uy = u.y;
    uz = u.z;
  }
  TTC_PROBE_E(2, ux);
  bool unsafe = *w_unsafe != 0;
  {
    const int l0 = h == 0 ? 0 : (h == 1 ? 4 : (h == 2 ? 7 : 10));
    const int nl = h == 0 ? 4 : (h == 3 ? 2 : 3);
    float xv[24];
#pragma unroll
    for (int i = 0; i < 24; ++i) xv[i] = 0.0f;
    if (h == 0) {
      if (live) {
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const float4 v = rstat[ri * kStat4 + 1 + k];
          xv[4 * k] = v.x;
          xv[4 * k + 1] = v.y;
          xv[4 * k + 2] = v.z;
          xv[4 * k + 3] = v.w;
        }
      }
      xv[23] = 1.0f;  // X column 47: the ones column of dW_0 (W_0's pad is 0)
      TTC_PROBE_E(3, xv[0]);
      put_units<3>(act0, act0_lo, r, 3, xv);
      mbar_wait(wbar, 0);  // the coarse levels have landed
      TTC_PROBE_E(4, 0.0f);
    }
    float2 f[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      f[k] = make_float2(0.f, 0.f);
      const int lvl = l0 + k;
      if (k < nl && live) {
        const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
        f[k] = lvl < P.dl.n ? level_features2_dense(dense + P.dl.off[lvl], P.dl.R[lvl], c)
                            : level_features2(theta + (size_t)lvl * T * 2, c, T - 1u);
      }
    }
    TTC_PROBE_E(5, f[0].x + f[1].x + f[2].x + f[3].x);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < nl) {
        put_level(act0, act0_lo, r, l0 + k, f[k]);
        unsafe |= !(fabsf(f[k].x) < kF16Max) || !(fabsf(f[k].y) < kF16Max);
      }
    unsafe |= f16_unsafe(xv, 24);
    if (dbg && live) {  // debug dump (tools/train_debug.py): X in input order
      float* d = dbg + row * kDbgStride;
      for (int k = 0; k < nl; ++k) {
        d[2 * (l0 + k)] = f[k].x;
        d[2 * (l0 + k) + 1] = f[k].y;
      }
      if (h == 0)
        for (int i = 0; i < 24; ++i) d[24 + i] = xv[i];
    }
  }
  TTC_PROBE(1);
  // bias of layer 0 -> Z_0 (the MMAs accumulate on top of it)
  {
    float b[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) b[j] = s_bias[16 * h + j];
    tmem_st16(tm + lane_off + 16 * h, b);
  }
  tmem_wait_st();
  fence_proxy_async();
  fence_before();
  __syncthreads();
  uint32_t ph_a = 0, ph_w = 0;
  if (w == 0) {
    fence_after();
    mbar_wait(wbar, 0);
    TTC_PROBE(2);
    if (elect_one()) {
      issue_fwd0(net, w_base, act0, tm);
      mma_commit(mbar_a);
    }
    __syncwarp();
  }
  // the shared coarse-level copy is dead after the encode: it becomes the
  // tile's coarse-level gradient accumulator
  if (dx_out == nullptr)
    for (int i = tid; i < P.dl.off[P.dl.n]; i += kThreads) dense[i] = make_float2(0.f, 0.f);
  // ---- forward: Z_l (hidden) stays in TMEM as the backward's stash ---------
  for (int l = 0; l < NL - 1; ++l) {
    mbar_wait(mbar_a, ph_a);
    ph_a ^= 1u;
    TTC_PROBE(3 + l);
    fence_after();
    float v[16];
    tmem_ld16(tm + lane_off + 64 * l + 16 * h, v);
    tmem_wait_ld();
    if (dbg && live)
      for (int j = 0; j < 16; ++j) dbg[row * kDbgStride + 48 + 64 * l + 16 * h + j] = v[j];
    float mx = 0.0f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      v[j] = relu(v[j]);
      mx = fmaxf(mx, v[j]);
    }
    unsafe |= !(mx < kF16Max);
    uint32_t hh[8], ll[8];
    PrecF16x2::split8(v, hh, ll);
    PrecF16x2::split8(v + 8, hh + 4, ll + 4);
    tmem_st8u(tm + lane_off + kColAop + 8 * h, hh);
    tmem_st8u(tm + lane_off + kColAop + 32 + 8 * h, ll);
    // bias of layer l + 1 -> its accumulator
    const bool last = l + 1 == NL - 1;
    const uint32_t dcol = last ? kColDA : 64u * (l + 1);
    if (!last || h == 0) {
      float b[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) b[j] = s_bias[(l + 1) * 64 + (last ? 0 : 16 * h) + j];
      tmem_st16(tm + lane_off + dcol + (last ? 0 : 16 * h), b);
    }
    tmem_wait_st();
    fence_before();
    __syncthreads();
    if (w == 0) {
      fence_after();
      if (elect_one()) {
        issue_fwd_ts(net, l + 1, w_base, tm + kColAop, tm + dcol);
        mma_commit(mbar_a);
      }
      __syncwarp();
    }
  }
  mbar_wait(mbar_a, ph_a);
  ph_a ^= 1u;
  TTC_PROBE(8);
  fence_after();
  float o[4];
  tmem_ld4(tm + lane_off + kColDA, o);
  tmem_wait_ld();
  if (dbg && live && h == 0)
    for (int j = 0; j < 4; ++j) dbg[row * kDbgStride + 304 + j] = o[j];
  if (dbg && live && unsafe) dbg[row * kDbgStride + 308] = 1.0f;
  // fp16 range guard: the whole tile goes to the fp32 kernel instead
  if (__syncthreads_or(unsafe)) {
    if (tid == 0) fix[1 + atomicAdd(fix, 1)] = (int32_t)tile;
    fence_before();
    __syncthreads();
    if (w == 0) {
      fence_after();
      tmem_dealloc(tm, kTmemCols);
    }
    return;
  }
  // ---- loss gradient (losses.py:23-42, f64, the reference's promotions):
  // output j of row r by thread h = j
  const int dout = sp.dims[NL];
  {
    double lsum = 0.0;
    float g = 0.0f;
    if (live && h < dout) {
      const double pdf = rec.pdf[ri];
      if (h == 0 && !(pdf > 0.0)) atomicOr(flags, 1);
      const double n_total = (double)(B * 3);
      float z = o[0];
#pragma unroll
      for (int j = 1; j < 4; ++j)
        if (h == j) z = o[j];
      const float yf = sp.out_act == 0 ? relu(z) : 1.0f / (1.0f + expf(-z));
      const double yd = (double)yf, t = rec.target[3 * ri + h];
      const double diff = dsub(yd, t);
      double gd;
      if (loss_kind == 0) {
        lsum = ddiv(dmul(diff, diff), pdf);
        gd = ddiv(ddiv(dmul(2.0, diff), pdf), n_total);
      } else {
        const float den32 = __fadd_rn(__fmul_rn(yf, yf), (float)loss_eps);
        const double den = dmul(pdf, (double)den32);
        lsum = ddiv(dmul(diff, diff), den);
        gd = ddiv(ddiv(dmul(2.0, diff), den), n_total);
      }
      const float gf = __double2float_rn(gd);
      g = sp.out_act == 0 ? (z >= 0.0f ? gf : 0.0f) : gf * yf * (1.0f - yf);
    }
    s_dzo[h][r] = g;
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) lsum += __shfl_down_sync(0xffffffffu, lsum, o2);
    if (lane == 0) s_loss[w] = lsum;
  }
  __syncthreads();
  TTC_PROBE(9);
  // ---- backward --------------------------------------------------------------
  // dz: this thread's 16 columns of dZ_l (the output layer's <= 16 columns
  // all belong to h = 0).  Per layer: maxima -> scales -> operands -> MMAs
  // (dA and dW committed separately: the dW MMA runs under the dA epilogue
  // and the next layer's maxima) -> staged, coalesced dW / db partials.
  float* wpart = partials + (int64_t)blockIdx.x * part_stride(sp);
  float dz[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) dz[j] = 0.0f;
  if (h == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) dz[j] = s_dzo[j][r];
  }
  if (tid == 0) {
    double t = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) t += s_loss[k];
    loss_part[blockIdx.x] = t;  // deterministic tile loss partial
  }
  // maxima of dZ_out -> s_rmax / s_cmax[(NL - 1) & 1]
  auto maxima = [&](int l) {
    const bool owns = l != NL - 1 || h == 0;
    const int c0 = l == NL - 1 ? 0 : 16 * h;
    uint32_t rm = 0u;
#pragma unroll
    for (int j = 0; j < 16; ++j) rm = max(rm, __float_as_uint(fabsf(dz[j])));
    s_rmax[h][r] = rm;
    uint32_t mine = 0u;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const uint32_t v = __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(dz[c])));
      if (lane == c) mine = v;
    }
    if (owns && lane < 16) atomicMax(&s_cmax[l & 1][c0 + lane], mine);
  };
  auto flush_stage = [&](int l) {  // staged [dW_l | db_l] -> the tile's partials
    // one warp per row j: the row's din weights are contiguous in theta
    const int din = sp.dims[l], dl_out = sp.dims[l + 1];
    float* wg = wpart + (sp.w_off[l] - sp.grid_len);
    for (int j = w; j < dl_out; j += kThreads / 32) {
      const float* srow = stage + j * kSt;
      for (int i = lane; i < din; i += 32) wg[j * din + i] = srow[i];
      if (lane == 0) wpart[(sp.b_off[l] - sp.grid_len) + j] = srow[din];
    }
  };
  maxima(NL - 1);
  __syncthreads();
  float dxv[6];
  for (int l = NL - 1; l >= 0; --l) {
    const bool out_layer = l == NL - 1;
    const bool owns = !out_layer || h == 0;
    const int c0 = out_layer ? 0 : 16 * h;
    uint32_t* cm = s_cmax[l & 1];
    TTC_PROBE(10 + 5 * l);
    float srow, irow;
    pow2_scale(max(max(s_rmax[0][r], s_rmax[1][r]), max(s_rmax[2][r], s_rmax[3][r])), srow, irow);
    if (!out_layer) flush_stage(l + 1);
    if (tid < 64) s_cmax[(l + 1) & 1][tid] = 0u;  // layer l - 1's buffer (read last by l + 1)
    // (B) operands: row-scaled dZ -> TMEM (dA), column-scaled dZ -> dZt (dW);
    // dZt / act are free: layer l + 1's dW MMA completed before the barrier
    if (owns) {
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = dz[j] * srow;
      uint32_t hh[8], ll[8];
      PrecF16x2::split8(v, hh, ll);
      PrecF16x2::split8(v + 8, hh + 4, ll + 4);
      tmem_st8u(tm + lane_off + kColAop + c0 / 2, hh);
      tmem_st8u(tm + lane_off + kColAop + 32 + c0 / 2, ll);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float sc, inv;
        pow2_scale(cm[c0 + j], sc, inv);
        v[j] = dz[j] * sc;
      }
      put_units<2>(dzt, 8 * kChunk, r, c0 / 8, v);
    }
    // a_{l-1} = relu(Z_{l-1}) -> act (l >= 1; layer 0 reads X from act0)
    float zprev[16];
    if (l >= 1) {
      tmem_ld16(tm + lane_off + 64 * (l - 1) + 16 * h, zprev);
      tmem_wait_ld();
      float a[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) a[j] = relu(zprev[j]);
      put_units<2>(act, act_lo, r, 2 * h, a);
    }
    tmem_wait_st();
    fence_proxy_async();
    fence_before();
    TTC_PROBE(11 + 5 * l);
    __syncthreads();
    if (w == 0) {
      fence_after();
      if (elect_one()) {
        issue_dA(net, l, w_base, tm + kColAop, tm + kColDA, l == 0 ? 32 : 64);
        mma_commit(mbar_a);
        issue_dW(dzt, l == 0 ? act0 : act, l == 0 ? act0_lo : act_lo, tm + kColDW,
                 l == 0 ? kAct0Cols : kActCols);
        mma_commit(mbar_w);
      }
      __syncwarp();
    }
    // (C) dA -> dz of layer l - 1 (ReLU' = z >= 0, mlp.py:149), or dX for l = 0
    mbar_wait(mbar_a, ph_a);
    ph_a ^= 1u;
    TTC_PROBE(12 + 5 * l);
    fence_after();
    {
      float v[32];
      if (l >= 1) {
        tmem_ld16(tm + lane_off + kColDA + 16 * h, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) dz[j] = zprev[j] >= 0.0f ? v[j] * irow : 0.0f;
        maxima(l - 1);  // next layer's scales, under the dW MMA
      } else {  // this thread's scatter levels h, h + 4, h + 8
        tmem_ld32(tm + lane_off + kColDA, v);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          float a0 = 0.f, a1 = 0.f;
#pragma unroll
          for (int hh = 0; hh < 4; ++hh)
            if (h == hh) {
              a0 = v[2 * (hh + 4 * k)];
              a1 = v[2 * (hh + 4 * k) + 1];
            }
          dxv[2 * k] = a0 * irow;
          dxv[2 * k + 1] = a1 * irow;
        }
      }
    }
    // (D) [dW | db] rows j < dout of the dW accumulator -> staging (x 1 / c_j)
    mbar_wait(mbar_w, ph_w);
    ph_w ^= 1u;
    fence_after();
    if (q < 2) {
      const int per = (l == 0 ? kAct0Cols : kActCols) / kSplit;  // 12 | 20 columns
      const int j = 32 * q + lane;
      float v[20];
#pragma unroll
      for (int k = 0; k < 5; ++k)
        if (4 * k < per) tmem_ld4(tm + lane_off + kColDW + per * h + 4 * k, v + 4 * k);
      tmem_wait_ld();
      if (j < sp.dims[l + 1]) {
        float sc, inv;
        pow2_scale(cm[j], sc, inv);
#pragma unroll
        for (int t = 0; t < 20; ++t)
          if (t < per) stage[j * kSt + per * h + t] = v[t] * inv;
      }
    }
    fence_before();
    TTC_PROBE(13 + 5 * l);
    __syncthreads();
  }
  flush_stage(0);
  TTC_PROBE(40);
  if (dbg && live)
    for (int k = 0; k < 3; ++k) {
      dbg[row * kDbgStride + 312 + 2 * (h + 4 * k)] = dxv[2 * k];
      dbg[row * kDbgStride + 312 + 2 * (h + 4 * k) + 1] = dxv[2 * k + 1];
    }
  // ---- hash-grid scatter (encoding.py:160-167): levels h, h + 4, h + 8 ------
  if (dx_out != nullptr) {  // deterministic mode: the rows' grid gradients + level maxima
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (live) {
        dx_out[row * 24 + 2 * (h + 4 * k)] = dxv[2 * k];
        dx_out[row * 24 + 2 * (h + 4 * k) + 1] = dxv[2 * k + 1];
      }
      const uint32_t m = __reduce_max_sync(
          0xffffffffu, max(__float_as_uint(fabsf(dxv[2 * k])), __float_as_uint(fabsf(dxv[2 * k + 1]))));
      if (lane == 0) atomicMax(lvlmax + h + 4 * k, m);
    }
  } else if (live) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int lvl = h + 4 * k;
      const float d0 = dxv[2 * k], d1 = dxv[2 * k + 1];
      if (d0 == 0.0f && d1 == 0.0f) continue;
      const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
      if (lvl < P.dl.n) {  // coarse level: shared-memory accumulator per grid vertex
        const int R = P.dl.R[lvl];
        float2* base = dense + P.dl.off[lvl] + (c.iz * R + c.iy) * R + c.ix;
#pragma unroll
        for (int kc = 0; kc < 8; ++kc) {
          const float wk = corner_weight(c, kc);
          float2* a = base + (kc & 1) + ((kc >> 1) & 1) * R + ((kc >> 2) & 1) * R * R;
          atomicAdd(&a->x, __fmul_rn(wk, d0));
          atomicAdd(&a->y, __fmul_rn(wk, d1));
        }
      } else {
        float* gl = grad + (size_t)lvl * T * 2;
#pragma unroll
        for (int kc = 0; kc < 8; kc += 2) {
          const float w0 = corner_weight(c, kc), w1 = corner_weight(c, kc + 1);
          const uint32_t h0 = corner_hash(c, kc, T - 1u), h1 = corner_hash(c, kc + 1, T - 1u);
          if ((c.ix & 1) == 0) {  // x even: the x-neighbour is slot h0 ^ 1 -> one 16-byte RED
            const float a0 = __fmul_rn(w0, d0), a1 = __fmul_rn(w0, d1);
            const float b0 = __fmul_rn(w1, d0), b1 = __fmul_rn(w1, d1);
            const float4 v4 = (h0 & 1u) ? make_float4(b0, b1, a0, a1) : make_float4(a0, a1, b0, b1);
            atomicAdd(reinterpret_cast<float4*>(gl + 2 * (h0 & ~1u)), v4);
          } else {
            atomicAdd(reinterpret_cast<float2*>(gl + 2 * h0),
                      make_float2(__fmul_rn(w0, d0), __fmul_rn(w0, d1)));
            atomicAdd(reinterpret_cast<float2*>(gl + 2 * h1),
                      make_float2(__fmul_rn(w1, d0), __fmul_rn(w1, d1)));
          }
        }
      }
    }
  }
  fence_before();
  TTC_PROBE(41);
  __syncthreads();
  TTC_PROBE(42);
  if (dx_out == nullptr) {  // flush the coarse levels: one RED per touched vertex
    for (int i = tid; i < P.dl.off[P.dl.n]; i += kThreads) {
      const float2 v = dense[i];
      if (v.x != 0.0f || v.y != 0.0f)
        atomicAdd(reinterpret_cast<float2*>(grad) + dslot[i], v);
    }
  }
  TTC_PROBE(43);
  if (w == 0) {
    fence_after();
    tmem_dealloc(tm, kTmemCols);
  }
}

}  // namespace ttc

float* g_train_dbg = nullptr;       // tools only: nirc_debug_train_probe
long long* g_train_prof = nullptr;  // tools only: nirc_debug_train_phases

bool train_tc_supported(const nirc_spec_t& sp) {
  if (!ttc::supported(sp)) return false;
  tc::TcNet net;
  if (!tc::tc_net_for(sp, &net, tc::PrecF16x2::kId)) return false;
  return ttc::plan_for(sp, net).total + 6144u <= 227u * 1024u;
}

// theta-independent per-record encoding blocks (once per frame)
int64_t train_static_bytes(int64_t n) { return n * ttc::kStat4 * 16; }
int launch_record_static(const nirc_spec_t& sp, const nirc_records_t& rec, float* out,
                         cudaStream_t s) {
  if (rec.n <= 0) return NIRC_OK;
  ttc::k_record_static<<<(unsigned)((rec.n + 127) / 128), 128, 0, s>>>(
      sp, rec, reinterpret_cast<float4*>(out));
  NIRC_LAUNCH_CHECK("k_record_static");
  return NIRC_OK;
}

// Tiles [tile0, tile1) on tcgen05; tiles beyond the fp16 range are appended
// to `fix` (count + tile ids, caller-zeroed count) for the fp32 kernel.
int launch_train_tc(const nirc_spec_t& sp, const float* theta, const float* rstat,
                    const nirc_records_t& rec, const int64_t* idx, int64_t B, int loss_kind,
                    double loss_eps, float* grad, float* partials, double* loss_part,
                    int32_t* flags, cudaStream_t s, int64_t tile0, int64_t tile1, int32_t* fix,
                    float* dx_out, uint32_t* lvlmax, void* zero_b, int64_t zero_b_bytes,
                    int32_t* adam_bad) {
  tc::TcNet net;
  if (!tc::tc_net_for(sp, &net, tc::PrecF16x2::kId)) return NIRC_E_UNSUPPORTED;
  const ttc::Plan P = ttc::plan_for(sp, net);
  const int ntiles = (int)(tile1 - tile0);
  if (ntiles <= 0) return NIRC_OK;
  AsyncBuf buf(s);
  const size_t img_bytes = ((size_t)net.wbytes + 255) & ~(size_t)255;
  NIRC_CUDA_TRY(buf.alloc(img_bytes + tc::kMaxTcLayers * 64 * 4 + 256 + P.dense_bytes +
                          (size_t)P.dl.off[P.dl.n] * 4 + 16));
  uint8_t* img = static_cast<uint8_t*>(buf.p);
  float* bias = reinterpret_cast<float*>(img + img_bytes);
  int32_t* unsafe = reinterpret_cast<int32_t*>(bias + tc::kMaxTcLayers * 64);
  float2* dense = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(unsafe) + 256);
  uint32_t* dslot = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(dense) + P.dense_bytes);
  NIRC_CUDA_TRY(cudaMemsetAsync(unsafe, 0, 4, s));
  int total = P.dl.off[P.dl.n] + net.nl * 64;
  for (int l = 0; l < net.nl; ++l) total += net.N[l] * net.K[l];
  // grad's grid part is zeroed by the prepare kernel (atomic scatter target)
  const int64_t nza = sp.grid_len / 4, nzb = zero_b_bytes / 16;
  int64_t blocks = (total + 255) / 256;
  blocks = blocks < 4 * 148 ? 4 * 148 : blocks;
  ttc::k_train_prepare<<<(unsigned)blocks, 256, 0, s>>>(
      sp, net, P.dl, theta, img, bias, unsafe, dense, dslot, reinterpret_cast<float4*>(grad), nza,
      reinterpret_cast<float4*>(zero_b), nzb, fix, adam_bad);
  NIRC_LAUNCH_CHECK("k_train_prepare");
  NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)ttc::k_train_tc,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.total));
  ttc::k_train_tc<<<ntiles, ttc::kThreads, P.total, s>>>(
      sp, net, P, img, bias, unsafe, dense, dslot, theta, reinterpret_cast<const float4*>(rstat),
      rec, idx,
      B, loss_kind, loss_eps, grad, partials, loss_part, flags, tile0, fix, dx_out, lvlmax,
      g_train_dbg, g_train_prof);
  NIRC_LAUNCH_CHECK("k_train_tc");
  return NIRC_OK;
}

}  // namespace nirc

extern "C" void nirc_debug_train_probe(float* buf) { nirc::g_train_dbg = buf; }
extern "C" void nirc_debug_train_phases(long long* buf) { nirc::g_train_prof = buf; }
