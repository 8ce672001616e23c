// Fused online-training step (train_frame body, pkg/src/nirclab/caches.py:
// 330-350) for the l2 / relative-L2 losses: ONE kernel per optimizer step,
// one CTA of 512 threads per 128-row tile of the batch, four threads per row
// (each owns 16 of a hidden layer's 64 columns and 3 of the 12 hash levels):
//   encode (bit-exact, encoding.py:111-157) -> forward (mlp.py:102-122) ->
//   loss gradient (losses.py:23-42, f64) -> backward (mlp.py:125-154,
//   ReLU' = z >= 0) -> hash-grid scatter (encoding.py:160-167).
// Each thread keeps its column slice of the row's layer outputs / input
// gradients in registers and reads the weights as broadcast 16-byte
// shared-memory rows (W^T for the forward, W for the backward); every layer's
// pre-activations and the encoded input are stashed in TENSOR memory (the
// row's TMEM lane, 4 x 64 + 64 columns) instead of shared memory, which
// leaves room for both weight images and keeps the whole batch in one wave
// (B / 128 = 128 CTAs on 148 SMs, 16 warps each).  Weight/bias gradients are
// per-CTA partials from a shared-memory block GEMM over the tile's rows,
// summed in a fixed order by k_reduce_grad (deterministic); the hash-grid
// scatter is the one atomic (non-deterministic) sum.
//
// fp32 SIMT: the reference's accuracy class.
#include <cmath>
#include "common.cuh"
#include "tc_common.cuh"

namespace nirc {

constexpr int kTR = 128;         // rows per tile
#ifndef NIRC_TRAIN_SPLIT
#define NIRC_TRAIN_SPLIT 4
#endif
constexpr int kSplit = NIRC_TRAIN_SPLIT;  // threads per row (output column slices)
constexpr int kTT = kTR * kSplit;         // threads per CTA
constexpr int kLD2 = 132;        // row stride of the [feature][row] staging arrays
constexpr int kMaxW = 64;        // widest layer supported by the fused path
constexpr int kMaxNL = 8;

struct FusedLayout {
  int nl, din[kMaxNL], dout[kMaxNL];
  int ldw[kMaxNL], ldt[kMaxNL];    // row strides of W (dout x ldw) and W^T (din x ldt)
  int w_off[kMaxNL], t_off[kMaxNL], b_off[kMaxNL];  // float offsets in smem
  int dz_off, a_off, red_off, total_floats;
  int x_col, tmem_cols;            // TMEM: z of layer l at cols 64*l, X at x_col
};

__host__ __device__ inline int up4(int x) { return (x + 3) & ~3; }

__host__ __device__ inline FusedLayout fused_layout(const nirc_spec_t& sp) {
  FusedLayout L{};
  L.nl = sp.n_layers;
  int off = 0;
  for (int l = 0; l < sp.n_layers; ++l) {
    L.din[l] = sp.dims[l];
    L.dout[l] = sp.dims[l + 1];
    L.ldw[l] = up4(L.din[l]);
    L.ldt[l] = up4(L.dout[l]);
    L.w_off[l] = off;
    off += up4(L.dout[l]) * L.ldw[l];
    L.t_off[l] = off;
    off += up4(L.din[l]) * L.ldt[l];
    L.b_off[l] = off;
    off += kMaxW;
  }
  L.dz_off = off;
  off += kMaxW * kLD2;
  L.a_off = off;
  off += kMaxW * kLD2;
  L.red_off = off;
  off += 2 * kTT;  // f64 reduction scratch
  L.total_floats = off;
  L.x_col = (sp.n_layers - 1) * 64;
  int need = L.x_col + 64;
  int c = 32;
  while (c < need) c <<= 1;
  L.tmem_cols = c;
  return L;
}

bool fused_supported(const nirc_spec_t& sp) {
  if (sp.n_layers < 2 || sp.n_layers > kMaxNL || sp.in_dim > kMaxW || sp.feats != 2 ||
      sp.levels > 12)
    return false;
  for (int l = 1; l < sp.n_layers; ++l)
    if (sp.dims[l] > kMaxW) return false;
  if (sp.dims[sp.n_layers] > 4) return false;
  return fused_layout(sp).tmem_cols <= 512;
}

size_t fused_smem_bytes(const nirc_spec_t& sp) {
  return (size_t)fused_layout(sp).total_floats * 4 + 16;
}

__device__ __forceinline__ float relu(float z) { return z > 0.0f ? z : 0.0f; }

// Thread (r, h): row r of the tile, column slice h (columns kCols*h ..).
constexpr int kCols = kMaxW / kSplit;   // hidden columns per thread
constexpr int kLvl = 12 / kSplit;       // hash levels per thread
constexpr int kDX = 2 * kLvl;           // encoded-grid gradient columns per thread

// out[j] = b[c0 + j] + sum_i in[i][r] * W[c0 + j][i], j < NOUT, c0 = column
// offset; the input column read from the staging array, W^T row segments as
// broadcast float4.
template <int NOUT>
__device__ __forceinline__ void row_forward(const float* __restrict__ in, int din,
                                            const float* __restrict__ WT, int ldt, int c0,
                                            const float* __restrict__ b, int r, float* out) {
#pragma unroll
  for (int j = 0; j < NOUT; ++j) out[j] = b[c0 + j];
#pragma unroll 2
  for (int i = 0; i < din; ++i) {
    const float ai = in[i * kLD2 + r];
    const float4* w = reinterpret_cast<const float4*>(WT + i * ldt + c0);
#pragma unroll
    for (int q = 0; q < NOUT / 4; ++q) {
      const float4 v = w[q];
      out[4 * q] = fmaf(ai, v.x, out[4 * q]);
      out[4 * q + 1] = fmaf(ai, v.y, out[4 * q + 1]);
      out[4 * q + 2] = fmaf(ai, v.z, out[4 * q + 2]);
      out[4 * q + 3] = fmaf(ai, v.w, out[4 * q + 3]);
    }
  }
}

// da[i] = sum_j dz[j][r] * W[j][c0 + i], i < NIN.
template <int NIN>
__device__ __forceinline__ void row_backward(const float* __restrict__ dz, int dout,
                                             const float* __restrict__ W, int ldw, int c0, int r,
                                             float* da) {
#pragma unroll
  for (int i = 0; i < NIN; ++i) da[i] = 0.0f;
#pragma unroll 2
  for (int j = 0; j < dout; ++j) {
    const float g = dz[j * kLD2 + r];
    if constexpr (NIN % 4 == 0) {
      const float4* w = reinterpret_cast<const float4*>(W + j * ldw + c0);
#pragma unroll
      for (int q = 0; q < NIN / 4; ++q) {
        const float4 v = w[q];
        da[4 * q] = fmaf(g, v.x, da[4 * q]);
        da[4 * q + 1] = fmaf(g, v.y, da[4 * q + 1]);
        da[4 * q + 2] = fmaf(g, v.z, da[4 * q + 2]);
        da[4 * q + 3] = fmaf(g, v.w, da[4 * q + 3]);
      }
    } else {
      const float2* w = reinterpret_cast<const float2*>(W + j * ldw + c0);
#pragma unroll
      for (int q = 0; q < NIN / 2; ++q) {
        const float2 v = w[q];
        da[2 * q] = fmaf(g, v.x, da[2 * q]);
        da[2 * q + 1] = fmaf(g, v.y, da[2 * q + 1]);
      }
    }
  }
}

// Per-CTA partial dW[j][i] = sum_r dz[j][r] a[i][r], db[j] = sum_r dz[j][r]:
// the threads as a kJG x 16 grid over the 64 x 64 outputs, kP x 4 each, rows
// in float4 steps.
constexpr int kJG = kTT / 16, kP = kMaxW / kJG;
__device__ __forceinline__ void tile_wgrad(const float* __restrict__ dz, int dout,
                                           const float* __restrict__ a, int din,
                                           float* __restrict__ part_w,
                                           float* __restrict__ part_b) {
  const int tid = threadIdx.x, jg = tid >> 4, ig = tid & 15;
  float acc[kP][4];
#pragma unroll
  for (int p = 0; p < kP; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[p][q] = 0.0f;
  if (jg < dout) {
    for (int r = 0; r < kTR; r += 4) {
      float4 g[kP], x[4];
#pragma unroll
      for (int p = 0; p < kP; ++p) {
        const int j = jg + kJG * p;
        g[p] = j < dout ? *reinterpret_cast<const float4*>(dz + j * kLD2 + r)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = ig + 16 * q;
        x[q] = i < din ? *reinterpret_cast<const float4*>(a + i * kLD2 + r)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int p = 0; p < kP; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[p][q] = fmaf(g[p].x, x[q].x, acc[p][q]);
          acc[p][q] = fmaf(g[p].y, x[q].y, acc[p][q]);
          acc[p][q] = fmaf(g[p].z, x[q].z, acc[p][q]);
          acc[p][q] = fmaf(g[p].w, x[q].w, acc[p][q]);
        }
    }
  }
#pragma unroll
  for (int p = 0; p < kP; ++p) {
    const int j = jg + kJG * p;
    if (j >= dout) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = ig + 16 * q;
      if (i < din) part_w[j * din + i] = acc[p][q];
    }
  }
  if (tid < dout) {
    float s = 0.0f;
    for (int r = 0; r < kTR; ++r) s += dz[tid * kLD2 + r];
    part_b[tid] = s;
  }
}

// kCols TMEM columns of this thread's lane <-> v[kCols]
__device__ __forceinline__ void tmem_put(uint32_t taddr, const float* v) {
#pragma unroll
  for (int c = 0; c < kCols; c += 16) tc::tmem_st16(taddr + c, v + c);
}
__device__ __forceinline__ void tmem_get(uint32_t taddr, float* v) {
  if constexpr (kCols == 32) {
    tc::tmem_ld32(taddr, v);
  } else {
#pragma unroll
    for (int c = 0; c < kCols; c += 16) tc::tmem_ld16(taddr + c, v + c);
  }
  tc::tmem_wait_ld();
}

// The step's weight image in the kernel's shared-memory layout: W (dout x
// ldw) and W^T (din x ldt) zero padded, and the biases, per layer -- built
// once per step so that every tile CTA stages it with TMA bulk copies.
__global__ void k_pack_train_weights(nirc_spec_t sp, FusedLayout L,
                                     const float* __restrict__ theta, float* __restrict__ img) {
  const int l = blockIdx.y;
  const float* Wg = theta + sp.w_off[l];
  const int din = L.din[l], dout = L.dout[l], ldw = L.ldw[l], ldt = L.ldt[l];
  const int nw = up4(dout) * ldw, nt = up4(din) * ldt;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nw + nt + kMaxW;
       e += gridDim.x * blockDim.x) {
    float v;
    if (e < nw) {
      const int j = e / ldw, i = e - j * ldw;
      v = (j < dout && i < din) ? Wg[j * din + i] : 0.0f;
      img[L.w_off[l] + e] = v;
    } else if (e < nw + nt) {
      const int i = (e - nw) / ldt, j = (e - nw) - i * ldt;
      v = (j < dout && i < din) ? Wg[j * din + i] : 0.0f;
      img[L.t_off[l] + (e - nw)] = v;
    } else {
      const int j = e - nw - nt;
      img[L.b_off[l] + j] = j < dout ? theta[sp.b_off[l] + j] : 0.0f;
    }
  }
}

// One 128-row tile of the batch per CTA (tiles tile0 + blockIdx.x); rows
// idx[tile*128 + r]; thread (r, h) = (tid & 127, tid >> 7).
__global__ void __launch_bounds__(kTT, 1)
    k_train_tile(nirc_spec_t sp, FusedLayout L, const float* __restrict__ theta,
                 const float* __restrict__ wimg, nirc_records_t rec,
                 const int64_t* __restrict__ idx, int64_t B, int loss_kind, double loss_eps,
                 float* __restrict__ grad, float* __restrict__ partials,
                 double* __restrict__ loss_part, int32_t* __restrict__ flags, int64_t tile0) {
  extern __shared__ __align__(16) float fsm[];
  __shared__ uint32_t tmem_holder;
  __shared__ __align__(8) uint64_t wbar;
  if (flags[0] & 3) return;
  const int tid = threadIdx.x;
  const int r = tid & (kTR - 1), h = tid / kTR;
  const int c0 = kCols * h;
  const int lane_base = ((tid >> 5) & 3) * 32;
  const int64_t row = (tile0 + blockIdx.x) * kTR + r;
  const bool live = row < B;
  // ---- weights: the step's image by TMA bulk copies, in flight during the
  // encode below (waited for before the forward) --------------------------
  const uint32_t wb = tc::smem_u32(&wbar);
  if (tid == 0) {
    tc::mbar_init(wb, 1);
    tc::mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t bytes = (uint32_t)L.dz_off * 4u;
    tc::mbar_expect_tx(wb, bytes);
    for (uint32_t off = 0; off < bytes; off += 32768u) {
      const uint32_t sz = bytes - off < 32768u ? bytes - off : 32768u;
      tc::bulk_g2s(tc::smem_u32(fsm) + off, reinterpret_cast<const uint8_t*>(wimg) + off, sz, wb);
    }
  }
  if (tid < 32) tc::tmem_alloc(tc::smem_u32(&tmem_holder), (uint32_t)L.tmem_cols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_holder + ((uint32_t)lane_base << 16);
  float* A = fsm + L.a_off;   // [feature][row]: the current layer's input
  float* DZ = fsm + L.dz_off;
  // ---- encode (bit-exact): levels kLvl*h ..; h == 0 also SH + aux ---------
  const uint32_t T = 1u << sp.table_log2;
  int64_t ri = 0;
  float ux = 0.0f, uy = 0.0f, uz = 0.0f;
  if (live) {
    ri = idx[row];
    const double* p = rec.pos + 3 * ri;
    ux = norm_coord(p[0], sp.bb_min[0], sp.bb_inv[0]);
    uy = norm_coord(p[1], sp.bb_min[1], sp.bb_inv[1]);
    uz = norm_coord(p[2], sp.bb_min[2], sp.bb_inv[2]);
  }
#pragma unroll
  for (int q = 0; q < kLvl; ++q) {
    const int lvl = kLvl * h + q;
    if (lvl < sp.levels) {
      float2 f = make_float2(0.0f, 0.0f);
      if (live) {
        const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
        f = level_features2(theta + (size_t)lvl * T * 2, c, T - 1u);
      }
      A[(2 * lvl) * kLD2 + r] = f.x;
      A[(2 * lvl + 1) * kLD2 + r] = f.y;
    }
  }
  if (h == 0) {
    const int g = sp.levels * 2;
    if (live) {
      const double* d = rec.dirs + 3 * ri;
      sh_eval<true>(d[0], d[1], d[2], sp.bands, sp.sh_k,
                    [&](int i, double v) { A[(g + i) * kLD2 + r] = __double2float_rn(v); });
      const int a0 = g + sp.bands * sp.bands;
      const double* nn = rec.ns + 3 * ri;
      const double* al = rec.alb + 3 * ri;
      for (int c = 0; c < 3; ++c) {
        A[(a0 + c) * kLD2 + r] = __double2float_rn(dmul(dadd(nn[c], 1.0), 0.5));
        A[(a0 + 3 + c) * kLD2 + r] = __double2float_rn(al[c]);
      }
      A[(a0 + 6) * kLD2 + r] = __double2float_rn(rec.rough[ri]);
    } else {
      for (int i = g; i < sp.in_dim; ++i) A[i * kLD2 + r] = 0.0f;
    }
  }
  __syncthreads();
  {  // the encoded row -> TMEM (layer 0's a_prev for its weight gradient)
    float x[kCols];
#pragma unroll
    for (int i = 0; i < kCols; ++i) x[i] = (c0 + i) < sp.in_dim ? A[(c0 + i) * kLD2 + r] : 0.0f;
    tmem_put(tbase + L.x_col + c0, x);
  }
  tc::mbar_wait(wb, 0);  // the weight image has landed
  // ---- forward: hidden layers stash z in TMEM, write relu(z) as next input
  const int NL = L.nl;
  for (int l = 0; l < NL - 1; ++l) {
    float z[kCols];
    row_forward<kCols>(A, L.din[l], fsm + L.t_off[l], L.ldt[l], c0, fsm + L.b_off[l], r, z);
    tmem_put(tbase + 64 * l + c0, z);
    __syncthreads();  // both halves finished reading this layer's input
#pragma unroll
    for (int j = 0; j < kCols; ++j) A[(c0 + j) * kLD2 + r] = relu(z[j]);
    __syncthreads();
  }
  float y[4];
  row_forward<4>(A, L.din[NL - 1], fsm + L.t_off[NL - 1], L.ldt[NL - 1], 0, fsm + L.b_off[NL - 1],
                 r, y);
  tc::tmem_wait_st();
  // ---- loss gradient (f64, the reference's promotions), half 0 ------------
  const int dout = L.dout[NL - 1];
  double lsum = 0.0;
  if (h == 0) {
    if (live) {
      const double pdf = rec.pdf[ri];
      if (!(pdf > 0.0)) atomicOr(flags, 1);
      const double n_total = (double)(B * 3);
      for (int j = 0; j < dout; ++j) {
        const float z = y[j];
        const float yf = sp.out_act == 0 ? (z > 0.0f ? z : 0.0f) : 1.0f / (1.0f + expf(-z));
        const double yd = (double)yf, t = rec.target[3 * ri + j];
        const double diff = dsub(yd, t);
        double g, v;
        if (loss_kind == 0) {
          v = ddiv(dmul(diff, diff), pdf);
          g = ddiv(ddiv(dmul(2.0, diff), pdf), n_total);
        } else {
          const float den32 = __fadd_rn(__fmul_rn(yf, yf), (float)loss_eps);
          const double den = dmul(pdf, (double)den32);
          v = ddiv(dmul(diff, diff), den);
          g = ddiv(ddiv(dmul(2.0, diff), den), n_total);
        }
        lsum += v;
        const float gf = __double2float_rn(g);
        DZ[j * kLD2 + r] = sp.out_act == 0 ? (z >= 0.0f ? gf : 0.0f) : gf * yf * (1.0f - yf);
      }
    } else {
      for (int j = 0; j < dout; ++j) DZ[j * kLD2 + r] = 0.0f;
    }
  }
  // deterministic per-tile loss partial (fixed shuffle tree per warp, then
  // the warp sums in order)
  double* red = reinterpret_cast<double*>(fsm + L.red_off);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_down_sync(0xffffffffu, lsum, o);
  if ((tid & 31) == 0) red[tid >> 5] = lsum;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kTT / 32; ++w) t += red[w];
    loss_part[blockIdx.x] = t;
  }
  // ---- backward ----------------------------------------------------------
  float* wpart = partials + (int64_t)blockIdx.x * (sp.theta_len - sp.grid_len);
  float dX[kDX];
  for (int l = NL - 1; l >= 0; --l) {
    {  // a_prev of layer l -> staging (relu(z_{l-1}) or the encoded input)
      float v[kCols];
      tmem_get(tbase + (l == 0 ? L.x_col : 64 * (l - 1)) + c0, v);
#pragma unroll
      for (int i = 0; i < kCols; ++i)
        if (c0 + i < L.din[l]) A[(c0 + i) * kLD2 + r] = l == 0 ? v[i] : relu(v[i]);
    }
    __syncthreads();  // DZ (layer l's dz) and A complete for the block GEMM
    tile_wgrad(DZ, L.dout[l], A, L.din[l], wpart + (sp.w_off[l] - sp.grid_len),
               wpart + (sp.b_off[l] - sp.grid_len));
    if (l > 0) {
      float da[kCols];
      row_backward<kCols>(DZ, L.dout[l], fsm + L.w_off[l], L.ldw[l], c0, r, da);
      float zp[kCols];
      tmem_get(tbase + 64 * (l - 1) + c0, zp);
      __syncthreads();  // everyone finished reading DZ / A of layer l
#pragma unroll
      for (int i = 0; i < kCols; ++i) DZ[(c0 + i) * kLD2 + r] = zp[i] >= 0.0f ? da[i] : 0.0f;
    } else {
      row_backward<kDX>(DZ, L.dout[0], fsm + L.w_off[0], L.ldw[0], kDX * h, r, dX);
    }
  }
  // ---- hash-grid scatter (encoding.py:160-167), levels kLvl*h .. ----------
  if (live) {
#pragma unroll
    for (int q = 0; q < kLvl; ++q) {
      const int lvl = kLvl * h + q;
      if (lvl >= sp.levels) continue;
      const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
      float* gl = grad + (size_t)lvl * T * 2;
      const float d0 = dX[2 * q], d1 = dX[2 * q + 1];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float w = corner_weight(c, k);
        const uint32_t hh = corner_hash(c, k, T - 1u);
        if (d0 != 0.0f || d1 != 0.0f)  // one 8-byte vector RED per corner
          atomicAdd(reinterpret_cast<float2*>(gl + 2 * hh),
                    make_float2(__fmul_rn(w, d0), __fmul_rn(w, d1)));
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (tid < 32) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_holder, (uint32_t)L.tmem_cols);
  }
}

// grad[mlp] = sum over tiles (tile order) of the partials.
// mode 0 (whole batch on this GPU): loss = mean; flags: 2 = non-finite loss
//   (stop), adam_bad = any non-finite gradient.
// mode 1 (one shard of a multi-GPU batch): aux[0] = this shard's raw loss
//   sum, aux[1] = 1 if a row of this shard had pdf <= 0; the finiteness
//   checks run after the cross-GPU sum (nirc_train_apply).
__global__ void k_reduce_grad(nirc_spec_t sp, const float* __restrict__ partials, int ntiles,
                              const double* __restrict__ loss_part, int64_t B,
                              float* __restrict__ grad, double* __restrict__ loss_out,
                              int32_t* __restrict__ flags, int32_t* __restrict__ adam_bad,
                              int mode) {
  if (mode == 0 && (flags[0] & 3)) return;
  // block = 8 warps x 32 consecutive parameters; warp w sums a contiguous
  // chunk of tiles, the 8 chunk sums are added in warp order (deterministic)
  __shared__ float part[8][33];
  const int np = (int)(sp.theta_len - sp.grid_len);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int per = (ntiles + 7) / 8;
  const int t0 = wid * per, t1 = min(ntiles, t0 + per);
  int bad = 0;
  for (int pb = blockIdx.x * 32; pb < np; pb += gridDim.x * 32) {
    const int p = pb + lane;
    float s = 0.0f;
    if (p < np) {
#pragma unroll 8
      for (int t = t0; t < t1; ++t) s += partials[(int64_t)t * np + p];
    }
    part[wid][lane] = s;
    __syncthreads();
    if (wid == 0 && p < np) {
      float tot = part[0][lane];
      for (int w = 1; w < 8; ++w) tot += part[w][lane];
      grad[sp.grid_len + p] = tot;
      bad |= !isfinite(tot);
    }
    __syncthreads();
  }
  if (mode == 1) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      double s = 0.0;
      for (int t = 0; t < ntiles; ++t) s += loss_part[t];
      loss_out[0] = s;
      loss_out[1] = (flags[0] & 1) ? 1.0 : 0.0;
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sp.grid_len;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(grad[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(adam_bad, 1);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int t = 0; t < ntiles; ++t) s += loss_part[t];
    const double v = s / (double)(B * 3);
    loss_out[0] = v;
    if (!isfinite(v)) atomicOr(flags, 2);
  }
}


// Tiles [tile0, tile1) of the batch (all of it on one GPU; one shard of it
// per GPU in the multi-GPU frame, mode 1).
int launch_fused_train(const nirc_spec_t& sp, const float* theta, const nirc_records_t& rec,
                       const int64_t* idx, int64_t B, int loss_kind, double loss_eps,
                       float* grad, float* partials, double* loss_part, double* loss_out,
                       int32_t* flags, int32_t* adam_bad, cudaStream_t s, int64_t tile0,
                       int64_t tile1, int mode) {
  const FusedLayout L = fused_layout(sp);
  const size_t sm = (size_t)L.total_floats * 4;
  NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)k_train_tile,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const int ntiles = (int)(tile1 > tile0 ? tile1 - tile0 : 0);
  NIRC_CUDA_TRY(cudaMemsetAsync(grad, 0, sp.grid_len * 4, s));
  if (adam_bad) NIRC_CUDA_TRY(cudaMemsetAsync(adam_bad, 0, 4, s));
  AsyncBuf img(s);
  if (ntiles > 0) {
    NIRC_CUDA_TRY(img.alloc((size_t)L.dz_off * 4));
    k_pack_train_weights<<<dim3(16, L.nl), 256, 0, s>>>(sp, L, theta,
                                                       static_cast<float*>(img.p));
    NIRC_LAUNCH_CHECK("k_pack_train_weights");
    k_train_tile<<<ntiles, kTT, sm, s>>>(sp, L, theta, static_cast<const float*>(img.p), rec,
                                         idx, B, loss_kind, loss_eps, grad, partials, loss_part,
                                         flags, tile0);
    NIRC_LAUNCH_CHECK("k_train_tile");
  }
  const int np = (int)(sp.theta_len - sp.grid_len);
  k_reduce_grad<<<(np + 31) / 32, 256, 0, s>>>(sp, partials, ntiles, loss_part, B, grad, loss_out,
                                               flags, adam_bad, mode);
  NIRC_LAUNCH_CHECK("k_reduce_grad");
  return NIRC_OK;
}

}  // namespace nirc
