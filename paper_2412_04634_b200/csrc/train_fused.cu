// Fused online-training step (train_frame body, pkg/src/nirclab/caches.py:
// 330-350) for the l2 / relative-L2 losses: ONE kernel per optimizer step
// runs, per 64-row tile of the batch,
//   encode (bit-exact, encoding.py:111-157) -> forward with pre-activation
//   stash (mlp.py:102-122) -> loss gradient (losses.py:23-42, f64) ->
//   backward (mlp.py:125-154, ReLU' = z >= 0) -> hash-grid scatter
//   (encoding.py:160-167) straight from registers,
// keeping every activation in shared memory.  Weight/bias gradients are
// written as per-CTA partials and summed in a fixed order by k_reduce_grad
// (deterministic), which also folds the loss, flags a non-finite loss
// (DivergenceError) or gradient (Adam skip) and feeds the dense Adam kernels.
//
// fp32 SIMT, register-blocked 4x4 micro-tiles: all GEMMs here are 64 wide
// and the batch is 16384 rows, so the step is latency- not FLOP-bound.
#include <cmath>
#include "common.cuh"

namespace nirc {

constexpr int kTR = 64;          // rows per tile
constexpr int kTT = 256;         // threads per CTA
constexpr int kLDR = 68;         // row stride of [feature][row] arrays (68/4 odd)
constexpr int kMaxW = 64;        // widest layer supported by the fused path

struct FusedLayout {
  int nl, din[8], dout[8], ldw[8];
  int woff[8], boff[8];          // float offsets in the smem weight block
  int wfloats;                   // weight block size (floats)
  int x_off, z_off[8], dz_off[2], dy_off, red_off, total_floats;
};

__host__ __device__ inline FusedLayout fused_layout(const nirc_spec_t& sp) {
  FusedLayout L{};
  L.nl = sp.n_layers;
  int off = 0;
  for (int l = 0; l < sp.n_layers; ++l) {
    L.din[l] = sp.dims[l];
    L.dout[l] = sp.dims[l + 1];
    L.ldw[l] = sp.dims[l] | 1;  // odd stride: strided-column loads hit distinct banks
    L.woff[l] = off;
    off += L.dout[l] * L.ldw[l];
    L.boff[l] = off;
    off += (L.dout[l] + 3) & ~3;
  }
  L.wfloats = (off + 3) & ~3;
  int f = L.wfloats;
  L.x_off = f;
  f += sp.in_dim * kLDR;
  for (int l = 0; l < sp.n_layers; ++l) {
    L.z_off[l] = f;
    f += L.dout[l] * kLDR;
  }
  L.dz_off[0] = f;
  f += kMaxW * kLDR;
  L.dz_off[1] = f;
  f += kMaxW * kLDR;
  L.dy_off = f;
  f += 4 * kLDR;
  L.red_off = f;
  f += kTT * 2;  // f64 reduction scratch (as 2 floats each)
  L.total_floats = f;
  return L;
}

bool fused_supported(const nirc_spec_t& sp) {
  if (sp.n_layers > 8 || sp.in_dim > kMaxW || sp.feats != 2) return false;
  for (int l = 1; l <= sp.n_layers; ++l)
    if (sp.dims[l] > kMaxW) return false;
  return sp.dims[sp.n_layers] <= 4;
}

__device__ inline float act_hidden(float z) { return z > 0.0f ? z : 0.0f; }

// out[j][r] (+)= sum_i in[i][r] * W[j][i] (+ b[j]) over a 64-row tile.
// Thread (rg, cg): rows 4rg..4rg+3, outputs cg + 16q.  `relu_in` applies
// max(.,0) to the stashed pre-activations on the fly.
__device__ inline void tile_gemm_fwd(const float* __restrict__ in, int din, bool relu_in,
                                     const float* __restrict__ W, int ldw,
                                     const float* __restrict__ b, int dout,
                                     float* __restrict__ out) {
  const int tid = threadIdx.x, rg = tid >> 4, cg = tid & 15;
  float acc[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[q][r] = 0.0f;
  for (int i = 0; i < din; ++i) {
    float4 a = *reinterpret_cast<const float4*>(in + i * kLDR + 4 * rg);
    if (relu_in) {
      a.x = act_hidden(a.x);
      a.y = act_hidden(a.y);
      a.z = act_hidden(a.z);
      a.w = act_hidden(a.w);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = cg + 16 * q;
      const float w = j < dout ? W[j * ldw + i] : 0.0f;
      acc[q][0] = fmaf(a.x, w, acc[q][0]);
      acc[q][1] = fmaf(a.y, w, acc[q][1]);
      acc[q][2] = fmaf(a.z, w, acc[q][2]);
      acc[q][3] = fmaf(a.w, w, acc[q][3]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = cg + 16 * q;
    if (j < dout) {
      const float bj = b[j];
      float4 o;
      o.x = acc[q][0] + bj;
      o.y = acc[q][1] + bj;
      o.z = acc[q][2] + bj;
      o.w = acc[q][3] + bj;
      *reinterpret_cast<float4*>(out + j * kLDR + 4 * rg) = o;
    }
  }
}

// da[i][r] = sum_j dz[j][r] W[j][i]; optionally masked by (z_prev[i][r] >= 0).
__device__ inline void tile_gemm_bwd(const float* __restrict__ dz, int dout,
                                     const float* __restrict__ W, int ldw, int din,
                                     const float* __restrict__ zprev, float* __restrict__ out) {
  const int tid = threadIdx.x, rg = tid >> 4, ig = tid & 15;
  float acc[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[q][r] = 0.0f;
  for (int j = 0; j < dout; ++j) {
    const float4 g = *reinterpret_cast<const float4*>(dz + j * kLDR + 4 * rg);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = ig + 16 * q;
      const float w = i < din ? W[j * ldw + i] : 0.0f;
      acc[q][0] = fmaf(g.x, w, acc[q][0]);
      acc[q][1] = fmaf(g.y, w, acc[q][1]);
      acc[q][2] = fmaf(g.z, w, acc[q][2]);
      acc[q][3] = fmaf(g.w, w, acc[q][3]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = ig + 16 * q;
    if (i < din) {
      float4 o = make_float4(acc[q][0], acc[q][1], acc[q][2], acc[q][3]);
      if (zprev) {
        const float4 z = *reinterpret_cast<const float4*>(zprev + i * kLDR + 4 * rg);
        o.x = z.x >= 0.0f ? o.x : 0.0f;
        o.y = z.y >= 0.0f ? o.y : 0.0f;
        o.z = z.z >= 0.0f ? o.z : 0.0f;
        o.w = z.w >= 0.0f ? o.w : 0.0f;
      }
      *reinterpret_cast<float4*>(out + i * kLDR + 4 * rg) = o;
    }
  }
}

// Per-CTA partial dW[j][i] = sum_r dz[j][r] a[i][r] and db[j] = sum_r dz[j][r].
__device__ inline void tile_wgrad(const float* __restrict__ dz, int dout,
                                  const float* __restrict__ a, bool relu_a, int din, int nrows,
                                  float* __restrict__ part_w, float* __restrict__ part_b) {
  const int tid = threadIdx.x, jg = tid >> 4, ig = tid & 15;
  float acc[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[p][q] = 0.0f;
  for (int r = 0; r < nrows; r += 4) {
    float4 g[4], x[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int j = jg + 16 * p;
      g[p] = j < dout ? *reinterpret_cast<const float4*>(dz + j * kLDR + r)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = ig + 16 * q;
      float4 v = i < din ? *reinterpret_cast<const float4*>(a + i * kLDR + r)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      if (relu_a) {
        v.x = act_hidden(v.x);
        v.y = act_hidden(v.y);
        v.z = act_hidden(v.z);
        v.w = act_hidden(v.w);
      }
      x[q] = v;
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[p][q] = fmaf(g[p].x, x[q].x, acc[p][q]);
        acc[p][q] = fmaf(g[p].y, x[q].y, acc[p][q]);
        acc[p][q] = fmaf(g[p].z, x[q].z, acc[p][q]);
        acc[p][q] = fmaf(g[p].w, x[q].w, acc[p][q]);
      }
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int j = jg + 16 * p;
    if (j >= dout) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = ig + 16 * q;
      if (i < din) part_w[j * din + i] = acc[p][q];
    }
  }
  if (tid < dout) {
    float s = 0.0f;
    for (int r = 0; r < nrows; ++r) s += dz[tid * kLDR + r];
    part_b[tid] = s;
  }
}

// One 64-row tile of the batch per CTA.  rec rows idx[tile*64 + r].
__global__ void __launch_bounds__(kTT, 1)
    k_train_tile(nirc_spec_t sp, FusedLayout L, const float* __restrict__ theta,
                 nirc_records_t rec, const int64_t* __restrict__ idx, int64_t B, int loss_kind,
                 double loss_eps, float* __restrict__ grad, float* __restrict__ partials,
                 double* __restrict__ loss_part, int32_t* __restrict__ flags, int64_t tile0) {
  extern __shared__ __align__(16) float fsm[];
  if (flags[0] & 3) return;
  const int tid = threadIdx.x;
  const int64_t row0 = (tile0 + blockIdx.x) * kTR;
  const int nrows = (int)((B - row0) < kTR ? (B - row0) : kTR);
  // ---- stage the network (odd-stride rows) ---------------------------------
  for (int l = 0; l < L.nl; ++l) {
    const float* Wg = theta + sp.w_off[l];
    for (int e = tid; e < L.dout[l] * L.din[l]; e += kTT) {
      const int j = e / L.din[l], i = e % L.din[l];
      fsm[L.woff[l] + j * L.ldw[l] + i] = Wg[e];
    }
    for (int j = tid; j < L.dout[l]; j += kTT) fsm[L.boff[l] + j] = theta[sp.b_off[l] + j];
  }
  // ---- encode: thread (row r, part p) does levels 3p..3p+2; p == 0 also SH+aux
  const int r = tid & 63, part = tid >> 6;
  float* X = fsm + L.x_off;
  LevelCell cells[3];
  const bool live = r < nrows;
  int64_t ri = 0;
  const uint32_t T = 1u << sp.table_log2;
  if (live) {
    ri = idx[row0 + r];
    const double* p = rec.pos + 3 * ri;
    const float ux = norm_coord(p[0], sp.bb_min[0], sp.bb_inv[0]);
    const float uy = norm_coord(p[1], sp.bb_min[1], sp.bb_inv[1]);
    const float uz = norm_coord(p[2], sp.bb_min[2], sp.bb_inv[2]);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int lvl = 3 * part + q;
      if (lvl < sp.levels) {
        cells[q] = level_cell(ux, uy, uz, sp.res[lvl]);
        const float2 f = level_features2(theta + (size_t)lvl * T * 2, cells[q], T - 1u);
        X[(2 * lvl) * kLDR + r] = f.x;
        X[(2 * lvl + 1) * kLDR + r] = f.y;
      }
    }
    if (part == 0) {
      const int g = sp.levels * 2;
      const double* d = rec.dirs + 3 * ri;
      sh_eval<true>(d[0], d[1], d[2], sp.bands, sp.sh_k,
                    [&](int i, double v) { X[(g + i) * kLDR + r] = __double2float_rn(v); });
      const int a0 = g + sp.bands * sp.bands;
      const double* nn = rec.ns + 3 * ri;
      const double* al = rec.alb + 3 * ri;
      for (int c = 0; c < 3; ++c) {
        X[(a0 + c) * kLDR + r] = __double2float_rn(dmul(dadd(nn[c], 1.0), 0.5));
        X[(a0 + 3 + c) * kLDR + r] = __double2float_rn(al[c]);
      }
      X[(a0 + 6) * kLDR + r] = __double2float_rn(rec.rough[ri]);
    }
  } else if (part == 0) {
    for (int i = 0; i < sp.in_dim; ++i) X[i * kLDR + r] = 0.0f;
  }
  __syncthreads();
  // ---- forward, stashing every pre-activation -----------------------------
  const int NL = L.nl;
  for (int l = 0; l < NL; ++l) {
    const float* in = l == 0 ? X : fsm + L.z_off[l - 1];
    tile_gemm_fwd(in, L.din[l], l > 0, fsm + L.woff[l], L.ldw[l], fsm + L.boff[l], L.dout[l],
                  fsm + L.z_off[l]);
    __syncthreads();
  }
  // ---- loss gradient (f64, the reference's promotions) --------------------
  const int dout = L.dout[NL - 1];
  const float* zo = fsm + L.z_off[NL - 1];
  float* dz = fsm + L.dz_off[0];
  double lsum = 0.0;
  if (tid < kTR) {
    const int rr = tid;
    if (rr < nrows) {
      const int64_t rj = idx[row0 + rr];
      const double pdf = rec.pdf[rj];
      if (!(pdf > 0.0)) atomicOr(flags, 1);
      const double n_total = (double)(B * 3);
      for (int j = 0; j < dout; ++j) {
        const float z = zo[j * kLDR + rr];
        const float yf = sp.out_act == 0 ? (z > 0.0f ? z : 0.0f) : 1.0f / (1.0f + expf(-z));
        const double y = (double)yf, t = rec.target[3 * rj + j];
        const double diff = dsub(y, t);
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
        float gz;
        if (sp.out_act == 0) gz = z >= 0.0f ? gf : 0.0f;
        else gz = gf * yf * (1.0f - yf);
        dz[j * kLDR + rr] = gz;
      }
    } else {
      for (int j = 0; j < dout; ++j) dz[j * kLDR + rr] = 0.0f;
    }
  }
  // deterministic per-tile loss partial (tree over the 64 row threads)
  double* red = reinterpret_cast<double*>(fsm + L.red_off);
  red[tid] = lsum;
  __syncthreads();
  for (int s = kTT / 2; s > 0; s >>= 1) {
    if (tid < s) red[tid] += red[tid + s];
    __syncthreads();
  }
  if (tid == 0) loss_part[blockIdx.x] = red[0];
  // ---- backward ----------------------------------------------------------
  float* wpart = partials + (int64_t)blockIdx.x * (sp.theta_len - sp.grid_len);
  int cur = 0;
  float dX[3][2];
  for (int l = NL - 1; l >= 0; --l) {
    float* dzc = fsm + L.dz_off[cur];
    const float* a_prev = l == 0 ? X : fsm + L.z_off[l - 1];
    tile_wgrad(dzc, L.dout[l], a_prev, l > 0, L.din[l], kTR,
               wpart + (sp.w_off[l] - sp.grid_len), wpart + (sp.b_off[l] - sp.grid_len));
    if (l > 0) {
      tile_gemm_bwd(dzc, L.dout[l], fsm + L.woff[l], L.ldw[l], L.din[l], fsm + L.z_off[l - 1],
                    fsm + L.dz_off[1 - cur]);
      __syncthreads();
      cur = 1 - cur;
    } else {
      // dX for the hash-grid block only: thread (r, part) needs its 3 levels
      const float* W0 = fsm + L.woff[0];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int lvl = 3 * part + q;
        float s0 = 0.0f, s1 = 0.0f;
        if (lvl < sp.levels)
          for (int j = 0; j < L.dout[0]; ++j) {
            const float g = dzc[j * kLDR + r];
            s0 = fmaf(g, W0[j * L.ldw[0] + 2 * lvl], s0);
            s1 = fmaf(g, W0[j * L.ldw[0] + 2 * lvl + 1], s1);
          }
        dX[q][0] = s0;
        dX[q][1] = s1;
      }
    }
  }
  // ---- hash-grid scatter (encoding.py:160-167) from registers -------------
  if (live) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int lvl = 3 * part + q;
      if (lvl >= sp.levels) continue;
      float* gl = grad + (size_t)lvl * T * 2;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float w = corner_weight(cells[q], k);
        const uint32_t h = corner_hash(cells[q], k, T - 1u);
        if (dX[q][0] != 0.0f) atomicAdd(gl + 2 * h, __fmul_rn(w, dX[q][0]));
        if (dX[q][1] != 0.0f) atomicAdd(gl + 2 * h + 1, __fmul_rn(w, dX[q][1]));
      }
    }
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

size_t fused_smem_bytes(const nirc_spec_t& sp) {
  return (size_t)fused_layout(sp).total_floats * 4;
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
  if (ntiles > 0) {
    k_train_tile<<<ntiles, kTT, sm, s>>>(sp, L, theta, rec, idx, B, loss_kind, loss_eps, grad,
                                         partials, loss_part, flags, tile0);
    NIRC_LAUNCH_CHECK("k_train_tile");
  }
  const int np = (int)(sp.theta_len - sp.grid_len);
  k_reduce_grad<<<(np + 31) / 32, 256, 0, s>>>(sp, partials, ntiles, loss_part, B, grad, loss_out,
                                               flags, adam_bad, mode);
  NIRC_LAUNCH_CHECK("k_reduce_grad");
  return NIRC_OK;
}

}  // namespace nirc
