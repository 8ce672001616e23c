// NIRC neural substrate on sm_100a: encoding, fp32 SIMT network twin,
// losses, backward + hash-grid scatter, dense Adam, and the fused online
// training step.  Reference: pkg/src/nirclab/{encoding,mlp,losses,adam,
// caches}.py (file:line cited per function).
#include <cstdio>
#include <cstring>
#include <cmath>
#include <climits>
#include "common.cuh"

namespace nirc {

constexpr int kRowsPerBlock = 128;

// ----------------------------------------------------------------------
// Encoding of one row into a caller-provided store functor.
// encode_batch (encoding.py:111-157): hash block [0, L*F), SH block
// [L*F, L*F+bands^2), aux block (n+1)/2, albedo, rough.
// ----------------------------------------------------------------------
template <typename StoreX>
__device__ void encode_row(const nirc_spec_t& sp, const float* __restrict__ theta,
                           const double* p, const double* nrm, const double* alb,
                           double rough, const double* d, StoreX store,
                           int64_t* __restrict__ ent, float* __restrict__ wts) {
  const float ux = norm_coord(p[0], sp.bb_min[0], sp.bb_inv[0]);
  const float uy = norm_coord(p[1], sp.bb_min[1], sp.bb_inv[1]);
  const float uz = norm_coord(p[2], sp.bb_min[2], sp.bb_inv[2]);
  const uint32_t T = 1u << sp.table_log2;
  const uint32_t mask = T - 1u;
  const int F = sp.feats;
  for (int lvl = 0; lvl < sp.levels; ++lvl) {
    const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
    const float* table = theta + (int64_t)lvl * T * F;
    if (F == 2 && ent == nullptr) {
      const float2 x = level_features2(table, c, mask);
      store(lvl * 2, x.x);
      store(lvl * 2 + 1, x.y);
    } else {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int k = 0; k < 8; ++k) {
        const float w = corner_weight(c, k);
        const uint32_t h = corner_hash(c, k, mask);
        if (ent) {
          ent[lvl * 8 + k] = (int64_t)lvl * T + h;
          wts[lvl * 8 + k] = w;
        }
        for (int f = 0; f < F && f < 4; ++f)
          acc[f] = __fadd_rn(acc[f], __fmul_rn(w, __ldg(table + (int64_t)h * F + f)));
      }
      for (int f = 0; f < F && f < 4; ++f) store(lvl * F + f, acc[f]);
    }
  }
  const int g = sp.levels * F;
  sh_eval<true>(d[0], d[1], d[2], sp.bands, sp.sh_k,
                [&](int i, double v) { store(g + i, __double2float_rn(v)); });
  const int a0 = g + sp.bands * sp.bands;
  store(a0 + 0, __double2float_rn(dmul(dadd(nrm[0], 1.0), 0.5)));
  store(a0 + 1, __double2float_rn(dmul(dadd(nrm[1], 1.0), 0.5)));
  store(a0 + 2, __double2float_rn(dmul(dadd(nrm[2], 1.0), 0.5)));
  store(a0 + 3, __double2float_rn(alb[0]));
  store(a0 + 4, __double2float_rn(alb[1]));
  store(a0 + 5, __double2float_rn(alb[2]));
  store(a0 + 6, __double2float_rn(rough));
}

__global__ void k_encode(nirc_spec_t sp, const float* __restrict__ theta,
                         const double* __restrict__ pos, const double* __restrict__ nrm,
                         const double* __restrict__ alb, const double* __restrict__ rough,
                         const double* __restrict__ dirs, int64_t n, float* __restrict__ X,
                         int64_t* __restrict__ entries, float* __restrict__ weights) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float* xr = X + i * sp.in_dim;
  encode_row(sp, theta, pos + 3 * i, nrm + 3 * i, alb + 3 * i, rough[i], dirs + 3 * i,
             [&](int k, float v) { xr[k] = v; },
             entries ? entries + i * sp.levels * 8 : nullptr,
             weights ? weights + i * sp.levels * 8 : nullptr);
}

// scatter_grid_grad (encoding.py:160-167).  np.add.at accumulates
// (w * dG) in row order; the device sums the same f32 products with
// atomics (order-free, tolerance stated in DESIGN.md).
__global__ void k_scatter(nirc_spec_t sp, float* __restrict__ grad,
                          const int64_t* __restrict__ entries, const float* __restrict__ weights,
                          const float* __restrict__ dX, int64_t n, int64_t stride) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = n * sp.levels * 8;
  if (t >= total) return;
  const int64_t row = t / (sp.levels * 8);
  const int lvl = (int)((t / 8) % sp.levels);
  const int64_t slot = entries[t];
  const float w = weights[t];
  for (int f = 0; f < sp.feats; ++f)
    atomicAdd(grad + slot * sp.feats + f, __fmul_rn(w, dX[row * stride + lvl * sp.feats + f]));
}

// ----------------------------------------------------------------------
// fp32 SIMT network twin: one thread per row, weights in shared memory,
// activations in a padded per-thread shared slab (stride dmax+1 words ->
// conflict-free).  mlp_forward (mlp.py:102-122) / mlp_forward_s
// (mlp.py:160-192): z = a W^T + b, ReLU hidden, ReLU or sigmoid output.
// ----------------------------------------------------------------------
__host__ __device__ inline int net_param_count(const nirc_spec_t& sp) {
  return (int)(sp.theta_len - sp.grid_len);
}
__host__ __device__ inline int net_dmax(const nirc_spec_t& sp) {
  int m = 0;
  for (int l = 0; l <= sp.n_layers; ++l) m = sp.dims[l] > m ? sp.dims[l] : m;
  return m;
}
__host__ __device__ inline int zs_width(const nirc_spec_t& sp) {
  int s = 0;
  for (int l = 1; l <= sp.n_layers; ++l) s += sp.dims[l];
  return s;
}
inline size_t simt_smem_bytes(const nirc_spec_t& sp) {
  return (size_t)net_param_count(sp) * 4 + (size_t)2 * kRowsPerBlock * (net_dmax(sp) + 1) * 4;
}

// Runs the network on the activation slab `a` (dmax+1 stride per thread)
// and returns the output in a (first dims[nl] entries).  W is the smem copy
// of theta[grid_len:].  zs (optional) receives every pre-activation.
__device__ inline void simt_forward_row(const nirc_spec_t& sp, const float* __restrict__ W,
                                        float* a, float* b, int stride, float* zs_row) {
  int zoff = 0;
  for (int l = 0; l < sp.n_layers; ++l) {
    const int din = sp.dims[l], dout = sp.dims[l + 1];
    const float* w = W + (sp.w_off[l] - sp.grid_len);
    const float* bias = W + (sp.b_off[l] - sp.grid_len);
    const bool last = (l == sp.n_layers - 1);
    for (int j = 0; j < dout; ++j) {
      const float* wr = w + j * din;
      float acc = 0.0f;
      for (int i = 0; i < din; ++i) acc = fmaf(a[i * stride], wr[i], acc);
      const float z = acc + bias[j];
      if (zs_row) zs_row[zoff + j] = z;
      float y;
      if (!last || sp.out_act == 0) y = z > 0.0f ? z : 0.0f;
      else y = 1.0f / (1.0f + expf(-z));
      b[j * stride] = y;
    }
    zoff += dout;
    float* t = a; a = b; b = t;
  }
  // the output sits in the caller's `b` slab for odd depth, `a` for even
}

__device__ inline void stage_params(const nirc_spec_t& sp, const float* __restrict__ theta,
                                    float* W) {
  const int np = net_param_count(sp);
  const float* src = theta + sp.grid_len;
  for (int i = threadIdx.x; i < np; i += blockDim.x) W[i] = __ldg(src + i);
}

__global__ void k_mlp_forward(nirc_spec_t sp, const float* __restrict__ theta,
                              const float* __restrict__ X, int64_t n, float* __restrict__ Y,
                              float* __restrict__ zs, int32_t* __restrict__ nonfinite) {
  extern __shared__ float smem[];
  float* W = smem;
  stage_params(sp, theta, W);
  if (nonfinite) {  // mlp.py:104-105 raises DivergenceError on any non-finite theta
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sp.theta_len;
         i += (int64_t)gridDim.x * blockDim.x)
      bad |= !isfinite(theta[i]);
    if (bad) atomicExch(nonfinite, 1);
  }
  const int dmax = net_dmax(sp);
  // thread t owns column t of two [dmax+1][128] slabs: a[i*128 + t]
  float* a = W + net_param_count(sp) + threadIdx.x;
  float* b = a + (dmax + 1) * kRowsPerBlock;
  __syncthreads();
  const int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + threadIdx.x;
  if (row >= n) return;
  for (int i = 0; i < sp.in_dim; ++i) a[i * kRowsPerBlock] = X[row * sp.in_dim + i];
  simt_forward_row(sp, W, a, b, kRowsPerBlock, zs ? zs + row * zs_width(sp) : nullptr);
  const float* out = (sp.n_layers % 2 == 1) ? b : a;
  const int dout = sp.dims[sp.n_layers];
  for (int j = 0; j < dout; ++j) Y[row * dout + j] = out[j * kRowsPerBlock];
}

// ----------------------------------------------------------------------
// Losses (losses.py:23-70).  Computed in f64 from the f32 prediction,
// exactly the reference's promotions: the relative-L2 denominator is
// f32(f32(y*y) + f32(eps)) (numpy NEP-50 weak scalar), everything else f64.
// Gradient = reference gradient cast to f32 (caches.py:349).
// ----------------------------------------------------------------------
constexpr int kLossThreads = 256;

__device__ inline double loss_elem(int kind, float yf, double t, double p, double rm,
                                   double eps, double n_total, float* dy) {
  const double y = (double)yf;
  switch (kind) {
    case 0: {  // loss_l2 :23-30
      const double diff = dsub(y, t);
      *dy = __double2float_rn(ddiv(ddiv(dmul(2.0, diff), p), n_total));
      return ddiv(dmul(diff, diff), p);
    }
    case 1: {  // loss_relative_l2 :33-42
      const float den32 = __fadd_rn(__fmul_rn(yf, yf), (float)eps);
      const double den = dmul(p, (double)den32);
      const double diff = dsub(y, t);
      *dy = __double2float_rn(ddiv(ddiv(dmul(2.0, diff), den), n_total));
      return ddiv(dmul(diff, diff), den);
    }
    case 2: {  // loss_variance :50-61
      const double dev = dsub(ddiv(dsub(t, y), p), rm);
      *dy = __double2float_rn(ddiv(ddiv(dmul(-2.0, dev), p), n_total));
      return dmul(dev, dev);
    }
    default: {  // loss_bce :64-70
      double q = y < 1e-6 ? 1e-6 : (y > 1.0 - 1e-6 ? 1.0 - 1e-6 : y);
      const double v = -(dadd(dmul(t, log(q)), dmul(dsub(1.0, t), log(dsub(1.0, q)))));
      *dy = __double2float_rn(ddiv(ddiv(dsub(q, t), dmul(q, dsub(1.0, q))), n_total));
      return v;
    }
  }
}

// Pass 1: per-block partial sums of the loss (and, for the variance loss,
// of (t - y)/pdf per channel when `dev_partial` is set).
__global__ void k_loss(int kind, const float* __restrict__ Y, const double* __restrict__ T,
                       const double* __restrict__ pdf, const double* __restrict__ rmean,
                       double eps, int64_t n, float* __restrict__ dY,
                       double* __restrict__ partial, int32_t* __restrict__ flags,
                       const int64_t* __restrict__ idx, int dev_pass) {
  __shared__ double red[kLossThreads][3];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc[3] = {0.0, 0.0, 0.0};
  if (flags && (flags[0] & 2)) return;  // an earlier step diverged
  if (i < n) {
    const int64_t r = idx ? idx[i] : i;
    const double p = kind == 3 ? 1.0 : pdf[r];
    if (kind != 3 && !(p > 0.0)) atomicOr(flags, 1);
    for (int c = 0; c < 3; ++c) {
      if (dev_pass) {
        acc[c] = ddiv(dsub(T[r * 3 + c], (double)Y[i * 3 + c]), p);
      } else {
        float g;
        acc[c] = loss_elem(kind, Y[i * 3 + c], T[r * 3 + c], p, rmean ? rmean[c] : 0.0, eps,
                           (double)(n * 3), &g);
        dY[i * 3 + c] = g;
      }
    }
  }
  for (int c = 0; c < 3; ++c) red[threadIdx.x][c] = acc[c];
  __syncthreads();
  for (int s = kLossThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int c = 0; c < 3; ++c) red[threadIdx.x][c] += red[threadIdx.x + s][c];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int c = 0; c < 3; ++c) partial[blockIdx.x * 3 + c] = red[0][c];
}

// Pass 2 (one block): fold the partials in block order (deterministic).
// mode 0: loss mean -> out[0], non-finite -> flags |= 2.
// mode 1: variance EMA  rm = 0.95 rm + 0.05 mean((t-y)/pdf) (caches.py:340-343).
__global__ void k_loss_final(const double* __restrict__ partial, int nblk, int64_t n,
                             double* __restrict__ out, int32_t* __restrict__ flags,
                             double* __restrict__ rmean, int mode) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (flags && (flags[0] & 2)) return;
  double s[3] = {0.0, 0.0, 0.0};
  for (int b = 0; b < nblk; ++b)
    for (int c = 0; c < 3; ++c) s[c] += partial[b * 3 + c];
  if (mode == 0) {
    const double v = (s[0] + s[1] + s[2]) / (double)(n * 3);
    out[0] = v;
    if (!isfinite(v)) atomicOr(flags, 2);
  } else {
    for (int c = 0; c < 3; ++c)
      rmean[c] = dadd(dmul(0.95, rmean[c]), dmul(dsub(1.0, 0.95), s[c] / (double)n));
  }
}

// ----------------------------------------------------------------------
// Backward (mlp.py:125-154).  ReLU' uses (z >= 0) for hidden AND output
// layers (:134-138, :149).  Row pass: dz per layer (stored for the weight
// gradient), dX = dz0 W0.  Weight pass: dW = dz^T a_prev, db = sum dz.
// ----------------------------------------------------------------------
__device__ inline float act_of(const nirc_spec_t& sp, int layer, float z) {
  // activation applied to the pre-activation of `layer`
  if (layer < sp.n_layers - 1 || sp.out_act == 0) return z > 0.0f ? z : 0.0f;
  return 1.0f / (1.0f + expf(-z));
}

__global__ void k_backward_rows(nirc_spec_t sp, const float* __restrict__ theta,
                                const float* __restrict__ zs, const float* __restrict__ dY,
                                int64_t n, float* __restrict__ dzs, float* __restrict__ dX,
                                const int32_t* __restrict__ flags) {
  extern __shared__ float smem[];
  if (flags && (flags[0] & 3)) return;
  float* W = smem;
  stage_params(sp, theta, W);
  const int dmax = net_dmax(sp);
  float* cur = W + net_param_count(sp) + threadIdx.x;
  float* nxt = cur + (dmax + 1) * kRowsPerBlock;
  __syncthreads();
  const int64_t row = (int64_t)blockIdx.x * kRowsPerBlock + threadIdx.x;
  if (row >= n) return;
  const int zw = zs_width(sp);
  int zoff[NIRC_MAX_LAYERS + 1];
  zoff[0] = 0;
  for (int l = 0; l < sp.n_layers; ++l) zoff[l + 1] = zoff[l] + sp.dims[l + 1];
  const float* zr = zs + row * zw;
  float* dzr = dzs + row * zw;
  const int L = sp.n_layers - 1;
  const int dout = sp.dims[sp.n_layers];
  for (int j = 0; j < dout; ++j) {
    const float z = zr[zoff[L] + j];
    float g;
    if (sp.out_act == 0) {
      g = z >= 0.0f ? dY[row * dout + j] : 0.0f;
    } else {
      const float s = 1.0f / (1.0f + expf(-z));
      g = dY[row * dout + j] * s * (1.0f - s);
    }
    cur[j * kRowsPerBlock] = g;
    dzr[zoff[L] + j] = g;
  }
  for (int l = L; l >= 0; --l) {
    const int din = sp.dims[l], do_ = sp.dims[l + 1];
    const float* w = W + (sp.w_off[l] - sp.grid_len);
    for (int i = 0; i < din; ++i) {
      float acc = 0.0f;
      for (int j = 0; j < do_; ++j) acc = fmaf(cur[j * kRowsPerBlock], w[j * din + i], acc);
      if (l > 0) {
        const float z = zr[zoff[l - 1] + i];
        const float g = z >= 0.0f ? acc : 0.0f;
        nxt[i * kRowsPerBlock] = g;
        dzr[zoff[l - 1] + i] = g;
      } else {
        dX[row * sp.in_dim + i] = acc;
      }
    }
    float* t = cur; cur = nxt; nxt = t;
  }
}

// dW_l[j][i] = sum_b dz_l[b][j] * a_{l-1}[b][i]; db_l[j] = sum_b dz_l[b][j].
// grid = (chunks, layers); each block reduces kDwRows rows of one layer in
// registers then adds its partial into grad with one atomic per weight.
constexpr int kDwRows = 256;
constexpr int kDwThreads = 256;

__global__ void k_weight_grad(nirc_spec_t sp, const float* __restrict__ X,
                              const float* __restrict__ zs, const float* __restrict__ dzs,
                              int64_t n, float* __restrict__ grad,
                              const int32_t* __restrict__ flags) {
  if (flags && (flags[0] & 3)) return;
  const int l = blockIdx.y;
  const int din = sp.dims[l], dout = sp.dims[l + 1];
  const int zw = zs_width(sp);
  int zoff_l = 0, zoff_prev = 0;
  for (int k = 0; k < l; ++k) zoff_l += sp.dims[k + 1];
  zoff_prev = zoff_l - (l > 0 ? sp.dims[l] : 0);
  __shared__ float s_a[32][129];
  __shared__ float s_dz[32][129];
  const int64_t r0 = (int64_t)blockIdx.x * kDwRows;
  const int64_t r1 = (n < r0 + kDwRows) ? n : r0 + kDwRows;
  const int nw = dout * (din + 1);  // +1 column: bias
  if (blockIdx.z * 32 * kDwThreads >= nw) return;
  // each thread owns up to 32 (j,i) pairs
  float acc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = 0.0f;
  for (int64_t rb = r0; rb < r1; rb += 32) {
    const int nr = (int)((r1 - rb) < 32 ? (r1 - rb) : 32);
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 128; e += blockDim.x) {
      const int rr = e / 128, c = e % 128;
      if (rr < nr) {
        const int64_t row = rb + rr;
        if (c < din) {
          float a;
          if (l == 0) a = X[row * sp.in_dim + c];
          else a = act_of(sp, l - 1, zs[row * zw + zoff_prev + c]);
          s_a[rr][c] = a;
        }
        if (c < dout) s_dz[rr][c] = dzs[row * zw + zoff_l + c];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int e = blockIdx.z * 32 * kDwThreads + threadIdx.x + k * kDwThreads;
      if (e < nw) {
        const int j = e / (din + 1), i = e % (din + 1);
        float s = acc[k];
        for (int rr = 0; rr < nr; ++rr) s = fmaf(s_dz[rr][j], i < din ? s_a[rr][i] : 1.0f, s);
        acc[k] = s;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int e = blockIdx.z * 32 * kDwThreads + threadIdx.x + k * kDwThreads;
    if (e < nw) {
      const int j = e / (din + 1), i = e % (din + 1);
      float* dst = (i < din) ? grad + sp.w_off[l] + j * din + i : grad + sp.b_off[l] + j;
      atomicAdd(dst, acc[k]);
    }
  }
}

// ----------------------------------------------------------------------
// Dense Adam (adam.py:20-33).  All arithmetic is the reference's f32
// sequence: m += f32(1-b1)*(g-m); v += f32(1-b2)*(g*g-v);
// theta -= (f32(lr)*(m/f32(1-b1^t))) / (sqrt(v/f32(1-b2^t)) + f32(eps)).
// Pass 1 flags any non-finite gradient; pass 2 applies or counts a skip.
// ----------------------------------------------------------------------
__global__ void k_adam_check(const float* __restrict__ g, int64_t n, int32_t* __restrict__ bad,
                             const int32_t* __restrict__ gate) {
  if (gate && gate[0]) return;
  int found = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    found |= !isfinite(g[i]);
  found = __syncthreads_or(found);
  if (found && threadIdx.x == 0) atomicExch(bad, 1);
}

__global__ void k_adam_apply(float* __restrict__ theta, float* __restrict__ m,
                             float* __restrict__ v, const float* __restrict__ g, int64_t n,
                             int64_t* __restrict__ t, int64_t* __restrict__ skipped, float lr,
                             double b1, double b2, float eps, const int32_t* __restrict__ bad,
                             const int32_t* __restrict__ gate) {
  if (gate && gate[0]) return;
  if (bad[0]) {
    if (blockIdx.x == 0 && threadIdx.x == 0) skipped[0] += 1;
    return;
  }
  const int64_t tn = t[0] + 1;  // read before block 0 publishes (see k_adam_tick)
  const float c1 = (float)(1.0 - b1);
  const float c2 = (float)(1.0 - b2);
  const float bc1 = (float)(1.0 - pow(b1, (double)tn));
  const float bc2 = (float)(1.0 - pow(b2, (double)tn));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    float mi = m[i], vi = v[i];
    mi = __fadd_rn(mi, __fmul_rn(c1, __fsub_rn(gi, mi)));
    vi = __fadd_rn(vi, __fmul_rn(c2, __fsub_rn(__fmul_rn(gi, gi), vi)));
    m[i] = mi;
    v[i] = vi;
    const float mh = __fdiv_rn(mi, bc1);
    const float vh = __fdiv_rn(vi, bc2);
    const float upd = __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), eps));
    theta[i] = __fsub_rn(theta[i], upd);
  }
}

// Same update, 4 parameters per thread through 16-byte loads (all of theta,
// m, v, g 16-byte aligned); the n % 4 tail is done by the first threads.
__device__ __forceinline__ void adam_one(float& th, float& mi, float& vi, float gi, float c1,
                                         float c2, float bc1, float bc2, float lr, float eps) {
  mi = __fadd_rn(mi, __fmul_rn(c1, __fsub_rn(gi, mi)));
  vi = __fadd_rn(vi, __fmul_rn(c2, __fsub_rn(__fmul_rn(gi, gi), vi)));
  const float mh = __fdiv_rn(mi, bc1);
  const float vh = __fdiv_rn(vi, bc2);
  th = __fsub_rn(th, __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), eps)));
}

__global__ void k_adam_apply4(float* __restrict__ theta, float* __restrict__ m,
                              float* __restrict__ v, const float* __restrict__ g, int64_t n,
                              int64_t* __restrict__ t, int64_t* __restrict__ skipped, float lr,
                              double b1, double b2, float eps, const int32_t* __restrict__ bad,
                              const int32_t* __restrict__ gate, const float* __restrict__ bc_in) {
  if (gate && gate[0]) return;
  if (bad[0]) {
    if (blockIdx.x == 0 && threadIdx.x == 0) skipped[0] += 1;
    return;
  }
  // bias corrections precomputed (k_reduce_grad): no block reads t, so
  // block 0 advances it here (no k_adam_tick launch)
  if (bc_in != nullptr && blockIdx.x == 0 && threadIdx.x == 0) t[0] += 1;
  const float c1 = (float)(1.0 - b1);
  const float c2 = (float)(1.0 - b2);
  const int64_t n4 = n >> 2;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // this thread's first float4s are requested before the bias corrections
  // (f64 pow, the reference's python float arithmetic; one lane per warp,
  // broadcast by shuffle) are computed, so their latencies overlap; t is
  // read before block 0 publishes (see k_adam_tick)
  const bool first = tid < n4;
  float4 th = make_float4(0.f, 0.f, 0.f, 0.f), mi = th, vi = th, gi = th;
  if (first) {
    th = reinterpret_cast<float4*>(theta)[tid];
    mi = reinterpret_cast<float4*>(m)[tid];
    vi = reinterpret_cast<float4*>(v)[tid];
    gi = reinterpret_cast<const float4*>(g)[tid];
  }
  float bc1 = 0.0f, bc2 = 0.0f;
  if (bc_in != nullptr) {
    bc1 = bc_in[0];
    bc2 = bc_in[1];
  } else {
    if ((threadIdx.x & 31) == 0) {
      const int64_t tn = t[0] + 1;
      bc1 = (float)(1.0 - pow(b1, (double)tn));
      bc2 = (float)(1.0 - pow(b2, (double)tn));
    }
    bc1 = __shfl_sync(0xffffffffu, bc1, 0);
    bc2 = __shfl_sync(0xffffffffu, bc2, 0);
  }
  for (int64_t i = tid; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    if (i != tid) {
      th = reinterpret_cast<float4*>(theta)[i];
      mi = reinterpret_cast<float4*>(m)[i];
      vi = reinterpret_cast<float4*>(v)[i];
      gi = reinterpret_cast<const float4*>(g)[i];
    }
    adam_one(th.x, mi.x, vi.x, gi.x, c1, c2, bc1, bc2, lr, eps);
    adam_one(th.y, mi.y, vi.y, gi.y, c1, c2, bc1, bc2, lr, eps);
    adam_one(th.z, mi.z, vi.z, gi.z, c1, c2, bc1, bc2, lr, eps);
    adam_one(th.w, mi.w, vi.w, gi.w, c1, c2, bc1, bc2, lr, eps);
    reinterpret_cast<float4*>(theta)[i] = th;
    reinterpret_cast<float4*>(m)[i] = mi;
    reinterpret_cast<float4*>(v)[i] = vi;
  }
  if (tid < (n & 3)) {
    const int64_t i = 4 * n4 + tid;
    float th = theta[i], mi = m[i], vi = v[i];
    adam_one(th, mi, vi, g[i], c1, c2, bc1, bc2, lr, eps);
    theta[i] = th;
    m[i] = mi;
    v[i] = vi;
  }
}

__global__ void k_adam_tick(int64_t* __restrict__ t, const int32_t* __restrict__ bad,
                            const int32_t* __restrict__ gate) {
  if (gate && gate[0]) return;
  if (!bad[0]) t[0] += 1;
}

// ----------------------------------------------------------------------
// Batch selection (caches.py:327-329): keys x_i = mix64(K + G*(step*n+i))>>11
// with K = stream_key(seed, P_SHUFFLE, 0, frame, 0) (rng.py:100-106 puts
// the stream in the pixel slot); idx = stable argsort(x)[:min(cap, n)].
__device__ inline uint64_t shuffle_key(uint64_t K, uint64_t dim) {
  return rand_u64(K, dim) >> 11;
}

// Multi-CTA exact selection (the production path): bucket the 53-bit keys
// by their top 14 bits, find the bucket holding rank B-1, scatter every key
// of the buckets up to it into bucket order, then sort each bucket by
// (key, index) with one thread per bucket (~n/4096 keys each).  The result
// is exactly argsort(key, stable)[:B] in O(n) work with no single-CTA pass.
constexpr int kSelBins = 16384;
constexpr int kSelShift = 53 - 14;

struct SelWs {
  // one slice per optimizer step (blockIdx.y), strides n / kSelBins
  uint64_t* keys;      // (steps, n)
  uint32_t* hist;      // (steps, kSelBins)
  uint32_t* fill;      // (steps, kSelBins)
  uint32_t* boff;      // (steps, kSelBins + 1) exclusive offsets
  int32_t* bstar;      // (steps, 2): [0] last bucket taken, [1] staged count
  uint64_t* skey;      // (steps, n) staged keys
  int64_t* sidx;       // (steps, n) staged indices -- step s's batch is sidx[s*n : s*n+B]
};

// keys of step s = blockIdx.y: dims offset + s*n + i (caches.py:327-328)
__global__ void k_sel_hist(uint64_t K, uint64_t offset, int64_t n, SelWs w,
                           const int32_t* __restrict__ flags) {
  extern __shared__ uint32_t h[];  // kSelBins
  if (flags && (flags[0] & 3)) return;
  const int s = blockIdx.y;
  uint64_t* keys = w.keys + (int64_t)s * n;
  uint32_t* hist = w.hist + (int64_t)s * kSelBins;
  const uint64_t off = offset + (uint64_t)s * (uint64_t)n;
  for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = shuffle_key(K, off + i);
    keys[i] = k;
    atomicAdd(&h[k >> kSelShift], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSelBins; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

__global__ void k_sel_scan(int64_t n, int B, SelWs w, const int32_t* __restrict__ flags) {
  __shared__ uint32_t part[1024];
  if (flags && (flags[0] & 3)) return;
  const int sy = blockIdx.y;
  const uint32_t* hist = w.hist + (int64_t)sy * kSelBins;
  uint32_t* boff = w.boff + (int64_t)sy * (kSelBins + 1);
  uint32_t* fill = w.fill + (int64_t)sy * kSelBins;
  int32_t* bstar = w.bstar + 2 * sy;
  const int t = threadIdx.x;  // 1024 threads x 16 consecutive bins (4 x 16-byte loads)
  constexpr int kPer = kSelBins / 1024;
  uint32_t v[kPer], s = 0;
#pragma unroll
  for (int q = 0; q < kPer; q += 4) {
    const uint4 x = reinterpret_cast<const uint4*>(hist + t * kPer)[q / 4];
    v[q] = x.x;
    v[q + 1] = x.y;
    v[q + 2] = x.z;
    v[q + 3] = x.w;
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q) s += v[q];
  // block-wide inclusive scan of the per-thread sums (warp shuffles)
  const int lane = t & 31, wid = t >> 5;
  uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) part[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t z = part[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    part[lane] = z;
  }
  __syncthreads();
  uint32_t run = x - s + (wid > 0 ? part[wid - 1] : 0u);
  uint32_t o[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    o[q] = run;
    // the bucket containing rank B-1 (or the last bucket when n <= B)
    if (run < (uint32_t)B && run + v[q] >= (uint32_t)B) {
      bstar[0] = t * kPer + q;
      bstar[1] = (int32_t)(run + v[q]);
    }
    run += v[q];
  }
  // boff is kSelBins + 1 long: 4-byte stores; fill via 16-byte stores
#pragma unroll
  for (int q = 0; q < kPer; ++q) boff[t * kPer + q] = o[q];
#pragma unroll
  for (int q = 0; q < kPer; q += 4)
    reinterpret_cast<uint4*>(fill + t * kPer)[q / 4] = make_uint4(0u, 0u, 0u, 0u);
  if (t == 1023) boff[kSelBins] = run;
  if (n <= B && t == 0) {
    bstar[0] = kSelBins - 1;
    bstar[1] = (int32_t)n;
  }
}

__global__ void k_sel_scatter(int64_t n, SelWs w, const int32_t* __restrict__ flags) {
  if (flags && (flags[0] & 3)) return;
  const int s = blockIdx.y;
  const uint64_t* keys = w.keys + (int64_t)s * n;
  const uint32_t* boff = w.boff + (int64_t)s * (kSelBins + 1);
  uint32_t* fill = w.fill + (int64_t)s * kSelBins;
  uint64_t* skey = w.skey + (int64_t)s * n;
  int64_t* sidx = w.sidx + (int64_t)s * n;
  const int bs = w.bstar[2 * s];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const int b = (int)(k >> kSelShift);
    if (b <= bs) {
      const uint32_t pos = boff[b] + atomicAdd(&fill[b], 1u);
      skey[pos] = k;
      sidx[pos] = i;
    }
  }
}

__global__ void k_sel_sort(int64_t n, SelWs w, const int32_t* __restrict__ flags) {
  if (flags && (flags[0] & 3)) return;
  const int s = blockIdx.y;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > w.bstar[2 * s]) return;
  const uint32_t* boff = w.boff + (int64_t)s * (kSelBins + 1);
  uint64_t* skey = w.skey + (int64_t)s * n;
  int64_t* sidx = w.sidx + (int64_t)s * n;
  const uint32_t lo = boff[b], hi = boff[b + 1];
  constexpr uint32_t kLocal = 32;
  if (hi - lo <= kLocal) {  // small bucket (the common case): sort in registers / L1
    uint64_t k[kLocal];
    int64_t x[kLocal];
    const uint32_t nb = hi - lo;
    for (uint32_t i = 0; i < nb; ++i) {
      k[i] = skey[lo + i];
      x[i] = sidx[lo + i];
    }
    for (uint32_t i = 1; i < nb; ++i) {  // insertion sort by (key, index)
      const uint64_t kk = k[i];
      const int64_t xx = x[i];
      uint32_t j = i;
      while (j > 0 && (k[j - 1] > kk || (k[j - 1] == kk && x[j - 1] > xx))) {
        k[j] = k[j - 1];
        x[j] = x[j - 1];
        --j;
      }
      k[j] = kk;
      x[j] = xx;
    }
    for (uint32_t i = 0; i < nb; ++i) {
      skey[lo + i] = k[i];
      sidx[lo + i] = x[i];
    }
    return;
  }
  for (uint32_t i = lo + 1; i < hi; ++i) {  // insertion sort by (key, index)
    const uint64_t k = skey[i];
    const int64_t x = sidx[i];
    uint32_t j = i;
    while (j > lo && (skey[j - 1] > k || (skey[j - 1] == k && sidx[j - 1] > x))) {
      skey[j] = skey[j - 1];
      sidx[j] = sidx[j - 1];
      --j;
    }
    skey[j] = k;
    sidx[j] = x;
  }
}

// Gather + encode + forward for the training batch: row i of the batch is
// record idx[i] (caches.py:330-333).
__global__ void k_train_forward(nirc_spec_t sp, const float* __restrict__ theta,
                                nirc_records_t rec, const int64_t* __restrict__ idx, int64_t B,
                                float* __restrict__ X, float* __restrict__ zs,
                                float* __restrict__ Y, const int32_t* __restrict__ flags) {
  extern __shared__ float smem[];
  if (flags && (flags[0] & 3)) return;
  float* W = smem;
  stage_params(sp, theta, W);
  const int dmax = net_dmax(sp);
  float* a = W + net_param_count(sp) + threadIdx.x;
  float* b = a + (dmax + 1) * kRowsPerBlock;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kRowsPerBlock + threadIdx.x;
  if (i >= B) return;
  const int64_t r = idx[i];
  float* xr = X + i * sp.in_dim;
  encode_row(sp, theta, rec.pos + 3 * r, rec.ns + 3 * r, rec.alb + 3 * r, rec.rough[r],
             rec.dirs + 3 * r,
             [&](int k, float v) {
               xr[k] = v;
               a[k * kRowsPerBlock] = v;
             },
             nullptr, nullptr);
  simt_forward_row(sp, W, a, b, kRowsPerBlock, zs + i * zs_width(sp));
  const float* out = (sp.n_layers % 2 == 1) ? b : a;
  const int dout = sp.dims[sp.n_layers];
  for (int j = 0; j < dout; ++j) Y[i * dout + j] = out[j * kRowsPerBlock];
}

// Hash-grid scatter for the training batch: slots and weights are recomputed
// from the record position (bit-identical to encode_batch's entries/weights)
// instead of being stored.  One thread per (row, level).
__global__ void k_train_scatter(nirc_spec_t sp, nirc_records_t rec,
                                const int64_t* __restrict__ idx, int64_t B,
                                const float* __restrict__ dX, float* __restrict__ grad,
                                const int32_t* __restrict__ flags) {
  if (flags && (flags[0] & 3)) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B * sp.levels) return;
  const int64_t i = t / sp.levels;
  const int lvl = (int)(t % sp.levels);
  const int64_t r = idx[i];
  const double* p = rec.pos + 3 * r;
  const float ux = norm_coord(p[0], sp.bb_min[0], sp.bb_inv[0]);
  const float uy = norm_coord(p[1], sp.bb_min[1], sp.bb_inv[1]);
  const float uz = norm_coord(p[2], sp.bb_min[2], sp.bb_inv[2]);
  const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
  const uint32_t T = 1u << sp.table_log2;
  const int F = sp.feats;
  float* gl = grad + (int64_t)lvl * T * F;
  for (int f = 0; f < F; ++f) {
    const float d = dX[i * sp.in_dim + lvl * F + f];
    if (d == 0.0f) continue;
    for (int k = 0; k < 8; ++k)
      atomicAdd(gl + (int64_t)corner_hash(c, k, T - 1u) * F + f, __fmul_rn(corner_weight(c, k), d));
  }
}

}  // namespace nirc

namespace nirc {
bool fused_supported(const nirc_spec_t& sp);
size_t fused_smem_bytes(const nirc_spec_t& sp);
int launch_fused_train(const nirc_spec_t& sp, const float* theta, const nirc_records_t& rec,
                       const int64_t* idx, int64_t B, int loss_kind, double loss_eps,
                       float* grad, float* partials, double* loss_part, double* loss_out,
                       int32_t* flags, int32_t* adam_bad, cudaStream_t s, int64_t tile0,
                       int64_t tile1, int mode, const float* rstat, bool deterministic,
                       const int64_t* t, float* bc, double b1, double b2);
template <typename T>
int ordered_scatter(const nirc_spec_t& sp, T* grad, const int64_t* entries, const float* weights,
                    const T* dX, int64_t n, int64_t stride, const double* pos, const int64_t* idx,
                    int64_t r0, cudaStream_t s);
int64_t train_static_bytes(int64_t n);
int launch_record_static(const nirc_spec_t& sp, const nirc_records_t& rec, float* out,
                         cudaStream_t s);
bool train_tc_supported(const nirc_spec_t& sp);
constexpr int kFusedTileRows = 128;  // rows per k_train_tile CTA (train_fused.cu kTR)
}  // namespace nirc

using namespace nirc;

// ======================================================================
// C ABI
// ======================================================================
static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline int blocks_for(int64_t n, int t) { return (int)((n + t - 1) / t); }

static int check_spec(const nirc_spec_t* sp) {
  if (!sp) { set_last_error("spec is NULL"); return NIRC_E_CONFIG; }
  if (sp->levels < 1 || sp->levels > NIRC_MAX_LEVELS || sp->feats < 1 || sp->feats > 4 ||
      sp->bands < 1 || sp->bands > NIRC_MAX_BANDS || sp->n_layers < 1 ||
      sp->n_layers > NIRC_MAX_LAYERS || sp->table_log2 < 1 || sp->table_log2 > 30) {
    set_last_error("unsupported spec (levels=%d feats=%d bands=%d layers=%d)", sp->levels,
                   sp->feats, sp->bands, sp->n_layers);
    return NIRC_E_CONFIG;
  }
  if (net_dmax(*sp) > 128) {
    set_last_error("layer width %d > 128 unsupported", net_dmax(*sp));
    return NIRC_E_UNSUPPORTED;
  }
  if (simt_smem_bytes(*sp) > 200 * 1024) {
    set_last_error("network too large for the shared-memory SIMT path");
    return NIRC_E_UNSUPPORTED;
  }
  return NIRC_OK;
}

static unsigned dw_zsplit(const nirc_spec_t& sp) {
  int mx = 0;
  for (int l = 0; l < sp.n_layers; ++l) {
    const int nw = sp.dims[l + 1] * (sp.dims[l] + 1);
    mx = nw > mx ? nw : mx;
  }
  return (unsigned)((mx + 32 * kDwThreads - 1) / (32 * kDwThreads));
}

static int set_smem(const void* fn, size_t bytes) {
  NIRC_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return NIRC_OK;
}

extern "C" int nirc_encode(const nirc_spec_t* spec, const float* theta, const double* pos,
                           const double* normal, const double* albedo, const double* rough,
                           const double* dirs, int64_t n, float* X, int64_t* entries,
                           float* weights, void* stream) {
  int st = check_spec(spec);
  if (st) return st;
  if (n <= 0) return NIRC_OK;
  k_encode<<<blocks_for(n, 128), 128, 0, S(stream)>>>(*spec, theta, pos, normal, albedo, rough,
                                                     dirs, n, X, entries, weights);
  NIRC_LAUNCH_CHECK("k_encode");
  return NIRC_OK;
}

extern "C" int nirc_scatter_grid_grad(const nirc_spec_t* spec, float* grad,
                                      const int64_t* entries, const float* weights,
                                      const float* dX, int64_t n, int64_t dx_stride,
                                      void* stream) {
  int st = check_spec(spec);
  if (st) return st;
  if (n <= 0) return NIRC_OK;
  return ordered_scatter<float>(*spec, grad, entries, weights, dX, n, dx_stride, nullptr, nullptr,
                                0, S(stream));
}

extern "C" int nirc_mlp_forward(const nirc_spec_t* spec, const float* theta, const float* X,
                                int64_t n, float* Y, float* zs, int32_t* nonfinite_flag,
                                void* stream) {
  int st = check_spec(spec);
  if (st) return st;
  if (n <= 0) return NIRC_OK;
  const size_t sm = simt_smem_bytes(*spec);
  if ((st = set_smem((const void*)k_mlp_forward, sm))) return st;
  k_mlp_forward<<<blocks_for(n, kRowsPerBlock), kRowsPerBlock, sm, S(stream)>>>(
      *spec, theta, X, n, Y, zs, nonfinite_flag);
  NIRC_LAUNCH_CHECK("k_mlp_forward");
  return NIRC_OK;
}

extern "C" int nirc_mlp_backward(const nirc_spec_t* spec, const float* theta, const float* X,
                                 const float* zs, const float* dY, int64_t n, float* grad,
                                 float* dX, float* scratch, void* stream) {
  int st = check_spec(spec);
  if (st) return st;
  if (n <= 0) return NIRC_OK;
  const size_t sm = simt_smem_bytes(*spec);
  if ((st = set_smem((const void*)k_backward_rows, sm))) return st;
  k_backward_rows<<<blocks_for(n, kRowsPerBlock), kRowsPerBlock, sm, S(stream)>>>(
      *spec, theta, zs, dY, n, scratch, dX, nullptr);
  NIRC_LAUNCH_CHECK("k_backward_rows");
  dim3 g(blocks_for(n, kDwRows), spec->n_layers, dw_zsplit(*spec));
  k_weight_grad<<<g, kDwThreads, 0, S(stream)>>>(*spec, X, zs, scratch, n, grad, nullptr);
  NIRC_LAUNCH_CHECK("k_weight_grad");
  return NIRC_OK;
}

extern "C" int nirc_loss(int32_t kind, const float* Y, const double* target, const double* pdf,
                         const double* running_mean, double eps, int64_t n, float* dY,
                         double* loss_out, int32_t* status_flags, double* scratch,
                         void* stream) {
  if (kind < 0 || kind > 3) { set_last_error("unknown loss kind %d", kind); return NIRC_E_CONFIG; }
  if (n <= 0) return NIRC_OK;
  const int nb = blocks_for(n, kLossThreads);
  k_loss<<<nb, kLossThreads, 0, S(stream)>>>(kind, Y, target, pdf, running_mean, eps, n, dY,
                                             scratch, status_flags, nullptr, 0);
  NIRC_LAUNCH_CHECK("k_loss");
  k_loss_final<<<1, 32, 0, S(stream)>>>(scratch, nb, n, loss_out, status_flags, nullptr, 0);
  NIRC_LAUNCH_CHECK("k_loss_final");
  return NIRC_OK;
}

static nirc_train_opts_t opts_or_default(const nirc_train_opts_t* o) {
  nirc_train_opts_t d{0.9, 0.99, 1e-8, 0, 0};  // AdamState defaults (adam.py:8-17)
  return o != nullptr ? *o : d;
}

// Dense Adam apply + tick; the non-finite check already ran (adam_bad).
static int launch_adam(float* theta, float* m, float* v, const float* grad, int64_t n,
                       int64_t* t, int64_t* skipped, float lr, const int32_t* bad,
                       const int32_t* gate, cudaStream_t s, double b1 = 0.9, double b2 = 0.99,
                       double eps = 1e-8, const float* bc = nullptr) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(m) |
                         reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(grad)) &
                        15u) == 0;
  if (aligned) {
    const int64_t n4 = (n >> 2) > 0 ? (n >> 2) : 1;
    const int nb = (int)((n4 + 255) / 256 < 148 * 8 ? (n4 + 255) / 256 : 148 * 8);
    k_adam_apply4<<<nb, 256, 0, s>>>(theta, m, v, grad, n, t, skipped, lr, b1, b2, (float)eps,
                                     bad, gate, bc);
    if (bc != nullptr) {  // t advanced by k_adam_apply4
      NIRC_LAUNCH_CHECK("k_adam_apply4");
      return NIRC_OK;
    }
  } else {
    k_adam_apply<<<148 * 4, 256, 0, s>>>(theta, m, v, grad, n, t, skipped, lr, b1, b2,
                                         (float)eps, bad, gate);
  }
  NIRC_LAUNCH_CHECK("k_adam_apply");
  k_adam_tick<<<1, 1, 0, s>>>(t, bad, gate);
  NIRC_LAUNCH_CHECK("k_adam_tick");
  return NIRC_OK;
}

extern "C" int nirc_adam_step(float* theta, float* m, float* v, const float* grad, int64_t n,
                              int64_t* t, int64_t* skipped, double lr, double beta1,
                              double beta2, double eps, const int32_t* gate_flags,
                              int32_t* scratch, void* stream) {
  if (n <= 0) return NIRC_OK;
  NIRC_CUDA_TRY(cudaMemsetAsync(scratch, 0, sizeof(int32_t), S(stream)));
  const int nb = 148 * 4;
  k_adam_check<<<nb, 256, 0, S(stream)>>>(grad, n, scratch, gate_flags);
  NIRC_LAUNCH_CHECK("k_adam_check");
  return launch_adam(theta, m, v, grad, n, t, skipped, (float)lr, scratch, gate_flags,
                     S(stream), beta1, beta2, eps);
}

// ---------------------------------------------------------------- train --
namespace {
struct TrainWs {
  SelWs sel;
  float *X, *zs, *Y, *dY, *dzs, *dX, *grad;
  double* partial;
  int32_t* adam_bad;
  float* fpart;      // fused path: per-tile MLP gradient partials
  double* floss;     // fused path: per-tile loss partials
  float* rstat;      // tcgen05 path: per-record static encoding (u, SH, aux)
  size_t bytes;
};
size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }
// `steps` selection slices (all optimizer steps of a frame are selected at
// once: the batch never depends on theta).
TrainWs carve_train(const nirc_spec_t& sp, int64_t n, int64_t B, int steps, void* base) {
  TrainWs w{};
  char* p = reinterpret_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = p ? p + off : nullptr;
    off += align_up(bytes);
    return r;
  };
  const int zw = zs_width(sp);
  w.sel.keys = (uint64_t*)take(steps * n * 8);
  w.sel.hist = (uint32_t*)take(steps * kSelBins * 4);
  w.sel.fill = (uint32_t*)take(steps * kSelBins * 4);
  w.sel.boff = (uint32_t*)take(steps * (kSelBins + 1) * 4);
  w.sel.bstar = (int32_t*)take(steps * 8 + 8);
  w.sel.skey = (uint64_t*)take(steps * n * 8);
  w.sel.sidx = (int64_t*)take(steps * n * 8);
  w.X = (float*)take(B * sp.in_dim * 4);
  w.zs = (float*)take(B * zw * 4);
  w.Y = (float*)take(B * 3 * 4 + 16);
  w.dY = (float*)take(B * 3 * 4 + 16);
  w.dzs = (float*)take(B * zw * 4);
  w.dX = (float*)take(B * sp.in_dim * 4);
  w.grad = (float*)take(sp.theta_len * 4);
  w.partial = (double*)take((B / kLossThreads + 2) * 3 * 8);
  w.adam_bad = (int32_t*)take(16);
  // partial slots: one per CTA; a launch of k tiles runs k, 2k or 4k CTAs
  // with 4k, 2k <= the SM count (train_fused.cu tile_rows_for)
  const int64_t ntiles = (B + kFusedTileRows - 1) / kFusedTileRows;
  const int64_t slots = ntiles > 256 ? ntiles : 256;
  w.fpart = (float*)take(slots * part_stride(sp) * 4);
  w.floss = (double*)take(slots * 8);
  w.rstat = (float*)take(train_static_bytes(n));
  w.bytes = off;
  return w;
}
}  // namespace

extern "C" int64_t nirc_train_workspace_bytes(const nirc_spec_t* spec, int64_t n_records,
                                              int32_t batch_cap) {
  const int64_t B = n_records < batch_cap ? n_records : batch_cap;
  return (int64_t)carve_train(*spec, n_records, B, 1, nullptr).bytes;
}

extern "C" int64_t nirc_train_frame_workspace_bytes(const nirc_spec_t* spec, int64_t n_records,
                                                    int32_t batch_cap, int32_t steps) {
  const int64_t B = n_records < batch_cap ? n_records : batch_cap;
  return (int64_t)carve_train(*spec, n_records, B, steps < 1 ? 1 : steps, nullptr).bytes;
}

// Batch selection of optimizer steps step0 .. step0+steps-1 (caches.py:
// 327-329): slice s of w.sel.sidx holds argsort(keys of step step0+s)[:B].
static int select_batches(const TrainWs& w, uint64_t seed, int64_t frame, int32_t step0,
                          int32_t steps, int64_t n, int64_t B, int32_t* status_flags,
                          cudaStream_t s) {
  const uint64_t K = stream_key(seed, P_SHUFFLE, 0, (uint64_t)frame, 0);
  const uint64_t off = (uint64_t)step0 * (uint64_t)n;
  NIRC_CUDA_TRY(cudaMemsetAsync(w.sel.hist, 0, (size_t)steps * kSelBins * 4, s));
  int sel_grid = (int)((n + 255) / 256 < 4 * 148 ? (n + 255) / 256 : 4 * 148);
  sel_grid = (sel_grid + steps - 1) / steps;
  NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)k_sel_hist,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSelBins * 4));
  k_sel_hist<<<dim3(sel_grid, steps), 256, kSelBins * 4, s>>>(K, off, n, w.sel, status_flags);
  k_sel_scan<<<dim3(1, steps), 1024, 0, s>>>(n, (int)B, w.sel, status_flags);
  k_sel_scatter<<<dim3(sel_grid, steps), 256, 0, s>>>(n, w.sel, status_flags);
  k_sel_sort<<<dim3(kSelBins / 128, steps), 128, 0, s>>>(n, w.sel, status_flags);
  NIRC_LAUNCH_CHECK("k_sel_*");
  return NIRC_OK;
}

static int train_args_ok(const nirc_spec_t* spec, const nirc_records_t* rec, int32_t batch_cap) {
  int st = check_spec(spec);
  if (st) return st;
  if (!rec || rec->n <= 0) {
    set_last_error("cannot train on an empty record set");
    return NIRC_E_CONFIG;
  }
  if (batch_cap < 1) { set_last_error("batch must be positive"); return NIRC_E_CONFIG; }
  if (rec->n > INT_MAX) { set_last_error("too many records"); return NIRC_E_UNSUPPORTED; }
  return NIRC_OK;
}

static bool use_fused(const nirc_spec_t& sp, int loss_kind) {
  return (loss_kind == 0 || loss_kind == 1) && fused_supported(sp) &&
         fused_smem_bytes(sp) <= 227 * 1024;
}

// One optimizer step on the batch rows idx[0:B] (caches.py:330-350).
static int step_body(const nirc_spec_t* spec, float* theta, float* m, float* v, int64_t* t,
                     int64_t* skipped, const nirc_records_t* rec, const int64_t* idx,
                     int64_t B, int32_t loss_kind, double loss_eps, double lr,
                     const nirc_train_opts_t& o, double* running_mean, double* loss_out,
                     int32_t* status_flags, const TrainWs& w, void* stream, const float* rstat) {
  cudaStream_t s = S(stream);
  int st;
  if (use_fused(*spec, loss_kind)) {
    // one fused kernel per step: encode, forward, loss, backward, scatter
    const int64_t ntiles = (B + kFusedTileRows - 1) / kFusedTileRows;
    float* bc = reinterpret_cast<float*>(w.adam_bad + 2);  // [bad | pad | bc1 | bc2]
    if ((st = launch_fused_train(*spec, theta, *rec, idx, B, loss_kind, loss_eps, w.grad,
                                 w.fpart, w.floss, loss_out, status_flags, w.adam_bad, s, 0,
                                 ntiles, 0, rstat, o.deterministic != 0, t, bc, o.beta1,
                                 o.beta2)))
      return st;
    return launch_adam(theta, m, v, w.grad, spec->theta_len, t, skipped, (float)lr, w.adam_bad,
                       status_flags, s, o.beta1, o.beta2, o.eps, bc);
  }
  const size_t sm = simt_smem_bytes(*spec);
  if ((st = set_smem((const void*)k_train_forward, sm))) return st;
  k_train_forward<<<blocks_for(B, kRowsPerBlock), kRowsPerBlock, sm, s>>>(
      *spec, theta, *rec, idx, B, w.X, w.zs, w.Y, status_flags);
  NIRC_LAUNCH_CHECK("k_train_forward");
  const int nb = blocks_for(B, kLossThreads);
  if (loss_kind == 2) {  // variance: EMA of the residual mean first (caches.py:340-343)
    k_loss<<<nb, kLossThreads, 0, s>>>(loss_kind, w.Y, rec->target, rec->pdf, running_mean,
                                        loss_eps, B, w.dY, w.partial, status_flags, idx, 1);
    k_loss_final<<<1, 32, 0, s>>>(w.partial, nb, B, loss_out, status_flags, running_mean, 1);
  }
  k_loss<<<nb, kLossThreads, 0, s>>>(loss_kind, w.Y, rec->target, rec->pdf, running_mean,
                                      loss_eps, B, w.dY, w.partial, status_flags, idx, 0);
  NIRC_LAUNCH_CHECK("k_loss");
  k_loss_final<<<1, 32, 0, s>>>(w.partial, nb, B, loss_out, status_flags, nullptr, 0);
  NIRC_LAUNCH_CHECK("k_loss_final");
  NIRC_CUDA_TRY(cudaMemsetAsync(w.grad, 0, spec->theta_len * 4, s));
  if ((st = set_smem((const void*)k_backward_rows, sm))) return st;
  k_backward_rows<<<blocks_for(B, kRowsPerBlock), kRowsPerBlock, sm, s>>>(
      *spec, theta, w.zs, w.dY, B, w.dzs, w.dX, status_flags);
  NIRC_LAUNCH_CHECK("k_backward_rows");
  dim3 g(blocks_for(B, kDwRows), spec->n_layers, dw_zsplit(*spec));
  k_weight_grad<<<g, kDwThreads, 0, s>>>(*spec, w.X, w.zs, w.dzs, B, w.grad, status_flags);
  NIRC_LAUNCH_CHECK("k_weight_grad");
  if (o.deterministic) {
    if ((st = ordered_scatter<float>(*spec, w.grad, nullptr, nullptr, w.dX, B, spec->in_dim,
                                     rec->pos, idx, 0, s)))
      return st;
  } else {
    k_train_scatter<<<blocks_for(B * spec->levels, 256), 256, 0, s>>>(*spec, *rec, idx, B, w.dX,
                                                                     w.grad, status_flags);
    NIRC_LAUNCH_CHECK("k_train_scatter");
  }
  return nirc_adam_step(theta, m, v, w.grad, spec->theta_len, t, skipped, lr, o.beta1, o.beta2,
                        o.eps, status_flags, w.adam_bad, stream);
}

extern "C" int nirc_train_step(const nirc_spec_t* spec, float* theta, float* m, float* v,
                               int64_t* t, int64_t* skipped, const nirc_records_t* rec,
                               uint64_t seed, int64_t frame, int32_t step, int32_t batch_cap,
                               int32_t loss_kind, double loss_eps, double lr,
                               const nirc_train_opts_t* opts, double* running_mean,
                               double* loss_out, int32_t* status_flags,
                               int64_t* batch_idx_out, void* workspace,
                               int64_t workspace_bytes, void* stream) {
  int st = train_args_ok(spec, rec, batch_cap);
  if (st) return st;
  const int64_t n = rec->n;
  const int64_t B = n < batch_cap ? n : batch_cap;
  TrainWs w = carve_train(*spec, n, B, 1, workspace);
  if ((int64_t)w.bytes > workspace_bytes) {
    set_last_error("train workspace too small (%lld < %lld)", (long long)workspace_bytes,
                   (long long)w.bytes);
    return NIRC_E_CONFIG;
  }
  cudaStream_t s = S(stream);
  if ((st = select_batches(w, seed, frame, step, 1, n, B, status_flags, s))) return st;
  if (batch_idx_out)
    NIRC_CUDA_TRY(cudaMemcpyAsync(batch_idx_out, w.sel.sidx, B * 8, cudaMemcpyDeviceToDevice, s));
  return step_body(spec, theta, m, v, t, skipped, rec, w.sel.sidx, B, loss_kind, loss_eps, lr,
                   opts_or_default(opts), running_mean, loss_out, status_flags, w, stream,
                   nullptr);
}

extern "C" int nirc_train_frame(const nirc_spec_t* spec, float* theta, float* m, float* v,
                                int64_t* t, int64_t* skipped, const nirc_records_t* rec,
                                uint64_t seed, int64_t frame, int32_t steps, int32_t batch_cap,
                                int32_t loss_kind, double loss_eps, double lr,
                                const nirc_train_opts_t* opts, double* running_mean,
                                double* loss_out, int32_t* status_flags, void* workspace,
                                int64_t workspace_bytes, void* stream) {
  int st = train_args_ok(spec, rec, batch_cap);
  if (st) return st;
  if (steps < 1) { set_last_error("steps must be positive"); return NIRC_E_CONFIG; }
  const int64_t n = rec->n;
  const int64_t B = n < batch_cap ? n : batch_cap;
  TrainWs w = carve_train(*spec, n, B, steps, workspace);
  if ((int64_t)w.bytes > workspace_bytes) {
    set_last_error("train workspace too small (%lld < %lld)", (long long)workspace_bytes,
                   (long long)w.bytes);
    return NIRC_E_CONFIG;
  }
  if ((st = select_batches(w, seed, frame, 0, steps, n, B, status_flags, S(stream)))) return st;
  const float* rstat = nullptr;  // theta-independent encoding blocks: once for all steps
  if (use_fused(*spec, loss_kind) && train_tc_supported(*spec)) {
    if ((st = launch_record_static(*spec, *rec, w.rstat, S(stream)))) return st;
    rstat = w.rstat;
  }
  for (int k = 0; k < steps; ++k)
    if ((st = step_body(spec, theta, m, v, t, skipped, rec, w.sel.sidx + (int64_t)k * n, B,
                        loss_kind, loss_eps, lr, opts_or_default(opts), running_mean,
                        loss_out + k, status_flags, w, stream, rstat)))
      return st;
  return NIRC_OK;
}

// ---- multi-GPU split of nirc_train_step ------------------
extern "C" int64_t nirc_train_tiles(int64_t n_records, int32_t batch_cap) {
  if (n_records <= 0 || batch_cap < 1) return 0;
  const int64_t B = n_records < batch_cap ? n_records : batch_cap;
  return (B + kFusedTileRows - 1) / kFusedTileRows;
}

extern "C" int nirc_train_grad(const nirc_spec_t* spec, const float* theta,
                               const nirc_records_t* rec, uint64_t seed, int64_t frame,
                               int32_t step, int32_t batch_cap, int32_t loss_kind,
                               double loss_eps, const nirc_train_opts_t* opts,
                               int64_t tile_begin, int64_t tile_end,
                               float* grad, double* aux, int32_t* status_flags,
                               int64_t* batch_idx_out, void* workspace, int64_t workspace_bytes,
                               void* stream) {
  int st = train_args_ok(spec, rec, batch_cap);
  if (st) return st;
  if (!use_fused(*spec, loss_kind)) {
    set_last_error("sharded training needs the fused l2 / relative_l2 path");
    return NIRC_E_UNSUPPORTED;
  }
  const int64_t n = rec->n;
  const int64_t B = n < batch_cap ? n : batch_cap;
  const int64_t ntiles = (B + kFusedTileRows - 1) / kFusedTileRows;
  if (tile_begin < 0 || tile_end > ntiles || tile_begin > tile_end) {
    set_last_error("tile range [%lld, %lld) outside [0, %lld)", (long long)tile_begin,
                   (long long)tile_end, (long long)ntiles);
    return NIRC_E_CONFIG;
  }
  TrainWs w = carve_train(*spec, n, B, 1, workspace);
  if ((int64_t)w.bytes > workspace_bytes) {
    set_last_error("train workspace too small (%lld < %lld)", (long long)workspace_bytes,
                   (long long)w.bytes);
    return NIRC_E_CONFIG;
  }
  cudaStream_t s = S(stream);
  if ((st = select_batches(w, seed, frame, step, 1, n, B, status_flags, s))) return st;
  if (batch_idx_out)
    NIRC_CUDA_TRY(cudaMemcpyAsync(batch_idx_out, w.sel.sidx, B * 8, cudaMemcpyDeviceToDevice, s));
  return launch_fused_train(*spec, theta, *rec, w.sel.sidx, B, loss_kind, loss_eps, grad, w.fpart,
                            w.floss, aux, status_flags, nullptr, s, tile_begin, tile_end, 1,
                            nullptr, opts_or_default(opts).deterministic != 0, nullptr, nullptr,
                            0.9, 0.99);
}

namespace nirc {
// Folds the cross-GPU sums: loss = sum / (B*3) (flag 2 if non-finite), flag
// 1 if any shard saw pdf <= 0.
__global__ void k_train_fold(const double* __restrict__ aux, int64_t B,
                             double* __restrict__ loss_out, int32_t* __restrict__ flags) {
  if (flags[0] & 3) return;
  if (aux[1] > 0.0) atomicOr(flags, 1);
  const double v = aux[0] / (double)(B * 3);
  loss_out[0] = v;
  if (!isfinite(v)) atomicOr(flags, 2);
}
}  // namespace nirc

extern "C" int nirc_train_apply(const nirc_spec_t* spec, float* theta, float* m, float* v,
                                int64_t* t, int64_t* skipped, const float* grad,
                                const double* aux, int64_t batch, double lr,
                                const nirc_train_opts_t* opts, double* loss_out,
                                int32_t* status_flags, int32_t* scratch, void* stream) {
  int st = check_spec(spec);
  if (st) return st;
  if (batch < 1) { set_last_error("batch must be positive"); return NIRC_E_CONFIG; }
  k_train_fold<<<1, 1, 0, S(stream)>>>(aux, batch, loss_out, status_flags);
  NIRC_LAUNCH_CHECK("k_train_fold");
  const nirc_train_opts_t o = opts_or_default(opts);
  return nirc_adam_step(theta, m, v, grad, spec->theta_len, t, skipped, lr, o.beta1, o.beta2,
                        o.eps, status_flags, scratch, stream);
}
