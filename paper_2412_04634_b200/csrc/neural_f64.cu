// The reference's 64-bit shadow mode: init_theta(dtype=f64)
// (mlp.py:65), encode_batch(dtype=f64) (encoding.py:111-157), mlp_forward /
// mlp_backward on f64 parameters (mlp.py:102-154), scatter_grid_grad on an
// f64 gradient (encoding.py:160-167), the losses on f64 predictions
// (losses.py:23-70, including relative-L2's frozen denominator for the
// finite-difference check) and Adam on f64 state (adam.py:20-33).  Used by
// the reference's verification helpers (gradient_check's five-point
// stencil, test_training_is_bit_reproducible).  fp64 SIMT, one thread per
// row; every reduction over rows is a fixed-order per-block partial sum, so
// results are run-to-run deterministic.  Not the hot path.
#include <cmath>
#include "common.cuh"

namespace nirc {

template <typename T>
int ordered_scatter(const nirc_spec_t& sp, T* grad, const int64_t* entries, const float* weights,
                    const T* dX, int64_t n, int64_t stride, const double* pos, const int64_t* idx,
                    int64_t r0, cudaStream_t s);

namespace {

constexpr int kRows = 128;  // rows per block of the row kernels
constexpr int kMaxW = 128;  // widest layer

__host__ __device__ inline int zsw(const nirc_spec_t& sp) {
  int s = 0;
  for (int l = 1; l <= sp.n_layers; ++l) s += sp.dims[l];
  return s;
}

// encode_batch(dtype=f64): u, cells, weights and slots exactly as the f32
// path (f32 cell arithmetic); features accumulate w (f32 -> f64) * grid
// (f64) in f64 over the corners in order; SH and aux stay f64.
__global__ void k_encode_f64(nirc_spec_t sp, const double* __restrict__ theta,
                             const double* __restrict__ pos, const double* __restrict__ nrm,
                             const double* __restrict__ alb, const double* __restrict__ rough,
                             const double* __restrict__ dirs, int64_t n, double* __restrict__ X,
                             int64_t* __restrict__ ent, float* __restrict__ wts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* x = X + i * sp.in_dim;
  const double* p = pos + 3 * i;
  const float ux = norm_coord(p[0], sp.bb_min[0], sp.bb_inv[0]);
  const float uy = norm_coord(p[1], sp.bb_min[1], sp.bb_inv[1]);
  const float uz = norm_coord(p[2], sp.bb_min[2], sp.bb_inv[2]);
  const uint32_t T = 1u << sp.table_log2;
  const int F = sp.feats;
  for (int lvl = 0; lvl < sp.levels; ++lvl) {
    const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < 8; ++k) {
      const float w = corner_weight(c, k);
      const uint32_t h = corner_hash(c, k, T - 1u);
      const int64_t slot = (int64_t)lvl * T + h;
      if (ent) {
        ent[(i * sp.levels + lvl) * 8 + k] = slot;
        wts[(i * sp.levels + lvl) * 8 + k] = w;
      }
      for (int f = 0; f < F && f < 4; ++f)
        acc[f] = __dadd_rn(acc[f], __dmul_rn((double)w, theta[slot * F + f]));
    }
    for (int f = 0; f < F && f < 4; ++f) x[lvl * F + f] = acc[f];
  }
  const int g = sp.levels * F;
  const double* d = dirs + 3 * i;
  sh_eval<true>(d[0], d[1], d[2], sp.bands, sp.sh_k, [&](int k, double v) { x[g + k] = v; });
  const int a0 = g + sp.bands * sp.bands;
  for (int c = 0; c < 3; ++c) x[a0 + c] = dmul(dadd(nrm[3 * i + c], 1.0), 0.5);
  for (int c = 0; c < 3; ++c) x[a0 + 3 + c] = alb[3 * i + c];
  x[a0 + 6] = rough[i];
}

// mlp_forward: z_l = a W^T + b (f64), ReLU hidden, ReLU / sigmoid output.
__global__ void k_forward_f64(nirc_spec_t sp, const double* __restrict__ theta,
                              const double* __restrict__ X, int64_t n, double* __restrict__ Y,
                              double* __restrict__ zs) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  double a[kMaxW], b[kMaxW];
  for (int i = 0; i < sp.in_dim; ++i) a[i] = X[row * sp.in_dim + i];
  int zoff = 0;
  for (int l = 0; l < sp.n_layers; ++l) {
    const int din = sp.dims[l], dout = sp.dims[l + 1];
    const double* W = theta + sp.w_off[l];
    const double* bias = theta + sp.b_off[l];
    const bool last = l == sp.n_layers - 1;
    for (int j = 0; j < dout; ++j) {
      double acc = 0.0;
      for (int i = 0; i < din; ++i) acc = fma(a[i], W[j * din + i], acc);
      const double z = acc + bias[j];
      if (zs) zs[row * zsw(sp) + zoff + j] = z;
      b[j] = (!last || sp.out_act == 0) ? (z > 0.0 ? z : 0.0) : 1.0 / (1.0 + exp(-z));
    }
    for (int j = 0; j < dout; ++j) a[j] = b[j];
    zoff += dout;
  }
  for (int j = 0; j < sp.dims[sp.n_layers]; ++j) Y[row * sp.dims[sp.n_layers] + j] = a[j];
}

// mlp_backward rows: dz per layer (ReLU' = z >= 0 on hidden AND output,
// mlp.py:134-138,149; sigmoid' = s (1 - s)), dX = dz_0 W_0.
__global__ void k_backward_rows_f64(nirc_spec_t sp, const double* __restrict__ theta,
                                    const double* __restrict__ zs, const double* __restrict__ dY,
                                    int64_t n, double* __restrict__ dzs, double* __restrict__ dX) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const int zw = zsw(sp);
  int zoff[NIRC_MAX_LAYERS + 1];
  zoff[0] = 0;
  for (int l = 0; l < sp.n_layers; ++l) zoff[l + 1] = zoff[l] + sp.dims[l + 1];
  const double* zr = zs + row * zw;
  double* dzr = dzs + row * zw;
  const int L = sp.n_layers - 1, dout = sp.dims[sp.n_layers];
  double cur[kMaxW], nxt[kMaxW];
  for (int j = 0; j < dout; ++j) {
    const double z = zr[zoff[L] + j];
    double g;
    if (sp.out_act == 0) {
      g = z >= 0.0 ? dY[row * dout + j] : 0.0;
    } else {
      const double s = 1.0 / (1.0 + exp(-z));
      g = dY[row * dout + j] * s * (1.0 - s);
    }
    cur[j] = g;
    dzr[zoff[L] + j] = g;
  }
  for (int l = L; l >= 0; --l) {
    const int din = sp.dims[l], dl = sp.dims[l + 1];
    const double* W = theta + sp.w_off[l];
    for (int i = 0; i < din; ++i) {
      double acc = 0.0;
      for (int j = 0; j < dl; ++j) acc = fma(cur[j], W[j * din + i], acc);
      if (l > 0) {
        const double g = zr[zoff[l - 1] + i] >= 0.0 ? acc : 0.0;
        nxt[i] = g;
        dzr[zoff[l - 1] + i] = g;
      } else {
        dX[row * sp.in_dim + i] = acc;
      }
    }
    for (int i = 0; i < din; ++i) cur[i] = nxt[i];
  }
}

// Per-block partials of dW_l = dz_l^T a_{l-1}, db_l = sum dz_l over the
// block's rows (rows in order); grid = (row blocks, layers).
__global__ void k_wgrad_part_f64(nirc_spec_t sp, const double* __restrict__ X,
                                 const double* __restrict__ zs, const double* __restrict__ dzs,
                                 int64_t n, double* __restrict__ part, int64_t np) {
  const int l = blockIdx.y;
  const int din = sp.dims[l], dout = sp.dims[l + 1];
  const int zw = zsw(sp);
  int zoff_l = 0;
  for (int k = 0; k < l; ++k) zoff_l += sp.dims[k + 1];
  const int zoff_prev = zoff_l - (l > 0 ? sp.dims[l] : 0);
  const int64_t r0 = (int64_t)blockIdx.x * kRows, r1 = n < r0 + kRows ? n : r0 + kRows;
  double* pb = part + (int64_t)blockIdx.x * np;
  for (int e = threadIdx.x; e < dout * (din + 1); e += blockDim.x) {
    const int j = e / (din + 1), i = e % (din + 1);
    double acc = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      double a = 1.0;
      if (i < din) {
        if (l == 0) {
          a = X[r * sp.in_dim + i];
        } else {
          const double z = zs[r * zw + zoff_prev + i];
          a = z > 0.0 ? z : 0.0;  // hidden activations are ReLU
        }
      }
      acc = fma(dzs[r * zw + zoff_l + j], a, acc);
    }
    if (i < din) pb[(sp.w_off[l] - sp.grid_len) + j * din + i] = acc;
    else pb[(sp.b_off[l] - sp.grid_len) + j] = acc;
  }
}

// grad[grid_len + p] += sum over blocks (block order) of the partials.
__global__ void k_wgrad_reduce_f64(const double* __restrict__ part, int nblk, int64_t np,
                                   double* __restrict__ grad_mlp) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * np + p];
  grad_mlp[p] += s;
}

// losses.py:23-70 on f64 predictions (every operation f64, as numpy does
// for an f64 prediction); den (nullable) = the frozen relative-L2
// denominator (losses.py:33-42 frozen_denom).
constexpr int kLossThreads = 256;
__global__ void k_loss_f64(int kind, const double* __restrict__ Y, const double* __restrict__ T,
                           const double* __restrict__ pdf, const double* __restrict__ rmean,
                           const double* __restrict__ den, double eps, int64_t n,
                           double* __restrict__ dY, double* __restrict__ partial,
                           int32_t* __restrict__ flags) {
  __shared__ double red[kLossThreads];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (i < n) {
    const double p = kind == 3 ? 1.0 : pdf[i];
    if (kind != 3 && !(p > 0.0)) atomicOr(flags, 1);
    const double nt = (double)(n * 3);
    for (int c = 0; c < 3; ++c) {
      const double y = Y[i * 3 + c], t = T[i * 3 + c];
      double v, g;
      switch (kind) {
        case 0: {
          const double diff = y - t;
          v = diff * diff / p;
          g = 2.0 * diff / p / nt;
          break;
        }
        case 1: {
          const double d = den ? den[i * 3 + c] : y * y + eps;
          const double diff = y - t;
          v = diff * diff / (p * d);
          g = 2.0 * diff / (p * d) / nt;
          break;
        }
        case 2: {
          const double dv = (t - y) / p - rmean[c];
          v = dv * dv;
          g = -2.0 * dv / p / nt;
          break;
        }
        default: {
          const double q = y < 1e-6 ? 1e-6 : (y > 1.0 - 1e-6 ? 1.0 - 1e-6 : y);
          v = -(t * log(q) + (1.0 - t) * log(1.0 - q));
          g = (q - t) / (q * (1.0 - q)) / nt;
        }
      }
      acc += v;
      dY[i * 3 + c] = g;
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kLossThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void k_loss_final_f64(const double* __restrict__ partial, int nblk, int64_t n,
                                 double* __restrict__ out, int32_t* __restrict__ flags) {
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[b];
  const double v = s / (double)(n * 3);
  out[0] = v;
  if (!isfinite(v)) atomicOr(flags, 2);
}

// adam.py:20-33 on f64 state: a non-finite gradient skips the step (t
// unchanged); m += (1 - b1)(g - m), v += (1 - b2)(g^2 - v), theta -=
// lr m^ / (sqrt(v^) + eps), all f64.
__global__ void k_adam_check_f64(const double* __restrict__ g, int64_t n, int32_t* __restrict__ bad) {
  int found = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    found |= !isfinite(g[i]);
  if (__syncthreads_or(found) && threadIdx.x == 0) atomicExch(bad, 1);
}

__global__ void k_adam_apply_f64(double* __restrict__ theta, double* __restrict__ m,
                                 double* __restrict__ v, const double* __restrict__ g, int64_t n,
                                 const int64_t* __restrict__ t, double lr, double b1, double b2,
                                 double eps, const int32_t* __restrict__ bad) {
  if (bad[0]) return;
  const double tn = (double)(t[0] + 1);
  const double bc1 = 1.0 - pow(b1, tn), bc2 = 1.0 - pow(b2, tn);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = g[i];
    double mi = m[i], vi = v[i];
    mi = __dadd_rn(mi, __dmul_rn(__dsub_rn(1.0, b1), __dsub_rn(gi, mi)));
    vi = __dadd_rn(vi, __dmul_rn(__dsub_rn(1.0, b2), __dsub_rn(__dmul_rn(gi, gi), vi)));
    m[i] = mi;
    v[i] = vi;
    const double mh = __ddiv_rn(mi, bc1), vh = __ddiv_rn(vi, bc2);
    theta[i] = __dsub_rn(theta[i], __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps)));
  }
}

__global__ void k_adam_tick_f64(int64_t* __restrict__ t, int64_t* __restrict__ skipped,
                                const int32_t* __restrict__ bad) {
  if (bad[0]) skipped[0] += 1;
  else t[0] += 1;
}

int check_f64_spec(const nirc_spec_t* sp) {
  if (!sp) {
    set_last_error("spec is NULL");
    return NIRC_E_CONFIG;
  }
  for (int l = 0; l <= sp->n_layers; ++l)
    if (sp->dims[l] > kMaxW) {
      set_last_error("f64 path: layer width %d > %d", sp->dims[l], kMaxW);
      return NIRC_E_UNSUPPORTED;
    }
  return NIRC_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline int nb(int64_t n, int t) { return (int)((n + t - 1) / t); }

}  // namespace
}  // namespace nirc

using namespace nirc;

extern "C" int nirc_encode_f64(const nirc_spec_t* spec, const double* theta, const double* pos,
                               const double* normal, const double* albedo, const double* rough,
                               const double* dirs, int64_t n, double* X, int64_t* entries,
                               float* weights, void* stream) {
  int st = check_f64_spec(spec);
  if (st) return st;
  if (n <= 0) return NIRC_OK;
  k_encode_f64<<<nb(n, 128), 128, 0, S(stream)>>>(*spec, theta, pos, normal, albedo, rough, dirs,
                                                  n, X, entries, weights);
  NIRC_LAUNCH_CHECK("k_encode_f64");
  return NIRC_OK;
}

extern "C" int nirc_mlp_forward_f64(const nirc_spec_t* spec, const double* theta,
                                    const double* X, int64_t n, double* Y, double* zs,
                                    int32_t* nonfinite_flag, void* stream) {
  int st = check_f64_spec(spec);
  if (st) return st;
  if (n <= 0) return NIRC_OK;
  if (nonfinite_flag) {  // mlp.py:104-105 raises DivergenceError
    k_adam_check_f64<<<4 * 148, 256, 0, S(stream)>>>(theta, spec->theta_len, nonfinite_flag);
    NIRC_LAUNCH_CHECK("k_finite_f64");
  }
  k_forward_f64<<<nb(n, kRows), kRows, 0, S(stream)>>>(*spec, theta, X, n, Y, zs);
  NIRC_LAUNCH_CHECK("k_forward_f64");
  return NIRC_OK;
}

extern "C" int nirc_mlp_backward_f64(const nirc_spec_t* spec, const double* theta,
                                     const double* X, const double* zs, const double* dY,
                                     int64_t n, double* grad, double* dX, double* scratch,
                                     void* stream) {
  int st = check_f64_spec(spec);
  if (st) return st;
  if (n <= 0) return NIRC_OK;
  cudaStream_t s = S(stream);
  k_backward_rows_f64<<<nb(n, kRows), kRows, 0, s>>>(*spec, theta, zs, dY, n, scratch, dX);
  NIRC_LAUNCH_CHECK("k_backward_rows_f64");
  const int64_t np = spec->theta_len - spec->grid_len;
  const int blocks = nb(n, kRows);
  AsyncBuf part(s);
  NIRC_CUDA_TRY(part.alloc((size_t)blocks * np * 8));
  k_wgrad_part_f64<<<dim3(blocks, spec->n_layers), 256, 0, s>>>(
      *spec, X, zs, scratch, n, static_cast<double*>(part.p), np);
  NIRC_LAUNCH_CHECK("k_wgrad_part_f64");
  k_wgrad_reduce_f64<<<nb(np, 256), 256, 0, s>>>(static_cast<const double*>(part.p), blocks, np,
                                                grad + spec->grid_len);
  NIRC_LAUNCH_CHECK("k_wgrad_reduce_f64");
  return NIRC_OK;
}

extern "C" int nirc_scatter_grid_grad_f64(const nirc_spec_t* spec, double* grad,
                                          const int64_t* entries, const float* weights,
                                          const double* dX, int64_t n, int64_t dx_stride,
                                          void* stream) {
  int st = check_f64_spec(spec);
  if (st) return st;
  if (n <= 0) return NIRC_OK;
  return ordered_scatter<double>(*spec, grad, entries, weights, dX, n, dx_stride, nullptr,
                                 nullptr, 0, S(stream));
}

extern "C" int nirc_loss_f64(int32_t kind, const double* Y, const double* target,
                             const double* pdf, const double* running_mean,
                             const double* frozen_denom, double eps, int64_t n, double* dY,
                             double* loss_out, int32_t* status_flags, void* stream) {
  if (kind < 0 || kind > 3) {
    set_last_error("unknown loss kind %d", kind);
    return NIRC_E_CONFIG;
  }
  if (n <= 0) return NIRC_OK;
  cudaStream_t s = S(stream);
  const int blocks = nb(n, kLossThreads);
  AsyncBuf part(s);
  NIRC_CUDA_TRY(part.alloc((size_t)blocks * 8));
  k_loss_f64<<<blocks, kLossThreads, 0, s>>>(kind, Y, target, pdf, running_mean, frozen_denom, eps,
                                             n, dY, static_cast<double*>(part.p), status_flags);
  NIRC_LAUNCH_CHECK("k_loss_f64");
  k_loss_final_f64<<<1, 1, 0, s>>>(static_cast<const double*>(part.p), blocks, n, loss_out,
                                   status_flags);
  NIRC_LAUNCH_CHECK("k_loss_final_f64");
  return NIRC_OK;
}

extern "C" int nirc_adam_step_f64(double* theta, double* m, double* v, const double* grad,
                                  int64_t n, int64_t* t, int64_t* skipped, double lr,
                                  double beta1, double beta2, double eps, int32_t* scratch,
                                  void* stream) {
  if (n <= 0) return NIRC_OK;
  cudaStream_t s = S(stream);
  NIRC_CUDA_TRY(cudaMemsetAsync(scratch, 0, 4, s));
  k_adam_check_f64<<<4 * 148, 256, 0, s>>>(grad, n, scratch);
  k_adam_apply_f64<<<4 * 148, 256, 0, s>>>(theta, m, v, grad, n, t, lr, beta1, beta2, eps, scratch);
  k_adam_tick_f64<<<1, 1, 0, s>>>(t, skipped, scratch);
  NIRC_LAUNCH_CHECK("k_adam_f64");
  return NIRC_OK;
}
