// full_forward (pkg/src/nirclab/mlp.py:216-224 = encode_batch + mlp_forward)
// as ONE persistent sm_100a kernel: every thread encodes its query row
// (12-level hash grid, 8-corner gathers from the L2-resident tables, f64
// SH, aux) straight into the SMEM A tile, then the group runs the network
// on tcgen05 (tc_mlp.cuh).  No X, entries or weights ever touch HBM.
#include <cstdlib>
#include <mutex>
#include "common.cuh"
#include "tc_mlp.cuh"

namespace nirc {
namespace tc {
// Packs theta's layers into hi/lo operand images (tf32 or fp16) in the
// canonical K-major layout (N rows, K columns).  One thread per (layer, n, k).
// `unsafe` (zeroed by the caller) is set when a weight is outside the fp16
// range of the F16x2 split: the launch then recomputes every row in fp32.
__global__ void k_pack_weights(nirc_spec_t sp, TcNet net, const float* __restrict__ theta,
                               uint8_t* __restrict__ img, float* __restrict__ bias,
                               int32_t* __restrict__ unsafe) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  int base = 0;
  for (int l = 0; l < net.nl; ++l) {
    const int cnt = net.N[l] * net.K[l];
    if (t >= base && t < base + cnt) {
      const int e = t - base;
      const int nrow = e / net.K[l], k = e % net.K[l];
      const int din = sp.dims[l], dout = sp.dims[l + 1];
      float w = 0.0f;
      if (nrow < dout && k < din) w = theta[sp.w_off[l] + (int64_t)nrow * din + k];
      if (net.prec == PrecF16x2::kId) {
        if (!(fabsf(w) < kF16Max)) atomicExch(unsafe, 1);
        const __half hi = __float2half_rn(w);
        const __half lo = __float2half_rn(w - __half2float(hi));
        const uint32_t o = op_offset<PrecF16x2>(nrow, k, net.N[l]);
        *reinterpret_cast<__half*>(img + net.woff[l] + o) = hi;
        *reinterpret_cast<__half*>(img + net.woff[l] + net.N[l] * net.K[l] * 2 + o) = lo;
      } else {
        const float hi = tf32_hi(w);
        const uint32_t o = op_offset<PrecTF32x3>(nrow, k, net.N[l]);
        *reinterpret_cast<float*>(img + net.woff[l] + o) = hi;
        *reinterpret_cast<float*>(img + net.woff[l] + net.N[l] * net.K[l] * 4 + o) = w - hi;
      }
    }
    base += cnt;
  }
  if (t < net.nl * 64) {
    const int l = t / 64, j = t % 64;
    bias[t] = j < sp.dims[l + 1] ? theta[sp.b_off[l] + j] : 0.0f;
  }
}

}  // namespace tc

// The default NIRC input layout (test_default_layout_dimensions,
// tests/test_neural.py:81-88): 12 levels x 2 feats, 4 SH bands, 7 aux.
constexpr int kL = 12, kF = 2, kBands = 4, kIn = 47, kK0 = 48;
constexpr int kDenseLevels = 4;  // dense coarse levels of the cfg2 kernel (measured best)


__host__ __device__ inline bool is_default_layout(const nirc_spec_t& sp) {
  return sp.levels == kL && sp.feats == kF && sp.bands == kBands && sp.in_dim == kIn &&
         sp.dims[0] == kIn;
}

// Encodes one query row into x[48] (x[47] = 0 pad) as encode_batch
// (encoding.py:111-157): hash + aux blocks bit-identical; the SH block
// bit-identical with the f64 recurrences (F32SH = false; measured faster in
// the fused kernel too: the f64 pipe is otherwise idle there) or within
// 5e-7 abs in fp32 (F32SH = true).  Levels < ND are
// gathered from the CTA's dense shared-memory copies, the rest from the
// L2-resident tables.
template <int ND, bool F32SH, bool kPairs = false>
__device__ __forceinline__ void encode_default(const nirc_spec_t& sp,
                                               const float* __restrict__ theta, const double* p,
                                               const double* nrm, const double* alb,
                                               double rough, const double* d, float* x,
                                               const DenseLevels& dl, const float2* dense) {
  const float ux = norm_coord(p[0], sp.bb_min[0], sp.bb_inv[0]);
  const float uy = norm_coord(p[1], sp.bb_min[1], sp.bb_inv[1]);
  const float uz = norm_coord(p[2], sp.bb_min[2], sp.bb_inv[2]);
  const uint32_t T = 1u << sp.table_log2;
#pragma unroll
  for (int lvl = 0; lvl < kL; ++lvl) {
    const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
    // ND is a compile-time count: the 12 levels stay straight-line code and
    // the gathers of all levels overlap in flight
    // (kPairs: the dense levels are stored as x-pairs, fill_dense_levels_x2)
    const float2 f = lvl < ND
                         ? (kPairs ? level_features2_dense_x2(
                                         reinterpret_cast<const float4*>(dense) + dl.off[lvl],
                                         dl.R[lvl], c)
                                   : level_features2_dense(dense + dl.off[lvl], dl.R[lvl], c))
                     : (kPairs ? level_features2_pairs(theta + (size_t)lvl * T * kF, c, T - 1u)
                               : level_features2(theta + (size_t)lvl * T * kF, c, T - 1u));
    x[2 * lvl] = f.x;
    x[2 * lvl + 1] = f.y;
  }
  if (F32SH)
    sh4_f32((float)d[0], (float)d[1], (float)d[2], sp.sh_k, x + 24);
  else
    sh_eval<true>(d[0], d[1], d[2], kBands, sp.sh_k,
                  [&](int i, double v) { x[24 + i] = __double2float_rn(v); });
  x[40] = __double2float_rn(dmul(dadd(nrm[0], 1.0), 0.5));
  x[41] = __double2float_rn(dmul(dadd(nrm[1], 1.0), 0.5));
  x[42] = __double2float_rn(dmul(dadd(nrm[2], 1.0), 0.5));
  x[43] = __double2float_rn(alb[0]);
  x[44] = __double2float_rn(alb[1]);
  x[45] = __double2float_rn(alb[2]);
  x[46] = __double2float_rn(rough);
  x[47] = 0.0f;
}

template <class P, int NG, int ND, bool kPairs = false>
__global__ void __launch_bounds__(NG * 128, 1)
    k_full_forward_tc(nirc_spec_t sp, tc::TcNet net, tc::TcSmem L,
                      const float* __restrict__ theta, const uint8_t* __restrict__ wimg,
                      const float* __restrict__ bias_g, const double* __restrict__ pos,
                      const double* __restrict__ nrm, const double* __restrict__ alb,
                      const double* __restrict__ rough, const double* __restrict__ dirs,
                      int64_t n, float* __restrict__ Y, DenseLevels dl,
                      const int32_t* __restrict__ w_unsafe, int32_t* __restrict__ fix) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t tmem_base;
  const bool all_unsafe = w_unsafe != nullptr && *w_unsafe != 0;
  // dense coarse levels live in the region after the group A buffers
  float2* dense = reinterpret_cast<float2*>(smem + L.a_off + NG * L.abuf_bytes);
  if (ND > 0) {
    if (kPairs) fill_dense_levels_x2(sp, dl, theta, reinterpret_cast<float4*>(dense));
    else fill_dense_levels(sp, dl, theta, dense);
  }
  tc::tc_prologue(smem, L, net, NG, wimg, bias_g, tmem_base);
  const uint32_t s0 = tc::smem_u32(smem);
  const int group = threadIdx.x >> 7;
  const int tg = threadIdx.x & 127;
  const uint32_t a_hi = s0 + L.a_off + group * L.abuf_bytes;
  const uint32_t a_lo = a_hi + L.abuf_bytes / 2;
  const uint32_t mbar = s0 + L.bar_off + 8 * (1 + group);
  constexpr bool kTS = P::kId == tc::PrecF16x2::kId;
  const uint32_t tmem_d = tmem_base + group * (kTS ? tc::kTsColsPerGroup : 64u);
  const uint32_t lane_off = (uint32_t)((tg >> 5) * 32) << 16;
  const float* s_bias = reinterpret_cast<const float*>(smem + L.bias_off);
  const int dout = sp.dims[sp.n_layers];
  uint32_t phase = 0;
  const int64_t ntiles = (n + tc::kTileRows - 1) / tc::kTileRows;
  for (int64_t tile = (int64_t)blockIdx.x * NG + group; tile < ntiles;
       tile += (int64_t)gridDim.x * NG) {
    const int64_t row = tile * tc::kTileRows + tg;
    float x[kK0];
    if (row < n) {
      encode_default<ND, false, kPairs>(sp, theta, pos + 3 * row, nrm + 3 * row, alb + 3 * row,
                                        rough[row], dirs + 3 * row, x, dl, dense);
    } else {
#pragma unroll
      for (int k = 0; k < kK0; ++k) x[k] = 0.0f;
    }
    float y[4];
    if constexpr (kTS) {
      bool unsafe = all_unsafe || tc::f16_unsafe(x, kK0);
      tc::write_a_row_ts<kK0>(tmem_d + 64 + lane_off, tmem_d + 96 + lane_off, x);
      tc::run_chain_ts(net, s0 + L.w_off, s_bias, group, tg, tmem_d, mbar, phase, y, unsafe);
      // fp16 range guard: this warp's 32 rows go to the fp32 fix-up list
      if (__any_sync(0xffffffffu, unsafe && row < n) && (tg & 31) == 0)
        fix[1 + atomicAdd(fix, 1)] = (int32_t)(tile * 4 + (tg >> 5));
    } else {
      tc::write_a_row<P, kK0>(a_hi, a_lo, tg, x);
      tc::run_chain<P>(net, s0 + L.w_off, s_bias, group, tg, a_hi, a_lo, tmem_d, mbar, phase, y);
    }
    if (row < n)
      for (int j = 0; j < dout; ++j) Y[row * dout + j] = y[j];
  }
  tc::tc_epilogue(tmem_base, NG, P::kId);
}

__device__ inline void stage_net(const nirc_spec_t& sp, const float* __restrict__ theta, float* W) {
  const int np = (int)(sp.theta_len - sp.grid_len);
  for (int i = threadIdx.x; i < np; i += blockDim.x) W[i] = __ldg(theta + sp.grid_len + i);
}

__device__ inline void simt_full_row(const nirc_spec_t& sp, const float* __restrict__ theta,
                                     const float* __restrict__ W, const double* __restrict__ pos,
                                     const double* __restrict__ nrm,
                                     const double* __restrict__ alb,
                                     const double* __restrict__ rough,
                                     const double* __restrict__ dirs, int64_t row,
                                     float* __restrict__ Y) {
  float a[64], b[64];
  DenseLevels none{};
  encode_default<0, false>(sp, theta, pos + 3 * row, nrm + 3 * row, alb + 3 * row, rough[row],
                           dirs + 3 * row, a, none, nullptr);
  simt_net_row(sp, W, a, b);
  const int dout = sp.dims[sp.n_layers];
  for (int j = 0; j < dout; ++j) Y[row * dout + j] = a[j];
}

// fp32 SIMT twin of the same fusion (precision == 1): weights in smem,
// one thread per row, the reference's accuracy class.
__global__ void k_full_forward_simt(nirc_spec_t sp, const float* __restrict__ theta,
                                    const double* __restrict__ pos, const double* __restrict__ nrm,
                                    const double* __restrict__ alb,
                                    const double* __restrict__ rough,
                                    const double* __restrict__ dirs, int64_t n,
                                    float* __restrict__ Y) {
  extern __shared__ float smem_f[];
  stage_net(sp, theta, smem_f);
  __syncthreads();
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  simt_full_row(sp, theta, smem_f, pos, nrm, alb, rough, dirs, row, Y);
}

// fp16 range fix-up of k_full_forward_tc<F16x2>: recomputes the flagged
// 32-row units (fix[1 .. fix[0]]) with the fp32 twin; a no-op launch when
// nothing was flagged.
__global__ void k_full_forward_fix(nirc_spec_t sp, const float* __restrict__ theta,
                                   const double* __restrict__ pos, const double* __restrict__ nrm,
                                   const double* __restrict__ alb, const double* __restrict__ rough,
                                   const double* __restrict__ dirs, int64_t n,
                                   float* __restrict__ Y, const int32_t* __restrict__ fix) {
  extern __shared__ float smem_f[];
  const int cnt = fix[0];
  if (cnt == 0) return;
  stage_net(sp, theta, smem_f);
  __syncthreads();
  const int warps = blockDim.x >> 5;
  for (int e = blockIdx.x * warps + (threadIdx.x >> 5); e < cnt; e += gridDim.x * warps) {
    const int64_t row = (int64_t)fix[1 + e] * 32 + (threadIdx.x & 31);
    if (row < n) simt_full_row(sp, theta, smem_f, pos, nrm, alb, rough, dirs, row, Y);
  }
}

// status_flags[0] |= bit when x[0:n] holds a non-finite value (the
// reference's mlp_forward raises DivergenceError, mlp.py:104-105).
__global__ void k_finite_flag(const float* __restrict__ x, int64_t n, int32_t* __restrict__ flags,
                              int32_t bit) {
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, bit);
}

// The packed weight image of one launch lives in a stream-ordered buffer
// owned by the caller (no library state is shared between calls or streams).
int pack_weights(const nirc_spec_t& sp, const tc::TcNet& net, const float* theta,
                 cudaStream_t s, AsyncBuf& buf, PackedNet* out) {
  const size_t img_bytes = ((size_t)net.wbytes + 255) & ~(size_t)255;
  NIRC_CUDA_TRY(buf.alloc(img_bytes + tc::kMaxTcLayers * 64 * 4 + 16));
  out->img = static_cast<uint8_t*>(buf.p);
  out->bias = reinterpret_cast<float*>(out->img + img_bytes);
  out->unsafe = reinterpret_cast<int32_t*>(out->bias + tc::kMaxTcLayers * 64);
  NIRC_CUDA_TRY(cudaMemsetAsync(out->unsafe, 0, 4, s));
  int total = 0;
  for (int l = 0; l < net.nl; ++l) total += net.N[l] * net.K[l];
  total = total > net.nl * 64 ? total : net.nl * 64;
  tc::k_pack_weights<<<(total + 255) / 256, 256, 0, s>>>(sp, net, theta, out->img, out->bias,
                                                         out->unsafe);
  NIRC_LAUNCH_CHECK("k_pack_weights");
  return NIRC_OK;
}

int finite_flag(const float* x, int64_t n, int32_t* flags, int32_t bit, cudaStream_t s) {
  if (!flags || n <= 0) return NIRC_OK;
  const int64_t nb = (n + 255) / 256;
  k_finite_flag<<<(int)(nb < 4 * 148 ? nb : 4 * 148), 256, 0, s>>>(x, n, flags, bit);
  NIRC_LAUNCH_CHECK("k_finite_flag");
  return NIRC_OK;
}

int sm_count() {
  static int cached[16] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return 148;
  if (!cached[dev]) {
    int c = 0;
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = c > 0 ? c : 148;
  }
  return cached[dev];
}

// Chooses the number of 128-row groups per CTA that fit in shared memory.
int tc_groups_for(const tc::TcNet& net, uint32_t extra_per_group) {
  const int gmax = net.prec == tc::PrecF16x2::kId ? 4 : 2;
  for (int g = gmax; g >= 1; --g)
    if (tc::tc_smem_layout(net, g, g * extra_per_group).total <= 227u * 1024u - 256u) return g;
  return 0;
}

}  // namespace nirc

using namespace nirc;

extern "C" int nirc_device_sm_count(void) { return sm_count(); }

namespace nirc {
// The fused forward of n rows into Y (the body of nirc_full_forward).
static int full_forward_impl(const nirc_spec_t* spec, const float* theta, const double* pos,
                             const double* normal, const double* albedo, const double* rough,
                             const double* dirs, int64_t n, float* Y, int32_t precision,
                             cudaStream_t s) {
  if (!is_default_layout(*spec)) {
    set_last_error("fused forward needs the default 12x2 hash + 4-band SH layout");
    return NIRC_E_UNSUPPORTED;
  }
  const size_t simt_sm = (size_t)(spec->theta_len - spec->grid_len) * 4;
  if (precision == 1) {
    if (simt_sm > 200 * 1024 || spec->dims[1] > 64) return NIRC_E_UNSUPPORTED;
    NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)k_full_forward_simt,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)simt_sm));
    k_full_forward_simt<<<(int)((n + 127) / 128), 128, simt_sm, s>>>(*spec, theta, pos, normal,
                                                                    albedo, rough, dirs, n, Y);
    NIRC_LAUNCH_CHECK("k_full_forward_simt");
    return NIRC_OK;
  }
  const int prec = precision == 2 ? tc::PrecF16x2::kId : tc::PrecTF32x3::kId;
  tc::TcNet net;
  if (!tc::tc_net_for(*spec, &net, prec)) {
    set_last_error("network shape not supported by the tcgen05 path");
    return NIRC_E_UNSUPPORTED;
  }
  const int ng = tc_groups_for(net, 0);
  if (ng == 0) {
    set_last_error("network too large for the tcgen05 shared-memory plan");
    return NIRC_E_UNSUPPORTED;
  }
  AsyncBuf wbuf(s), fbuf(s);
  PackedNet pn;
  int st = pack_weights(*spec, net, theta, s, wbuf, &pn);
  if (st) return st;
  const int64_t ntiles = (n + tc::kTileRows - 1) / tc::kTileRows;
  int32_t* fix = nullptr;
  if (prec == tc::PrecF16x2::kId) {  // fp16 range fix-up list: count + 32-row units
    if (simt_sm > 200 * 1024 || spec->dims[1] > 64) return NIRC_E_UNSUPPORTED;
    NIRC_CUDA_TRY(fbuf.alloc((size_t)(4 * ntiles + 1) * 4));
    fix = static_cast<int32_t*>(fbuf.p);
    NIRC_CUDA_TRY(cudaMemsetAsync(fix, 0, 4, s));
  }
  // coarse levels as dense shared-memory arrays (levels 0..ND-1), if the
  // plan leaves room; NIRC_DENSE_LEVELS overrides (0 = all from L2/L1)
  int nd_want = kDenseLevels;
  if (const char* e = getenv("NIRC_DENSE_LEVELS")) nd_want = atoi(e);
  const uint32_t base_total = tc::tc_smem_layout(net, ng, 0).total;
  DenseLevels dl = dense_levels_for(*spec, 227u * 1024u - 1024u - base_total, nd_want);
  if (dl.n != 0 && dl.n != 4 && dl.n != 5) dl = dense_levels_for(*spec, 0, 0);
  // paired 16-byte gathers need 16-byte aligned level tables (NIRC_PAIRS=0: 8-byte only)
  dl.pairs = (reinterpret_cast<uintptr_t>(theta) & 15u) == 0;
  if (const char* e = getenv("NIRC_PAIRS")) dl.pairs = dl.pairs && atoi(e) != 0;
  // the paired kernel keeps its dense levels as x-pairs (16 bytes per entry)
  // where they fit, else the 8-byte layout of the unpaired kernel
  if (dl.pairs && !(ng == 4 && dl.n == 4 &&
                    base_total + (uint32_t)dl.off[dl.n] * 16u <= 227u * 1024u - 1024u))
    dl.pairs = 0;
  const uint32_t dense_entry = (ng == 4 && dl.n == 4 && dl.pairs) ? 16u : 8u;
  const tc::TcSmem L = tc::tc_smem_layout(net, ng, (uint32_t)dl.off[dl.n] * dense_entry);
  const int64_t want = (ntiles + ng - 1) / ng;
  const int grid = (int)(want < sm_count() ? want : sm_count());
  auto launch = [&](auto kern, int threads) -> int {
    NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)kern,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    kern<<<grid, threads, L.total, s>>>(*spec, net, L, theta, pn.img, pn.bias, pos, normal, albedo,
                                        rough, dirs, n, Y, dl, pn.unsafe, fix);
    return NIRC_OK;
  };
  if (prec == tc::PrecF16x2::kId) {
    if (ng == 4 && dl.n == 4 && dl.pairs)
      st = launch(k_full_forward_tc<tc::PrecF16x2, 4, 4, true>, 512);
    else if (ng == 4 && dl.n == 5) st = launch(k_full_forward_tc<tc::PrecF16x2, 4, 5>, 512);
    else if (ng == 4 && dl.n == 4) st = launch(k_full_forward_tc<tc::PrecF16x2, 4, 4>, 512);
    else if (ng == 4) st = launch(k_full_forward_tc<tc::PrecF16x2, 4, 0>, 512);
    else if (ng == 3) st = launch(k_full_forward_tc<tc::PrecF16x2, 3, 0>, 384);
    else if (ng == 2) st = launch(k_full_forward_tc<tc::PrecF16x2, 2, 0>, 256);
    else st = launch(k_full_forward_tc<tc::PrecF16x2, 1, 0>, 128);
  } else {
    if (ng == 2) st = launch(k_full_forward_tc<tc::PrecTF32x3, 2, 0>, 256);
    else st = launch(k_full_forward_tc<tc::PrecTF32x3, 1, 0>, 128);
  }
  if (st) return st;
  NIRC_LAUNCH_CHECK("k_full_forward_tc");
  if (fix) {
    NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)k_full_forward_fix,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)simt_sm));
    k_full_forward_fix<<<sm_count(), 128, simt_sm, s>>>(*spec, theta, pos, normal, albedo, rough,
                                                       dirs, n, Y, fix);
    NIRC_LAUNCH_CHECK("k_full_forward_fix");
  }
  return NIRC_OK;
}
}  // namespace nirc

extern "C" int nirc_full_forward(const nirc_spec_t* spec, const float* theta, const double* pos,
                                 const double* normal, const double* albedo, const double* rough,
                                 const double* dirs, int64_t n, float* Y, int32_t precision,
                                 int32_t* status_flags, void* stream) {
  if (!spec) return NIRC_E_CONFIG;
  if (n <= 0) return NIRC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st = finite_flag(theta, spec->theta_len, status_flags, NIRC_FLAG_DIVERGED, s);
  if (st) return st;
  return full_forward_impl(spec, theta, pos, normal, albedo, rough, dirs, n, Y, precision, s);
}

// ---------------------------------------------------------------------
// Cache._query / nirc_query (caches.py:211-233), amortised as the reference
// does it: each surface's 12-level hash block is encoded ONCE
// (k_surface_features, one thread per (surface, level)), then every
// direction row reads its surface's 24 features + aux and evaluates SH and
// the network in the fused tcgen05 chain (k_query_tc).
namespace nirc {
__global__ void k_surface_features(nirc_spec_t sp, const float* __restrict__ theta,
                                   const double* __restrict__ surf, int64_t n_surf,
                                   float* __restrict__ feat) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_surf * kL) return;
  const int64_t k = t / kL;
  const int lvl = (int)(t % kL);
  const double* r = surf + 10 * k;
  const float ux = norm_coord(r[0], sp.bb_min[0], sp.bb_inv[0]);
  const float uy = norm_coord(r[1], sp.bb_min[1], sp.bb_inv[1]);
  const float uz = norm_coord(r[2], sp.bb_min[2], sp.bb_inv[2]);
  const uint32_t T = 1u << sp.table_log2;
  const float2 f = level_features2(theta + (size_t)lvl * T * kF, level_cell(ux, uy, uz, sp.res[lvl]),
                                   T - 1u);
  reinterpret_cast<float2*>(feat)[k * kL + lvl] = f;
}

// Encoded row of direction i: the surface's shared hash block, SH of the
// direction (f64 recurrences, bit-identical to encode_batch), aux block.
__device__ inline bool query_row(const nirc_spec_t& sp, const float* __restrict__ feat,
                                 const double* __restrict__ surf, int64_t n_surf,
                                 const double* __restrict__ dirs,
                                 const int32_t* __restrict__ dir_to_surf, int64_t i, float* x) {
  const int32_t k = dir_to_surf[i];
  if (k < 0 || k >= n_surf) return false;
  const float4* f4 = reinterpret_cast<const float4*>(feat + (int64_t)k * 24);
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const float4 v = f4[q];
    x[4 * q] = v.x;
    x[4 * q + 1] = v.y;
    x[4 * q + 2] = v.z;
    x[4 * q + 3] = v.w;
  }
  const double* d = dirs + 3 * i;
  sh_eval<true>(d[0], d[1], d[2], kBands, sp.sh_k,
                [&](int j, double v) { x[24 + j] = __double2float_rn(v); });
  const double* r = surf + 10 * (int64_t)k;
  x[40] = __double2float_rn(dmul(dadd(r[3], 1.0), 0.5));
  x[41] = __double2float_rn(dmul(dadd(r[4], 1.0), 0.5));
  x[42] = __double2float_rn(dmul(dadd(r[5], 1.0), 0.5));
  x[43] = __double2float_rn(r[6]);
  x[44] = __double2float_rn(r[7]);
  x[45] = __double2float_rn(r[8]);
  x[46] = __double2float_rn(r[9]);
  x[47] = 0.0f;
  return true;
}

template <int NG>
__global__ void __launch_bounds__(NG * 128, 1)
    k_query_tc(nirc_spec_t sp, tc::TcNet net, tc::TcSmem L, const uint8_t* __restrict__ wimg,
               const float* __restrict__ bias_g, const float* __restrict__ feat,
               const double* __restrict__ surf, int64_t n_surf, const double* __restrict__ dirs,
               const int32_t* __restrict__ dir_to_surf, int64_t n, float* __restrict__ Y,
               const int32_t* __restrict__ w_unsafe, int32_t* __restrict__ fix,
               int32_t* __restrict__ flags) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t tmem_base;
  const bool all_unsafe = *w_unsafe != 0;
  tc::tc_prologue(smem, L, net, NG, wimg, bias_g, tmem_base);
  const uint32_t s0 = tc::smem_u32(smem);
  const int group = threadIdx.x >> 7;
  const int tg = threadIdx.x & 127;
  const uint32_t mbar = s0 + L.bar_off + 8 * (1 + group);
  const uint32_t tmem_d = tmem_base + group * tc::kTsColsPerGroup;
  const uint32_t lane_off = (uint32_t)((tg >> 5) * 32) << 16;
  const float* s_bias = reinterpret_cast<const float*>(smem + L.bias_off);
  const int dout = sp.dims[sp.n_layers];
  uint32_t phase = 0;
  const int64_t ntiles = (n + tc::kTileRows - 1) / tc::kTileRows;
  for (int64_t tile = (int64_t)blockIdx.x * NG + group; tile < ntiles;
       tile += (int64_t)gridDim.x * NG) {
    const int64_t row = tile * tc::kTileRows + tg;
    float x[kK0];
    bool ok = true;
    if (row < n) ok = query_row(sp, feat, surf, n_surf, dirs, dir_to_surf, row, x);
    if (row >= n || !ok) {
#pragma unroll
      for (int k = 0; k < kK0; ++k) x[k] = 0.0f;
    }
    if (!ok) atomicOr(flags, NIRC_FLAG_BAD_INDEX);
    float y[4];
    bool unsafe = all_unsafe || tc::f16_unsafe(x, kK0);
    tc::write_a_row_ts<kK0>(tmem_d + 64 + lane_off, tmem_d + 96 + lane_off, x);
    tc::run_chain_ts(net, s0 + L.w_off, s_bias, group, tg, tmem_d, mbar, phase, y, unsafe);
    if (__any_sync(0xffffffffu, unsafe && row < n && ok) && (tg & 31) == 0)
      fix[1 + atomicAdd(fix, 1)] = (int32_t)(tile * 4 + (tg >> 5));
    if (row < n)
      for (int j = 0; j < dout; ++j) Y[row * dout + j] = ok ? y[j] : __int_as_float(0x7fc00000);
  }
  tc::tc_epilogue(tmem_base, NG, tc::PrecF16x2::kId);
}

// fp32 fix-up / twin of k_query_tc: the rows of fix's 32-row units (all rows
// when fix == nullptr).
__global__ void k_query_simt(nirc_spec_t sp, const float* __restrict__ theta,
                             const float* __restrict__ feat, const double* __restrict__ surf,
                             int64_t n_surf, const double* __restrict__ dirs,
                             const int32_t* __restrict__ dir_to_surf, int64_t n,
                             float* __restrict__ Y, const int32_t* __restrict__ fix,
                             int32_t* __restrict__ flags) {
  extern __shared__ float smem_f[];
  const int64_t cnt = fix ? fix[0] : (n + 31) / 32;
  if (cnt == 0) return;
  stage_net(sp, theta, smem_f);
  __syncthreads();
  const int warps = blockDim.x >> 5;
  const int dout = sp.dims[sp.n_layers];
  for (int64_t e = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); e < cnt;
       e += (int64_t)gridDim.x * warps) {
    const int64_t row = (fix ? (int64_t)fix[1 + e] : e) * 32 + (threadIdx.x & 31);
    if (row >= n) continue;
    float a[64], b[64];
    if (!query_row(sp, feat, surf, n_surf, dirs, dir_to_surf, row, a)) {
      atomicOr(flags, NIRC_FLAG_BAD_INDEX);
      for (int j = 0; j < dout; ++j) Y[row * dout + j] = __int_as_float(0x7fc00000);
      continue;
    }
    simt_net_row(sp, smem_f, a, b);
    for (int j = 0; j < dout; ++j) Y[row * dout + j] = a[j];
  }
}
}  // namespace nirc

extern "C" int nirc_query(const nirc_spec_t* spec, const float* theta, const double* surf,
                          int64_t n_surf, const double* dirs, const int32_t* dir_to_surf,
                          int64_t n_dirs, float* Y, int32_t precision, int32_t* status_flags,
                          void* stream) {
  if (!spec) return NIRC_E_CONFIG;
  if (n_dirs <= 0) return NIRC_OK;
  if (n_surf <= 0) {
    set_last_error("directions given without surfaces");
    return NIRC_E_CONFIG;
  }
  if (!status_flags) {
    set_last_error("nirc_query needs status_flags (bad indices are reported there)");
    return NIRC_E_CONFIG;
  }
  if (!is_default_layout(*spec)) {
    set_last_error("amortised query needs the default 12x2 hash + 4-band SH layout");
    return NIRC_E_UNSUPPORTED;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st = finite_flag(theta, spec->theta_len, status_flags, NIRC_FLAG_DIVERGED, s);
  if (st) return st;
  const size_t simt_sm = (size_t)(spec->theta_len - spec->grid_len) * 4;
  if (simt_sm > 200 * 1024 || spec->dims[1] > 64) return NIRC_E_UNSUPPORTED;
  AsyncBuf fbuf(s), wbuf(s), xbuf(s);
  NIRC_CUDA_TRY(fbuf.alloc((size_t)n_surf * 24 * 4));
  float* feat = static_cast<float*>(fbuf.p);
  k_surface_features<<<(unsigned)((n_surf * kL + 255) / 256), 256, 0, s>>>(*spec, theta, surf,
                                                                          n_surf, feat);
  NIRC_LAUNCH_CHECK("k_surface_features");
  NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)k_query_simt,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)simt_sm));
  tc::TcNet net;
  const bool tc_ok = precision == 2 && tc::tc_net_for(*spec, &net, tc::PrecF16x2::kId) &&
                     tc_groups_for(net, 0) == 4;
  if (!tc_ok) {  // fp32 twin (precision 1; 0 also lands here: amortised rows are fp32-class)
    const int64_t units = (n_dirs + 31) / 32;
    k_query_simt<<<(int)((units + 3) / 4 < 4 * 148 ? (units + 3) / 4 : 4 * 148), 128, simt_sm, s>>>(
        *spec, theta, feat, surf, n_surf, dirs, dir_to_surf, n_dirs, Y, nullptr, status_flags);
    NIRC_LAUNCH_CHECK("k_query_simt");
    return NIRC_OK;
  }
  PackedNet pn;
  if ((st = pack_weights(*spec, net, theta, s, wbuf, &pn))) return st;
  const int64_t ntiles = (n_dirs + tc::kTileRows - 1) / tc::kTileRows;
  NIRC_CUDA_TRY(xbuf.alloc((size_t)(4 * ntiles + 1) * 4));
  int32_t* fix = static_cast<int32_t*>(xbuf.p);
  NIRC_CUDA_TRY(cudaMemsetAsync(fix, 0, 4, s));
  const tc::TcSmem L = tc::tc_smem_layout(net, 4, 0);
  const int64_t want = (ntiles + 3) / 4;
  const int grid = (int)(want < sm_count() ? want : sm_count());
  NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)k_query_tc<4>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
  k_query_tc<4><<<grid, 512, L.total, s>>>(*spec, net, L, pn.img, pn.bias, feat, surf, n_surf, dirs,
                                           dir_to_surf, n_dirs, Y, pn.unsafe, fix, status_flags);
  NIRC_LAUNCH_CHECK("k_query_tc");
  k_query_simt<<<sm_count(), 128, simt_sm, s>>>(*spec, theta, feat, surf, n_surf, dirs, dir_to_surf,
                                                n_dirs, Y, fix, status_flags);
  NIRC_LAUNCH_CHECK("k_query_simt");
  return NIRC_OK;
}
