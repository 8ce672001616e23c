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
__global__ void k_pack_weights(nirc_spec_t sp, TcNet net, const float* __restrict__ theta,
                               uint8_t* __restrict__ img, float* __restrict__ bias) {
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
template <int ND, bool F32SH>
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
    const float2 f = lvl < ND ? level_features2_dense(dense + dl.off[lvl], dl.R[lvl], c)
                              : level_features2(theta + (size_t)lvl * T * kF, c, T - 1u);
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

template <class P, int NG, int ND>
__global__ void __launch_bounds__(NG * 128, 1)
    k_full_forward_tc(nirc_spec_t sp, tc::TcNet net, tc::TcSmem L,
                      const float* __restrict__ theta, const uint8_t* __restrict__ wimg,
                      const float* __restrict__ bias_g, const double* __restrict__ pos,
                      const double* __restrict__ nrm, const double* __restrict__ alb,
                      const double* __restrict__ rough, const double* __restrict__ dirs,
                      int64_t n, float* __restrict__ Y, DenseLevels dl) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t tmem_base;
  // dense coarse levels live in the region after the group A buffers
  float2* dense = reinterpret_cast<float2*>(smem + L.a_off + NG * L.abuf_bytes);
  if (ND > 0) fill_dense_levels(sp, dl, theta, dense);
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
      encode_default<ND, false>(sp, theta, pos + 3 * row, nrm + 3 * row, alb + 3 * row,
                                rough[row], dirs + 3 * row, x, dl, dense);
    } else {
#pragma unroll
      for (int k = 0; k < kK0; ++k) x[k] = 0.0f;
    }
    float y[4];
    if constexpr (kTS) {
      tc::write_a_row_ts<kK0>(tmem_d + 64 + lane_off, tmem_d + 96 + lane_off, x);
      tc::run_chain_ts(net, s0 + L.w_off, s_bias, group, tg, tmem_d, mbar, phase, y);
    } else {
      tc::write_a_row<P, kK0>(a_hi, a_lo, tg, x);
      tc::run_chain<P>(net, s0 + L.w_off, s_bias, group, tg, a_hi, a_lo, tmem_d, mbar, phase, y);
    }
    if (row < n)
      for (int j = 0; j < dout; ++j) Y[row * dout + j] = y[j];
  }
  tc::tc_epilogue(tmem_base, NG, P::kId);
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
  const int np = (int)(sp.theta_len - sp.grid_len);
  float* W = smem_f;
  for (int i = threadIdx.x; i < np; i += blockDim.x) W[i] = __ldg(theta + sp.grid_len + i);
  __syncthreads();
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  float a[64], b[64];
  DenseLevels none{};
  encode_default<0, false>(sp, theta, pos + 3 * row, nrm + 3 * row, alb + 3 * row, rough[row],
                 dirs + 3 * row, a, none, nullptr);
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
  const int dout = sp.dims[sp.n_layers];
  for (int j = 0; j < dout; ++j) Y[row * dout + j] = a[j];
}

// Per-device cache of packed weight images (the library's only state).
struct WeightCache {
  uint8_t* img = nullptr;
  float* bias = nullptr;
};
static WeightCache g_wcache[16];
static std::mutex g_wmutex;

int get_weight_cache(uint8_t** img, float** bias) {
  int dev = 0;
  NIRC_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) return NIRC_E_CUDA;
  std::lock_guard<std::mutex> lk(g_wmutex);
  WeightCache& c = g_wcache[dev];
  if (!c.img) {
    NIRC_CUDA_TRY(cudaMalloc(&c.img, 192 * 1024));
    NIRC_CUDA_TRY(cudaMalloc(&c.bias, tc::kMaxTcLayers * 64 * 4));
  }
  *img = c.img;
  *bias = c.bias;
  return NIRC_OK;
}

int pack_weights(const nirc_spec_t& sp, const tc::TcNet& net, const float* theta,
                 cudaStream_t s, uint8_t** img, float** bias) {
  int st = get_weight_cache(img, bias);
  if (st) return st;
  int total = 0;
  for (int l = 0; l < net.nl; ++l) total += net.N[l] * net.K[l];
  total = total > net.nl * 64 ? total : net.nl * 64;
  tc::k_pack_weights<<<(total + 255) / 256, 256, 0, s>>>(sp, net, theta, *img, *bias);
  NIRC_LAUNCH_CHECK("k_pack_weights");
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
    if (tc::tc_smem_layout(net, g, g * extra_per_group).total <= 227u * 1024u) return g;
  return 0;
}

}  // namespace nirc

using namespace nirc;

extern "C" int nirc_device_sm_count(void) { return sm_count(); }

extern "C" int nirc_full_forward(const nirc_spec_t* spec, const float* theta, const double* pos,
                                 const double* normal, const double* albedo, const double* rough,
                                 const double* dirs, int64_t n, float* Y, int32_t precision,
                                 void* stream) {
  if (!spec) return NIRC_E_CONFIG;
  if (n <= 0) return NIRC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!is_default_layout(*spec)) {
    set_last_error("fused forward needs the default 12x2 hash + 4-band SH layout");
    return NIRC_E_UNSUPPORTED;
  }
  if (precision == 1) {
    const size_t sm = (size_t)(spec->theta_len - spec->grid_len) * 4;
    if (sm > 200 * 1024 || spec->dims[1] > 64) return NIRC_E_UNSUPPORTED;
    NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)k_full_forward_simt,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_full_forward_simt<<<(int)((n + 127) / 128), 128, sm, s>>>(*spec, theta, pos, normal, albedo,
                                                               rough, dirs, n, Y);
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
  uint8_t* img;
  float* bias;
  int st = pack_weights(*spec, net, theta, s, &img, &bias);
  if (st) return st;
  // coarse levels as dense shared-memory arrays (levels 0..ND-1), if the
  // plan leaves room; NIRC_DENSE_LEVELS overrides (0 = all from L2/L1)
  int nd_want = kDenseLevels;
  if (const char* e = getenv("NIRC_DENSE_LEVELS")) nd_want = atoi(e);
  const uint32_t base_total = tc::tc_smem_layout(net, ng, 0).total;
  DenseLevels dl = dense_levels_for(*spec, 227u * 1024u - 1024u - base_total, nd_want);
  if (dl.n != 0 && dl.n != 4 && dl.n != 5) dl = dense_levels_for(*spec, 0, 0);
  const tc::TcSmem L = tc::tc_smem_layout(net, ng, (uint32_t)dl.off[dl.n] * 8u);
  const int64_t ntiles = (n + tc::kTileRows - 1) / tc::kTileRows;
  const int64_t want = (ntiles + ng - 1) / ng;
  const int grid = (int)(want < sm_count() ? want : sm_count());
  auto launch = [&](auto kern, int threads) -> int {
    NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)kern,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    kern<<<grid, threads, L.total, s>>>(*spec, net, L, theta, img, bias, pos, normal, albedo,
                                        rough, dirs, n, Y, dl);
    return NIRC_OK;
  };
  if (prec == tc::PrecF16x2::kId) {
    if (ng == 4 && dl.n == 5) st = launch(k_full_forward_tc<tc::PrecF16x2, 4, 5>, 512);
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
  return NIRC_OK;
}

// ---------------------------------------------------------------------
// Cache._query / nirc_query (caches.py:211-233): directions against a set
// of shared surfaces.  Each direction's surface row (pos, ns, albedo,
// roughness) is gathered next to it and the rows go through the fused
// encode + MLP kernel; directions of one surface hit the same hash cells, so
// their repeated gathers are L1 hits.
namespace nirc {
__global__ void k_gather_surfaces(const double* __restrict__ surf, int64_t n_surf,
                                  const int32_t* __restrict__ dir_to_surf, int64_t n,
                                  double* pos, double* ns, double* alb, double* rough,
                                  int32_t* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t k = dir_to_surf[i];
  if (k < 0 || k >= n_surf) {
    atomicOr(bad, 1);
    return;
  }
  const double* r = surf + 10 * (int64_t)k;
  for (int c = 0; c < 3; ++c) {
    pos[3 * i + c] = r[c];
    ns[3 * i + c] = r[3 + c];
    alb[3 * i + c] = r[6 + c];
  }
  rough[i] = r[9];
}
}  // namespace nirc

extern "C" int nirc_query(const nirc_spec_t* spec, const float* theta, const double* surf,
                          int64_t n_surf, const double* dirs, const int32_t* dir_to_surf,
                          int64_t n_dirs, float* Y, int32_t precision, void* stream) {
  if (!spec) return NIRC_E_CONFIG;
  if (n_dirs <= 0) return NIRC_OK;
  if (n_surf <= 0) {
    set_last_error("directions given without surfaces");
    return NIRC_E_CONFIG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  AsyncBuf buf(s);
  NIRC_CUDA_TRY(buf.alloc((size_t)n_dirs * 10 * sizeof(double) + 16));
  double* pos = static_cast<double*>(buf.p);
  double* ns = pos + 3 * n_dirs;
  double* alb = ns + 3 * n_dirs;
  double* rough = alb + 3 * n_dirs;
  int32_t* bad = reinterpret_cast<int32_t*>(rough + n_dirs);
  NIRC_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int32_t), s));
  k_gather_surfaces<<<(unsigned)((n_dirs + 255) / 256), 256, 0, s>>>(surf, n_surf, dir_to_surf,
                                                                   n_dirs, pos, ns, alb, rough,
                                                                   bad);
  NIRC_LAUNCH_CHECK("k_gather_surfaces");
  int32_t h_bad = 0;
  NIRC_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  NIRC_CUDA_TRY(cudaStreamSynchronize(s));
  if (h_bad) {
    set_last_error("dir_to_surf index outside [0, n_surf)");
    return NIRC_E_CONFIG;
  }
  return nirc_full_forward(spec, theta, pos, ns, alb, rough, dirs, n_dirs, Y, precision, stream);
}
