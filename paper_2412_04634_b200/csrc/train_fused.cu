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
#include <cstdlib>
#include "common.cuh"
#include "tc_common.cuh"

namespace nirc {

constexpr int kTT = 512;         // threads per tile CTA
constexpr int kMaxW = 64;        // widest layer supported by the fused path
constexpr int kMaxNL = 8;
constexpr int kTileRows = 128;   // the API's tile (nirc_train_tiles); a CTA
                                 // takes all of one, or a half / quarter of
                                 // one when a launch has few tiles

struct FusedLayout {
  int nl, din[kMaxNL], dout[kMaxNL];
  int ldw[kMaxNL], ldt[kMaxNL];    // row strides of W (dout x ldw) and W^T (din x ldt)
  int w_off[kMaxNL], t_off[kMaxNL], b_off[kMaxNL];  // float offsets in smem
  int dz_off, a_off, red_off, total_floats;
  int x_col, tmem_cols;            // TMEM: z of layer l at cols 64*l, X at x_col
  int ld2;                         // row stride of the [feature][row] staging arrays
};

__host__ __device__ inline int up4(int x) { return (x + 3) & ~3; }

__host__ __device__ inline FusedLayout fused_layout(const nirc_spec_t& sp, int tr = kTileRows) {
  FusedLayout L{};
  L.ld2 = tr + 4;
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
  off += kMaxW * L.ld2;
  L.a_off = off;
  off += kMaxW * L.ld2;
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

// The step's weight image in the kernel's shared-memory layout: W (dout x
// ldw) and W^T (din x ldt) zero padded, and the biases, per layer -- built
// once per step so that every tile CTA stages it with TMA bulk copies.
__global__ void k_pack_train_weights(nirc_spec_t sp, FusedLayout L,
                                     const float* __restrict__ theta, float* __restrict__ img,
                                     const int32_t* __restrict__ gate = nullptr) {
  if (gate != nullptr && gate[0] == 0) return;  // fix-up list empty: nothing to pack
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

int sm_count();  // fused.cu

namespace t128 {
constexpr int kTR = 128;
#include "train_tile_body.cuh"
}  // namespace t128
namespace t64 {
constexpr int kTR = 64;
#include "train_tile_body.cuh"
}  // namespace t64
namespace t32 {
constexpr int kTR = 32;
#include "train_tile_body.cuh"
}  // namespace t32

// Rows per CTA for a launch of `ntiles` API tiles: a quarter or half tile
// when the launch would otherwise occupy a quarter / half of the SMs or
// less (small batches, the per-rank share of a sharded step), so the step's
// latency -- each thread's serial share of a row -- shrinks with it.
inline int tile_rows_for(int64_t ntiles) {
  const int64_t sms = sm_count();
  if (ntiles * 4 <= sms) return 32;
  if (ntiles * 2 <= sms) return 64;
  return 128;
}

// grad[mlp] = sum over tiles (tile order) of the partials.
// mode 0 (whole batch on this GPU): loss = mean; flags: 2 = non-finite loss
//   (stop), adam_bad = any non-finite gradient; bc (when given) = the Adam
//   bias corrections of the coming step, f32(1 - b^(t+1)) computed in f64
//   (the reference's python-float arithmetic, adam.py:30-31).
// mode 1 (one shard of a multi-GPU batch): aux[0] = this shard's raw loss
//   sum, aux[1] = 1 if a row of this shard had pdf <= 0; the finiteness
//   checks run after the cross-GPU sum (nirc_train_apply).
// Blocks [0, nb_mlp): 32 float4 columns of the MLP block each, warp w sums
// the tiles of chunk w (8 chunks) -- the chunk sums are added in warp order
// (deterministic); the remaining blocks check the grid gradient.
constexpr int kRedMlpCols = 32;
__global__ void __launch_bounds__(256) k_reduce_grad(
    nirc_spec_t sp, const float* __restrict__ partials, int ntiles,
    const double* __restrict__ loss_part, int64_t B, float* __restrict__ grad,
    double* __restrict__ loss_out, int32_t* __restrict__ flags, int32_t* __restrict__ adam_bad,
    int mode, int nb_mlp, const int64_t* __restrict__ t, float* __restrict__ bc, double b1,
    double b2) {
  if (mode == 0 && (flags[0] & 3)) return;
  const int np = (int)(sp.theta_len - sp.grid_len);
  const int64_t ps = part_stride(sp);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int bad = 0;
  if ((int)blockIdx.x < nb_mlp) {
    __shared__ float4 part[8][kRedMlpCols];
    const int c4 = blockIdx.x * kRedMlpCols + lane;  // float4 column
    const int per = (ntiles + 7) / 8;
    const int t0 = wid * per, t1 = min(ntiles, t0 + per);
    float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (4 * c4 + 4 > np && 4 * c4 < np) {
      // the column holding the last parameters: scalar loads, so the
      // partials' padding past np (never written) is not read
      const float* src = partials + 4 * c4;
      float* acc = &s4.x;
      for (int tt = t0; tt < t1; ++tt)
        for (int k = 0; 4 * c4 + k < np; ++k) acc[k] += src[(int64_t)tt * ps + k];
    } else if (4 * c4 < np) {
      const float4* src = reinterpret_cast<const float4*>(partials) + c4;
      int tt = t0;
      for (; tt + 8 <= t1; tt += 8) {  // 8 independent 16-byte loads in flight
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = src[(int64_t)(tt + u) * (ps / 4)];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          s4.x += v[u].x;
          s4.y += v[u].y;
          s4.z += v[u].z;
          s4.w += v[u].w;
        }
      }
      for (; tt < t1; ++tt) {
        const float4 v = src[(int64_t)tt * (ps / 4)];
        s4.x += v.x;
        s4.y += v.y;
        s4.z += v.z;
        s4.w += v.w;
      }
    }
    part[wid][lane] = s4;
    __syncthreads();
    if (wid == 0 && 4 * c4 < np) {
      float4 tot = part[0][lane];
      for (int w = 1; w < 8; ++w) {
        tot.x += part[w][lane].x;
        tot.y += part[w][lane].y;
        tot.z += part[w][lane].z;
        tot.w += part[w][lane].w;
      }
      const float vv[4] = {tot.x, tot.y, tot.z, tot.w};
      for (int k = 0; k < 4 && 4 * c4 + k < np; ++k) {
        grad[sp.grid_len + 4 * c4 + k] = vv[k];
        bad |= !isfinite(vv[k]);
      }
    }
  } else if (mode == 0) {  // the grid gradient's finiteness (float4 sweeps)
    const int64_t n4 = sp.grid_len / 4;
    const float4* g4 = reinterpret_cast<const float4*>(grad);
    for (int64_t i = (int64_t)(blockIdx.x - nb_mlp) * blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)(gridDim.x - nb_mlp) * blockDim.x) {
      const float4 v = g4[i];
      bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
    }
  }
  // the tiles' loss partials: 32 lanes sum contiguous chunks, then a fixed
  // shuffle tree (deterministic, no serial 128-long load chain)
  auto loss_sum = [&]() -> double {
    const int per = (ntiles + 31) / 32;
    double s = 0.0;
    for (int k = lane * per; k < min(ntiles, lane * per + per); ++k) s += loss_part[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    return s;
  };
  if (mode == 1) {
    if (blockIdx.x == 0 && wid == 0) {
      const double s = loss_sum();
      if (lane == 0) {
        loss_out[0] = s;
        loss_out[1] = (flags[0] & 1) ? 1.0 : 0.0;
      }
    }
    return;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(adam_bad, 1);
  if (blockIdx.x == gridDim.x - 1 && wid == 0) {
    const double s = loss_sum();
    if (lane != 0) return;
    const double v = s / (double)(B * 3);
    loss_out[0] = v;
    if (!isfinite(v)) atomicOr(flags, 2);
    if (bc != nullptr) {
      const double tn = (double)(t[0] + 1);
      bc[0] = (float)(1.0 - pow(b1, tn));
      bc[1] = (float)(1.0 - pow(b2, tn));
    }
  }
}

inline int reduce_blocks_mlp(const nirc_spec_t& sp) {
  const int64_t c4 = part_stride(sp) / 4;
  return (int)((c4 + kRedMlpCols - 1) / kRedMlpCols);
}

bool train_tc_supported(const nirc_spec_t& sp);
int launch_train_tc(const nirc_spec_t& sp, const float* theta, const float* rstat,
                    const nirc_records_t& rec, const int64_t* idx, int64_t B, int loss_kind,
                    double loss_eps, float* grad, float* partials, double* loss_part,
                    int32_t* flags, cudaStream_t s, int64_t tile0, int64_t tile1, int32_t* fix,
                    float* dx_out, uint32_t* lvlmax, void* zero_b, int64_t zero_b_bytes,
                    int32_t* adam_bad);
int64_t train_static_bytes(int64_t n);
int launch_record_static(const nirc_spec_t& sp, const nirc_records_t& rec, float* out,
                         cudaStream_t s);

// Tiles [tile0, tile1) of the batch (all of it on one GPU; one shard of it
// per GPU in the multi-GPU frame, mode 1).  The default layout trains on
// tcgen05 (train_tc.cu) with the fp32 SIMT kernel as the fp16-range fix-up;
// other layouts (or NIRC_TRAIN_SIMT=1) run the SIMT kernel throughout.
int fixed_scatter_rows(const nirc_spec_t& sp, float* grad, const float* dX, int64_t nrows,
                       const uint32_t* lvlmax, const double* pos, const int64_t* idx, int64_t r0,
                       int64_t batch_rows, unsigned long long* acc, cudaStream_t s);

int launch_fused_train(const nirc_spec_t& sp, const float* theta, const nirc_records_t& rec,
                       const int64_t* idx, int64_t B, int loss_kind, double loss_eps,
                       float* grad, float* partials, double* loss_part, double* loss_out,
                       int32_t* flags, int32_t* adam_bad, cudaStream_t s, int64_t tile0,
                       int64_t tile1, int mode, const float* rstat, bool deterministic,
                       const int64_t* t, float* bc, double b1, double b2) {
  const int ntiles = (int)(tile1 > tile0 ? tile1 - tile0 : 0);
  const bool force_simt = getenv("NIRC_TRAIN_SIMT") != nullptr;  // read per call (tests switch it)
  // deterministic mode: the tile kernels write the rows' grid gradients (and
  // each level's max |dX|); the 64-bit fixed-point scatter sums them
  // order-independently (scatter.cu)
  AsyncBuf dxb(s);
  float* dx_out = nullptr;
  uint32_t* lvlmax = nullptr;
  unsigned long long* acc = nullptr;
  const int64_t r0 = tile0 * kTileRows, r1 = tile1 * kTileRows < B ? tile1 * kTileRows : B;
  if (deterministic && ntiles > 0) {
    const size_t dxbytes = ((size_t)B * 24 * 4 + 255) & ~(size_t)255;
    NIRC_CUDA_TRY(dxb.alloc(dxbytes + 256 + (size_t)sp.grid_len * 8));
    dx_out = static_cast<float*>(dxb.p);
    lvlmax = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(dxb.p) + dxbytes);
    acc = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(dxb.p) + dxbytes + 256);
  }
  const bool tc_path = !force_simt && train_tc_supported(sp);
  if (lvlmax != nullptr && !(tc_path && ntiles > 0))  // the tc path zeroes them in its prepare
    NIRC_CUDA_TRY(cudaMemsetAsync(lvlmax, 0, 256 + (size_t)sp.grid_len * 8, s));
  auto det_scatter = [&]() -> int {
    if (!dx_out || r1 <= r0) return NIRC_OK;
    return fixed_scatter_rows(sp, grad, dx_out + r0 * 24, r1 - r0, lvlmax, rec.pos, idx, r0, B,
                              acc, s);
  };
  if (tc_path) {
    if (ntiles == 0) {
      NIRC_CUDA_TRY(cudaMemsetAsync(grad, 0, sp.grid_len * 4, s));
      if (adam_bad) NIRC_CUDA_TRY(cudaMemsetAsync(adam_bad, 0, 4, s));
    }
    if (ntiles > 0) {
      AsyncBuf fb(s), img(s), sb(s);
      NIRC_CUDA_TRY(fb.alloc((size_t)(ntiles + 1) * 4));
      int32_t* fix = static_cast<int32_t*>(fb.p);  // zeroed by k_train_prepare
      if (rstat == nullptr) {  // per-record static encoding (train_frame computes it once)
        NIRC_CUDA_TRY(sb.alloc((size_t)train_static_bytes(rec.n)));
        int st = launch_record_static(sp, rec, static_cast<float*>(sb.p), s);
        if (st) return st;
        rstat = static_cast<const float*>(sb.p);
      }
      int st = launch_train_tc(sp, theta, rstat, rec, idx, B, loss_kind, loss_eps, grad, partials,
                               loss_part, flags, s, tile0, tile1, fix, dx_out, lvlmax, lvlmax,
                               lvlmax ? 256 + (int64_t)sp.grid_len * 8 : 0, adam_bad);
      if (st) return st;
      // fp32 fix-up of the tiles beyond the fp16 range (CTAs past the list exit)
      const FusedLayout L = fused_layout(sp, kTileRows);
      const size_t sm = (size_t)L.total_floats * 4;
      NIRC_CUDA_TRY(img.alloc((size_t)L.dz_off * 4));
      k_pack_train_weights<<<dim3(16, L.nl), 256, 0, s>>>(sp, L, theta,
                                                         static_cast<float*>(img.p), fix);
      NIRC_LAUNCH_CHECK("k_pack_train_weights");
      NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)t128::k_train_tile,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      t128::k_train_tile<<<ntiles < 32 ? ntiles : 32, kTT, sm, s>>>(
          sp, L, theta, static_cast<const float*>(img.p), rec, idx, B, loss_kind, loss_eps, grad,
          partials, loss_part, flags, tile0, fix, dx_out, lvlmax);
      NIRC_LAUNCH_CHECK("k_train_tile(fix)");
      if ((st = det_scatter())) return st;
    }
    const int nbm = reduce_blocks_mlp(sp);
    k_reduce_grad<<<nbm + (mode == 0 ? 64 : 0), 256, 0, s>>>(
        sp, partials, ntiles, loss_part, B, grad, loss_out, flags, adam_bad, mode, nbm, t, bc,
        b1, b2);
    NIRC_LAUNCH_CHECK("k_reduce_grad");
    return NIRC_OK;
  }
  const int tr = tile_rows_for(ntiles);
  const int nsub = kTileRows / tr;
  const FusedLayout L = fused_layout(sp, tr);
  const size_t sm = (size_t)L.total_floats * 4;
  NIRC_CUDA_TRY(cudaMemsetAsync(grad, 0, sp.grid_len * 4, s));
  if (adam_bad) NIRC_CUDA_TRY(cudaMemsetAsync(adam_bad, 0, 4, s));
  AsyncBuf img(s);
  if (ntiles > 0) {
    NIRC_CUDA_TRY(img.alloc((size_t)L.dz_off * 4));
    k_pack_train_weights<<<dim3(16, L.nl), 256, 0, s>>>(sp, L, theta,
                                                       static_cast<float*>(img.p));
    NIRC_LAUNCH_CHECK("k_pack_train_weights");
    auto launch = [&](auto kern) -> int {
      NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)kern,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      kern<<<ntiles * nsub, kTT, sm, s>>>(sp, L, theta, static_cast<const float*>(img.p), rec,
                                          idx, B, loss_kind, loss_eps, grad, partials, loss_part,
                                          flags, tile0, nullptr, dx_out, lvlmax);
      return NIRC_OK;
    };
    int st = tr == 32 ? launch(t32::k_train_tile)
                      : tr == 64 ? launch(t64::k_train_tile) : launch(t128::k_train_tile);
    if (st) return st;
    NIRC_LAUNCH_CHECK("k_train_tile");
    if ((st = det_scatter())) return st;
  }
  const int nbm = reduce_blocks_mlp(sp);
  k_reduce_grad<<<nbm + (mode == 0 ? 64 : 0), 256, 0, s>>>(sp, partials, ntiles * nsub, loss_part,
                                                           B, grad, loss_out, flags, adam_bad,
                                                           mode, nbm, t, bc, b1, b2);
  NIRC_LAUNCH_CHECK("k_reduce_grad");
  return NIRC_OK;
}

}  // namespace nirc
