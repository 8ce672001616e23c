// Ordered hash-grid gradient scatter: scatter_grid_grad
// (pkg/src/nirclab/encoding.py:160-167) with np.add.at's exact semantics --
// every slot accumulates its contributions sequentially in entry order
// ((row, level, corner) row-major), starting from the slot's current value.
// Run-to-run deterministic, and bit-identical to the reference given the same
// weights and input gradients (the reference adds w * dG, an f32 product for
// f32 theta and an f64 one for its f64 shadow mode).
//
//   1. keys[e] = slot of entry e, vals[e] = e         (entries given, or
//      recomputed from the records' positions for the training rows)
//   2. stable radix sort of (key, e) pairs            (cub::DeviceRadixSort)
//   3. one thread per run of equal keys sums it in e order
//
// Used by the batch API (nirc_scatter_grid_grad[_f64]) and by the training
// step's deterministic mode (the tile kernels write the rows' dX instead of
// issuing atomics).
#include <cub/device/device_radix_sort.cuh>
#include "common.cuh"

namespace nirc {

namespace {

__global__ void k_keys_from_entries(const int64_t* __restrict__ entries, int64_t ne,
                                    uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  keys[e] = (uint32_t)entries[e];
  vals[e] = (uint32_t)e;
}

// Training rows: row r of the batch is record idx[r0 + r]; entry e =
// (r * L + lvl) * 8 + c, slot = lvl * T + hash (encode_batch's entries).
__device__ inline LevelCell row_cell(const nirc_spec_t& sp, const double* __restrict__ pos,
                                     const int64_t* __restrict__ idx, int64_t row, int lvl) {
  const double* p = pos + 3 * idx[row];
  const float ux = norm_coord(p[0], sp.bb_min[0], sp.bb_inv[0]);
  const float uy = norm_coord(p[1], sp.bb_min[1], sp.bb_inv[1]);
  const float uz = norm_coord(p[2], sp.bb_min[2], sp.bb_inv[2]);
  return level_cell(ux, uy, uz, sp.res[lvl]);
}

__global__ void k_keys_from_rows(nirc_spec_t sp, const double* __restrict__ pos,
                                 const int64_t* __restrict__ idx, int64_t r0, int64_t nrows,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows * sp.levels) return;
  const int64_t r = t / sp.levels;
  const int lvl = (int)(t % sp.levels);
  const LevelCell c = row_cell(sp, pos, idx, r0 + r, lvl);
  const uint32_t T = 1u << sp.table_log2;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int64_t e = t * 8 + k;
    keys[e] = (uint32_t)lvl * T + corner_hash(c, k, T - 1u);
    vals[e] = (uint32_t)e;
  }
}

// One thread per sorted position; the first of each run of equal keys sums
// the run in entry order.  weights == nullptr: recompute the trilinear
// weight from the record position (training rows).
template <typename T>
__global__ void k_sum_runs(nirc_spec_t sp, int64_t ne, const uint32_t* __restrict__ skeys,
                           const uint32_t* __restrict__ svals, const float* __restrict__ weights,
                           const T* __restrict__ dX, int64_t stride, T* __restrict__ grad,
                           const double* __restrict__ pos, const int64_t* __restrict__ idx,
                           int64_t r0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ne) return;
  const uint32_t key = skeys[i];
  if (i > 0 && skeys[i - 1] == key) return;
  const int F = sp.feats, L = sp.levels;
  T acc[4];
  for (int f = 0; f < F && f < 4; ++f) acc[f] = grad[(int64_t)key * F + f];
  int64_t end = i + 1;
  while (end < ne && skeys[end] == key) ++end;
  // the run's contributions are loaded 8 at a time (independent gathers in
  // flight) and added strictly in entry order
  for (int64_t j0 = i; j0 < end; j0 += 8) {
    float w[8];
    T d[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (j0 + u < end) {
        const uint32_t e = svals[j0 + u];
        const int64_t row = e / (8 * L);
        const int lvl = (int)((e / 8) % L), c = (int)(e % 8);
        w[u] = weights != nullptr ? weights[e]
                                  : corner_weight(row_cell(sp, pos, idx, r0 + row, lvl), c);
        for (int f = 0; f < F && f < 4; ++f) d[u][f] = dX[row * stride + lvl * F + f];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (j0 + u < end) {
        for (int f = 0; f < F && f < 4; ++f) {
          if constexpr (sizeof(T) == 4) {
            acc[f] = __fadd_rn(acc[f], __fmul_rn(w[u], d[u][f]));
          } else {
            acc[f] = __dadd_rn(acc[f], __dmul_rn((double)w[u], d[u][f]));
          }
        }
      }
    }
  }
  for (int f = 0; f < F && f < 4; ++f) grad[(int64_t)key * F + f] = acc[f];
}

int key_bits(const nirc_spec_t& sp) {
  const uint64_t nslots = (uint64_t)sp.levels << sp.table_log2;
  int b = 1;
  while ((1ull << b) < nslots) ++b;
  return b;
}

}  // namespace

// ne = n * levels * 8 entries; keys from `entries` when given, otherwise
// from the training rows (pos, idx, r0).  T = float or double.
template <typename T>
int ordered_scatter(const nirc_spec_t& sp, T* grad, const int64_t* entries, const float* weights,
                    const T* dX, int64_t n, int64_t stride, const double* pos, const int64_t* idx,
                    int64_t r0, cudaStream_t s) {
  const int64_t ne = n * sp.levels * 8;
  if (ne <= 0) return NIRC_OK;
  if (ne >= (1ll << 31)) {
    set_last_error("ordered scatter: too many entries (%lld)", (long long)ne);
    return NIRC_E_UNSUPPORTED;
  }
  const int bits = key_bits(sp);
  size_t temp = 0;
  NIRC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t*)nullptr,
                                                (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                                (uint32_t*)nullptr, (int)ne, 0, bits, s));
  AsyncBuf buf(s);
  const size_t arr = ((size_t)ne * 4 + 255) & ~(size_t)255;
  NIRC_CUDA_TRY(buf.alloc(4 * arr + temp + 256));
  uint8_t* p = static_cast<uint8_t*>(buf.p);
  uint32_t *keys = (uint32_t*)p, *vals = (uint32_t*)(p + arr), *skeys = (uint32_t*)(p + 2 * arr),
           *svals = (uint32_t*)(p + 3 * arr);
  void* tmp = p + 4 * arr;
  if (entries != nullptr) {
    k_keys_from_entries<<<(unsigned)((ne + 255) / 256), 256, 0, s>>>(entries, ne, keys, vals);
  } else {
    const int64_t nt = n * sp.levels;
    k_keys_from_rows<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(sp, pos, idx, r0, n, keys, vals);
  }
  NIRC_LAUNCH_CHECK("k_keys");
  NIRC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, temp, keys, skeys, vals, svals, (int)ne, 0,
                                                bits, s));
  k_sum_runs<T><<<(unsigned)((ne + 255) / 256), 256, 0, s>>>(sp, ne, skeys, svals, weights, dX,
                                                            stride, grad, pos, idx, r0);
  NIRC_LAUNCH_CHECK("k_sum_runs");
  return NIRC_OK;
}

template int ordered_scatter<float>(const nirc_spec_t&, float*, const int64_t*, const float*,
                                    const float*, int64_t, int64_t, const double*, const int64_t*,
                                    int64_t, cudaStream_t);
template int ordered_scatter<double>(const nirc_spec_t&, double*, const int64_t*, const float*,
                                     const double*, int64_t, int64_t, const double*,
                                     const int64_t*, int64_t, cudaStream_t);

// ---------------------------------------------------------------------
// Deterministic grid gradient of a training step (the tile kernels' rows):
// integer addition is associative, so every slot accumulates in 64-bit fixed
// point with atomics and the result is independent of their order.  Per
// level, contributions w * dX are scaled by 2^k with k chosen from the
// level's max |dX| (written by the tile kernels) so that 8 B of them fit in
// 2^61: absolute resolution 2^-44 of the level's largest contribution, i.e.
// fp32-class relative accuracy for every slot within 2^-20 of it (smaller
// ones move Adam by < 1e-6 of a step).  Coarse levels aggregate per CTA in
// shared memory first.  The float gradient is written back by
// k_fixed_to_float.
namespace {
__device__ inline double fixed_scale(uint32_t maxbits, int64_t nrows, bool inverse) {
  int e = (int)(maxbits >> 23) - 126;  // |x| < 2^e
  if (maxbits == 0u) e = 0;
  int lg = 0;
  while ((1ll << lg) < nrows * 8) ++lg;  // 2^lg >= the contributions one slot can get
  const int k = 61 - lg - e;
  return inverse ? ldexp(1.0, -k) : ldexp(1.0, k);
}

__global__ void __launch_bounds__(256) k_fixed_scatter(nirc_spec_t sp, const float* __restrict__ dX,
                                                       int64_t nrows, const uint32_t* __restrict__ lvlmax,
                                                       const double* __restrict__ pos,
                                                       const int64_t* __restrict__ idx, int64_t r0,
                                                       unsigned long long* __restrict__ acc,
                                                       DenseLevels dl, int64_t bnrows) {
  extern __shared__ unsigned long long s_acc[];  // coarse levels, 2 features per vertex
  __shared__ double s_sc[NIRC_MAX_LEVELS];
  const int ncoarse = dl.off[dl.n];
  for (int i = threadIdx.x; i < 2 * ncoarse; i += blockDim.x) s_acc[i] = 0ull;
  if (threadIdx.x < sp.levels) s_sc[threadIdx.x] = fixed_scale(lvlmax[threadIdx.x], bnrows, false);
  __syncthreads();
  const uint32_t T = 1u << sp.table_log2;
  // block b: rows [b * 64, b * 64 + 64) x all levels
  const int64_t rbase = (int64_t)blockIdx.x * 64;
  for (int t = threadIdx.x; t < 64 * sp.levels; t += blockDim.x) {
    const int64_t r = rbase + t / sp.levels;
    const int lvl = t % sp.levels;
    if (r >= nrows) continue;
    const float d0 = dX[r * 24 + 2 * lvl], d1 = dX[r * 24 + 2 * lvl + 1];
    if (d0 == 0.0f && d1 == 0.0f) continue;
    const double sc = s_sc[lvl];
    const LevelCell c = row_cell(sp, pos, idx, r0 + r, lvl);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float w = corner_weight(c, k);
      const long long q0 = __double2ll_rn((double)__fmul_rn(w, d0) * sc);
      const long long q1 = __double2ll_rn((double)__fmul_rn(w, d1) * sc);
      if (lvl < dl.n) {
        const int R = dl.R[lvl];
        const int v = dl.off[lvl] + ((c.iz + ((k >> 2) & 1)) * R + (c.iy + ((k >> 1) & 1))) * R +
                      c.ix + (k & 1);
        atomicAdd(&s_acc[2 * v], (unsigned long long)q0);
        atomicAdd(&s_acc[2 * v + 1], (unsigned long long)q1);
      } else {
        const uint64_t slot = (uint64_t)lvl * T + corner_hash(c, k, T - 1u);
        atomicAdd(&acc[2 * slot], (unsigned long long)q0);
        atomicAdd(&acc[2 * slot + 1], (unsigned long long)q1);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ncoarse; i += blockDim.x) {
    const unsigned long long a = s_acc[2 * i], b = s_acc[2 * i + 1];
    if (a == 0ull && b == 0ull) continue;
    int l = 0;
    while (i >= dl.off[l + 1]) ++l;
    const int R = dl.R[l], e = i - dl.off[l];
    const uint64_t slot = (uint64_t)l * T + hash3((uint32_t)(e % R), (uint32_t)((e / R) % R),
                                                  (uint32_t)(e / (R * R)), T - 1u);
    atomicAdd(&acc[2 * slot], a);
    atomicAdd(&acc[2 * slot + 1], b);
  }
}

__global__ void k_fixed_to_float(nirc_spec_t sp, unsigned long long* __restrict__ acc,
                                 const uint32_t* __restrict__ lvlmax, int64_t bnrows,
                                 float* __restrict__ grad) {
  __shared__ double s_inv[NIRC_MAX_LEVELS];
  if (threadIdx.x < sp.levels) s_inv[threadIdx.x] = fixed_scale(lvlmax[threadIdx.x], bnrows, true);
  __syncthreads();
  const int shift = sp.table_log2 + 1;  // grid entry i belongs to level i >> shift
  const int64_t n2 = sp.grid_len / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 a = reinterpret_cast<const ulonglong2*>(acc)[i];
    if (a.x == 0ull && a.y == 0ull) continue;
    const double inv = s_inv[(int)((2 * i) >> shift)];
    reinterpret_cast<float2*>(grad)[i] = make_float2(__double2float_rn((double)(long long)a.x * inv),
                                                     __double2float_rn((double)(long long)a.y * inv));
  }
}
}  // namespace

// dX rows [0, nrows) (row r = batch row r0 + r, stride 24) -> grad's grid
// part (overwritten where touched; the caller zeroes it); acc: grid_len
// zeroed u64 accumulators.
int fixed_scatter_rows(const nirc_spec_t& sp, float* grad, const float* dX, int64_t nrows,
                       const uint32_t* lvlmax, const double* pos, const int64_t* idx, int64_t r0,
                       int64_t batch_rows, unsigned long long* acc, cudaStream_t s) {
  if (nrows <= 0) return NIRC_OK;
  DenseLevels dl = dense_levels_for(sp, 80 * 1024, 4);
  const size_t sm = (size_t)dl.off[dl.n] * 16;
  NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)k_fixed_scatter,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_fixed_scatter<<<(unsigned)((nrows + 63) / 64), 256, sm, s>>>(sp, dX, nrows, lvlmax, pos, idx,
                                                                 r0, acc, dl, batch_rows);
  NIRC_LAUNCH_CHECK("k_fixed_scatter");
  k_fixed_to_float<<<4 * 148, 256, 0, s>>>(sp, acc, lvlmax, batch_rows, grad);
  NIRC_LAUNCH_CHECK("k_fixed_to_float");
  return NIRC_OK;
}

}  // namespace nirc
