// Shared device building blocks for the NIRC hot path on sm_100a.
//
// Everything that must be BIT-EXACT against the reference lives here and is
// written with explicit round-to-nearest intrinsics (__fmul_rn, __dadd_rn,
// ...) so nvcc can never contract it into FMAs:
//   * splitmix64 counter RNG          pkg/src/nirclab/rng.py:59-106
//   * real SH, no Condon-Shortley     pkg/src/nirclab/sh.py:36-127
//   * XOR-primes hash + trilinear     pkg/src/nirclab/encoding.py:38-157
//   * cosine sampling / ONB           pkg/src/nirclab/core.py:39-74
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/nirc_b200.h"

#define NIRC_HD __host__ __device__ __forceinline__
#define NIRC_D __device__ __forceinline__

namespace nirc {

// ---------------------------------------------------------------- rng ----
// rng.py:23-31 constants, :59-64 mix64, :67-73 stream_key, :76-89 draws.
constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ull;
constexpr uint64_t M1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t M2 = 0x94D049BB133111EBull;
constexpr uint64_t P_RENDER = 0x01, P_TRAIN = 0x02, P_INIT = 0x03,
                   P_SHUFFLE = 0x04, P_BASELINE = 0x05, P_MEASURE = 0x06;
// rng.py:45-56 per-vertex dimension layout
constexpr int DIM_JITTER_X = 0, DIM_JITTER_Y = 1, VERTEX_DIM_BASE = 8,
              DIMS_PER_VERTEX = 64, OFF_LIGHT_PICK = 0, OFF_LIGHT_U = 1,
              OFF_LIGHT_V = 2, OFF_BSDF_U = 3, OFF_BSDF_V = 4, OFF_RR = 5,
              OFF_TERM = 6, OFF_CACHE = 8;

NIRC_HD uint64_t mix64(uint64_t x) {
  x += GAMMA;
  x = (x ^ (x >> 30)) * M1;
  x = (x ^ (x >> 27)) * M2;
  return x ^ (x >> 31);
}
NIRC_HD uint64_t stream_key(uint64_t seed, uint64_t purpose, uint64_t frame,
                            uint64_t pixel, uint64_t sample) {
  uint64_t k = mix64(seed ^ purpose);
  k = mix64(k ^ frame);
  k = mix64(k ^ pixel);
  return mix64(k ^ sample);
}
NIRC_HD uint64_t rand_u64(uint64_t key, uint64_t dim) {
  return mix64(key + GAMMA * dim);
}
// (u64 >> 11) * 2^-53: both steps are exact in f64.
NIRC_HD double rand_uniform(uint64_t key, uint64_t dim) {
  return (double)(rand_u64(key, dim) >> 11) * (1.0 / 9007199254740992.0);
}
// (float)rand_uniform(key, dim) in one conversion: rounding the 53-bit
// integer to f32 and scaling by the power of two 2^-53 is the same rounding.
NIRC_D float rand_uniform_f32(uint64_t key, uint64_t dim) {
  return __ull2float_rn(rand_u64(key, dim) >> 11) * 0x1p-53f;
}

// ----------------------------------------------------- exact f64 helpers --
NIRC_D double dmul(double a, double b) { return __dmul_rn(a, b); }
NIRC_D double dadd(double a, double b) { return __dadd_rn(a, b); }
NIRC_D double dsub(double a, double b) { return __dsub_rn(a, b); }
NIRC_D double ddiv(double a, double b) { return __ddiv_rn(a, b); }
NIRC_D double dsqrt(double a) { return __dsqrt_rn(a); }

// ------------------------------------------------------------------ SH ---
// sh.py:36-76 (scalar, numba) and :89-127 (batch, numpy).  The two differ in
// one association: the batch path advances P_m^m as (pmm*(2m-1))*s, the
// scalar path as pmm*((2m-1)*s).  `BatchOrder` selects which one to follow.
// The Legendre recurrences and the K*P*cos products are otherwise identical.
template <bool BatchOrder, typename Store>
NIRC_D void sh_eval(double x, double y, double z, int bands,
                    const double* __restrict__ sh_k, Store store) {
  const double s = dsqrt(dadd(dmul(x, x), dmul(y, y)));
  double cphi = 1.0, sphi = 0.0;
  if (s > 0.0) {
    cphi = ddiv(x, s);
    sphi = ddiv(y, s);
  }
  double cm = 1.0, sm = 0.0, pmm = 1.0;
  for (int m = 0; m < bands; ++m) {
    if (m > 0) {
      const double f = (double)(2 * m - 1);
      pmm = BatchOrder ? dmul(dmul(pmm, f), s) : dmul(pmm, dmul(f, s));
      const double cn = dsub(dmul(cm, cphi), dmul(sm, sphi));
      const double sn = dadd(dmul(sm, cphi), dmul(cm, sphi));
      cm = cn;
      sm = sn;
    }
    double p_lm2 = 0.0, p_lm1 = 0.0;
    for (int l = m; l < bands; ++l) {
      double p;
      if (l == m) {
        p = pmm;
      } else if (l == m + 1) {
        p = dmul(dmul(z, (double)(2 * m + 1)), pmm);
      } else {
        const double a = dmul(dmul((double)(2 * l - 1), z), p_lm1);
        const double b = dmul((double)(l + m - 1), p_lm2);
        p = ddiv(dsub(a, b), (double)(l - m));
      }
      p_lm2 = p_lm1;
      p_lm1 = p;
      const int base = l * l + l;
      if (m == 0) {
        store(base, dmul(sh_k[l * 8], p));
      } else {
        const double k = dmul(sh_k[l * 8 + m], p);
        store(base + m, dmul(k, cm));
        store(base - m, dmul(k, sm));
      }
    }
  }
}

// Real SH (bands = 4), the scalar-path recurrences of sh.py:36-76 in fp32.
// sh_k may be the spec's f64 table or its f32 rounding (the same values).
// Closed form of the scalar-path recurrences (sh.py:36-76, no Condon-Shortley
// phase): out[l^2 + l +- m] = K_lm * Pt_lm(z) * Re / Im (x + i y)^m with
// Pt_lm = P_lm / s^m the polynomial the recurrence builds -- no sqrt or
// division; within an ulp or two of the fp32 recurrence.
template <class KT>
NIRC_D void sh4_f32(float x, float y, float z, const KT* sh_k, float* out) {
  const float z2 = z * z;
  const float c2 = x * x - y * y, s2 = 2.0f * x * y;     // (x + i y)^2
  const float c3 = x * c2 - y * s2, s3 = x * s2 + y * c2;  // (x + i y)^3
  const float p20 = 1.5f * z2 - 0.5f;
  const float p30 = z * (2.5f * z2 - 1.5f);
  const float p31 = 7.5f * z2 - 1.5f;
  out[0] = (float)sh_k[0];
  out[2] = (float)sh_k[8] * z;
  out[3] = (float)sh_k[9] * x;
  out[1] = (float)sh_k[9] * y;
  out[6] = (float)sh_k[16] * p20;
  const float k21 = (float)sh_k[17] * (3.0f * z);
  out[7] = k21 * x;
  out[5] = k21 * y;
  const float k22 = (float)sh_k[18] * 3.0f;
  out[8] = k22 * c2;
  out[4] = k22 * s2;
  out[12] = (float)sh_k[24] * p30;
  const float k31 = (float)sh_k[25] * p31;
  out[13] = k31 * x;
  out[11] = k31 * y;
  const float k32 = (float)sh_k[26] * (15.0f * z);
  out[14] = k32 * c2;
  out[10] = k32 * s2;
  const float k33 = (float)sh_k[27] * 15.0f;
  out[15] = k33 * c3;
  out[9] = k33 * s3;
}

// ----------------------------------------------------------- hash grid ---
// encoding.py:38-42: (x*1 ^ y*P1 ^ z*P2) & (T-1).  The mask is < 2^32 so
// the low 32 bits of the u64 products decide the slot; u32 math is exact.
constexpr uint32_t P1 = 2654435761u;
constexpr uint32_t P2 = 805459861u;

NIRC_HD uint32_t hash3(uint32_t x, uint32_t y, uint32_t z, uint32_t mask) {
  return (x ^ (y * P1) ^ (z * P2)) & mask;
}

// Position normalisation, encoding.py:49-66 / :126-127: f64 affine into the
// padded scene box, clamp to [0,1], then round to f32.
NIRC_D float norm_coord(double p, double lo, double inv) {
  double u = dmul(dsub(p, lo), inv);
  u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
  return __double2float_rn(u);
}

struct LevelCell {
  int32_t ix, iy, iz;
  float wx, wy, wz;
};

// encoding.py:129-131: s = u * f32(res) (f32 RN), i = floor, w = s - i.
NIRC_D LevelCell level_cell(float ux, float uy, float uz, int res) {
  const float r = (float)res;
  const float sx = __fmul_rn(ux, r), sy = __fmul_rn(uy, r), sz = __fmul_rn(uz, r);
  LevelCell c;
  c.ix = (int32_t)floorf(sx);
  c.iy = (int32_t)floorf(sy);
  c.iz = (int32_t)floorf(sz);
  c.wx = __fsub_rn(sx, (float)c.ix);
  c.wy = __fsub_rn(sy, (float)c.iy);
  c.wz = __fsub_rn(sz, (float)c.iz);
  return c;
}

// Corner c: x = bit0, y = bit1, z = bit2; w = ((wx|1-wx)*(wy|1-wy))*(wz|1-wz)
// in f32 (encoding.py:81-85, :140-143).
NIRC_D float corner_weight(const LevelCell& c, int corner) {
  const float ax = (corner & 1) ? c.wx : __fsub_rn(1.0f, c.wx);
  const float ay = (corner & 2) ? c.wy : __fsub_rn(1.0f, c.wy);
  const float az = (corner & 4) ? c.wz : __fsub_rn(1.0f, c.wz);
  return __fmul_rn(__fmul_rn(ax, ay), az);
}
NIRC_D uint32_t corner_hash(const LevelCell& c, int corner, uint32_t mask) {
  return hash3((uint32_t)(c.ix + (corner & 1)), (uint32_t)(c.iy + ((corner >> 1) & 1)),
               (uint32_t)(c.iz + ((corner >> 2) & 1)), mask);
}

// Hash-grid features of one level for feats == 2 (the NIRC default):
// x[f] = sum_{c=0..7} (w_c * theta[slot_c*2+f]) accumulated in corner order
// from 0.0f, f32 RN (encoding.py:144-151).  The 8 gathers are issued before
// the dependent accumulation so they overlap in the memory system.
NIRC_D float2 level_features2(const float* __restrict__ table, const LevelCell& c,
                              uint32_t mask) {
  float2 g[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    g[k] = __ldg(reinterpret_cast<const float2*>(table) + corner_hash(c, k, mask));
  float x0 = 0.0f, x1 = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float w = corner_weight(c, k);
    x0 = __fadd_rn(x0, __fmul_rn(w, g[k].x));
    x1 = __fadd_rn(x1, __fmul_rn(w, g[k].y));
  }
  return make_float2(x0, x1);
}

// The same features with paired gathers: corners (x, y, z) and (x+1, y, z)
// hash to slots h and h ^ 1 when x is even (x + 1 = x ^ 1, the mask keeps
// bit 0), i.e. one aligned 16-byte slot pair; so the x-even corner pairs take
// one 16-byte load each and the x-odd ones a 16-byte plus an 8-byte load.
// Measured on B200 (tools/l2_gather_peak.cu): a random 16-byte L2 gather
// costs 1.25x an 8-byte one, so a level costs 5 (even x) or 9 (odd x) load
// units instead of 8.  The table must be 16-byte aligned.  Same values, same
// f32 accumulation order as level_features2.
NIRC_D float2 level_features2_pairs(const float* __restrict__ table, const LevelCell& c,
                                    uint32_t mask) {
  const float4* t4 = reinterpret_cast<const float4*>(table);
  const float2* t2 = reinterpret_cast<const float2*>(table);
  const bool even = (c.ix & 1) == 0;
  float2 g[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t h0 = corner_hash(c, 2 * q, mask);
    const float4 A = __ldg(t4 + (h0 >> 1));
    const bool hi = (h0 & 1u) != 0u;
    g[2 * q] = hi ? make_float2(A.z, A.w) : make_float2(A.x, A.y);
    if (even) g[2 * q + 1] = hi ? make_float2(A.x, A.y) : make_float2(A.z, A.w);
    else g[2 * q + 1] = __ldg(t2 + corner_hash(c, 2 * q + 1, mask));
  }
  float x0 = 0.0f, x1 = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float w = corner_weight(c, k);
    x0 = __fadd_rn(x0, __fmul_rn(w, g[k].x));
    x1 = __fadd_rn(x1, __fmul_rn(w, g[k].y));
  }
  return make_float2(x0, x1);
}

// Dense shared-memory copies of the coarse levels (feats == 2).  Level l's
// cell coordinates lie in [0, res_l] and its corners in [0, res_l + 1], so a
// dense (res_l + 2)^3 array indexed by (z, y, x) holds every slot the level
// can touch: dense[(z*R + y)*R + x] = table_l[hash3(x, y, z)] -- the same
// values, gathered from shared memory instead of scattered L2 lines.
struct DenseLevels {
  int n;                          // levels 0..n-1 are dense
  int pairs;                      // sparse levels: paired 16-byte gathers (aligned table)
  int R[NIRC_MAX_LEVELS];         // res + 2
  int off[NIRC_MAX_LEVELS + 1];   // float2 offsets; off[n] = total entries
};

inline DenseLevels dense_levels_for(const nirc_spec_t& sp, size_t budget_bytes,
                                    int max_levels = NIRC_MAX_LEVELS) {
  DenseLevels d{};
  int total = 0;
  d.off[0] = 0;
  for (int l = 0; l < sp.levels && l < max_levels; ++l) {
    const int R = sp.res[l] + 2;
    const long long cnt = (long long)R * R * R;
    if (sp.feats != 2 || (total + cnt) * 8 > (long long)budget_bytes) break;
    d.R[l] = R;
    total += (int)cnt;
    d.n = l + 1;
    d.off[l + 1] = total;
  }
  return d;
}

// Cooperative fill of the dense levels by the whole CTA.
NIRC_D void fill_dense_levels(const nirc_spec_t& sp, const DenseLevels& d,
                              const float* __restrict__ theta, float2* dense) {
  const uint32_t T = 1u << sp.table_log2;
  for (int l = 0; l < d.n; ++l) {
    const int R = d.R[l];
    const float2* tab = reinterpret_cast<const float2*>(theta + (size_t)l * T * 2);
    for (int i = threadIdx.x; i < R * R * R; i += blockDim.x) {
      const int x = i % R, y = (i / R) % R, z = i / (R * R);
      dense[d.off[l] + i] = __ldg(tab + hash3((uint32_t)x, (uint32_t)y, (uint32_t)z, T - 1u));
    }
  }
}

NIRC_D float2 level_features2_dense(const float2* dense, int R, const LevelCell& c) {
  const int b = (c.iz * R + c.iy) * R + c.ix;
  float2 g[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    g[k] = dense[b + (k & 1) + ((k >> 1) & 1) * R + ((k >> 2) & 1) * R * R];
  float x0 = 0.0f, x1 = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float w = corner_weight(c, k);
    x0 = __fadd_rn(x0, __fmul_rn(w, g[k].x));
    x1 = __fadd_rn(x1, __fmul_rn(w, g[k].y));
  }
  return make_float2(x0, x1);
}

// The dense levels as x-pairs: entry (x, y, z) holds the slots of (x, y, z)
// and (x + 1, y, z) -- a cell's two x-corners in one 16-byte shared load,
// four loads per level instead of eight (the same values, accumulated in
// the same corner order as level_features2_dense).
NIRC_D void fill_dense_levels_x2(const nirc_spec_t& sp, const DenseLevels& d,
                                 const float* __restrict__ theta, float4* dense) {
  const uint32_t T = 1u << sp.table_log2;
  for (int l = 0; l < d.n; ++l) {
    const int R = d.R[l];
    const float2* tab = reinterpret_cast<const float2*>(theta + (size_t)l * T * 2);
    for (int i = threadIdx.x; i < R * R * R; i += blockDim.x) {
      const int x = i % R, y = (i / R) % R, z = i / (R * R);
      const float2 a = __ldg(tab + hash3((uint32_t)x, (uint32_t)y, (uint32_t)z, T - 1u));
      const float2 b = x + 1 < R
                           ? __ldg(tab + hash3((uint32_t)(x + 1), (uint32_t)y, (uint32_t)z, T - 1u))
                           : make_float2(0.0f, 0.0f);
      dense[d.off[l] + i] = make_float4(a.x, a.y, b.x, b.y);
    }
  }
}

NIRC_D float2 level_features2_dense_x2(const float4* dense, int R, const LevelCell& c) {
  const int b = (c.iz * R + c.iy) * R + c.ix;
  float2 g[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // q = (dy, dz): corners 2 q (x) and 2 q + 1 (x + 1)
    const float4 v = dense[b + (q & 1) * R + (q >> 1) * R * R];
    g[2 * q] = make_float2(v.x, v.y);
    g[2 * q + 1] = make_float2(v.z, v.w);
  }
  float x0 = 0.0f, x1 = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float w = corner_weight(c, k);
    x0 = __fadd_rn(x0, __fmul_rn(w, g[k].x));
    x1 = __fadd_rn(x1, __fmul_rn(w, g[k].y));
  }
  return make_float2(x0, x1);
}

// ------------------------------------------------------ sampling frames --
// core.py:39-54 onb_s (Duff et al.), :57-65 cosine_dir_s.  Used by the render
// and collection kernels (compiled with -fmad=false).
struct Onb {
  double tx, ty, tz, bx, by, bz;
};
__device__ inline Onb onb(double nx, double ny, double nz) {
  const double s = nz >= 0.0 ? 1.0 : -1.0;
  const double a = -1.0 / (s + nz);
  const double b = nx * ny * a;
  Onb o;
  o.tx = 1.0 + s * nx * nx * a;
  o.ty = s * b;
  o.tz = -s * nx;
  o.bx = b;
  o.by = s + ny * ny * a;
  o.bz = -ny;
  return o;
}

}  // namespace nirc

// ------------------------------------------------------------- errors ----
namespace nirc {
void set_last_error(const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
}  // namespace nirc

#define NIRC_CUDA_TRY(expr)                                        \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return nirc::check_cuda(_e, #expr);     \
  } while (0)

// Stream-ordered temporary: cudaFreeAsync on every exit path of the entry
// point that allocated it (early error returns included).
// Row stride (floats) of the training kernels' per-tile MLP-gradient
// partials: the MLP block of theta padded to 16 bytes (vector reduction).
NIRC_HD int64_t part_stride(const nirc_spec_t& sp) {
  return (sp.theta_len - sp.grid_len + 3) & ~(int64_t)3;
}

struct AsyncBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  explicit AsyncBuf(cudaStream_t st) : s(st) {}
  AsyncBuf(const AsyncBuf&) = delete;
  AsyncBuf& operator=(const AsyncBuf&) = delete;
  cudaError_t alloc(size_t bytes) {
    keep_pool();
    return cudaMallocAsync(&p, bytes, s);
  }
  // the device's default pool keeps freed blocks (threshold = max) so the
  // per-call temporaries are recycled instead of returned at every sync
  static void keep_pool() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
  }
  ~AsyncBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

#define NIRC_LAUNCH_CHECK(what)                                    \
  do {                                                             \
    cudaError_t _e = cudaGetLastError();                           \
    if (_e != cudaSuccess) return nirc::check_cuda(_e, what);      \
  } while (0)
