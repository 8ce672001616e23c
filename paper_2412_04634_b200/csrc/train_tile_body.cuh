// Body of the fused training tile kernel, instantiated once per tile height
// kTR (rows per CTA; 128, 64 or 32) by train_fused.cu, which defines kTR in
// the enclosing namespace before including this file.
// Thread (r, h): row r of the CTA's rows, column slice h (columns kCols*h ..).
constexpr int kSplit = kTT / kTR;                 // threads per row
constexpr int kLD2 = kTR + 4;                     // staging row stride (FusedLayout.ld2)
constexpr int kCols = kMaxW / kSplit;             // hidden columns per thread
constexpr int kLvl = (12 + kSplit - 1) / kSplit;  // hash levels per thread
constexpr int kDX = 2 * kLvl;                     // encoded-grid gradient columns per thread
static_assert(kCols == 4 || kCols == 8 || kCols == 16, "TMEM stash widths");

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

// kCols TMEM columns of this thread's lane <-> v[kCols].  Every thread owns
// one lane of its warp's quadrant and the columns of its slice, so the
// stash needs no row <-> lane correspondence: a thread reads back only what
// it wrote.
__device__ __forceinline__ void tmem_put(uint32_t taddr, const float* v) {
  if constexpr (kCols == 4) {
    tc::tmem_st4(taddr, v);
  } else if constexpr (kCols == 8) {
    tc::tmem_st8(taddr, v);
  } else {
    tc::tmem_st16(taddr, v);
  }
}
__device__ __forceinline__ void tmem_get(uint32_t taddr, float* v) {
  if constexpr (kCols == 4) {
    tc::tmem_ld4(taddr, v);
  } else if constexpr (kCols == 8) {
    tc::tmem_ld8(taddr, v);
  } else {
    tc::tmem_ld16(taddr, v);
  }
  tc::tmem_wait_ld();
}

// kTR rows of the batch per CTA: rows tile0 * 128 + blockIdx.x * kTR + r
// (r < kTR) of the selected order idx; thread (r, h) = (tid % kTR, tid / kTR).
__global__ void __launch_bounds__(kTT, 1)
    k_train_tile(nirc_spec_t sp, FusedLayout L, const float* __restrict__ theta,
                 const float* __restrict__ wimg, nirc_records_t rec,
                 const int64_t* __restrict__ idx, int64_t B, int loss_kind, double loss_eps,
                 float* __restrict__ grad, float* __restrict__ partials,
                 double* __restrict__ loss_part, int32_t* __restrict__ flags, int64_t tile0,
                 const int32_t* __restrict__ tile_list, float* __restrict__ dx_out,
                 uint32_t* __restrict__ lvlmax) {
  extern __shared__ __align__(16) float fsm[];
  __shared__ uint32_t tmem_holder;
  __shared__ __align__(8) uint64_t wbar;
  if (flags[0] & 3) return;
  // list mode (kTR == 128): the fp16-range fix-up of k_train_tc -- the CTAs
  // loop over the API tiles tile_list[1 ..] and write those tiles' partial
  // slots (a no-op launch when the list is empty)
  if (tile_list != nullptr && (int)blockIdx.x >= tile_list[0]) return;
  const int tid = threadIdx.x;
  const int r = tid & (kTR - 1), h = tid / kTR;
  const int c0 = kCols * h;
  const int lane_base = ((tid >> 5) & 3) * 32;
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
  const int nitems = tile_list != nullptr ? tile_list[0] : (int)blockIdx.x + 1;
  for (int item = blockIdx.x; item < nitems; item += (tile_list != nullptr ? gridDim.x : nitems)) {
  int64_t slot = item, row0 = tile0 * kTileRows + (int64_t)item * kTR;
  if (tile_list != nullptr) {
    const int64_t t = tile_list[1 + item];
    slot = t - tile0;
    row0 = t * kTileRows;
  }
  const int64_t row = row0 + r;
  const bool live = row < B;
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
    loss_part[slot] = t;
  }
  // ---- backward ----------------------------------------------------------
  float* wpart = partials + slot * part_stride(sp);
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
      const float d0 = dX[2 * q], d1 = dX[2 * q + 1];
      if (dx_out != nullptr) {  // deterministic mode: rows for the ordered scatter
        dx_out[row * 24 + 2 * lvl] = d0;
        dx_out[row * 24 + 2 * lvl + 1] = d1;
        atomicMax(lvlmax + lvl, max(__float_as_uint(fabsf(d0)), __float_as_uint(fabsf(d1))));
        continue;
      }
      const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
      float* gl = grad + (size_t)lvl * T * 2;
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
  __syncthreads();  // the next item reuses the staging arrays
  }
  tc::fence_before();
  __syncthreads();
  if (tid < 32) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_holder, (uint32_t)L.tmem_cols);
  }
}

