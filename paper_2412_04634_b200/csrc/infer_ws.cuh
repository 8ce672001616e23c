// Warp-specialised fused inference of the two-level frame (included by
// render.cu after the row / combine helpers).  Same work and the same
// results layout as k_infer_tc<F16x2> -- cache_lc_s + the residual
// (src/kernels.py:424-448, :593-601) for every deferred cache vertex -- but
// the per-tile phases run on different warps so they overlap:
//
//   producer warpgroups (NP x 128 threads)          chain groups (4 x 128 threads)
//   ------------------------------------           --------------------------------
//   records of tile t -> SMEM                      group g = t % 4 owns TMEM cols
//   shared surface encoding (vertex x level)       [128g, 128g+128): D | A_hi | A_lo
//   per row: Lambert direction + SH + aux          layer 0: SS MMAs from the A slot
//     -> layer-0 A operand (fp16 hi/lo, SMEM       layers 1..: TS MMAs, epilogue =
//        slot g) + per-row weights f, ci/pdf         ReLU + hi/lo split into TMEM
//     -> per-vertex combine data (T, T', slot)     combine: n(w) f cos/pdf per row,
//   arrive full[g]                                   k-ordered per-vertex sum, result
//
// So while a group runs the MMA -> epilogue chain of tile t, a producer builds
// tile t+4's rows, and the tensor pipe sees four chains at once.  Per group:
//   full[g]     producer -> chain: A slot g + meta buffer (n & 1) written
//   aempty[g]   tcgen05.commit after layer 0: A slot g may be overwritten
//   mempty[g][b] chain -> producer: meta buffer b's combine is done
//   mma[g]      tcgen05.commit of each layer (the chain's own wait)
// The epilogue split is x = hi + lo with hi = x truncated to fp16 precision
// (mask of the low 13 mantissa bits: exact in fp16 for |x| in [2^-14, 65504])
// and lo = fp16_rn(x - hi); ReLU rides in the conversion (cvt.relu on both
// parts: x < 0 gives two negative parts, both clamp to 0).  ~2^-21 relative
// per operand, the fp32 class of the reference (tests hold it to rtol 1e-4).
#pragma once
// (included inside namespace nirc)

namespace ws {

constexpr int kChainGroups = 4;   // one TMEM slot each
constexpr int kSlots = 4;
// register split per thread (setmaxnreg; 0 = none).  The CTA keeps the
// registers it was launched with (96 x 640 for NP = 1, 80 x 768 for NP = 2):
// what the chain warps release is all the producers may take, or
// setmaxnreg.inc blocks forever (checked on the host).  NP must divide 4 (a
// slot's tiles come from one producer, so its barrier phases stay in order).
// NP = 2 measured (1080p inference): 72 / 96 2.30 ms, 64 / 112 2.33 ms,
// 80 / 80 2.61 ms (the producers spill).
template <int NP> constexpr int kChainRegs = NP == 1 ? 88 : (NP == 2 ? 72 : 0);
template <int NP> constexpr int kProdRegs = NP == 1 ? 128 : (NP == 2 ? 96 : 0);

// Per-vertex data the combine needs (vertex_result), written by the producer.
struct VMeta {
  double T[3], Tp[3];
  double inv;  // 1 / ncq (the reference's 1.0 / N_c, computed once by the producer)
  int64_t slot;
  int32_t ncq, has_res, nrc, pad;
};

struct Layout {
  uint32_t w_off, bias_off, a_off, meta_off, meta_bytes, prod_off, prod_bytes, bar_off,
      holder_off, total;
  float shk[28];  // the SH constants sh4_f32 reads, as fp32 kernel-parameter operands
};

// meta buffer: 128 rows x {f.x, f.y, f.z, ci/pdf} doubles (the row's
// contribution overwrites them after the chain), S VMeta, 4 producer flags
__host__ __device__ inline uint32_t meta_bytes_for(int S) {
  return (uint32_t)(128 * 32 + S * (int)sizeof(VMeta) + 16 + 15) & ~15u;
}
// Per-vertex data of the producer: the Lambert frame, f = albedo / pi and the
// layer-0 operand chunks shared by the vertex's rows.
struct VFrame {
  LambertFrame F;
  int lambert, unsafe;
  double f[3];
};
// producer staging: records (double-buffered: the next tile's are in flight),
// features, per-vertex chunks (hi: feat 0-2, aux; lo: same), frames
__host__ __device__ inline uint32_t prod_bytes_for(int S) {
  const uint32_t cv = (uint32_t)(2 * S * (int)sizeof(CacheVertex) + 15) & ~15u;
  return cv + (uint32_t)(S * 24 * 4 + 15) / 16 * 16 + (uint32_t)S * 128u +
         ((uint32_t)(S * (int)sizeof(VFrame) + 15) & ~15u) + 64 * 4;
}
constexpr uint32_t kASlotBytes = 2u * 128u * 48u * 2u;  // hi + lo, K = 48 fp16

__host__ __device__ inline Layout layout(const tc::TcNet& net, int S, int NP) {
  Layout L;
  L.w_off = 0;
  // bias operands: a 128 x 16 fp16 "ones" tile (columns 0, 1 = 1.0) and per
  // layer an N x 16 tile holding the bias hi / lo parts in columns 0 / 1, so
  // one SS MMA (K = 16, accumulate off) writes D = b_hi + b_lo
  L.bias_off = (net.wbytes + 1023u) & ~1023u;
  L.a_off = (L.bias_off + 4096u + (uint32_t)net.nl * 2048u + 1023u) & ~1023u;
  L.meta_off = L.a_off + kSlots * kASlotBytes;
  L.meta_bytes = meta_bytes_for(S);
  L.prod_off = L.meta_off + kSlots * 2 * L.meta_bytes;
  L.prod_bytes = prod_bytes_for(S);
  L.bar_off = (L.prod_off + NP * L.prod_bytes + 7u) & ~7u;
  L.holder_off = L.bar_off + 8 * (1 + 5 * kSlots);
  L.total = L.holder_off + 16 + 4 * kSlots + 4 * tc::kMaxTcLayers;
  return L;
}

__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

// 16 fp32 accumulator columns -> 8 packed fp16x2 columns each of hi and lo,
// ReLU applied: hi = fp16_rz(relu(x)) (the truncation: hi <= x), lo =
// fp16_rn(relu(x - hi)) with x - hi formed exactly by a mixed f16/f32 FMA
// (4 instructions per pair); gmax accumulates max(x) for the fp16 range guard
// (NaN sticks).
template <bool kGuard>
__device__ __forceinline__ void relu_split16(const float* h, uint32_t* hi, uint32_t* lo,
                                             float& gmax) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float x0 = h[2 * c], x1 = h[2 * c + 1];
    asm("cvt.rz.relu.f16x2.f32 %0, %1, %2;" : "=r"(hi[c]) : "f"(x1), "f"(x0));
    float l0, l1;
    asm("{\n\t.reg .b16 h0, h1, m1;\n\t"
        "mov.b32 {h0, h1}, %2;\n\t"
        "mov.b16 m1, 0xBC00;\n\t"
        "fma.rn.f32.f16 %0, h0, m1, %3;\n\t"
        "fma.rn.f32.f16 %1, h1, m1, %4;\n\t}"
        : "=f"(l0), "=f"(l1)
        : "r"(hi[c]), "f"(x0), "f"(x1));
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(lo[c]) : "f"(l1), "f"(l0));
    if constexpr (kGuard)
      asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(gmax) : "f"(gmax), "f"(x0), "f"(x1));
  }
}

// 2 layer-0 inputs (any sign) -> fp16x2 hi (the truncation) and lo =
// fp16_rn(x - hi), as split8 below for one word.
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rz.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(x1), "f"(x0));
  float l0, l1;
  asm("{\n\t.reg .b16 h0, h1, m1;\n\t"
      "mov.b32 {h0, h1}, %2;\n\t"
      "mov.b16 m1, 0xBC00;\n\t"
      "fma.rn.f32.f16 %0, h0, m1, %3;\n\t"
      "fma.rn.f32.f16 %1, h1, m1, %4;\n\t}"
      : "=f"(l0), "=f"(l1)
      : "r"(hi), "f"(x0), "f"(x1));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(l1), "f"(l0));
}

// 8 layer-0 inputs (any sign) -> one 16-byte chunk each of fp16 hi (the
// truncation) and lo = fp16_rn(x - hi), as relu_split16 without the ReLU.
__device__ __forceinline__ void split8(const float* x, uint4& hi4, uint4& lo4) {
  uint32_t hi[4], lo[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float x0 = x[2 * c], x1 = x[2 * c + 1];
    asm("cvt.rz.f16x2.f32 %0, %1, %2;" : "=r"(hi[c]) : "f"(x1), "f"(x0));
    float l0, l1;
    asm("{\n\t.reg .b16 h0, h1, m1;\n\t"
        "mov.b32 {h0, h1}, %2;\n\t"
        "mov.b16 m1, 0xBC00;\n\t"
        "fma.rn.f32.f16 %0, h0, m1, %3;\n\t"
        "fma.rn.f32.f16 %1, h1, m1, %4;\n\t}"
        : "=f"(l0), "=f"(l1)
        : "r"(hi[c]), "f"(x0), "f"(x1));
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo[c]) : "f"(l1), "f"(l0));
  }
  hi4 = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  lo4 = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

__device__ __forceinline__ void sts128(uint32_t addr, const uint4& v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// A layer with A in TMEM (TS): K = 48 (layer 0) or 64, N = 64 (hidden) or
// 16 (output); accumulates on the bias the layer's tcgen05.cp put in D.
template <int K, int N>
__device__ __forceinline__ void issue_layer_ts(uint32_t w_l, uint32_t a_hi, uint32_t a_lo,
                                               uint32_t tmem_d) {
  constexpr uint32_t idesc = tc::PrecF16x2::kIdescFmt | ((uint32_t)(N >> 3) << 17) |
                             ((uint32_t)(tc::kTileRows >> 4) << 24);
  constexpr uint32_t w_lbo = (uint32_t)N * 16;
  const uint32_t w_lo = w_l + (uint32_t)(N * K * 2);
#pragma unroll
  for (int term = 0; term < 3; ++term) {  // hi*lo, lo*hi, then hi*hi
    const uint32_t A = term == 1 ? a_lo : a_hi;
    const uint32_t B = term == 0 ? w_lo : w_l;
#pragma unroll
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint64_t bd = tc::sdesc(B + kk * 2 * w_lbo, w_lbo, 128);
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "setp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
          "r"(A + kk * 8), "l"(bd), "n"(idesc), "n"(1));
    }
  }
}

// Layer 0 from the SMEM A slot (SS), accumulating on the bias in D.
__device__ __forceinline__ void issue_layer0_ss(uint32_t w_l0, uint32_t a_hi, uint32_t a_lo,
                                                uint32_t tmem_d) {
  constexpr int K = 48, N = 64;
  constexpr uint32_t idesc = tc::PrecF16x2::kIdescFmt | ((uint32_t)(N >> 3) << 17) |
                             ((uint32_t)(tc::kTileRows >> 4) << 24);
  constexpr uint32_t a_lbo = tc::kTileRows * 16, w_lbo = (uint32_t)N * 16;
  const uint32_t w_lo = w_l0 + (uint32_t)(N * K * 2);
#pragma unroll
  for (int term = 0; term < 3; ++term) {
    const uint32_t A = term == 1 ? a_lo : a_hi;
    const uint32_t B = term == 0 ? w_lo : w_l0;
#pragma unroll
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint64_t ad = tc::sdesc(A + kk * 2 * a_lbo, a_lbo, 128);
      const uint64_t bd = tc::sdesc(B + kk * 2 * w_lbo, w_lbo, 128);
      tc::mma_issue<tc::PrecF16x2>(tmem_d, ad, bd, idesc, 1u);
    }
  }
}

// D <- the layer's bias in every lane: one SS MMA, ones (128 x 16) x bias
// tile (N x 16: hi, lo in columns 0, 1), accumulate off.
template <int N>
__device__ __forceinline__ void mma_bias(uint32_t tmem_d, uint32_t ones, uint32_t btile) {
  constexpr uint32_t idesc = tc::PrecF16x2::kIdescFmt | ((uint32_t)(N >> 3) << 17) |
                             ((uint32_t)(tc::kTileRows >> 4) << 24);
  const uint64_t ad = tc::sdesc(ones, tc::kTileRows * 16, 128);
  const uint64_t bd = tc::sdesc(btile, (uint32_t)N * 16, 128);
  tc::mma_issue<tc::PrecF16x2>(tmem_d, ad, bd, idesc, 0u);
}
}  // namespace ws

// Waits for an mbarrier phase, sleeping between polls (producer side: not
// latency critical, and the chain warps need the issue slots).
__device__ __forceinline__ void ws_wait_sleep(uint32_t mbar, uint32_t parity) {
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(mbar), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(200);
  }
}

// Four chain groups, one TMEM slot each.  (Measured alternative, not kept:
// two groups alternating between two slots each, "ping-pong", 5.60 vs 5.31
// ms per 1080p render.)
template <int NP, bool kProbe, int NG = 4>
__global__ void __launch_bounds__((NG + NP) * 128, 1)
    k_infer_ws(nirc_spec_t sp, tc::TcNet net, ws::Layout L, const float* __restrict__ theta,
               const uint8_t* __restrict__ wimg, const float* __restrict__ bias_g, InferArgs a) {
  constexpr int NS = ws::kSlots;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t s0 = tc::smem_u32(smem);
  const int tid = threadIdx.x;
  const int R = a.rows_per_vertex, S = a.verts_per_tile;
  const int64_t nverts = (int64_t)a.counters[0];
  const int64_t ntiles = (nverts + S - 1) / S;
  // barriers: [0] weights, then per slot s: full, aempty, mempty0, mempty1, mma
  const uint32_t bar0 = s0 + L.bar_off + 8;
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + L.holder_off);
  int* s_unsafe = reinterpret_cast<int*>(smem + L.holder_off + 16);
  if (tid == 0) {
    // mempty (per slot entries 2, 3) counts every chain thread of the slot's group
    for (int i = 0; i < 1 + 5 * NS; ++i)
      tc::mbar_init(s0 + L.bar_off + 8 * i, (i >= 1 && ((i - 1) % 5 == 2 || (i - 1) % 5 == 3)) ? 128 : 1);
    tc::mbar_init_fence();
  }
  if (tid < NS) s_unsafe[tid] = 0;
  if ((tid >> 5) == 0) tc::tmem_alloc(tc::smem_u32(holder), 512);
  // bias operands (K-major canonical fp16: element (r, k) at (k / 8) * rows * 16
  // + (r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2): ones tile at bias_off,
  // layer l's bias tile at bias_off + 4096 + 2048 l
  {
    uint16_t* s_ones = reinterpret_cast<uint16_t*>(smem + L.bias_off);
    for (int i = tid; i < 128 * 16; i += blockDim.x) {
      const int r = i / 16, k = i % 16;
      s_ones[((k / 8) * 128 * 16 + (r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) / 2] =
          k < 2 ? (uint16_t)0x3c00u : (uint16_t)0u;
    }
    for (int i = tid; i < net.nl * 64 * 16; i += blockDim.x) {
      const int l = i / 1024, r = (i / 16) % 64, k = i % 16;
      const int N = net.N[l];
      if (r >= N) continue;
      uint16_t* bt = reinterpret_cast<uint16_t*>(smem + L.bias_off + 4096 + 2048 * l);
      const float b = bias_g[l * 64 + r];
      const __half hi = __float2half_rn(b);
      const __half lo = __float2half_rn(b - __half2float(hi));
      const __half v = k == 0 ? hi : (k == 1 ? lo : __float2half_rn(0.0f));
      bt[((k / 8) * N * 16 + (r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) / 2] =
          *reinterpret_cast<const uint16_t*>(&v);
    }
  }
  tc::fence_proxy_async();
  uint32_t* s_woff = reinterpret_cast<uint32_t*>(smem + L.holder_off + 16 + 4 * ws::kSlots);
  if (tid < tc::kMaxTcLayers) s_woff[tid] = tid < net.nl ? net.woff[tid] : 0u;
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *holder;
  if (tid == 0) {
    const uint32_t wbar = s0 + L.bar_off;
    tc::mbar_expect_tx(wbar, net.wbytes);
    for (uint32_t off = 0; off < net.wbytes; off += 32768u) {
      const uint32_t sz = net.wbytes - off < 32768u ? net.wbytes - off : 32768u;
      tc::bulk_g2s(s0 + L.w_off + off, wimg + off, sz, wbar);
    }
  }
  const int role = tid >> 7;  // 0..NG-1 chain groups, NG.. producers
  const int tg = tid & 127;
  const int warp = tg >> 5;

  if (role >= NG) {
    // ------------------------------------------------------- producer ---
    if constexpr (NG == 4 && ws::kProdRegs<NP> > 0)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(ws::kProdRegs<NP>));
    const int p = role - NG;
    uint8_t* pbase = smem + L.prod_off + p * L.prod_bytes;
    const uint32_t cv_bytes = (uint32_t)(2 * S * (int)sizeof(CacheVertex) + 15) & ~15u;
    CacheVertex* s_cvb = reinterpret_cast<CacheVertex*>(pbase);
    // (the S x 24 floats after the records are unused since the features
    // are split into s_vx as they are computed)
    uint4* s_vx = reinterpret_cast<uint4*>(pbase + cv_bytes + (uint32_t)(S * 24 * 4 + 15) / 16 * 16);
    ws::VFrame* s_vf = reinterpret_cast<ws::VFrame*>(reinterpret_cast<uint8_t*>(s_vx) + S * 128);
    if (tg < S) s_vf[tg].unsafe = 0;  // (ordered by the loop's first barrier)
    const uint32_t pbar = 1 + NG + p;
    const uint32_t T = 1u << sp.table_log2;
    const bool pairs = (reinterpret_cast<uintptr_t>(theta) & 15u) == 0;  // 16-byte slot pairs
    const int j = tg / R, k = tg % R;
    // asynchronous copy of a tile's records (8-byte cp.async per word)
    auto fetch = [&](int64_t i, int buf) {
      const int64_t tile = (int64_t)blockIdx.x + i * gridDim.x;
      if (tile < ntiles) {
        const int64_t v0 = tile * S;
        const int nv = (int)((nverts - v0) < S ? (nverts - v0) : S);
        const double* src = reinterpret_cast<const double*>(a.cv + v0);
        const uint32_t dst = tc::smem_u32(s_cvb + buf * S);
        const int words = nv * (int)(sizeof(CacheVertex) / 8);
        for (int w = tg; w < words; w += 128)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8 * w),
                       "l"(src + w)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    fetch(p, 0);
    int it = 0;
    for (int64_t i = p; ; i += NP, ++it) {
      const int64_t tile = (int64_t)blockIdx.x + i * gridDim.x;
      if (tile >= ntiles) break;
      const int slot = (int)(i % NS);
      const int64_t n = i / NS;  // the slot's tile number
      const int64_t v0 = tile * S;
      const int nv = (int)((nverts - v0) < S ? (nverts - v0) : S);
      CacheVertex* s_cv = s_cvb + (it & 1) * S;
      long long* pb = (kProbe && blockIdx.x == 0 && tg == 0 && p == 0 && it < 32)
                          ? a.dbg + 2048 + it * 8 : nullptr;
      if (kProbe && pb) pb[0] = clock64();
      if (a.ablate == 1) {  // timing experiment: only the handshake
        const int b = (int)(n & 1);
        if (warp == 0) {
          if (n >= 1) ws_wait_sleep(bar0 + 8 * (5 * slot + 1), (uint32_t)((n - 1) & 1));
          if (n >= 2) ws_wait_sleep(bar0 + 8 * (5 * slot + 2 + b), (uint32_t)(((n >> 1) - 1) & 1));
        }
        tc::named_bar_sync(pbar, 128);
        if (tg == 0) ws::mbar_arrive(bar0 + 8 * (5 * slot));
        continue;
      }
      // the next tile's records load while this one is built (its buffer's
      // last reader was the tile before this one, ordered by its barriers)
      fetch(i + NP, (it + 1) & 1);
      if (kProbe && pb) pb[7] = clock64();
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      // the slot's meta buffer b is free once the combine of its tile n-2
      // is done (checked here: the per-vertex meta is written below)
      const int b = (int)(n & 1);
      if (warp == 0 && n >= 2)
        ws_wait_sleep(bar0 + 8 * (5 * slot + 2 + b), (uint32_t)(((n >> 1) - 1) & 1));
      tc::named_bar_sync(pbar, 128);
      if (kProbe && pb) pb[1] = clock64();
      uint8_t* meta = smem + L.meta_off + (slot * 2 + b) * L.meta_bytes;
      ws::VMeta* vm = reinterpret_cast<ws::VMeta*>(meta + 128 * 32);
      // one pass: the shared surface encoding, one thread per (vertex, level),
      // each splitting its two features straight into the vertex's fp16
      // hi / lo operand chunks (features 8 c .. 8 c + 7 in chunk c); then,
      // from the next warp boundary on, the per-vertex items (aux chunk,
      // Lambert frame, combine meta), which need no encoding
      {
        const int ne = nv * 12;
        const int b2 = (ne + 31) & ~31;
        uint32_t* s_vw = reinterpret_cast<uint32_t*>(s_vx);
        for (int item = tg; item < b2 + 3 * nv; item += 128) {
          if (item < ne) {
            const int jj = item / 12, lvl = item % 12;
            const CacheVertex& r = s_cv[jj];
            const float ux = norm_coord(r.pos[0], sp.bb_min[0], sp.bb_inv[0]);
            const float uy = norm_coord(r.pos[1], sp.bb_min[1], sp.bb_inv[1]);
            const float uz = norm_coord(r.pos[2], sp.bb_min[2], sp.bb_inv[2]);
            const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
            const float2 f = pairs ? level_features2_pairs(theta + (size_t)lvl * T * 2, c, T - 1u)
                                   : level_features2(theta + (size_t)lvl * T * 2, c, T - 1u);
            uint32_t hw, lw;
            ws::split2(f.x, f.y, hw, lw);
            const int wi = (jj * 8 + (lvl >> 2)) * 4 + (lvl & 3);
            s_vw[wi] = hw;
            s_vw[wi + 16] = lw;
            if (!(fabsf(f.x) < tc::kF16Max) || !(fabsf(f.y) < tc::kF16Max))
              atomicOr(&s_vf[jj].unsafe, 1);
          } else if (item >= b2) {
            const int q = item - b2, jj = q % nv, what = q / nv;
            const CacheVertex& r = s_cv[jj];
            if (what == 0) {  // aux chunk: (n + 1) / 2, albedo, roughness
              float v[8];
              v[0] = (float)((r.ns[0] + 1.0) * 0.5);
              v[1] = (float)((r.ns[1] + 1.0) * 0.5);
              v[2] = (float)((r.ns[2] + 1.0) * 0.5);
              v[3] = (float)r.alb[0];
              v[4] = (float)r.alb[1];
              v[5] = (float)r.alb[2];
              v[6] = (float)r.rough;
              v[7] = 0.0f;
              uint4 hi, lo;
              ws::split8(v, hi, lo);
              s_vx[jj * 8 + 3] = hi;
              s_vx[jj * 8 + 7] = lo;
              if (tc::f16_unsafe(v, 8)) atomicOr(&s_vf[jj].unsafe, 1);
            } else if (what == 1) {
              ws::VFrame& vf = s_vf[jj];
              vf.F = lambert_frame(r);
              vf.lambert = r.mkind == pt::MAT_LAMBERT;
              vf.f[0] = r.alb[0] * pt::INV_PI;
              vf.f[1] = r.alb[1] * pt::INV_PI;
              vf.f[2] = r.alb[2] * pt::INV_PI;
            } else {
              ws::VMeta m;
              m.T[0] = r.T[0];
              m.T[1] = r.T[1];
              m.T[2] = r.T[2];
              m.Tp[0] = r.Tp[0];
              m.Tp[1] = r.Tp[1];
              m.Tp[2] = r.Tp[2];
              m.slot = r.slot;
              m.ncq = r.ncq;
              m.has_res = r.has_res;
              m.nrc = r.nrc;
              m.pad = 0;
              m.inv = r.ncq > 0 ? 1.0 / r.ncq : 0.0;
              vm[jj] = m;
            }
          }
        }
      }
      tc::named_bar_sync(pbar, 128);
      if (kProbe && pb) {
        pb[2] = clock64();
        pb[5] = pb[2];
      }
      // per row: the direction, its SH block and the combine weights
      int kind = 0;
      double sw = 0.0, f0 = 0.0, f1 = 0.0, f2 = 0.0;
      float w[3] = {0.0f, 0.0f, 1.0f};
      if (j < nv) {
        const CacheVertex& r = s_cv[j];
        const ws::VFrame& vf = s_vf[j];
        if (vf.lambert && k < r.ncq) {
          lambert_row(vf.F, r.key, r.base, k, w, &sw, &kind);
          if (kind == 0) {
            w[0] = 0.0f;
            w[1] = 0.0f;
            w[2] = 1.0f;
          }
          f0 = vf.f[0];
          f1 = vf.f[1];
          f2 = vf.f[2];
        } else {  // other lobes (f64 sampler), the residual and NRC rows
          const RowDir rd = row_direction(r, k);
          kind = rd.kind;
          w[0] = (float)rd.wi.x;
          w[1] = (float)rd.wi.y;
          w[2] = (float)rd.wi.z;
          sw = rd.s;
          f0 = rd.f.x;
          f1 = rd.f.y;
          f2 = rd.f.z;
        }
      }
      float sh[16];
      sh4_f32(w[0], w[1], w[2], L.shk, sh);
      uint4 shi0, slo0, shi1, slo1;
      ws::split8(sh, shi0, slo0);
      ws::split8(sh + 8, shi1, slo1);
      const bool unsafe = kind != 0 && s_vf[j < nv ? j : 0].unsafe != 0;
      if (kProbe && pb) pb[6] = clock64();
      // every warp observes the slot's A image free (layer 0 of its previous
      // tile complete) itself: no barrier needed before the stores
      if (n >= 1) ws_wait_sleep(bar0 + 8 * (5 * slot + 1), (uint32_t)((n - 1) & 1));
      if (kProbe && pb) pb[3] = clock64();
      // layer-0 row: chunks 0-2 features, 3-4 SH, 5 aux (K-major, 16-byte chunks)
      {
        const uint32_t a_hi = s0 + L.a_off + slot * ws::kASlotBytes;
        const uint32_t a_lo = a_hi + ws::kASlotBytes / 2;
        const uint32_t ro = (uint32_t)((tg >> 3) * 128 + (tg & 7) * 16);
        const int jv = j < nv ? j : 0;
        const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
        const bool live = j < nv;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ws::sts128(a_hi + c * 2048 + ro, live ? s_vx[jv * 8 + c] : z4);
          ws::sts128(a_lo + c * 2048 + ro, live ? s_vx[jv * 8 + 4 + c] : z4);
        }
        ws::sts128(a_hi + 3 * 2048 + ro, shi0);
        ws::sts128(a_lo + 3 * 2048 + ro, slo0);
        ws::sts128(a_hi + 4 * 2048 + ro, shi1);
        ws::sts128(a_lo + 4 * 2048 + ro, slo1);
        ws::sts128(a_hi + 5 * 2048 + ro, live ? s_vx[jv * 8 + 3] : z4);
        ws::sts128(a_lo + 5 * 2048 + ro, live ? s_vx[jv * 8 + 7] : z4);
      }
      double* mrow = reinterpret_cast<double*>(meta) + 4 * tg;
      if (kind == 1) {
        mrow[0] = f0;
        mrow[1] = f1;
        mrow[2] = f2;
        mrow[3] = sw;
      } else {  // residual / NRC rows: the prediction itself; invalid rows: 0
        const double v = kind >= 2 ? 1.0 : 0.0;
        mrow[0] = v;
        mrow[1] = v;
        mrow[2] = v;
        mrow[3] = kind >= 2 ? -1.0 : 0.0;  // < 0: unit weight, no ci/pdf factor
      }
      int* pflag = reinterpret_cast<int*>(meta + 128 * 32 + S * sizeof(ws::VMeta));
      const bool wu = __any_sync(0xffffffffu, unsafe);
      if ((tg & 31) == 0) pflag[warp] = wu ? 1 : 0;
      tc::fence_proxy_async();
      // the vertex flags are reset for the next tile after every row read them
      tc::named_bar_sync(pbar, 128);
      if (tg < S) s_vf[tg].unsafe = 0;
      if (tg == 0) ws::mbar_arrive(bar0 + 8 * (5 * slot));
      if (kProbe && pb) pb[4] = clock64();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    // ----------------------------------------------------------- chain ---
    if constexpr (NG == 4 && ws::kChainRegs<NP> > 0)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(ws::kChainRegs<NP>));
    {
    const int g = role;  // = the group's TMEM slot
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const uint32_t tmem_d = tmem_base + g * tc::kTsColsPerGroup;
    const uint32_t t_row = tmem_d + lane_off;  // this thread's lane of D
    const uint32_t a_hi = s0 + L.a_off + g * ws::kASlotBytes;
    const uint32_t w_base = s0 + L.w_off;
    const uint32_t b_img = s0 + L.bias_off;
    const uint32_t full = bar0 + 8 * (5 * g), mbar = full + 8 * 4;
    const uint32_t gbar = 1 + g;
    const bool all_unsafe = *a.w_unsafe != 0;
    const int nl = net.nl;
    uint32_t phase = 0;
    if (warp == 0) tc::mbar_wait(s0 + L.bar_off, 0);  // weights landed (warp 0 issues)
    int it = 0;
    // starts local tile i: layer 0 accumulates on its bias (D is free: the
    // previous tile's outputs were read); false when the CTA has no tile i
    auto start = [&](int64_t i) -> bool {
      const int64_t tile = (int64_t)blockIdx.x + i * gridDim.x;
      if (tile >= ntiles) return false;
      const int64_t n = i / NG;
      // the group's reads of D (the previous tile's outputs) are complete
      // before the bias MMA overwrites it
      tc::fence_before();
      if (warp == 0) tc::mbar_wait(full, (uint32_t)(n & 1));
      tc::named_bar_sync(gbar, 128);
      if (warp == 0) {
        tc::fence_after();
        if (tc::elect_one()) {
          long long* tl = (kProbe && blockIdx.x == 0 && n < 32) ? a.dbg + 4096 + g * 512 + n * 16
                                                               : nullptr;
          if (kProbe && tl) tl[0] = clock64();
          ws::mma_bias<64>(tmem_d, b_img, b_img + 4096);
          ws::issue_layer0_ss(w_base + s_woff[0], a_hi, a_hi + ws::kASlotBytes / 2, tmem_d);
          tc::mma_commit(mbar);
          tc::mma_commit(full + 8);  // aempty: the A slot is free once layer 0 completes
          if (kProbe && tl) tl[1] = clock64();
        }
        __syncwarp();
      }
      return true;
    };
    if (a.ablate == 2) {  // timing experiment: only the handshake
      for (int64_t i = g; ; i += NG) {
        const int64_t tile = (int64_t)blockIdx.x + i * gridDim.x;
        if (tile >= ntiles) break;
        const int64_t n = i / NG;
        if (warp == 0) tc::mbar_wait(full, (uint32_t)(n & 1));
        tc::named_bar_sync(gbar, 128);
        if (tg == 0) ws::mbar_arrive(full + 8);
        ws::mbar_arrive(full + 8 * (2 + (int)(n & 1)));
      }
    }
    bool have = a.ablate == 2 ? false : start(g);
    for (int64_t i = g; have; i += NG, ++it) {
      const int64_t tile = (int64_t)blockIdx.x + i * gridDim.x;
      const int64_t n = i / NG;
      const int b = (int)(n & 1);
      long long* pb = (kProbe && blockIdx.x == 0 && tg == 0 && g == 0 && it < 32)
                          ? a.dbg + it * 16 : nullptr;
      if (kProbe && pb) pb[0] = clock64();
      float gmax = 0.0f;
      float y[4];
      for (int l = 0; l < nl; ++l) {
        // one warp observes the layer's completion, the barrier releases the group
        if (warp == 0) tc::mbar_wait(mbar, phase);
        phase ^= 1u;
        long long* tl = (kProbe && blockIdx.x == 0 && n < 32) ? a.dbg + 4096 + g * 512 + n * 16
                                                             : nullptr;
        if (kProbe && tl && tg == 0) tl[2 + 3 * l] = clock64();
        tc::named_bar_sync(gbar, 128);
        tc::fence_after();
        if (kProbe && pb) pb[2 + l] = clock64();
        if (l < nl - 1) {
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float h[32];
            tc::tmem_ld32(t_row + half * 32, h);
            tc::tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              uint32_t hh[8], ll[8];
              ws::relu_split16<true>(h + 16 * c, hh, ll, gmax);
              tc::tmem_st8u(t_row + 64 + half * 16 + c * 8, hh);
              tc::tmem_st8u(t_row + 96 + half * 16 + c * 8, ll);
            }
          }
          if (kProbe && pb && l == 1) pb[9] = clock64();
          tc::tmem_wait_st();
          tc::fence_before();
          if (kProbe && pb && l == 1) pb[10] = clock64();
          tc::named_bar_sync(gbar, 128);
          if (kProbe && pb && l == 1) pb[11] = clock64();
          if (warp == 0) {
            tc::fence_after();
            if (tc::elect_one()) {
              if (kProbe && tl) tl[3 + 3 * l] = clock64();
              const uint32_t wl = w_base + s_woff[l + 1];
              const uint32_t bl = b_img + 4096 + 2048u * (uint32_t)(l + 1);
              if (l + 1 == nl - 1) {
                ws::mma_bias<16>(tmem_d, b_img, bl);
                ws::issue_layer_ts<64, 16>(wl, tmem_d + 64, tmem_d + 96, tmem_d);
              } else {
                ws::mma_bias<64>(tmem_d, b_img, bl);
                ws::issue_layer_ts<64, 64>(wl, tmem_d + 64, tmem_d + 96, tmem_d);
              }
              tc::mma_commit(mbar);
              if (kProbe && tl) tl[4 + 3 * l] = clock64();
            }
            __syncwarp();
          }
          if (kProbe && pb && l == 1) pb[12] = clock64();
        } else {
          float o[4];
          tc::tmem_ld4(t_row, o);
          tc::tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float z = o[c];
            y[c] = net.out_act == 0 ? (z > 0.0f ? z : 0.0f) : 1.0f / (1.0f + expf(-z));
          }
        }
      }
      // MLMC combine: the row's contribution replaces its weights in the meta row
      uint8_t* meta = smem + L.meta_off + (g * 2 + b) * L.meta_bytes;
      double* mrow = reinterpret_cast<double*>(meta) + 4 * tg;
      const double sw = mrow[3];
      double c0 = 0.0, c1 = 0.0, c2 = 0.0;
      if (sw > 0.0) {
        c0 = (double)y[0] * mrow[0] * sw;
        c1 = (double)y[1] * mrow[1] * sw;
        c2 = (double)y[2] * mrow[2] * sw;
      } else if (sw < 0.0) {
        c0 = (double)y[0];
        c1 = (double)y[1];
        c2 = (double)y[2];
      }
      mrow[0] = c0;
      mrow[1] = c1;
      mrow[2] = c2;
      const bool unsafe = sw != 0.0 && (all_unsafe || !(gmax < tc::kF16Max));
      if (__any_sync(0xffffffffu, unsafe) && (tg & 31) == 0) atomicOr(&s_unsafe[g], 1);
      // the next tile's layer 0 goes to the tensor pipe before this tile's
      // per-vertex combine (its barrier also publishes the contributions)
      have = start(i + NG);
      if (!have) tc::named_bar_sync(gbar, 128);
      if (kProbe && pb) pb[7] = clock64();
      const int64_t v0 = tile * S;
      const int nv = (int)((nverts - v0) < S ? (nverts - v0) : S);
      const ws::VMeta* vm = reinterpret_cast<const ws::VMeta*>(meta + 128 * 32);
      // (vertex, channel) items on warps 1-3 (warp 0 goes on to the next
      // layer-0 completion): the k-ordered f64 sum of cache_lc_s per channel
      const double* md = reinterpret_cast<const double*>(meta);
      for (int ct = tg - 32; ct >= 0 && ct < 3 * nv && a.ablate == 0; ct += 96) {
        const int v = ct / 3, ch = ct - 3 * v;
        const ws::VMeta& r = vm[v];
        const double* rows = md + 4 * (v * R) + ch;
        double o;
        if (r.nrc) {
          o = r.T[ch] * rows[0];
        } else {
          double acc = 0.0;
          for (int c = 0; c < r.ncq; ++c) acc += rows[4 * c];
          o = r.T[ch] * (acc * r.inv);
          if (r.has_res) o -= r.Tp[ch] * rows[4 * r.ncq];
        }
        a.result[3 * r.slot + ch] = o;
      }
      if (tg == 0 && a.ablate == 0) {
        const int* pflag = reinterpret_cast<const int*>(meta + 128 * 32 + S * sizeof(ws::VMeta));
        if (s_unsafe[g] | pflag[0] | pflag[1] | pflag[2] | pflag[3]) {
          s_unsafe[g] = 0;
          a.fix[1 + atomicAdd(a.fix, 1)] = (int32_t)tile;
        }
      }
      ws::mbar_arrive(full + 8 * (2 + b));  // mempty[b]: every chain thread is done with it
      if (kProbe && pb) pb[8] = clock64();
    }
  }
  }
  tc::fence_before();
  __syncthreads();
  if ((tid >> 5) == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_base, 512);
  }
}
