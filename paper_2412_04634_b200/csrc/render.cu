// Two-level (MLMC) frame estimator and training-record collection on
// sm_100a.  The fp64 path walks follow the reference's operation order (FMA
// contraction allowed, as numba fastmath allows it; build.py NIRC_RENDER_FMAD).
//
// Frame pipeline (nirc_render, one stream, no host sync):
//   K5  k_trace       one thread per (pixel, sample): fp64 path tracer
//                     (trace_sample MODE_PT/MODE_TL, kernels.py:451-608).
//                     The network output never steers the walk, so the
//                     two-level terms are DEFERRED: each cache vertex emits a
//                     record (surface, T, key/base, T', w_cont) and the walk
//                     continues exactly like plain PT.
//   K1+K2+K4  k_infer_tc  persistent tcgen05 kernel over cache-vertex tiles:
//                     shared surface hash encoding once per vertex, N_c BSDF
//                     directions + the residual direction per vertex encoded
//                     straight into the SMEM A tile, 3xTF32 MLP, and the MLMC
//                     combine  T*L_c - T'*n(w_cont)  reduced per vertex in
//                     deterministic order (cache_lc_s, kernels.py:424-448).
//   k_accumulate      per pixel: r = PT sum + cache terms; img += r,
//                     img2 += r*r, term += vertices (render_kernel :753-759).
#include <cstdlib>
#include <type_traits>
#include "common.cuh"
#include "pt_common.cuh"
#include "tc_mlp.cuh"

namespace nirc {

extern long long* g_infer_probe;
int sm_count();
int pack_weights(const nirc_spec_t& sp, const tc::TcNet& net, const float* theta, cudaStream_t s,
                 AsyncBuf& buf, PackedNet* out);
int tc_groups_for(const tc::TcNet& net, uint32_t extra_per_group);
bool default_layout(const nirc_spec_t& sp);

using pt::V3;

// One two-level cache vertex (the deferred work of kernels.py:559-601).
struct CacheVertex {
  double pos[3], ns[3], alb[3], rough;
  double wo[3];
  double T[3];    // throughput when the cache integral is added
  double Tp[3];   // post-roulette, post-bsdf throughput T' (residual weight)
  double wc[3];   // continuation direction w_cont
  uint64_t key;
  int32_t base, ncq, mkind, has_res;
  int32_t nrc, pad;  // nrc: one query at wo, added with +T (biased-nrc-sph stop)
  int64_t slot;   // sample * max_cv + cu
};

struct TraceOut {
  double* acc;       // (n_samples, 3)
  int32_t* term;     // (n_samples,)
  CacheVertex* cv;   // capacity n_samples * max_cv
  unsigned long long* counters;  // [0] cache vertices, [1] executed queries
};

// Per-lane path state of the persistent tracer.
struct PathState {
  V3 o, d, lns;
  double ar, ag, ab, tr, tg, tb, prev_pdf;
  double a0, a_sp;  // footprint spread state of the biased modes
  uint64_t key;
  int64_t sid;
  int v, cu, term, v1;
};

// Warp-aggregated fetch of the next sample index for the lanes in `want`.
__device__ inline int64_t fetch_sample(unsigned long long* ctr, bool want) {
  const unsigned mask = __activemask();
  const unsigned need = __ballot_sync(mask, want);
  if (!want) return -1;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(need) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(ctr, (unsigned long long)__popc(need));
  base = __shfl_sync(need, base, leader);
  return (int64_t)base + __popc(need & ((1u << lane) - 1u));
}

__device__ inline void start_path(PathState& p, const double* cam, const nirc_render_cfg_t& cfg,
                                  int64_t sid) {
  const int W = cfg.width;
  const int s = (int)(sid % cfg.spp);
  const int64_t lp = sid / cfg.spp;
  const int ix = (int)(lp % W);
  const int iy = cfg.row0 + (int)(lp / W);
  const int64_t pix = (int64_t)iy * W + ix;
  p.sid = sid;
  p.key = stream_key(cfg.seed, P_RENDER, cfg.frame, (uint64_t)pix, (uint64_t)s);
  pt::camera_ray(cam, ix, iy, rand_uniform(p.key, DIM_JITTER_X), rand_uniform(p.key, DIM_JITTER_Y),
                 p.o, p.d);
  p.ar = p.ag = p.ab = 0.0;
  p.tr = p.tg = p.tb = 1.0;
  p.prev_pdf = -1.0;
  p.lns = {0.0, 0.0, 0.0};
  p.v = p.cu = p.term = 0;
  p.a0 = 0.0;
  p.a_sp = 1.0;
  p.v1 = cfg.v1 ? cfg.v1[pix] : 0;
}

__device__ inline void fill_stop_vertex(CacheVertex& rec, const PathState& p, V3 pos, V3 ns,
                                        V3 alb, double rough, V3 wo, int base, int mkind,
                                        int ncq, int nrc, int max_cv) {
  rec.pos[0] = pos.x; rec.pos[1] = pos.y; rec.pos[2] = pos.z;
  rec.ns[0] = ns.x; rec.ns[1] = ns.y; rec.ns[2] = ns.z;
  rec.alb[0] = alb.x; rec.alb[1] = alb.y; rec.alb[2] = alb.z;
  rec.rough = rough;
  rec.wo[0] = wo.x; rec.wo[1] = wo.y; rec.wo[2] = wo.z;
  rec.T[0] = p.tr; rec.T[1] = p.tg; rec.T[2] = p.tb;
  rec.key = p.key;
  rec.base = base;
  rec.ncq = ncq;
  rec.mkind = mkind;
  rec.has_res = 0;
  rec.nrc = nrc;
  rec.pad = 0;
  rec.slot = p.sid * max_cv;
  rec.Tp[0] = rec.Tp[1] = rec.Tp[2] = 0.0;
  rec.wc[0] = rec.wc[1] = 0.0;
  rec.wc[2] = 1.0;
}

// One vertex of trace_sample's biased family (kernels.py:609-720): the
// spread / stochastic-brdf / first-vertex stop tests; the stop vertex is
// shaded by NEE + the cache integral over nbias directions (NIRC modes) or
// one NRC query at wo, deferred to the inference pass like the two-level
// cache vertices.  Returns true when the path ended.
__device__ inline bool trace_vertex_biased(const nirc_scene_t& scn, const nirc_render_cfg_t& cfg,
                                           PathState& p, CacheVertex& rec, int& pending) {
  pending = 0;
  const int v = p.v;
  const pt::Hit h = pt::intersect<false>(scn, p.o, p.d, pt::T_FAR);
  if (h.kind < 0) {
    if (scn.env_kind != pt::ENV_NONE) {
      const V3 e = pt::env_eval(scn, p.d);
      double w = 1.0;
      if (p.prev_pdf >= 0.0) {
        const double pn = pt::nee_pdf_for_env(scn, p.lns, p.d);
        w = p.prev_pdf / (p.prev_pdf + pn);
      }
      p.ar += p.tr * w * e.x;
      p.ag += p.tg * w * e.y;
      p.ab += p.tb * w * e.z;
    }
    return true;
  }
  p.term = v + 1;
  const V3 wo = {-p.d.x, -p.d.y, -p.d.z};
  const double flip = (h.n.x * wo.x + h.n.y * wo.y + h.n.z * wo.z) >= 0.0 ? 1.0 : -1.0;
  const V3 ns = {h.n.x * flip, h.n.y * flip, h.n.z * flip};
  const V3 em = pt::ld3(scn.mat_emit, h.mid);
  if (em.x > 0.0 || em.y > 0.0 || em.z > 0.0) {
    double w = 1.0;
    if (p.prev_pdf >= 0.0) {
      const double pn = pt::nee_pdf_for_hit(scn, h.kind, h.prim, h.t, p.d, h.n);
      w = p.prev_pdf / (p.prev_pdf + pn);
    }
    p.ar += p.tr * w * em.x;
    p.ag += p.tg * w * em.y;
    p.ab += p.tb * w * em.z;
  }
  const int mkind = scn.mat_kind[h.mid];
  const V3 alb = pt::ld3(scn.mat_albedo, h.mid);
  const double rough = scn.mat_rough[h.mid];
  const int base = VERTEX_DIM_BASE + v * DIMS_PER_VERTEX;
  const uint64_t key = p.key;
  if (mkind == pt::MAT_MIRROR) {  // delta vertex: no stop tests (kernels.py:520-548)
    double rr_div = 1.0;
    if (v >= pt::RR_START) {
      if (rand_uniform(key, base + OFF_RR) >= cfg.rr_survive) return true;
      rr_div = cfg.rr_survive;
    }
    const pt::BsdfSample b = pt::bsdf_sample(mkind, alb, rough, ns, wo,
                                             rand_uniform(key, base + OFF_BSDF_U),
                                             rand_uniform(key, base + OFF_BSDF_U + 1));
    if (b.pdf <= 0.0) return true;
    const double ci = b.wi.x * ns.x + b.wi.y * ns.y + b.wi.z * ns.z;
    if (ci <= 0.0) return true;
    const double inv = 1.0 / (b.pdf * rr_div);
    p.tr *= b.f.x * ci * inv;
    p.tg *= b.f.y * ci * inv;
    p.tb *= b.f.z * ci * inv;
    p.prev_pdf = -1.0;
    const double sg = (h.n.x * b.wi.x + h.n.y * b.wi.y + h.n.z * b.wi.z) > 0.0 ? 1.0 : -1.0;
    p.o = {h.p.x + sg * scn.eps * h.n.x, h.p.y + sg * scn.eps * h.n.y,
           h.p.z + sg * scn.eps * h.n.z};
    p.d = b.wi;
    p.lns = ns;
    p.v = v + 1;
    return p.v >= pt::MAXB;
  }
  // relative-footprint state (kernels.py:612-618)
  const double cs_arr = wo.x * ns.x + wo.y * ns.y + wo.z * ns.z;
  if (v == 0) {
    if (cs_arr > 0.0) p.a0 = h.t * h.t / (4.0 * pt::PI * cs_arr);
  } else if (p.prev_pdf > 0.0 && cs_arr > 0.0) {
    const double fac = h.t / (p.prev_pdf * cs_arr);
    p.a_sp *= fac * fac;
  }
  const double nb = (double)cfg.nbias;
  int stop = 0, have_cont = 0;
  pt::BsdfSample b;
  b.pdf = 0.0;
  if (cs_arr <= 0.0) {
    stop = 1;
  } else if (cfg.mode == 2) {  // MODE_BTH
    if (v >= 1 && p.a_sp > cfg.sph_c * p.a0) {
      stop = 1;
    } else {
      b = pt::bsdf_sample(mkind, alb, rough, ns, wo, rand_uniform(key, base + OFF_BSDF_U),
                          rand_uniform(key, base + OFF_BSDF_U + 1));
      double ps = 0.0;
      if (b.pdf > 0.0 && b.delta == 0) {
        const double ci = b.wi.x * ns.x + b.wi.y * ns.y + b.wi.z * ns.z;
        if (ci > 0.0) {
          have_cont = 1;
          ps = b.pdf / (b.pdf + nb / pt::PI);
        }
      }
      if (rand_uniform(key, base + OFF_TERM) > ps) stop = 1;
    }
  } else {
    if (v == 0) {
      if (p.v1 == 1 && (cfg.mode == 3 || rough >= cfg.rough_cut)) stop = 1;
    } else if (p.a_sp > cfg.sph_c * p.a0) {
      stop = 1;
    }
  }
  if (stop == 1) {
    if (cfg.mode == 4) {  // MODE_NRC_SPH: one outgoing-radiance query at wo
      if (cfg.cache_on == 1) {
        pending = 1;
        fill_stop_vertex(rec, p, h.p, ns, alb, rough, wo, base, mkind, 0, 1, cfg.max_cv);
      }
    } else {
      const V3 q = pt::nee_contrib(scn, h.p, ns, h.n, mkind, alb, rough, wo,
                                   rand_uniform(key, base + OFF_LIGHT_PICK),
                                   rand_uniform(key, base + OFF_LIGHT_U),
                                   rand_uniform(key, base + OFF_LIGHT_U + 1), 0);
      p.ar += p.tr * q.x;
      p.ag += p.tg * q.y;
      p.ab += p.tb * q.z;
      if (cfg.cache_on == 1) {
        pending = 1;
        fill_stop_vertex(rec, p, h.p, ns, alb, rough, wo, base, mkind, cfg.nbias, 0,
                         cfg.max_cv);
      }
    }
    return true;
  }
  const V3 q = pt::nee_contrib(scn, h.p, ns, h.n, mkind, alb, rough, wo,
                               rand_uniform(key, base + OFF_LIGHT_PICK),
                               rand_uniform(key, base + OFF_LIGHT_U),
                               rand_uniform(key, base + OFF_LIGHT_U + 1), 0);
  p.ar += p.tr * q.x;
  p.ag += p.tg * q.y;
  p.ab += p.tb * q.z;
  double rr_div = 1.0;
  if (v >= pt::RR_START) {
    if (rand_uniform(key, base + OFF_RR) >= cfg.rr_survive) return true;
    rr_div = cfg.rr_survive;
  }
  if (have_cont == 0) {
    b = pt::bsdf_sample(mkind, alb, rough, ns, wo, rand_uniform(key, base + OFF_BSDF_U),
                        rand_uniform(key, base + OFF_BSDF_U + 1));
    if (b.pdf <= 0.0) return true;
    const double ci = b.wi.x * ns.x + b.wi.y * ns.y + b.wi.z * ns.z;
    if (ci <= 0.0) return true;
  }
  const double ci = b.wi.x * ns.x + b.wi.y * ns.y + b.wi.z * ns.z;
  const double inv = 1.0 / (b.pdf * rr_div);
  p.tr *= b.f.x * ci * inv;
  p.tg *= b.f.y * ci * inv;
  p.tb *= b.f.z * ci * inv;
  p.prev_pdf = b.pdf;
  const double sg = (h.n.x * b.wi.x + h.n.y * b.wi.y + h.n.z * b.wi.z) > 0.0 ? 1.0 : -1.0;
  p.o = {h.p.x + sg * scn.eps * h.n.x, h.p.y + sg * scn.eps * h.n.y,
         h.p.z + sg * scn.eps * h.n.z};
  p.d = b.wi;
  p.lns = ns;
  p.v = v + 1;
  return p.v >= pt::MAXB;
}

// One vertex of trace_sample (kernels.py:481-608) for MODE_PT / MODE_TL.
// Returns true when the path ended.  A two-level cache vertex is returned in
// `rec` (pending == 1) instead of being evaluated inline.
__device__ inline bool trace_vertex_pt_tl(const nirc_scene_t& scn, const nirc_render_cfg_t& cfg,
                                          PathState& p, CacheVertex& rec, int& pending) {
  pending = 0;
  const int v = p.v;
  const pt::Hit h = pt::intersect<false>(scn, p.o, p.d, pt::T_FAR);
  if (h.kind < 0) {
    if (scn.env_kind != pt::ENV_NONE) {
      const V3 e = pt::env_eval(scn, p.d);
      double w = 1.0;
      if (p.prev_pdf >= 0.0) {
        const double pn = pt::nee_pdf_for_env(scn, p.lns, p.d);
        w = p.prev_pdf / (p.prev_pdf + pn);
      }
      p.ar += p.tr * w * e.x;
      p.ag += p.tg * w * e.y;
      p.ab += p.tb * w * e.z;
    }
    return true;
  }
  p.term = v + 1;
  const V3 wo = {-p.d.x, -p.d.y, -p.d.z};
  const double flip = (h.n.x * wo.x + h.n.y * wo.y + h.n.z * wo.z) >= 0.0 ? 1.0 : -1.0;
  const V3 ns = {h.n.x * flip, h.n.y * flip, h.n.z * flip};
  const V3 em = pt::ld3(scn.mat_emit, h.mid);
  if (em.x > 0.0 || em.y > 0.0 || em.z > 0.0) {
    double w = 1.0;
    if (p.prev_pdf >= 0.0) {
      const double pn = pt::nee_pdf_for_hit(scn, h.kind, h.prim, h.t, p.d, h.n);
      w = p.prev_pdf / (p.prev_pdf + pn);
    }
    p.ar += p.tr * w * em.x;
    p.ag += p.tg * w * em.y;
    p.ab += p.tb * w * em.z;
  }
  const int mkind = scn.mat_kind[h.mid];
  const V3 alb = pt::ld3(scn.mat_albedo, h.mid);
  const double rough = scn.mat_rough[h.mid];
  const int base = VERTEX_DIM_BASE + v * DIMS_PER_VERTEX;
  const uint64_t key = p.key;
  double rr_div = 1.0;
  if (mkind == pt::MAT_MIRROR) {  // delta vertex, kernels.py:520-548
    if (v >= pt::RR_START) {
      if (rand_uniform(key, base + OFF_RR) >= cfg.rr_survive) return true;
      rr_div = cfg.rr_survive;
    }
  } else {
    const V3 q = pt::nee_contrib(scn, h.p, ns, h.n, mkind, alb, rough, wo,
                                 rand_uniform(key, base + OFF_LIGHT_PICK),
                                 rand_uniform(key, base + OFF_LIGHT_U),
                                 rand_uniform(key, base + OFF_LIGHT_U + 1), 0);
    p.ar += p.tr * q.x;
    p.ag += p.tg * q.y;
    p.ab += p.tb * q.z;
    if (cfg.mode == 1 && cfg.cache_on == 1 && rough >= cfg.rough_cut && p.cu < cfg.max_cv) {
      const int ncq = cfg.nc[p.cu];
      p.cu += 1;
      if (ncq > 0) {
        pending = 1;
        rec.pos[0] = h.p.x; rec.pos[1] = h.p.y; rec.pos[2] = h.p.z;
        rec.ns[0] = ns.x; rec.ns[1] = ns.y; rec.ns[2] = ns.z;
        rec.alb[0] = alb.x; rec.alb[1] = alb.y; rec.alb[2] = alb.z;
        rec.rough = rough;
        rec.wo[0] = wo.x; rec.wo[1] = wo.y; rec.wo[2] = wo.z;
        rec.T[0] = p.tr; rec.T[1] = p.tg; rec.T[2] = p.tb;
        rec.key = key;
        rec.base = base;
        rec.ncq = ncq;
        rec.mkind = mkind;
        rec.has_res = 0;
        rec.nrc = 0;
        rec.pad = 0;
        rec.slot = p.sid * cfg.max_cv + (p.cu - 1);
        rec.Tp[0] = rec.Tp[1] = rec.Tp[2] = 0.0;
        rec.wc[0] = rec.wc[1] = 0.0;
        rec.wc[2] = 1.0;
      }
    }
    if (v >= pt::RR_START) {
      if (rand_uniform(key, base + OFF_RR) >= cfg.rr_survive) return true;
      rr_div = cfg.rr_survive;
    }
  }
  const pt::BsdfSample b = pt::bsdf_sample(mkind, alb, rough, ns, wo,
                                           rand_uniform(key, base + OFF_BSDF_U),
                                           rand_uniform(key, base + OFF_BSDF_U + 1));
  if (b.pdf <= 0.0) return true;
  const double ci = b.wi.x * ns.x + b.wi.y * ns.y + b.wi.z * ns.z;
  if (ci <= 0.0) return true;
  const double inv = 1.0 / (b.pdf * rr_div);
  p.tr *= b.f.x * ci * inv;
  p.tg *= b.f.y * ci * inv;
  p.tb *= b.f.z * ci * inv;
  if (pending) {  // residual along the continuation (kernels.py:593-601)
    rec.has_res = 1;
    rec.Tp[0] = p.tr; rec.Tp[1] = p.tg; rec.Tp[2] = p.tb;
    rec.wc[0] = b.wi.x; rec.wc[1] = b.wi.y; rec.wc[2] = b.wi.z;
  }
  p.prev_pdf = mkind == pt::MAT_MIRROR ? -1.0 : b.pdf;
  const double sg = (h.n.x * b.wi.x + h.n.y * b.wi.y + h.n.z * b.wi.z) > 0.0 ? 1.0 : -1.0;
  p.o = {h.p.x + sg * scn.eps * h.n.x, h.p.y + sg * scn.eps * h.n.y,
         h.p.z + sg * scn.eps * h.n.z};
  p.d = b.wi;
  p.lns = ns;
  p.v = v + 1;
  return p.v >= pt::MAXB;
}

// kBiased: the biased early-stop family, else MODE_PT / MODE_TL.  Compiled
// as separate tracer instantiations so each carries only its own code.
template <bool kBiased>
__device__ inline bool trace_vertex(const nirc_scene_t& scn, const nirc_render_cfg_t& cfg,
                                    PathState& p, CacheVertex& rec, int& pending) {
  if constexpr (kBiased) return trace_vertex_biased(scn, cfg, p, rec, pending);
  else return trace_vertex_pt_tl(scn, cfg, p, rec, pending);
}

// ---------------------------------------------------------------------
// Training records: walk_record (kernels.py:85-286) driven by
// collect_paths_kernel (:289-311).  Each path's vertices are kept in a
// vertex-major staging area and the backward sweep runs when the path ends;
// a scan turns per-path record counts into offsets and a compaction writes
// the records in (path, vertex) order -- the reference's row order.  The
// walk is written per lane (walk_start / walk_vertex / walk_finish) so the
// persistent tracer can interleave training paths with camera paths.
// Record kinds (caches.py:87-131): 0 nirc, 1 nirc_full, 2 nrc, 3 nvc, 4 nirc_env.
constexpr int REC_NIRC = 0, REC_NIRC_FULL = 1, REC_NRC = 2, REC_NVC = 3, REC_NIRC_ENV = 4;

struct Stage {
  // vertex-major: field[v * count + p]; one candidate record per vertex,
  // already in the requested kind's (dirs, pdf, target) form
  double *pos, *ns, *alb, *rough, *wi, *pdf, *tgt;
  uint8_t* keep;
  int32_t* nrec;   // per path
  int32_t* nvert;  // per path
  int64_t count;
  int64_t path0;   // global index of local path 0 (multi-GPU path shards)
  int32_t kind;    // REC_*
  int32_t pad;
};

struct WalkLane {
  V3 o, d, lns;
  double prev_pdf;
  uint64_t key;
  int64_t p;
  int v, esc;
  double env_m[3], env_r[3];
  // per-vertex backward-sweep inputs (local memory)
  double mise[pt::MAXB][3], emit[pt::MAXB][3], nee[pt::MAXB][3], fcp[pt::MAXB][3];
};

__device__ inline void walk_start(WalkLane& w, const double* cam, uint64_t seed, uint64_t frame,
                                  const Stage& st, int64_t p) {
  w.p = p;
  w.key = stream_key(seed, P_TRAIN, frame, (uint64_t)(st.path0 + p), 0);
  const double sx = rand_uniform(w.key, DIM_JITTER_X) * cam[14];
  const double sy = rand_uniform(w.key, DIM_JITTER_Y) * cam[15];
  const int ix = (int)sx, iy = (int)sy;
  pt::camera_ray(cam, ix, iy, sx - ix, sy - iy, w.o, w.d);
  w.prev_pdf = -1.0;
  w.lns = {0.0, 0.0, 0.0};
  w.v = 0;
  w.esc = 0;
  for (int c = 0; c < 3; ++c) w.env_m[c] = w.env_r[c] = 0.0;
}

// One vertex of walk_record; returns true when the path ended (w.v = the
// vertex count n).
__device__ inline bool walk_vertex(const nirc_scene_t& scn, WalkLane& w, const Stage& st) {
  const int v = w.v;
  const int64_t C = st.count, p = w.p;
  const pt::Hit hh = pt::intersect<false>(scn, w.o, w.d, pt::T_FAR);
  if (hh.kind < 0) {
    if (scn.env_kind != pt::ENV_NONE) {
      const V3 e = pt::env_eval(scn, w.d);
      w.env_r[0] = e.x; w.env_r[1] = e.y; w.env_r[2] = e.z;
      double wgt = 1.0;
      if (w.prev_pdf >= 0.0) {
        const double pn = pt::nee_pdf_for_env(scn, w.lns, w.d);
        wgt = w.prev_pdf / (w.prev_pdf + pn);
      }
      w.env_m[0] = wgt * e.x; w.env_m[1] = wgt * e.y; w.env_m[2] = wgt * e.z;
    }
    w.esc = 1;
    return true;
  }
  const V3 wo = {-w.d.x, -w.d.y, -w.d.z};
  const double flip = (hh.n.x * wo.x + hh.n.y * wo.y + hh.n.z * wo.z) >= 0.0 ? 1.0 : -1.0;
  const V3 ns = {hh.n.x * flip, hh.n.y * flip, hh.n.z * flip};
  const V3 em = pt::ld3(scn.mat_emit, hh.mid);
  if (em.x > 0.0 || em.y > 0.0 || em.z > 0.0) {
    double wgt = 1.0;
    if (w.prev_pdf >= 0.0) {
      const double pn = pt::nee_pdf_for_hit(scn, hh.kind, hh.prim, hh.t, w.d, hh.n);
      wgt = w.prev_pdf / (w.prev_pdf + pn);
    }
    w.mise[v][0] = wgt * em.x; w.mise[v][1] = wgt * em.y; w.mise[v][2] = wgt * em.z;
    w.emit[v][0] = em.x; w.emit[v][1] = em.y; w.emit[v][2] = em.z;
  } else {
    w.mise[v][0] = w.mise[v][1] = w.mise[v][2] = 0.0;
    w.emit[v][0] = w.emit[v][1] = w.emit[v][2] = 0.0;
  }
  const int mkind = scn.mat_kind[hh.mid];
  const int delta = mkind == pt::MAT_MIRROR ? 1 : 0;
  const V3 alb = pt::ld3(scn.mat_albedo, hh.mid);
  const double rough = scn.mat_rough[hh.mid];
  const int64_t at = (int64_t)v * C + p;
  st.pos[3 * at] = hh.p.x; st.pos[3 * at + 1] = hh.p.y; st.pos[3 * at + 2] = hh.p.z;
  st.ns[3 * at] = ns.x; st.ns[3 * at + 1] = ns.y; st.ns[3 * at + 2] = ns.z;
  st.alb[3 * at] = alb.x; st.alb[3 * at + 1] = alb.y; st.alb[3 * at + 2] = alb.z;
  st.rough[at] = rough;
  const int base = VERTEX_DIM_BASE + v * DIMS_PER_VERTEX;
  const uint64_t key = w.key;
  V3 q = {0.0, 0.0, 0.0};
  if (delta == 0)
    q = pt::nee_contrib(scn, hh.p, ns, hh.n, mkind, alb, rough, wo,
                        rand_uniform(key, base + OFF_LIGHT_PICK),
                        rand_uniform(key, base + OFF_LIGHT_U),
                        rand_uniform(key, base + OFF_LIGHT_U + 1), 0);
  w.nee[v][0] = q.x; w.nee[v][1] = q.y; w.nee[v][2] = q.z;
  const int kind = st.kind;
  if (kind == REC_NVC || kind == REC_NIRC_ENV) {
    // environment-visibility record (kernels.py:183-210)
    uint8_t ok = 0;
    if (delta == 0 && scn.env_kind != pt::ENV_NONE) {
      const pt::Cosine c = pt::cosine_dir(rand_uniform(key, base + OFF_CACHE),
                                          rand_uniform(key, base + OFF_CACHE + 1));
      if (c.pdf > 0.0) {
        const Onb b = onb(ns.x, ns.y, ns.z);
        const V3 e = {b.tx * c.x + b.bx * c.y + ns.x * c.z, b.ty * c.x + b.by * c.y + ns.y * c.z,
                      b.tz * c.x + b.bz * c.y + ns.z * c.z};
        const double sg = (hh.n.x * e.x + hh.n.y * e.y + hh.n.z * e.z) > 0.0 ? 1.0 : -1.0;
        const V3 so = {hh.p.x + sg * scn.eps * hh.n.x, hh.p.y + sg * scn.eps * hh.n.y,
                       hh.p.z + sg * scn.eps * hh.n.z};
        const double vis = pt::occluded(scn, so, e, pt::T_FAR) ? 0.0 : 1.0;
        const V3 er = pt::env_eval(scn, e);
        st.wi[3 * at] = e.x; st.wi[3 * at + 1] = e.y; st.wi[3 * at + 2] = e.z;
        st.pdf[at] = c.pdf;
        if (kind == REC_NVC) {
          st.tgt[3 * at] = st.tgt[3 * at + 1] = st.tgt[3 * at + 2] = vis;
        } else {
          st.tgt[3 * at] = vis * er.x; st.tgt[3 * at + 1] = vis * er.y;
          st.tgt[3 * at + 2] = vis * er.z;
        }
        ok = 1;
      }
    }
    st.keep[at] = ok;
  } else if (kind == REC_NRC) {
    // keyed at the vertex the sampled segment landed on (caches.py:107-116):
    // direction = -w_i of the previous vertex = wo, pdf of that segment
    st.wi[3 * at] = wo.x; st.wi[3 * at + 1] = wo.y; st.wi[3 * at + 2] = wo.z;
    st.pdf[at] = w.prev_pdf;
    st.keep[at] = (v >= 1 && delta == 0 && w.prev_pdf > 0.0) ? 1 : 0;
  }
  int alive = 1;
  double rr_div = 1.0;
  if (v >= pt::RR_START) {
    if (rand_uniform(key, base + OFF_RR) >= pt::RR_SURVIVE) alive = 0;
    else rr_div = pt::RR_SURVIVE;
  }
  int cont = 0;
  double vpdf = 0.0;
  V3 vwi = {0.0, 0.0, 0.0};
  w.fcp[v][0] = w.fcp[v][1] = w.fcp[v][2] = 0.0;
  if (alive == 1 && v < pt::MAXB - 1) {
    const pt::BsdfSample b = pt::bsdf_sample(mkind, alb, rough, ns, wo,
                                             rand_uniform(key, base + OFF_BSDF_U),
                                             rand_uniform(key, base + OFF_BSDF_U + 1));
    if (b.pdf > 0.0) {
      const double ci = b.wi.x * ns.x + b.wi.y * ns.y + b.wi.z * ns.z;
      if (ci > 0.0) {
        const double inv = 1.0 / (b.pdf * rr_div);
        vwi = b.wi;
        vpdf = b.delta == 1 ? -1.0 : b.pdf;
        w.fcp[v][0] = b.f.x * ci * inv;
        w.fcp[v][1] = b.f.y * ci * inv;
        w.fcp[v][2] = b.f.z * ci * inv;
        w.prev_pdf = vpdf;
        const double sg = (hh.n.x * b.wi.x + hh.n.y * b.wi.y + hh.n.z * b.wi.z) > 0.0 ? 1.0 : -1.0;
        w.o = {hh.p.x + sg * scn.eps * hh.n.x, hh.p.y + sg * scn.eps * hh.n.y,
               hh.p.z + sg * scn.eps * hh.n.z};
        w.d = b.wi;
        w.lns = ns;
        cont = 1;
      }
    }
  }
  if (kind == REC_NIRC || kind == REC_NIRC_FULL) {
    st.wi[3 * at] = vwi.x; st.wi[3 * at + 1] = vwi.y; st.wi[3 * at + 2] = vwi.z;
    st.pdf[at] = vpdf;
    st.keep[at] = (delta == 0 && vpdf > 0.0) ? 1 : 0;
  }
  w.v = v + 1;
  return cont == 0;
}

// Backward sweep (kernels.py:249-277) over the path's w.v vertices: the
// incident-radiance targets (MIS-weighted emission for nirc, raw emission
// for nirc_full) and the outgoing radiance at each vertex (nrc).
__device__ inline void walk_finish(const WalkLane& w, const Stage& st) {
  const int64_t C = st.count, p = w.p;
  const int n = w.v;
  const int kind = st.kind;
  double lr = 0.0, lg = 0.0, lb = 0.0;
  int nrec = 0;
  for (int v = n - 1; v >= 0; --v) {
    double cr, cg, cb, qr, qg, qb;
    if (v == n - 1) {
      cr = w.esc ? w.env_m[0] : 0.0; cg = w.esc ? w.env_m[1] : 0.0; cb = w.esc ? w.env_m[2] : 0.0;
      qr = w.esc ? w.env_r[0] : 0.0; qg = w.esc ? w.env_r[1] : 0.0; qb = w.esc ? w.env_r[2] : 0.0;
    } else {
      cr = w.mise[v + 1][0] + lr; cg = w.mise[v + 1][1] + lg; cb = w.mise[v + 1][2] + lb;
      qr = w.emit[v + 1][0] + lr; qg = w.emit[v + 1][1] + lg; qb = w.emit[v + 1][2] + lb;
    }
    const int64_t at = (int64_t)v * C + p;
    if (kind == REC_NIRC) {
      st.tgt[3 * at] = cr; st.tgt[3 * at + 1] = cg; st.tgt[3 * at + 2] = cb;
    } else if (kind == REC_NIRC_FULL) {
      st.tgt[3 * at] = qr; st.tgt[3 * at + 1] = qg; st.tgt[3 * at + 2] = qb;
    }
    lr = w.nee[v][0] + w.fcp[v][0] * cr;
    lg = w.nee[v][1] + w.fcp[v][1] * cg;
    lb = w.nee[v][2] + w.fcp[v][2] * cb;
    if (kind == REC_NRC) {
      st.tgt[3 * at] = lr; st.tgt[3 * at + 1] = lg; st.tgt[3 * at + 2] = lb;
    }
    nrec += st.keep[at];
  }
  st.nrec[p] = nrec;
  st.nvert[p] = n;
}

// Stand-alone collection (Cache.collect without a render): one thread per path.
__global__ void k_walk_record(nirc_scene_t scn, const double* __restrict__ cam, uint64_t seed,
                              uint64_t frame, Stage st) {
  __shared__ __align__(16) unsigned char scene_sm[pt::kSceneSmemBytes];
  pt::stage_scene(scn, scene_sm);
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= st.count) return;
  WalkLane w;
  walk_start(w, cam, seed, frame, st, p);
  while (!walk_vertex(scn, w, st)) {
  }
  walk_finish(w, st);
}

// K5: persistent path tracer.  Each lane owns one path at a time and pulls
// the next (pixel, sample) from a global counter as soon as its path ends,
// so lanes stay busy despite Russian-roulette path-length variance (a plain
// one-thread-per-sample megakernel idles ~80% of each warp).
// Training paths traced by the same persistent kernel (render + collect of
// one frame in one launch): work items [0, n) are walk_record paths, taken
// first so their long Russian-roulette tails overlap the camera paths.
struct WalkJob {
  Stage st;
  uint64_t seed, frame;
  int64_t n;  // 0: render only
};

#ifndef NIRC_TRACE_MINB
#define NIRC_TRACE_MINB 3  // measured with the fp32 pre-test: 3 CTAs/SM (168 regs) beat 4 and 2
#endif
#ifndef NIRC_TRACE_MINB_BVH
#define NIRC_TRACE_MINB_BVH 8  // BVH-traversed scenes: latency-bound, 8 CTAs/SM measured best (4..12)
#endif
// kWalks: the launch also traces the frame's training walks (render+collect);
// render-only launches are compiled without the walk lanes' state.  kMinB:
// CTAs per SM the register budget is sized for (the warp-uniform scan of
// small scenes wants registers, BVH traversal of larger ones wants warps).
template <bool kBiased, bool kWalks, int kMinB>
__global__ void __launch_bounds__(128, kMinB)
    k_trace(nirc_scene_t scn, const double* __restrict__ cam, nirc_render_cfg_t cfg, TraceOut out,
            WalkJob job) {
  // the staged scene, sized to it (dynamic: the rest of the SM's 256 KB
  // stays L1 for the lanes' local state)
  extern __shared__ __align__(16) unsigned char scene_sm[];
  pt::stage_scene(scn, scene_sm);
  const int64_t nsamp = (int64_t)(cfg.row1 - cfg.row0) * cfg.width * cfg.spp;
  const int64_t nwalk = kWalks ? job.n : 0;
  const int64_t nwork = nwalk + nsamp;
  PathState p;
  typename std::conditional<kWalks, WalkLane, char>::type wl;
  bool active = false, walking = false;
  auto start = [&](int64_t item) {
    if (item < nwalk) {
      if constexpr (kWalks) walk_start(wl, cam, job.seed, job.frame, job.st, item);
      walking = true;
    } else {
      start_path(p, cam, cfg, item - nwalk);
      walking = false;
    }
    active = true;
  };
  int64_t item = fetch_sample(out.counters + 2, true);
  if (item < nwork) start(item);
  while (__any_sync(0xffffffffu, active)) {
    CacheVertex rec;
    int pending = 0;
    bool done = false;
    if (active) {
      if (walking) {
        if constexpr (kWalks) {
          done = walk_vertex(scn, wl, job.st);
          if (done) walk_finish(wl, job.st);
        }
      } else {
        done = trace_vertex<kBiased>(scn, cfg, p, rec, pending);
      }
    }
    // warp-aggregated append of the cache-vertex records and query counts
    const unsigned pm = __ballot_sync(0xffffffffu, pending);
    if (pending) {
      const int lane = threadIdx.x & 31;
      const int leader = __ffs(pm) - 1;
      unsigned long long base = 0;
      const unsigned q = __reduce_add_sync(pm, (unsigned)(rec.ncq + rec.has_res + rec.nrc));
      if (lane == leader) {
        base = atomicAdd(out.counters, (unsigned long long)__popc(pm));
        atomicAdd(out.counters + 1, (unsigned long long)q);
      }
      base = __shfl_sync(pm, base, leader);
      out.cv[base + __popc(pm & ((1u << lane) - 1u))] = rec;
    }
    if (active && done) {
      if (!walking) {
        out.acc[3 * p.sid] = p.ar;
        out.acc[3 * p.sid + 1] = p.ag;
        out.acc[3 * p.sid + 2] = p.ab;
        out.term[p.sid] = p.term;
      }
      active = false;
    }
    const int64_t nxt = fetch_sample(out.counters + 2, !active);
    if (!active && nxt < nwork) start(nxt);
  }
}

// ---------------------------------------------------------------------
// Row of the amortised inference: direction + weights for query k of a
// cache vertex (cache_lc_s, kernels.py:432-446) or its residual row.
struct RowDir {
  V3 wi;
  double s;  // ci / pdf for cache rows
  V3 f;
  int kind;  // 0 invalid, 1 cache sample, 2 residual
};

__device__ inline RowDir row_direction(const CacheVertex& r, int k) {
  RowDir o;
  o.kind = 0;
  o.wi = {0.0, 0.0, 1.0};
  o.s = 0.0;
  o.f = {0.0, 0.0, 0.0};
  if (k < r.ncq) {
    const V3 ns = {r.ns[0], r.ns[1], r.ns[2]};
    const pt::BsdfSample b = pt::bsdf_sample(
        r.mkind, {r.alb[0], r.alb[1], r.alb[2]}, r.rough, ns, {r.wo[0], r.wo[1], r.wo[2]},
        rand_uniform(r.key, r.base + OFF_CACHE + 2 * k),
        rand_uniform(r.key, r.base + OFF_CACHE + 2 * k + 1));
    if (b.pdf <= 0.0 || b.delta == 1) return o;
    const double ci = b.wi.x * ns.x + b.wi.y * ns.y + b.wi.z * ns.z;
    if (ci <= 0.0) return o;
    o.kind = 1;
    o.wi = b.wi;
    o.s = ci / b.pdf;
    o.f = b.f;
  } else if (k == r.ncq && r.has_res) {
    o.kind = 2;
    o.wi = {r.wc[0], r.wc[1], r.wc[2]};
  } else if (k == 0 && r.nrc) {  // NRC stop: outgoing radiance along wo
    o.kind = 3;
    o.wi = {r.wo[0], r.wo[1], r.wo[2]};
  }
  return o;
}

// Encoded input of one inference row: shared surface features (24 floats
// computed once per vertex), SH of the row direction in the scalar-path
// order (encode_dir_into -> sh_eval_into, sh.py:36-76), aux block.
__device__ inline void build_row(const nirc_spec_t& sp, const float* feat, const CacheVertex& r,
                                 V3 wi, float* x) {
#pragma unroll
  for (int i = 0; i < 24; ++i) x[i] = feat[i];
  sh_eval<false>(wi.x, wi.y, wi.z, 4, sp.sh_k, [&](int i, double v) {
    x[24 + i] = __double2float_rn(v);
  });
  x[40] = __double2float_rn((r.ns[0] + 1.0) * 0.5);
  x[41] = __double2float_rn((r.ns[1] + 1.0) * 0.5);
  x[42] = __double2float_rn((r.ns[2] + 1.0) * 0.5);
  x[43] = __double2float_rn(r.alb[0]);
  x[44] = __double2float_rn(r.alb[1]);
  x[45] = __double2float_rn(r.alb[2]);
  x[46] = __double2float_rn(r.rough);
  x[47] = 0.0f;
}

// fp32 producer for the amortised inference rows (render path only; the
// reference-exact f64 sampler above stays for non-Lambert lobes).  The
// directions feed only the network input (SH) and the Lambert weight
// f*cos/pdf = albedo*cos/(cos/pi); fp32 changes either by ~1e-7 relative,
// far inside the two-level image tolerance (tests/test_gpu_render.py).
// Per-vertex part of the fp32 Lambert sampler: the ONB of the shading normal
// (core.py:39-54 onb_s, Duff et al.) and the visibility of wo.
struct LambertFrame {
  float nx, ny, nz, tx, ty, tz, bx, by, bz;
  bool co_pos;
};
__device__ inline LambertFrame lambert_frame(const CacheVertex& r) {
  LambertFrame F;
  F.nx = (float)r.ns[0];
  F.ny = (float)r.ns[1];
  F.nz = (float)r.ns[2];
  const float sg = F.nz >= 0.0f ? 1.0f : -1.0f;
  const float a = -1.0f / (sg + F.nz);
  const float bb = F.nx * F.ny * a;
  F.tx = 1.0f + sg * F.nx * F.nx * a;
  F.ty = sg * bb;
  F.tz = -sg * F.nx;
  F.bx = bb;
  F.by = sg + F.ny * F.ny * a;
  F.bz = -F.ny;
  const double co = r.ns[0] * r.wo[0] + r.ns[1] * r.wo[1] + r.ns[2] * r.wo[2];
  F.co_pos = co > 0.0;
  return F;
}
// Per-row part: cosine-weighted direction k (cosine_dir_s, core.py:57-65)
// from the vertex's stream; kind 1 with s = cos/pdf, or kind 0 (rejected).
__device__ inline void lambert_row(const LambertFrame& F, uint64_t key, int64_t base, int k,
                                   float* w, double* s_out, int* kind) {
  const float u1 = rand_uniform_f32(key, base + OFF_CACHE + 2 * k);
  const float u2 = rand_uniform_f32(key, base + OFF_CACHE + 2 * k + 1);
  // fast-math sampler: the directions feed the network input and the
  // Lambert weight only (hardware sin / cos of 2 pi u2 to ~1e-6 absolute)
  float sp, cp;
  __sincosf(6.28318530717958647692f * u2, &sp, &cp);
  float rr, lz;  // (approximate MUFU square roots, ~1 ulp)
  asm("sqrt.approx.f32 %0, %1;" : "=f"(rr) : "f"(u1));
  asm("sqrt.approx.f32 %0, %1;" : "=f"(lz) : "f"(fmaxf(0.0f, 1.0f - u1)));
  const float lx = rr * cp, ly = rr * sp;
  const float pdf = lz * (float)pt::INV_PI;
  w[0] = F.tx * lx + F.bx * ly + F.nx * lz;
  w[1] = F.ty * lx + F.by * ly + F.ny * lz;
  w[2] = F.tz * lx + F.bz * ly + F.nz * lz;
  *kind = 0;
  *s_out = 0.0;
  if (!F.co_pos || pdf <= 0.0f) return;
  const float ci = w[0] * F.nx + w[1] * F.ny + w[2] * F.nz;
  if (ci <= 0.0f) return;
  *kind = 1;
  *s_out = (double)__fdividef(ci, pdf);
}

// fp32 producer for the amortised inference rows (render path only; the
// reference-exact f64 sampler above stays for non-Lambert lobes).  The
// directions feed only the network input (SH) and the Lambert weight
// f*cos/pdf = albedo*cos/(cos/pi); fp32 changes either by ~1e-7 relative,
// far inside the two-level image tolerance (tests/test_gpu_render.py).
__device__ inline RowDir row_direction_fast(const CacheVertex& r, int k) {
  if (r.mkind != pt::MAT_LAMBERT || k >= r.ncq) return row_direction(r, k);
  RowDir o;
  o.f = {0.0, 0.0, 0.0};
  const LambertFrame F = lambert_frame(r);
  float w[3];
  lambert_row(F, r.key, r.base, k, w, &o.s, &o.kind);
  if (o.kind == 0) {
    o.wi = {0.0, 0.0, 1.0};
    return o;
  }
  o.wi = {w[0], w[1], w[2]};
  o.f = {r.alb[0] * pt::INV_PI, r.alb[1] * pt::INV_PI, r.alb[2] * pt::INV_PI};
  return o;
}

__device__ inline void build_row_fast(const float* feat, const CacheVertex& r, V3 wi,
                                      const double* sh_k, float* x) {
#pragma unroll
  for (int i = 0; i < 24; ++i) x[i] = feat[i];
  sh4_f32((float)wi.x, (float)wi.y, (float)wi.z, sh_k, x + 24);
  x[40] = (float)((r.ns[0] + 1.0) * 0.5);
  x[41] = (float)((r.ns[1] + 1.0) * 0.5);
  x[42] = (float)((r.ns[2] + 1.0) * 0.5);
  x[43] = (float)r.alb[0];
  x[44] = (float)r.alb[1];
  x[45] = (float)r.alb[2];
  x[46] = (float)r.rough;
  x[47] = 0.0f;
}

struct InferArgs {
  const CacheVertex* cv;
  const unsigned long long* counters;
  double* result;  // (n_samples * max_cv, 3)
  double* rowbuf;  // SIMT fallback only: per-row contributions (cap * R, 3)
  int rows_per_vertex;  // R = max(nc) + 1
  int verts_per_tile;   // S = 128 / R
  long long* dbg;       // optional phase timestamps (CTA 0, group 0, thread 0)
  const int32_t* w_unsafe;  // F16x2: a weight outside the fp16 range (every tile flagged)
  int32_t* fix;             // F16x2 range guard: [count, tile ids...] for k_infer_fix
  int ablate;               // tools only (NIRC_INFER_ABLATE): 1 = producers skip the
                            // row work, 2 = chains skip MMAs + epilogues (wrong results)
};

// Deferred vertex term from its rows' contributions (row k at rows[3k]):
// two-level / biased NIRC: T * (1/N_c) sum_k n(w_k) f cos/pdf in k order
// (cache_lc_s, kernels.py:424-448), minus T' * n(w_cont) for the residual
// (:593-601); NRC stop: T * n(wo) (:660-670).
__device__ inline void vertex_result(const CacheVertex& r, const double* rows, double* o) {
  if (r.nrc) {
    o[0] = r.T[0] * rows[0];
    o[1] = r.T[1] * rows[1];
    o[2] = r.T[2] * rows[2];
    return;
  }
  double sr = 0.0, sg = 0.0, sb = 0.0;
  for (int k = 0; k < r.ncq; ++k) {
    sr += rows[3 * k];
    sg += rows[3 * k + 1];
    sb += rows[3 * k + 2];
  }
  const double inv = 1.0 / r.ncq;
  o[0] = r.T[0] * (sr * inv);
  o[1] = r.T[1] * (sg * inv);
  o[2] = r.T[2] * (sb * inv);
  if (r.has_res) {
    o[0] -= r.Tp[0] * rows[3 * r.ncq];
    o[1] -= r.Tp[1] * rows[3 * r.ncq + 1];
    o[2] -= r.Tp[2] * rows[3 * r.ncq + 2];
  }
}

constexpr int kMaxVertsPerTile = 64;

template <class P, int NG>
__global__ void __launch_bounds__(NG * 128, 1)
    k_infer_tc(nirc_spec_t sp, tc::TcNet net, tc::TcSmem L, const float* __restrict__ theta,
               const uint8_t* __restrict__ wimg, const float* __restrict__ bias_g, InferArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t tmem_base;
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
  // per-group extra shared memory: surface features + row contributions
  uint8_t* extra = smem + L.a_off + NG * L.abuf_bytes;
  const int R = a.rows_per_vertex, S = a.verts_per_tile;
  double* s_con = reinterpret_cast<double*>(extra) + group * 128 * 3;
  float* s_feat = reinterpret_cast<float*>(extra + NG * 128 * 3 * 8) + group * S * 24;
  CacheVertex* s_cv = reinterpret_cast<CacheVertex*>(extra + NG * 128 * 3 * 8 + NG * S * 24 * 4 +
                                                     ((NG * S * 24 * 4) & 8)) + group * S;
  const uint32_t T = 1u << sp.table_log2;
  const int64_t nverts = (int64_t)a.counters[0];
  const int64_t ntiles = (nverts + S - 1) / S;
  uint32_t phase = 0;
  const bool probe = a.dbg && blockIdx.x == 0 && threadIdx.x == 0;
  __shared__ int s_unsafe[NG];
  if (tg == 0) s_unsafe[group] = 0;
  const bool all_unsafe = kTS && *a.w_unsafe != 0;
  int it = 0;
  for (int64_t tile = (int64_t)blockIdx.x * NG + group; tile < ntiles;
       tile += (int64_t)gridDim.x * NG, ++it) {
    const int64_t v0 = tile * S;
    long long* pb = (probe && it < 32) ? a.dbg + it * 64 : nullptr;
    if (pb) pb[0] = clock64();
    // 0) the tile's cache-vertex records -> shared memory (one coalesced copy)
    {
      const int nv = (int)((nverts - v0) < S ? (nverts - v0) : S);
      const double* src = reinterpret_cast<const double*>(a.cv + v0);
      double* dst = reinterpret_cast<double*>(s_cv);
      const int words = nv * (int)(sizeof(CacheVertex) / 8);
      for (int i = tg; i < words; i += tc::kGroupThreads) dst[i] = src[i];
    }
    tc::named_bar_sync(1 + group, tc::kGroupThreads);
    // 1) shared surface encoding: one thread per (vertex, level)
    for (int item = tg; item < S * 12; item += tc::kGroupThreads) {
      const int j = item / 12, lvl = item % 12;
      const int64_t vid = v0 + j;
      if (vid < nverts) {
        const CacheVertex& r = s_cv[j];
        const float ux = norm_coord(r.pos[0], sp.bb_min[0], sp.bb_inv[0]);
        const float uy = norm_coord(r.pos[1], sp.bb_min[1], sp.bb_inv[1]);
        const float uz = norm_coord(r.pos[2], sp.bb_min[2], sp.bb_inv[2]);
        const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
        const float2 f = level_features2(theta + (size_t)lvl * T * 2, c, T - 1u);
        s_feat[j * 24 + 2 * lvl] = f.x;
        s_feat[j * 24 + 2 * lvl + 1] = f.y;
      }
    }
    tc::named_bar_sync(1 + group, tc::kGroupThreads);
    if (pb) pb[1] = clock64();
    // 2) per-row direction sampling + SH straight into the A tile
    const int j = tg / R, k = tg % R;
    const int64_t vid = v0 + j;
    RowDir rd;
    rd.kind = 0;
    float x[48];
    if (j < S && vid < nverts) {
      const CacheVertex& r = s_cv[j];
      rd = row_direction_fast(r, k);
      build_row_fast(s_feat + j * 24, r, rd.wi, sp.sh_k, x);
    } else {
#pragma unroll
      for (int i = 0; i < 48; ++i) x[i] = 0.0f;
    }
    float y[4];
    if constexpr (kTS) {
      bool unsafe = all_unsafe || tc::f16_unsafe(x, 48);
      tc::write_a_row_ts<48>(tmem_d + 64 + lane_off, tmem_d + 96 + lane_off, x);
      if (pb) pb[2] = clock64();
      tc::run_chain_ts(net, s0 + L.w_off, s_bias, group, tg, tmem_d, mbar, phase, y, unsafe);
      // fp16 range guard: the tile is recomputed in fp32 by k_infer_fix
      if (__any_sync(0xffffffffu, unsafe && rd.kind != 0) && (tg & 31) == 0)
        atomicOr(&s_unsafe[group], 1);
    } else {
      tc::write_a_row<P, 48>(a_hi, a_lo, tg, x);
      if (pb) pb[2] = clock64();
      tc::run_chain<P>(net, s0 + L.w_off, s_bias, group, tg, a_hi, a_lo, tmem_d, mbar, phase, y,
                       pb ? pb + 5 : nullptr);
    }
    if (pb) pb[3] = clock64();
    // 3) MLMC combine: cache rows give n(w)*f*cos/pdf, the residual row n(w_cont)
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
    if (rd.kind == 1) {
      c0 = (double)y[0] * rd.f.x * rd.s;
      c1 = (double)y[1] * rd.f.y * rd.s;
      c2 = (double)y[2] * rd.f.z * rd.s;
    } else if (rd.kind >= 2) {  // residual row / NRC row: the prediction itself
      c0 = (double)y[0];
      c1 = (double)y[1];
      c2 = (double)y[2];
    }
    s_con[3 * tg] = c0;
    s_con[3 * tg + 1] = c1;
    s_con[3 * tg + 2] = c2;
    tc::named_bar_sync(1 + group, tc::kGroupThreads);
    if (tg < S && v0 + tg < nverts) {
      const CacheVertex& r = s_cv[tg];
      double o[3];
      vertex_result(r, s_con + 3 * (tg * R), o);
      a.result[3 * r.slot] = o[0];
      a.result[3 * r.slot + 1] = o[1];
      a.result[3 * r.slot + 2] = o[2];
    }
    if (kTS && tg == 0 && s_unsafe[group]) {
      s_unsafe[group] = 0;
      a.fix[1 + atomicAdd(a.fix, 1)] = (int32_t)tile;
    }
    tc::named_bar_sync(1 + group, tc::kGroupThreads);
    if (pb) pb[4] = clock64();
  }
  tc::tc_epilogue(tmem_base, NG, P::kId);
}

#include "infer_ws.cuh"

// fp16 range fix-up of k_infer_tc<F16x2>: recomputes every vertex of the
// flagged tiles (a.fix) with the fp32 twin -- same rows, same k-ordered
// combine -- and overwrites their results.  A no-op when nothing was flagged.
__global__ void __launch_bounds__(128) k_infer_fix(nirc_spec_t sp, const float* __restrict__ theta,
                                                   InferArgs a) {
  extern __shared__ float wsm[];
  __shared__ double s_con[128 * 3];
  const int cnt = a.fix[0];
  if (cnt == 0) return;
  const int np = (int)(sp.theta_len - sp.grid_len);
  for (int i = threadIdx.x; i < np; i += blockDim.x) wsm[i] = theta[sp.grid_len + i];
  __syncthreads();
  const int R = a.rows_per_vertex, S = a.verts_per_tile;
  const int64_t nverts = (int64_t)a.counters[0];
  const uint32_t T = 1u << sp.table_log2;
  const int tg = threadIdx.x;
  for (int e = blockIdx.x; e < cnt; e += gridDim.x) {
    const int64_t v0 = (int64_t)a.fix[1 + e] * S;
    const int j = tg / R, k = tg % R;
    const int64_t vid = v0 + j;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
    if (j < S && vid < nverts) {
      const CacheVertex& r = a.cv[vid];
      const RowDir rd = row_direction_fast(r, k);
      if (rd.kind != 0) {
        float feat[24];
        const float ux = norm_coord(r.pos[0], sp.bb_min[0], sp.bb_inv[0]);
        const float uy = norm_coord(r.pos[1], sp.bb_min[1], sp.bb_inv[1]);
        const float uz = norm_coord(r.pos[2], sp.bb_min[2], sp.bb_inv[2]);
        for (int lvl = 0; lvl < 12; ++lvl) {
          const float2 f = level_features2(theta + (size_t)lvl * T * 2,
                                           level_cell(ux, uy, uz, sp.res[lvl]), T - 1u);
          feat[2 * lvl] = f.x;
          feat[2 * lvl + 1] = f.y;
        }
        float x[64], b[64];
        build_row_fast(feat, r, rd.wi, sp.sh_k, x);
        simt_net_row(sp, wsm, x, b);
        if (rd.kind == 1) {
          c0 = (double)x[0] * rd.f.x * rd.s;
          c1 = (double)x[1] * rd.f.y * rd.s;
          c2 = (double)x[2] * rd.f.z * rd.s;
        } else {
          c0 = (double)x[0];
          c1 = (double)x[1];
          c2 = (double)x[2];
        }
      }
    }
    s_con[3 * tg] = c0;
    s_con[3 * tg + 1] = c1;
    s_con[3 * tg + 2] = c2;
    __syncthreads();
    if (tg < S && v0 + tg < nverts) {
      const CacheVertex& r = a.cv[v0 + tg];
      double o[3];
      vertex_result(r, s_con + 3 * (tg * R), o);
      a.result[3 * r.slot] = o[0];
      a.result[3 * r.slot + 1] = o[1];
      a.result[3 * r.slot + 2] = o[2];
    }
    __syncthreads();
  }
}

// Generic-shape fallback of the same stage (any NetSpec): one thread per
// row, weights in shared memory, fp32 SIMT; rows are reduced per vertex by
// k_combine_rows in the same k order.
__global__ void k_infer_simt(nirc_spec_t sp, const float* __restrict__ theta, InferArgs a) {
  extern __shared__ float wsm[];
  const int np = (int)(sp.theta_len - sp.grid_len);
  for (int i = threadIdx.x; i < np; i += blockDim.x) wsm[i] = theta[sp.grid_len + i];
  __syncthreads();
  const int64_t nverts = (int64_t)a.counters[0];
  const int R = a.rows_per_vertex;
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t vid = row / R;
  const int k = (int)(row % R);
  if (vid >= nverts) return;
  const CacheVertex& r = a.cv[vid];
  const RowDir rd = row_direction(r, k);
  double* out = a.rowbuf + 3 * row;
  out[0] = out[1] = out[2] = 0.0;
  if (rd.kind == 0) return;
  float act[2][136];
  float* x = act[0];
  const int F = sp.feats;
  const uint32_t T = 1u << sp.table_log2;
  const float ux = norm_coord(r.pos[0], sp.bb_min[0], sp.bb_inv[0]);
  const float uy = norm_coord(r.pos[1], sp.bb_min[1], sp.bb_inv[1]);
  const float uz = norm_coord(r.pos[2], sp.bb_min[2], sp.bb_inv[2]);
  for (int lvl = 0; lvl < sp.levels; ++lvl) {
    const LevelCell c = level_cell(ux, uy, uz, sp.res[lvl]);
    for (int f = 0; f < F; ++f) {
      float acc = 0.0f;
      for (int cc = 0; cc < 8; ++cc)
        acc = __fadd_rn(acc, __fmul_rn(corner_weight(c, cc),
                                       theta[((size_t)lvl * T + corner_hash(c, cc, T - 1u)) * F + f]));
      x[lvl * F + f] = acc;
    }
  }
  const int g = sp.levels * F;
  sh_eval<false>(rd.wi.x, rd.wi.y, rd.wi.z, sp.bands, sp.sh_k,
                 [&](int i, double v) { x[g + i] = __double2float_rn(v); });
  const int a0 = g + sp.bands * sp.bands;
  for (int i = 0; i < 3; ++i) x[a0 + i] = __double2float_rn((r.ns[i] + 1.0) * 0.5);
  for (int i = 0; i < 3; ++i) x[a0 + 3 + i] = __double2float_rn(r.alb[i]);
  x[a0 + 6] = __double2float_rn(r.rough);
  int cur = 0;
  for (int l = 0; l < sp.n_layers; ++l) {
    const int din = sp.dims[l], dout = sp.dims[l + 1];
    const float* w = wsm + (sp.w_off[l] - sp.grid_len);
    const float* bias = wsm + (sp.b_off[l] - sp.grid_len);
    const bool last = l == sp.n_layers - 1;
    for (int jj = 0; jj < dout; ++jj) {
      float acc = 0.0f;
      for (int i = 0; i < din; ++i) acc = fmaf(act[cur][i], w[jj * din + i], acc);
      const float z = acc + bias[jj];
      act[1 - cur][jj] =
          (!last || sp.out_act == 0) ? (z > 0.0f ? z : 0.0f) : 1.0f / (1.0f + expf(-z));
    }
    cur = 1 - cur;
  }
  const float* y = act[cur];
  if (rd.kind == 1) {
    out[0] = (double)y[0] * rd.f.x * rd.s;
    out[1] = (double)y[1] * rd.f.y * rd.s;
    out[2] = (double)y[2] * rd.f.z * rd.s;
  } else {
    out[0] = y[0];
    out[1] = y[1];
    out[2] = y[2];
  }
}

__global__ void k_combine_rows(InferArgs a) {
  const int64_t vid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vid >= (int64_t)a.counters[0]) return;
  const CacheVertex& r = a.cv[vid];
  const int R = a.rows_per_vertex;
  double o[3];
  vertex_result(r, a.rowbuf + 3 * vid * R, o);
  a.result[3 * r.slot] = o[0];
  a.result[3 * r.slot + 1] = o[1];
  a.result[3 * r.slot + 2] = o[2];
}

// render_kernel accumulation (kernels.py:753-759): per pixel, samples in
// order s = 0..spp-1; r = PT sum + sum over cache vertices (cu order).
__global__ void k_accumulate(nirc_render_cfg_t cfg, const double* __restrict__ acc,
                             const int32_t* __restrict__ term, const double* __restrict__ res,
                             int use_res, double* __restrict__ img, double* __restrict__ img2,
                             double* __restrict__ tsum) {
  const int W = cfg.width;
  const int64_t lp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (lp >= (int64_t)(cfg.row1 - cfg.row0) * W) return;
  const int64_t pix = (int64_t)cfg.row0 * W + lp;
  double i0 = img[3 * pix], i1 = img[3 * pix + 1], i2 = img[3 * pix + 2];
  double q0 = img2[3 * pix], q1 = img2[3 * pix + 1], q2 = img2[3 * pix + 2];
  double ts = tsum[pix];
  for (int s = 0; s < cfg.spp; ++s) {
    const int64_t sid = lp * cfg.spp + s;
    double r = acc[3 * sid], g = acc[3 * sid + 1], b = acc[3 * sid + 2];
    if (use_res) {
      for (int c = 0; c < cfg.max_cv; ++c) {
        const double* q = res + 3 * (sid * cfg.max_cv + c);
        r += q[0];
        g += q[1];
        b += q[2];
      }
    }
    i0 += r;
    i1 += g;
    i2 += b;
    q0 += r * r;
    q1 += g * g;
    q2 += b * b;
    ts += term[sid];
  }
  img[3 * pix] = i0;
  img[3 * pix + 1] = i1;
  img[3 * pix + 2] = i2;
  img2[3 * pix] = q0;
  img2[3 * pix + 1] = q1;
  img2[3 * pix + 2] = q2;
  tsum[pix] = ts;
}

// Exclusive scan of per-path record counts (one CTA; count is ~5e4).
// Exclusive scan of per-path record counts in two levels: k_scan_local
// scans each 1024-path chunk (warp shuffles) and emits the chunk totals,
// k_scan_top scans the totals (one warp); the compaction adds the chunk
// prefix.  Every level is coalesced and fully parallel.
constexpr int kScanChunk = 1024;

__global__ void k_scan_local(const int32_t* __restrict__ cnt, int64_t n,
                             int64_t* __restrict__ off, int64_t* __restrict__ chunk_sum) {
  __shared__ int32_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t i = (int64_t)blockIdx.x * kScanChunk + tid;
  const int32_t v = i < n ? cnt[i] : 0;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int32_t z = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    wsum[lane] = z;
  }
  __syncthreads();
  const int32_t incl = x + (w > 0 ? wsum[w - 1] : 0);
  if (i < n) off[i] = incl - v;
  if (tid == kScanChunk - 1) chunk_sum[blockIdx.x] = incl;
}

__global__ void k_scan_top(int64_t* __restrict__ chunk_sum, int64_t nchunks,
                           int64_t* __restrict__ total) {
  const int lane = threadIdx.x;
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nchunks; b0 += 32) {
    const int64_t b = b0 + lane;
    const int64_t v = b < nchunks ? chunk_sum[b] : 0;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (b < nchunks) chunk_sum[b] = carry + x - v;  // exclusive chunk prefix
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) *total = carry;
}

static inline int scan_counts(const int32_t* cnt, int64_t n, int64_t* off, int64_t* chunk,
                              int64_t* total, cudaStream_t s) {
  const int64_t nchunks = (n + kScanChunk - 1) / kScanChunk;
  k_scan_local<<<(int)nchunks, kScanChunk, 0, s>>>(cnt, n, off, chunk);
  k_scan_top<<<1, 32, 0, s>>>(chunk, nchunks, total);
  return cudaGetLastError() == cudaSuccess ? NIRC_OK : NIRC_E_CUDA;
}

// One warp per path: lanes take the path's vertices (<= 64, two rounds),
// ballot the kept ones and write them in vertex order at off[p] + rank --
// the reference's (path, vertex) row order with coalesced stores.
__global__ void k_compact_records(Stage st, const int64_t* __restrict__ off,
                                  const int64_t* __restrict__ chunk_pre,
                                  nirc_records_out_t out) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= st.count) return;
  int64_t o = off[p] + chunk_pre[p / kScanChunk];
  const int n = st.nvert[p];
  for (int v0 = 0; v0 < n; v0 += 32) {
    const int v = v0 + lane;
    const int64_t at = (int64_t)v * st.count + p;
    const bool keep = v < n && st.keep[at];
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int64_t q = o + __popc(m & ((1u << lane) - 1u));
      if (q < out.cap) {
        for (int c = 0; c < 3; ++c) {
          out.pos[3 * q + c] = st.pos[3 * at + c];
          out.ns[3 * q + c] = st.ns[3 * at + c];
          out.alb[3 * q + c] = st.alb[3 * at + c];
          out.dirs[3 * q + c] = st.wi[3 * at + c];
          out.target[3 * q + c] = st.tgt[3 * at + c];
        }
        out.rough[q] = st.rough[at];
        out.pdf[q] = st.pdf[at];
      }
    }
    o += __popc(m);
  }
}

long long* g_infer_probe = nullptr;  // set by nirc_debug_infer_probe (tools only)

// Optional per-stage timing of the render launch set (nirc_stage_timing):
// CUDA events on the launch stream around the tracer, the fused inference
// (+ its fp16 fix-up) and the accumulation of the last timed render.
struct StageTimer {
  bool on = false;
  bool created = false;
  cudaEvent_t ev[4];
};
StageTimer g_stage;
static void stage_mark(int i, cudaStream_t s) {
  if (g_stage.on) cudaEventRecord(g_stage.ev[i], s);
}

bool default_layout(const nirc_spec_t& sp) {
  return sp.levels == 12 && sp.feats == 2 && sp.bands == 4 && sp.in_dim == 47;
}

}  // namespace nirc

using namespace nirc;

namespace {
size_t aup(size_t x) { return (x + 255) & ~(size_t)255; }

struct RenderWs {
  double *acc, *result, *rowbuf;
  int32_t* term;
  int32_t* fix;  // F16x2 range-guard tile list (count + ids)
  CacheVertex* cv;
  unsigned long long* counters;
  size_t bytes;
};

// Inference rows per deferred vertex: N_c + the residual (two-level),
// nbias (biased NIRC stop), 1 (NRC stop).
int rows_per_vertex(const nirc_render_cfg_t& c) {
  if (c.mode == 4) return 1;
  if (c.mode >= 2) return c.nbias;
  int m = 0;
  for (int i = 0; i < c.max_cv && i < 8; ++i) m = c.nc[i] > m ? c.nc[i] : m;
  return m + 1;
}

RenderWs carve_render(const nirc_render_cfg_t& c, void* base) {
  RenderWs w{};
  char* p = reinterpret_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t b) {
    char* r = p ? p + off : nullptr;
    off += aup(b);
    return r;
  };
  const int64_t ns = (int64_t)(c.row1 - c.row0) * c.width * c.spp;
  const int64_t ncv = c.mode >= 1 && c.cache_on ? ns * c.max_cv : 0;
  w.acc = (double*)take(ns * 24);
  w.term = (int32_t*)take(ns * 4);
  w.result = (double*)take(ncv * 24 + 24);
  w.cv = (CacheVertex*)take(ncv * sizeof(CacheVertex) + 16);
  w.counters = (unsigned long long*)take(64);
  w.fix = (int32_t*)take((ncv + 2) * 4);
  w.rowbuf = (double*)take(0);  // sized on demand for the SIMT fallback
  w.bytes = off;
  return w;
}
}  // namespace

namespace {
Stage carve_stage(int64_t count, void* base, size_t* bytes) {
  Stage st{};
  char* p = reinterpret_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t b) {
    char* r = p ? p + off : nullptr;
    off += aup(b);
    return r;
  };
  const int64_t V = (int64_t)pt::MAXB * count;
  st.pos = (double*)take(V * 24);
  st.ns = (double*)take(V * 24);
  st.alb = (double*)take(V * 24);
  st.rough = (double*)take(V * 8);
  st.wi = (double*)take(V * 24);
  st.pdf = (double*)take(V * 8);
  st.tgt = (double*)take(V * 24);
  st.keep = (uint8_t*)take(V);
  st.nrec = (int32_t*)take(count * 4);
  st.nvert = (int32_t*)take(count * 4);
  take(count * 8);  // offsets
  take(((count + kScanChunk - 1) / kScanChunk) * 8 + 8);  // chunk prefixes
  st.count = count;
  *bytes = off;
  return st;
}
}  // namespace

extern "C" int64_t nirc_render_workspace_bytes(const nirc_render_cfg_t* cfg) {
  return (int64_t)carve_render(*cfg, nullptr).bytes;
}

static int check_render_cfg(const nirc_render_cfg_t& c) {
  if (c.mode < 0 || c.mode > 4) {
    set_last_error("unknown render mode %d", c.mode);
    return NIRC_E_UNSUPPORTED;
  }
  if (c.mode >= 2 && (c.nbias < 1 || c.nbias > 28 || !(c.sph_c > 0.0) || c.max_cv < 1)) {
    set_last_error("biased modes need 1 <= nbias <= 28, sph_c > 0 and max_cv >= 1");
    return NIRC_E_CONFIG;
  }
  if (c.spp < 1 || c.row0 < 0 || c.row1 > c.height || c.row0 >= c.row1 || c.max_cv > 8) {
    set_last_error("bad render configuration");
    return NIRC_E_CONFIG;
  }
  for (int i = 0; i < c.max_cv; ++i)
    if (c.nc[i] < 0 || c.nc[i] > 28) {
      set_last_error("nc entry outside 0..28");
      return NIRC_E_CONFIG;
    }
  return NIRC_OK;
}

// The frame pipeline: K5 trace (+ the training walks of `job`), fused
// inference/combine, accumulation.
static int render_impl(const nirc_scene_t* scene, const double* cam, const nirc_render_cfg_t& c,
                       const nirc_spec_t* spec, const float* theta, double* img, double* img2,
                       double* term, int64_t* queries_out, const RenderWs& w, const WalkJob& job,
                       cudaStream_t s) {
  const bool tl = c.mode >= 1 && c.cache_on;  // deferred cache vertices exist
  const int64_t ns = (int64_t)(c.row1 - c.row0) * c.width * c.spp;
  NIRC_CUDA_TRY(cudaMemsetAsync(w.counters, 0, 64, s));
  if (tl) NIRC_CUDA_TRY(cudaMemsetAsync(w.result, 0, ns * c.max_cv * 24, s));
  TraceOut to{w.acc, w.term, w.cv, w.counters};
  const size_t scene_bytes = pt::scene_smem_bytes(*scene);
  const size_t dyn = scene_bytes <= (size_t)pt::kSceneSmemBytes ? (scene_bytes + 15) & ~15ull : 0;
  auto launch_trace = [&](auto kern) -> int {
    int per_sm = 0;
    NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)kern,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       pt::kSceneSmemBytes));
    NIRC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, dyn));
    if (per_sm < 1) per_sm = 1;
    const int64_t tgrid_max = (ns + job.n + 127) / 128;
    const int64_t tgrid_pers = (int64_t)sm_count() * per_sm;
    kern<<<(int)(tgrid_max < tgrid_pers ? tgrid_max : tgrid_pers), 128, dyn, s>>>(*scene, cam, c,
                                                                                  to, job);
    return NIRC_OK;
  };
  int tst;
  stage_mark(0, s);
  constexpr int kS = NIRC_TRACE_MINB, kB = NIRC_TRACE_MINB_BVH;
  const bool bvh = scene->bvh_packed != nullptr;  // general scene: packed BVH traversal
  if (c.mode >= 2 && bvh)
    tst = job.n > 0 ? launch_trace(k_trace<true, true, kB>)
                    : launch_trace(k_trace<true, false, kB>);
  else if (c.mode >= 2)
    tst = job.n > 0 ? launch_trace(k_trace<true, true, kS>)
                    : launch_trace(k_trace<true, false, kS>);
  else if (bvh)
    tst = job.n > 0 ? launch_trace(k_trace<false, true, kB>)
                    : launch_trace(k_trace<false, false, kB>);
  else
    tst = job.n > 0 ? launch_trace(k_trace<false, true, kS>)
                    : launch_trace(k_trace<false, false, kS>);
  if (tst) return tst;
  NIRC_LAUNCH_CHECK("k_trace");
  stage_mark(1, s);
  if (tl) {
    if (!spec || !theta) return NIRC_E_CONFIG;
    const int R = rows_per_vertex(c);
    InferArgs a{w.cv, w.counters, w.result, nullptr, R, 128 / R, g_infer_probe, nullptr, w.fix, 0};
    if (const char* e = getenv("NIRC_INFER_ABLATE")) a.ablate = atoi(e);
    const int prec = c.precision == 2 ? tc::PrecF16x2::kId : tc::PrecTF32x3::kId;
    tc::TcNet net;
    const bool tc_ok =
        c.precision != 1 && default_layout(*spec) && tc::tc_net_for(*spec, &net, prec);
    const uint32_t extra =
        (uint32_t)(128 * 3 * 8 + a.verts_per_tile * 24 * 4 + 16 + a.verts_per_tile * sizeof(CacheVertex));
    const int ng = tc_ok ? tc_groups_for(net, extra) : 0;

    AsyncBuf wbuf(s);
    if (ng > 0) {
      PackedNet pn;
      int st = pack_weights(*spec, net, theta, s, wbuf, &pn);
      if (st) return st;
      a.w_unsafe = pn.unsafe;
      const bool ts = prec == tc::PrecF16x2::kId;
      const size_t fix_sm = (size_t)(spec->theta_len - spec->grid_len) * 4;
      if (ts) NIRC_CUDA_TRY(cudaMemsetAsync(w.fix, 0, 4, s));
      const tc::TcSmem L = tc::tc_smem_layout(net, ng, ng * extra);
      const int grid = sm_count();
      auto launch = [&](auto kern, int threads) -> int {
        NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)kern,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)L.total));
        kern<<<grid, threads, L.total, s>>>(*spec, net, L, theta, pn.img, pn.bias, a);
        return NIRC_OK;
      };
      // warp-specialised kernel (infer_ws.cuh) where its shared-memory plan fits
      int np_ws = 2;
      if (const char* e = getenv("NIRC_INFER_NP")) np_ws = atoi(e);  // 0 = k_infer_tc
      if (np_ws > 2) np_ws = 2;
      ws::Layout WL = ws::layout(net, a.verts_per_tile, np_ws > 0 ? np_ws : 1);
      for (int q = 0; q < 28; ++q) WL.shk[q] = (float)spec->sh_k[q];
      bool ws_shape = net.K[0] == 48 && net.N[0] == 64 && net.N[net.nl - 1] == 16;
      for (int l = 1; l < net.nl; ++l) ws_shape = ws_shape && net.K[l] == 64;
      for (int l = 0; l < net.nl - 1; ++l) ws_shape = ws_shape && net.N[l] == 64;
      const bool use_ws = prec == tc::PrecF16x2::kId && np_ws > 0 && ws_shape &&
                          WL.total <= 227u * 1024u - 256u;
      auto launch_ws = [&](auto kern, int threads, int chain_regs, int prod_regs) -> int {
        // setmaxnreg only redistributes the registers the CTA was launched
        // with: check the split against the compiled allocation
        cudaFuncAttributes fa;
        NIRC_CUDA_TRY(cudaFuncGetAttributes(&fa, (const void*)kern));
        const int npw = threads / 128 - ws::kChainGroups;
        if (chain_regs > 0 &&
            fa.numRegs * threads < ws::kChainGroups * 128 * chain_regs + npw * 128 * prod_regs) {
          set_last_error("k_infer_ws register split exceeds its allocation (%d x %d)",
                         fa.numRegs, threads);
          return NIRC_E_UNSUPPORTED;
        }
        NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)kern,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)WL.total));
        kern<<<grid, threads, WL.total, s>>>(*spec, net, WL, theta, pn.img, pn.bias, a);
        return NIRC_OK;
      };
#define NIRC_WS_LAUNCH(NPV, PROBE)                                                         \
  launch_ws(k_infer_ws<NPV, PROBE>, (ws::kChainGroups + NPV) * 128, ws::kChainRegs<NPV>, \
            ws::kProdRegs<NPV>)
      if (use_ws && a.dbg) {  // phase stamps (tools/infer_ab.py)
        if (np_ws == 1) st = NIRC_WS_LAUNCH(1, true);
        else st = NIRC_WS_LAUNCH(2, true);
      } else if (use_ws) {
        if (np_ws == 1) st = NIRC_WS_LAUNCH(1, false);
        else st = NIRC_WS_LAUNCH(2, false);
#undef NIRC_WS_LAUNCH
      } else if (prec == tc::PrecF16x2::kId) {
        if (ng == 4) st = launch(k_infer_tc<tc::PrecF16x2, 4>, 512);
        else if (ng == 3) st = launch(k_infer_tc<tc::PrecF16x2, 3>, 384);
        else if (ng == 2) st = launch(k_infer_tc<tc::PrecF16x2, 2>, 256);
        else st = launch(k_infer_tc<tc::PrecF16x2, 1>, 128);
      } else {
        if (ng == 2) st = launch(k_infer_tc<tc::PrecTF32x3, 2>, 256);
        else st = launch(k_infer_tc<tc::PrecTF32x3, 1>, 128);
      }
      if (st) return st;
      NIRC_LAUNCH_CHECK("k_infer_tc");
      if (ts) {
        NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)k_infer_fix,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)fix_sm));
        k_infer_fix<<<sm_count(), 128, fix_sm, s>>>(*spec, theta, a);
        NIRC_LAUNCH_CHECK("k_infer_fix");
      }
    }
    if (ng == 0) {
      // generic layouts: SIMT rows into a row buffer, then per-vertex combine
      const int64_t cap = ns * c.max_cv;
      AsyncBuf rowbuf(s);
      NIRC_CUDA_TRY(rowbuf.alloc((size_t)cap * R * 24 + 24));
      a.rowbuf = static_cast<double*>(rowbuf.p);
      const size_t sm = (size_t)(spec->theta_len - spec->grid_len) * 4;
      NIRC_CUDA_TRY(cudaFuncSetAttribute((const void*)k_infer_simt,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k_infer_simt<<<(int)((cap * R + 127) / 128), 128, sm, s>>>(*spec, theta, a);
      NIRC_LAUNCH_CHECK("k_infer_simt");
      k_combine_rows<<<(int)((cap + 127) / 128), 128, 0, s>>>(a);
      NIRC_LAUNCH_CHECK("k_combine_rows");
    }
  }
  stage_mark(2, s);
  const int64_t npix = (int64_t)(c.row1 - c.row0) * c.width;
  k_accumulate<<<(int)((npix + 127) / 128), 128, 0, s>>>(c, w.acc, w.term, w.result, tl ? 1 : 0,
                                                        img, img2, term);
  NIRC_LAUNCH_CHECK("k_accumulate");
  stage_mark(3, s);
  if (queries_out)
    NIRC_CUDA_TRY(cudaMemcpyAsync(queries_out, w.counters + 1, 8, cudaMemcpyDeviceToDevice, s));
  return NIRC_OK;
}

extern "C" int nirc_render(const nirc_scene_t* scene, const double* cam,
                           const nirc_render_cfg_t* cfg, const nirc_spec_t* spec,
                           const float* theta, double* img, double* img2, double* term,
                           int64_t* queries_out, void* workspace, int64_t workspace_bytes,
                           void* stream) {
  int st = check_render_cfg(*cfg);
  if (st) return st;
  RenderWs w = carve_render(*cfg, workspace);
  if ((int64_t)w.bytes > workspace_bytes) {
    set_last_error("render workspace too small");
    return NIRC_E_CONFIG;
  }
  WalkJob job{};
  return render_impl(scene, cam, *cfg, spec, theta, img, img2, term, queries_out, w, job,
                     reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int64_t nirc_render_collect_workspace_bytes(const nirc_render_cfg_t* cfg,
                                                       int64_t count) {
  size_t b = 0;
  carve_stage(count, nullptr, &b);
  return (int64_t)(aup(carve_render(*cfg, nullptr).bytes) + b);
}

extern "C" int nirc_render_collect(const nirc_scene_t* scene, const double* cam,
                                   const nirc_render_cfg_t* cfg, const nirc_spec_t* spec,
                                   const float* theta, double* img, double* img2, double* term,
                                   int64_t* queries_out, uint64_t train_seed,
                                   uint64_t train_frame, int64_t path0, int64_t count,
                                   int32_t kind, const nirc_records_out_t* out, int64_t* n_out,
                                   void* workspace, int64_t workspace_bytes, void* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int st = check_render_cfg(*cfg);
  if (st) return st;
  if (count <= 0 || path0 < 0) {
    set_last_error("count must be positive and path0 non-negative");
    return NIRC_E_CONFIG;
  }
  if (kind < 0 || kind > 4) {
    set_last_error("unknown record kind %d", kind);
    return NIRC_E_CONFIG;
  }
  RenderWs w = carve_render(*cfg, workspace);
  size_t sb = 0;
  Stage stg = carve_stage(count, reinterpret_cast<char*>(workspace) + aup(w.bytes), &sb);
  if ((int64_t)(aup(w.bytes) + sb) > workspace_bytes) {
    set_last_error("render+collect workspace too small");
    return NIRC_E_CONFIG;
  }
  stg.path0 = path0;
  stg.kind = kind;
  WalkJob job{stg, train_seed, train_frame, count};
  if ((st = render_impl(scene, cam, *cfg, spec, theta, img, img2, term, queries_out, w, job, s)))
    return st;
  int64_t* off = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(stg.nvert) + aup(count * 4));
  int64_t* chunk = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(off) + aup(count * 8));
  if ((st = scan_counts(stg.nrec, count, off, chunk, n_out, s))) return st;
  NIRC_LAUNCH_CHECK("k_scan_*");
  k_compact_records<<<(int)((count * 32 + 255) / 256), 256, 0, s>>>(stg, off, chunk, *out);
  NIRC_LAUNCH_CHECK("k_compact_records");
  return NIRC_OK;
}


extern "C" int64_t nirc_collect_workspace_bytes(int64_t count) {
  size_t b = 0;
  carve_stage(count, nullptr, &b);
  return (int64_t)b;
}

extern "C" int nirc_collect_range(const nirc_scene_t* scene, const double* cam, uint64_t seed,
                                  uint64_t frame, int64_t path0, int64_t count, int32_t kind,
                                  const nirc_records_out_t* out, int64_t* n_out, void* workspace,
                                  int64_t workspace_bytes, void* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (count <= 0 || path0 < 0) {
    set_last_error("count must be positive and path0 non-negative");
    return NIRC_E_CONFIG;
  }
  if (kind < 0 || kind > 4) {
    set_last_error("unknown record kind %d", kind);
    return NIRC_E_CONFIG;
  }
  size_t need = 0;
  Stage st = carve_stage(count, workspace, &need);
  if ((int64_t)need > workspace_bytes) {
    set_last_error("collect workspace too small");
    return NIRC_E_CONFIG;
  }
  st.path0 = path0;
  st.kind = kind;
  int64_t* off = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(st.nvert) + aup(count * 4));
  int64_t* chunk = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(off) + aup(count * 8));
  k_walk_record<<<(int)((count + 63) / 64), 64, 0, s>>>(*scene, cam, seed, frame, st);
  NIRC_LAUNCH_CHECK("k_walk_record");
  if (scan_counts(st.nrec, count, off, chunk, n_out, s)) return NIRC_E_CUDA;
  NIRC_LAUNCH_CHECK("k_scan_*");
  k_compact_records<<<(int)((count * 32 + 255) / 256), 256, 0, s>>>(st, off, chunk, *out);
  NIRC_LAUNCH_CHECK("k_compact_records");
  return NIRC_OK;
}

extern "C" int nirc_collect(const nirc_scene_t* scene, const double* cam, uint64_t seed,
                            uint64_t frame, int64_t count, int32_t kind,
                            const nirc_records_out_t* out, int64_t* n_out, void* workspace,
                            int64_t workspace_bytes, void* stream) {
  return nirc_collect_range(scene, cam, seed, frame, 0, count, kind, out, n_out, workspace,
                            workspace_bytes, stream);
}

// Tools only (not part of include/nirc_b200.h): route per-phase clock64()
// stamps of CTA 0 / group 0 of the next k_infer_tc launches into `buf`
// (device, >= 64*8 int64), or disable with NULL.
extern "C" void nirc_debug_infer_probe(long long* buf) { nirc::g_infer_probe = buf; }

extern "C" int nirc_stage_timing(int32_t on) {
  if (on && !g_stage.created) {
    for (int i = 0; i < 4; ++i) NIRC_CUDA_TRY(cudaEventCreate(&g_stage.ev[i]));
    g_stage.created = true;
  }
  g_stage.on = on != 0;
  return NIRC_OK;
}

extern "C" int nirc_stage_times(float* ms, int32_t n) {
  if (!g_stage.created) {
    set_last_error("stage timing was never enabled");
    return NIRC_E_CONFIG;
  }
  NIRC_CUDA_TRY(cudaEventSynchronize(g_stage.ev[3]));
  for (int i = 0; i < 3 && i < n; ++i)
    NIRC_CUDA_TRY(cudaEventElapsedTime(&ms[i], g_stage.ev[i], g_stage.ev[i + 1]));
  return NIRC_OK;
}

// Tools/tests only (not part of include/nirc_b200.h): the fp32 pre-filtered
// triangle scan against the plain f64 scan on n random rays through the
// scene (origins inside its box, random directions; a third of the rays aimed
// exactly at triangle vertices / edge points; occlusion windows at the hit
// distance and one ulp either side).  counts[0] = mismatches (hit kind,
// primitive or t bit pattern, or occlusion boolean), counts[1] = hits.
namespace nirc {
__global__ void k_debug_intersect(nirc_scene_t scn, int64_t n, uint64_t seed,
                                  unsigned long long* counts, double* detail, int aim) {
  __shared__ __align__(16) unsigned char scene_sm[pt::kSceneSmemBytes];
  pt::stage_scene(scn, scene_sm);
  nirc_scene_t plain = scn;  // the reference-order f64 scan / stack walk
  plain.tri_f32 = nullptr;
  plain.bvh_packed = nullptr;
  plain.prim_packed = nullptr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = stream_key(seed, 77, 0, (uint64_t)i, 0);
    auto U = [&](int dim) { return rand_uniform(key, dim); };
    const double ext = 1.0 / scn.bbox_inv_ext[0];
    V3 o = {scn.bbox_min[0] + U(0) / scn.bbox_inv_ext[0], scn.bbox_min[1] + U(1) / scn.bbox_inv_ext[1],
            scn.bbox_min[2] + U(2) / scn.bbox_inv_ext[2]};
    V3 d = {U(3) - 0.5, U(4) - 0.5, U(5) - 0.5};
    if (aim && U(6) < 0.33 && scn.n_tri > 0) {  // aim at a vertex or an edge point of a triangle
      const int t = (int)(U(7) * scn.n_tri) % scn.n_tri;
      const V3 v0 = pt::ld3(scn.tri_v0, t), e1 = pt::ld3(scn.tri_e1, t), e2 = pt::ld3(scn.tri_e2, t);
      const double a = U(8) < 0.5 ? 0.0 : U(9), b = U(10) < 0.5 ? 0.0 : 1.0 - a;
      const V3 tp = {v0.x + a * e1.x + b * e2.x, v0.y + a * e1.y + b * e2.y,
                     v0.z + a * e1.z + b * e2.z};
      d = {tp.x - o.x, tp.y - o.y, tp.z - o.z};
    }
    const double dl = sqrt(d.x * d.x + d.y * d.y + d.z * d.z);
    if (!(dl > 0.0)) continue;
    d = {d.x / dl, d.y / dl, d.z / dl};
    (void)ext;
    const pt::Hit a = pt::intersect<false>(scn, o, d, pt::T_FAR);
    const pt::Hit b = pt::intersect<false>(plain, o, d, pt::T_FAR);
    // counts: [0] nearest-hit mismatches, [1] hits, [2] occlusion mismatches
    // at t_max = t and one ulp either side of the hit
    bool bad = a.kind != b.kind || a.prim != b.prim ||
               (a.kind >= 0 && __double_as_longlong(a.t) != __double_as_longlong(b.t));
    bool bad_occ = false;
    if (b.kind >= 0) {
      atomicAdd(counts + 1, 1ull);
      const double tm[3] = {b.t, nextafter(b.t, 0.0), nextafter(b.t, 1e300)};
      for (int q = 0; q < 3; ++q)
        bad_occ |= pt::occluded(scn, o, d, tm[q]) != pt::occluded(plain, o, d, tm[q]);
    }
    if (bad_occ) atomicAdd(counts + 2, 1ull);
    if (bad || bad_occ) {
      const unsigned long long m = bad ? atomicAdd(counts, 1ull) : 16ull;
      if (detail && m < 16) {  // first mismatches: ray, both hits, occlusion answers
        double* q = detail + 16 * m;
        q[0] = o.x; q[1] = o.y; q[2] = o.z; q[3] = d.x; q[4] = d.y; q[5] = d.z;
        q[6] = a.kind; q[7] = a.prim; q[8] = a.t; q[9] = b.kind; q[10] = b.prim; q[11] = b.t;
        if (b.kind >= 0) {
          q[12] = pt::occluded(scn, o, d, b.t);
          q[13] = pt::occluded(plain, o, d, b.t);
          q[14] = pt::occluded(scn, o, d, nextafter(b.t, 1e300));
          q[15] = pt::occluded(plain, o, d, nextafter(b.t, 1e300));
        }
      }
    }
  }
}
}  // namespace nirc

extern "C" int nirc_debug_intersect_check(const nirc_scene_t* scene, int64_t n, uint64_t seed,
                                          unsigned long long* counts) {
  nirc::k_debug_intersect<<<148 * 4, 128>>>(*scene, n, seed, counts, nullptr, 1);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

extern "C" int nirc_debug_intersect_detail(const nirc_scene_t* scene, int64_t n, uint64_t seed,
                                           unsigned long long* counts, double* detail,
                                           int32_t aim) {
  nirc::k_debug_intersect<<<148 * 4, 128>>>(*scene, n, seed, counts, detail, aim);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

// ---------------------------------------------------------------------
// Per-interaction helpers of the drop-in API (estimators.py:240-320,
// caches.py:134-155): BSDF draws at one surface, repeated incident-radiance
// walks along one ray, one path-traced pixel sample.
namespace nirc {

// estimators.py _surface_dirs: n draws (u pairs) of bsdf_sample at one
// interaction; delta / pdf <= 0 / below-horizon draws give zero rows.
__global__ void k_surface_samples(nirc_scene_t scn, V3 ns, V3 wo, int mat, const double* u,
                                  int n, double* dirs, double* pdf, double* f, double* cosv) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int mkind = scn.mat_kind[mat];
  const V3 alb = pt::ld3(scn.mat_albedo, mat);
  const pt::BsdfSample b = pt::bsdf_sample(mkind, alb, scn.mat_rough[mat], ns, wo, u[2 * k],
                                           u[2 * k + 1]);
  double c = 0.0;
  bool ok = b.pdf > 0.0 && b.delta == 0;
  if (ok) {
    c = b.wi.x * ns.x + b.wi.y * ns.y + b.wi.z * ns.z;
    ok = c > 0.0;
  }
  dirs[3 * k] = ok ? b.wi.x : 0.0;
  dirs[3 * k + 1] = ok ? b.wi.y : 0.0;
  dirs[3 * k + 2] = ok ? b.wi.z : 0.0;
  pdf[k] = ok ? b.pdf : 0.0;
  f[3 * k] = ok ? b.f.x : 0.0;
  f[3 * k + 1] = ok ? b.f.y : 0.0;
  f[3 * k + 2] = ok ? b.f.z : 0.0;
  cosv[k] = ok ? c : 0.0;
}

// walk_record's return value (kernels.py:249-286): runs the walk w (key,
// ray, prev_pdf / prev_ns already set) to its end and sweeps it backwards;
// res[1:4] -> out, res[4:7] -> out_full.
__device__ inline void walk_incident(const nirc_scene_t& scn, WalkLane& w, const Stage& st,
                                     double* out, double* out_full) {
  w.v = 0;
  w.esc = 0;
  for (int c = 0; c < 3; ++c) w.env_m[c] = w.env_r[c] = 0.0;
  while (!walk_vertex(scn, w, st)) {
  }
  walk_finish(w, st);
  const int n = w.v;
  if (n == 0) {
    for (int c = 0; c < 3; ++c) {
      out[c] = w.env_m[c];
      out_full[c] = w.env_r[c];
    }
    return;
  }
  double l[3] = {0.0, 0.0, 0.0};
  for (int v = n - 1; v >= 0; --v) {
    double cc[3];
    for (int c = 0; c < 3; ++c) {
      cc[c] = v == n - 1 ? (w.esc ? w.env_m[c] : 0.0) : w.mise[v + 1][c] + l[c];
    }
    for (int c = 0; c < 3; ++c) l[c] = w.nee[v][c] + w.fcp[v][c] * cc[c];
  }
  for (int c = 0; c < 3; ++c) {
    out[c] = w.mise[0][c] + l[c];
    out_full[c] = w.emit[0][c] + l[c];
  }
}

// incident_targets_kernel (kernels.py:315-338): walk i keys
// stream_key(seed, P_TRAIN, frame, i, 0) and starts on the given ray.
__global__ void k_incident_targets(nirc_scene_t scn, uint64_t seed, uint64_t frame, V3 o, V3 d,
                                   double pv_pdf, V3 pns, int count, Stage st, double* out,
                                   double* out_full) {
  __shared__ __align__(16) unsigned char scene_sm[pt::kSceneSmemBytes];
  pt::stage_scene(scn, scene_sm);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  WalkLane w;
  w.p = i;
  w.key = stream_key(seed, P_TRAIN, frame, (uint64_t)i, 0);
  w.o = o;
  w.d = d;
  w.prev_pdf = pv_pdf;
  w.lns = pns;
  walk_incident(scn, w, st, out + 3 * i, out_full + 3 * i);
}

// integrand_samples_kernel (kernels.py:342-421): draw k of pixel p (one
// thread each, draws [q0, q0 + n) of the flattened (P, K) grid) at the
// centre ray's primary hit; the draw keys stream_key(seed, P_BASELINE,
// frame, p, k), samples the BSDF with dims (2, 3) and estimates the
// incident radiance with one recording walk (stage slot = draw - q0).
// Outputs the reference leaves untouched (missed / mirror pixels, dead
// draws' dir / f / frc) are not written.
__global__ void k_integrand_samples(nirc_scene_t scn, const double* cam, uint64_t seed,
                                    uint64_t frame, int K, int64_t q0, int64_t n, Stage st,
                                    double* o_dir, double* o_f, double* o_frc, double* o_pdf,
                                    uint8_t* o_valid, double* o_spos, double* o_sns,
                                    double* o_salb, double* o_srough) {
  __shared__ __align__(16) unsigned char scene_sm[pt::kSceneSmemBytes];
  pt::stage_scene(scn, scene_sm);
  const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= n) return;
  const int64_t q = q0 + slot, p = q / K;
  const int k = (int)(q - p * K);
  const int W = (int)cam[14];
  const int ix = (int)(p % W), iy = (int)(p / W);
  V3 o, d;
  pt::camera_ray(cam, ix, iy, 0.5, 0.5, o, d);
  const pt::Hit hh = pt::intersect<false>(scn, o, d, pt::T_FAR);
  if (k == 0) o_valid[p] = 0;
  if (hh.kind < 0) return;
  const int mkind = scn.mat_kind[hh.mid];
  if (mkind == pt::MAT_MIRROR) return;
  const V3 wo = {-d.x, -d.y, -d.z};
  const double flip = (hh.n.x * wo.x + hh.n.y * wo.y + hh.n.z * wo.z) >= 0.0 ? 1.0 : -1.0;
  const V3 ns = {hh.n.x * flip, hh.n.y * flip, hh.n.z * flip};
  const V3 alb = pt::ld3(scn.mat_albedo, hh.mid);
  const double rough = scn.mat_rough[hh.mid];
  if (k == 0) {
    o_valid[p] = 1;
    o_spos[3 * p] = hh.p.x; o_spos[3 * p + 1] = hh.p.y; o_spos[3 * p + 2] = hh.p.z;
    o_sns[3 * p] = ns.x; o_sns[3 * p + 1] = ns.y; o_sns[3 * p + 2] = ns.z;
    o_salb[3 * p] = alb.x; o_salb[3 * p + 1] = alb.y; o_salb[3 * p + 2] = alb.z;
    o_srough[p] = rough;
  }
  o_pdf[q] = 0.0;
  const uint64_t key = stream_key(seed, P_BASELINE, frame, (uint64_t)p, (uint64_t)k);
  const pt::BsdfSample b =
      pt::bsdf_sample(mkind, alb, rough, ns, wo, rand_uniform(key, 2), rand_uniform(key, 3));
  if (b.pdf <= 0.0 || b.delta == 1) return;
  const double ci = b.wi.x * ns.x + b.wi.y * ns.y + b.wi.z * ns.z;
  if (ci <= 0.0) return;
  const double sg = (hh.n.x * b.wi.x + hh.n.y * b.wi.y + hh.n.z * b.wi.z) > 0.0 ? 1.0 : -1.0;
  WalkLane w;
  w.p = slot;
  w.key = key;
  w.o = {hh.p.x + sg * scn.eps * hh.n.x, hh.p.y + sg * scn.eps * hh.n.y,
         hh.p.z + sg * scn.eps * hh.n.z};
  w.d = b.wi;
  w.prev_pdf = b.pdf;
  w.lns = ns;
  double res[3], res_full[3];
  walk_incident(scn, w, st, res, res_full);
  o_dir[3 * q] = b.wi.x; o_dir[3 * q + 1] = b.wi.y; o_dir[3 * q + 2] = b.wi.z;
  o_frc[3 * q] = b.f.x * ci; o_frc[3 * q + 1] = b.f.y * ci; o_frc[3 * q + 2] = b.f.z * ci;
  o_f[3 * q] = res[0] * b.f.x * ci;
  o_f[3 * q + 1] = res[1] * b.f.y * ci;
  o_f[3 * q + 2] = res[2] * b.f.z * ci;
  o_pdf[q] = b.pdf;
}

// occluded (geometry.py:206-210) over a batch of shadow rays.
__global__ void k_occluded(nirc_scene_t scn, const double* o, const double* d, int64_t n,
                           double t_max, uint8_t* out) {
  __shared__ __align__(16) unsigned char scene_sm[pt::kSceneSmemBytes];
  pt::stage_scene(scn, scene_sm);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const V3 oi = {o[3 * i], o[3 * i + 1], o[3 * i + 2]};
  const V3 di = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
  out[i] = pt::occluded(scn, oi, di, t_max) ? 1 : 0;
}

// pt_radiance (estimators.py:240-257): one MODE_PT sample of one pixel.
__global__ void k_pt_radiance(nirc_scene_t scn, const double* cam, nirc_render_cfg_t cfg,
                              int ix, int iy, int sample, double* out) {
  __shared__ __align__(16) unsigned char scene_sm[pt::kSceneSmemBytes];
  pt::stage_scene(scn, scene_sm);
  if (threadIdx.x != 0) return;
  PathState p;
  cfg.row0 = iy;
  cfg.spp = sample + 1;
  const int64_t sid = (int64_t)ix * cfg.spp + sample;  // row band [iy, iy+1)
  start_path(p, cam, cfg, sid);
  CacheVertex rec;
  int pending;
  while (!trace_vertex<false>(scn, cfg, p, rec, pending)) {
  }
  out[0] = p.ar;
  out[1] = p.ag;
  out[2] = p.ab;
}
}  // namespace nirc

extern "C" int nirc_surface_samples(const nirc_scene_t* scene, const double* ns_host,
                                    const double* wo_host, int32_t mat, const double* u,
                                    int32_t n, double* dirs, double* pdf, double* f,
                                    double* cosv, void* stream) {
  if (n <= 0) return NIRC_OK;
  if (mat < 0 || mat >= scene->n_mat) {
    set_last_error("material %d out of range", mat);
    return NIRC_E_CONFIG;
  }
  const V3 ns = {ns_host[0], ns_host[1], ns_host[2]};
  const V3 wo = {wo_host[0], wo_host[1], wo_host[2]};
  k_surface_samples<<<(n + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      *scene, ns, wo, mat, u, n, dirs, pdf, f, cosv);
  NIRC_LAUNCH_CHECK("k_surface_samples");
  return NIRC_OK;
}

extern "C" int nirc_incident_targets(const nirc_scene_t* scene, uint64_t seed, uint64_t frame,
                                     const double* origin_host, const double* dir_host,
                                     double prev_pdf, const double* prev_ns_host, int32_t count,
                                     double* out, double* out_full, void* stream) {
  if (count <= 0) return NIRC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  size_t bytes = 0;
  carve_stage(count, nullptr, &bytes);
  AsyncBuf ws(s);
  NIRC_CUDA_TRY(ws.alloc(bytes));
  size_t b2 = 0;
  Stage st = carve_stage(count, ws.p, &b2);
  st.kind = REC_NIRC;
  const V3 o = {origin_host[0], origin_host[1], origin_host[2]};
  const V3 d = {dir_host[0], dir_host[1], dir_host[2]};
  const V3 pns = {prev_ns_host[0], prev_ns_host[1], prev_ns_host[2]};
  k_incident_targets<<<(count + 63) / 64, 64, 0, s>>>(*scene, seed, frame, o, d, prev_pdf, pns,
                                                      count, st, out, out_full);
  NIRC_LAUNCH_CHECK("k_incident_targets");
  return NIRC_OK;
}

extern "C" int nirc_integrand_samples(const nirc_scene_t* scene, const double* cam,
                                      uint64_t seed, uint64_t frame, int32_t per_round,
                                      double* o_dir, double* o_f, double* o_frc, double* o_pdf,
                                      uint8_t* o_valid, double* o_spos, double* o_sns,
                                      double* o_salb, double* o_srough, void* stream) {
  if (per_round <= 0) {
    set_last_error("per_round must be positive");
    return NIRC_E_CONFIG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  double dims[2];
  NIRC_CUDA_TRY(cudaMemcpyAsync(dims, cam + 14, sizeof(dims), cudaMemcpyDeviceToHost, s));
  NIRC_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t P = (int64_t)dims[0] * (int64_t)dims[1], total = P * per_round;
  if (total == 0) return NIRC_OK;
  // the walks' per-vertex scratch is reused across chunks of draws
  const int64_t chunk = total < (int64_t(1) << 18) ? total : (int64_t(1) << 18);
  size_t bytes = 0;
  carve_stage(chunk, nullptr, &bytes);
  AsyncBuf ws(s);
  NIRC_CUDA_TRY(ws.alloc(bytes));
  size_t b2 = 0;
  Stage st = carve_stage(chunk, ws.p, &b2);
  st.kind = REC_NIRC;
  for (int64_t q0 = 0; q0 < total; q0 += chunk) {
    const int64_t n = total - q0 < chunk ? total - q0 : chunk;
    k_integrand_samples<<<(unsigned)((n + 63) / 64), 64, 0, s>>>(
        *scene, cam, seed, frame, per_round, q0, n, st, o_dir, o_f, o_frc, o_pdf, o_valid,
        o_spos, o_sns, o_salb, o_srough);
    NIRC_LAUNCH_CHECK("k_integrand_samples");
  }
  return NIRC_OK;
}

extern "C" int nirc_occluded(const nirc_scene_t* scene, const double* origins,
                             const double* dirs, int64_t n, double t_max, uint8_t* out,
                             void* stream) {
  if (n <= 0) return NIRC_OK;
  k_occluded<<<(unsigned)((n + 127) / 128), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      *scene, origins, dirs, n, t_max, out);
  NIRC_LAUNCH_CHECK("k_occluded");
  return NIRC_OK;
}

extern "C" int nirc_pt_radiance(const nirc_scene_t* scene, const double* cam,
                                const nirc_render_cfg_t* cfg, int32_t ix, int32_t iy,
                                int32_t sample, double* out, void* stream) {
  if (ix < 0 || iy < 0 || ix >= cfg->width || iy >= cfg->height || sample < 0) {
    set_last_error("pixel / sample out of range");
    return NIRC_E_CONFIG;
  }
  nirc_render_cfg_t c = *cfg;
  c.mode = 0;
  c.cache_on = 0;
  k_pt_radiance<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*scene, cam, c, ix, iy,
                                                                      sample, out);
  NIRC_LAUNCH_CHECK("k_pt_radiance");
  return NIRC_OK;
}
