// fp64 path-tracing building blocks (device).  Compiled with -fmad=false so
// every expression follows the reference's operation order:
//   geometry   pkg/src/nirclab/geometry.py:19-210
//   bsdf       pkg/src/nirclab/bsdf.py:27-154
//   lights     pkg/src/nirclab/lights.py:20-216
//   NEE        pkg/src/nirclab/kernels.py:44-82
#pragma once
#include "common.cuh"
#include "pt_packed.cuh"

namespace nirc {
namespace pt {

constexpr double T_FAR = 1.0e30;
constexpr double INV_PI = 1.0 / 3.141592653589793;
constexpr double PI = 3.141592653589793;
constexpr double TWO_PI = 2.0 * 3.141592653589793;
constexpr double FOUR_PI = 4.0 * 3.141592653589793;
constexpr double ALPHA_MIN = 1e-3;
constexpr int MAT_LAMBERT = 0, MAT_CONDUCTOR = 1, MAT_MIRROR = 2;
constexpr int LIGHT_TRI = 0, LIGHT_SPHERE = 1, LIGHT_ENV = 2;
constexpr int ENV_NONE = 0, ENV_CONSTANT = 1, ENV_SKY = 2, ENV_LATLONG = 3;
constexpr int MAXB = 64;
constexpr double RR_SURVIVE = 0.9;
constexpr int RR_START = 1;

struct V3 {
  double x, y, z;
};
__device__ inline V3 ld3(const double* a, int i) { return {a[3 * i], a[3 * i + 1], a[3 * i + 2]}; }
__device__ inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

// ---------------------------------------------------------- geometry ----
// ray_tri (geometry.py:19-44), Moller-Trumbore in f64.
__device__ inline double ray_tri(V3 o, V3 d, V3 v0, V3 e1, V3 e2) {
  const double px = d.y * e2.z - d.z * e2.y;
  const double py = d.z * e2.x - d.x * e2.z;
  const double pz = d.x * e2.y - d.y * e2.x;
  const double det = e1.x * px + e1.y * py + e1.z * pz;
  if (det > -1e-12 && det < 1e-12) return -1.0;
  const double inv = 1.0 / det;
  const double tx = o.x - v0.x, ty = o.y - v0.y, tz = o.z - v0.z;
  const double u = (tx * px + ty * py + tz * pz) * inv;
  if (u < -1e-9 || u > 1.0 + 1e-9) return -1.0;
  const double qx = ty * e1.z - tz * e1.y;
  const double qy = tz * e1.x - tx * e1.z;
  const double qz = tx * e1.y - ty * e1.x;
  const double v = (d.x * qx + d.y * qy + d.z * qz) * inv;
  if (v < -1e-9 || u + v > 1.0 + 1e-9) return -1.0;
  const double t = (e2.x * qx + e2.y * qy + e2.z * qz) * inv;
  if (t <= 0.0) return -1.0;
  return t;
}

__device__ inline double ray_sph(V3 o, V3 d, V3 c, double r) {
  const double lx = o.x - c.x, ly = o.y - c.y, lz = o.z - c.z;
  const double b = d.x * lx + d.y * ly + d.z * lz;
  const double cc = lx * lx + ly * ly + lz * lz - r * r;
  const double disc = b * b - cc;
  if (disc < 0.0) return -1.0;
  const double sq = sqrt(disc);
  const double t0 = -b - sq;
  if (t0 > 0.0) return t0;
  const double t1 = -b + sq;
  if (t1 > 0.0) return t1;
  return -1.0;
}

// _box_hit (geometry.py:66-99).  inv_d[a] = 1.0 / d[a] is computed once per
// ray: it is the same IEEE quotient the reference recomputes per box, so the
// slab test is bit-identical.
__device__ inline bool box_hit(V3 o, V3 d, const double* inv_d, const double* lo,
                               const double* hi, double t_best) {
  double t0 = 0.0, t1 = t_best;
  const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (dd[a] > -1e-30 && dd[a] < 1e-30) {
      if (oo[a] < lo[a] || oo[a] > hi[a]) return false;
    } else {
      double ta = (lo[a] - oo[a]) * inv_d[a];
      double tb = (hi[a] - oo[a]) * inv_d[a];
      if (ta > tb) {
        const double s = ta;
        ta = tb;
        tb = s;
      }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
      if (t0 > t1) return false;
    }
  }
  return true;
}

struct Hit {
  int kind, prim, mid;
  double t;
  V3 p, n;
};

// intersect_bvh (geometry.py:153-202): nearest hit with t in (eps, t_max).
// any_hit stops at the first accepted primitive (occlusion queries only
// need the boolean, which is identical).
// Scenes up to this many primitives are intersected by a warp-uniform scan
// over the BVH's primitive order instead of a per-lane stack traversal: every
// lane runs the same loop (no divergence; broadcast shared-memory reads), and
// the test order is the BVH's depth-first leaf order, so exact ties resolve
// to the same primitive.
constexpr int kLinearMaxPrims = 64;

// Conservative fp32 pre-test of one scan-order triangle (the linear-scan
// path): returns false only when ray_tri's f64 result is certainly rejected
// by the caller's window t in (t_lo, t_hi).  The fp32 evaluation of
// ray_tri's numerators (det, u*det, v*det, t*det) differs from the f64 one
// by at most ~9 unit roundoffs of the magnitude bounds below (inputs
// rounded to fp32 included); K = 16 u gives 2x headroom, and the 1e-9
// thresholds carry a 1e-12 relative slack for ray_tri's own rounding of
// 1/det and the products.  Rows of T (48 B per triangle, 16 B aligned):
//   (v0.xyz, |e1|_1), (e1.xyz, |e2|_1), (e2.xyz, |v0|_1).
constexpr float kFilterK = 16.0f * 5.9604645e-8f * 1.0001f;  // 16 unit roundoffs
#ifndef NIRC_FILTER_UNROLL
#define NIRC_FILTER_UNROLL 1  // measured: 1 < 2 < 4 < 8 (instruction-cache pressure)
#endif
constexpr int kFilterUnroll = NIRC_FILTER_UNROLL;
struct RayF32 {
  float ox, oy, oz, dx, dy, dz, kd, no;  // kd = K * |d|_1, no = |o|_1
};
__device__ inline RayF32 ray_f32(V3 o, V3 d) {
  RayF32 r;
  r.ox = (float)o.x; r.oy = (float)o.y; r.oz = (float)o.z;
  r.dx = (float)d.x; r.dy = (float)d.y; r.dz = (float)d.z;
  r.kd = kFilterK * (fabsf(r.dx) + fabsf(r.dy) + fabsf(r.dz)) * 1.0001f;
  r.no = (fabsf(r.ox) + fabsf(r.oy) + fabsf(r.oz)) * 1.0001f;
  return r;
}
// One scan item: a triangle (cu = 1: u, v >= 0, u + v <= 1) or a
// parallelogram v0 + u e1 + v e2 (cu = 0: u, v in [0, 1]) covering two
// scan-order triangles (v0, e1, e1 + e2) and (v0, e1 + e2, e2) -- their
// union, so the test stays conservative for both.  `slack` is the
// barycentric tolerance the item needs (the reference's 1e-9, doubled for a
// parallelogram whose triangles carry it in their own coordinates).
__device__ inline bool tri_candidate(const RayF32& r, const float4* T, float t_lo, float t_hi) {
  const float4 A = T[0], B = T[1], C = T[2], D = T[3];
  const float px = r.dy * C.z - r.dz * C.y;
  const float py = r.dz * C.x - r.dx * C.z;
  const float pz = r.dx * C.y - r.dy * C.x;
  const float det = B.x * px + B.y * py + B.z * pz;
  const float tx = r.ox - A.x, ty = r.oy - A.y, tz = r.oz - A.z;
  const float un = tx * px + ty * py + tz * pz;
  const float qx = ty * B.z - tz * B.y;
  const float qy = tz * B.x - tx * B.z;
  const float qz = tx * B.y - ty * B.x;
  const float vn = r.dx * qx + r.dy * qy + r.dz * qz;
  const float tn = C.x * qx + C.y * qy + C.z * qz;
  // magnitude bounds: |e1|_1 |d|_1 |e2|_1 etc., |t|_1 <= |o|_1 + |v0|_1
  const float nt = (r.no + C.w) * 1.0001f;
  const float Ed = r.kd * A.w * B.w;
  const float Eu = r.kd * nt * B.w;
  const float Ev = r.kd * nt * A.w;
  const float Et = kFilterK * nt * A.w * B.w;
  const float ad = fabsf(det);
  const float sgn = det > 0.0f ? 1.0f : -1.0f;
  const float u = un * sgn, v = vn * sgn, t = tn * sgn;
  const float hi = ad + Ed, lo = ad - Ed;
  const float cu = D.x, sl = D.y;
  // branch-free: every condition is a predicate, the scan loop stays straight
  const bool out = (u + Eu < -sl * hi) |                        // u < -slack
                   (u - Eu > (1.0f + sl) * hi) |                // u > 1 + slack
                   (v + Ev < -sl * hi) |                        // v < -slack
                   (v - Ev > (1.0f + 2.0f * sl) * hi) |         // v > 1 + 2 slack
                   (cu * (u - Eu) + v - Ev > (1.0f + sl) * hi) |  // u + v > 1 + slack
                   (t + Et < t_lo * lo * 0.999999f) |           // t <= t_lo (t_lo > 0)
                   (t - Et > t_hi * hi * 1.000001f);            // t >= t_hi (inf: never)
  return !(ad > Ed) | !out;  // sign of det uncertain: the exact test decides
}
// scan-order triangles an item covers, as a candidate bit mask (stored as
// two 32-bit words in the row's last two lanes)
__device__ inline uint64_t item_bits(const float4* T) {
  return ((uint64_t)__float_as_uint(T[3].w) << 32) | __float_as_uint(T[3].z);
}

// Traversal image (nirc_pack_scene): per internal node both child boxes and
// child references (n > 0: leaf, primitives [c, c + n) of the leaf order;
// n == 0: internal node c), primitives in leaf order with geometry inline.
// (layouts in pt_packed.cuh)

// _box_hit's slab test (the same arithmetic and accept rule as box_hit),
// returning the entry distance t0 as well.
__device__ inline bool box_entry(const double* oo, const double* inv_d, const double* lo,
                                 const double* hi, double t_best, double& t_in) {
  double t0 = 0.0, t1 = t_best;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (fabs(inv_d[a]) == __longlong_as_double(0x7ff0000000000000ll)) {  // |d| < 1e-30
      if (oo[a] < lo[a] || oo[a] > hi[a]) return false;
    } else {
      double ta = (lo[a] - oo[a]) * inv_d[a];
      double tb = (hi[a] - oo[a]) * inv_d[a];
      if (ta > tb) {
        const double s = ta;
        ta = tb;
        tb = s;
      }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
      if (t0 > t1) return false;
    }
  }
  t_in = t0;
  return true;
}

// Conservative fp32 slab test of a packed (outward-rounded) child box: accepts
// every box _box_hit accepts for the f64 ray (it may accept a few more,
// which only costs primitive tests).  Each slab distance is widened by the
// fp32 rounding of the origin (w = |o| 2^-22 |1/d|, precomputed per ray) and
// of the subtraction / inverse / product (2^-20 relative); t_in is a lower
// bound of the f64 entry distance.
struct RayBox32 {
  float o[3], inv[3], w[3];
  bool par[3];  // |d| < 1e-30: the reference's parallel-slab case
};
__device__ inline RayBox32 ray_box32(V3 o, V3 d) {
  RayBox32 r;
  const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    r.o[a] = (float)oo[a];
    r.par[a] = dd[a] > -1e-30 && dd[a] < 1e-30;
    r.inv[a] = r.par[a] ? 0.0f : (float)(1.0 / dd[a]);
    r.w[a] = (fabsf(r.o[a]) * 2.384185791e-7f + 1e-30f) * fabsf(r.inv[a]);  // 2^-22
  }
  return r;
}
__device__ inline bool box_entry32(const RayBox32& r, const float* lo, const float* hi,
                                   float t_best, float& t_in) {
  float t0 = 0.0f, t1 = t_best;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (r.par[a]) {
      const float m = fabsf(r.o[a]) * 2.384185791e-7f + 1e-30f;
      if (r.o[a] < lo[a] - m || r.o[a] > hi[a] + m) return false;
    } else {
      const float ta = (lo[a] - r.o[a]) * r.inv[a];
      const float tb = (hi[a] - r.o[a]) * r.inv[a];
      const float tn = fminf(ta, tb), tf = fmaxf(ta, tb);
      const float tn_w = tn - (fabsf(tn) * 9.5367431640625e-7f + r.w[a]);  // 2^-20
      const float tf_w = tf + (fabsf(tf) * 9.5367431640625e-7f + r.w[a]);
      t0 = fmaxf(t0, tn_w);
      t1 = fminf(t1, tf_w);
    }
  }
  t_in = t0;
  return t0 <= t1;
}

// Front-to-back traversal of the packed image: at an internal node both
// child boxes are tested (fp32, conservatively) against the current best
// distance and the nearer child is visited first (child 0 on equal entry
// distances); popped subtrees whose entry lies beyond the best hit are
// skipped.  The reference's left-first walk meets primitives in leaf order
// and keeps the first of equal distances, so its hit is the minimum of
// (t, leaf index): ties here resolve the same way, and the nearest hit (kind,
// primitive, t) and the any-hit boolean equal the reference's exactly.
template <bool AnyHit>
__device__ __noinline__ void bvh_scan_packed(const nirc_scene_t& s, V3 o, V3 d, double& best,
                                             int& kind, int& prim) {
  const double eps = s.eps;
  const double oo[3] = {o.x, o.y, o.z};
  const double dd[3] = {d.x, d.y, d.z};
  double inv_d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)  // parallel axes (|d| < 1e-30) marked by an infinite inverse
    inv_d[a] = (dd[a] > -1e-30 && dd[a] < 1e-30) ? __longlong_as_double(0x7ff0000000000000ll)
                                                 : 1.0 / dd[a];
  const PackedNode* N = reinterpret_cast<const PackedNode*>(s.bvh_packed);
  const PackedPrim* Pp = reinterpret_cast<const PackedPrim*>(s.prim_packed);
  double t_root;
  if (s.bvh_b[0] == 0 && s.bvh_a[0] == 0 && s.n_tri + s.n_sph == 0) return;
  if (!box_entry(oo, inv_d, s.bvh_lo, s.bvh_hi, best, t_root)) return;
  const RayBox32 rb32 = ray_box32(o, d);
  int cur = s.bvh_b[0] > 0 ? (s.bvh_a[0] << 3 | s.bvh_b[0]) : 0;
  int best_k = 0x7fffffff;
  int st_ref[40];
  float st_t[40];
  int sp = 0;
  while (true) {
    const int n = cur & 7, idx = cur >> 3;
    if (n > 0) {
      for (int k = idx; k < idx + n; ++k) {
        const PackedPrim& q = Pp[k];
        const double t = q.kind == 0
                             ? ray_tri(o, d, {q.g[0], q.g[1], q.g[2]}, {q.g[3], q.g[4], q.g[5]},
                                       {q.g[6], q.g[7], q.g[8]})
                             : ray_sph(o, d, {q.g[0], q.g[1], q.g[2]}, q.g[3]);
        // equal distances resolve to the earlier leaf-order primitive: the
        // one the reference's left-first walk meets first
        if (t > eps && (t < best || (t == best && kind >= 0 && k < best_k))) {
          best = t;
          best_k = k;
          kind = q.kind;
          prim = q.id;
          if (AnyHit) return;
        }
      }
    } else {
      const PackedNode& nd = N[idx];
      float ta = 0.0f, tb = 0.0f;
      const float best_up = __double2float_ru(best);
      const bool ha = box_entry32(rb32, nd.lo0, nd.hi0, best_up, ta);
      const bool hb = box_entry32(rb32, nd.lo1, nd.hi1, best_up, tb);
      int ra = nd.c0 << 3 | nd.n0, rb = nd.c1 << 3 | nd.n1;
      if (ha && hb) {
        if (tb < ta) {
          const int r = ra;
          ra = rb;
          rb = r;
          const float t = ta;
          ta = tb;
          tb = t;
        }
        // visit the nearer child; push the farther one with its entry (a
        // lower bound: the pop test stays conservative)
        st_ref[sp] = rb;
        st_t[sp] = tb;
        ++sp;
        cur = ra;
        continue;
      }
      if (ha) {
        cur = ra;
        continue;
      }
      if (hb) {
        cur = rb;
        continue;
      }
    }
    do {
      if (sp == 0) return;
      --sp;
    } while ((double)st_t[sp] > best);
    cur = st_ref[sp];
  }
}

// Linear f64 scan (no staged fp32 table) or BVH traversal (spheres, larger
// scenes) -- the reference's intersect_bvh order; kept out of line.
template <bool AnyHit>
__device__ __noinline__ void bvh_scan(const nirc_scene_t& s, V3 o, V3 d, double& best, int& kind,
                                      int& prim) {
  const double eps = s.eps;
  if (s.n_tri + s.n_sph <= kLinearMaxPrims && s.n_sph == 0) {
    const int np = s.n_tri;
    for (int k = 0; k < np; ++k) {
      const int pid = s.bvh_prim[k];
      const double t = ray_tri(o, d, ld3(s.tri_v0, pid), ld3(s.tri_e1, pid), ld3(s.tri_e2, pid));
      if (t > eps && t < best) {
        best = t;
        kind = 0;
        prim = pid;
        if (AnyHit) break;
      }
    }
  } else {
  int stack[64];
  int top = 0;
  stack[top++] = 0;
  const double inv_d[3] = {1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
  while (top > 0) {
    const int node = stack[--top];
    if (!box_hit(o, d, inv_d, s.bvh_lo + 3 * node, s.bvh_hi + 3 * node, best)) continue;
    const int count = s.bvh_b[node];
    if (count > 0) {
      const int first = s.bvh_a[node];
      for (int k = first; k < first + count; ++k) {
        const int pid = s.bvh_prim[k];
        if (pid < s.n_tri) {
          const double t = ray_tri(o, d, ld3(s.tri_v0, pid), ld3(s.tri_e1, pid),
                                   ld3(s.tri_e2, pid));
          if (t > eps && t < best) {
            best = t;
            kind = 0;
            prim = pid;
          }
        } else {
          const int j = pid - s.n_tri;
          const double t = ray_sph(o, d, ld3(s.sph_c, j), s.sph_r[j]);
          if (t > eps && t < best) {
            best = t;
            kind = 1;
            prim = j;
          }
        }
        if (AnyHit && kind >= 0) return;
      }
    } else if (count == 0 && s.bvh_a[node] != node) {
      stack[top++] = s.bvh_a[node];
      stack[top++] = node + 1;
    }
  }
  }
}

template <bool AnyHit>
__device__ inline Hit intersect(const nirc_scene_t& s, V3 o, V3 d, double t_max) {
  const double eps = s.eps;
  double best = t_max;
  int kind = -1, prim = -1;
  if (s.tri_f32 && s.n_sph == 0 && s.n_tri <= kLinearMaxPrims) {
    // warp-uniform fp32 pre-test over the scan order, then ray_tri (f64,
    // the reference's arithmetic) on each lane's own candidates in scan
    // order: the accepted hit (and any-hit boolean) equal the full scan's
    const int ni = s.n_filter;
    const RayF32 r = ray_f32(o, d);
    const float4* T = reinterpret_cast<const float4*>(s.tri_f32);
    const float f_lo = (float)eps;
    const float f_hi = t_max < 1e29 ? (float)t_max : __int_as_float(0x7f800000);
    uint64_t cand = 0;
#pragma unroll(kFilterUnroll)
    for (int k = 0; k < ni; ++k)
      cand |= tri_candidate(r, T + 4 * k, f_lo, f_hi) ? item_bits(T + 4 * k) : 0ull;
    while (cand) {
      const int k = __ffsll((long long)cand) - 1;
      cand &= cand - 1;
      const int pid = s.bvh_prim[k];
      const double t = ray_tri(o, d, ld3(s.tri_v0, pid), ld3(s.tri_e1, pid), ld3(s.tri_e2, pid));
      if (t > eps && t < best) {
        best = t;
        kind = 0;
        prim = pid;
        if (AnyHit) break;
      }
    }
  } else if (s.bvh_packed) {
    // general scenes with a traversal image: front to back, out of line
    bvh_scan_packed<AnyHit>(s, o, d, best, kind, prim);
  } else {
    // general scenes (spheres, > 64 primitives): out of line, see below
    bvh_scan<AnyHit>(s, o, d, best, kind, prim);
  }
  Hit h;
  h.kind = kind;
  h.prim = prim;
  h.mid = -1;
  h.t = -1.0;
  if (kind < 0) return h;
  h.t = best;
  h.p = {o.x + d.x * best, o.y + d.y * best, o.z + d.z * best};
  if (kind == 0) {
    h.n = ld3(s.tri_ng, prim);
    h.mid = s.tri_mat[prim];
  } else {
    const double inv = 1.0 / s.sph_r[prim];
    const V3 c = ld3(s.sph_c, prim);
    h.n = {(h.p.x - c.x) * inv, (h.p.y - c.y) * inv, (h.p.z - c.z) * inv};
    h.mid = s.sph_mat[prim];
  }
  return h;
}

__device__ inline bool occluded(const nirc_scene_t& s, V3 o, V3 d, double t_max) {
  return intersect<true>(s, o, d, t_max).kind >= 0;
}

// ------------------------------------------------------------- frames ---
struct Cosine {
  double x, y, z, pdf;
};
// core.py:57-65
__device__ inline Cosine cosine_dir(double u1, double u2) {
  const double r = sqrt(u1);
  const double phi = TWO_PI * u2;
  Cosine c;
  c.x = r * cos(phi);
  c.y = r * sin(phi);
  const double t = 1.0 - u1;
  c.z = sqrt(t > 0.0 ? t : 0.0);
  c.pdf = c.z * INV_PI;
  return c;
}

// ---------------------------------------------------------------- BSDF --
__device__ inline double ggx_d(double alpha, double ch) {
  const double a2 = alpha * alpha;
  const double d = ch * ch * (a2 - 1.0) + 1.0;
  return a2 / (PI * d * d);
}
__device__ inline double ggx_g1(double alpha, double cv) {
  const double a2 = alpha * alpha;
  return 2.0 * cv / (cv + sqrt(a2 + (1.0 - a2) * cv * cv));
}

// The conductor (GGX) lobe is kept out of line (__noinline__): scenes of
// Lambert walls never execute it, and the tracer is instruction-cache bound.
__device__ __noinline__ V3 ggx_eval(V3 a, double rough, V3 n, V3 wo, V3 wi, double ci,
                                    double co);
__device__ __noinline__ double ggx_pdf(double rough, V3 n, V3 wo, V3 wi);
struct BsdfSample;

// bsdf_eval_s (bsdf.py:38-72)
__device__ inline V3 bsdf_eval(int kind, V3 a, double rough, V3 n, V3 wo, V3 wi) {
  const double ci = n.x * wi.x + n.y * wi.y + n.z * wi.z;
  const double co = n.x * wo.x + n.y * wo.y + n.z * wo.z;
  if (ci <= 0.0 || co <= 0.0 || kind == MAT_MIRROR) return {0.0, 0.0, 0.0};
  if (kind == MAT_LAMBERT) return {a.x * INV_PI, a.y * INV_PI, a.z * INV_PI};
  return ggx_eval(a, rough, n, wo, wi, ci, co);
}

__device__ __noinline__ V3 ggx_eval(V3 a, double rough, V3 n, V3 wo, V3 wi, double ci,
                                    double co) {
  const double alpha = rough > ALPHA_MIN ? rough : ALPHA_MIN;
  double hx = wi.x + wo.x, hy = wi.y + wo.y, hz = wi.z + wo.z;
  const double hl = sqrt(hx * hx + hy * hy + hz * hz);
  if (hl < 1e-12) return {0.0, 0.0, 0.0};
  hx /= hl;
  hy /= hl;
  hz /= hl;
  const double ch = n.x * hx + n.y * hy + n.z * hz;
  if (ch <= 0.0) return {0.0, 0.0, 0.0};
  const double D = ggx_d(alpha, ch);
  const double G = ggx_g1(alpha, ci) * ggx_g1(alpha, co);
  double cd = wo.x * hx + wo.y * hy + wo.z * hz;
  if (cd < 0.0) cd = 0.0;
  double s5 = (1.0 - cd);
  s5 = s5 * s5 * s5 * s5 * s5;
  const double scale = D * G / (4.0 * ci * co);
  return {(a.x + (1.0 - a.x) * s5) * scale, (a.y + (1.0 - a.y) * s5) * scale,
          (a.z + (1.0 - a.z) * s5) * scale};
}

// bsdf_pdf_s (bsdf.py:75-100)
__device__ inline double bsdf_pdf(int kind, double rough, V3 n, V3 wo, V3 wi) {
  const double ci = n.x * wi.x + n.y * wi.y + n.z * wi.z;
  const double co = n.x * wo.x + n.y * wo.y + n.z * wo.z;
  if (ci <= 0.0 || co <= 0.0 || kind == MAT_MIRROR) return 0.0;
  if (kind == MAT_LAMBERT) return ci * INV_PI;
  return ggx_pdf(rough, n, wo, wi);
}

__device__ __noinline__ double ggx_pdf(double rough, V3 n, V3 wo, V3 wi) {
  const double alpha = rough > ALPHA_MIN ? rough : ALPHA_MIN;
  double hx = wi.x + wo.x, hy = wi.y + wo.y, hz = wi.z + wo.z;
  const double hl = sqrt(hx * hx + hy * hy + hz * hz);
  if (hl < 1e-12) return 0.0;
  hx /= hl;
  hy /= hl;
  hz /= hl;
  const double ch = n.x * hx + n.y * hy + n.z * hz;
  if (ch <= 0.0) return 0.0;
  const double cd = wo.x * hx + wo.y * hy + wo.z * hz;
  if (cd < 1e-9) return 0.0;
  return ggx_d(alpha, ch) * ch / (4.0 * cd);
}

struct BsdfSample {
  V3 wi;
  double pdf;
  V3 f;
  int delta;
};

__device__ __noinline__ BsdfSample ggx_sample(int kind, V3 a, double rough, V3 n, V3 wo,
                                              double u1, double u2);

// bsdf_sample_s (bsdf.py:103-154)
__device__ inline BsdfSample bsdf_sample(int kind, V3 a, double rough, V3 n, V3 wo, double u1,
                                         double u2) {
  BsdfSample r;
  r.wi = {0.0, 0.0, 1.0};
  r.pdf = 0.0;
  r.f = {0.0, 0.0, 0.0};
  r.delta = 0;
  if (kind == MAT_MIRROR) {
    r.delta = 1;
    const double co = n.x * wo.x + n.y * wo.y + n.z * wo.z;
    const V3 wi = {2.0 * co * n.x - wo.x, 2.0 * co * n.y - wo.y, 2.0 * co * n.z - wo.z};
    const double ci = n.x * wi.x + n.y * wi.y + n.z * wi.z;
    if (ci < 1e-9) return r;
    const double inv = 1.0 / ci;
    r.wi = wi;
    r.pdf = 1.0;
    r.f = {a.x * inv, a.y * inv, a.z * inv};
    return r;
  }
  if (kind == MAT_LAMBERT) {
    const Onb b = onb(n.x, n.y, n.z);
    const Cosine c = cosine_dir(u1, u2);
    const V3 wi = {b.tx * c.x + b.bx * c.y + n.x * c.z, b.ty * c.x + b.by * c.y + n.y * c.z,
                   b.tz * c.x + b.bz * c.y + n.z * c.z};
    const double co = n.x * wo.x + n.y * wo.y + n.z * wo.z;
    if (co <= 0.0 || c.pdf <= 0.0) return r;
    r.wi = wi;
    r.pdf = c.pdf;
    r.f = {a.x * INV_PI, a.y * INV_PI, a.z * INV_PI};
    return r;
  }
  return ggx_sample(kind, a, rough, n, wo, u1, u2);
}

__device__ __noinline__ BsdfSample ggx_sample(int kind, V3 a, double rough, V3 n, V3 wo,
                                              double u1, double u2) {
  BsdfSample r;
  r.wi = {0.0, 0.0, 1.0};
  r.pdf = 0.0;
  r.f = {0.0, 0.0, 0.0};
  r.delta = 0;
  const double alpha = rough > ALPHA_MIN ? rough : ALPHA_MIN;
  const double ch = sqrt((1.0 - u1) / (1.0 + (alpha * alpha - 1.0) * u1));
  const double sh = sqrt(ch < 1.0 ? 1.0 - ch * ch : 0.0);
  const double phi = TWO_PI * u2;
  const Onb b = onb(n.x, n.y, n.z);
  const double hlx = sh * cos(phi), hly = sh * sin(phi);
  const V3 h = {b.tx * hlx + b.bx * hly + n.x * ch, b.ty * hlx + b.by * hly + n.y * ch,
                b.tz * hlx + b.bz * hly + n.z * ch};
  const double cd = wo.x * h.x + wo.y * h.y + wo.z * h.z;
  if (cd < 1e-9) return r;
  const V3 wi = {2.0 * cd * h.x - wo.x, 2.0 * cd * h.y - wo.y, 2.0 * cd * h.z - wo.z};
  const double pdf = ggx_d(alpha, ch) * ch / (4.0 * cd);
  const V3 f = bsdf_eval(kind, a, rough, n, wo, wi);
  const double ci = n.x * wi.x + n.y * wi.y + n.z * wi.z;
  if (ci <= 0.0 || pdf <= 0.0) return r;
  r.wi = wi;
  r.pdf = pdf;
  r.f = f;
  return r;
}

// -------------------------------------------------------------- lights --
// env_eval_s (lights.py:20-58); out of line (cold for closed scenes)
__device__ __noinline__ V3 env_eval(const nirc_scene_t& s, V3 d) {
  if (s.env_kind == ENV_NONE) return {0.0, 0.0, 0.0};
  if (s.env_kind == ENV_CONSTANT) return {s.env_c0[0], s.env_c0[1], s.env_c0[2]};
  if (s.env_kind == ENV_SKY) {
    double t;
    const double* b;
    if (d.y >= 0.0) {
      t = d.y;
      b = s.env_c0;
    } else {
      t = -d.y;
      b = s.env_c2;
    }
    const double* a = s.env_c1;
    return {a[0] + (b[0] - a[0]) * t, a[1] + (b[1] - a[1]) * t, a[2] + (b[2] - a[2]) * t};
  }
  double cy = d.y;
  if (cy > 1.0) cy = 1.0;
  else if (cy < -1.0) cy = -1.0;
  const double v = acos(cy) / PI;
  const double u = 0.5 + atan2(d.x, -d.z) / TWO_PI;
  int col = (int)(u * s.env_w);
  int row = (int)(v * s.env_h);
  if (col >= s.env_w) col = s.env_w - 1;
  if (col < 0) col = 0;
  if (row >= s.env_h) row = s.env_h - 1;
  if (row < 0) row = 0;
  const double* px = s.env_img + 3 * ((int64_t)row * s.env_w + col);
  return {px[0], px[1], px[2]};
}

struct LightSample {
  V3 wi;
  double dist;
  V3 e;
  double pdf;
  int src;
};

// sample_light_s (lights.py:61-135)
__device__ inline LightSample sample_light(const nirc_scene_t& s, V3 p, V3 ns, double u_pick,
                                          double u1, double u2) {
  LightSample r;
  r.wi = {0.0, 0.0, 1.0};
  r.dist = 0.0;
  r.e = {0.0, 0.0, 0.0};
  r.pdf = 0.0;
  r.src = -1;
  const int n = s.n_light;
  if (n == 0) return r;
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (s.lt_cdf[mid] < u_pick) lo = mid + 1;
    else hi = mid;
  }
  const double q = s.lt_q[lo];
  const int kind = s.lt_kind[lo];
  const int prim = s.lt_prim[lo];
  if (kind == LIGHT_ENV) {
    const Onb b = onb(ns.x, ns.y, ns.z);
    const Cosine c = cosine_dir(u1, u2);
    const V3 wi = {b.tx * c.x + b.bx * c.y + ns.x * c.z, b.ty * c.x + b.by * c.y + ns.y * c.z,
                   b.tz * c.x + b.bz * c.y + ns.z * c.z};
    r.wi = wi;
    r.dist = T_FAR;
    r.e = env_eval(s, wi);
    r.pdf = q * c.pdf;
    r.src = LIGHT_ENV;
    return r;
  }
  V3 lp, ln;
  double area;
  int mid;
  if (kind == LIGHT_TRI) {
    const double r1 = sqrt(u1);
    const double b1 = r1 * (1.0 - u2);
    const double b2 = r1 * u2;
    const V3 v0 = ld3(s.tri_v0, prim), e1 = ld3(s.tri_e1, prim), e2 = ld3(s.tri_e2, prim);
    lp = {v0.x + e1.x * b1 + e2.x * b2, v0.y + e1.y * b1 + e2.y * b2,
          v0.z + e1.z * b1 + e2.z * b2};
    ln = ld3(s.tri_ng, prim);
    area = s.tri_area[prim];
    mid = s.tri_mat[prim];
  } else {
    const double z = 1.0 - 2.0 * u1;
    const double sn = sqrt(z * z < 1.0 ? 1.0 - z * z : 0.0);
    const double phi = TWO_PI * u2;
    ln = {sn * cos(phi), sn * sin(phi), z};
    const double rr = s.sph_r[prim];
    const V3 c = ld3(s.sph_c, prim);
    lp = {c.x + rr * ln.x, c.y + rr * ln.y, c.z + rr * ln.z};
    area = FOUR_PI * rr * rr;
    mid = s.sph_mat[prim];
  }
  const double dx = lp.x - p.x, dy = lp.y - p.y, dz = lp.z - p.z;
  const double d2 = dx * dx + dy * dy + dz * dz;
  const double dist = sqrt(d2);
  if (dist < 1e-9) return r;
  const V3 wi = {dx / dist, dy / dist, dz / dist};
  double cos_l = -(wi.x * ln.x + wi.y * ln.y + wi.z * ln.z);
  if (cos_l < 0.0) cos_l = -cos_l;
  if (cos_l < 1e-9 || area < 1e-12) return r;
  r.wi = wi;
  r.dist = dist;
  r.e = ld3(s.mat_emit, mid);
  r.pdf = q * d2 / (area * cos_l);
  r.src = kind;
  return r;
}

// nee_pdf_for_hit_s (lights.py:138-159)
__device__ inline double nee_pdf_for_hit(const nirc_scene_t& s, int hit_kind, int prim, double t,
                                         V3 wi, V3 ln) {
  double q, area;
  if (hit_kind == 0) {
    q = s.tri_lq[prim];
    area = s.tri_area[prim];
  } else {
    q = s.sph_lq[prim];
    area = FOUR_PI * s.sph_r[prim] * s.sph_r[prim];
  }
  if (q <= 0.0 || area < 1e-12) return 0.0;
  double cos_l = -(wi.x * ln.x + wi.y * ln.y + wi.z * ln.z);
  if (cos_l < 0.0) cos_l = -cos_l;
  if (cos_l < 1e-9) return 0.0;
  return q * t * t / (area * cos_l);
}

// nee_pdf_for_env_s (lights.py:162-169)
__device__ inline double nee_pdf_for_env(const nirc_scene_t& s, V3 ns, V3 wi) {
  if (s.env_q <= 0.0) return 0.0;
  const double c = ns.x * wi.x + ns.y * wi.y + ns.z * wi.z;
  if (c <= 0.0) return 0.0;
  return s.env_q * c / PI;
}

// camera_ray_s (lights.py:205-216)
__device__ inline void camera_ray(const double* cam, int ix, int iy, double u, double v, V3& o,
                                  V3& d) {
  const double w = cam[14], h = cam[15];
  const double sx = ((ix + u) / w * 2.0 - 1.0) * cam[12] * cam[13];
  const double sy = (1.0 - (iy + v) / h * 2.0) * cam[12];
  const double dx = cam[3] * sx + cam[6] * sy + cam[9];
  const double dy = cam[4] * sx + cam[7] * sy + cam[10];
  const double dz = cam[5] * sx + cam[8] * sy + cam[11];
  const double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
  o = {cam[0], cam[1], cam[2]};
  d = {dx * inv, dy * inv, dz * inv};
}

// nee_contrib_s (kernels.py:44-82)
__device__ inline V3 nee_contrib(const nirc_scene_t& s, V3 p, V3 ns, V3 gn, int mkind, V3 alb,
                                 double rough, V3 wo, double u_pick, double u1, double u2,
                                 int terminal) {
  const V3 zero = {0.0, 0.0, 0.0};
  if (s.n_light == 0) return zero;
  const LightSample L = sample_light(s, p, ns, u_pick, u1, u2);
  if (L.pdf <= 0.0) return zero;
  const double cs = L.wi.x * ns.x + L.wi.y * ns.y + L.wi.z * ns.z;
  if (cs <= 0.0) return zero;
  const V3 f = bsdf_eval(mkind, alb, rough, ns, wo, L.wi);
  if (f.x == 0.0 && f.y == 0.0 && f.z == 0.0) return zero;
  const double sgn = (gn.x * L.wi.x + gn.y * L.wi.y + gn.z * L.wi.z) > 0.0 ? 1.0 : -1.0;
  const V3 o = {p.x + sgn * s.eps * gn.x, p.y + sgn * s.eps * gn.y, p.z + sgn * s.eps * gn.z};
  const double t_lim = L.dist - 2.0 * s.eps;
  if (t_lim <= 0.0) return zero;
  if (occluded(s, o, L.wi, t_lim)) return zero;
  double w;
  if (terminal != 0) {
    w = 1.0;
  } else {
    const double pb = bsdf_pdf(mkind, rough, ns, wo, L.wi);
    w = L.pdf / (L.pdf + pb);
  }
  const double sc = w * cs / L.pdf;
  return {f.x * L.e.x * sc, f.y * L.e.y * sc, f.z * L.e.z * sc};
}

// Copies the geometry the traversal touches (triangles, spheres, BVH) into
// shared memory when it fits and redirects the scene pointers there; the
// kernel then reads it through generic loads that resolve to shared memory.
constexpr int kSceneSmemBytes = 40 * 1024;

__host__ __device__ inline size_t scene_smem_bytes(const nirc_scene_t& s) {
  return (size_t)s.n_tri * (4 * 3 * 8 + 4) + (size_t)s.n_sph * (4 * 8 + 4) +
         (size_t)s.n_bvh * (6 * 8 + 8) + (size_t)(s.n_tri + s.n_sph) * 4 + 64 +
         (size_t)s.n_tri * 64 + 16;  // fp32 filter table
}

__device__ inline void stage_scene(nirc_scene_t& s, unsigned char* sm) {
  if (scene_smem_bytes(s) > (size_t)kSceneSmemBytes) return;
  double* dp = reinterpret_cast<double*>(sm);
  auto cp = [&](const double* src, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dp[i] = src[i];
    const double* r = dp;
    dp += n;
    return r;
  };
  s.tri_v0 = cp(s.tri_v0, 3 * s.n_tri);
  s.tri_e1 = cp(s.tri_e1, 3 * s.n_tri);
  s.tri_e2 = cp(s.tri_e2, 3 * s.n_tri);
  s.tri_ng = cp(s.tri_ng, 3 * s.n_tri);
  s.sph_c = cp(s.sph_c, 3 * s.n_sph);
  s.sph_r = cp(s.sph_r, s.n_sph);
  s.bvh_lo = cp(s.bvh_lo, 3 * s.n_bvh);
  s.bvh_hi = cp(s.bvh_hi, 3 * s.n_bvh);
  int* ip = reinterpret_cast<int*>(dp);
  auto cpi = [&](const int* src, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) ip[i] = src[i];
    const int* r = ip;
    ip += n;
    return r;
  };
  s.tri_mat = cpi(s.tri_mat, s.n_tri);
  s.sph_mat = cpi(s.sph_mat, s.n_sph);
  s.bvh_a = cpi(s.bvh_a, s.n_bvh);
  s.bvh_b = cpi(s.bvh_b, s.n_bvh);
  s.bvh_prim = cpi(s.bvh_prim, s.n_tri + s.n_sph);
  s.tri_f32 = nullptr;
  if (s.n_sph == 0 && s.n_tri <= kLinearMaxPrims) {
    // fp32 filter table in scan order (16-byte aligned after the int arrays)
    uintptr_t a = reinterpret_cast<uintptr_t>(ip);
    a = (a + 15) & ~(uintptr_t)15;
    float* f = reinterpret_cast<float*>(a);
    if (s.filter_items) {  // host-built items (paired parallelograms)
      for (int i = threadIdx.x; i < 16 * s.n_filter; i += blockDim.x) f[i] = s.filter_items[i];
    } else {
      __syncthreads();  // the staged doubles / prim order are read below
      for (int k = threadIdx.x; k < s.n_tri; k += blockDim.x) {
        const int pid = s.bvh_prim[k];
        const double* v0 = s.tri_v0 + 3 * pid;
        const double* e1 = s.tri_e1 + 3 * pid;
        const double* e2 = s.tri_e2 + 3 * pid;
        float* row = f + 16 * k;
        for (int c = 0; c < 3; ++c) {
          row[c] = (float)v0[c];
          row[4 + c] = (float)e1[c];
          row[8 + c] = (float)e2[c];
        }
        // L1 norms of the fp32-rounded vectors, rounded up
        row[3] = (fabsf(row[4]) + fabsf(row[5]) + fabsf(row[6])) * 1.0001f;
        row[7] = (fabsf(row[8]) + fabsf(row[9]) + fabsf(row[10])) * 1.0001f;
        row[11] = (fabsf(row[0]) + fabsf(row[1]) + fabsf(row[2])) * 1.0001f;
        row[12] = 1.0f;            // triangle
        row[13] = 1.000001e-9f;    // the reference's barycentric slack
        row[14] = __uint_as_float(k < 32 ? 1u << k : 0u);  // candidate mask
        row[15] = __uint_as_float(k >= 32 ? 1u << (k - 32) : 0u);
      }
      s.n_filter = s.n_tri;
    }
    s.tri_f32 = f;
  }
  __syncthreads();
}

}  // namespace pt
}  // namespace nirc
