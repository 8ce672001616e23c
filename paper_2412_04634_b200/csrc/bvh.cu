// Device BVH build: the reference's median-split BVH (build_bvh,
// pkg/src/nirclab/geometry.py:213-274) built on the GPU with an identical
// node array, so traversal order -- and with it every tie between equal hit
// distances -- is the host build's (larger scenes).
//
// The split positions depend only on segment sizes (a node over n > 4
// primitives sends n / 2 to the left child), so the node layout -- DFS
// preorder index, [start, start + count) range of the primitive order,
// depth, right-child link -- is planned on the host from P alone.  What
// depends on the geometry is the permutation: every internal node sorts its
// range stably by the centroid coordinate along the axis of largest centroid
// extent.  The device runs that level by level:
//   1. centroid bounds of every internal node at this depth (one thread per
//      primitive slot, binary search for its node, atomics on order-
//      preserving 64-bit keys -- min / max are exact, so the result equals
//      numpy's c.min / c.max);
//   2. key1 = the centroid coordinate along the node's axis (argmax of the
//      extents, first on ties), key2 = the node's start; slots outside this
//      depth's internal nodes (finished leaves) key on their own position;
//   3. two stable radix sorts (key1, then key2) = a stable sort of every
//      node's range by its centroid key, leaving finished ranges in place.
// Node bounds are min / max over the node's primitives, computed bottom-up
// afterwards (leaf: its <= 4 primitives; internal: union of the children --
// the same exact min / max).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "nirc_b200.h"
#include "common.cuh"
#include "pt_packed.cuh"

namespace nirc {
namespace {

constexpr int kLeafMax = 4;

// order-preserving map of a double to uint64 (total order, -0 < +0 is
// avoided by canonicalising the zero before the map)
__device__ __forceinline__ uint64_t okey(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(__dadd_rn(x, 0.0));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void k_prim_bounds(const double* v0, const double* e1, const double* e2, int64_t nt,
                              const double* sc, const double* sr, int64_t ns, double* plo,
                              double* phi, double* cent, int32_t* perm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt + ns) return;
  for (int c = 0; c < 3; ++c) {
    double lo, hi;
    if (i < nt) {
      const double a = v0[3 * i + c];
      const double b = __dadd_rn(a, e1[3 * i + c]);
      const double d = __dadd_rn(a, e2[3 * i + c]);
      lo = fmin(fmin(a, b), d);
      hi = fmax(fmax(a, b), d);
    } else {
      const int64_t j = i - nt;
      lo = __dsub_rn(sc[3 * j + c], sr[j]);
      hi = __dadd_rn(sc[3 * j + c], sr[j]);
    }
    plo[3 * i + c] = lo;
    phi[3 * i + c] = hi;
    cent[3 * i + c] = __dmul_rn(0.5, __dadd_rn(lo, hi));
  }
  perm[i] = (int32_t)i;
}

// index of the internal node (of this depth) whose range holds slot i, or -1
__device__ __forceinline__ int find_node(const int64_t* start, const int64_t* count, int n,
                                         int64_t i) {
  int lo = 0, hi = n;  // first start > i
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (start[mid] <= i) lo = mid + 1;
    else hi = mid;
  }
  const int s = lo - 1;
  return (s >= 0 && i < start[s] + count[s]) ? s : -1;
}

__global__ void k_init_bounds(uint64_t* cb, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int c = 0; c < 3; ++c) {
    cb[6 * i + c] = ~0ull;     // min
    cb[6 * i + 3 + c] = 0ull;  // max
  }
}

__global__ void k_cent_bounds(const int64_t* start, const int64_t* count, int n, int64_t P,
                              const int32_t* perm, const double* cent, uint64_t* cb) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int s = i < P ? find_node(start, count, n, i) : -1;
  uint64_t mn[3], mx[3];
  if (s >= 0) {
    const int32_t p = perm[i];
    for (int c = 0; c < 3; ++c) mn[c] = mx[c] = okey(cent[3 * p + c]);
  } else {
    for (int c = 0; c < 3; ++c) {
      mn[c] = ~0ull;
      mx[c] = 0ull;
    }
  }
  // warp-level combine when the whole warp works on one node (the common
  // case above the bottom levels), else per-thread atomics
  const int s0 = __shfl_sync(0xffffffffu, s, 0);
  const bool uniform = __all_sync(0xffffffffu, s == s0);
  if (uniform) {
    if (s0 < 0) return;
    for (int o = 16; o > 0; o >>= 1)
      for (int c = 0; c < 3; ++c) {
        mn[c] = min(mn[c], (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)mn[c], o));
        mx[c] = max(mx[c], (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)mx[c], o));
      }
    if ((threadIdx.x & 31) != 0) return;
  } else if (s < 0) {
    return;
  }
  const int t = uniform ? s0 : s;
  for (int c = 0; c < 3; ++c) {
    atomicMin(reinterpret_cast<unsigned long long*>(cb + 6 * t + c), (unsigned long long)mn[c]);
    atomicMax(reinterpret_cast<unsigned long long*>(cb + 6 * t + 3 + c),
              (unsigned long long)mx[c]);
  }
}

__global__ void k_split_keys(const int64_t* start, const int64_t* count, int n, int64_t P,
                             const int32_t* perm, const double* cent, const uint64_t* cb,
                             uint64_t* key1, uint64_t* val) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int s = find_node(start, count, n, i);
  const int32_t p = perm[i];
  uint64_t k1, k2;
  if (s >= 0) {
    // axis = argmax(c.max(axis=0) - c.min(axis=0)), the first on ties
    int axis = 0;
    double best = 0.0;
    for (int c = 0; c < 3; ++c) {
      const double e = __dsub_rn(okey_inv(cb[6 * s + 3 + c]), okey_inv(cb[6 * s + c]));
      if (c == 0 || e > best) {
        best = e;
        axis = c;
      }
    }
    k1 = okey(cent[3 * p + axis]);
    k2 = (uint64_t)start[s];
  } else {
    k1 = (uint64_t)i;
    k2 = (uint64_t)i;
  }
  key1[i] = k1;
  val[i] = (k2 << 32) | (uint32_t)p;
}

__global__ void k_unpack(const uint64_t* val, uint32_t* key2, int32_t* perm, int64_t P) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  key2[i] = (uint32_t)(val[i] >> 32);
  perm[i] = (int32_t)(val[i] & 0xffffffffu);
}

// bottom-up node bounds over the nodes of one depth
__global__ void k_node_bounds(const int32_t* nodes, int n, const int32_t* a, const int32_t* b,
                              const int32_t* perm, const double* plo, const double* phi,
                              double* lo, double* hi) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int node = nodes[k];
  for (int c = 0; c < 3; ++c) {
    double l, h;
    if (b[node] > 0) {
      l = plo[3 * perm[a[node]] + c];
      h = phi[3 * perm[a[node]] + c];
      for (int j = 1; j < b[node]; ++j) {
        l = fmin(l, plo[3 * perm[a[node] + j] + c]);
        h = fmax(h, phi[3 * perm[a[node] + j] + c]);
      }
    } else {
      l = fmin(lo[3 * (node + 1) + c], lo[3 * a[node] + c]);
      h = fmax(hi[3 * (node + 1) + c], hi[3 * a[node] + c]);
    }
    lo[3 * node + c] = l;
    hi[3 * node + c] = h;
  }
}

struct Plan {
  std::vector<int64_t> start, count;
  std::vector<int32_t> depth, a, b;
  int max_depth = 0;
};

// build_bvh's emit recursion on sizes alone: DFS preorder, left subtree first
Plan plan_nodes(int64_t P) {
  Plan pl;
  struct Item {
    int64_t start, count;
    int32_t depth, patch;
  };
  std::vector<Item> st{{0, P, 0, -1}};
  while (!st.empty()) {
    const Item it = st.back();
    st.pop_back();
    const int32_t me = (int32_t)pl.a.size();
    if (it.patch >= 0) pl.a[it.patch] = me;
    pl.start.push_back(it.start);
    pl.count.push_back(it.count);
    pl.depth.push_back(it.depth);
    pl.max_depth = std::max(pl.max_depth, (int)it.depth);
    if (it.count <= kLeafMax) {
      pl.a.push_back((int32_t)it.start);
      pl.b.push_back((int32_t)it.count);
      continue;
    }
    pl.a.push_back(0);
    pl.b.push_back(0);
    const int64_t half = it.count / 2;
    st.push_back({it.start + half, it.count - half, it.depth + 1, me});
    st.push_back({it.start, half, it.depth + 1, -1});
  }
  return pl;
}

int64_t node_count(int64_t P) {
  if (P <= kLeafMax) return 1;
  return 1 + node_count(P / 2) + node_count(P - P / 2);
}

}  // namespace
}  // namespace nirc

using namespace nirc;

extern "C" int64_t nirc_bvh_node_count(int64_t n_prims) {
  return n_prims <= 0 ? 1 : node_count(n_prims);
}

extern "C" int nirc_build_bvh(const double* tri_v0, const double* tri_e1, const double* tri_e2,
                              int64_t n_tri, const double* sph_c, const double* sph_r,
                              int64_t n_sph, double* lo, double* hi, int32_t* a, int32_t* b,
                              int32_t* prim, void* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t P = n_tri + n_sph;
  if (n_tri < 0 || n_sph < 0 || P >= (int64_t(1) << 31)) {
    set_last_error("primitive counts out of range");
    return NIRC_E_CONFIG;
  }
  if (P == 0) {  // a single empty leaf pointing at itself
    NIRC_CUDA_TRY(cudaMemsetAsync(lo, 0, 3 * sizeof(double), s));
    NIRC_CUDA_TRY(cudaMemsetAsync(hi, 0, 3 * sizeof(double), s));
    NIRC_CUDA_TRY(cudaMemsetAsync(a, 0, sizeof(int32_t), s));
    NIRC_CUDA_TRY(cudaMemsetAsync(b, 0, sizeof(int32_t), s));
    return NIRC_OK;
  }
  const Plan pl = plan_nodes(P);
  const int N = (int)pl.a.size();
  // per-depth lists: internal nodes (start, count) for the sorts, all nodes
  // for the bottom-up bounds
  const int D = pl.max_depth + 1;
  std::vector<std::vector<int32_t>> internal(D), all(D);
  for (int i = 0; i < N; ++i) {
    all[pl.depth[i]].push_back(i);
    if (pl.b[i] == 0) internal[pl.depth[i]].push_back(i);
  }
  std::vector<int64_t> h_start, h_count;
  std::vector<int32_t> h_nodes;
  std::vector<int> in_off(D + 1, 0), all_off(D + 1, 0);
  for (int d = 0; d < D; ++d) {
    in_off[d] = (int)h_start.size();
    for (int i : internal[d]) {
      h_start.push_back(pl.start[i]);
      h_count.push_back(pl.count[i]);
    }
    all_off[d] = (int)h_nodes.size();
    for (int i : all[d]) h_nodes.push_back(i);
  }
  in_off[D] = (int)h_start.size();
  all_off[D] = (int)h_nodes.size();
  int max_in = 1;
  for (int d = 0; d < D; ++d) max_in = std::max(max_in, in_off[d + 1] - in_off[d]);

  // workspace
  size_t sort_bytes = 0, sort2_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint64_t*)nullptr,
                                  (uint64_t*)nullptr, (const uint64_t*)nullptr,
                                  (uint64_t*)nullptr, (int)P, 0, 64, s);
  cub::DeviceRadixSort::SortPairs(nullptr, sort2_bytes, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)P, 0, 32, s);
  sort_bytes = std::max(sort_bytes, sort2_bytes);
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t b_pd = up(9 * P * sizeof(double));                       // plo, phi, cent
  const size_t b_perm = up(2 * P * sizeof(int32_t));                    // perm x2
  const size_t b_keys = up(4 * P * sizeof(uint64_t));                   // key1 x2, val x2
  const size_t b_k2 = up(2 * P * sizeof(uint32_t));                     // key2 x2
  const size_t b_plan = up(h_start.size() * 2 * sizeof(int64_t) + 8);   // starts, counts
  const size_t b_nodes = up(h_nodes.size() * sizeof(int32_t) + 4);
  const size_t b_ab = up(2 * (size_t)N * sizeof(int32_t));
  const size_t b_cb = up((size_t)max_in * 6 * sizeof(uint64_t));
  const size_t total = b_pd + b_perm + b_keys + b_k2 + b_plan + b_nodes + b_ab + b_cb +
                       up(sort_bytes);
  AsyncBuf wsb(s);
  NIRC_CUDA_TRY(wsb.alloc(total));
  char* q = static_cast<char*>(wsb.p);
  double* plo = reinterpret_cast<double*>(q);
  double* phi = plo + 3 * P;
  double* cent = phi + 3 * P;
  q += b_pd;
  int32_t* perm = reinterpret_cast<int32_t*>(q);
  int32_t* perm2 = perm + P;
  q += b_perm;
  uint64_t* key1 = reinterpret_cast<uint64_t*>(q);
  uint64_t* key1s = key1 + P;
  uint64_t* val = key1s + P;
  uint64_t* vals = val + P;
  q += b_keys;
  uint32_t* key2 = reinterpret_cast<uint32_t*>(q);
  uint32_t* key2s = key2 + P;
  q += b_k2;
  int64_t* d_start = reinterpret_cast<int64_t*>(q);
  int64_t* d_count = d_start + h_start.size();
  q += b_plan;
  int32_t* d_nodes = reinterpret_cast<int32_t*>(q);
  q += b_nodes;
  int32_t* d_a = reinterpret_cast<int32_t*>(q);
  int32_t* d_b = d_a + N;
  q += b_ab;
  uint64_t* cb = reinterpret_cast<uint64_t*>(q);
  q += b_cb;
  void* tmp = q;

  if (!h_start.empty()) {
    NIRC_CUDA_TRY(cudaMemcpyAsync(d_start, h_start.data(), h_start.size() * sizeof(int64_t),
                                  cudaMemcpyHostToDevice, s));
    NIRC_CUDA_TRY(cudaMemcpyAsync(d_count, h_count.data(), h_count.size() * sizeof(int64_t),
                                  cudaMemcpyHostToDevice, s));
  }
  NIRC_CUDA_TRY(cudaMemcpyAsync(d_nodes, h_nodes.data(), h_nodes.size() * sizeof(int32_t),
                                cudaMemcpyHostToDevice, s));
  NIRC_CUDA_TRY(cudaMemcpyAsync(d_a, pl.a.data(), N * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  NIRC_CUDA_TRY(cudaMemcpyAsync(d_b, pl.b.data(), N * sizeof(int32_t), cudaMemcpyHostToDevice, s));

  const unsigned gP = (unsigned)((P + 255) / 256);
  k_prim_bounds<<<gP, 256, 0, s>>>(tri_v0, tri_e1, tri_e2, n_tri, sph_c, sph_r, n_sph, plo, phi,
                                   cent, perm);
  NIRC_LAUNCH_CHECK("k_prim_bounds");
  for (int d = 0; d < D; ++d) {
    const int n = in_off[d + 1] - in_off[d];
    if (n == 0) continue;
    const int64_t* st = d_start + in_off[d];
    const int64_t* ct = d_count + in_off[d];
    k_init_bounds<<<(n + 255) / 256, 256, 0, s>>>(cb, n);
    k_cent_bounds<<<gP, 256, 0, s>>>(st, ct, n, P, perm, cent, cb);
    k_split_keys<<<gP, 256, 0, s>>>(st, ct, n, P, perm, cent, cb, key1, val);
    NIRC_LAUNCH_CHECK("k_split_keys");
    size_t tb = sort_bytes;
    NIRC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, key1, key1s, val, vals, (int)P, 0, 64,
                                                  s));
    k_unpack<<<gP, 256, 0, s>>>(vals, key2, perm2, P);
    tb = sort_bytes;
    NIRC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, key2, key2s, perm2, perm, (int)P, 0,
                                                  32, s));
  }
  for (int d = D - 1; d >= 0; --d) {
    const int n = all_off[d + 1] - all_off[d];
    k_node_bounds<<<(n + 127) / 128, 128, 0, s>>>(d_nodes + all_off[d], n, d_a, d_b, perm, plo,
                                                  phi, lo, hi);
  }
  NIRC_LAUNCH_CHECK("k_node_bounds");
  NIRC_CUDA_TRY(cudaMemcpyAsync(a, d_a, N * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  NIRC_CUDA_TRY(cudaMemcpyAsync(b, d_b, N * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  NIRC_CUDA_TRY(cudaMemcpyAsync(prim, perm, P * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  // the host plan vectors are read by the async copies above
  NIRC_CUDA_TRY(cudaStreamSynchronize(s));
  return NIRC_OK;
}

// ---------------------------------------------------------------------
// Traversal image for the front-to-back walk (pt_common.cuh
// bvh_scan_packed): per internal node both child boxes + references, and
// the primitives in leaf order with their geometry inline.
namespace nirc {
namespace {

__global__ void k_pack_nodes(nirc_scene_t s, pt::PackedNode* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.n_bvh) return;
  pt::PackedNode nd{};
  if (s.bvh_b[i] == 0 && s.bvh_a[i] != i) {
    const int ch[2] = {i + 1, s.bvh_a[i]};
    for (int c = 0; c < 2; ++c) {
      const int k = ch[c];
      float* lo = c == 0 ? nd.lo0 : nd.lo1;
      float* hi = c == 0 ? nd.hi0 : nd.hi1;
      for (int a = 0; a < 3; ++a) {
        lo[a] = __double2float_rd(s.bvh_lo[3 * k + a]);
        hi[a] = __double2float_ru(s.bvh_hi[3 * k + a]);
      }
      const bool leaf = s.bvh_b[k] > 0;
      (c == 0 ? nd.c0 : nd.c1) = leaf ? s.bvh_a[k] : k;
      (c == 0 ? nd.n0 : nd.n1) = leaf ? s.bvh_b[k] : 0;
    }
  }
  out[i] = nd;
}

__global__ void k_pack_prims(nirc_scene_t s, pt::PackedPrim* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= s.n_tri + s.n_sph) return;
  pt::PackedPrim q{};
  const int pid = s.bvh_prim[k];
  if (pid < s.n_tri) {
    for (int a = 0; a < 3; ++a) {
      q.g[a] = s.tri_v0[3 * pid + a];
      q.g[3 + a] = s.tri_e1[3 * pid + a];
      q.g[6 + a] = s.tri_e2[3 * pid + a];
    }
    q.id = pid;
    q.kind = 0;
  } else {
    const int j = pid - s.n_tri;
    for (int a = 0; a < 3; ++a) q.g[a] = s.sph_c[3 * j + a];
    q.g[3] = s.sph_r[j];
    q.id = j;
    q.kind = 1;
  }
  out[k] = q;
}

size_t packed_node_bytes(const nirc_scene_t& s) {
  return ((size_t)s.n_bvh * sizeof(pt::PackedNode) + 255) & ~size_t(255);
}

}  // namespace
}  // namespace nirc

extern "C" int64_t nirc_scene_packed_bytes(const nirc_scene_t* scene) {
  return (int64_t)(packed_node_bytes(*scene) +
                   (size_t)(scene->n_tri + scene->n_sph + 1) * sizeof(pt::PackedPrim));
}

extern "C" int nirc_pack_scene(nirc_scene_t* scene, void* out, int64_t out_bytes, void* stream) {
  if (out_bytes < nirc_scene_packed_bytes(scene)) {
    set_last_error("packed scene buffer too small");
    return NIRC_E_CONFIG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto* nodes = reinterpret_cast<pt::PackedNode*>(out);
  auto* prims = reinterpret_cast<pt::PackedPrim*>(reinterpret_cast<char*>(out) +
                                                   packed_node_bytes(*scene));
  nirc_scene_t sc = *scene;
  sc.bvh_packed = nullptr;
  sc.prim_packed = nullptr;
  if (sc.n_bvh > 0)
    k_pack_nodes<<<(sc.n_bvh + 127) / 128, 128, 0, s>>>(sc, nodes);
  const int np = sc.n_tri + sc.n_sph;
  if (np > 0) k_pack_prims<<<(np + 127) / 128, 128, 0, s>>>(sc, prims);
  NIRC_LAUNCH_CHECK("k_pack_scene");
  scene->bvh_packed = nodes;
  scene->prim_packed = prims;
  return NIRC_OK;
}
