// Layouts of the BVH traversal image (nirc_pack_scene in bvh.cu, walked by
// bvh_scan_packed in pt_common.cuh).
#pragma once

namespace nirc {
namespace pt {

// per internal node: both child boxes -- fp32, rounded outward (lo down, hi
// up) -- and child references (n > 0: leaf, primitives [c, c + n) of the
// leaf order; n == 0: internal node c)
struct alignas(16) PackedNode {
  float lo0[3], hi0[3], lo1[3], hi1[3];
  int c0, n0, c1, n1;
};
// primitives in leaf order with their geometry inline
struct alignas(16) PackedPrim {
  double g[9];   // triangle: v0, e1, e2; sphere: centre, radius
  int id, kind;  // triangle / sphere index; 0 = triangle, 1 = sphere
};
static_assert(sizeof(PackedNode) == 64, "PackedNode layout");
static_assert(sizeof(PackedPrim) == 80, "PackedPrim layout");

}  // namespace pt
}  // namespace nirc
