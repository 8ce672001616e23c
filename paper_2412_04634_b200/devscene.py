"""Device copy of a scene pack + the ``nirc_scene_t`` the C ABI consumes."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib


LINEAR_MAX_PRIMS = 64  # pt_common.cuh kLinearMaxPrims
TRI_SLACK = np.float32(1.000001e-9)   # the reference's barycentric 1e-9 (ray_tri_s)
PAIR_SLACK = np.float32(2.2e-9)       # a parallelogram's union of two triangles


def _l1_up(v):
    return np.float32((np.abs(v).sum()) * np.float32(1.0001))


def filter_items(p):
    """fp32 pre-test items of the warp-uniform scan (pt_common.cuh
    tri_candidate) for a small triangle-only scene: the triangles in BVH
    scan order, with each pair (v0, a, a + b), (v0, a + b, b) -- a quad the
    scene file split along its diagonal -- merged into one parallelogram
    item (v0, a, b) when the diagonal is a + b to 1e-13.  (n_items, 16) f32."""
    order = np.asarray(p.bvh_prim, np.int64)
    v0 = np.asarray(p.tri_v0, np.float64)[order]
    e1 = np.asarray(p.tri_e1, np.float64)[order]
    e2 = np.asarray(p.tri_e2, np.float64)[order]
    n = len(order)
    by_a = {}
    for k in range(n):
        by_a.setdefault((v0[k].tobytes(), e2[k].tobytes()), []).append(k)
    partner = [-1] * n
    for k in range(n):  # k as the second triangle (v0, a + b, b)
        if partner[k] >= 0:
            continue
        for j in by_a.get((v0[k].tobytes(), e1[k].tobytes()), []):
            if j == k or partner[j] >= 0:
                continue
            a, b = e1[j], e2[k]
            if np.abs(e2[j] - (a + b)).sum() <= 1e-13 * (np.abs(a).sum() + np.abs(b).sum()):
                partner[j], partner[k] = k, j
                break
    rows = []
    done = [False] * n
    for k in range(n):
        if done[k]:
            continue
        row = np.zeros(16, np.float32)
        j = partner[k]
        if j >= 0:  # k and j: the item is v0 + u a + v b over the unit square
            ka, kb = (k, j) if e2[k].tobytes() == e1[j].tobytes() else (j, k)
            ea, eb = e1[ka], e2[kb]
            cu, slack, bits = 0.0, PAIR_SLACK, (1 << k) | (1 << j)
            done[j] = True
        else:
            ka, ea, eb = k, e1[k], e2[k]
            cu, slack, bits = 1.0, TRI_SLACK, 1 << k
        f0, fa, fb = (v0[ka].astype(np.float32), ea.astype(np.float32),
                      eb.astype(np.float32))
        row[0:3], row[3] = f0, _l1_up(fa)
        row[4:7], row[7] = fa, _l1_up(fb)
        row[8:11], row[11] = fb, _l1_up(f0)
        row[12], row[13] = cu, slack
        row[14:16] = np.array([bits & 0xFFFFFFFF, bits >> 32], np.uint32).view(np.float32)
        done[k] = True
        rows.append(row)
    return np.stack(rows) if rows else np.zeros((0, 16), np.float32)


class DeviceScene:
    _F64 = ("tri_v0", "tri_e1", "tri_e2", "tri_ng", "tri_area", "tri_lq", "sph_c", "sph_r",
            "sph_lq", "mat_albedo", "mat_rough", "mat_emit", "lt_cdf", "lt_q", "env_img",
            "bvh_lo", "bvh_hi")
    _I32 = ("tri_mat", "sph_mat", "mat_kind", "lt_kind", "lt_prim", "bvh_a", "bvh_b",
            "bvh_prim")

    def __init__(self, scene):
        p = scene.pack
        self.tensors = {}
        s = _lib.NircScene()
        for name in self._F64:
            self._put(s, name, np.asarray(getattr(p, name), np.float64))
        for name in self._I32:
            self._put(s, name, np.asarray(getattr(p, name), np.int32))
        s.n_tri = len(p.tri_v0)
        s.n_sph = len(p.sph_c)
        s.n_mat = len(p.mat_kind)
        s.n_light = len(p.lt_kind)
        s.n_bvh = len(p.bvh_a)
        s.env_kind = int(p.env_kind)
        s.env_h, s.env_w = int(p.env_img.shape[0]), int(p.env_img.shape[1])
        for i in range(3):
            s.env_c0[i], s.env_c1[i], s.env_c2[i] = p.env_c0[i], p.env_c1[i], p.env_c2[i]
            s.bbox_min[i] = p.bbox_min[i]
            s.bbox_inv_ext[i] = p.bbox_inv_ext[i]
        s.env_q = float(p.env_q)
        s.eps = float(p.eps)
        s.diag = float(p.diag)
        s.bvh_packed = None
        s.prim_packed = None
        s.filter_items = None
        s.n_filter = 0
        if s.n_sph == 0 and 0 < s.n_tri <= LINEAR_MAX_PRIMS:
            items = filter_items(p)
            self._put(s, "filter_items", items)
            s.n_filter = items.shape[0]
        self.struct = s
        self.cam = torch.from_numpy(np.ascontiguousarray(scene.camera, np.float64)).cuda()
        if s.n_sph > 0 or s.n_tri > LINEAR_MAX_PRIMS:
            # front-to-back traversal image for general scenes (the small
            # triangle-only scenes take the warp-uniform scan)
            lib = _lib.load()
            nbytes = int(lib.nirc_scene_packed_bytes(C.byref(s)))
            self.tensors["packed"] = t = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            _lib.check(lib.nirc_pack_scene(C.byref(s), t.data_ptr(), nbytes,
                                           torch.cuda.current_stream().cuda_stream),
                       "nirc_pack_scene")

    def _put(self, s, name, arr):
        t = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1).copy()
                             if arr.size else np.zeros(1, arr.dtype)).cuda()
        self.tensors[name] = t
        setattr(s, name, t.data_ptr())

    def ptr(self):
        return C.byref(self.struct)
