"""Device copy of a scene pack + the ``nirc_scene_t`` the C ABI consumes."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib


LINEAR_MAX_PRIMS = 64  # pt_common.cuh kLinearMaxPrims


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
