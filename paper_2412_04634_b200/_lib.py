"""ctypes binding of the C-ABI library (include/nirc_b200.h).

The library is the product path: if ``libnirc_b200.so`` is missing or a CUDA
device is absent, every compute call raises instead of falling back to a CPU
implementation.  ``load()`` builds the library in-tree when sources are newer
(nvcc cross-compiles; no GPU is needed to build).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import threading

import numpy as np

from .errors import ConfigError, DivergenceError, InvalidSampleError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnirc_b200.so")

NIRC_OK = 0
NIRC_E_CONFIG = 2
NIRC_E_DIVERGENCE = 3
NIRC_E_BAD_PDF = 4
NIRC_E_CUDA = 5
NIRC_E_UNSUPPORTED = 6

MAX_LAYERS = 9
MAX_LEVELS = 16


class NircSpec(C.Structure):
    """Mirror of ``nirc_spec_t`` (NetSpec, pkg/src/nirclab/mlp.py:26-33)."""

    _fields_ = [
        ("levels", C.c_int32), ("table_log2", C.c_int32), ("feats", C.c_int32),
        ("bands", C.c_int32), ("in_dim", C.c_int32), ("n_layers", C.c_int32),
        ("out_act", C.c_int32), ("pad0", C.c_int32),
        ("dims", C.c_int32 * (MAX_LAYERS + 1)),
        ("pad1", C.c_int32 * 2),
        ("w_off", C.c_int64 * MAX_LAYERS),
        ("b_off", C.c_int64 * MAX_LAYERS),
        ("res", C.c_int32 * MAX_LEVELS),
        ("bb_min", C.c_double * 3),
        ("bb_inv", C.c_double * 3),
        ("grid_len", C.c_int64), ("theta_len", C.c_int64),
        ("sh_k", C.c_double * 64),
    ]


class NircRecords(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in
                ("pos", "ns", "alb", "rough", "dirs", "target", "pdf")] + [
        ("n", C.c_int64)]


class NircTrainOpts(C.Structure):
    """nirc_train_opts_t: Adam hyper-parameters + the deterministic switch."""
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("deterministic", C.c_int32), ("reserved", C.c_int32)]


def train_opts(adam, deterministic=False):
    return NircTrainOpts(float(adam.beta1), float(adam.beta2), float(adam.eps),
                         1 if deterministic else 0, 0)


class NircRecordsOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in
                ("pos", "ns", "alb", "rough", "dirs", "target", "pdf")] + [
        ("cap", C.c_int64)]


class NircScene(C.Structure):
    _fields_ = [
        ("n_tri", C.c_int32), ("n_sph", C.c_int32), ("n_mat", C.c_int32),
        ("n_light", C.c_int32), ("n_bvh", C.c_int32), ("env_kind", C.c_int32),
        ("env_h", C.c_int32), ("env_w", C.c_int32),
        ("tri_v0", C.c_void_p), ("tri_e1", C.c_void_p), ("tri_e2", C.c_void_p),
        ("tri_ng", C.c_void_p), ("tri_area", C.c_void_p), ("tri_lq", C.c_void_p),
        ("tri_mat", C.c_void_p),
        ("sph_c", C.c_void_p), ("sph_r", C.c_void_p), ("sph_lq", C.c_void_p),
        ("sph_mat", C.c_void_p),
        ("mat_kind", C.c_void_p),
        ("mat_albedo", C.c_void_p), ("mat_rough", C.c_void_p), ("mat_emit", C.c_void_p),
        ("lt_kind", C.c_void_p), ("lt_prim", C.c_void_p),
        ("lt_cdf", C.c_void_p), ("lt_q", C.c_void_p),
        ("env_img", C.c_void_p),
        ("env_c0", C.c_double * 3), ("env_c1", C.c_double * 3), ("env_c2", C.c_double * 3),
        ("env_q", C.c_double), ("eps", C.c_double), ("diag", C.c_double),
        ("bbox_min", C.c_double * 3), ("bbox_inv_ext", C.c_double * 3),
        ("bvh_lo", C.c_void_p), ("bvh_hi", C.c_void_p),
        ("bvh_a", C.c_void_p), ("bvh_b", C.c_void_p), ("bvh_prim", C.c_void_p),
        ("tri_f32", C.c_void_p),
        ("bvh_packed", C.c_void_p), ("prim_packed", C.c_void_p),
        ("filter_items", C.c_void_p), ("n_filter", C.c_int32), ("pad_filter", C.c_int32),
    ]


class NircRenderCfg(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("spp", C.c_int32), ("cache_on", C.c_int32),
        ("max_cv", C.c_int32), ("nc", C.c_int32 * 8),
        ("rough_cut", C.c_double), ("rr_survive", C.c_double),
        ("seed", C.c_uint64), ("frame", C.c_uint64),
        ("width", C.c_int32), ("height", C.c_int32),
        ("row0", C.c_int32), ("row1", C.c_int32),
        ("precision", C.c_int32), ("nbias", C.c_int32),
        ("sph_c", C.c_double), ("v1", C.c_void_p),
    ]


P = C.c_void_p
I32, I64, U64, F64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
SPEC = C.POINTER(NircSpec)

# name -> (restype, argtypes); exactly the declarations of include/nirc_b200.h
SIGNATURES = {
    "nirc_version": (C.c_char_p, []),
    "nirc_last_error": (I32, [C.c_char_p, I32]),
    "nirc_device_sm_count": (I32, []),
    "nirc_stage_timing": (I32, [I32]),
    "nirc_stage_times": (I32, [P, I32]),
    "nirc_encode": (I32, [SPEC, P, P, P, P, P, P, I64, P, P, P, P]),
    "nirc_scatter_grid_grad": (I32, [SPEC, P, P, P, P, I64, I64, P]),
    "nirc_mlp_forward": (I32, [SPEC, P, P, I64, P, P, P, P]),
    "nirc_mlp_backward": (I32, [SPEC, P, P, P, P, I64, P, P, P, P]),
    "nirc_full_forward": (I32, [SPEC, P, P, P, P, P, P, I64, P, I32, P, P]),
    "nirc_loss": (I32, [I32, P, P, P, P, F64, I64, P, P, P, P, P]),
    "nirc_encode_f64": (I32, [SPEC, P, P, P, P, P, P, I64, P, P, P, P]),
    "nirc_mlp_forward_f64": (I32, [SPEC, P, P, I64, P, P, P, P]),
    "nirc_mlp_backward_f64": (I32, [SPEC, P, P, P, P, I64, P, P, P, P]),
    "nirc_scatter_grid_grad_f64": (I32, [SPEC, P, P, P, P, I64, I64, P]),
    "nirc_loss_f64": (I32, [I32, P, P, P, P, P, F64, I64, P, P, P, P]),
    "nirc_adam_step_f64": (I32, [P, P, P, P, I64, P, P, F64, F64, F64, F64, P, P]),
    "nirc_adam_step": (I32, [P, P, P, P, I64, P, P, F64, F64, F64, F64, P, P, P]),
    "nirc_train_step": (I32, [SPEC, P, P, P, P, P, C.POINTER(NircRecords), U64, I64, I32,
                              I32, I32, F64, F64, C.POINTER(NircTrainOpts), P, P, P, P, P,
                              I64, P]),
    "nirc_train_workspace_bytes": (I64, [SPEC, I64, I32]),
    "nirc_train_frame": (I32, [SPEC, P, P, P, P, P, C.POINTER(NircRecords), U64, I64, I32,
                               I32, I32, F64, F64, C.POINTER(NircTrainOpts), P, P, P, P, I64,
                               P]),
    "nirc_train_frame_workspace_bytes": (I64, [SPEC, I64, I32, I32]),
    "nirc_train_tiles": (I64, [I64, I32]),
    "nirc_train_grad": (I32, [SPEC, P, C.POINTER(NircRecords), U64, I64, I32, I32, I32, F64,
                              C.POINTER(NircTrainOpts), I64, I64, P, P, P, P, P, I64, P]),
    "nirc_train_apply": (I32, [SPEC, P, P, P, P, P, P, P, I64, F64, C.POINTER(NircTrainOpts),
                               P, P, P, P]),
    "nirc_render": (I32, [C.POINTER(NircScene), P, C.POINTER(NircRenderCfg), SPEC, P, P, P,
                          P, P, P, I64, P]),
    "nirc_render_workspace_bytes": (I64, [C.POINTER(NircRenderCfg)]),
    "nirc_render_collect": (I32, [C.POINTER(NircScene), P, C.POINTER(NircRenderCfg), SPEC, P,
                                  P, P, P, P, U64, U64, I64, I64, I32,
                                  C.POINTER(NircRecordsOut), P, P, I64, P]),
    "nirc_render_collect_workspace_bytes": (I64, [C.POINTER(NircRenderCfg), I64]),
    "nirc_collect": (I32, [C.POINTER(NircScene), P, U64, U64, I64, I32,
                           C.POINTER(NircRecordsOut), P, P, I64, P]),
    "nirc_collect_workspace_bytes": (I64, [I64]),
    "nirc_surface_samples": (I32, [C.POINTER(NircScene), P, P, I32, P, I32, P, P, P, P, P]),
    "nirc_incident_targets": (I32, [C.POINTER(NircScene), U64, U64, P, P, F64, P, I32, P, P,
                                    P]),
    "nirc_integrand_samples": (I32, [C.POINTER(NircScene), P, U64, U64, I32, P, P, P, P, P, P,
                                     P, P, P, P]),
    "nirc_query": (I32, [SPEC, P, P, I64, P, P, I64, P, I32, P, P]),
    "nirc_bvh_node_count": (I64, [I64]),
    "nirc_scene_packed_bytes": (I64, [C.POINTER(NircScene)]),
    "nirc_pack_scene": (I32, [C.POINTER(NircScene), P, I64, P]),
    "nirc_build_bvh": (I32, [P, P, P, I64, P, P, I64, P, P, P, P, P, P]),
    "nirc_occluded": (I32, [C.POINTER(NircScene), P, P, I64, F64, P, P]),
    "nirc_pt_radiance": (I32, [C.POINTER(NircScene), P, C.POINTER(NircRenderCfg), I32, I32, I32,
                               P, P]),
    "nirc_collect_range": (I32, [C.POINTER(NircScene), P, U64, U64, I64, I64, I32,
                                 C.POINTER(NircRecordsOut), P, P, I64, P]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load (building if stale) the sm_100a library; raises if impossible."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        from . import build as _build

        # build only when the library is absent (or NIRC_REBUILD=1): a
        # snapshot copied to the GPU box may carry shuffled mtimes and must
        # use the library built by __graft_entry__.build()
        if not os.path.exists(LIB_PATH) or os.environ.get("NIRC_REBUILD") == "1":
            _build.build(force=os.environ.get("NIRC_REBUILD") == "1")
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension missing: {LIB_PATH}")
        # NIRC_LIB_PATH: another in-tree build of the same library (tools' A/B runs)
        lib = C.CDLL(os.environ.get("NIRC_LIB_PATH", LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error():
    buf = C.create_string_buffer(512)
    load().nirc_last_error(buf, 512)
    return buf.value.decode(errors="replace")


FLAG_BAD_PDF = 1       # include/nirc_b200.h NIRC_FLAG_*
FLAG_DIVERGED = 2
FLAG_BAD_INDEX = 4


def check_flags(flags, what="nirc call"):
    """Raise the reference's exception for a device status word (reads it:
    synchronises with the stream that wrote it)."""
    v = int(flags[0].item()) if hasattr(flags, "item") else int(flags)
    if v & FLAG_DIVERGED:
        raise DivergenceError(f"{what}: non-finite network parameter")
    if v & FLAG_BAD_PDF:
        raise InvalidSampleError(f"{what}: pdf <= 0")
    if v & FLAG_BAD_INDEX:
        raise ConfigError(f"{what}: dir_to_surf index outside [0, n_surf)")


def check(status, what="nirc call"):
    """Map a C status onto the reference's exception types."""
    if status == NIRC_OK:
        return
    msg = f"{what}: {last_error()}"
    if status == NIRC_E_CONFIG:
        raise ConfigError(msg)
    if status == NIRC_E_DIVERGENCE:
        raise DivergenceError(msg)
    if status == NIRC_E_BAD_PDF:
        raise InvalidSampleError(msg)
    if status == NIRC_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------- spec ----

def _sh_k_table():
    """NORM[l,0] and sqrt(2)*NORM[l,m] with sh.py:21-33's expression order."""
    out = np.zeros(64)
    sqrt2 = math.sqrt(2.0)
    for l in range(8):
        for m in range(l + 1):
            norm = math.sqrt((2 * l + 1) / (4.0 * math.pi) * math.factorial(l - m)
                             / math.factorial(l + m))
            out[l * 8 + m] = norm if m == 0 else sqrt2 * norm
    return out


_SH_K = _sh_k_table()


def make_c_spec(spec):
    """nirc_spec_t for a NetSpec namedtuple (cached on the spec object id)."""
    s = NircSpec()
    table = int(spec.table)
    if table & (table - 1):
        raise ConfigError(f"hash table size {table} is not a power of two")
    s.levels = int(spec.levels)
    s.table_log2 = table.bit_length() - 1
    s.feats = int(spec.feats)
    s.bands = int(spec.bands)
    s.in_dim = int(spec.in_dim)
    s.n_layers = int(spec.nl)
    s.out_act = int(spec.out_act)
    if s.n_layers > MAX_LAYERS or s.levels > MAX_LEVELS:
        raise ConfigError("network exceeds the C-ABI limits")
    for i, d in enumerate(spec.dims):
        s.dims[i] = int(d)
    for i in range(s.n_layers):
        s.w_off[i] = int(spec.w_off[i])
        s.b_off[i] = int(spec.b_off[i])
    for i, r in enumerate(spec.res):
        s.res[i] = int(r)
    for i in range(3):
        s.bb_min[i] = float(spec.bb_min[i])
        s.bb_inv[i] = float(spec.bb_inv[i])
    s.grid_len = int(spec.grid_len)
    s.theta_len = int(spec.theta_len)
    for i in range(64):
        s.sh_k[i] = float(_SH_K[i])
    return s
