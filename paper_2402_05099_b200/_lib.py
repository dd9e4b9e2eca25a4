"""ctypes binding of libhydra.so (include/hydra.h): argument marshalling only.

The shared library is built in-tree by `paper_2402_05099_b200.build` (nvcc,
sm_100a).  There is no fallback: if the library is missing or fails to load,
every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HYDRA_LIB_PATH: load another build of the library (A/B timing of two builds on one box);
# HYDRA_TESTING=1: the testing build libhydra_test.so (diagnostics and the parity suite's
# sabotage switches, which the release libhydra.so does not contain).
RELEASE_LIB = os.path.join(_HERE, "libhydra.so")
TEST_LIB = os.path.join(_HERE, "libhydra_test.so")
LIB_PATH = os.environ.get("HYDRA_LIB_PATH") or (TEST_LIB if os.environ.get("HYDRA_TESTING") == "1" else RELEASE_LIB)

HYDRA_OK, HYDRA_EINVAL, HYDRA_ESHAPE, HYDRA_EUNSUPPORTED, HYDRA_ECUDA, HYDRA_ENCCL, HYDRA_ENOMEM = range(7)
HYDRA_BF16, HYDRA_F32, HYDRA_F16 = 0, 1, 2
HYDRA_OP_PREFIX, HYDRA_OP_SUFFIX, HYDRA_OP_ATTN, HYDRA_OP_PARTS = 0, 1, 2, 3
_STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ESHAPE", 3: "EUNSUPPORTED", 4: "ECUDA", 5: "ENCCL", 6: "ENOMEM"}

EXPORTED = ["hydra_prefix_attn", "hydra_suffix_attn", "hydra_combine", "hydra_attn", "hydra_tree_create",
            "hydra_tree_destroy", "hydra_tree_depth", "hydra_tree_group_size", "hydra_tree_workspace_size",
            "hydra_tree_attn", "hydra_workspace_size", "hydra_set_config", "hydra_get_config",
            "hydra_last_error", "hydra_version", "hydra_append_kv", "hydra_suffix_attn_paged", "hydra_attn_paged",
            "hydra_append_kv_paged", "hydra_tree_attn_paged", "hydra_tree_prepare", "hydra_debug_lens_violations",
            "hydra_combine_ex"]


class HydraError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: HYDRA_{_STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Heads(ctypes.Structure):
    _fields_ = [("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("scale", ctypes.c_float), ("dtype", ctypes.c_int32)]


class Paging(ctypes.Structure):
    """hydra_paging (include/hydra.h): block table [B, bt_stride] of a paged suffix cache."""
    _fields_ = [("block_table", ctypes.c_void_p), ("bt_stride", ctypes.c_int64), ("page_size", ctypes.c_int32),
                ("n_pages", ctypes.c_int64)]


class CombineDesc(ctypes.Structure):
    """hydra_combine_desc (include/hydra.h): two part groups with part / row strides."""
    _fields_ = [("rows", ctypes.c_int64), ("d", ctypes.c_int32), ("n_parts", ctypes.c_int32),
                ("o_parts", ctypes.c_void_p), ("o_dtype", ctypes.c_int32), ("o_part_stride", ctypes.c_int64),
                ("o_row_stride", ctypes.c_int64), ("lse_parts", ctypes.c_void_p), ("lse_part_stride", ctypes.c_int64),
                ("lse_row_stride", ctypes.c_int64), ("n_parts_f32", ctypes.c_int32), ("o_parts_f32", ctypes.c_void_p),
                ("o_f32_part_stride", ctypes.c_int64), ("o_f32_row_stride", ctypes.c_int64),
                ("lse_parts_f32", ctypes.c_void_p), ("lse_f32_part_stride", ctypes.c_int64),
                ("lse_f32_row_stride", ctypes.c_int64), ("out", ctypes.c_void_p), ("out_dtype", ctypes.c_int32),
                ("out_row_stride", ctypes.c_int64), ("lse_out", ctypes.c_void_p),
                ("lse_out_row_stride", ctypes.c_int64), ("out_table", ctypes.c_void_p),
                ("lse_out_table", ctypes.c_void_p), ("table_rows", ctypes.c_int64)]


_lib = None
_i64, _i32, _vp, _sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t
_HP = ctypes.POINTER(Heads)
_PP = ctypes.POINTER(Paging)


def load():
    """Load libhydra.so (raises if it is missing -- there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2402_05099_b200.build` "
                           "(or __graft_entry__.build()); the CUDA library is required")
    lib = ctypes.CDLL(LIB_PATH)
    st = ctypes.c_int32
    sig = {
        "hydra_prefix_attn": (st, [_HP, _i64, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
        "hydra_suffix_attn": (st, [_HP, _i64, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp,
                                   _vp, _sz, _vp]),
        "hydra_combine": (st, [_i64, _i32, _i32, _vp, _i32, _i64, _vp, _i64, _vp, _i32, _vp, _vp]),
        "hydra_combine_ex": (st, [ctypes.POINTER(CombineDesc), _vp]),
        "hydra_attn": (st, [_HP, _i64, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _i64,
                            _i64, _vp, _vp, _i32, _vp, _vp, _sz, _vp, _vp]),
        "hydra_tree_create": (st, [_vp, _vp, _vp, _i32, _vp, _i64, ctypes.POINTER(_vp)]),
        "hydra_tree_destroy": (None, [_vp]),
        "hydra_tree_prepare": (st, [_vp, _HP]),
        "hydra_debug_lens_violations": (_i64, [_i32]),
        "hydra_tree_depth": (_i32, [_vp]),
        "hydra_tree_group_size": (_i64, [_vp, _i32]),
        "hydra_tree_workspace_size": (_sz, [_HP, _vp, _i64]),
        "hydra_tree_attn": (st, [_HP, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _i64,
                                 _i64, _vp, _vp, _i32, _vp, _vp, _sz, _vp, _vp]),
        "hydra_workspace_size": (_sz, [ctypes.c_int, _HP, _i64, _i64, _i64, _i32]),
        "hydra_append_kv": (st, [_HP, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp]),
        "hydra_suffix_attn_paged": (st, [_HP, _i64, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _i64, _PP, _i64, _vp,
                                         _vp, _vp, _vp, _sz, _vp]),
        "hydra_attn_paged": (st, [_HP, _i64, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64,
                                  _i64, _PP, _i64, _vp, _vp, _i32, _vp, _vp, _sz, _vp, _vp]),
        "hydra_append_kv_paged": (st, [_HP, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _i64, _PP, _i64, _vp,
                                       _vp]),
        "hydra_tree_attn_paged": (st, [_HP, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64,
                                       _i64, _PP, _i64, _vp, _vp, _i32, _vp, _vp, _sz, _vp, _vp]),
        "hydra_set_config": (st, [ctypes.c_char_p, _i64]),
        "hydra_get_config": (_i64, [ctypes.c_char_p]),
        "hydra_last_error": (ctypes.c_char_p, []),
        "hydra_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(status: int, where: str) -> None:
    if status != HYDRA_OK:
        raise HydraError(status, where, load().hydra_last_error().decode())


def version() -> str:
    return load().hydra_version().decode()


def set_config(key: str, value: int) -> None:
    check(load().hydra_set_config(key.encode(), int(value)), f"set_config({key})")


def get_config(key: str) -> int:
    return int(load().hydra_get_config(key.encode()))
