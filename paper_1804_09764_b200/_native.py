"""ctypes binding of libcc.so (include/cc.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  There is no
fallback: if libcc.so is missing or fails to load, importing this module
raises ImportError."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1804_09764_b200.build` "
                      "(or __graft_entry__.build())")

lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)

c_i32, c_i64, c_u32, c_u64, c_dbl, vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                         ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p)


class cc_options(ctypes.Structure):
    _fields_ = [("precision", c_i32), ("device", c_i32), ("world", c_i32), ("rank", c_i32),
                ("nccl_id", vp), ("chunk_cols", c_i64), ("segment_len", c_i32),
                ("use_graphs", c_i32), ("relabel_seed", c_u64), ("fixed_root", c_i32), ("replicas", c_i32),
                ("loopback", vp), ("exchange", c_i32)]


CC_OK, CC_ERR_ARG, CC_ERR_GRAPH, CC_ERR_TEMPLATE, CC_ERR_STATE, CC_ERR_OOM, CC_ERR_CUDA, \
    CC_ERR_NCCL, CC_ERR_NONFINITE = range(9)
CC_FP64, CC_FP32 = 0, 1
CC_EXCHANGE_AUTO, CC_EXCHANGE_GROUPED, CC_EXCHANGE_RING, CC_EXCHANGE_ALLTOALL, CC_EXCHANGE_DEVICE = 0, 1, 2, 3, 4
STATUS_NAMES = ["CC_OK", "CC_ERR_ARG", "CC_ERR_GRAPH", "CC_ERR_TEMPLATE", "CC_ERR_STATE", "CC_ERR_OOM",
                "CC_ERR_CUDA", "CC_ERR_NCCL", "CC_ERR_NONFINITE"]

# every symbol declared in include/cc.h, with its signature
SIGNATURES = {
    "cc_default_options": (c_i32, [vp]),
    "cc_nccl_unique_id": (c_i32, [vp]),
    "cc_nccl_selftest": (c_i32, [c_i32]),
    "cc_nccl_device_selftest": (c_i32, [c_i32]),
    "cc_loopback_create": (c_i32, [c_i32, vp]),
    "cc_loopback_destroy": (None, [vp]),
    "cc_create": (c_i32, [vp, vp]),
    "cc_destroy": (None, [vp]),
    "cc_last_error": (ctypes.c_char_p, [vp]),
    "cc_load_graph": (c_i32, [vp, c_i64, vp, vp]),
    "cc_set_template": (c_i32, [vp, c_i32, vp]),
    "cc_set_template_colors": (c_i32, [vp, c_i32, vp, c_i32]),
    "cc_color": (c_i32, [vp, c_u64]),
    "cc_count_colorful": (c_i32, [vp, vp]),
    "cc_count_colorful_multi": (c_i32, [vp, c_i32, vp, vp, vp]),
    "cc_estimate": (c_i32, [vp, c_i32, c_u64, vp, vp]),
    "cc_set_colors": (c_i32, [vp, vp]),
    "cc_get_colors": (c_i32, [vp, vp]),
    "cc_template_info": (c_i32, [vp, vp, vp, vp]),
    "cc_get_subtree_counts": (c_i32, [vp, c_i32, vp]),
    "cc_get_subtree_rows": (c_i32, [vp, c_i32, vp, c_i32, vp]),
    "cc_estimate_mom": (c_i32, [vp, c_i32, c_u64, c_i32, vp, vp]),
    "cc_median_of_means": (c_i32, [vp, c_i32, c_i32, c_i64, c_i32, vp]),
    "cc_niter": (c_i32, [c_dbl, c_dbl, c_i32, c_dbl, vp]),
    "cc_last_profile": (c_i32, [vp, vp, c_i32, vp]),
    "cc_set_profiling": (c_i32, [vp, c_i32]),
    "cc_set_knob": (c_i32, [vp, ctypes.c_char_p, c_i32]),
    "cc_get_knob": (c_i32, [vp, ctypes.c_char_p, vp]),
    "cc_last_stats": (c_i32, [vp, vp, c_i32]),
    "cc_colex_rank": (c_i64, [c_u32]),
    "cc_colex_unrank": (c_u32, [c_i32, c_i64]),
    "cc_split_table": (c_i32, [c_i32, c_i32, c_i32, vp, c_i64]),
    "cc_zblock_table": (c_i32, [c_i32, c_i32, c_i32, vp, c_i64, vp, vp]),
    "cc_plan_template": (c_i32, [c_i32, vp, vp, c_i32, vp, vp, vp, vp, vp]),
    "cc_plan_template_auto": (c_i32, [c_i32, vp, c_dbl, c_i32, vp, c_i32, vp, vp, vp]),
    "cc_partition_plan":(c_i32, [c_i64, vp, vp, c_i32, c_i32, c_u64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "cc_exchange_model": (c_i32, [c_i64, vp, vp, c_i32, c_i32, c_u64, c_dbl, vp]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
