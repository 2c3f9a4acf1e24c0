"""ctypes loader for libtrigraph_b200.so (the C ABI in include/trigraph_b200.h).

There is no fallback: if the in-tree library is missing, importing the
package raises.  Build it with ``python -c "import __graft_entry__ as g; g.build()"``
or ``make -C paper_1706_05151_b200/csrc``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TG_LIB_PATH: an alternative build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("TG_LIB_PATH") or os.path.join(HERE, "libtrigraph_b200.so")

TG_OK = 0
TG_ERR_INVALID_ARGUMENT = 1
TG_ERR_CUDA = 2
TG_ERR_OOM = 3
TG_ERR_CAPACITY = 4
TG_ERR_INTERNAL = 5
TG_ERR_PARSE = 6


class TgConfig(C.Structure):
    _fields_ = [
        ("engine", C.c_int32),
        ("cost", C.c_int32),
        ("ranks", C.c_uint64),
        ("boundaries", C.c_void_p),
        ("track_nodes", C.c_int32),
        ("collect_triangles", C.c_int32),
        ("sparsify", C.c_int32),
        ("sparsify_q", C.c_double),
        ("sparsify_seed", C.c_uint64),
        ("order_set", C.c_int32),
        ("order", C.c_int32),
        ("order_seed", C.c_uint64),
    ]


class TgRankStats(C.Structure):
    _fields_ = [
        ("triangles", C.c_uint64),
        ("data_sent", C.c_uint64),
        ("data_recv", C.c_uint64),
        ("realized_cost", C.c_uint64),
        ("stored_entries", C.c_uint64),
    ]


# Every symbol include/trigraph_b200.h declares, with its ctypes signature.
_vp, _u64, _u32, _i32, _dbl = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_double
_pvp, _pu64 = C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)
SIGNATURES = {
    "tg_graph_from_edges": (_i32, [C.c_int, _vp, _u64, _u64, _pvp]),
    "tg_graph_from_csr": (_i32, [C.c_int, _u64, _vp, _vp, _pvp]),
    "tg_count_from_csr": (_i32, [C.c_int, _u64, _vp, _vp, _pu64]),
    "tg_count_from_csr_range": (_i32, [C.c_int, _u64, _vp, _vp, _u64, _u64, _pu64]),
    "tg_graph_free": (_i32, [_vp]),
    "tg_graph_info": (_i32, [_vp, _pu64, _pu64]),
    "tg_graph_csr": (_i32, [_vp, _vp, _vp]),
    "tg_set_stream": (_i32, [_vp, _vp]),
    "tg_set_order": (_i32, [_vp, _i32, _u64]),
    "tg_set_order_rank": (_i32, [_vp, _vp]),
    "tg_comm_unique_id": (_i32, [_vp]),
    "tg_comm_init": (_i32, [C.c_int, C.c_int, C.c_int, _vp, _pvp]),
    "tg_comm_init_local": (_i32, [C.c_int, _vp, _vp]),
    "tg_comm_free": (_i32, [_vp]),
    "tg_comm_info": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i32)]),
    "tg_graph_from_rows": (_i32, [C.c_int, _u64, _u32, _u32, _vp, _vp, _vp, _pvp]),
    "tg_run_engine_comm": (_i32, [_vp, _vp, C.POINTER(TgConfig), _pu64, _vp, _vp]),
    "tg_aop_step_comm": (_i32, [_vp, _vp, _vp, _vp]),
    "tg_orient_rows_device": (_i32, [_vp, _u32, _u32, _pu64]),
    "tg_clustering_comm": (_i32, [_vp, _vp, C.POINTER(TgConfig), _vp, _vp, _vp]),
    "tg_eff_from_csr": (_i32, [C.c_int, _u64, _vp, _vp, _pvp]),
    "tg_eff_free": (_i32, [_vp]),
    "tg_eff_count": (_i32, [_vp, _pu64, _vp, _vp, _u64, _i32, _pu64]),
    "tg_graph_from_text": (_i32, [C.c_int, _vp, _u64, _u64, _pvp, _pu64]),
    "tg_parse_edge_list": (_i32, [C.c_int, _vp, _u64, _vp, _u64, _pu64, _pu64]),
    "tg_write_edge_list": (_i32, [_vp, _vp, _u64, _pu64]),
    "tg_coreness": (_i32, [_vp, _vp]),
    "tg_compute_order": (_i32, [_vp, _vp]),
    "tg_effective_adjacency": (_i32, [_vp, _vp, _vp]),
    "tg_ordering_cost": (_i32, [_vp, _pu64]),
    "tg_node_costs": (_i32, [_vp, _i32, _vp, _vp]),
    "tg_compute_boundaries": (_i32, [_vp, _i32, _u64, _vp]),
    "tg_count": (_i32, [_vp, _pu64]),
    "tg_count_node_iterator_pp": (_i32, [_vp, _i32, _pu64]),
    "tg_run_engine": (_i32, [_vp, C.POINTER(TgConfig), _pu64, _vp, _vp, _vp, _vp, _u64, _pu64]),
    "tg_clustering_coefficients": (_i32, [_vp, C.POINTER(TgConfig), _vp, _vp]),
    "tg_approx_count": (_i32, [_vp, _u64, _i32, _dbl, _u64, _vp, _i32, C.POINTER(_dbl)]),
    "tg_per_edge_triangle_counts": (_i32, [_vp, _vp]),
    "tg_variance_report": (_i32, [_vp, _vp, _u64, _dbl, _vp, _vp]),
    "tg_step_device": (_i32, [_vp, _vp]),
    "tg_orient_device": (_i32, [_vp]),
    "tg_count_device": (_i32, [_vp, _vp]),
    "tg_aop_rank_device": (_i32, [_vp, _vp, _u64, _u64, _vp]),
    "tg_aop_rank_sinks_device": (_i32, [_vp, _vp, _u64, _u64, _vp, _vp, _vp, _u64, _vp]),
    "tg_cc_from_tally_device": (_i32, [_vp, _vp, _vp]),
    "tg_surrogate_pack_sizes": (_i32, [_vp, _vp, _u64, _u64, _vp, _vp]),
    "tg_surrogate_pack_device": (_i32, [_vp, _vp, _u64, _u64, _vp, _vp]),
    "tg_surrogate_count_device": (_i32, [_vp, _vp, _u64, _u64, _vp, _u64, _vp, _vp]),
    "tg_last_error": (C.c_char_p, []),
    "tg_status_string": (C.c_char_p, [_i32]),
    "tg_kernel_launches": (_u64, []),
    "tg_last_intersect_ms": (_dbl, [_vp]),
    "tg_debug_set_block_cap": (None, [_u32]),
    "tg_debug_set_chunk_entries": (None, [_u64]),
    "tg_debug_set_warp_variant": (None, [_i32]),
    "tg_debug_set_paths": (None, [_i32, _i32]),
    "tg_debug_set_window": (None, [_i32]),
    "tg_debug_set_slab": (None, [_i32]),
    "tg_debug_set_rank_bitmap": (None, [_i32, _u32]),
    "tg_gen_pa": (_i32, [_u64, _u64, _u64, _pvp, _pu64]),
    "tg_gen_gnp": (_i32, [_u64, _dbl, _u64, _pvp, _pu64]),
    "tg_gen_gnm": (_i32, [_u64, _u64, _u64, _pvp, _pu64]),
    "tg_gen_rmat": (_i32, [_u32, _u64, _dbl, _dbl, _dbl, _u64, _pvp, _pu64]),
    "tg_gen_ws": (_i32, [_u64, _u64, _dbl, _u64, _pvp, _pu64]),
    "tg_free_host": (None, [_vp]),
    "tg_graph_from_rmat": (_i32, [C.c_int, _u32, _u64, _dbl, _dbl, _dbl, _u64, _pvp]),
    "tg_graph_from_ws": (_i32, [C.c_int, _u64, _u64, _dbl, _u64, _pvp]),
}

_lib = None


class TrigraphError(RuntimeError):
    """A non-argument failure reported by the library (CUDA, OOM, internal)."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


class ParseError(RuntimeError):
    """io.hpp:18-22 trigraph::ParseError: what() = "line N: ...", .line = N."""

    def __init__(self, line: int, msg: str):
        super().__init__(msg)
        self.line = line


def check(status: int, err_line: int = 0) -> None:
    """Map tg_status to the reference's exception types."""
    if status == TG_OK:
        return
    msg = lib().tg_last_error().decode(errors="replace")
    if status == TG_ERR_PARSE:
        raise ParseError(err_line, msg)
    if status == TG_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)  # reference: std::invalid_argument
    if status == TG_ERR_OOM:
        raise MemoryError(msg)
    raise TrigraphError(status, f"{lib().tg_status_string(status).decode()}: {msg}")
