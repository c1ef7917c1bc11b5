"""ctypes declaration of libinferlog_b200.so (include/il.h).  Argument marshalling only.

There is no fallback: if the shared library is missing or fails to load this module raises,
and every entry point of the package fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libinferlog_b200.so")
# profiling builds of the same sources (scripts/attn_variants.py) may be selected by name
if os.environ.get("IL_LIB_VARIANT"):
    LIB_PATH = os.path.join(HERE, "variants", f"libinferlog_b200_{os.environ['IL_LIB_VARIANT']}.so")

IL_OK, IL_ERR_ARG, IL_ERR_CAPACITY, IL_ERR_STATE, IL_ERR_INTERNAL, IL_ERR_CUDA = range(6)
STATUS_NAMES = {0: "IL_OK", 1: "IL_ERR_ARG", 2: "IL_ERR_CAPACITY", 3: "IL_ERR_STATE",
                4: "IL_ERR_INTERNAL", 5: "IL_ERR_CUDA"}
IL_SIM_COSINE, IL_SIM_JACCARD = 0, 1
IL_F_PAIR, IL_F_GUARD, IL_F_EXCLUDE_SELF, IL_F_VERIFY, IL_F_DEDUP = 1, 2, 4, 8, 16

# every symbol include/il.h declares (checked by tests/test_abi.py)
EXPORTS = ["il_workspace_bytes", "il_create", "il_destroy", "il_status_sync", "il_stats_sync", "il_stats_async",
           "il_last_error", "il_pool_load", "il_refine_batch", "il_prefix_match", "il_prefill_attn",
           "il_commit", "il_commit_index", "il_commit_records", "il_synth_qkv", "il_index_dump",
           "il_table_dump", "il_evicted_dump", "il_record_bytes", "il_commit_export", "il_commit_apply",
           "il_box_hit_dump", "il_select_batch", "il_synth_qkv_paged", "il_set_sm_split",
           "il_decode_attn"]


class ILError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class il_config(C.Structure):
    _fields_ = [("k", C.c_uint32), ("table_capacity", C.c_uint32), ("kv_pages", C.c_uint32),
                ("max_batch", C.c_uint32), ("max_prompt_tokens", C.c_uint32), ("max_pool", C.c_uint32),
                ("max_pool_tokens", C.c_uint32), ("max_log_tokens", C.c_uint32),
                ("max_suffix_tokens", C.c_uint32), ("n_q_heads", C.c_uint32), ("n_kv_heads", C.c_uint32),
                ("head_dim", C.c_uint32), ("metric", C.c_uint32), ("flags", C.c_uint32),
                ("hash_seed", C.c_uint64), ("max_global_batch", C.c_uint32), ("max_block_records", C.c_uint32),
                ("max_decode_tokens", C.c_uint32), ("reserved1", C.c_uint32)]


class il_refine_info(C.Structure):
    _fields_ = [("target_stamp", C.c_uint64), ("target_slot", C.c_int32), ("pmc", C.c_uint8),
                ("rule", C.c_uint8), ("reverted", C.c_uint8), ("matched", C.c_uint8)]


class il_stats(C.Structure):
    _fields_ = [("batch", C.c_uint64), ("resident_blocks", C.c_uint32), ("free_pages", C.c_uint32),
                ("table_entries", C.c_uint32), ("evicted_blocks", C.c_uint32), ("need_pages", C.c_uint32),
                ("suffix_tokens", C.c_uint32), ("index_rebuilds", C.c_uint32), ("status", C.c_uint32),
                ("launches", C.c_uint64), ("hit_blocks", C.c_uint32), ("box_hit_blocks", C.c_uint32),
                ("full_blocks", C.c_uint32), ("record_backlog", C.c_uint32), ("map_slots_used", C.c_uint32),
                ("dedup_blocks", C.c_uint32)]


assert C.sizeof(il_refine_info) == 16
assert C.sizeof(il_stats) == 72


_lib = None


def load():
    """Load libinferlog_b200.so (raises if it was not built: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    P, U32, U64, F32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_float
    sig = {
        "il_workspace_bytes": [C.POINTER(il_config), C.POINTER(C.c_size_t)],
        "il_create": [C.POINTER(il_config), P, C.c_size_t, P, C.POINTER(P)],
        "il_destroy": [P],
        "il_status_sync": [P, P],
        "il_stats_sync": [P, P, C.POINTER(il_stats)],
        "il_stats_async": [P, P, P],
        "il_pool_load": [P, U32, P, P, P, P, P, P, P, U32, P],
        "il_refine_batch": [P, U32, P, P, P, P, P, P, P, P, P],
        "il_prefix_match": [P, U32, P, P, P, P, P, P, P, P],
        "il_prefill_attn": [P, U32, P, P, P, P, P, P, P, P, P, P, F32, P],
        "il_decode_attn": [P, U32, P, P, P, P, P, P, P, P, P, F32, P],
        "il_commit": [P, P],
        "il_commit_index": [P, P],
        "il_commit_records": [P, U32, P, P, P],
        "il_synth_qkv": [P, U32, P, P, P, U64, F32, P, P, P, P],
        "il_synth_qkv_paged": [P, U32, P, P, P, P, U64, F32, P, P, P, P],
        "il_index_dump": [P, P, P, P, P, P, P],
        "il_table_dump": [P, P, P, P],
        "il_evicted_dump": [P, P, P, P],
        "il_record_bytes": [C.POINTER(il_config), C.POINTER(C.c_size_t)],
        "il_commit_export": [P, P, P],
        "il_commit_apply": [P, P, U32, P, P],
        "il_box_hit_dump": [P, P, P, U32],
        "il_select_batch": [P, U32, P, P, P, P, P],
        "il_set_sm_split": [P, U32],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.il_last_error.argtypes = []
    lib.il_last_error.restype = C.c_char_p
    _lib = lib
    return lib


def check(status: int, where: str) -> None:
    if status != IL_OK:
        raise ILError(status, where, load().il_last_error().decode(errors="replace"))
