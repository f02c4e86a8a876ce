"""ctypes binding of libforkattn.so (include/forkattn.h).

This is the binding a reference maintainer would add next to
semflow/engine.py: plain pointers and sizes, no torch
types.  The library is built in-tree by `make -C paper_2405_19888_b200/csrc`
(or __graft_entry__.build()); importing this module without it raises.
"""

from __future__ import annotations

import array
import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int32, c_int64, c_size_t, c_uint8, c_uint32, c_uint64, c_void_p

from .errors import ContextBusy, KernelError, OutOfMemory, UnknownContext, UnknownParentContext

LIB_PATH = os.environ.get("FK_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libforkattn.so")

FK_OK = 0
FK_OUT_OF_MEMORY = 1
FK_UNKNOWN_CONTEXT = 2
FK_UNKNOWN_PARENT_CONTEXT = 3
FK_CONTEXT_BUSY = 4
FK_INVALID_ARGUMENT = 5
FK_CUDA_ERROR = 6
FK_NO_DEVICE = 7

FK_OPT_TC_MIN_FANOUT = 1
FK_OPT_PREFIX_TARGET_CTAS = 2
FK_OPT_LAUNCH_ORDER = 3
FK_OPT_MIN_SPLIT_PAGES = 4
FK_OPT_CORUN = 5
FK_OPT_PREFIX_RATE_PCT = 6
FK_OPT_PDL = 7
FK_OPT_PRIV_MIN_CHUNK = 8
FK_OPT_PRIV_STATIC_FIRST = 9
FK_OPT_PRIV_WARPS = 11
FK_OPT_GRAPH = 12
FK_OPT_TC_BOUNDARY_COST = 14
FK_OPT_APPEND_FIRST = 16
FK_OPT_GROUP_FANOUT = 18
FK_OPT_DEBUG_SKIP_MERGE = 90


class PoolDesc(ctypes.Structure):
    _fields_ = [
        ("num_layers", c_int32),
        ("num_heads", c_int32),
        ("head_dim", c_int32),
        ("block_size", c_int32),
        ("total_blocks", c_int64),
        ("num_pages", c_int64),
        ("device", c_int32),
        ("reserved", c_int32),
    ]


class PoolStats(ctypes.Structure):
    _fields_ = [
        ("used_blocks", c_int64),
        ("free_blocks", c_int64),
        ("peak_used", c_int64),
        ("total_blocks", c_int64),
        ("next_block", c_int64),
        ("num_pages", c_int64),
        ("free_pages", c_int64),
        ("arena_bytes", c_int64),
        ("host_wait_ns", c_int64),
        ("graph_replays", c_int64),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("batch_tokens", c_int64),
        ("shared_tokens", c_int64),
        ("private_tokens", c_int64),
        ("num_rows", c_int32),
        ("num_shared_ctx", c_int32),
        ("num_prefix_ctas", c_int32),
        ("max_slots", c_int32),
        ("num_tc_items", c_int32),
        ("num_mma_items", c_int32),
        ("fused_merge", c_int32),
        ("streamed_tokens", c_int64),
    ]


# (name, restype, argtypes) for every symbol of include/forkattn.h
SIGNATURES = [
    ("fk_pool_create", c_int32, [POINTER(PoolDesc), POINTER(c_void_p)]),
    ("fk_pool_destroy", c_int32, [c_void_p]),
    ("fk_pool_set_total_blocks", c_int32, [c_void_p, c_int64]),
    ("fk_pool_reserve_pages", c_int32, [c_void_p, c_int64]),
    ("fk_pool_stats_get", c_int32, [c_void_p, POINTER(PoolStats)]),
    ("fk_pool_set_option", c_int32, [c_void_p, c_int32, c_int64]),
    ("fk_last_error", c_char_p, []),
    ("fk_ctx_create", c_int32, [c_void_p, c_int64, c_int64]),
    ("fk_ctx_grow", c_int32, [c_void_p, c_int64, c_int64, POINTER(c_int64), c_int64, POINTER(c_int64)]),
    ("fk_ctx_release", c_int32, [c_void_p, c_int64]),
    ("fk_ctx_info", c_int32, [c_void_p, c_int64, POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
    ("fk_ctx_tokens", c_int64, [c_void_p, c_int64]),
    ("fk_ctx_blocks", c_int32, [c_void_p, c_int64, POINTER(c_int64), POINTER(c_int32), c_int64, POINTER(c_int64)]),
    ("fk_step_plan", c_int32, [c_void_p, POINTER(c_int64), c_int32, c_int32, c_void_p, POINTER(PlanInfo)]),
    ("fk_attn_decode", c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("fk_attn_decode_layers", c_int32, [c_void_p, c_int32, c_int32, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                        c_int64, c_void_p]),
    ("fk_step_grow", c_int32, [c_void_p, POINTER(c_int64), POINTER(c_int64), POINTER(c_int32)]),
    ("fk_step_commit", c_int32, [c_void_p, POINTER(c_int64), c_void_p]),
    ("fk_append_kv", c_int32, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    ("fk_append_kv_layers", c_int32, [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    ("fk_fill_kv", c_int32, [c_void_p, c_int64, c_int64, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    ("fk_ctx_copy_kv", c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p]),
    ("fk_synth_fill", c_int32, [c_void_p, c_int64, c_int64, c_int64, c_uint64, c_float, c_void_p]),
    ("fk_synth_queries", c_int32, [c_void_p, c_uint64, c_void_p, c_int32, c_void_p]),
    ("fk_synth_append", c_int32, [c_void_p, c_uint64, c_float, c_void_p]),
    ("fk_fnv1a64_u32", c_uint64, [POINTER(c_uint32), c_size_t, c_uint64]),
    ("fk_fnv1a64_chain", c_int32, [POINTER(c_uint32), POINTER(c_int64), c_int32, c_uint64, POINTER(c_uint64)]),
    ("fk_build_info", c_char_p, []),
]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2405_19888_b200/csrc` "
            "(the product path has no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

_ERRORS = {
    FK_OUT_OF_MEMORY: OutOfMemory,
    FK_UNKNOWN_CONTEXT: UnknownContext,
    FK_UNKNOWN_PARENT_CONTEXT: UnknownParentContext,
    FK_CONTEXT_BUSY: ContextBusy,
}


def last_error() -> str:
    msg = lib.fk_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    if status == FK_OK:
        return
    cls = _ERRORS.get(status, KernelError)
    raise cls(last_error() or f"forkattn status {status}")


def build_info() -> str:
    return lib.fk_build_info().decode()


def _u32_buffer(ids):
    """Token ids as a contiguous u32 buffer (array.array: one C loop, no
    per-element ctypes objects); ids outside u32 wrap like struct.pack would
    refuse to -- the reference only hashes u32 ids."""
    try:
        return array.array("I", ids)
    except (OverflowError, TypeError):
        return array.array("I", [int(t) & 0xFFFFFFFF for t in ids])


def fnv1a64_u32(ids, seed: int) -> int:
    """hash_token_ids (tokenizer.py:47-49) through the C-ABI."""
    arr = _u32_buffer(ids)
    n = len(arr)
    ptr = arr.buffer_info()[0] if n else None
    return int(lib.fk_fnv1a64_u32(ctypes.cast(ptr, POINTER(c_uint32)) if ptr else None, n,
                                  seed & 0xFFFFFFFFFFFFFFFF))


def fnv1a64_chain(segments, seed: int):
    """Chained segment hashes (prefix.py:78-85) in one C call."""
    flat = _u32_buffer([t for seg in segments for t in seg])
    offs = [0]
    for seg in segments:
        offs.append(offs[-1] + len(seg))
    ids = ctypes.cast(flat.buffer_info()[0], POINTER(c_uint32)) if len(flat) else (c_uint32 * 1)()
    off = (c_int64 * len(offs))(*offs)
    out = (c_uint64 * max(len(segments), 1))()
    check(lib.fk_fnv1a64_chain(ids, off, len(segments), seed & 0xFFFFFFFFFFFFFFFF, out))
    return [int(out[i]) for i in range(len(segments))]
