"""C-ABI library: loads on CPU, exports every symbol include/forkattn.h
declares, host-only pool semantics, hashing known answers (no GPU calls)."""

import ctypes
import json
import os
import re

import pytest

from paper_2405_19888_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "forkattn.h")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(syms) == bound, set(syms) ^ bound


def test_library_is_sm100a():
    info = _lib.build_info()
    assert "sm_100a" in info
    # the fatbin must carry sm_100a SASS, not only PTX
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_fnv_known_answers():
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    assert _lib.fnv1a64_u32([], 0xCBF29CE484222325) == int(kat["empty"])
    for case in kat["ids"]:
        assert _lib.fnv1a64_u32(case["ids"], int(case["seed"])) == int(case["hash"])
    for case in kat["chains"]:
        assert _lib.fnv1a64_chain(case["segments"], 0xCBF29CE484222325) == [int(h) for h in case["chain"]]


def _pool(total=100, device=-1, L=1, H=4):
    desc = _lib.PoolDesc(num_layers=L, num_heads=H, head_dim=128, block_size=16, total_blocks=total,
                         num_pages=0, device=device, reserved=0)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.fk_pool_create(ctypes.byref(desc), ctypes.byref(h)))
    return h


def test_host_only_pool_grow_release_and_errors():
    h = _pool(total=10)
    L = _lib.lib
    assert L.fk_ctx_create(h, 1, -1) == _lib.FK_OK
    assert L.fk_ctx_create(h, 2, 99) == _lib.FK_UNKNOWN_PARENT_CONTEXT
    assert L.fk_ctx_create(h, 2, 1) == _lib.FK_OK
    ids = (ctypes.c_int64 * 16)()
    n = ctypes.c_int64()
    assert L.fk_ctx_grow(h, 1, 100, ids, 16, ctypes.byref(n)) == _lib.FK_OK
    assert n.value == 7 and list(ids[:7]) == list(range(7))
    # atomic OOM: 4 more blocks do not fit in 3 free
    assert L.fk_ctx_grow(h, 2, 64, ids, 16, ctypes.byref(n)) == _lib.FK_OUT_OF_MEMORY
    st = _lib.PoolStats()
    L.fk_pool_stats_get(h, ctypes.byref(st))
    assert (st.used_blocks, st.free_blocks, st.peak_used, st.next_block) == (7, 3, 7, 7)
    assert L.fk_ctx_release(h, 1) == _lib.FK_CONTEXT_BUSY  # still has a child
    assert L.fk_ctx_release(h, 2) == _lib.FK_OK
    assert L.fk_ctx_release(h, 1) == _lib.FK_OK
    assert L.fk_ctx_release(h, 1) == _lib.FK_UNKNOWN_CONTEXT
    L.fk_pool_stats_get(h, ctypes.byref(st))
    assert (st.used_blocks, st.peak_used, st.next_block) == (0, 7, 7)  # ids never recycled
    # compute entry points refuse on a host-only pool
    assert L.fk_attn_decode(h, 0, None, None, None, None) in (_lib.FK_NO_DEVICE, _lib.FK_INVALID_ARGUMENT)
    assert L.fk_pool_destroy(h) == _lib.FK_OK


def test_invalid_geometry_rejected():
    for kw in (dict(block_size=8), dict(head_dim=64), dict(num_layers=0)):
        base = dict(num_layers=1, num_heads=4, head_dim=128, block_size=16, total_blocks=10, num_pages=0,
                    device=-1, reserved=0)
        base.update(kw)
        desc = _lib.PoolDesc(**base)
        h = ctypes.c_void_p()
        assert _lib.lib.fk_pool_create(ctypes.byref(desc), ctypes.byref(h)) == _lib.FK_INVALID_ARGUMENT
        assert "must" in _lib.last_error() or "geometry" in _lib.last_error()


def test_status_maps_to_reference_exception_classes():
    from paper_2405_19888_b200 import errors

    with pytest.raises(errors.OutOfMemory) as e:
        _lib.check(_lib.FK_OUT_OF_MEMORY)
    assert e.value.code == "out_of_memory"
    with pytest.raises(errors.UnknownContext):
        _lib.check(_lib.FK_UNKNOWN_CONTEXT)
    with pytest.raises(errors.UnknownParentContext):
        _lib.check(_lib.FK_UNKNOWN_PARENT_CONTEXT)
    with pytest.raises(errors.ContextBusy):
        _lib.check(_lib.FK_CONTEXT_BUSY)
    with pytest.raises(errors.KernelError):
        _lib.check(_lib.FK_CUDA_ERROR)


def test_step_grow_sequential_oom_rule():
    """fk_step_grow: rows grow one token in row order; a row whose page does
    not fit fails alone (engine.py:431-438), later rows that need no new page
    still grow, ids come from the monotonic counter."""
    h = _pool(total=4)
    L = _lib.lib
    for ctx, parent in ((1, -1), (2, 1), (3, 1), (4, 1)):
        assert L.fk_ctx_create(h, ctx, parent) == _lib.FK_OK
    ids = (ctypes.c_int64 * 8)()
    n = ctypes.c_int64()
    assert L.fk_ctx_grow(h, 1, 16, ids, 8, ctypes.byref(n)) == _lib.FK_OK  # block 0
    assert L.fk_ctx_grow(h, 2, 16, ids, 8, ctypes.byref(n)) == _lib.FK_OK  # block 1 (full page)
    assert L.fk_ctx_grow(h, 3, 5, ids, 8, ctypes.byref(n)) == _lib.FK_OK   # block 2 (room left)
    assert L.fk_ctx_grow(h, 4, 16, ids, 8, ctypes.byref(n)) == _lib.FK_OK  # block 3: pool full
    leaves = (ctypes.c_int64 * 3)(2, 3, 4)
    info = _lib.PlanInfo()
    assert L.fk_step_plan(h, leaves, 3, 1, None, ctypes.byref(info)) == _lib.FK_OK
    assert info.batch_tokens == 16 + 16 + 5 + 16
    pos = (ctypes.c_int64 * 3)()
    new = (ctypes.c_int64 * 3)()
    nf = ctypes.c_int32()
    assert L.fk_step_grow(h, pos, new, ctypes.byref(nf)) == _lib.FK_OK
    # row 0 (ctx 2) needs a new page -> OOM; row 1 (ctx 3) fits its page; row 2 needs one -> OOM
    assert list(pos) == [-1, 5, -1] and nf.value == 2
    assert list(new) == [-1, -1, -1]
    tok = ctypes.c_int64()
    nb = ctypes.c_int64()
    par = ctypes.c_int64()
    L.fk_ctx_info(h, 3, ctypes.byref(tok), ctypes.byref(nb), ctypes.byref(par))
    assert (tok.value, nb.value, par.value) == (6, 1, 1)
    assert L.fk_ctx_tokens(h, 3) == 6 and L.fk_ctx_tokens(h, 99) == -1
    L.fk_pool_destroy(h)


def test_device_entry_points_refuse_host_only_pools():
    h = _pool(total=10)
    L = _lib.lib
    assert L.fk_ctx_create(h, 1, -1) == _lib.FK_OK
    ids = (ctypes.c_int64 * 4)()
    n = ctypes.c_int64()
    assert L.fk_ctx_grow(h, 1, 20, ids, 4, ctypes.byref(n)) == _lib.FK_OK
    assert L.fk_fill_kv(h, 1, 0, 20, 0, 1, None, None, None) == _lib.FK_NO_DEVICE
    assert L.fk_ctx_copy_kv(h, 1, h, 1, 20, None) == _lib.FK_NO_DEVICE
    assert L.fk_synth_fill(h, 1, 0, 20, 1, 1.0, None) == _lib.FK_NO_DEVICE
    leaves = (ctypes.c_int64 * 1)(1)
    info = _lib.PlanInfo()
    assert L.fk_step_plan(h, leaves, 1, 1, None, ctypes.byref(info)) == _lib.FK_OK
    assert L.fk_attn_decode_layers(h, 0, 1, None, 0, None, 0, None, 0, None) == _lib.FK_NO_DEVICE
    L.fk_pool_destroy(h)


def test_options_validate():
    h = _pool()
    L = _lib.lib
    for opt, val in ((_lib.FK_OPT_TC_MIN_FANOUT, 0), (_lib.FK_OPT_CORUN, 0), (_lib.FK_OPT_PREFIX_RATE_PCT, 60),
                     (_lib.FK_OPT_PDL, 2), (_lib.FK_OPT_PRIV_MIN_CHUNK, 4), (_lib.FK_OPT_PRIV_STATIC_FIRST, 0),
                     (_lib.FK_OPT_LAUNCH_ORDER, 1), (_lib.FK_OPT_GRAPH, 0), (_lib.FK_OPT_TC_BOUNDARY_COST, 2),
                     (_lib.FK_OPT_APPEND_FIRST, 1)):
        assert L.fk_pool_set_option(h, opt, val) == _lib.FK_OK
    # unknown, and the options removed in round 2 (tcgen05 dynamic tail: 10 and
    # 13; fused merge: 15 -- measured slower)
    for opt in (999, 10, 13, 15):
        assert L.fk_pool_set_option(h, opt, 1) == _lib.FK_INVALID_ARGUMENT
    for warps in (8, 10, 12):
        assert L.fk_pool_set_option(h, _lib.FK_OPT_PRIV_WARPS, warps) == _lib.FK_OK
    for warps in (5, 6, 9, 11, 13, 14):
        assert L.fk_pool_set_option(h, _lib.FK_OPT_PRIV_WARPS, warps) == _lib.FK_INVALID_ARGUMENT
    L.fk_pool_destroy(h)
