"""Subprocess helper of tests/test_plan.py::test_auto_min_chunk (needs
FK_DEBUG_PLAN_DIGEST=1 at process start): for small fork groups with no
prefix grid, the plan built with the automatic minimum private chunk equals,
digest for digest, the plan built with FK_OPT_PRIV_MIN_CHUNK set to the value
the rule below predicts (restated from fk_pool.cpp's planner): over mc in
4..8, minimise (ceil(n/W) - n/W) * mc + 2 n/W, n = the guided chunk count, W
= the warps that start at once.  Prints one line per case and 'ok'."""

import ctypes
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2405_19888_b200 import _lib  # noqa: E402

W = 148 * 10      # host-only pool: 148 SMs, 10 private warps per CTA
MAX_CHUNK = 32


def chunk_count(U, mc):
    n, pos, w2 = 0, 0, 2 * W
    while pos < U:
        sz = min(max(-(-(U - pos) // w2), mc), MAX_CHUNK)
        n += 1
        pos += sz
    return n


def predicted_mc(U):
    best, mc = None, None
    for m in range(8, 3, -1):
        f = chunk_count(U, m) / W
        cost = (math.ceil(f - 1e-9) - f) * m + 2 * f
        if best is None or cost < best - 1e-9:
            best, mc = cost, m
    return mc


def plan_digest(P, B, S, H, opts):
    lib = _lib.lib
    desc = _lib.PoolDesc(1, H, 128, 16, 1 << 22, 0, -1, 0)
    pool = ctypes.c_void_p()
    _lib.check(lib.fk_pool_create(ctypes.byref(desc), ctypes.byref(pool)))
    for k, v in opts.items():
        _lib.check(lib.fk_pool_set_option(pool, k, v))
    ids = (ctypes.c_int64 * 4096)()
    n = ctypes.c_int64()
    _lib.check(lib.fk_ctx_create(pool, 0, -1))
    _lib.check(lib.fk_ctx_grow(pool, 0, P, ids, 4096, ctypes.byref(n)))
    for b in range(B):
        _lib.check(lib.fk_ctx_create(pool, 1 + b, 0))
        _lib.check(lib.fk_ctx_grow(pool, 1 + b, S, ids, 4096, ctypes.byref(n)))
    lv = (ctypes.c_int64 * B)(*range(1, B + 1))
    info = _lib.PlanInfo()
    _lib.check(lib.fk_step_plan(pool, lv, B, 1, None, ctypes.byref(info)))
    d = lib.fk_debug_plan_digest(pool)
    prefix_ctas = info.num_prefix_ctas
    lib.fk_pool_destroy(pool)
    return d, prefix_ctas


def main():
    assert os.environ.get("FK_DEBUG_PLAN_DIGEST"), "set FK_DEBUG_PLAN_DIGEST=1"
    _lib.lib.fk_debug_plan_digest.restype = ctypes.c_uint64
    _lib.lib.fk_debug_plan_digest.argtypes = [ctypes.c_void_p]
    seen = set()
    for P, B, S, H in ((6000, 1, 256, 40), (6000, 2, 256, 40), (6000, 3, 256, 40), (6000, 4, 256, 40),
                       (6000, 6, 256, 40), (6000, 8, 256, 40), (2000, 5, 700, 32), (0, 1, 4000, 40)):
        pages = -(-P // 16) + B * -(-S // 16)  # contexts start on page boundaries
        U = pages * H
        assert U < 32768
        mc = predicted_mc(U)
        auto, ctas = plan_digest(P, B, S, H, {})
        fixed, _ = plan_digest(P, B, S, H, {_lib.FK_OPT_PRIV_MIN_CHUNK: mc})
        other, _ = plan_digest(P, B, S, H, {_lib.FK_OPT_PRIV_MIN_CHUNK: 4 if mc != 4 else 5})
        assert ctas == 0, (P, B, S, "expected no prefix grid")
        assert auto == fixed, (P, B, S, H, U, mc)
        seen.add(mc)
        print(P, B, S, H, "units", U, "mc", mc, "differs from fixed 4/5:", auto != other)
    assert len(seen) >= 2, seen  # the rule is not a constant over these shapes
    print("ok")


if __name__ == "__main__":
    main()
