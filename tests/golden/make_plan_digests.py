"""Pins the work-list planner's output (fk_step_plan): for random forests and
option sets on host-only pools, the FNV-1a digest of every array and scalar
the plan uploads (FK_DEBUG_PLAN_DIGEST, fk_pool.cpp), over a few steps with
the one-token growth in between.

    FK_DEBUG_PLAN_DIGEST=1 python tests/golden/make_plan_digests.py [--check]

Written once with the round-1 planner (plan_digests.json); the planner was
then rewritten for host speed and must reproduce every digest
(tests/test_plan.py::test_plan_digests_pinned runs --check in a subprocess).
The FK_OPT_GROUP_FANOUT option sets (opt9, opt10) were added afterwards by the
grouped planner (--add: writes only keys the file does not have).
"""

import ctypes
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2405_19888_b200 import _lib  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "plan_digests.json")

OPTION_SETS = [
    {},
    {_lib.FK_OPT_TC_MIN_FANOUT: 0},
    {_lib.FK_OPT_TC_MIN_FANOUT: 8},
    {_lib.FK_OPT_CORUN: 0},
    {_lib.FK_OPT_PREFIX_TARGET_CTAS: 40},
    {_lib.FK_OPT_PRIV_WARPS: 8, _lib.FK_OPT_PRIV_MIN_CHUNK: 4},
    {_lib.FK_OPT_PRIV_STATIC_FIRST: 0, _lib.FK_OPT_TC_BOUNDARY_COST: 0},
    {_lib.FK_OPT_APPEND_FIRST: 1},
    {_lib.FK_OPT_MIN_SPLIT_PAGES: 16, _lib.FK_OPT_TC_MIN_FANOUT: 0, _lib.FK_OPT_LAUNCH_ORDER: 1},
    # (round 2, written by the grouped planner: regression pins, not round-1 parity)
    {_lib.FK_OPT_GROUP_FANOUT: 8},
    {_lib.FK_OPT_GROUP_FANOUT: 16, _lib.FK_OPT_TC_MIN_FANOUT: 0, _lib.FK_OPT_APPEND_FIRST: 1},
]


def forest_cases():
    """(name, heads, builder) -- builder(rng) -> (contexts [(id, parent, tokens)], leaves)."""
    def fork(P, B, S):
        def b(rng):
            ctxs = [(0, -1, P)] + [(1 + r, 0, S + rng.randint(0, 40)) for r in range(B)]
            return ctxs, [1 + r for r in range(B)]
        return b

    def nested(rng):
        ctxs, leaves, n = [(0, -1, 4000)], [], 1
        for a in range(4):
            app = n
            ctxs.append((app, 0, 1000 + rng.randint(0, 30)))
            n += 1
            for u in range(rng.randint(3, 40)):
                ctxs.append((n, app, rng.randint(0, 300)))
                leaves.append(n)
                n += 1
        return ctxs, leaves

    def mapreduce(rng):
        ctxs, leaves, n = [], [], 0
        for g in range(rng.randint(2, 6)):
            root = n
            ctxs.append((root, -1, 2000 + rng.randint(0, 100)))
            n += 1
            for u in range(rng.randint(2, 40)):
                ctxs.append((n, root, rng.randint(128, 1024)))
                leaves.append(n)
                n += 1
        return ctxs, leaves

    def random_forest(rng):
        ctxs, ids = [], []
        for i in range(rng.randint(1, 60)):
            parent = rng.choice(ids) if ids and rng.random() < 0.7 else -1
            ctxs.append((i, parent, rng.choice([0, 1, 15, 16, 17, rng.randint(0, 900)])))
            ids.append(i)
        leaves = [rng.choice(ids) for _ in range(rng.randint(1, 80))]
        return ctxs, leaves

    cases = [("fork_6000x64", 40, fork(6000, 64, 256)), ("fork_6000x256", 8, fork(6000, 256, 256)),
             ("fork_6000x150", 8, fork(6000, 150, 100)), ("fork_300x6", 8, fork(300, 6, 10)),
             ("single", 32, fork(0, 1, 700)), ("nested", 40, nested), ("mapreduce", 40, mapreduce)]
    cases += [(f"random{i}", random.Random(i).choice([1, 8, 40]), random_forest) for i in range(24)]
    return cases


def run():
    lib = _lib.lib
    lib.fk_debug_plan_digest.restype = ctypes.c_uint64
    lib.fk_debug_plan_digest.argtypes = [ctypes.c_void_p]
    out = {}
    for ci, (name, H, build) in enumerate(forest_cases()):
        for oi, opts in enumerate(OPTION_SETS):
            for di, dedup in enumerate((1, 0)):
                # (the seeds of the 9 round-1 option sets are their original enumeration index)
                rng = random.Random((ci * 9 + oi) * 2 + di + 17 if oi < 9 else 100000 + (ci * 100 + oi) * 2 + di)
                ctxs, leaves = build(rng)
                desc = _lib.PoolDesc(2, H, 128, 16, 1 << 22, 0, -1, 0)
                pool = ctypes.c_void_p()
                _lib.check(lib.fk_pool_create(ctypes.byref(desc), ctypes.byref(pool)))
                # (the round-1 planner had no row groups, a fixed 2-page minimum
                # chunk and a boundary cost of 4 tiles: its sets run that way; the
                # grouped sets were pinned with the latter two as well)
                base = {_lib.FK_OPT_PRIV_MIN_CHUNK: 2, _lib.FK_OPT_TC_BOUNDARY_COST: 4}
                for k, v in ({_lib.FK_OPT_GROUP_FANOUT: 0, **base, **opts} if oi < 9 else {**base, **opts}).items():
                    _lib.check(lib.fk_pool_set_option(pool, k, v))
                ids = (ctypes.c_int64 * 4096)()
                n = ctypes.c_int64()
                for cid, parent, tok in ctxs:
                    _lib.check(lib.fk_ctx_create(pool, cid, parent))
                    _lib.check(lib.fk_ctx_grow(pool, cid, tok, ids, 4096, ctypes.byref(n)))
                B = len(leaves)
                lv = (ctypes.c_int64 * B)(*leaves)
                pos = (ctypes.c_int64 * B)()
                nid = (ctypes.c_int64 * B)()
                nf = ctypes.c_int32()
                info = _lib.PlanInfo()
                digs = []
                for step in range(3):
                    _lib.check(lib.fk_step_plan(pool, lv, B, dedup, None, ctypes.byref(info)))
                    digs.append("%016x" % lib.fk_debug_plan_digest(pool))
                    _lib.check(lib.fk_step_grow(pool, pos, nid, ctypes.byref(nf)))
                lib.fk_pool_destroy(pool)
                out[f"{name}/opt{oi}/dedup{dedup}"] = digs
    return out


def main():
    assert os.environ.get("FK_DEBUG_PLAN_DIGEST"), "set FK_DEBUG_PLAN_DIGEST=1"
    got = run()
    if "--check" in sys.argv:
        want = json.load(open(OUT))
        bad = [k for k in want if want[k] != got.get(k)]
        print(f"{len(want) - len(bad)}/{len(want)} plan digests match")
        for k in bad[:10]:
            print("MISMATCH", k, want[k], got.get(k))
        sys.exit(1 if bad else 0)
    if "--add" in sys.argv:
        want = json.load(open(OUT))
        assert all(want[k] == got[k] for k in want), "existing digests changed"
        got = {**got, **want}
    with open(OUT, "w") as f:
        json.dump(got, f, indent=0, sort_keys=True)
    print(f"wrote {len(got)} digests to {OUT}")


if __name__ == "__main__":
    main()
