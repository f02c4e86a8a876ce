"""Per-CTA start/end of the prefix (tcgen05) and private kernels for the last
two layers of a bench-shaped step (debug build, FK_LIB_PATH=profiles/build/
libforkattn_tl.so; stamps are kept per layer parity).  Diagnostic only.

    python profiles/cta_timeline.py [--config ...] [--opt PREFIX_RATE_PCT=50]
"""
import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FK_LIB_PATH", os.path.join(ROOT, "profiles", "build", "libforkattn_tl.so"))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2405_19888_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--isolated", action="store_true",
                    help="stamps of bench.time_layers_isolated (direct launches, a foreign kernel between layers)")
    ap.add_argument("--shape", default=None, help="P,B,S[,L,H]: fork group shape instead of --config")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    if args.shape:
        v = [int(x) for x in args.shape.split(",")]
        cfg = dict(model="custom", P=v[0], B=v[1], S=v[2], L=v[3] if len(v) > 3 else 40, H=v[4] if len(v) > 4 else 40)
    eng, rows = bench.build_engine(cfg, 0, torch, out_len=32)
    for kv in args.opt:
        k, v = kv.split("=")
        eng.set_option(getattr(_lib, "FK_OPT_" + k), int(v))
    for _ in range(4):
        eng.step()
    torch.cuda.synchronize()
    if args.isolated:
        bench.time_layers_isolated(eng, 1, torch)
        torch.cuda.synchronize()
    info = eng.last_plan
    out = {}
    for name in ("prefix", "priv", "merge"):
        fn = getattr(_lib.lib, "fk_debug_cta_timeline_" + name)
        fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
        buf = (ctypes.c_ulonglong * 8192)()
        assert fn(buf, 1024) == 0
        out[name] = [[(buf[par * 4096 + 4 * i], buf[par * 4096 + 4 * i + 1]) for i in range(1024)] for par in (0, 1)]
        if name == "prefix":
            notes = [[(buf[par * 4096 + 4 * i + 2], buf[par * 4096 + 4 * i + 3]) for i in range(1024)] for par in (0, 1)]
    L = cfg["L"]
    pars = [(L - 2) & 1, (L - 1) & 1]  # second-to-last layer, last layer
    t0 = None
    for par in pars:
        pre = [x for x in out["prefix"][par][:info.num_prefix_ctas] if x[0]]
        if pre:
            t_last = max(s for s, _ in pre)
            pre = [x for x in pre if x[0] >= t_last - 20000]
        else:  # (no prefix kernel: small fan-outs stream in the private kernel)
            t_last = max(s for s, _ in out["priv"][par] if s)
        priv = [x for x in out["priv"][par] if x[0] and abs(x[0] - t_last) < 60000 and x[1] >= x[0]]
        if t0 is None:
            t0 = min(s for s, _ in pre + priv)
        mer = [x for x in out["merge"][par] if x[0] and abs(x[0] - t_last) < 200000 and x[1] >= x[0]]
        for name, xs in (("prefix", pre), ("private", priv), ("merge*", mer)):
            if not xs:
                print(f"layer%2 {par} {name:8s} none")
                continue
            st = sorted((s - t0) / 1e3 for s, _ in xs)
            en = sorted((e - t0) / 1e3 for _, e in xs)
            print(f"layer%2 {par} {name:8s} ctas={len(xs):4d} start min/med/max {st[0]:7.2f} {statistics.median(st):7.2f} "
                  f"{st[-1]:7.2f}   end min/med/max {en[0]:7.2f} {statistics.median(en):7.2f} {en[-1]:7.2f}")
    print("(merge* start = after its griddepcontrol.wait; the wide merge stamps its launch)")
    par = pars[-1]
    late = sorted(((e, s, i) for i, (s, e) in enumerate(out["merge"][par]) if s and e >= s and abs(s - t_last) < 200000),
                  reverse=True)[:6]
    print("last layer, latest merge CTAs (index: start, end us):",
          " ".join("%d: %.2f, %.2f" % (i, (s - t0) / 1e3, (e - t0) / 1e3) for e, s, i in late))
    par = pars[-1]
    print("last layer prefix CTAs (tiles, pieces, duration us):")
    print(" ".join("%d/%d/%.0f" % (notes[par][i][0], notes[par][i][1], (out["prefix"][par][i][1] - out["prefix"][par][i][0]) / 1e3)
                   for i in range(info.num_prefix_ctas)) or "-")
    print("plan:", info.num_rows, "rows", info.num_prefix_ctas, "prefix CTAs", info.max_slots, "slots")


if __name__ == "__main__":
    main()
