"""Interleaved A/B of pool options on one engine (diagnostic): for R rounds,
each option set runs N engine steps timed with CUDA events; prints the median
algorithmic GB/s per set (the suffixes grow every step).  Interleaving cancels the clock drift between separate runs.

    python profiles/ab.py --set PREFIX_RATE_PCT=40 --set PREFIX_RATE_PCT=50 [--rounds 5 --steps 8]
    (a set may hold several options: --set "CORUN=0,PDL=1")
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2405_19888_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--set", action="append", required=True)
    ap.add_argument("--base", default="", help="K=V,... applied before every set (options persist otherwise)")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--shape", default=None, help="P,B,S[,L,H]: fork group shape instead of --config")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    if args.shape:
        v = [int(x) for x in args.shape.split(",")]
        cfg = dict(model="custom", P=v[0], B=v[1], S=v[2], L=v[3] if len(v) > 3 else 40, H=v[4] if len(v) > 4 else 40)
    eng, rows = bench.build_engine(cfg, 0, torch, out_len=args.rounds * len(args.set) * (args.steps + 2) + 32)
    sets = [[kv.split("=") for kv in s.split(",")] for s in args.set]
    res = {s: [] for s in args.set}
    st = eng.stream
    for _ in range(3):
        eng.step()
    for r in range(args.rounds):
        base = [kv.split("=") for kv in args.base.split(",") if kv]
        for name, opts in zip(args.set, sets):
            for k, v in base + opts:
                eng.set_option(getattr(_lib, "FK_OPT_" + k), int(v))
            eng.step()
            eng.step()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            nbytes = 0
            a.record(st)
            for _ in range(args.steps):
                eng.step()
                nbytes += cfg["L"] * bench.alg_bytes_per_layer(eng.last_plan, rows, cfg["H"])
            b.record(st)
            b.synchronize()
            res[name].append(nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)  # algorithmic GB/s
            if res[name][-1] < 0.7 * max(res[name]):
                ps = eng.pool_stats()
                print(f"outlier: round {r} set {name}: {a.elapsed_time(b) / args.steps:.3f} ms/step, pages "
                      f"{ps.num_pages} free {ps.free_pages}, slots {eng.last_plan.max_slots}", flush=True)
    for name in args.set:
        v = res[name]
        print(f"{name:40s} median {statistics.median(v):7.0f} GB/s (alg., whole step)  max {max(v):7.0f}  all {' '.join('%.0f' % x for x in v)}")


if __name__ == "__main__":
    main()
