"""Interleaved A/B of pool options in the isolated-layer mode (diagnostic):
one fk_attn_decode per layer, direct launches, PDL within the layer only and
a foreign kernel between layers (bench.time_layers_isolated), so each layer's
ramp, tail and merge are fully exposed.  Prints per-set median layer us.

    python profiles/iso_ab.py --set DEBUG_SKIP_MERGE=0 --set DEBUG_SKIP_MERGE=1 [--rounds 5]
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
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--graph-too", action="store_true", help="also time the PDL=2 graph path per set")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    eng, rows = bench.build_engine(cfg, 0, torch, out_len=64)
    for _ in range(4):
        eng.step()
    torch.cuda.synchronize()
    eng.set_option(_lib.FK_OPT_GRAPH, 0)
    sets = [[kv.split("=") for kv in s.split(",")] for s in args.set]
    res = {s: [] for s in args.set}
    alg = bench.alg_bytes_per_layer(eng.last_plan, rows, cfg["H"])
    for r in range(args.rounds):
        for name, opts in zip(args.set, sets):
            for k, v in opts:
                eng.set_option(getattr(_lib, "FK_OPT_" + k), int(v))
            eng.step()  # plan-time options take effect with a new plan
            t, tf = bench.time_layers_isolated(eng, args.reps, torch)
            res[name].append(t * 1e6)
            for k, v in opts:  # back to defaults for the next set
                if k == "DEBUG_SKIP_MERGE":
                    eng.set_option(_lib.FK_OPT_DEBUG_SKIP_MERGE, 0)
    for name in args.set:
        med = statistics.median(res[name])
        print(f"{name:40s} layer {med:7.2f} us  {alg / (med * 1e-6) / 1e9:7.1f} GB/s  "
              f"(rounds {', '.join(f'{x:.2f}' for x in res[name])})", flush=True)


if __name__ == "__main__":
    main()
