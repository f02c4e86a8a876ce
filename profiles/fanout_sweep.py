"""Whole-step throughput vs fan-out on the final kernels (diagnostic):
LLaMA-13B attention shape, 6000-token shared prefix, B forks x 256-token
suffixes, B in {2, 4, 8, 16, 32, 64}.  Prints algorithmic GB/s and the
fraction of the measured HBM peak per fan-out (graph path, PDL level 2), and
the isolated-layer fraction.

    python profiles/fanout_sweep.py [--steps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2405_19888_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--fanouts", default="2,4,8,16,32,64")
    ap.add_argument("--opt", action="append", default=[], metavar="NAME=V", help="FK_OPT_<NAME> on every engine")
    args = ap.parse_args()
    peak, kind = bench.load_peaks()
    for b in [int(x) for x in args.fanouts.split(",")]:
        cfg = dict(model="LLaMA-13B", L=40, H=40, P=6000, B=b, S=256)
        eng, rows = bench.build_engine(cfg, 0, torch, out_len=2 * args.steps + 32)
        for kv in args.opt:
            k, v = kv.split("=")
            eng.set_option(getattr(_lib, "FK_OPT_" + k), int(v))
        for _ in range(3):
            eng.step()
        t = bench.time_steps(eng, args.steps, torch)
        info = eng.last_plan
        nbytes = bench.alg_bytes_per_layer(info, rows, 40)
        t_layer = bench.time_layers(eng, 5, torch)
        t_iso, _ = bench.time_layers_isolated(eng, 3, torch)
        print(json.dumps({"fanout": b, "tokens_per_s": rows * args.steps / t, "layer_us": t_layer * 1e6,
                          "layer_gbs": nbytes / t_layer / 1e9, "frac": nbytes / t_layer / 1e9 / peak,
                          "frac_isolated": nbytes / t_iso / 1e9 / peak, "batch_tokens": int(info.batch_tokens),
                          "prefix_ctas": info.num_prefix_ctas, "tc_items": info.num_tc_items}), flush=True)
        eng.close()
        del eng
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
