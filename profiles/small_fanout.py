"""Per-kernel view of small fan-outs (diagnostic, run under ncu): one fork
group (6000-token prefix, B forks x 256-token suffixes, 13B shape) stepped a
few times with the given pool options, so an ncu launch list shows what each
kernel costs.  Never a bench number.

    ncu --metrics gpu__time_duration.sum -k regex:fk_ -s 300 -c 9 \
        python profiles/small_fanout.py --b 2 --set GROUP_FANOUT=16
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2405_19888_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=2)
    ap.add_argument("--set", default="")
    ap.add_argument("--steps", type=int, default=4)
    args = ap.parse_args()
    cfg = dict(model="LLaMA-13B", L=40, H=40, P=6000, B=args.b, S=256)
    eng, rows = bench.build_engine(cfg, 0, torch, out_len=64)
    for kv in [x for x in args.set.split(",") if x]:
        k, v = kv.split("=")
        eng.set_option(getattr(_lib, "FK_OPT_" + k), int(v))
    eng.set_option(_lib.FK_OPT_GRAPH, 0)  # direct launches: ncu sees each kernel
    for _ in range(args.steps):
        eng.step()
    torch.cuda.synchronize()
    info = eng.last_plan
    print("plan: rows", info.num_rows, "shared", info.num_shared_ctx, "prefix CTAs", info.num_prefix_ctas,
          "max slots", info.max_slots, flush=True)


if __name__ == "__main__":
    main()
