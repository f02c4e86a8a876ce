"""Where does a decode step's time go?  Kernel timeline of a few bench steps
(torch.profiler / CUPTI) -> busy time per kernel, idle gaps between kernels,
host time per step.  Diagnostic only (not product code, not a bench number).

    python profiles/step_gaps.py [--config llama13b_p6000_b64] [--steps 3]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--opt", action="append", default=[], help="NAME=VALUE pool option, e.g. CORUN=0")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    eng, rows = bench.build_engine(cfg, 0, torch, out_len=64)
    from paper_2405_19888_b200 import _lib
    for kv in args.opt:
        k, v = kv.split("=")
        eng.set_option(getattr(_lib, "FK_OPT_" + k), int(v))
    for _ in range(4):
        eng.step()
    torch.cuda.synchronize()
    # host time per step with the GPU drained before each step
    t_host = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.step()
        t_host.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    print("host step (GPU drained before):", ["%.2f ms" % (1e3 * t) for t in t_host])
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(args.steps):
            eng.step()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    busy = {}
    gaps = []
    prev_end = None
    for e in evs:
        s, t = e.time_range.start, e.time_range.end
        busy[e.name[:40]] = busy.get(e.name[:40], 0) + (t - s)
        if prev_end is not None:
            gaps.append((s - prev_end, e.name[:40]))
        prev_end = t if prev_end is None else max(prev_end, t)
    span = evs[-1].time_range.end - evs[0].time_range.start
    print(f"span {span / 1e3:.3f} ms for {args.steps} steps, {len(evs)} device events")
    for k, v in sorted(busy.items(), key=lambda kv: -kv[1]):
        print(f"  {k:40s} {v / 1e3:9.3f} ms")
    pos = [g for g in gaps if g[0] > 0]
    print(f"idle between events: {sum(g for g, _ in pos) / 1e3:.3f} ms over {len(pos)} gaps;"
          f" overlap (negative gaps): {sum(-g for g, _ in gaps if g < 0) / 1e3:.3f} ms")
    big = sorted(pos, reverse=True)[:12]
    print("largest gaps (us, before kernel):", [(round(g, 1), n) for g, n in big])
    # one layer in the middle of the last step: start/end offsets per kernel
    ks = [e for e in evs if "fk_" in e.name]
    mid = [e for e in ks if "prefix" in e.name][-20]
    t0 = mid.time_range.start
    print("layer timeline (us from prefix start):")
    for e in ks:
        if t0 - 5 <= e.time_range.start <= t0 + 400:
            print(f"  {e.name.split('(')[0][4:]:22s} {e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f}")
    print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=15))


if __name__ == "__main__":
    main()
