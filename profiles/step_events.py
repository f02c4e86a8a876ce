"""Step time vs back-to-back layer time (diagnostic, not a bench number).

Times each engine step with CUDA events on the engine stream, the host time
of each step() call, and the same 40-layer attention loop bench.py's
roofline uses, in one process.

    python profiles/step_events.py [--config ...] [--steps 20] [--opt CORUN=0]
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--host", action="store_true", help="pinned-host Q/K/V (the e2e path)")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    eng, rows = bench.build_engine(cfg, 0, torch, host_inputs=args.host, out_len=4 * args.steps + 16)
    from paper_2405_19888_b200 import _lib
    for kv in args.opt:
        k, v = kv.split("=")
        eng.set_option(getattr(_lib, "FK_OPT_" + k), int(v))
    for _ in range(5):
        eng.step()
    torch.cuda.synchronize()
    st = eng.stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    host = []
    ev[0].record(st)
    for i in range(args.steps):
        t0 = time.perf_counter()
        eng.step()
        host.append(time.perf_counter() - t0)
        ev[i + 1].record(st)
    ev[-1].synchronize()
    dev = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    print("device ms/step:", " ".join("%.3f" % d for d in dev))
    print("host   ms/step:", " ".join("%.3f" % (1e3 * h) for h in host))
    print("median device %.3f ms, host %.3f ms" % (statistics.median(dev), 1e3 * statistics.median(host)))
    if args.host:
        return
    t_layer = bench.time_layers(eng, 5, torch)
    print("back-to-back layer %.1f us -> x%d = %.3f ms" % (1e6 * t_layer, cfg["L"], 1e3 * t_layer * cfg["L"]))
    # step with the device drained before it: the host cost alone
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.step()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print("drained host step %.3f ms, device done %.3f ms later" % (1e3 * (t1 - t0), 1e3 * (time.perf_counter() - t1)))


if __name__ == "__main__":
    main()
