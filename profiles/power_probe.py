"""Steady-state power, SM clock and algorithmic HBM throughput of the
attention layers (diagnostic): for each fork-group shape, the engine's
40-layer graph replayed back to back for --seconds, nvidia-smi sampled every
50 ms; the last half of the window is reported (median power, median SM
clock, GB/s from CUDA events over that half), plus J per GB streamed.

    python profiles/power_probe.py [--shapes 6000,64,256 6000,1,256] [--seconds 4] [--opt NAME=V]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2405_19888_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", nargs="+", default=["6000,64,256", "6000,1,256", "6000,256,256"])
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--read-baseline", action="store_true",
                    help="also a plain HBM read (torch sum over 8 GiB of bf16) for the J/GB floor")
    args = ap.parse_args()
    if args.read_baseline:
        x = torch.randn(1 << 32, device="cuda", dtype=torch.bfloat16)  # 8 GiB (random bits toggle like K/V)
        acc = torch.empty((), device="cuda", dtype=torch.float32)
        sampler = bench.ClockSampler(0)
        sampler.start()
        time.sleep(0.5)
        t_end = time.perf_counter() + args.seconds
        t_half = t_end - args.seconds / 2
        nb, secs = 0, 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        while time.perf_counter() < t_end:
            e0.record()
            for _ in range(10):
                acc = torch.sum(x, dtype=torch.float32)
            e1.record()
            e1.synchronize()
            if time.perf_counter() >= t_half:
                nb += 10 * x.numel() * 2
                secs += e0.elapsed_time(e1) / 1e3
        lines = [ln for t, ln in sampler.lines if t >= t_half]
        sampler.stop()
        pw = [float(ln.split(",")[3]) for ln in lines if ln.count(",") >= 3]
        mhz = [float(ln.split(",")[1]) for ln in lines if ln.count(",") >= 3]
        gbs = nb / secs / 1e9
        print(json.dumps({"shape": "read-baseline (torch.sum, 8 GiB bf16)", "gb_s": round(gbs, 1),
                          "power_w": statistics.median(pw), "sm_mhz": statistics.median(mhz),
                          "j_per_gb": round(statistics.median(pw) / gbs, 4), "samples": len(pw)}), flush=True)
        del x
        torch.cuda.empty_cache()
        time.sleep(2.0)
    for shape in args.shapes:
        P, B, S = (int(x) for x in shape.split(","))
        cfg = dict(model="LLaMA-13B", L=40, H=40, P=P, B=B, S=S)
        eng, rows = bench.build_engine(cfg, 0, torch, out_len=64)
        for kv in args.opt:
            k, v = kv.split("=")
            eng.set_option(getattr(_lib, "FK_OPT_" + k), int(v))
        for _ in range(3):
            eng.step()
        torch.cuda.synchronize()
        info = eng.last_plan
        nbytes = bench.alg_bytes_per_layer(info, rows, 40)
        sampler = bench.ClockSampler(0)
        sampler.start()
        time.sleep(0.5)
        t_end = time.perf_counter() + args.seconds
        chunks = []  # (host time at end, layers, seconds)
        while time.perf_counter() < t_end:
            dt = bench.time_layers(eng, 10, torch)  # 10 passes x 40 layers
            chunks.append((time.perf_counter(), 400, dt * 400))
        t_half = t_end - args.seconds / 2
        sampler.mark()
        sampler.t_mark = t_half
        lines = [ln for t, ln in sampler.lines if t >= t_half]
        sampler.stop()
        pw, mhz = [], []
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            try:
                mhz.append(float(f[1]))
                pw.append(float(f[3]))
            except (ValueError, IndexError):
                pass
        late = [c for c in chunks if c[0] >= t_half]
        secs = sum(c[2] for c in late)
        layers = sum(c[1] for c in late)
        gbs = nbytes * layers / secs / 1e9
        p = statistics.median(pw) if pw else None
        print(json.dumps({"shape": shape, "opts": args.opt, "gb_s": round(gbs, 1), "layer_us": round(secs / layers * 1e6, 2),
                          "power_w": p, "sm_mhz": statistics.median(mhz) if mhz else None,
                          "j_per_gb": round(p / gbs, 4) if p else None, "samples": len(pw)}), flush=True)
        eng.close()
        del eng
        torch.cuda.empty_cache()
        time.sleep(2.0)  # let the power average settle between shapes


if __name__ == "__main__":
    main()
