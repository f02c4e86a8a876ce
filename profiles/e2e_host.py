"""Host view of the e2e path (pinned-host Q/K/V in, output back every step;
diagnostic): per-step host time of GpuEngine.step and the part of it the
planner spent blocked on the GPU (PoolStats.host_wait_ns), against the
device time per step.  If step() blocks, the host is in lock-step with the
GPU and its own time adds to every step.

    python profiles/e2e_host.py [--config ...] [--steps 30] [--device-inputs]
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
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--device-inputs", action="store_true")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    eng, rows = bench.build_engine(cfg, 0, torch, host_inputs=not args.device_inputs, out_len=args.steps + 40)
    for _ in range(5):
        eng.step()
    torch.cuda.synchronize()
    st = eng.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host, waits = [], []
    w_prev = eng.pool_stats().host_wait_ns
    e0.record(st)
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t = time.perf_counter()
        eng.step()
        host.append((time.perf_counter() - t) * 1e6)
        w = eng.pool_stats().host_wait_ns
        waits.append((w - w_prev) / 1e3)
        w_prev = w
    e1.record(st)
    e1.synchronize()
    wall = (time.perf_counter() - t_all) * 1e6 / args.steps
    dev = e0.elapsed_time(e1) * 1e3 / args.steps
    print(f"{'host' if not args.device_inputs else 'device'} inputs: device us/step {dev:.1f}, wall us/step {wall:.1f}, "
          f"step() host us median {statistics.median(host):.1f} (min {min(host):.1f}, max {max(host):.1f}), "
          f"planner GPU wait us median {statistics.median(waits):.1f}")


if __name__ == "__main__":
    main()
