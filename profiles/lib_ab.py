"""Interleaved A/B of two builds of libforkattn.so on one box (diagnostic):
runs bench.py alternately with FK_LIB_PATH = A and B and prints each run's
tokens/s, layer us and isolated fraction, then the medians.

    python profiles/lib_ab.py --a .ab/libforkattn_old.so --b paper_2405_19888_b200/libforkattn.so [--config ...]
    python profiles/lib_ab.py --a L --b L --opt-b PREFIX_JOINS=1     (an option A/B on one build)
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--a", required=True)
    ap.add_argument("--b", required=True)
    ap.add_argument("--config", default=None)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--opt-a", action="append", default=[], help="bench.py --opt for arm A (NAME=V)")
    ap.add_argument("--opt-b", action="append", default=[], help="bench.py --opt for arm B (NAME=V)")
    args = ap.parse_args()
    res = {"A": [], "B": []}
    for r in range(args.rounds):
        for name, lib in (("A", args.a), ("B", args.b)):
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", str(args.steps), "--warmup", "5",
                   "--no-cpu-baseline", "--no-e2e", "--no-check"]
            if args.config:
                cmd += ["--config", args.config]
            for kv in args.opt_a if name == "A" else args.opt_b:
                cmd += ["--opt", kv]
            out = subprocess.run(cmd, env={**os.environ, "FK_LIB_PATH": os.path.abspath(lib)}, capture_output=True,
                                 text=True, timeout=600)
            line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
            if not line:
                print(name, "failed:", out.stderr[-500:], flush=True)
                continue
            d = json.loads(line[-1])
            rf = d.get("roofline", {})
            row = (d["value"], rf.get("layer_us"), rf.get("frac_isolated"), d.get("clocks", {}).get("sm_mhz"))
            res[name].append(row)
            print(name, "round", r, "tokens/s %.0f layer %.2f us iso %.4f MHz %s" % row, flush=True)
    for name in ("A", "B"):
        if res[name]:
            print(name, "median tokens/s %.0f layer %.2f us iso %.4f" % tuple(
                statistics.median(x[i] for x in res[name]) for i in range(3)))


if __name__ == "__main__":
    main()
