"""Host cost of the engine step with several GpuEngines in one process.

The reference manager steps its engines serially on one thread
(run_until_idle, manager.py:638-657), so with one engine per GPU the host
time of GpuEngine.step must stay well under the GPU step time.  This runs
the unmodified reference runtime (semflow from /root/reference or
baseline/_ref) over Config(engines=N) with engine_factory: N shared-prompt
groups (64 users each, 6000-token system prompt, 200-token unique part), one
group per engine, and reports the host microseconds spent inside
GpuEngine.step (plan, launches, growth, bookkeeping; the GPU runs
asynchronously) and the whole manager loop per engine step.

    python profiles/host_step.py [--engines 8] [--output-len 64] [--layers 32 --heads 32]

All engines live on the visible GPU(s) (engine eI -> cuda:(I mod ndev));
LLaMA-7B attention shape by default so that 8 engines fit on one B200.
"""

import argparse
import dataclasses
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for ref in (os.environ.get("FK_REFERENCE", "/root/reference/pkg/src"), os.path.join(ROOT, "baseline", "_ref")):
    if os.path.isdir(os.path.join(ref, "semflow")):
        sys.path.insert(1, ref)
        break


def direct(args):
    """One engine built exactly as bench.py builds it (headline shape by
    default), stepped in a loop: per-step host time minus the plan's GPU
    waits, and the per-phase split."""
    import torch

    import bench

    cfg = bench.CONFIGS[args.config]
    eng, rows = bench.build_engine(cfg, 0, torch, out_len=2 * args.steps + 16)
    for _ in range(5):
        eng.step()
    torch.cuda.synchronize()
    if args.cprofile:  # where the host time goes (tottime per function)
        import cProfile
        import pstats
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(args.steps):
            eng.step()
        pr.disable()
        torch.cuda.synchronize()
        pstats.Stats(pr).sort_stats("tottime").print_stats(25)
    us = []
    for _ in range(args.steps):
        w0 = eng.pool_stats().host_wait_ns
        t0 = time.perf_counter()
        eng.step()
        t1 = time.perf_counter()
        us.append((t1 - t0) * 1e6 - (eng.pool_stats().host_wait_ns - w0) / 1e3)
    torch.cuda.synchronize()
    out = {"mode": "direct", "config": args.config, "rows": rows, "steps": args.steps,
           "step_host_us_median": statistics.median(us), "step_host_us_mean": statistics.mean(us)}
    ph = eng.__dict__.get("phase_steps")
    if ph:
        out["phase_us_median"] = {k: statistics.median(x[k] for x in ph) for k in ph[0]}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--direct", action="store_true", help="one bench.py engine, no manager")
    ap.add_argument("--cprofile", action="store_true", help="(direct) cProfile the steps first")
    ap.add_argument("--config", default="llama13b_p6000_b64")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--engines", type=int, default=8)
    ap.add_argument("--pages", type=int, default=0, help="KV arena pages per engine (default: the workload's need)")
    ap.add_argument("--users", type=int, default=64)
    ap.add_argument("--output-len", type=int, default=64)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--py-hash", action="store_true",
                    help="keep the reference's pure-Python FNV (default: rebind it to the C one, INTEGRATION.md §3)")
    args = ap.parse_args()
    if args.direct:
        return direct(args)

    import torch

    import paper_2405_19888_b200 as P
    import semflow.manager as sm
    from semflow.config import Config
    from semflow.experiments import run_workload_manager
    from semflow.workloads import Workload, shared_prompt_serving

    apps = []
    for g in range(args.engines):
        wl = shared_prompt_serving(100 + g, users=args.users, system_prompt_len=6000, unique_len=200,
                                   output_len=args.output_len)
        apps += [dataclasses.replace(a, app_id=f"g{g}.{a.app_id}") for a in wl.apps]
    work = Workload("GroupsPerEngine", 7, {"groups": args.engines}, apps)

    step_us, full, slow = [], [], []
    orig_step = P.GpuEngine.step

    def timed_step(self):
        w0 = self.pool_stats().host_wait_ns if self.device is not None else 0
        t0 = time.perf_counter()
        r = orig_step(self)
        t1 = time.perf_counter()
        w1 = self.pool_stats().host_wait_ns if self.device is not None else 0
        # host CPU time of the step: wall time minus the time the plan waited
        # for the GPU to release a plan slot (the host runs <= 1 step ahead)
        step_us.append((t1 - t0) * 1e6 - (w1 - w0) / 1e3)
        if step_us[-1] > 1000:  # where the slow steps happen (engine, its step, rows)
            slow.append((round(step_us[-1]), self.engine_id, len(self.reports), self.last_plan.num_rows))
        full.append(r is not None and r.batch_tokens > 0 and self.last_plan.num_rows == args.users)
        return r

    P.GpuEngine.step = timed_step
    if not args.py_hash:  # render_prefix / end hashes through fk_fnv1a64_u32
        import semflow.engine as se
        import semflow.prefix as sp
        import semflow.tokenizer as st
        st.hash_token_ids = sp.hash_token_ids = se.hash_token_ids = P.hash_token_ids
    # the KV arena sized up front (a serving deployment sizes its pool at
    # start-up; growing it is a device-wide copy): prompt + users x (unique +
    # output) tokens per engine, in 16-token pages
    pages = args.pages or (-(-6000 // 16) + args.users * (-(-(200 + args.output_len) // 16) + 2) + 64)
    sm.Engine = P.engine_factory(P.ModelGeometry(args.layers, args.heads, 128), num_pages=pages)
    t0 = time.perf_counter()
    if args.cprofile:
        import cProfile
        import pstats
        pr = cProfile.Profile()
        pr.enable()
    mgr, _, end_ns = run_workload_manager(work, "semflow", Config(engines=args.engines, kv_tokens=1 << 21))
    wall = time.perf_counter() - t0
    if args.cprofile:
        pr.disable()
        st_ = pstats.Stats(pr)
        st_.sort_stats("tottime").print_stats("paper_2405_19888_b200|torch", 30)
    for e in mgr.engines.values():
        if e.stream is not None:
            e.stream.synchronize()
    gpu_wall = time.perf_counter() - t0
    decode = [len(e.history) for e in mgr.engines.values()]
    steps_per_engine = [len(e.reports) for e in mgr.engines.values()]
    # the first steps include the one-time graph captures: report the steady part too
    steady = step_us[len(step_us) // 4:]
    out = {
        "engines": args.engines, "c_hash": not args.py_hash, "devices": torch.cuda.device_count(), "layers": args.layers, "heads": args.heads,
        "users_per_engine": args.users, "steps_per_engine": steps_per_engine,
        "engine_steps": len(step_us),
        "step_host_us_mean": statistics.mean(step_us), "step_host_us_median": statistics.median(step_us),
        "step_host_us_steady_mean": statistics.mean(steady), "step_host_us_steady_median": statistics.median(steady),
        # decode steps with every user of the engine's group in the batch (B = users)
        "full_batch_steps": sum(full),
        "full_batch_step_host_us_median": statistics.median([u for u, f in zip(step_us, full) if f] or [0.0]),
        "full_batch_step_host_us_mean": statistics.mean([u for u, f in zip(step_us, full) if f] or [0.0]),
        "step_host_us_p90": sorted(steady)[int(0.9 * (len(steady) - 1))],
        "step_host_us_p99": sorted(steady)[int(0.99 * (len(steady) - 1))],
        "step_host_us_max": max(step_us), "steps_over_1ms": sum(u > 1000 for u in step_us),
        "slow_steps": slow[:60],
        "manager_loop_us_per_engine_step": wall / max(len(step_us), 1) * 1e6,
        "wall_s": wall, "wall_with_gpu_drain_s": gpu_wall, "virtual_end_ms": end_ns / 1e6,
        "max_batch": max(max((r.batch_tokens for r in e.reports), default=0) for e in mgr.engines.values()),
    }
    del decode
    ph = [x for e in mgr.engines.values() for x in e.__dict__.get("phase_steps", [])]
    if ph:  # FK_DEBUG_TIMING=1: per-phase host us per step, medians (plan includes its GPU wait)
        out["phase_us_median"] = {k: statistics.median(x[k] for x in ph) for k in ph[0]}
        n = len(ph)
        waits = sum(e.pool_stats().host_wait_ns for e in mgr.engines.values() if e.device is not None)
        out["plan_gpu_wait_us_mean"] = waits / 1e3 / n
    print(json.dumps(out))


if __name__ == "__main__":
    main()
