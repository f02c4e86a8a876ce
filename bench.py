#!/usr/bin/env python
"""Benchmark: shared-prefix decode attention tokens/s and HBM GB/s vs roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

A "step" is one engine decode step through the public API (GpuEngine.step:
plan -> per-layer prefix/private/merge attention kernels for all L layers ->
one-token growth -> K/V append) for the B forks of one prefix-affinity group.
Per GPU the workload is fixed (one group per rank, weak scaling); under
torchrun every rank runs its own engine on its own GPU with no collective
on the data path.  Rank 0 prints one JSON line.

  value : tokens/s with inputs (Q, new K/V rows) resident in HBM, device
          timed with CUDA events on the engine stream, max over ranks.
  e2e   : the same through the engine API with host (pinned) inputs: Q and
          K/V rows copied H2D and the attention output copied D2H each step.
  roofline : the per-layer attention (fk_attn_decode) against measured HBM
          peak with algorithmic bytes = (batch_tokens * H * D * 2 * 2) + Q + out.
  cpu_baseline : the numpy oracle on the host cores, bounded sample.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[2] (headline): LLaMA-13B shape, 6k prefix x 64 forks, S=256
    "llama13b_p6000_b64": dict(model="LLaMA-13B", L=40, H=40, P=6000, B=64, S=256),
    "llama13b_p6000_b128": dict(model="LLaMA-13B", L=40, H=40, P=6000, B=128, S=256),
    "llama13b_p6000_b256": dict(model="LLaMA-13B", L=40, H=40, P=6000, B=256, S=256),
    # BASELINE.json configs[1]: LLaMA-7B shape
    "llama7b_p6000_b64": dict(model="LLaMA-7B", L=32, H=32, P=6000, B=64, S=256),
    # BASELINE.json configs[3]: map-reduce, 2 groups of 32 forks over 2k prefixes per GPU
    "mapreduce_13b": dict(model="LLaMA-13B", L=40, H=40, P=2000, B=32, S=None, groups=2),
    # BASELINE.json configs[4]: nested 4k -> 1k -> 64 users x 256 per GPU
    "nested_13b": dict(model="LLaMA-13B", L=40, H=40, P=4096, B=64, S=256, app=1024),
    # the same two workloads at the BASELINE totals, dealt over the ranks
    # (strong scaling): 16 map-reduce groups of 32 forks; 8 apps x 64 users
    # (512 requests) under one 4k system prompt, replicated per GPU
    "mapreduce_13b_16x32": dict(model="LLaMA-13B", L=40, H=40, P=2000, B=32, S=None, groups=16, strong=True),
    "nested_13b_8apps": dict(model="LLaMA-13B", L=40, H=40, P=4096, B=64, S=256, app=1024, apps=8, strong=True),
    # launcher smoke (tests): the strong deal at a 2-layer, 8-head shape, so
    # several ranks fit on one GPU
    "nested_smoke_8apps": dict(model="smoke (2 layers x 8 heads)", L=2, H=8, P=4096, B=64, S=256, app=1024, apps=8,
                               strong=True),
}
DEFAULT_CONFIG = "llama13b_p6000_b64"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []
        self.t_mark = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self):
        """Start of the timed region: only samples after this count."""
        self.t_mark = time.perf_counter()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = [ln for t, ln in self.lines if self.t_mark is None or t >= self.t_mark]
        if not lines:  # timed region shorter than one sample period
            lines = [ln for _, ln in self.lines[-2:]]
        for ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            try:
                pw.append(float(parts[3]))
            except ValueError:
                pass
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        # (board power: nvidia-smi's averaged reading, it trails the load by
        # ~1 s; sustained runs settle at the 1000 W cap, profiles/r02/power/)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(pw) if pw else None}


# ------------------------------------------------------------------ workload
def rank_units(cfg, rank=0, world=1):
    """Fork groups (map-reduce) or apps (nested) this rank serves: every one
    at the per-GPU configs, a round-robin deal of the BASELINE totals over the
    ranks at the strong-scaling ones (cluster.rank_groups)."""
    from paper_2405_19888_b200.cluster import rank_groups

    n = cfg.get("groups") or cfg.get("apps") or 1
    return rank_groups(rank, n, world) if cfg.get("strong") else list(range(n))


class DoesNotFit(RuntimeError):
    """The config's share for this rank does not fit one GPU's memory."""


def build_engine(cfg, device, torch, host_inputs=False, seed=0x5EED, out_len=4096, rank=0, world=1):
    import paper_2405_19888_b200 as P
    from paper_2405_19888_b200.workloads import drain_fills, fork_group, nested_forest

    L, H = cfg["L"], cfg["H"]
    geo = P.ModelGeometry(L, H, 128)
    eng = P.GpuEngine("e0", P.CostModel(), kv_tokens=1 << 30, device=device, geometry=geo,
                      model=P.SyntheticDecodeModel(seed))
    units = rank_units(cfg, rank, world)
    # back every page the run will use up front: growing the arena later is
    # a device-wide copy with old and new arenas live at once
    pg = lambda n: -(-n // 16)  # noqa: E731
    grow = pg(out_len) + 1
    if "app" in cfg:
        pages = pg(cfg["P"]) + len(units) * (pg(cfg["app"]) + cfg["B"] * (pg(cfg["S"]) + grow))
    elif cfg.get("groups"):
        pages = len(units) * (pg(cfg["P"]) + cfg["B"] * (pg(1024) + grow))
    else:
        pages = pg(cfg["P"]) + cfg["B"] * (pg(cfg["S"]) + grow)
    need = pages * L * 2 * H * 16 * 128 * 2
    free = torch.cuda.mem_get_info(device)[0]
    if need > 0.9 * free:  # (the strong-scaling configs hold the BASELINE totals: several GPUs)
        eng.close()
        raise DoesNotFit(f"KV arena {need / 1e9:.0f} GB for this rank's {len(units)} of {cfg.get('groups') or cfg.get('apps') or 1} "
                         f"group(s) > {free / 1e9:.0f} GB free on the GPU: run it over more GPUs (torchrun)")
    eng.reserve_pages(pages)
    if "app" in cfg:
        nested_forest(eng, cfg["P"], cfg["app"], len(units), cfg["S"], cfg["B"], out_len=out_len, seed=seed)
    elif cfg.get("groups"):
        import random
        rng = random.Random(0)
        lens = [[rng.randint(128, 1024) for _ in range(cfg["B"])] for _ in range(cfg["groups"])]
        for gi in units:
            fork_group(eng, cfg["P"], lens[gi], out_len=out_len, tag=f"g{gi}", seed=seed + gi)
    else:
        fork_group(eng, cfg["P"], [cfg["S"]] * cfg["B"], out_len=out_len, seed=seed)
    drain_fills(eng)
    rows = len(eng.gens)
    # leaf tokens when the model rows take over (the parity check's oracle:
    # positions >= n0 of a request's leaf hold its model K/V row)
    eng.bench_leaf_n0 = {eng.contexts[g.context_id].uid: (eng.contexts[g.context_id].token_count, r)
                         for r, g in enumerate(eng.gens.values())}
    # back the whole run's decode growth now, so no arena growth (a device-wide
    # copy) lands in the timed region
    st = eng.pool_stats()
    eng.reserve_pages(st.num_pages - st.free_pages + rows * (out_len // 16 + 2))
    shape = (L, rows, H, 128)
    gen = torch.Generator(device="cpu").manual_seed(seed)
    q = torch.randn(shape, generator=gen).to(torch.bfloat16)
    k = torch.randn(shape, generator=gen).to(torch.bfloat16)
    v = torch.randn(shape, generator=gen).to(torch.bfloat16)
    if host_inputs:
        q, k, v = q.pin_memory(), k.pin_memory(), v.pin_memory()
        eng.model = P.TensorDecodeModel(q, k, v, copy_out=True)
        eng.model.seed = seed
    else:
        dev = torch.device("cuda", device)
        q = q.to(dev)
        eng.model = P.TensorDecodeModel(q, k.to(dev), v.to(dev), out=torch.empty_like(q))
        eng.model.seed = seed
    torch.cuda.synchronize(device)
    return eng, rows


def alg_bytes_per_layer(info, rows, H, D=128):
    """(_batch_tokens) * H * D * 2 (K,V) * 2 B + Q + out."""
    return info.batch_tokens * H * D * 2 * 2 + 2 * rows * H * D * 2


def time_steps(eng, steps, torch):
    st = eng.stream
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(st)
    for _ in range(steps):
        eng.step()
    end.record(st)
    end.synchronize()
    return start.elapsed_time(end) / 1e3


def time_layers(eng, steps, torch):
    """Device time of the per-layer attention alone (same plan, same inputs,
    layers back to back as in the step)."""
    from paper_2405_19888_b200 import _lib

    L = eng.geometry.num_layers
    rows = eng.last_plan.num_rows
    H = eng.geometry.num_heads
    q = eng.model.q
    out = torch.empty_like(q)
    le = rows * H * 128 * 2
    st = eng.stream
    sp = ctypes.c_void_p(st.cuda_stream)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the engine's own path: all layers through fk_attn_decode_layers (one
    # CUDA graph replay per pass), per-layer kernels and PDL chain unchanged
    def one_pass():
        _lib.check(_lib.lib.fk_attn_decode_layers(eng._pool.handle, 0, L, ctypes.c_void_p(q.data_ptr()), le,
                                                  ctypes.c_void_p(out.data_ptr()), le, None, 0, sp))

    one_pass()  # (re)capture outside the timed region
    start.record(st)
    for _ in range(steps):
        one_pass()
    end.record(st)
    end.synchronize()
    return start.elapsed_time(end) / 1e3 / (steps * L)


def time_layers_isolated(eng, reps, torch):
    """Per-layer attention as a model sees it: one fk_attn_decode per layer,
    PDL only between the layer's own kernels (FK_OPT_PDL=1), and a foreign
    kernel between consecutive layers (the rest of the transformer layer),
    so nothing of layer l+1 overlaps layer l.  The L-layer sequence is
    captured in a CUDA graph (as a served model replays its decode step), so
    the host's launch rate is out of the measurement; the foreign kernels'
    own time, replayed alone in a graph, is subtracted.  Returns (mean layer
    seconds, foreign-kernel seconds per layer)."""
    from paper_2405_19888_b200 import _lib

    L = eng.geometry.num_layers
    rows = eng.last_plan.num_rows
    H = eng.geometry.num_heads
    q = eng.model.q
    out = torch.empty_like(q)
    le = rows * H * 128 * 2
    st = eng.stream
    sp = ctypes.c_void_p(st.cuda_stream)
    foreign = torch.empty(1 << 16, dtype=torch.float32, device=q.device)
    eng.set_option(_lib.FK_OPT_PDL, 1)
    eng.set_option(_lib.FK_OPT_GRAPH, 0)  # direct launches, captured below

    def one_pass(attn=True):
        for layer in range(L):
            foreign.add_(1.0)
            if attn:
                _lib.check(_lib.lib.fk_attn_decode(eng._pool.handle, layer, ctypes.c_void_p(q.data_ptr() + layer * le),
                                                   ctypes.c_void_p(out.data_ptr() + layer * le), None, sp))

    def timed(graph):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        graph.replay()
        start.record(st)
        for _ in range(reps):
            graph.replay()
        end.record(st)
        end.synchronize()
        return start.elapsed_time(end) / 1e3

    try:
        with torch.cuda.stream(st):
            one_pass()  # (warm: every kernel's attributes set before capture)
            st.synchronize()
            g_all, g_foreign = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_all, stream=st):
                one_pass()
            with torch.cuda.graph(g_foreign, stream=st):
                one_pass(attn=False)
            t_all = timed(g_all)
            t_foreign = timed(g_foreign)
    finally:
        eng.set_option(_lib.FK_OPT_PDL, 2)
        eng.set_option(_lib.FK_OPT_GRAPH, 1)
    return (t_all - t_foreign) / (reps * L), t_foreign / (reps * L)


def ncu_layer(eng, torch, batch_tokens, bytes_layer):
    """One layer's kernels inside a cudaProfilerStart/Stop range, on the plan
    the roofline is timed on, so an `ncu --profile-from-start off` run of
    bench.py measures DRAM traffic at exactly this batch_tokens (written with
    the algorithmic bytes to gpurun_out/ncu_layer.json)."""
    from paper_2405_19888_b200 import _lib

    q = eng.model.q
    out = torch.empty_like(q)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    _lib.check(_lib.lib.fk_attn_decode(eng._pool.handle, 0, ctypes.c_void_p(q.data_ptr()),
                                       ctypes.c_void_p(out.data_ptr()), None, ctypes.c_void_p(eng.stream.cuda_stream)))
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "ncu_layer.json"), "w") as f:
        json.dump({"batch_tokens": batch_tokens, "alg_bytes_per_layer": bytes_layer}, f)


def parity_check(eng, torch):
    """Outside the timed region: one more GpuEngine.step on the benchmarked
    engine (same plan path, kernels and CUDA graph as the timed steps) with the
    fp32 pre-cast output captured; layers 0 and L-1 against the fp64 oracle
    (the engine's synthetic prefill rows + the model's appended K/V rows)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from gpu_check import MAX_ABS, MEAN_REL_F32, REL_L2, check_history, tensor_model_oracle

    eng.capture_f32, eng.keep_history = True, True
    eng.history.clear()
    eng.step()
    eng.stream.synchronize()
    eng.capture_f32, eng.keep_history = False, False
    L = eng.geometry.num_layers
    kv, queries = tensor_model_oracle(eng, eng.bench_leaf_n0)
    t0 = time.perf_counter()
    w = check_history(eng, layers=[0, L - 1], kv=kv, queries=queries, strict=False)
    eng.history.clear()
    return {"max_abs": w["max_abs"], "rel_l2": w["rel_l2"], "mean_rel_f32": w["mean_rel_f32"], "pass": w["pass"],
            "layers": [0, L - 1], "rows": eng.last_plan.num_rows, "batch_tokens": int(eng.last_plan.batch_tokens),
            "tolerance": {"max_abs": MAX_ABS, "rel_l2": REL_L2, "mean_rel_f32": MEAN_REL_F32},
            "oracle": "fp64 un-decomposed softmax over each row's chain (oracle/forkattn_oracle.py attend_forest)",
            "step": "one GpuEngine.step after the timed region (same plan path and graph)",
            "check_s": round(time.perf_counter() - t0, 1)}


def cpu_baseline(cfg, budget_s=12.0, impl_steps=None):
    """numpy fp32 oracle (matmul form) on the host cores for one layer of the
    workload; tokens/s extrapolated x L.  Returns (tokens/s, sample, cores, secs)."""
    import numpy as np

    from oracle import forkattn_oracle as O

    H, P, B = cfg["H"], cfg["P"], cfg["B"]
    S = cfg["S"] or 576
    rng = np.random.default_rng(0)
    q = O.bf16_round(rng.standard_normal((B, H, 128), dtype=np.float32))
    pk = O.bf16_round(rng.standard_normal((P, H, 128), dtype=np.float32))
    pv = O.bf16_round(rng.standard_normal((P, H, 128), dtype=np.float32))
    sk = [O.bf16_round(rng.standard_normal((S, H, 128), dtype=np.float32)) for _ in range(B)]
    sv = [O.bf16_round(rng.standard_normal((S, H, 128), dtype=np.float32)) for _ in range(B)]
    O.attend_shared_batch(q, pk, pv, sk, sv)  # warm
    times = []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        O.attend_shared_batch(q, pk, pv, sk, sv)
        times.append(time.perf_counter() - t0)
        if impl_steps is not None:
            if len(times) >= impl_steps:
                break
        elif time.perf_counter() - t_all > budget_s:
            break
    t_layer = statistics.median(times)
    cores = len(os.sched_getaffinity(0))
    sample = (f"1 of {cfg['L']} layers ({H} heads, {B} rows, P={P}, S={S}) numpy fp32 matmul form, "
              f"{len(times)} reps, median, extrapolated x{cfg['L']} layers")
    return B / (cfg["L"] * t_layer), sample, cores, t_layer


# ----------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the post-run parity check against the oracle")
    ap.add_argument("--no-isolated", action="store_true", help="skip the isolated-layer timing")
    ap.add_argument("--tc-min-fanout", type=int, default=None)
    ap.add_argument("--corun", type=int, default=None, help="FK_OPT_CORUN (default: library default, 1)")
    ap.add_argument("--prefix-rate-pct", type=int, default=None)
    ap.add_argument("--opt", action="append", default=[], metavar="NAME=V",
                    help="any FK_OPT_<NAME> (repeatable; A/B experiments)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    strong = bool(cfg.get("strong"))
    units = cfg.get("groups") or cfg.get("apps") or 1
    workload = dict(workload=args.config, model=cfg["model"], layers=cfg["L"], heads=cfg["H"], head_dim=128,
                    prefix_tokens=cfg["P"], forks=cfg["B"] * units,
                    suffix_tokens=cfg["S"] if cfg["S"] else "U[128,1024]",
                    per_gpu=("BASELINE totals dealt over the GPUs by whole fork group / app (strong scaling)"
                             if strong else "one prefix-affinity group set per GPU (weak scaling)"),
                    l2="inputs larger than L2 (KV per layer >> 126 MB; layers stream distinct pages)",
                    parallelism=f"dp{args.gpus} (independent engines, no collective)")
    if "app" in cfg:
        workload["app_tokens"] = cfg["app"]
    metric = "shared-prefix decode attn tokens/s + HBM GB/s vs roofline, 1/2/4/8 B200"

    if args.impl == "reference":
        if rank != 0:
            return
        rows = cfg["B"] * units
        c = dict(cfg, B=rows)
        t0 = time.perf_counter()
        tok_s, sample, cores, t_layer = cpu_baseline(c, impl_steps=max(1, args.steps) + max(0, args.warmup))
        # one "step" of this arm is one sampled layer (the whole 40-layer step
        # would take minutes per step on the host); tokens/s is extrapolated
        # to all L layers and says so
        line = {"metric": metric, "value": tok_s, "unit": "tokens/s", "impl": "reference", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_layer,
                "step_is": f"one sampled layer of the {cfg['L']}-layer step (median); value extrapolated x{cfg['L']}",
                "extrapolated": True, "layer_ms": 1e3 * t_layer, "layers": cfg["L"],
                "wall_s": round(time.perf_counter() - t0, 2),
                "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic", "config": workload,
                "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample},
                "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch

    dist = None
    if world > 1:
        # the process group only carries the barrier and the out-of-region
        # timing reductions (no collective on the data path): gloo on the
        # host, so several ranks can even share one GPU (smoke tests)
        import torch.distributed as dist  # noqa: F811

        dist.init_process_group("gloo")
    device = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(device)
    from paper_2405_19888_b200 import _lib
    from paper_2405_19888_b200.cluster import max_over_ranks, sum_over_ranks

    out_len = 2 * (args.steps + args.warmup) + 64
    why = None
    try:
        eng, rows = build_engine(cfg, device, torch, out_len=out_len, rank=rank, world=world)
    except DoesNotFit as e:
        why = str(e)
    if dist is not None:  # every rank stops when one cannot hold its share
        flag = torch.tensor([0 if why else 1], dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not flag.item() and why is None:
            why = "another rank's share does not fit its GPU"
            eng.close()
    if why:
        if rank == 0:
            print(json.dumps({"metric": metric, "config": workload, "n_gpus": args.gpus, "unavailable": why}))
        return

    def apply_options(e):
        if args.tc_min_fanout is not None:
            e.set_option(_lib.FK_OPT_TC_MIN_FANOUT, args.tc_min_fanout)
        if args.corun is not None:
            e.set_option(_lib.FK_OPT_CORUN, args.corun)
        if args.prefix_rate_pct is not None:
            e.set_option(_lib.FK_OPT_PREFIX_RATE_PCT, args.prefix_rate_pct)
        for kv in args.opt:
            k, v = kv.split("=")
            e.set_option(getattr(_lib, "FK_OPT_" + k), int(v))

    apply_options(eng)
    L, H = cfg["L"], cfg["H"]
    # the clock sampler starts before the warm-up so nvidia-smi's own start-up
    # (NVML init) is outside the timed region
    clocks = ClockSampler(device)
    clocks.start()
    for _ in range(max(args.warmup, 3)):
        eng.step()
    torch.cuda.synchronize(device)

    def barrier():
        torch.cuda.synchronize(device)
        if dist is not None:
            dist.barrier()

    barrier()
    clocks.mark()
    t_steps = time_steps(eng, args.steps, torch)
    barrier()
    info = eng.last_plan
    batch_tokens = int(info.batch_tokens)
    bytes_layer = alg_bytes_per_layer(info, rows, H)
    plan_line = {"rows": info.num_rows, "shared_ctx": info.num_shared_ctx, "prefix_ctas": info.num_prefix_ctas,
                 "max_slots": info.max_slots, "tc_items": info.num_tc_items, "mma_items": info.num_mma_items}
    # per-layer attention alone for the roofline (same plan as the last step);
    # the isolated-layer figure is measured in alternation with it (the
    # part's clock moves under its power cap), medians of five rounds each
    t_layers, t_isos, t_foreign = [], [], 0.0
    for _ in range(5):
        t_layers.append(time_layers(eng, max(args.steps // 6, 3), torch))
        if not args.no_isolated:
            ti, t_foreign = time_layers_isolated(eng, 3, torch)
            t_isos.append(ti)
    t_layer = statistics.median(t_layers)
    barrier()
    if os.environ.get("FK_NCU_LAYER"):  # profiles/traffic_all.sh: ncu --profile-from-start off
        ncu_layer(eng, torch, batch_tokens, bytes_layer)
    clk = clocks.stop()
    iso = (max_over_ranks(statistics.median(t_isos)), t_foreign) if t_isos else None
    parity = None if args.no_check else parity_check(eng, torch)
    t_steps = max_over_ranks(t_steps)
    t_layer = max_over_ranks(t_layer)
    total_rows = int(sum_over_ranks(rows))
    peak, peak_kind = load_peaks()
    achieved = bytes_layer / t_layer / 1e9
    value = total_rows * args.steps / t_steps
    # per layer: prefix kernel(s) + private + merge; per step: one K/V append
    launches_per_step = L * (2 + int(info.num_mma_items > 0) + int(info.num_tc_items > 0)) + 1

    # ---- e2e: host (pinned) inputs through the engine API
    e2e = None
    if not args.no_e2e:
        eng.close()
        del eng
        torch.cuda.empty_cache()
        eng2, rows2 = build_engine(cfg, device, torch, host_inputs=True, out_len=out_len, rank=rank, world=world)
        apply_options(eng2)
        for _ in range(max(args.warmup, 3)):
            eng2.step()
        barrier()
        t0 = time.perf_counter()
        t_e2e = time_steps(eng2, args.steps, torch)
        wall = time.perf_counter() - t0
        barrier()
        t_e2e = max_over_ranks(max(t_e2e, wall))
        bi = 3 * L * rows2 * H * 128 * 2
        bo = L * rows2 * H * 128 * 2
        e2e = {"value": total_rows * args.steps / t_e2e, "unit": "tokens/s", "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo, "ms_per_step": 1e3 * t_e2e / args.steps}
        eng2.close()
    else:
        eng.close()

    traffic, traffic_src, traffic_tok = None, None, None
    try:  # DRAM bytes per layer (prefix + private + merge) from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(args.config)
        if tr:
            traffic_src = tr["source"]
            traffic_tok = tr.get("bytes_per_token")
            if tr.get("batch_tokens") == batch_tokens:  # captured at this run's final plan
                traffic = tr["layer_bytes"]
            elif traffic_tok:  # another run length: the measured bytes per streamed token, scaled
                traffic = traffic_tok * batch_tokens
                traffic_src += f" (captured at {tr.get('batch_tokens')} tokens, scaled per token)"
    except Exception:
        pass

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:  # the CPU baseline is an N=1 figure
            tok_s, sample, cores, _ = cpu_baseline(dict(cfg, B=rows))
            cpu = {"value": tok_s, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample}
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "traffic_bytes_per_token": traffic_tok,
                "alg_bytes_per_token": H * 128 * 2 * 2, "peak_kind": peak_kind,
                "kernel": "fk_attn_decode (prefix + private/merge kernels, one layer)",
                "alg_bytes_per_layer": bytes_layer, "layer_us": t_layer * 1e6,
                "batch_tokens": batch_tokens,
                "roofline_tokens_per_s": rows * peak * 1e9 / (L * bytes_layer)}
        if iso is not None:
            roof["layer_us_isolated"] = iso[0] * 1e6
            roof["frac_isolated"] = bytes_layer / iso[0] / 1e9 / peak
            roof["isolated_mode"] = ("one fk_attn_decode per layer, PDL within the layer only, a foreign kernel "
                                     f"between layers ({iso[1] * 1e6:.2f} us, subtracted); the layer sequence "
                                     "replayed as a CUDA graph")
        line = {
            "metric": metric,
            "value": value,
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": 1e3 * t_steps / args.steps,
            "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic",
            "config": workload,
            "roofline": roof,
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
            "plan": plan_line,
        }
        if world > 1:
            line["rows_total"] = total_rows
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
