"""The reference runtime drives the B200 path.

semflow's SemanticManager builds its engines at one site
(manager.py:130-139); rebinding `semflow.manager.Engine` to
`engine_factory(...)` puts a GpuEngine per engine id on the GPUs
(eI -> cuda:(I mod ndev)).  The reference's own experiment harness then runs
a shared-prompt serving workload end to end -- `_place_one` forks every
request from the 6k system prompt (manager.py:465-511), `_step_engine`
steps the engines (manager.py:623-636), `_complete_request` finishes them --
and every decode step executes the attention kernels on the device.

Checked: the manager's view (traces, step reports, end time, peak blocks)
is identical to the unmodified reference Engine's run, and every recorded
decode step's attention agrees with the fp64 oracle.  semflow comes from
/root/reference (build container) or baseline/_ref (the unmodified install
that travels to the GPU box).
"""

import dataclasses

import pytest

import paper_2405_19888_b200 as P

from gpu_check import check_history

pytestmark = pytest.mark.gpu

semflow = pytest.importorskip("semflow", reason="the reference runtime (semflow) is not importable")


def run_manager(factory, engines=1, **cfg):
    import semflow.manager as sm
    from semflow.config import Config
    from semflow.experiments import run_workload_manager
    from semflow.workloads import shared_prompt_serving

    wl = shared_prompt_serving(1, users=64, system_prompt_len=6000, unique_len=200, output_len=8)
    saved = sm.Engine
    if factory is not None:
        sm.Engine = factory
    try:
        mgr, runners, end_ns = run_workload_manager(wl, "semflow", Config(total_blocks=30000, engines=engines, **cfg))
    finally:
        sm.Engine = saved
    return mgr, end_ns


def manager_view(mgr, end_ns):
    view = {"end_ns": end_ns}
    for eid, e in sorted(mgr.engines.items()):
        view[eid] = {
            "trace": list(e.trace),
            "reports": [dataclasses.astuple(r) for r in e.reports],
            "peak": e.store.peak_used,
            "emitted": e.total_emitted,
            "clock": e.clock_ns,
        }
    return view


@pytest.mark.parametrize("engines", [1, 2])
def test_reference_manager_drives_gpu_engines(cuda_device, engines):
    import torch

    want = manager_view(*run_manager(None, engines))
    factory = P.engine_factory(P.ModelGeometry(2, 8, 128), capture_f32=True, keep_history=True)
    mgr, end_ns = run_manager(factory, engines)
    got = manager_view(mgr, end_ns)
    assert got == want
    ndev = torch.cuda.device_count()
    decode_steps = 0
    for i, (eid, eng) in enumerate(sorted(mgr.engines.items())):
        assert isinstance(eng, P.GpuEngine) and eng.device == i % ndev
        if not eng.history:
            continue
        eng.stream.synchronize()
        decode_steps += len(eng.history)
        # the 6000-token system prompt is one shared context read by the forks
        assert max(r["batch_tokens"] for r in eng.history) >= 6000
        check_history(eng)
    assert decode_steps >= 8
    assert sum(e.kv_tokens_streamed for e in mgr.engines.values()) == sum(
        r.batch_tokens for e in mgr.engines.values() for r in e.reports)


def test_shared_ctx_fallback_migrates_the_prefix(cuda_device):
    """With a throughput capacity the prefix holder cannot absorb, the
    scheduler's `shared-ctx` placement falls back to `solo` on the second
    engine (scheduler.py:198-222), which must then fill the 6k system
    prompt.  With engine_factory(migrate_prefixes=True) that fill copies the
    holder's K/V (fk_ctx_copy_kv) instead of prefilling: the manager's view
    is unchanged, the copied context holds the holder's rows (oracle alias),
    and every decode step still matches the oracle."""
    import oracle.forkattn_oracle as O

    cfg = dict(throughput_capacity=10000)
    want = manager_view(*run_manager(None, 2, **cfg))
    factory = P.engine_factory(P.ModelGeometry(2, 8, 128), capture_f32=True, keep_history=True,
                               migrate_prefixes=True)
    mgr, end_ns = run_manager(factory, 2, **cfg)
    assert manager_view(mgr, end_ns) == want
    engines = [e for _, e in sorted(mgr.engines.items())]
    assert sum(e.prefix_migrations for e in engines) >= 1
    assert sum(e.migrated_tokens for e in engines) >= 6000
    for eng in engines:
        if not eng.history:
            continue
        eng.stream.synchronize()
        alias = {dst: src for dst, (_, src, _) in eng.migrated.items()}
        kv = O.KVCache(eng.model_seed, eng.geometry.num_heads, eng.model_k_scale, alias=alias)
        check_history(eng, kv=kv)


def test_graph_replay_key_under_a_serving_load(cuda_device, monkeypatch):
    """Under the manager the batch changes from step to step (requests join
    and finish).  The engine-owned q/out buffers keep their pointers (row
    capacity), the prefix grid its size (hysteresis), so most steps replay
    the cached CUDA graph without recording (fk_attn_decode_layers' replay
    key).  FK_DEBUG_GRAPH_CHECK=1 records every step anyway and fails if a
    replayed step's launches would have differed; outputs (bf16, no f32
    capture, which would change a pointer every step) match the oracle."""
    monkeypatch.setenv("FK_DEBUG_GRAPH_CHECK", "1")
    want = manager_view(*run_manager(None, 1))
    factory = P.engine_factory(P.ModelGeometry(2, 8, 128), keep_history=True)
    mgr, end_ns = run_manager(factory, 1)
    assert manager_view(mgr, end_ns) == want
    (eng,) = mgr.engines.values()
    eng.stream.synchronize()
    steps = len(eng.history)
    replays = eng.pool_stats().graph_replays
    assert steps >= 8 and replays >= steps // 2, (steps, replays)
    check_history(eng, f32=False)
