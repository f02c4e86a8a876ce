"""GPU parity: decode attention through the C-ABI vs the CPU oracle.

Every case builds a forest through the reference engine surface (fill /
create_context / generate), runs real engine steps on cuda:0 (plan ->
per-layer prefix/private/merge kernels -> one-token growth -> append) and
compares each recorded step with the oracle's un-decomposed softmax.
Integer side-conditions (batch_tokens == dedup walk, block ids) are
asserted alongside.
"""

import random

import numpy as np
import pytest

import paper_2405_19888_b200 as P
from paper_2405_19888_b200 import _lib
from paper_2405_19888_b200.workloads import fork_group, nested_forest

from gpu_check import check_history

pytestmark = pytest.mark.gpu


PATH = {"path": "mma"}


@pytest.fixture(params=["mma", "tc", "grp"], autouse=True)
def prefix_path(request):
    """Every case runs with the shared prefixes on the warp-level mma.sync
    kernel, on the tcgen05 kernel (fan-out threshold 2), and with shared
    contexts of fan-out <= 16 streamed by the private kernel for groups of up
    to 8 rows (FK_OPT_GROUP_FANOUT=16; larger fan-outs on tcgen05)."""
    PATH["path"] = request.param
    yield request.param


_OPEN = []


@pytest.fixture(autouse=True)
def close_engines():
    """Engines are closed when their test ends: a process holds at most 64
    device pools, and under compute-sanitizer the interpreter's frames (held
    from C) keep finished tests' engines alive, so release cannot wait for
    garbage collection (profiles/sanitize_full.sh runs this whole file)."""
    yield
    while _OPEN:
        _OPEN.pop().close()


def make_engine(cuda_device, H, L=1, shared=True, k_scale=1.0, seed=0x5EED, kv_tokens=1 << 20, **kw):
    eng = P.GpuEngine("e0", P.CostModel(shared_kernel=shared), kv_tokens=kv_tokens, device=cuda_device,
                      geometry=P.ModelGeometry(L, H, 128), model=P.SyntheticDecodeModel(seed, k_scale),
                      capture_f32=True, keep_history=True, **kw)
    eng.set_option(_lib.FK_OPT_TC_MIN_FANOUT, 0 if PATH["path"] == "mma" else 2)
    eng.set_option(_lib.FK_OPT_GROUP_FANOUT, 16 if PATH["path"] == "grp" else 0)
    _OPEN.append(eng)
    return eng


def run_steps(eng, n):
    for _ in range(n):
        rep = eng.step()
        if rep is None:
            break
        running = [g for g in eng.gens.values()]
        assert rep.batch_tokens >= 0
    eng.stream.synchronize()


def assert_plan_matches_walk(eng):
    for rec in eng.history:
        # batch_tokens from the C++ planner == reference dedup walk over the snapshot
        if eng.cost.shared_kernel:
            seen = {}
            for chain in rec["chains"]:
                for uid, n in chain:
                    seen[uid] = n
            assert rec["batch_tokens"] == sum(seen.values())
        else:
            assert rec["batch_tokens"] == sum(n for chain in rec["chains"] for uid, n in chain)


def test_tiny_config1(cuda_device):
    """BASELINE config 1: 1 layer, 32x128, 1k prefix, 8 forks x 64 suffix."""
    eng = make_engine(cuda_device, H=32)
    fork_group(eng, 1024, [64] * 8, out_len=3)
    run_steps(eng, 3)
    assert eng.last_plan.num_shared_ctx == 1 and eng.last_plan.num_rows == 8
    assert eng.history[0]["batch_tokens"] == 1024 + 8 * 64
    w = check_history(eng)
    assert_plan_matches_walk(eng)
    print("tiny", w)


def test_ragged_suffixes_cross_pages(cuda_device):
    rng = random.Random(1)
    eng = make_engine(cuda_device, H=4, L=2)
    # 7, 8, 9, 24, 25: last pages on either side of the private kernel's
    # half-page load (<= 8 tokens: rows 0..7 only); 20 steps move each
    # chain's last page through both forms
    lens = [rng.randint(0, 70) for _ in range(13)] + [0, 1, 7, 8, 9, 15, 16, 17, 24, 25]
    fork_group(eng, 100, lens, out_len=20, seed=3)  # 100 = partial last prefix page
    run_steps(eng, 20)
    check_history(eng)
    assert_plan_matches_walk(eng)


def test_nested_three_levels(cuda_device):
    eng = make_engine(cuda_device, H=8, L=1)
    nested_forest(eng, root_len=300, app_len=50, n_apps=3, user_len=33, users_per_app=4, out_len=5)
    run_steps(eng, 5)
    assert eng.last_plan.num_shared_ctx == 4  # root + 3 apps
    check_history(eng)
    assert_plan_matches_walk(eng)


def test_unshared_mode_streams_whole_chains(cuda_device):
    eng = make_engine(cuda_device, H=8, shared=False)
    fork_group(eng, 500, [40] * 6, out_len=4)
    run_steps(eng, 4)
    assert eng.last_plan.num_shared_ctx == 0
    assert eng.history[0]["batch_tokens"] == 6 * 540
    check_history(eng)


def test_two_generations_on_one_leaf(cuda_device):
    eng = make_engine(cuda_device, H=4)
    eng.fill([1] * 200, "root", None, boundary_hash=1)
    eng.fill([1] * 30, "leaf", "root", boundary_hash=2)
    eng.generate("a", "leaf", [1] * 4, "")
    eng.generate("b", "leaf", [1] * 4, "")
    eng.fill([1] * 20, "solo", "root", boundary_hash=3)
    eng.generate("c", "solo", [1] * 4, "")
    run_steps(eng, 4)
    assert eng.contexts["leaf"].token_count == 30 + 8  # both rows grow the shared leaf
    check_history(eng)


def test_stress_peaky_softmax(cuda_device):
    eng = make_engine(cuda_device, H=8, k_scale=8.0)
    fork_group(eng, 700, [50, 90, 3], out_len=3)
    run_steps(eng, 3)
    check_history(eng)


@pytest.mark.parametrize("order", [0, 1])
def test_merge_by_either_kernel(cuda_device, order):
    """launch order 1 runs the private kernel first, so the prefix kernel's
    CTAs are the last arrivers and perform the LSE merge."""
    eng = make_engine(cuda_device, H=4)
    eng.set_option(_lib.FK_OPT_LAUNCH_ORDER, order)
    fork_group(eng, 333, [7, 64, 129, 0], out_len=3)
    run_steps(eng, 3)
    check_history(eng)


def test_large_fanout_multiple_query_blocks(cuda_device):
    eng = make_engine(cuda_device, H=2)
    fork_group(eng, 260, [5] * 150, out_len=2)  # 150 queries -> 3 blocks of 64
    run_steps(eng, 2)
    check_history(eng)


def test_many_splits(cuda_device):
    eng = make_engine(cuda_device, H=2)
    eng.set_option(_lib.FK_OPT_MIN_SPLIT_PAGES, 1)  # mma path: one split per page
    eng.set_option(_lib.FK_OPT_PREFIX_TARGET_CTAS, 4096)  # tcgen05 path: one-tile ranges
    fork_group(eng, 1000, [20, 21], out_len=2)
    run_steps(eng, 2)
    assert eng.last_plan.max_slots > 5
    check_history(eng)


def test_stream_k_pieces_cross_items(cuda_device):
    """Few CTAs over many prefix tiles: stream-K ranges cut items mid-way and
    span head / context boundaries (tcgen05), many splits (mma)."""
    eng = make_engine(cuda_device, H=5, L=2)
    eng.set_option(_lib.FK_OPT_PREFIX_TARGET_CTAS, 7)
    fork_group(eng, 2100, [33] * 9, out_len=2, tag="a", seed=1)
    fork_group(eng, 700, [3] * 140, out_len=2, tag="b", seed=2)  # 140 rows: 2 x 128-query blocks
    run_steps(eng, 2)
    check_history(eng)


def test_headline_shape_one_layer(cuda_device):
    """LLaMA-13B head count, 6k prefix x 64 forks x 256: the bench shape, 1 layer."""
    eng = make_engine(cuda_device, H=40, L=1)
    fork_group(eng, 6000, [256] * 64, out_len=1)
    run_steps(eng, 1)
    check_history(eng)


def test_single_request_and_empty_chain(cuda_device):
    eng = make_engine(cuda_device, H=4)
    eng.fill([1] * 77, "only", None)
    eng.generate("r", "only", [1] * 3, "")
    eng.create_context("empty", None)  # zero tokens: output defined as 0
    eng.generate("z", "empty", [1] * 2, "")
    run_steps(eng, 3)
    check_history(eng)
    first = eng.history[0]
    z = first["rows"].index("z")
    assert np.abs(first["output"][:, z].float().numpy()).max() == 0.0


def test_decode_oom_skips_append(cuda_device):
    eng = make_engine(cuda_device, H=4, kv_tokens=16 * 12)
    eng.fill([1] * 16 * 10, "root", None)
    eng.fill([1] * 16, "a", "root")
    eng.fill([1] * 15, "b", "root")
    eng.generate("ra", "a", [1] * 3, "")
    eng.generate("rb", "b", [1] * 3, "")
    reps = [eng.step() for _ in range(3)]
    eng.stream.synchronize()
    assert any(r.failed for r in reps)
    check_history(eng)


def test_engine_pages_are_physical_and_logical_ids_monotonic(cuda_device):
    eng = make_engine(cuda_device, H=2)
    fork_group(eng, 64, [16, 16], out_len=1)
    logical, physical = eng.context_pages("e0.c0")
    assert logical == list(range(4))
    assert len(set(physical)) == 4


@pytest.mark.parametrize("corun", [0, 1])
def test_corun_and_serial_sm_split(cuda_device, corun):
    """FK_OPT_CORUN=1 splits the SMs between the tcgen05 prefix CTAs and the
    private stream (launched back to back); 0 gives each kernel every SM."""
    eng = make_engine(cuda_device, H=8, L=2)
    eng.set_option(_lib.FK_OPT_CORUN, corun)
    fork_group(eng, 1500, [300, 17, 64, 250, 129] * 4, out_len=3)
    run_steps(eng, 3)
    check_history(eng)


def test_host_tensor_pipeline_matches_device_tensors(cuda_device):
    """Pinned-host Q/K/V (copied in per layer on a copy stream, output copied
    back per layer) give bit-identical outputs to device-resident rows."""
    import torch

    outs = []
    for host in (False, True):
        eng = make_engine(cuda_device, H=8, L=3)
        fork_group(eng, 700, [40, 90, 3, 17], out_len=3)
        from paper_2405_19888_b200.workloads import drain_fills
        drain_fills(eng)
        rows = len(eng.gens)
        g = torch.Generator().manual_seed(7)
        q, k, v = (torch.randn((3, rows, 8, 128), generator=g).to(torch.bfloat16) for _ in range(3))
        if host:
            eng.model = P.TensorDecodeModel(q.pin_memory(), k.pin_memory(), v.pin_memory(), copy_out=True)
        else:
            dev = torch.device("cuda", cuda_device)
            eng.model = P.TensorDecodeModel(q.to(dev), k.to(dev), v.to(dev))
        eng.capture_f32 = False
        got = []
        for _ in range(3):
            eng.step()
            eng.stream.synchronize()
            got.append(eng.last_output.cpu().clone())
            if host:
                assert torch.equal(eng.model.host_out, got[-1])
        outs.append(got)
        eng.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_fill_with_model_kv_rows(cuda_device):
    """fill(kv=(k, v)) writes the caller's prefill rows (fk_fill_kv); decode
    attention over them matches fp64 softmax over the same bf16 values, for
    a shared prefix, ragged leaves (partial pages) and the step's appended
    rows."""
    import torch

    from oracle import forkattn_oracle as O

    H, L = 4, 2
    dev = torch.device("cuda", cuda_device)
    eng = make_engine(cuda_device, H=H, L=L)
    g = torch.Generator().manual_seed(11)

    def rows(n):
        return [torch.randn((L, n, H, 128), generator=g).to(torch.bfloat16) for _ in range(2)]

    ctx_kv = {}
    pk, pv = rows(333)
    eng.fill([1] * 333, "root", None, boundary_hash=1, kv=(pk.to(dev), pv.to(dev)))
    ctx_kv["root"] = (pk, pv)
    lens = [5, 16, 17, 40]
    for i, n in enumerate(lens):
        lk, lv = rows(n)
        eng.fill([1] * n, f"leaf{i}", "root", boundary_hash=10 + i, kv=(lk.to(dev), lv.to(dev)))
        ctx_kv[f"leaf{i}"] = (lk, lv)
        eng.generate(f"r{i}", f"leaf{i}", [1] * 3, "")
    from paper_2405_19888_b200.workloads import drain_fills
    drain_fills(eng)
    B = len(lens)
    q = torch.randn((L, B, H, 128), generator=g).to(torch.bfloat16)
    k_new, v_new = rows(B)
    eng.model = P.TensorDecodeModel(q.to(dev), k_new.to(dev), v_new.to(dev))
    eng.capture_f32 = False
    outs = []
    for _ in range(2):
        eng.step()
        eng.stream.synchronize()
        outs.append(eng.last_output.float().cpu().numpy())
    for step, out in enumerate(outs):
        for b in range(B):
            kk = torch.cat([ctx_kv["root"][0], ctx_kv[f"leaf{b}"][0]] + ([k_new[:, b:b + 1]] if step else []), 1)
            vv = torch.cat([ctx_kv["root"][1], ctx_kv[f"leaf{b}"][1]] + ([v_new[:, b:b + 1]] if step else []), 1)
            for layer in range(L):
                want = O.attend(q[layer, b].float().numpy(), kk[layer].float().numpy(),
                                vv[layer].float().numpy())
                r = O.tolerance_report(out[layer, b], want)
                assert r["max_abs"] <= 2e-2 and r["rel_l2"] <= 4e-3, (step, b, layer, r)


def test_prefix_migration_between_pools(cuda_device):
    """fill(kv_from=(engine, ctx)) copies a context's KV from another pool
    (fk_ctx_copy_kv; NVLink peer reads when the pools are on different GPUs,
    here both on cuda_device): decoding the migrated forest gives outputs
    bit-identical to decoding it where it was prefilled."""
    import torch

    H, L = 4, 2
    a = make_engine(cuda_device, H=H, L=L)
    b = make_engine(cuda_device, H=H, L=L)
    b.fill([7] * 16, "pad", None)  # different physical pages in b
    lens = [3, 16, 40]
    a.fill([1] * 700, "root", None, boundary_hash=1)
    b.fill([1] * 700, "root", None, boundary_hash=1, kv_from=(a, "root"))
    for i, n in enumerate(lens):
        a.fill([1] * n, f"l{i}", "root", boundary_hash=10 + i)
        b.fill([1] * n, f"l{i}", "root", boundary_hash=10 + i, kv_from=(a, f"l{i}"))
        for e in (a, b):
            e.generate(f"r{i}", f"l{i}", [1] * 2, "")
    from paper_2405_19888_b200.workloads import drain_fills
    g = torch.Generator().manual_seed(5)
    dev = torch.device("cuda", cuda_device)
    q, k, v = (torch.randn((L, len(lens), H, 128), generator=g).to(torch.bfloat16).to(dev) for _ in range(3))
    outs = []
    for e in (a, b):
        drain_fills(e)
        e.model = P.TensorDecodeModel(q, k, v)
        e.capture_f32 = False
        got = []
        for _ in range(2):
            e.step()
            e.stream.synchronize()
            got.append(e.last_output.cpu().clone())
        outs.append(got)
    assert a.context_pages("root")[1] != b.context_pages("root")[1]
    for x, y in zip(*outs):
        assert torch.equal(x, y)
    a.close()
    b.close()


def test_mapreduce_shape_one_layer(cuda_device):
    """BASELINE config 4 per GPU: 2 groups of 32 forks over 2k-token chunk
    prefixes, suffixes U[128, 1024] (random.Random(0)), 13B head count."""
    rng = random.Random(0)
    eng = make_engine(cuda_device, H=40, L=1)
    for gi in range(2):
        fork_group(eng, 2000, [rng.randint(128, 1024) for _ in range(32)], out_len=1, tag=f"g{gi}", seed=gi)
    run_steps(eng, 1)
    assert eng.last_plan.num_shared_ctx == 2 and eng.last_plan.num_rows == 64
    check_history(eng)
    assert_plan_matches_walk(eng)


def test_nested_shape_one_layer(cuda_device):
    """BASELINE config 5 per GPU: 4k system prompt -> 1k app prompt -> 64
    users x 256, 13B head count (three-level chain, two shared levels)."""
    eng = make_engine(cuda_device, H=40, L=1)
    nested_forest(eng, root_len=4096, app_len=1024, n_apps=1, user_len=256, users_per_app=64, out_len=1)
    run_steps(eng, 1)
    assert eng.last_plan.num_shared_ctx == 2 and eng.last_plan.num_rows == 64
    check_history(eng)
    assert_plan_matches_walk(eng)


def test_fanout_256_two_query_blocks(cuda_device):
    """BASELINE config 3 at 256 forks: two 128-query tcgen05 blocks per head
    (or four 64-query mma blocks) over one 6k prefix, 8 heads."""
    eng = make_engine(cuda_device, H=8, L=1)
    fork_group(eng, 6000, [64] * 256, out_len=1)
    run_steps(eng, 1)
    check_history(eng)


def test_fill_while_decoding(cuda_device):
    """Fills run on their own stream: a new fork group is prefilled between
    decode steps of another, and finished contexts' pages are recycled into
    it; decode waits only for the fills of contexts it reads."""
    eng = make_engine(cuda_device, H=4, L=2)
    fork_group(eng, 300, [20, 33], out_len=6, tag="a", seed=1)
    run_steps(eng, 2)
    fork_group(eng, 500, [7, 64, 90], out_len=3, tag="b", seed=2)  # joins mid-run
    run_steps(eng, 3)
    freed = 0
    for rid, g in [(r, g) for r, g in eng.gens.items() if g.done]:
        eng.finish_generation(rid)
        if eng.contexts[g.context_id].refcount == 0:
            eng.free_context(g.context_id)  # its pages go back to the free stack
            freed += 1
    assert freed > 0
    free_before = eng.pool_stats().free_pages
    fork_group(eng, 250, [16, 17], out_len=2, tag="c", seed=3)
    assert eng.pool_stats().free_pages < free_before  # group c reuses recycled pages
    run_steps(eng, 4)
    check_history(eng)
    assert_plan_matches_walk(eng)


def test_discarded_fill_then_decode_growth_into_its_pages(cuda_device):
    """A context freed while its fill may still be writing (the manager frees
    just-filled contexts on OutOfMemory, manager.py:489-492): its pages go
    back to the free stack and the next decode growth hands them to running
    leaves, whose new K/V rows must land after the old fill (the engine
    stream waits for it at discard time)."""
    eng = make_engine(cuda_device, H=8, L=4)
    fork_group(eng, 64, [16, 32, 48], out_len=4)  # leaves end on page boundaries: step 1 grows
    eng.fill([1] * 4000, "junk", None)  # 250 pages, filled on the fill stream
    junk_pages = set(eng.context_pages("junk")[1])
    eng.free_context("junk")            # back on the free stack, fill possibly still running
    run_steps(eng, 4)
    grown = {eng.context_pages(leaf)[1][-1] for leaf in ("e0.c1", "e0.c2", "e0.c3")}
    assert grown <= junk_pages  # decode growth took the recycled pages
    check_history(eng)


@pytest.mark.parametrize("suffix", [600, 2100])
def test_merge_many_partials(cuda_device, suffix):
    """One-page private chunks cut a long suffix into one partial per page:
    > 32 partials (the merge's multi-round fast path) and > 128 (its
    one-slot-at-a-time fallback) per (row, head)."""
    eng = make_engine(cuda_device, H=2)
    eng.set_option(_lib.FK_OPT_PRIV_MIN_CHUNK, 1)
    fork_group(eng, 100, [suffix, 5], out_len=2)
    run_steps(eng, 2)
    assert eng.last_plan.max_slots > (128 if suffix > 2048 else 32)
    check_history(eng)


@pytest.mark.parametrize("ctas", [1, 3])
def test_prefix_chunk_queue_wraps(cuda_device, ctas):
    """Few tcgen05 CTAs over many items: each CTA streams 20+ chunks, so the
    producer's chunk queue (16 entries) wraps several times, chunks of
    several heads and both query-block layouts (32- and 16-lane) interleave."""
    eng = make_engine(cuda_device, H=16, L=1)
    eng.set_option(_lib.FK_OPT_PREFIX_TARGET_CTAS, ctas)
    fork_group(eng, 700, [9] * 70, out_len=2, tag="a", seed=1)   # 70 rows: 32-lane layout
    fork_group(eng, 300, [4] * 20, out_len=2, tag="b", seed=2)   # 20 rows: 16-lane layout
    fork_group(eng, 140, [4] * 3, out_len=2, tag="c", seed=3)
    run_steps(eng, 2)
    check_history(eng)


@pytest.mark.parametrize("warps", [8, 12])
def test_private_ring_shapes(cuda_device, warps):
    """FK_OPT_PRIV_WARPS: the private CTA shapes besides the default 10 x 2
    (8 warps x 3 stages, 12 x 2) give the same attention."""
    eng = make_engine(cuda_device, H=4, L=2)
    eng.set_option(_lib.FK_OPT_PRIV_WARPS, warps)
    fork_group(eng, 400, [33, 100, 7, 260], out_len=3)
    run_steps(eng, 3)
    check_history(eng)


@pytest.mark.parametrize("cost", [0, 8])
def test_prefix_boundary_cost(cuda_device, cost):
    """FK_OPT_TC_BOUNDARY_COST 0 / 8: the cost-balanced static ranges cut
    items at different points (more or fewer pieces per head)."""
    eng = make_engine(cuda_device, H=8, L=2)
    eng.set_option(_lib.FK_OPT_TC_BOUNDARY_COST, cost)
    fork_group(eng, 3000, [40] * 50, out_len=2, tag="a", seed=4)
    fork_group(eng, 900, [5, 77, 130], out_len=2, tag="b", seed=5)
    run_steps(eng, 2)
    check_history(eng)


def test_model_style_layer_chain_with_pdl(cuda_device):
    """A model-style chain: layer l+1's queries are computed by a torch kernel
    from layer l's attention output, right before fk_attn_decode(l + 1).
    With the engine's cross-layer PDL (level 2) the outputs are bit-identical
    to plain stream order (level 0): the prefix kernel reads q only after
    griddepcontrol.wait."""
    import ctypes

    import torch

    L, H = 4, 8
    outs = {}
    for pdl in (0, 2):
        eng = make_engine(cuda_device, H=H, L=L)
        eng.set_option(_lib.FK_OPT_PDL, pdl)
        fork_group(eng, 900, [30, 64, 5, 100], out_len=2)
        from paper_2405_19888_b200.workloads import drain_fills
        drain_fills(eng)
        running = [g for g in eng.gens.values() if g.started and not g.done]
        eng._plan(running)
        rows = len(running)
        dev = torch.device("cuda", cuda_device)
        g = torch.Generator().manual_seed(3)
        q0 = torch.randn((rows, H, 128), generator=g).to(torch.bfloat16).to(dev)
        res = []
        with torch.cuda.stream(eng.stream):
            q = q0
            for layer in range(L):
                out = torch.empty_like(q)
                _lib.check(_lib.lib.fk_attn_decode(eng._pool.handle, layer, ctypes.c_void_p(q.data_ptr()),
                                                   ctypes.c_void_p(out.data_ptr()), None, eng._sp()))
                res.append(out)
                q = (out.float() * 8.0 + q.float()).to(torch.bfloat16)  # the "rest of the layer"
        eng.stream.synchronize()
        outs[pdl] = [r.cpu() for r in res]
        eng.close()
    for a, b in zip(outs[0], outs[2]):
        assert torch.equal(a, b)


def test_full_size_dedup_equals_unshared_streams(cuda_device):
    """Size-independent property at the full headline shape (13B heads, 6k
    prefix x 64 forks x 256, 2 layers): the shared-prefix decomposition
    (tcgen05 prefix + private + merge) and the unshared mode (every row
    streams its whole chain privately) compute the same attention."""
    outs = []
    for shared in (True, False):
        eng = make_engine(cuda_device, H=40, L=2, shared=shared)
        eng.keep_history = False
        fork_group(eng, 6000, [256] * 64, out_len=2)
        run_steps(eng, 2)
        outs.append(eng.last_output.float().cpu())
        eng.close()
    d = (outs[0] - outs[1]).abs()
    rel = d.norm() / outs[1].norm()
    assert d.max().item() <= 1e-2 and rel.item() <= 4e-3, (d.max().item(), rel.item())


def test_full_size_fork_permutation(cuda_device):
    """Reordering the forks of a group permutes the outputs and changes
    nothing else (headline shape, 1 layer, model K/V rows and queries given
    per fork; compared within the decomposition's own rounding noise)."""
    import torch

    H, n = 40, 64
    dev = torch.device("cuda", cuda_device)
    rng = random.Random(11)
    lens = [rng.randint(200, 300) for _ in range(n)]

    def rows(seed, ntok):
        g = torch.Generator().manual_seed(seed)
        return [torch.randn((1, ntok, H, 128), generator=g).to(torch.bfloat16).to(dev) for _ in range(2)]

    root_kv = rows(0, 6000)
    leaf_kv = [rows(1000 + i, lens[i]) for i in range(n)]
    g = torch.Generator().manual_seed(5)
    qbase = torch.randn((n, H, 128), generator=g).to(torch.bfloat16)

    def run(order):
        eng = make_engine(cuda_device, H=H, L=1)
        eng.keep_history = False
        eng.capture_f32 = False
        root = eng.new_context_id()
        eng.fill([1] * 6000, root, None, boundary_hash=1, kv=tuple(root_kv))
        for i in order:
            eng.fill([1] * lens[i], f"leaf{i}", root, boundary_hash=100 + i, kv=tuple(leaf_kv[i]))
            eng.generate(f"r{i}", f"leaf{i}", [1] * 2, "")
        from paper_2405_19888_b200.workloads import drain_fills
        drain_fills(eng)
        q = qbase[list(order)].unsqueeze(0).to(dev)
        eng.model = P.TensorDecodeModel(q, torch.zeros_like(q), torch.zeros_like(q))
        run_steps(eng, 1)
        rowpos = {rid: k for k, rid in enumerate(eng.last_rows)}
        out = eng.last_output[0].float().cpu()
        eng.close()
        return torch.stack([out[rowpos[f"r{i}"]] for i in range(n)])

    a = run(list(range(n)))
    b = run(list(reversed(range(n))))
    d = (a - b).abs()
    assert d.max().item() <= 1e-2 and (d.norm() / a.norm()).item() <= 4e-3, (d.max().item(),)


@pytest.mark.parametrize("shape", ["ragged", "nested", "shared_leaf", "oom"])
def test_attend_own_token_synthetic(cuda_device, shape):
    """attend_own_token (FK_OPT_APPEND_FIRST): each row's new K/V row is
    written before attention and is part of its span (a real decoder); the
    oracle attends over the chain including the step's own token."""
    if shape == "oom":
        eng = make_engine(cuda_device, H=4, L=2, kv_tokens=16 * 12, attend_own_token=True)
        eng.fill([1] * 16 * 10, "root", None)
        eng.fill([1] * 16, "a", "root")
        eng.fill([1] * 15, "b", "root")
        eng.generate("ra", "a", [1] * 3, "")
        eng.generate("rb", "b", [1] * 3, "")
        reps = [eng.step() for _ in range(3)]
        eng.stream.synchronize()
        assert any(r.failed for r in reps)
    else:
        eng = make_engine(cuda_device, H=8, L=2, attend_own_token=True)
        if shape == "ragged":
            fork_group(eng, 100, [0, 1, 15, 16, 17, 40], out_len=18, seed=3)
            run_steps(eng, 18)
        elif shape == "nested":
            nested_forest(eng, root_len=300, app_len=50, n_apps=2, user_len=33, users_per_app=3, out_len=4)
            run_steps(eng, 4)
        else:
            eng.fill([1] * 200, "root", None, boundary_hash=1)
            eng.fill([1] * 30, "leaf", "root", boundary_hash=2)
            eng.generate("a", "leaf", [1] * 4, "")
            eng.generate("b", "leaf", [1] * 4, "")
            run_steps(eng, 4)
    for rec in eng.history:
        # the span includes the step's new tokens; the reference count does not
        assert rec["streamed_tokens"] == rec["batch_tokens"] + sum(p >= 0 for p in rec["positions"])
    check_history(eng)


def test_attend_own_token_model_rows(cuda_device):
    """attend_own_token with model K/V rows: the output of a step includes
    the row the model produced for that very step (compared with the oracle
    over prefill rows + every appended model row so far)."""
    import torch

    from gpu_check import tensor_model_oracle
    from paper_2405_19888_b200.workloads import drain_fills

    H, L = 8, 3
    eng = make_engine(cuda_device, H=H, L=L, attend_own_token=True)
    fork_group(eng, 900, [30, 64, 5, 100, 0], out_len=4)
    drain_fills(eng)
    rows = len(eng.gens)
    n0 = {eng.contexts[g.context_id].uid: (eng.contexts[g.context_id].token_count, r)
          for r, g in enumerate(eng.gens.values())}
    g = torch.Generator().manual_seed(9)
    dev = torch.device("cuda", cuda_device)
    q, k, v = (torch.randn((L, rows, H, 128), generator=g).to(torch.bfloat16).to(dev) for _ in range(3))
    eng.model = P.TensorDecodeModel(q, k, v)
    run_steps(eng, 3)
    kv, queries = tensor_model_oracle(eng, n0)
    check_history(eng, kv=kv, queries=queries)
    # and it differs from the reference span (the own token matters)
    eng2 = make_engine(cuda_device, H=H, L=L)
    fork_group(eng2, 900, [30, 64, 5, 100, 0], out_len=4)
    drain_fills(eng2)
    eng2.model = P.TensorDecodeModel(q, k, v)
    run_steps(eng2, 1)
    assert not torch.equal(eng.history[0]["output"], eng2.history[0]["output"])
