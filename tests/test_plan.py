"""Work-list planner (fk_step_plan) on host-only pools: the work-list
invariant sum(tokens of prefix items and private streams) == the reference
dedup count _batch_tokens (engine.py:470-484), in both shared_kernel modes,
over random forests; the oracle twin agrees."""

import random

import pytest

import paper_2405_19888_b200 as P
from oracle import forkattn_oracle as O


def random_forest(seed, shared=True):
    rng = random.Random(seed)
    eng = P.GpuEngine("e0", P.CostModel(shared_kernel=shared), kv_tokens=1 << 22)
    twin = O.BlockTwin(16, -(-(1 << 22) // 16))
    ids = []
    for i in range(rng.randint(1, 40)):
        parent = rng.choice(ids) if ids and rng.random() < 0.7 else None
        cid = f"c{i}"
        n = rng.choice([0, 1, 15, 16, 17, rng.randint(0, 600)])
        eng.fill([1] * n, cid, parent)
        twin.create(cid, parent)
        assert twin.grow(cid, n)
        ids.append(cid)
    leaves = []
    for j in range(rng.randint(1, 30)):
        leaf = rng.choice(ids)
        eng.generate(f"r{j}", leaf, [1] * 3, "")
        leaves.append(leaf)
    return eng, twin, leaves


@pytest.mark.parametrize("shared,group", [(True, 0), (False, 0), (True, 8), (True, 16)])
def test_plan_batch_tokens_matches_walk_and_twin(shared, group):
    """(group > 0: small-fan-out shared contexts go to the private kernel as
    row groups -- FK_OPT_GROUP_FANOUT -- and still count once)"""
    for seed in range(60):
        eng, twin, leaves = random_forest(seed, shared)
        eng.set_option(P._lib.FK_OPT_GROUP_FANOUT, group)
        running = [g for g in eng.gens.values() if g.started and not g.done]
        bt = eng._plan(running)
        info = eng.last_plan
        assert bt == eng._batch_tokens(running) == twin.batch_tokens(leaves, shared)
        assert info.num_rows == len(running)
        if shared:
            assert info.shared_tokens + info.private_tokens == bt
        else:
            assert info.num_shared_ctx == 0 and info.private_tokens == bt
        assert info.max_slots >= 1


def test_block_ids_match_twin():
    eng, twin, _ = random_forest(7)
    for cid in twin.blocks:
        assert eng.contexts[cid].block_ids == twin.blocks[cid]
    st = eng.pool_stats()
    assert st.used_blocks == twin.used and st.peak_used == twin.peak


def test_headline_plan_shape():
    """LLaMA-13B headline: one 6000-token prefix shared by 64 forks of 256."""
    eng = P.GpuEngine("e0", P.CostModel(), kv_tokens=1 << 22, geometry=P.LLAMA_13B)
    from paper_2405_19888_b200.workloads import fork_group

    fork_group(eng, 6000, [256] * 64, out_len=2)
    running = list(eng.gens.values())
    assert eng._plan(running) == 6000 + 64 * 256 == 22384
    info = eng.last_plan
    assert info.num_shared_ctx == 1 and info.shared_tokens == 6000 and info.private_tokens == 64 * 256
    # prefix split into about one wave of CTAs
    assert 40 <= info.num_prefix_ctas <= 2 * 148


def test_nested_plan_counts_every_level_once():
    eng = P.GpuEngine("e0", P.CostModel(), kv_tokens=1 << 22)
    from paper_2405_19888_b200.workloads import nested_forest

    nested_forest(eng, 4096, 1024, 8, 256, 8, out_len=2)
    running = list(eng.gens.values())
    assert eng._plan(running) == 4096 + 8 * 1024 + 64 * 256
    assert eng.last_plan.num_shared_ctx == 9


def test_plan_digests_pinned():
    """Every array and scalar the planner uploads, for 682 (forest, options,
    dedup) cases x 3 steps, equals the pinned digests
    (tests/golden/make_plan_digests.py): 558 were written by the round-1
    planner, so the host-speed rewrite of fk_step_plan changed no plan; the
    124 FK_OPT_GROUP_FANOUT cases pin the grouped planner."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "golden", "make_plan_digests.py"), "--check"],
                       env={**os.environ, "FK_DEBUG_PLAN_DIGEST": "1"}, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_auto_min_chunk():
    """Small plans without a prefix grid: the automatic minimum private chunk
    is the one the last-round rule predicts (tests/plan_min_chunk_check.py
    restates it and compares plan digests against the explicit option)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "plan_min_chunk_check.py")],
                       env={**os.environ, "FK_DEBUG_PLAN_DIGEST": "1"}, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
