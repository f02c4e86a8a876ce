"""World-size-2 (gloo, CPU) coverage of the multi-GPU partition: each rank
owns whole prefix-affinity groups, runs its own engine, and only the timing
reduction crosses ranks."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2405_19888_b200 as P
    from paper_2405_19888_b200 import cluster
    from paper_2405_19888_b200.workloads import fork_group

    groups = cluster.rank_groups(rank, 4, world)
    eng = P.GpuEngine(f"e{rank}", P.CostModel(), kv_tokens=1 << 20)
    for g in groups:
        fork_group(eng, 2000, [128 + 16 * g] * 32, out_len=3, tag=f"g{g}", seed=g)
    tokens = 0
    steps = 0
    while eng.has_work() and steps < 50:
        rep = eng.step()
        tokens += len(rep.emitted)
        steps += 1
    total = cluster.sum_over_ranks(tokens)
    slowest = cluster.max_over_ranks(float(steps + rank))
    q.put((rank, groups, tokens, total, slowest, eng.store.peak_used))
    dist.destroy_process_group()


def test_two_rank_group_partition():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, g0, t0, tot0, s0, pk0), (r1, g1, t1, tot1, s1, pk1) = res
    assert g0 == [0, 2] and g1 == [1, 3]  # whole groups, disjoint
    assert tot0 == tot1 == t0 + t1 == 4 * 32 * 3  # every fork emitted its 3 tokens
    assert s0 == s1 == max(s0, s1)
    # each rank stores its own prefixes once (no replication of others' groups)
    assert pk0 == 2 * 125 + sum(32 * -(-(128 + 16 * g + 3) // 16) for g in g0)
