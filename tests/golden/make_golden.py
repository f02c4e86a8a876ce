"""Generate the golden fixtures of tests/golden from the REFERENCE package.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Outputs (committed):
    kat.json             FNV-1a known answers (reference test vectors +
                         reference-computed hash_token_ids / chains)
    engine_streams.json  op streams recorded on semflow.engine.Engine
    plans.json           per-step batch_tokens of manager-driven workloads
"""

from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("FK_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, HERE)

from semflow.config import Config  # noqa: E402
from semflow.engine import CostModel, Engine  # noqa: E402
from semflow.experiments import run_workload_manager  # noqa: E402
from semflow.tokenizer import FNV64_EMPTY, fnv1a64, hash_token_ids  # noqa: E402
from semflow.workloads import mapreduce_summary, shared_prompt_serving  # noqa: E402

import streams  # noqa: E402

N_STREAMS = 24
OPS_PER_STREAM = 90


def kat():
    rng = random.Random(2405)
    ids_cases = []
    for _ in range(64):
        ids = [rng.randrange(1 << 32) for _ in range(rng.randint(0, 40))]
        seed = rng.choice([FNV64_EMPTY, rng.randrange(1 << 64)])
        ids_cases.append({"ids": ids, "seed": str(seed), "hash": str(hash_token_ids(ids, seed))})
    chains = []
    for _ in range(16):
        segs = [[rng.randrange(1 << 32) for _ in range(rng.randint(0, 30))] for _ in range(rng.randint(1, 5))]
        h = FNV64_EMPTY
        out = []
        for s in segs:
            h = hash_token_ids(s, h)
            out.append(str(h))
        chains.append({"segments": segs, "chain": out})
    return {
        # tests/test_tokenizer.py:20-35 (standard FNV-1a-64 vectors)
        "bytes": [[d.hex(), str(fnv1a64(d))] for d in (b"", b"a", b"foobar")],
        "expected_bytes": [["", str(0xCBF29CE484222325)], ["61", str(0xAF63DC4C8601EC8C)],
                           ["666f6f626172", str(0x85944171F73967E8)]],
        "ids": ids_cases,
        "chains": chains,
        "empty": str(FNV64_EMPTY),
    }


def engine_streams():
    out = []
    for i in range(N_STREAMS):
        spec = streams.make_ops(9000 + i, OPS_PER_STREAM)
        rec = streams.record_stream(
            lambda kv, sk: Engine("e0", CostModel(shared_kernel=sk), kv_tokens=kv), spec)
        out.append({"spec": spec, "record": rec})
    return out


def plans():
    cases = {
        "shared_prompt_small": (shared_prompt_serving(1, users=12, system_prompt_len=600, unique_len=40,
                                                      output_len=30), Config(total_blocks=4000)),
        "mapreduce_small": (mapreduce_summary(2, maps=4, chunk_size=300, output_len=20),
                            Config(total_blocks=4000)),
        "shared_prompt_2eng": (shared_prompt_serving(3, users=8, system_prompt_len=300, unique_len=20,
                                                     output_len=16), Config(engines=2, total_blocks=4000)),
    }
    res = {}
    for name, (wl, cfg) in cases.items():
        mgr, _, end_ns = run_workload_manager(wl, "semflow", cfg)
        res[name] = {
            "end_ns": end_ns,
            "engines": {eid: {"reports": [streams.report_tuple(r) for r in e.reports],
                              "trace": list(e.trace), "peak": e.store.peak_used}
                        for eid, e in sorted(mgr.engines.items())},
        }
    return res


def main():
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat(), f)
    with open(os.path.join(HERE, "engine_streams.json"), "w") as f:
        json.dump(engine_streams(), f)
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(plans(), f)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
