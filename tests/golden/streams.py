"""Randomised engine op streams with recorded outcomes.

`record_stream` drives an engine with the reference's surface through a
seeded op mix modelled on the reference's block-conservation property suite
(/root/reference/pkg/tests/oracles.py:556-608) and records, after every op,
the outcome plus a digest of the full observable state (contexts, blocks,
refcounts, hashes, registry, store counters, step reports, trace).
`make_golden.py` runs it on the REFERENCE Engine and commits the result;
tests replay the same ops on GpuEngine and require identical records.
"""

from __future__ import annotations

import hashlib
import json
import random
from typing import Any, Callable, Dict, List


def engine_state(eng) -> Dict[str, Any]:
    ctxs = {}
    for cid, c in sorted(eng.contexts.items()):
        ctxs[cid] = [c.parent_id, c.token_count, list(c.block_ids), c.refcount, c.dropped,
                     [str(h) for h in c.chain_hashes], [str(h) for h in c.registered_hashes]]
    gens = {rid: [g.context_id, g.emitted, g.started, g.done, len(g.token_ids)] for rid, g in sorted(eng.gens.items())}
    return {
        "contexts": ctxs,
        "gens": gens,
        "registry": {str(h): c for h, c in sorted(eng.registry.items())},
        "store": [eng.store.used_blocks, eng.store.free_blocks, eng.store.peak_used, eng.store.total_blocks],
        "owner": {str(b): c for b, c in sorted(eng.store.owner.items())},
        "pending": {k: v for k, v in sorted(eng.pending_fills.items())},
        "fill_queue": [[t.request_id, t.context_id, len(t.token_ids)] for t in eng.fill_queue],
        "clock": [eng.clock_ns, eng.busy_ns, eng.fill_ns_total, eng.decode_ns_total, eng.total_emitted],
        "trace_len": len(eng.trace),
        "request_leaf": dict(sorted(eng.request_leaf.items())),
    }


def digest(obj: Any) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()[:16]


def report_tuple(r) -> List[Any]:
    if r is None:
        return None
    return [r.started_ns, r.elapsed_ns, r.fill_tokens, r.batch_tokens, sorted(r.emitted.items()),
            list(r.finished), [list(f) for f in r.failed], list(r.fill_completed)]


def make_ops(seed: int, n_ops: int) -> Dict[str, Any]:
    """A seeded op list, generated without looking at any engine: ids and
    choices only reference names; invalid picks exercise the error paths."""
    rng = random.Random(seed)
    ops: List[Dict[str, Any]] = []
    ctx_names: List[str] = []
    req_names: List[str] = []
    for i in range(n_ops):
        roll = rng.random()
        if roll < 0.34 or not ctx_names:
            cid = f"k{i}"
            parent = rng.choice(ctx_names) if ctx_names and rng.random() < 0.65 else None
            if ctx_names and rng.random() < 0.15:  # extend an existing context
                cid, parent = rng.choice(ctx_names), None
            rid = f"r{i}" if rng.random() < 0.3 else None
            ops.append({"op": "fill", "ctx": cid, "parent": parent, "n": rng.randint(0, 70), "rid": rid,
                        "bh": rng.randrange(1 << 40) if rng.random() < 0.8 else None,
                        "tok": rng.randrange(1 << 32)})
            if cid not in ctx_names:
                ctx_names.append(cid)
            if rid:
                req_names.append(rid)
        elif roll < 0.40:
            ops.append({"op": "create", "ctx": f"k{i}", "parent": rng.choice(ctx_names)})
            ctx_names.append(f"k{i}")
        elif roll < 0.52:
            rid = rng.choice(req_names) if req_names and rng.random() < 0.4 else f"g{i}"
            ops.append({"op": "generate", "rid": rid, "ctx": rng.choice(ctx_names),
                        "toks": [rng.randrange(1 << 32) for _ in range(rng.randint(0, 6))]})
            req_names.append(rid)
        elif roll < 0.76:
            ops.append({"op": "step"})
        elif roll < 0.84:
            ops.append({"op": "finish", "rid": rng.choice(req_names) if req_names else "none"})
        elif roll < 0.90:
            ops.append({"op": "free", "ctx": rng.choice(ctx_names)})
        elif roll < 0.96:
            ops.append({"op": "drop", "ctx": rng.choice(ctx_names)})
        else:
            ops.append({"op": "cancel", "rid": rng.choice(req_names) if req_names else "none"})
    return {"seed": seed, "kv_tokens": 16 * rng.choice([12, 24, 48, 96]), "shared_kernel": rng.random() < 0.8,
            "ops": ops}


def apply_op(eng, op: Dict[str, Any]) -> Any:
    kind = op["op"]
    if kind == "fill":
        return eng.fill([op["tok"]] * op["n"], op["ctx"], op["parent"], request_id=op["rid"],
                        boundary_hash=op["bh"])
    if kind == "create":
        eng.create_context(op["ctx"], op["parent"])
        return None
    if kind == "generate":
        t = eng.generate(op["rid"], op["ctx"], op["toks"], "v")
        return [t.started]
    if kind == "step":
        return report_tuple(eng.step())
    if kind == "finish":
        h = eng.finish_generation(op["rid"])
        return None if h is None else str(h)
    if kind == "free":
        eng.free_context(op["ctx"])
        return None
    if kind == "drop":
        eng.mark_dropped(op["ctx"])
        return None
    if kind == "cancel":
        eng.cancel_request(op["rid"])
        return None
    raise ValueError(kind)


def record_stream(make_engine: Callable[[int, bool], Any], spec: Dict[str, Any]) -> List[Any]:
    eng = make_engine(spec["kv_tokens"], spec["shared_kernel"])
    out = []
    for op in spec["ops"]:
        try:
            res = ["ok", apply_op(eng, op)]
        except Exception as exc:  # error class names are part of the contract
            res = ["err", type(exc).__name__, str(exc)]
        out.append([res, digest(engine_state(eng))])
    out.append(["final", engine_state(eng), list(eng.trace)])
    return out
