"""Fork-group builders over the engine API (the shapes of BASELINE.json).

These call only the reference surface (fill / create_context / generate),
the way the manager's `_place_one` does (manager.py:465-511), so the forest,
block ids and chain hashes are the ones the reference would produce.
Token ids are synthetic; KV content comes from the engine's fill path.
"""

from __future__ import annotations

import random
from typing import List, Optional, Sequence

from .engine import FNV64_EMPTY, hash_token_ids


def _tokens(rng: random.Random, n: int) -> List[int]:
    return [rng.randrange(1 << 32) for _ in range(n)]


def fork_group(eng, prefix_len: int, suffix_lens: Sequence[int], out_len: int, tag: str = "g0",
               seed: int = 0, parent: Optional[str] = None, parent_hash: int = FNV64_EMPTY) -> List[str]:
    """One shared prefix context + one leaf per request; returns request ids
    in generate() order (= the gens order the decode batch follows)."""
    rng = random.Random(seed)
    root = eng.new_context_id()
    toks = _tokens(rng, prefix_len)
    h_root = hash_token_ids(toks, parent_hash)
    eng.fill(toks, root, parent, boundary_hash=h_root)
    rids = []
    for i, s in enumerate(suffix_lens):
        leaf = eng.new_context_id()
        stoks = _tokens(rng, s)
        eng.fill(stoks, leaf, root, boundary_hash=hash_token_ids(stoks, h_root))
        rid = f"{tag}.r{i}"
        eng.generate(rid, leaf, _tokens(rng, out_len), "")
        rids.append(rid)
    return rids


def nested_forest(eng, root_len: int, app_len: int, n_apps: int, user_len: int, users_per_app: int,
                  out_len: int, tag: str = "n", seed: int = 0) -> List[str]:
    """System prompt -> per-app prompt -> per-user suffix (BASELINE config 5)."""
    rng = random.Random(seed)
    root = eng.new_context_id()
    rt = _tokens(rng, root_len)
    h0 = hash_token_ids(rt)
    eng.fill(rt, root, None, boundary_hash=h0)
    rids = []
    for a in range(n_apps):
        app = eng.new_context_id()
        at = _tokens(rng, app_len)
        h1 = hash_token_ids(at, h0)
        eng.fill(at, app, root, boundary_hash=h1)
        for u in range(users_per_app):
            leaf = eng.new_context_id()
            ut = _tokens(rng, user_len)
            eng.fill(ut, leaf, app, boundary_hash=hash_token_ids(ut, h1))
            rid = f"{tag}.a{a}.u{u}"
            eng.generate(rid, leaf, _tokens(rng, out_len), "")
            rids.append(rid)
    return rids


def drain_fills(eng) -> None:
    """Retire queued fill chunks (cost-model bookkeeping only: the KV was
    written at fill time) without running a decode step."""
    while eng.fill_queue:
        task = eng.fill_queue.popleft()
        if task.request_id is not None:
            eng.pending_fills[task.request_id] = eng.pending_fills.get(task.request_id, 0) - 1
