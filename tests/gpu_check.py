"""Shared GPU-vs-oracle comparison for the parity tests, smoke() and
bench.py --check.

Tolerances:
  bf16 output vs the fp64-accumulated oracle: max-abs <= 2e-2 AND rel-L2 <= 4e-3
  fp32 pre-cast merge output (capture_f32):   mean-rel <= 1e-3
"""

from __future__ import annotations

import numpy as np

from oracle import forkattn_oracle as O

MAX_ABS = 2e-2
REL_L2 = 4e-3
MEAN_REL_F32 = 1e-3


def to_np(t):
    import torch

    return t.detach().to("cpu", torch.float32).numpy()


def synthetic_queries(eng, rec, layer):
    """Q rows of the synthetic model, keyed by (leaf uid, leaf tokens before
    the step's growth): the chains' leaf count, or rec["qpos"] when the span
    already includes the step's own token (attend_own_token)."""
    chains = rec["chains"]
    qpos = rec.get("qpos") or [c[-1][1] for c in chains]
    return O.row_queries(eng.model_seed, [c[-1][0] for c in chains], qpos, layer, eng.geometry.num_heads)


def tensor_model_oracle(eng, leaf_n0):
    """KV cache + queries of a TensorDecodeModel engine (bench.py's model):
    every context holds the synthetic prefill rows, except that positions >=
    n0 of a leaf hold the model K/V row of its request (the same row every
    step); queries are the model's q rows.  leaf_n0: {leaf uid: (n0, row)}
    captured when the model was attached."""
    model = eng.model
    qh = to_np(model.q)
    kh, vh = to_np(model.k), to_np(model.v)
    H = eng.geometry.num_heads

    def rows_of(row):
        def rows(layer, kv, pos):
            src = kh if kv == 0 else vh
            return np.broadcast_to(src[layer, row], (len(pos), H, 128))
        return rows

    app = {uid: (n0, rows_of(row)) for uid, (n0, row) in leaf_n0.items()}
    kv = O.KVCache(eng.model_seed, H, eng.model_k_scale, appended=app)
    return kv, (lambda rec, layer: qh[layer, :len(rec["rows"])])


def check_history(eng, steps=None, f32=True, layers=None, kv=None, queries=None, strict=True):
    """Compare every recorded step (or the listed ones) and layer (or the
    listed ones) against the oracle; returns the worst error report (and
    asserts the tolerances unless strict=False)."""
    if kv is None:
        kv = O.KVCache(eng.model_seed, eng.geometry.num_heads, eng.model_k_scale)
    if queries is None:
        queries = lambda rec, layer: synthetic_queries(eng, rec, layer)  # noqa: E731
    worst = {"max_abs": 0.0, "rel_l2": 0.0, "mean_rel_f32": 0.0}
    recs = eng.history if steps is None else [eng.history[i] for i in steps]
    assert recs, "no decode step recorded"
    for rec in recs:
        out = to_np(rec["output"])
        out32 = to_np(rec["output_f32"]) if rec.get("output_f32") is not None else None
        for layer in (range(eng.geometry.num_layers) if layers is None else layers):
            want = O.attend_forest(rec["chains"], queries(rec, layer), kv, layer)
            r = O.tolerance_report(out[layer], want)
            finite = bool(np.isfinite(out[layer]).all())
            worst["finite"] = worst.get("finite", True) and finite
            assert finite or not strict
            assert not strict or (r["max_abs"] <= MAX_ABS and r["rel_l2"] <= REL_L2), (layer, r)
            worst["max_abs"] = max(worst["max_abs"], r["max_abs"])
            worst["rel_l2"] = max(worst["rel_l2"], r["rel_l2"])
            if f32 and out32 is not None:
                r32 = O.tolerance_report(out32[layer], want)
                assert not strict or r32["mean_rel"] <= MEAN_REL_F32, (layer, r32)
                worst["mean_rel_f32"] = max(worst["mean_rel_f32"], r32["mean_rel"])
    worst["pass"] = bool(worst.get("finite", True) and worst["max_abs"] <= MAX_ABS and worst["rel_l2"] <= REL_L2
                         and worst["mean_rel_f32"] <= MEAN_REL_F32)
    return worst
