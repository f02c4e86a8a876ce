"""Shared GPU-vs-oracle comparison for the parity tests and smoke().

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


def oracle_step(eng, rec, layer, kv):
    chains = rec["chains"]
    leaf_uids = [c[-1][0] for c in chains]
    leaf_pos = [c[-1][1] for c in chains]
    q = O.row_queries(eng.model_seed, leaf_uids, leaf_pos, layer, eng.geometry.num_heads)
    return O.attend_rows(chains, q, kv, layer)


def check_history(eng, steps=None, f32=True):
    """Compare every recorded step (or the listed ones) against the oracle;
    returns the worst error report."""
    kv = O.KVCache(eng.model_seed, eng.geometry.num_heads, eng.model_k_scale)
    worst = {"max_abs": 0.0, "rel_l2": 0.0, "mean_rel_f32": 0.0}
    recs = eng.history if steps is None else [eng.history[i] for i in steps]
    assert recs, "no decode step recorded"
    for rec in recs:
        out = to_np(rec["output"])
        out32 = to_np(rec["output_f32"]) if rec.get("output_f32") is not None else None
        for layer in range(eng.geometry.num_layers):
            want = oracle_step(eng, rec, layer, kv)
            r = O.tolerance_report(out[layer], want)
            assert np.isfinite(out[layer]).all()
            assert r["max_abs"] <= MAX_ABS and r["rel_l2"] <= REL_L2, (layer, r)
            worst["max_abs"] = max(worst["max_abs"], r["max_abs"])
            worst["rel_l2"] = max(worst["rel_l2"], r["rel_l2"])
            if f32 and out32 is not None:
                r32 = O.tolerance_report(out32[layer], want)
                assert r32["mean_rel"] <= MEAN_REL_F32, (layer, r32)
                worst["mean_rel_f32"] = max(worst["mean_rel_f32"], r32["mean_rel"])
    return worst
