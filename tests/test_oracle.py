"""The oracle is pinned before it is trusted: FNV against the reference's
known-answer vectors and reference-computed fixtures, the block twin against
the reference PagedKvStore, the numpy generator against the C restatement,
and the attention forms against each other."""

import ctypes
import json
import os
import random
import subprocess

import numpy as np
import pytest

from oracle import forkattn_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def oracle_c():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "build", "liboracle_c.so"))
    lib.oracle_fnv1a64_u32.restype = ctypes.c_uint64
    lib.oracle_fnv1a64_u32.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint64, ctypes.c_uint64]
    lib.oracle_synth_chunk.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_float,
                                       ctypes.POINTER(ctypes.c_uint16)]
    lib.oracle_ceil_blocks.restype = ctypes.c_int64
    lib.oracle_ceil_blocks.argtypes = [ctypes.c_int64, ctypes.c_int64]
    return lib


def test_fnv_reference_test_vectors():
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    # tests/test_tokenizer.py:20-35 standard vectors
    for hexdata, want in kat["expected_bytes"]:
        assert O.fnv1a64_bytes(bytes.fromhex(hexdata)) == int(want)
    for hexdata, want in kat["bytes"]:
        assert O.fnv1a64_bytes(bytes.fromhex(hexdata)) == int(want)
    for case in kat["ids"]:
        assert O.hash_token_ids(case["ids"], int(case["seed"])) == int(case["hash"])
    for case in kat["chains"]:
        assert O.chain_hashes(case["segments"]) == [int(h) for h in case["chain"]]


def test_c_restatement_matches_numpy(oracle_c):
    kat = json.load(open(os.path.join(GOLDEN, "kat.json")))
    for case in kat["ids"][:32]:
        ids = case["ids"]
        arr = (ctypes.c_uint32 * max(len(ids), 1))(*ids)
        assert oracle_c.oracle_fnv1a64_u32(arr, len(ids), int(case["seed"])) == int(case["hash"])
    for t in (0, 1, 15, 16, 17, 6000):
        assert oracle_c.oracle_ceil_blocks(t, 16) == -(-t // 16)
    rng = random.Random(5)
    out = (ctypes.c_uint16 * 4)()
    for _ in range(40):
        seed, tag = rng.randrange(1 << 64), rng.choice([1, 2, 3])
        uid, pos, layer, head = rng.randrange(1 << 20), rng.randrange(1 << 41), rng.randrange(80), rng.randrange(64)
        scale = rng.choice([1.0, 8.0])
        rows = O.synth_rows(seed, tag, uid, [pos], layer, head + 1, scale)[0, head]
        bits = rows.view(np.uint32) >> 16
        for j in (0, 7, 31):
            oracle_c.oracle_synth_chunk(seed, tag, uid, pos, layer, head, j, scale, out)
            assert list(out) == [int(b) for b in bits[4 * j:4 * j + 4]]


def test_bf16_rounding_is_rne():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5e-5, 3.0e38], dtype=np.float32)
    r = O.bf16_round(x)
    assert r[0] == 1.0 and r[1] == 1.0  # tie -> even
    assert r[2] == np.float32(1.0078125)
    assert np.isfinite(r).all()


def test_attention_forms_agree():
    rng = np.random.default_rng(3)
    B, H, Pn = 6, 4, 123
    q = O.bf16_round(rng.standard_normal((B, H, 128), dtype=np.float32))
    pk = O.bf16_round(rng.standard_normal((Pn, H, 128), dtype=np.float32))
    pv = O.bf16_round(rng.standard_normal((Pn, H, 128), dtype=np.float32))
    sk = [O.bf16_round(rng.standard_normal((s, H, 128), dtype=np.float32)) for s in (0, 1, 5, 16, 17, 40)]
    sv = [O.bf16_round(rng.standard_normal((s, H, 128), dtype=np.float32)) for s in (0, 1, 5, 16, 17, 40)]
    got = O.attend_shared_batch(q, pk, pv, sk, sv)
    for b in range(B):
        want = O.attend(q[b], np.concatenate([pk, sk[b]]), np.concatenate([pv, sv[b]]))
        assert np.abs(got[b] - want).max() < 1e-5


def test_attend_rows_decomposition_identity():
    """Splitting a chain into contexts does not change the oracle output."""
    kv = O.KVCache(0x5EED, 2)
    q = O.row_queries(0x5EED, [7, 7, 9], [10, 10, 3], 0, 2)
    chains = [[(1, 40), (7, 10)], [(1, 40), (7, 10)], [(1, 40), (2, 16), (9, 3)]]
    out = O.attend_rows(chains, q, kv, 0)
    k1, v1 = kv.get(1, 40, 0)
    k2, v2 = kv.get(2, 16, 0)
    k9, v9 = kv.get(9, 3, 0)
    want = O.attend(q[2], np.concatenate([k1, k2, k9]), np.concatenate([v1, v2, v9]))
    assert np.allclose(out[2], want)
    assert not np.allclose(q[0], q[1])  # rank keys distinct queries on one leaf


@pytest.mark.reference
def test_block_twin_matches_reference_store():
    from semflow.engine import Context, PagedKvStore
    from semflow.errors import OutOfMemory

    rng = random.Random(11)
    for trial in range(30):
        total = rng.choice([5, 20, 80])
        ref = PagedKvStore(16, total)
        twin = O.BlockTwin(16, total)
        ctxs = {}
        for i in range(60):
            if ctxs and rng.random() < 0.2:
                cid = rng.choice(list(ctxs))
                ref.release(ctxs.pop(cid))
                twin.release(cid)
                continue
            cid = rng.choice(list(ctxs)) if ctxs and rng.random() < 0.5 else f"c{i}"
            if cid not in ctxs:
                ctxs[cid] = Context(cid, "e0", None)
                twin.create(cid, None)
            n = ctxs[cid].token_count + rng.randint(0, 50)
            try:
                ref.grow(ctxs[cid], n)
                ok = True
            except OutOfMemory:
                ok = False
            assert twin.grow(cid, n) == ok
            assert twin.blocks[cid] == ctxs[cid].block_ids
            assert (twin.used, twin.peak) == (ref.used_blocks, ref.peak_used)


def test_attend_matches_torch_sdpa_fp64():
    """The attention oracle is plain softmax(q k^T / sqrt(D)) v: an
    independent implementation (torch.nn.functional.scaled_dot_product_attention
    on the CPU, fp64) gives the same rows, including a peaky (K x 8) case and
    one-token / page-boundary lengths."""
    import torch

    rng = np.random.default_rng(11)
    for T, kscale in ((1, 1.0), (16, 1.0), (17, 8.0), (300, 1.0), (300, 8.0)):
        q = O.bf16_round(rng.standard_normal((4, 128), dtype=np.float32))
        k = O.bf16_round(rng.standard_normal((T, 4, 128), dtype=np.float32) * kscale)
        v = O.bf16_round(rng.standard_normal((T, 4, 128), dtype=np.float32))
        got = O.attend(q, k, v)
        tq = torch.from_numpy(q.astype(np.float64))[:, None, :]           # [H, 1, D]
        tk = torch.from_numpy(k.astype(np.float64)).permute(1, 0, 2)      # [H, T, D]
        tv = torch.from_numpy(v.astype(np.float64)).permute(1, 0, 2)
        want = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv)[:, 0, :].numpy()
        assert np.abs(got - want).max() < 1e-12, (T, kscale)


def test_bulk_c_rows_match_numpy_generator():
    """oracle_synth_rows (C, used for full-size checks) == synth_rows (numpy)."""
    for seed, tag, uid, pos0, n, layer, heads, scale in ((1, 1, 0, 0, 33, 0, 3, 1.0),
                                                         (0x5EED, 2, 77, 6000, 17, 39, 40, 1.0),
                                                         (12345, 1, 5, 1 << 41, 4, 7, 2, 8.0)):
        want = O.synth_rows(seed, tag, uid, np.arange(pos0, pos0 + n), layer, heads, scale)
        got = O.synth_rows_range(seed, tag, uid, pos0, n, layer, heads, scale)
        assert np.array_equal(want, got)


def test_forest_form_equals_per_row_form():
    """attend_forest (context-batched products, one softmax per whole row)
    == attend_rows (per-row concatenated chain) on nested, ragged, empty and
    shared-leaf forests, with model-appended rows."""
    rng = np.random.default_rng(2)
    app = {3: (10, lambda layer, kv, pos: np.full((len(pos), 4, 128), 0.25 * (kv + 1) + layer, np.float32)),
           5: (0, lambda layer, kv, pos: rng.standard_normal((len(pos), 4, 128)).astype(np.float32))}
    for k_scale in (1.0, 8.0):
        kv = O.KVCache(11, 4, k_scale, appended=app)
        chains = [[(0, 300), (1, 33)], [(0, 300), (2, 0)], [(0, 300), (3, 17), (4, 5)],
                  [(0, 300), (3, 17), (5, 40)], [(6, 0)], [(7, 64)], [(0, 300), (1, 33)]]
        q = O.bf16_round(rng.standard_normal((len(chains), 4, 128), dtype=np.float32))
        for layer in (0, 2):
            a = O.attend_rows(chains, q, kv, layer)
            b = O.attend_forest(chains, q, kv, layer)
            assert np.abs(a - b).max() < 1e-12
            assert np.abs(b[4]).max() == 0.0  # empty chain -> zeros
