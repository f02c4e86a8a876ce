"""CPU oracle for the shared-prefix decode path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker or the timed CPU
baseline; the product path (paper_2405_19888_b200) never routes through it.

What it restates (each function cites the reference it follows):

* FNV-1a-64 chained over little-endian u32 token ids
  (semflow/tokenizer.py:36-49) — pinned against the reference's own known
  answer vectors (tests/test_tokenizer.py:20-35) in tests/golden.
* Block accounting + the shared-kernel dedup count (semflow/engine.py:66-106,
  470-484) as `BlockTwin` — pinned against op streams run through the
  reference Engine (tests/golden/engine_streams.json, made by
  tests/golden/make_golden.py).
* The synthetic K/V/Q generator of the device path (fk_common.cuh
  synth_key/synth_chunk), restated independently in numpy.
* Attention: the reference has NO attention math (SPEC.md:8 models the
  kernel as a cost flag), so the numerics are "parity unpinned" by reference
  tests.  `attend_rows` computes plain, un-decomposed softmax attention over
  each request's concatenated chain (engine.py:53-63 segments, span = chain
  tokens at step start, engine.py:416-434), which checks the device path's
  prefix/suffix/merge decomposition independently.
"""

from __future__ import annotations

import math
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

FNV64_BASIS = 0xCBF29CE484222325
FNV64_PRIME = 0x00000100000001B3
MASK64 = (1 << 64) - 1


# --------------------------------------------------------------- hashing
def fnv1a64_bytes(data: bytes, seed: int = FNV64_BASIS) -> int:
    """tokenizer.fnv1a64 (tokenizer.py:36-41)."""
    h = seed
    for b in data:
        h = ((h ^ b) * FNV64_PRIME) & MASK64
    return h


def hash_token_ids(ids: Iterable[int], seed: int = FNV64_BASIS) -> int:
    """tokenizer.hash_token_ids (tokenizer.py:47-49): LE u32 bytes, chained."""
    h = seed
    for t in ids:
        h = fnv1a64_bytes(int(t).to_bytes(4, "little"), h)
    return h


def chain_hashes(segments: Sequence[Sequence[int]], seed: int = FNV64_BASIS) -> List[int]:
    """Boundary chain of render_prefix (prefix.py:78-85)."""
    out = []
    h = seed
    for seg in segments:
        h = hash_token_ids(seg, h)
        out.append(h)
    return out


# ------------------------------------------------------ block accounting
class BlockTwin:
    """Restatement of PagedKvStore + the forest walk of _batch_tokens.

    engine.py:84-85 ceil packing; :87-100 atomic grow with ids from a
    monotonic counter (:74); :102-106 release; :470-484 dedup count.
    """

    def __init__(self, block_size: int, total_blocks: int):
        self.block_size = block_size
        self.total_blocks = total_blocks
        self.next_id = 0
        self.used = 0
        self.peak = 0
        self.parent: Dict[str, Optional[str]] = {}
        self.tokens: Dict[str, int] = {}
        self.blocks: Dict[str, List[int]] = {}

    def create(self, cid: str, parent: Optional[str]) -> None:
        self.parent[cid] = parent
        self.tokens[cid] = 0
        self.blocks[cid] = []

    def grow(self, cid: str, new_tokens: int) -> bool:
        need = -(-new_tokens // self.block_size) - len(self.blocks[cid])
        if need > self.total_blocks - self.used:
            return False
        for _ in range(max(need, 0)):
            self.blocks[cid].append(self.next_id)
            self.next_id += 1
        self.used += max(need, 0)
        self.tokens[cid] = new_tokens
        self.peak = max(self.peak, self.used)
        return True

    def release(self, cid: str) -> None:
        self.used -= len(self.blocks.pop(cid))
        del self.tokens[cid]
        del self.parent[cid]

    def chain(self, leaf: str) -> List[str]:
        out = []
        cur: Optional[str] = leaf
        while cur is not None and cur in self.parent:
            out.append(cur)
            cur = self.parent[cur]
        return out

    def batch_tokens(self, leaves: Sequence[str], shared_kernel: bool = True) -> int:
        if shared_kernel:
            seen = set()
            for leaf in leaves:
                seen.update(self.chain(leaf))
            return sum(self.tokens[c] for c in seen)
        return sum(self.tokens[c] for leaf in leaves for c in self.chain(leaf))


# ------------------------------------------------- synthetic generator
TAG_K, TAG_V, TAG_Q = 1, 2, 3
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(x: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer on uint64 arrays (wrapping arithmetic)."""
    x = x ^ (x >> np.uint64(30))
    x = x * _M1
    x = x ^ (x >> np.uint64(27))
    x = x * _M2
    x = x ^ (x >> np.uint64(31))
    return x


def _u64(v) -> np.ndarray:
    return np.asarray(np.asarray(v, dtype=np.int64), dtype=np.uint64) if np.ndim(v) else np.uint64(int(v) & MASK64)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 (round to nearest even) -> float32."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def synth_rows(seed: int, tag: int, uid, pos, layer: int, heads: int, scale: float = 1.0) -> np.ndarray:
    """Rows of the counter-hash generator: returns [n, heads, 128] float32
    holding bf16 values, for n = len(pos) token keys (uid broadcast)."""
    with np.errstate(over="ignore"):
        pos = np.atleast_1d(np.asarray(pos, dtype=np.int64)).astype(np.uint64)
        uid = np.broadcast_to(np.asarray(uid, dtype=np.int64), pos.shape).astype(np.uint64)
        k = _mix(np.full(pos.shape, (int(seed) ^ (tag << 56)) & MASK64, dtype=np.uint64))
        k = _mix(k ^ uid)
        k = _mix(k ^ pos)
        k = _mix(k ^ np.uint64(layer))
        kh = _mix(k[:, None] ^ np.arange(heads, dtype=np.uint64)[None, :])  # [n, H]
        w = _mix(kh[:, :, None] ^ np.arange(32, dtype=np.uint64)[None, None, :])  # [n, H, 32]
        u = (w[..., None] >> (np.uint64(16) * np.arange(4, dtype=np.uint64))) & np.uint64(0xFFFF)
    v = (u.astype(np.int64) - 32768).astype(np.float32) * np.float32(5.340576171875e-05) * np.float32(scale)
    return bf16_round(v.reshape(pos.shape[0], heads, 128))


def context_kv(seed: int, uid: int, ntok: int, layer: int, heads: int, k_scale: float = 1.0):
    """K, V of one context's first ntok tokens: two [ntok, H, 128] arrays."""
    pos = np.arange(ntok, dtype=np.int64)
    return (synth_rows(seed, TAG_K, uid, pos, layer, heads, k_scale),
            synth_rows(seed, TAG_V, uid, pos, layer, heads, 1.0))


def row_queries(seed: int, leaf_uids: Sequence[int], leaf_pos: Sequence[int], layer: int, heads: int) -> np.ndarray:
    """Q rows keyed by (leaf uid, leaf tokens at plan time + rank << 40)."""
    ranks: Dict[int, int] = {}
    keys = []
    for u in leaf_uids:
        r = ranks.get(u, 0)
        ranks[u] = r + 1
        keys.append(r)
    pos = np.asarray(leaf_pos, dtype=np.int64) + (np.asarray(keys, dtype=np.int64) << 40)
    out = np.empty((len(leaf_uids), heads, 128), dtype=np.float32)
    for i, (u, p) in enumerate(zip(leaf_uids, pos)):
        out[i] = synth_rows(seed, TAG_Q, u, [p], layer, heads)[0]
    return out


# ------------------------------------------------------------ attention
def attend(q: np.ndarray, k: np.ndarray, v: np.ndarray, dtype=np.float64) -> np.ndarray:
    """softmax(q k^T / sqrt(D)) v for one row: q [H, D], k/v [T, H, D]."""
    H, D = q.shape
    if k.shape[0] == 0:
        return np.zeros((H, D), dtype=dtype)
    qd = q.astype(dtype)
    kd = k.astype(dtype)
    vd = v.astype(dtype)
    s = np.einsum("hd,thd->ht", qd, kd) * dtype(1.0 / math.sqrt(D))
    s = s - s.max(axis=1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=1, keepdims=True)
    return np.einsum("ht,thd->hd", p, vd)


_C_LIB = None


def c_lib():
    """oracle_c.c (the C restatement, built by oracle/Makefile) via ctypes, or
    None when it cannot be built (numpy restatement then)."""
    global _C_LIB
    if _C_LIB is None:
        import ctypes
        import os
        import subprocess

        here = os.path.dirname(os.path.abspath(__file__))
        path = os.path.join(here, "build", "liboracle_c.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", here], check=False)
        try:
            lib = ctypes.CDLL(path)
            lib.oracle_synth_rows.restype = None
            lib.oracle_synth_rows.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_float,
                                              ctypes.c_void_p]
            _C_LIB = lib
        except OSError:
            _C_LIB = False
    return _C_LIB or None


def synth_rows_range(seed: int, tag: int, uid: int, pos0: int, n: int, layer: int, heads: int,
                     scale: float = 1.0) -> np.ndarray:
    """synth_rows for the contiguous positions [pos0, pos0 + n), through the C
    restatement when available (same values, pinned by test_oracle)."""
    lib = c_lib()
    if lib is None or n == 0:
        return synth_rows(seed, tag, uid, np.arange(pos0, pos0 + n), layer, heads, scale)
    out = np.empty((n, heads, 128), dtype=np.float32)
    lib.oracle_synth_rows(int(seed) & MASK64, tag, int(uid), int(pos0), int(n), int(layer), int(heads),
                          float(scale), out.ctypes.data)
    return out


class KVCache:
    """Generated K/V per (context uid, layer), grown on demand.

    `appended[uid] = (n0, rows)`: positions >= n0 of that context hold model
    rows instead of generated ones (the K/V a TensorDecodeModel appended
    during decode); rows(layer, kv, positions) -> [n, H, 128] float32."""

    def __init__(self, seed: int, heads: int, k_scale: float = 1.0, appended=None, alias=None):
        self.seed, self.heads, self.k_scale = seed, heads, k_scale
        self.appended = appended or {}
        # alias[uid] = src_uid: a context whose K/V was copied from another
        # engine's context (prefix migration) holds that context's rows
        self.alias = alias or {}
        self._c: Dict[Tuple[int, int], Tuple[np.ndarray, np.ndarray]] = {}

    def _gen(self, uid: int, ntok: int, layer: int):
        n0, rows = self.appended.get(uid, (ntok, None))
        n0 = min(n0, ntok)
        src = self.alias.get(uid, uid)
        k = synth_rows_range(self.seed, TAG_K, src, 0, n0, layer, self.heads, self.k_scale)
        v = synth_rows_range(self.seed, TAG_V, src, 0, n0, layer, self.heads, 1.0)
        if ntok > n0:
            pos = np.arange(n0, ntok)
            k = np.concatenate([k, np.asarray(rows(layer, 0, pos), dtype=np.float32)])
            v = np.concatenate([v, np.asarray(rows(layer, 1, pos), dtype=np.float32)])
        return k, v

    def get(self, uid: int, ntok: int, layer: int):
        key = (uid, layer)
        have = self._c.get(key)
        if have is None or have[0].shape[0] < ntok:
            have = self._gen(uid, max(ntok, 1), layer)
            self._c[key] = have
        return have[0][:ntok], have[1][:ntok]


def attend_rows(chains: Sequence[Sequence[Tuple[int, int]]], q: np.ndarray, kv: KVCache, layer: int,
                dtype=np.float64) -> np.ndarray:
    """Per row: full softmax attention over the concatenated chain
    [(uid, tokens)] root -> leaf.  q: [B, H, D] -> out [B, H, D]."""
    out = np.zeros(q.shape, dtype=dtype)
    for b, chain in enumerate(chains):
        ks, vs = [], []
        for uid, ntok in chain:
            if ntok > 0:
                k, v = kv.get(uid, ntok, layer)
                ks.append(k)
                vs.append(v)
        if ks:
            out[b] = attend(q[b], np.concatenate(ks), np.concatenate(vs), dtype)
    return out


def attend_forest(chains: Sequence[Sequence[Tuple[int, int]]], q: np.ndarray, kv: KVCache, layer: int,
                  dtype=np.float64) -> np.ndarray:
    """Same math as attend_rows -- one exact softmax over each row's whole
    concatenated chain, no split-K / partial merging -- with the products
    batched per context: every context's K/V is multiplied once with the
    queries of all rows that read it (BLAS), the max and the sum are taken over
    the row's full score vector.  For full-size checks (6k-token prefixes,
    40 heads, 64-256 rows)."""
    B, H, D = q.shape
    scale = dtype(1.0 / math.sqrt(D))
    qh = np.ascontiguousarray(q.astype(dtype).transpose(1, 0, 2))  # [H, B, D]
    users: Dict[int, List[int]] = {}
    ntok: Dict[int, int] = {}
    for b, chain in enumerate(chains):
        for uid, n in chain:
            if n > 0:
                users.setdefault(uid, []).append(b)
                ntok[uid] = n
    scores = {}
    m = np.full((H, B), -np.inf, dtype=dtype)
    for uid, rows in users.items():
        k, _ = kv.get(uid, ntok[uid], layer)
        kt = np.ascontiguousarray(k.astype(dtype).transpose(1, 2, 0))  # [H, D, T]
        idx = np.asarray(rows)
        s = np.matmul(qh[:, idx, :], kt) * scale  # [H, nr, T]
        scores[uid] = (idx, s)
        m[:, idx] = np.maximum(m[:, idx], s.max(axis=2))  # (a row reads a context once)
    mm = np.where(np.isfinite(m), m, 0.0)
    l = np.zeros((H, B), dtype=dtype)
    o = np.zeros((H, B, D), dtype=dtype)
    for uid, (idx, s) in scores.items():
        _, v = kv.get(uid, ntok[uid], layer)
        p = np.exp(s - mm[:, idx, None])
        vh = np.ascontiguousarray(v.astype(dtype).transpose(1, 0, 2))  # [H, T, D]
        l[:, idx] += p.sum(axis=2)
        o[:, idx] += np.matmul(p, vh)
    out = np.where(l[:, :, None] > 0, o / np.where(l > 0, l, 1.0)[:, :, None], 0.0)
    return out.transpose(1, 0, 2)


def attend_shared_batch(q: np.ndarray, prefix_k: np.ndarray, prefix_v: np.ndarray,
                        suffix_k: Sequence[np.ndarray], suffix_v: Sequence[np.ndarray],
                        dtype=np.float32) -> np.ndarray:
    """Matmul form of the same math for one shared prefix + per-row suffixes
    (the CPU baseline: batched BLAS over heads); exact softmax over the
    concatenated chain, no split-K decomposition."""
    B, H, D = q.shape
    scale = dtype(1.0 / math.sqrt(D))
    qh = np.ascontiguousarray(q.astype(dtype).transpose(1, 0, 2))          # [H, B, D]
    kp = np.ascontiguousarray(prefix_k.astype(dtype).transpose(1, 2, 0))   # [H, D, P]
    vp = np.ascontiguousarray(prefix_v.astype(dtype).transpose(1, 0, 2))   # [H, P, D]
    sp = np.matmul(qh, kp) * scale                                          # [H, B, P]
    ss = []
    for b in range(B):
        ks = suffix_k[b].astype(dtype).transpose(1, 2, 0)                   # [H, D, S]
        ss.append(np.matmul(qh[:, b:b + 1, :], ks)[:, 0, :] * scale)        # [H, S]
    m = sp.max(axis=2)                                                      # [H, B]
    for b in range(B):
        if ss[b].shape[1]:
            m[:, b] = np.maximum(m[:, b], ss[b].max(axis=1))
    ep = np.exp(sp - m[:, :, None])
    l = ep.sum(axis=2)
    o = np.matmul(ep, vp)                                                   # [H, B, D]
    for b in range(B):
        if ss[b].shape[1]:
            es = np.exp(ss[b] - m[:, b:b + 1])                              # [H, S]
            l[:, b] += es.sum(axis=1)
            vs = suffix_v[b].astype(dtype).transpose(1, 0, 2)               # [H, S, D]
            o[:, b, :] += np.matmul(es[:, None, :], vs)[:, 0, :]
    return (o / l[:, :, None]).transpose(1, 0, 2)


def tolerance_report(got: np.ndarray, want: np.ndarray) -> Dict[str, float]:
    """max-abs, relative L2 and mean-relative error."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    diff = got - want
    denom = np.linalg.norm(want)
    return {
        "max_abs": float(np.abs(diff).max()) if diff.size else 0.0,
        "rel_l2": float(np.linalg.norm(diff) / denom) if denom > 0 else float(np.linalg.norm(diff)),
        "mean_rel": float(np.abs(diff).sum() / max(np.abs(want).sum(), 1e-30)),
    }
