"""GPU-backed engine behind the reference's Fill/Generate/FreeContext surface.

`GpuEngine` is a drop-in for `semflow.engine.Engine`
(/root/reference/pkg/src/semflow/engine.py:157-538): same constructor, same
methods, same live attributes the manager, scheduler and report builder read
(SURVEY.md §8b).  Bookkeeping that the reference keeps in Python dicts is
split as follows:

* block accounting, the context forest topology and the per-step work list
  live in the C++ pool of libforkattn.so (PagedKvStore, engine.py:66-106,
  and the `_batch_tokens` walk, engine.py:470-484);
* refcounts, the dropped flag, the hash registry, the fill queue and the
  generation tasks stay here, because the manager and the scheduler read
  and write them directly;
* with a device, every decode step runs the shared-prefix attention kernels
  for all layers over the running batch before the
  one-token growth, exactly where the reference charges `batch_tokens`.

Without a device (``device=None``) the engine is the same native block
manager with no attention — the integer twin the CPU parity suites drive.
"""

from __future__ import annotations

import ctypes
import itertools
import os
import time
from collections import deque
from dataclasses import dataclass, field
from typing import Any, Deque, Dict, List, Optional, Sequence, Set, Tuple

from . import _lib
from .errors import ContextBusy, OutOfMemory, UnknownContext, UnknownParentContext

MS = 1_000_000  # ns per millisecond
_PHASES = bool(os.environ.get("FK_DEBUG_TIMING"))  # per-phase host time of step() (profiles/host_step.py)
_NVTX = bool(os.environ.get("FK_NVTX"))  # an NVTX range per GpuEngine.step (the C++ entry points always emit theirs)
FNV64_EMPTY = 0xCBF29CE484222325


def hash_token_ids(token_ids: Sequence[int], seed: int = FNV64_EMPTY) -> int:
    """tokenizer.hash_token_ids (tokenizer.py:47-49) via the C-ABI."""
    return _lib.fnv1a64_u32(list(token_ids), seed)


class Context:
    """Forest node (engine.py:53-63) plus the pool uid that keys it in C++.

    The C++ pool is authoritative for the block accounting: token_count and
    block_ids are read from it on demand (a decode step then touches no
    Python object per row); refcount, dropped and the hashes live here."""

    __slots__ = ("context_id", "engine_id", "parent_id", "refcount", "dropped", "chain_hashes",
                 "registered_hashes", "uid", "_pool", "_released")

    def __init__(self, context_id: str, engine_id: str, parent_id: Optional[str], refcount: int = 0,
                 dropped: bool = False, chain_hashes: Optional[List[int]] = None,
                 registered_hashes: Optional[List[int]] = None, uid: int = -1, pool: Any = None):
        self.context_id = context_id
        self.engine_id = engine_id
        self.parent_id = parent_id
        self.refcount = refcount
        self.dropped = dropped
        self.chain_hashes = [] if chain_hashes is None else chain_hashes
        self.registered_hashes = [] if registered_hashes is None else registered_hashes
        self.uid = uid
        self._pool = pool
        self._released = False

    @property
    def token_count(self) -> int:
        if self._released or self._pool is None:
            return 0
        return int(_lib.lib.fk_ctx_tokens(self._pool.handle, self.uid))

    @property
    def block_ids(self) -> List[int]:
        if self._released or self._pool is None:
            return []
        return self._pool.blocks(self.uid)[0]

    def __repr__(self) -> str:
        return (f"Context({self.context_id!r}, parent={self.parent_id!r}, tokens={self.token_count}, "
                f"refcount={self.refcount}, dropped={self.dropped})")


class GenerationTask:
    """engine.py:116-128.  `emitted` is derived from the engine's decode
    counter: a running generation emits one token per decode iteration until
    it finishes or fails (engine.py:431-443), so the step updates no
    per-row Python state -- only the rows that finish or fail."""

    __slots__ = ("request_id", "context_id", "token_ids", "value_text", "started", "done",
                 "_base", "_clock", "_t0", "_t_end")

    def __init__(self, request_id: str, context_id: str, token_ids: List[int], value_text: str,
                 emitted: int = 0, started: bool = False, done: bool = False, clock: Optional[List[int]] = None):
        self.request_id = request_id
        self.context_id = context_id
        self.token_ids = token_ids
        self.value_text = value_text
        self.started = started
        self.done = done
        self._base = emitted
        self._clock = clock if clock is not None else [0]
        self._t0 = -1      # decode counter when it first ran (-1: never)
        self._t_end = -1   # decode counter when it stopped (-1: still running)

    @property
    def emitted(self) -> int:
        if self._t0 < 0:
            return self._base
        end = self._t_end if self._t_end >= 0 else self._clock[0]
        return self._base + end - self._t0

    @property
    def remaining(self) -> int:
        return len(self.token_ids) - self.emitted

    def __repr__(self) -> str:
        return (f"GenerationTask({self.request_id!r}, ctx={self.context_id!r}, emitted={self.emitted}/"
                f"{len(self.token_ids)}, started={self.started}, done={self.done})")


@dataclass(frozen=True)
class ModelGeometry:
    """Attention shape of the served model (new ctor args: Config rejects
    unknown keys, config.py:39-42, so they cannot live there)."""

    num_layers: int
    num_heads: int
    head_dim: int = 128


LLAMA_7B = ModelGeometry(32, 32, 128)
LLAMA_13B = ModelGeometry(40, 40, 128)
TINY = ModelGeometry(1, 32, 128)


class GpuKvStore:
    """PagedKvStore (engine.py:66-106) over the C++ pool.

    Logical ids come from the pool's monotonic counter and are never
    recycled, physical pages are.  `owner` (block id -> context id, read by
    the reference's conservation oracle, tests/oracles.py:543-553) is built
    from the pool on demand."""

    def __init__(self, pool: "_Pool", block_size: int, contexts: Dict[str, "Context"]):
        self._pool = pool
        self.block_size = block_size
        self._contexts = contexts

    @property
    def owner(self) -> Dict[int, str]:
        return {bid: ctx.context_id for ctx in self._contexts.values() for bid in ctx.block_ids}

    @property
    def total_blocks(self) -> int:
        return self._pool.stats().total_blocks

    @total_blocks.setter
    def total_blocks(self, value: int) -> None:  # manager.py:138 writes this
        _lib.check(_lib.lib.fk_pool_set_total_blocks(self._pool.handle, int(value)))

    @property
    def peak_used(self) -> int:
        return self._pool.stats().peak_used

    @property
    def used_blocks(self) -> int:
        return self._pool.stats().used_blocks

    @property
    def free_blocks(self) -> int:
        return self._pool.stats().free_blocks

    def blocks_for(self, tokens: int) -> int:
        return -(-tokens // self.block_size)

    def grow(self, ctx: Context, new_token_count: int) -> None:
        status = _lib.lib.fk_ctx_grow(self._pool.handle, ctx.uid, int(new_token_count), None, 0, None)
        if status == _lib.FK_OUT_OF_MEMORY:
            need = self.blocks_for(new_token_count) - len(ctx.block_ids)
            raise OutOfMemory(f"engine {ctx.engine_id}: need {need} blocks, {self.free_blocks} free")
        _lib.check(status)

    def release(self, ctx: Context) -> None:
        _lib.check(_lib.lib.fk_ctx_release(self._pool.handle, ctx.uid))
        ctx._released = True


class _Pool:
    """Owns one fk_pool* (one per engine / GPU)."""

    def __init__(self, geometry: ModelGeometry, block_size: int, total_blocks: int, device: Optional[int],
                 num_pages: int = 0):
        desc = _lib.PoolDesc(
            num_layers=geometry.num_layers,
            num_heads=geometry.num_heads,
            head_dim=geometry.head_dim,
            block_size=block_size,
            total_blocks=total_blocks,
            num_pages=num_pages if device is not None else 0,
            device=-1 if device is None else int(device),
            reserved=0,
        )
        h = ctypes.c_void_p()
        rc = _lib.lib.fk_pool_create(ctypes.byref(desc), ctypes.byref(h))
        if rc == _lib.FK_INVALID_ARGUMENT and device is not None:
            # A process holds at most 64 device pools (two __constant__ plan
            # slots each).  Engines dropped without close() inside reference
            # cycles keep theirs until the cycle collector runs: run it, retry.
            import gc

            gc.collect()
            rc = _lib.lib.fk_pool_create(ctypes.byref(desc), ctypes.byref(h))
        _lib.check(rc)
        self.handle = h
        self._ids = (ctypes.c_int64 * 64)()
        self._stats = _lib.PoolStats()

    def id_buffer(self, n: int):
        if n > len(self._ids):
            self._ids = (ctypes.c_int64 * max(n, 2 * len(self._ids)))()
        return self._ids

    def blocks(self, uid: int) -> Tuple[List[int], List[int]]:
        """(logical ids, physical pages) of a context, read back from C++."""
        n = ctypes.c_int64(0)
        _lib.check(_lib.lib.fk_ctx_blocks(self.handle, uid, None, None, 0, ctypes.byref(n)))
        lg = (ctypes.c_int64 * max(n.value, 1))()
        ph = (ctypes.c_int32 * max(n.value, 1))()
        _lib.check(_lib.lib.fk_ctx_blocks(self.handle, uid, lg, ph, n.value, ctypes.byref(n)))
        return lg[:n.value], ph[:n.value]

    def stats(self) -> _lib.PoolStats:
        _lib.check(_lib.lib.fk_pool_stats_get(self.handle, ctypes.byref(self._stats)))
        return self._stats

    def set_option(self, option: int, value: int) -> None:
        _lib.check(_lib.lib.fk_pool_set_option(self.handle, option, int(value)))

    def close(self) -> None:
        if self.handle:
            _lib.lib.fk_pool_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SyntheticDecodeModel:
    """Deterministic stand-in for the QKV projection: Q rows and the step's
    new K/V rows come from the counter-hash generator on the device
    (oracle/forkattn_oracle.py restates it).  Fills use the same generator."""

    def __init__(self, seed: int = 0x5EED, k_scale: float = 1.0):
        self.seed = seed
        self.k_scale = k_scale


class TensorDecodeModel:
    """Caller-supplied rows: q[L][B][H][D] and k/v[L][B][H][D] bf16, device
    resident or host (pinned) — host tensors are copied in the step, and the
    output is copied back, which is the end-to-end path of bench.py.
    `out` (device, same shape as q) is the model's own attention-output
    buffer: the step writes it in place (on the engine stream) instead of
    allocating a new tensor every step."""

    def __init__(self, q, k=None, v=None, copy_out: bool = False, out=None):
        self.q, self.k, self.v = q, k, v
        self.copy_out = copy_out
        self.host_out = None
        self.out = out


# ---- the reference runtime ------------------------------------------------------
# GpuEngine plugs into semflow (the reference runtime: manager, scheduler,
# API).  Where semflow is importable, the engine's pure bookkeeping -- the
# report / plan / fill dataclasses, the cost model, prefix planning, the
# live-context walk, context freeing -- is the reference's own code
# (GpuEngine subclasses semflow.engine.Engine and overrides only what the
# device path changes: the context forest and block store live in the C++
# pool, fills write K/V, the step runs the kernels).  Without semflow (a
# standalone bench run) the restatement below stands in, pinned to the
# reference by the golden op streams (tests/golden) and the rebound suites.
_ref = None
if not os.environ.get("FK_STANDALONE_ENGINE"):
    try:
        from semflow import engine as _ref  # noqa: F811
    except ImportError:
        _ref = None

if _ref is not None:
    CostModel = _ref.CostModel
    FillTask = _ref.FillTask
    StepReport = _ref.StepReport
    ContextPlan = _ref.ContextPlan
    format_ms = _ref.format_ms
    _EngineBase = _ref.Engine
else:
    def format_ms(ns: int) -> str:
        """engine.format_ms (engine.py:541-545): ms with <= 3 decimals, zeros trimmed."""
        text = "%.3f" % (ns / MS)
        if "." in text:
            text = text.rstrip("0").rstrip(".")
        return text

    @dataclass
    class CostModel:
        """Virtual clock of the reference (engine.py:25-50); kept so reports and
        traces stay byte-identical.  Any object with the same attributes works."""

        c0_ms: float = 2.0
        c1_ms: float = 0.0062
        c2_ms: float = 5.0
        c3_ms: float = 0.002
        shared_kernel: bool = True
        block_size: int = 16

        def __post_init__(self) -> None:
            self.c0_ns = round(self.c0_ms * MS)
            self.c1_ns = round(self.c1_ms * MS)
            self.c2_ns = round(self.c2_ms * MS)
            self.c3_ns = round(self.c3_ms * MS)

        def iteration_ns(self, batch_tokens: int) -> int:
            return self.c0_ns + self.c1_ns * batch_tokens

        def fill_ns(self, fill_tokens: int) -> int:
            return self.c2_ns + self.c3_ns * fill_tokens

        def latency_threshold_ms(self, capacity: int) -> float:
            return self.iteration_ns(capacity) / MS

    @dataclass
    class FillTask:
        request_id: Optional[str]
        context_id: str
        token_ids: List[int]

    @dataclass
    class StepReport:
        engine_id: str
        started_ns: int
        elapsed_ns: int
        fill_tokens: int
        batch_tokens: int
        emitted: Dict[str, int]
        finished: List[str]
        failed: List[Tuple[str, str]]
        fill_completed: List[str]

    @dataclass
    class ContextPlan:
        reuse_context_id: Optional[str]
        reused_tokens: int
        fill_segments: List[Tuple[List[int], int]]
        marginal_tokens: int
        adopted_tokens: int = 0

    class _EngineBase:
        """Restatement of the reference Engine's bookkeeping (engine.py:186-387,
        534-538) for runs without semflow; GpuEngine supplies the state."""

        def new_context_id(self) -> str:
            return f"{self.engine_id}.c{next(self._ctx_counter)}"

        def get_context(self, context_id: str) -> Context:
            ctx = self.contexts.get(context_id)
            if ctx is None:
                raise UnknownContext(f"unknown context {context_id}")
            return ctx

        def free_context(self, context_id: str) -> None:
            ctx = self.get_context(context_id)
            if ctx.refcount > 0:
                raise ContextBusy(f"context {context_id} has refcount {ctx.refcount}")
            self._discard_context(ctx)

        def mark_dropped(self, context_id: str) -> None:
            ctx = self.get_context(context_id)
            ctx.dropped = True
            if ctx.refcount == 0:
                self._discard_context(ctx)

        # -- planning (engine.py:304-382) -------------------------------------------

        def plan_prefix(self, chain_hashes: Sequence[int], segment_tokens: Sequence[Sequence[int]],
                        overlay: Optional[Dict[int, str]] = None) -> ContextPlan:
            """Deepest chain boundary held by the registry (or the overlay of
            this scheduling pass) -> context to fork from; see engine.py:304-363."""
            n = len(chain_hashes)
            cumulative: List[int] = []
            acc = 0
            for i in range(n):
                if i < len(segment_tokens):
                    acc += len(segment_tokens[i])
                cumulative.append(acc)
            reuse_id: Optional[str] = None
            depth = credited = 0
            if self.reuse_enabled:
                live: Optional[Set[str]] = None
                for i in reversed(range(n)):
                    if cumulative[i] == 0:
                        break
                    h = chain_hashes[i]
                    holder = self.registry.get(h)
                    planned = overlay is not None and h in overlay
                    if holder is None and not planned:
                        continue
                    if reuse_id is None:
                        reuse_id = holder if holder is not None else overlay[h]
                        depth = i + 1
                    if planned:
                        credited = i + 1
                        break
                    if live is None:
                        live = self._live_context_ids()
                    if holder in live:
                        credited = i + 1
                        break
            fills: List[Tuple[List[int], int]] = []
            marginal = 0
            for i in range(depth, len(segment_tokens)):
                seg = list(segment_tokens[i])
                if seg:
                    fills.append((seg, chain_hashes[i]))
                    marginal += len(seg)
            reused = 0
            if reuse_id is not None and reuse_id in self.contexts:
                reused = self._chain_tokens(self.contexts[reuse_id])
            adopted = 0
            if depth > credited:
                adopted = cumulative[depth - 1] - (cumulative[credited - 1] if credited else 0)
            return ContextPlan(reuse_id, reused, fills, marginal, adopted)

        def _live_context_ids(self) -> Set[str]:
            live: Set[str] = set()
            for leaf in self.request_leaf.values():
                for c in self._ancestors(self.contexts.get(leaf)):
                    if c.context_id in live:
                        break
                    live.add(c.context_id)
            return live

        def _chain_tokens(self, ctx: Context) -> int:
            return sum(c.token_count for c in self._ancestors(ctx))

        def has_work(self) -> bool:
            return bool(self.fill_queue) or any(not g.done for g in self.gens.values())

        @property
        def charged_tokens(self) -> int:
            return sum(self.charges.values())

        def admitted_classes(self) -> List[str]:
            return sorted(set(self.holder_class.values()))


class GpuEngine(_EngineBase):
    """Drop-in `Engine` (engine.py:157-538) with a B200 decode path."""

    def __init__(
        self,
        engine_id: str,
        cost: Any,
        kv_tokens: int = 120_000,
        token_capacity: int = 64_000,
        *,
        device: Optional[int] = None,
        geometry: ModelGeometry = TINY,
        model: Any = None,
        num_pages: int = 0,
        capture_f32: bool = False,
        keep_history: bool = False,
        attend_own_token: bool = False,
        peers: Optional[List["GpuEngine"]] = None,
    ):
        self.engine_id = engine_id
        self.cost = cost
        self.token_capacity = token_capacity
        self.latency_threshold_ms = cost.latency_threshold_ms(token_capacity)
        block_size = getattr(cost, "block_size", 16)
        self.geometry = geometry
        self.device = device
        self._pool = _Pool(geometry, block_size, -(-kv_tokens // block_size), device, num_pages)
        self.contexts: Dict[str, Context] = {}
        self.store = GpuKvStore(self._pool, block_size, self.contexts)
        self.clock_ns = 0
        self.registry: Dict[int, str] = {}
        self.fill_queue: Deque[FillTask] = deque()
        self.gens: Dict[str, GenerationTask] = {}
        self.pending_fills: Dict[str, int] = {}
        self.charges: Dict[str, int] = {}
        self.holder_class: Dict[str, str] = {}
        self.request_leaf: Dict[str, str] = {}
        self.trace: List[str] = []
        self.reports: List[StepReport] = []
        self.reuse_enabled = True
        self.busy_ns = 0
        self.fill_ns_total = 0
        self.decode_ns_total = 0
        self.total_emitted = 0
        self._ctx_counter = itertools.count()
        self._uid_counter = itertools.count()
        # decode iterations so far (GenerationTask.emitted derives from it), the
        # running rows in gens order (rebuilt only when the set changes) and
        # the running generations by the counter value they finish at
        self._dclock = [0]
        self._running: Optional[List[GenerationTask]] = None
        self._running_rids: List[str] = []
        self._finish_at: Dict[int, List[GenerationTask]] = {}
        # device state
        self.model = model if model is not None else SyntheticDecodeModel()
        self.capture_f32 = capture_f32
        self.keep_history = keep_history
        self.history: List[Dict[str, Any]] = []
        self.last_output = None
        self.last_output_f32 = None
        self._last_running: List[GenerationTask] = []
        self.last_plan = _lib.PlanInfo()
        self.kv_tokens_streamed = 0  # sum of batch_tokens over decode steps (per layer)
        # prefix migration (engine_factory(migrate_prefixes=True)): the engines
        # of one process whose registries a fill may copy a prefix from
        self._peers = peers
        self.prefix_migrations = 0
        self.migrated_tokens = 0
        self.migrated: Dict[int, Tuple[str, int, int]] = {}  # dst uid -> (src engine id, src uid, tokens)
        self._stream = None
        self._plan_rows: List[GenerationTask] = []  # rows of _leaf_buf
        self._nfail = ctypes.c_int32(0)
        self._zero_len: List[GenerationTask] = []
        self._leaf_buf = (ctypes.c_int64 * 64)()
        self._leaf_pos0 = (ctypes.c_int64 * 64)()
        self._pos_buf = (ctypes.c_int64 * 64)()
        self._id_buf = (ctypes.c_int64 * 64)()
        if device is not None:
            import torch

            self._torch = torch
            self._dev = torch.device("cuda", device)
            with torch.cuda.device(self._dev):
                self._stream = torch.cuda.Stream(self._dev)
                # fills (prefill KV writes, prefix migrations) run on their own
                # stream: decode waits only for the fills of contexts it reads
                self._fill_stream = torch.cuda.Stream(self._dev)
            self._spv = self._stream.cuda_stream  # (plain int: ctypes passes it as void*)
            self._ev_caller = torch.cuda.Event()  # the caller's stream position, per step
            self._dev_index = int(device)
            self._caller_raw = None  # the caller's stream (cached Stream object, by raw handle)
            self._caller = None
            self._fill_pending: Dict[str, Any] = {}  # context id -> event of its last fill
            self._release_event = None  # engine-stream fence of the last page release
            # The engine owns Q's producer side (its own buffers, ordered by
            # stream events), so a layer's kernels may start under the previous
            # layer's merge (cross-layer programmatic dependent launch).
            self._pool.set_option(_lib.FK_OPT_PDL, 2)
        # FK_OPT_APPEND_FIRST: each row's new K/V row is
        # appended before attention and is part of its span, as in a real
        # decoder; the default is the reference's span (engine.py:416-434)
        self.attend_own_token = bool(attend_own_token)
        if self.attend_own_token:
            self._pool.set_option(_lib.FK_OPT_APPEND_FIRST, 1)

    # -- device plumbing ------------------------------------------------------

    @property
    def stream(self):
        return self._stream

    def _sp(self):
        return ctypes.c_void_p(self._stream.cuda_stream) if self._stream is not None else None

    def set_option(self, option: int, value: int) -> None:
        self._pool.set_option(option, value)

    def reserve_pages(self, num_pages: int) -> None:
        """Back at least `num_pages` physical pages now (fk_pool_reserve_pages).
        The arena otherwise grows on demand, and a growth is a device-wide
        copy of every live page -- do it before latency matters."""
        _lib.check(_lib.lib.fk_pool_reserve_pages(self._pool.handle, int(num_pages)))

    def pool_stats(self) -> _lib.PoolStats:
        return self._pool.stats()

    def context_pages(self, context_id: str) -> Tuple[List[int], List[int]]:
        """(logical ids, physical pages) of a context, read back from C++."""
        return self._pool.blocks(self.get_context(context_id).uid)

    def close(self) -> None:
        if self._stream is not None:
            self._fill_stream.synchronize()
            self._stream.synchronize()
        self._pool.close()

    # -- context primitives (engine.py:192-300) --------------------------------

    def create_context(self, context_id: str, parent_context_id: Optional[str], request_id: Optional[str] = None) -> Context:
        inherited: List[int] = []
        parent_uid = -1
        if parent_context_id is not None:
            parent = self.contexts.get(parent_context_id)
            if parent is None:
                raise UnknownParentContext(f"unknown parent {parent_context_id}")
            parent.refcount += 1
            inherited = list(parent.chain_hashes)
            parent_uid = parent.uid
        ctx = Context(context_id, self.engine_id, parent_context_id, chain_hashes=inherited,
                      uid=next(self._uid_counter), pool=self._pool)
        _lib.check(_lib.lib.fk_ctx_create(self._pool.handle, ctx.uid, parent_uid))
        self.contexts[context_id] = ctx
        if request_id is not None:
            self.request_leaf[request_id] = context_id
        return ctx

    def fill(self, token_ids: Sequence[int], context_id: str, parent_context_id: Optional[str] = None,
             request_id: Optional[str] = None, boundary_hash: Optional[int] = None, *, kv=None,
             kv_from=None) -> int:
        """Allocate pages for the new tokens, write their KV and queue the
        fill work; atomic on OutOfMemory (engine.py:225-255).

        `kv=(k, v)`: the model's K/V rows for these tokens, device tensors
        [L][len(token_ids)][H][D] bf16, written into the pages (fk_fill_kv).
        `kv_from=(engine, context_id)`: copy the first len(token_ids) tokens'
        K/V of a context held by another GpuEngine (another GPU: NVLink peer
        reads, fk_ctx_copy_kv) -- a shared prefix migrates instead of being
        prefilled again.  The new context must be fresh.
        Without either, the deterministic synthetic generator stands in for
        the prefill (tests, bench)."""
        if kv is not None:
            self._check_rows(kv, len(token_ids))
        if (kv is None and kv_from is None and self._peers and boundary_hash is not None and self.device is not None
                and token_ids and context_id not in self.contexts):
            kv_from = self._peer_prefix(boundary_hash, parent_context_id, len(token_ids))
        if kv_from is not None:
            src_eng, src_id = kv_from
            src_ctx = src_eng.get_context(src_id)
            if context_id in self.contexts or len(token_ids) > src_ctx.token_count or self.device is None:
                raise ValueError("kv_from needs a fresh context on a device engine and <= source tokens")
        fresh = context_id not in self.contexts
        ctx = self.create_context(context_id, parent_context_id) if fresh else self.get_context(context_id)
        before = ctx.token_count
        try:
            self.store.grow(ctx, before + len(token_ids))
        except OutOfMemory:
            if fresh:
                self._discard_context(ctx)
            raise
        if self.device is not None and len(token_ids) > 0:
            torch = self._torch
            fs = self._fill_stream
            fsp = ctypes.c_void_p(fs.cuda_stream)
            if self._release_event is not None:  # recycled pages: earlier decode work is done with them
                fs.wait_event(self._release_event)
            prev = self._fill_pending.get(context_id)
            if prev is not None:
                fs.wait_event(prev)
            if kv_from is not None:
                ev = torch.cuda.Event()
                ev.record(src_eng.stream)  # the source pages are written
                fs.wait_event(ev)
                src_fill = src_eng._fill_pending.get(src_id)
                if src_fill is not None:
                    fs.wait_event(src_fill)
                _lib.check(_lib.lib.fk_ctx_copy_kv(self._pool.handle, ctx.uid, src_eng._pool.handle, src_ctx.uid,
                                                   len(token_ids), fsp))
            elif kv is not None:
                k, v = kv
                with torch.cuda.device(self._dev):
                    fs.wait_stream(torch.cuda.current_stream(self._dev))  # the caller's tensors
                _lib.check(_lib.lib.fk_fill_kv(self._pool.handle, ctx.uid, before, ctx.token_count, 0,
                                               self.geometry.num_layers, ctypes.c_void_p(k.data_ptr()),
                                               ctypes.c_void_p(v.data_ptr()), fsp))
                k.record_stream(fs)
                v.record_stream(fs)
            else:
                _lib.check(_lib.lib.fk_synth_fill(self._pool.handle, ctx.uid, before, ctx.token_count,
                                                  self.model_seed, self.model_k_scale, fsp))
            done = torch.cuda.Event()
            done.record(fs)
            self._fill_pending[context_id] = done
            if kv_from is not None:
                src_eng.stream.wait_event(done)  # the source may not recycle its pages before the copy
                self.prefix_migrations += 1
                self.migrated_tokens += len(token_ids)
                self.migrated[ctx.uid] = (src_eng.engine_id, src_ctx.uid, len(token_ids))
        if boundary_hash is not None:
            ctx.chain_hashes.append(boundary_hash)
            if boundary_hash not in self.registry:
                self.registry[boundary_hash] = context_id
                ctx.registered_hashes.append(boundary_hash)
        self.fill_queue.append(FillTask(request_id, context_id, list(token_ids)))
        if request_id is not None:
            self.pending_fills[request_id] = self.pending_fills.get(request_id, 0) + 1
            self.request_leaf[request_id] = context_id
        return len(token_ids)

    def _boundary(self, context_id: Optional[str]) -> Optional[int]:
        """Chain hash at the end of a context (None: the root side)."""
        ctx = self.contexts.get(context_id) if context_id else None
        return ctx.chain_hashes[-1] if ctx is not None and ctx.chain_hashes else None

    def _peer_prefix(self, boundary_hash: int, parent_context_id: Optional[str], ntok: int):
        """The reference scheduler's `shared-ctx` fallback (scheduler.py:198-222)
        places a request on an engine without its prefix when the engines that
        hold it are full; the new engine would prefill the prefix again.
        Instead, a fill whose segment ends at a chain hash another engine of
        the process holds -- same segment (same parent boundary), at least as
        many tokens -- copies that context's K/V (fill(kv_from=...):
        fk_ctx_copy_kv, NVLink peer reads across GPUs).  Returns (engine,
        context id) or None."""
        want_parent = self._boundary(parent_context_id)
        for e in self._peers:
            if e is self or e.device is None:
                continue
            cid = e.registry.get(boundary_hash)
            src = e.contexts.get(cid) if cid is not None else None
            if src is None or src.token_count < ntok or e._boundary(src.parent_id) != want_parent:
                continue
            if e.geometry != self.geometry:
                continue
            return (e, cid)
        return None

    def _check_rows(self, kv, n: int) -> None:
        if self.device is None:
            raise ValueError("kv rows need a device engine")
        geo = self.geometry
        want = (geo.num_layers, n, geo.num_heads, geo.head_dim)
        for t in kv:
            if (tuple(t.shape) != want or t.dtype != self._torch.bfloat16 or t.device != self._dev
                    or not t.is_contiguous()):
                raise ValueError(f"kv rows must be contiguous bf16 {want} on {self._dev}, got "
                                 f"{tuple(t.shape)} {t.dtype} {t.device}")

    @property
    def model_seed(self) -> int:
        return int(getattr(self.model, "seed", 0x5EED))

    @property
    def model_k_scale(self) -> float:
        return float(getattr(self.model, "k_scale", 1.0))

    def generate(self, request_id: str, context_id: str, token_ids: Sequence[int], value_text: str) -> GenerationTask:
        ctx = self.get_context(context_id)
        ctx.refcount += 1  # the active generation holds its leaf
        self.request_leaf[request_id] = context_id
        task = GenerationTask(request_id, context_id, list(token_ids), value_text, clock=self._dclock)
        task.started = self.pending_fills.get(request_id, 0) == 0
        if not task.token_ids:
            self._zero_len.append(task)
        self.gens[request_id] = task
        self._running = None
        return task

    def _discard_context(self, ctx: Context) -> None:
        if self.device is not None:
            # Pages freed here may be handed out again by decode growth (their
            # new rows are written on the engine stream) or by a fill (which
            # waits for _release_event): the engine stream first waits for any
            # fill still writing the discarded contexts, so both reuses are
            # ordered after it.
            c = ctx
            while c is not None:
                ev = self._fill_pending.pop(c.context_id, None)
                if ev is not None:
                    self._stream.wait_event(ev)
                parent = self.contexts.get(c.parent_id) if c.parent_id is not None else None
                c = parent if (parent is not None and parent.refcount == 1 and parent.dropped) else None
            self._release_event = self._torch.cuda.Event()
            self._release_event.record(self._stream)
        while ctx is not None:
            self.store.release(ctx)
            if self.device is not None:
                self._fill_pending.pop(ctx.context_id, None)
            for h in ctx.registered_hashes:
                if self.registry.get(h) == ctx.context_id:
                    del self.registry[h]
            ctx.registered_hashes = []
            del self.contexts[ctx.context_id]
            parent = self.contexts.get(ctx.parent_id) if ctx.parent_id is not None else None
            ctx = None
            if parent is not None:
                parent.refcount -= 1
                if parent.refcount == 0 and parent.dropped:
                    ctx = parent  # cascade (engine.py:280-285)

    def _ancestors(self, ctx: Optional[Context]):
        while ctx is not None:
            yield ctx
            ctx = self.contexts.get(ctx.parent_id) if ctx.parent_id else None

    # -- stepping (engine.py:386-484) ---------------------------------------------

    def _batch_tokens(self, running: List[GenerationTask]) -> int:
        """Host restatement of the dedup walk; the step itself takes the
        number from the C++ planner (they are asserted equal in tests)."""
        if not running:
            return 0
        if self.cost.shared_kernel:
            seen: Set[str] = set()
            total = 0
            for g in running:
                for c in self._ancestors(self.contexts.get(g.context_id)):
                    if c.context_id not in seen:
                        seen.add(c.context_id)
                        total += c.token_count
            return total
        return sum(self._chain_tokens(self.contexts[g.context_id]) for g in running)

    def _plan(self, running: List[GenerationTask]) -> int:
        B = len(running)
        if B > len(self._leaf_buf):
            self._plan_rows = []
            self._leaf_buf = (ctypes.c_int64 * (2 * B))()
            self._leaf_pos0 = (ctypes.c_int64 * (2 * B))()
            self._pos_buf = (ctypes.c_int64 * (2 * B))()
            self._id_buf = (ctypes.c_int64 * (2 * B))()
        prev = self._plan_rows
        if prev is not running and (len(prev) != B or any(a is not b for a, b in zip(prev, running))):
            # the running set changed: new leaf list (a generation keeps its leaf)
            for i, g in enumerate(running):
                self._leaf_buf[i] = self.contexts[g.context_id].uid
            self._plan_rows = running
        if self.keep_history:  # leaf tokens before the step (the synthetic query key)
            for i, g in enumerate(running):
                self._leaf_pos0[i] = self.contexts[g.context_id].token_count
        _lib.check(_lib.lib.fk_step_plan(self._pool.handle, self._leaf_buf, B,
                                         1 if self.cost.shared_kernel else 0, self._sp(),
                                         ctypes.byref(self.last_plan)))
        return int(self.last_plan.batch_tokens)

    def _host_pipeline(self, shape):
        """Device buffers, copy streams and per-layer events for host-resident
        TensorDecodeModel rows (allocated once per shape)."""
        torch = self._torch
        hp = getattr(self, "_hp", None)
        if hp is None or hp["shape"] != shape:
            L = shape[0]
            with torch.cuda.device(self._dev):
                hp = {
                    "shape": shape,
                    "q": torch.empty(shape, dtype=torch.bfloat16, device=self._dev),
                    "k": torch.empty(shape, dtype=torch.bfloat16, device=self._dev),
                    "v": torch.empty(shape, dtype=torch.bfloat16, device=self._dev),
                    "out": torch.empty(shape, dtype=torch.bfloat16, device=self._dev),
                    "h2d": torch.cuda.Stream(self._dev),
                    "d2h": torch.cuda.Stream(self._dev),
                    "ev_q": [torch.cuda.Event() for _ in range(L)],
                    "ev_o": [torch.cuda.Event() for _ in range(L)],
                    # copy granularity: layer chunks (see _layer_chunks)
                    "chunks": self._layer_chunks(L),
                    "ev_kv": torch.cuda.Event(),
                    "ev_d2h": torch.cuda.Event(),
                    "ev_start": torch.cuda.Event(),
                }
            self._hp = hp
        return hp

    @staticmethod
    def _layer_chunks(L: int) -> List[Tuple[int, int]]:
        """Copy chunks of the e2e path: 1 and 3 layers first (layer 0 waits
        for one layer's rows), 8 in the middle, then 2, 1, 1 at the end (the
        step ends with the last chunk's output copy: one layer's rows, ≈13 us
        over PCIe, instead of four).  Each chunk boundary is an event wait in
        the stream, which breaks the PDL chain between layers, so the middle
        chunks stay large."""
        sizes, rest = [], L
        for n in (1, 3):
            if rest > 0:
                sizes.append(min(n, rest))
                rest -= sizes[-1]
        while rest > 12:
            sizes.append(8)
            rest -= 8
        if rest > 4:
            sizes.append(rest - 4)
            rest = 4
        for n in (2, 1, 1):
            if rest > 0:
                sizes.append(min(n, rest))
                rest -= sizes[-1]
        out, a = [], 0
        for n in sizes:
            out.append((a, a + n))
            a += n
        return out

    def _decode_attention_host(self, running: List[GenerationTask]) -> None:
        """Host (pinned) Q/K/V in, host output out, pipelined per layer: the
        H2D copy of layer l+1's Q and the D2H copy of layer l-1's output run
        on their own streams (copy engines) under layer l's attention."""
        torch = self._torch
        geo = self.geometry
        model = self.model
        B = len(running)
        shape = (geo.num_layers, B, geo.num_heads, geo.head_dim)
        hp = self._host_pipeline(shape)
        st, h2d, d2h = self._stream, hp["h2d"], hp["d2h"]
        if model.host_out is None or tuple(model.host_out.shape) != shape:
            model.host_out = torch.empty(shape, dtype=torch.bfloat16, pin_memory=True)
        with torch.cuda.device(self._dev):
            # Copies start once this step's plan upload (on the engine stream,
            # after the previous step's append) has gone: the buffers are free
            # then, and the plan never queues behind this step's 50 MB of K/V
            # rows on the copy engine.
            hp["ev_start"].record(st)
            h2d.wait_event(hp["ev_start"])
            d2h.wait_event(hp["ev_start"])
            chunks = hp["chunks"]
            with torch.cuda.stream(h2d):
                for ci, (a, b) in enumerate(chunks):
                    hp["q"][a:b].copy_(model.q[a:b], non_blocking=True)
                    hp["ev_q"][ci].record(h2d)
                if model.k is not None and not self.attend_own_token:  # (appended before attention otherwise)
                    hp["k"].copy_(model.k, non_blocking=True)
                    hp["v"].copy_(model.v, non_blocking=True)
                    hp["ev_kv"].record(h2d)
            q, out = hp["q"], hp["out"]
            layer_elems = B * geo.num_heads * geo.head_dim
            qp, op, handle, sp = q.data_ptr(), out.data_ptr(), self._pool.handle, self._sp()
            for ci, (a, b) in enumerate(chunks):
                st.wait_event(hp["ev_q"][ci])
                _lib.check(_lib.lib.fk_attn_decode_layers(handle, a, b - a, ctypes.c_void_p(qp + a * layer_elems * 2),
                                                          layer_elems * 2, ctypes.c_void_p(op + a * layer_elems * 2),
                                                          layer_elems * 2, None, 0, sp))
                hp["ev_o"][ci].record(st)
                d2h.wait_event(hp["ev_o"][ci])
                with torch.cuda.stream(d2h):
                    model.host_out[a:b].copy_(out[a:b], non_blocking=True)
            hp["ev_d2h"].record(d2h)
            # the step completes with its output on the host: the engine stream
            # waits for the last output copy at the end of step(), so the K/V
            # append (enqueued after attention) runs under that copy
            self._pending_d2h = hp["ev_d2h"]
        self.last_output = out
        self.last_output_f32 = None
        self._last_running = running

    def _decode_attention(self, running: List[GenerationTask]) -> None:
        torch = self._torch
        model = self.model
        tensor_model = isinstance(model, TensorDecodeModel)
        if tensor_model and model.q.device.type != "cuda" and not self.capture_f32:
            self._decode_attention_host(running)
            return
        geo = self.geometry
        B = len(running)
        shape = (geo.num_layers, B, geo.num_heads, geo.head_dim)
        st = self._stream
        caller = self._caller  # (_caller_sync: the engine stream is past the caller's producers)
        # The step's buffers are allocated on the engine stream (so the caching
        # allocator never hands the engine memory another stream still uses).
        # (set_stream instead of the context managers: this is the per-step
        # host path.)
        torch.cuda.set_stream(st)
        # Engine-owned buffers hold `cap` >= B rows per layer (B rounded up to
        # a power of two): the pointers and layer strides the kernels get stay
        # the same while the batch moves, so the step's CUDA graph replays
        # without node updates (under a serving load B changes every step).
        cap = self._row_cap(B)
        row_bytes = geo.num_heads * geo.head_dim * 2
        try:
            if tensor_model:
                q = model.q
                if q.device.type != "cuda":
                    q = q.to(self._dev, non_blocking=True)
                q_stride = B * row_bytes
            else:  # synthetic queries into an engine-owned buffer (only the engine stream touches it)
                q = self.__dict__.get("_synth_q")
                if q is None or q.shape[1] != cap:
                    q = self._synth_q = torch.empty((geo.num_layers, cap, geo.num_heads, geo.head_dim),
                                                    dtype=torch.bfloat16, device=self._dev)
                _lib.check(_lib.lib.fk_synth_queries(self._pool.handle, self.model_seed, q.data_ptr(), cap, self._spv))
                q_stride = cap * row_bytes
            out = model.out if tensor_model else None
            if out is None or tuple(out.shape) != shape or out.dtype != torch.bfloat16 or out.device != self._dev:
                # engine-owned outputs: a ring of two, alternating with the
                # plan slots, so a step's graph sees the same pointers as the
                # step two before it (no node updates); last_output stays
                # valid until two steps later (pass TensorDecodeModel(out=...)
                # to own the buffer)
                ring = self.__dict__.setdefault("_out_ring", [None, None])
                i = self._ring_i = self.__dict__.get("_ring_i", 1) ^ 1
                full = ring[i]
                if full is None or full.shape[1] != cap:
                    full = ring[i] = torch.empty((geo.num_layers, cap, geo.num_heads, geo.head_dim),
                                                 dtype=torch.bfloat16, device=self._dev)
                out, out_stride = full[:, :B], cap * row_bytes
            else:
                out_stride = B * row_bytes
            f32 = torch.empty(shape, dtype=torch.float32, device=self._dev) if self.capture_f32 else None
            # every layer's queries are already on the device: one C call
            # replays the layers' kernels (fk_attn_decode_layers, a CUDA graph)
            _lib.check(_lib.lib.fk_attn_decode_layers(
                self._pool.handle, 0, geo.num_layers, q.data_ptr(), q_stride, out.data_ptr(), out_stride,
                f32.data_ptr() if f32 is not None else None, B * row_bytes * 2 if f32 is not None else 0, self._spv))
            self.last_output = out
            self.last_output_f32 = f32
            if tensor_model and model.copy_out:
                if model.host_out is None or tuple(model.host_out.shape) != shape:
                    model.host_out = torch.empty(shape, dtype=torch.bfloat16, pin_memory=True)
                model.host_out.copy_(out, non_blocking=True)
        finally:
            torch.cuda.set_stream(caller)
        self._last_running = running

    def _row_cap(self, B: int) -> int:
        """Rows of the engine-owned q/out buffers: B rounded up to a power of
        two, at least 64 (a batch that builds up request by request then
        never reallocates -- a reallocation costs milliseconds under a
        serving load), shrunk only when B falls below a quarter of it."""
        cap = self.__dict__.get("_cap", 0)
        if B > cap or 4 * B < cap:
            cap = self._cap = max(64, 1 << (B - 1).bit_length())
        return cap

    @property
    def last_rows(self) -> List[str]:
        """Request ids of the rows of last_output, in row order."""
        return [g.request_id for g in self._last_running]

    def _append(self, running: List[GenerationTask]) -> None:
        """The step's new K/V rows into their (page, slot), positions from
        fk_step_grow (still in _pos_buf)."""
        torch = self._torch
        _lib.check(_lib.lib.fk_step_commit(self._pool.handle, self._pos_buf, self._spv))
        model = self.model
        if isinstance(model, TensorDecodeModel) and model.k is not None and model.k.device.type == "cuda":
            # (the engine stream already waits for the caller: _caller_sync)
            geo = self.geometry
            _lib.check(_lib.lib.fk_append_kv_layers(self._pool.handle, 0, geo.num_layers,
                                                    model.k.data_ptr(), model.v.data_ptr(), self._spv))
        elif isinstance(model, TensorDecodeModel) and model.k is not None:
            geo = self.geometry
            with torch.cuda.device(self._dev), torch.cuda.stream(self._stream):
                k, v = model.k, model.v
                hp = getattr(self, "_hp", None)
                if (k.device.type != "cuda" and hp is not None and hp["shape"] == tuple(k.shape)
                        and not self.attend_own_token):
                    # copied in under this step's attention (_decode_attention_host)
                    self._stream.wait_event(hp["ev_kv"])
                    k, v = hp["k"], hp["v"]
                else:
                    k = k.to(self._dev, non_blocking=True)
                    v = v.to(self._dev, non_blocking=True)
                _lib.check(_lib.lib.fk_append_kv_layers(self._pool.handle, 0, geo.num_layers,
                                                        ctypes.c_void_p(k.data_ptr()),
                                                        ctypes.c_void_p(v.data_ptr()), self._sp()))
        else:
            _lib.check(_lib.lib.fk_synth_append(self._pool.handle, self.model_seed, self.model_k_scale,
                                                self._sp()))

    def _caller_sync(self) -> None:
        """Once per step: the engine stream waits for the caller's current
        stream (where a TensorDecodeModel's q/k/v were produced), and device
        model tensors are marked as used by the engine stream (caching
        allocator).  The attention and the append read them afterwards."""
        torch = self._torch
        raw = torch._C._cuda_getCurrentRawStream(self._dev_index)
        if raw != self._caller_raw:
            self._caller = torch.cuda.current_stream(self._dev)
            self._caller_raw = raw
        if raw == self._spv:
            return
        model = self.model
        if isinstance(model, TensorDecodeModel) and model.q.device.type == "cuda":
            self._ev_caller.record(self._caller)
            self._stream.wait_event(self._ev_caller)
            st = self._stream
            model.q.record_stream(st)
            if model.k is not None:
                model.k.record_stream(st)
                model.v.record_stream(st)
            if model.out is not None:
                model.out.record_stream(st)

    def _wait_fills(self, running: List[GenerationTask]) -> None:
        """The decode stream waits for the pending fills of the contexts this
        step reads (and only those: other fills keep overlapping decode)."""
        seen: Set[str] = set()
        for g in running:
            for c in self._ancestors(self.contexts.get(g.context_id)):
                if c.context_id in seen:
                    break
                seen.add(c.context_id)
                ev = self._fill_pending.pop(c.context_id, None)
                if ev is not None:
                    self._stream.wait_event(ev)
            if not self._fill_pending:
                break

    def _snapshot(self, running: List[GenerationTask]) -> List[List[Tuple[int, int]]]:
        """Per row: [(context uid, tokens)] root -> leaf at plan time."""
        rows = []
        for g in running:
            chain = [(c.uid, c.token_count) for c in self._ancestors(self.contexts.get(g.context_id))]
            rows.append(list(reversed(chain)))
        return rows

    def step(self) -> Optional[StepReport]:
        if not self.has_work():
            return None
        if _NVTX and self.device is not None:
            self._torch.cuda.nvtx.range_push(f"GpuEngine.step {self.engine_id}")
            try:
                return self._step()
            finally:
                self._torch.cuda.nvtx.range_pop()
        return self._step()

    def _step(self) -> Optional[StepReport]:
        if _PHASES:
            tm = [time.perf_counter()]
        started_ns = self.clock_ns
        emitted: Dict[str, int] = {}
        finished: List[str] = []
        failed: List[Tuple[str, str]] = []
        fill_completed: List[str] = []

        if self._zero_len:  # zero-length generations (engine.py:398-402)
            for g in list(self.gens.values()):
                if g.started and not g.done and not g.token_ids:
                    g.done = True
                    finished.append(g.request_id)
                    self._running = None
            self._zero_len = [g for g in self._zero_len if not g.done]

        fill_tokens = 0
        if self.fill_queue:  # one fill chunk per step, FIFO (engine.py:404-414)
            task = self.fill_queue.popleft()
            fill_tokens = len(task.token_ids)
            if task.request_id is not None:
                left = self.pending_fills.get(task.request_id, 0) - 1
                self.pending_fills[task.request_id] = left
                if left <= 0:
                    fill_completed.append(task.request_id)

        running = self._running_rows()
        if _PHASES:
            tm.append(time.perf_counter())
        batch_tokens = self._plan(running) if running else 0
        if _PHASES:
            tm.append(time.perf_counter())
        if running and self.device is not None:
            self._caller_sync()
            if self._fill_pending:
                self._wait_fills(running)
        snapshot = None
        emitted: Dict[str, int] = {}
        if self.attend_own_token:
            # real-decoder order: grow (the plan already did, fk_step_plan
            # under FK_OPT_APPEND_FIRST), write the new K/V rows, then attend
            # over spans that include them
            if running:
                emitted = self._grow_rows(running, finished, failed)
            snapshot = self._snapshot(running) if (self.keep_history and running) else None
            if running and self.device is not None:
                self._append(running)
                self._decode_attention(running)
        else:
            snapshot = self._snapshot(running) if (self.keep_history and running) else None
            if running and self.device is not None:
                self._decode_attention(running)
        if running and self.device is not None:
            self.kv_tokens_streamed += int(self.last_plan.streamed_tokens)
        if _PHASES:
            tm.append(time.perf_counter())

        elapsed = 0
        if fill_tokens > 0:
            part = self.cost.fill_ns(fill_tokens)
            elapsed += part
            self.fill_ns_total += part
        if running:
            part = self.cost.iteration_ns(batch_tokens)
            elapsed += part
            self.decode_ns_total += part
        self.clock_ns += elapsed
        self.busy_ns += elapsed

        if not self.attend_own_token and running:
            emitted = self._grow_rows(running, finished, failed)
            if self.device is not None:
                self._append(running)

        if self.__dict__.get("_pending_d2h") is not None:
            self._stream.wait_event(self._pending_d2h)
            self._pending_d2h = None
        if _PHASES:
            tm.append(time.perf_counter())
        for rid in fill_completed:  # fills done this step decode next step
            g = self.gens.get(rid)
            if g is not None and not g.started:
                g.started = True
                self._running = None

        self.total_emitted += len(emitted)
        self.trace.append("t=%s engine=%s fill=%d batch=%d emitted=%d"
                          % (format_ms(self.clock_ns), self.engine_id, fill_tokens, batch_tokens, len(emitted)))
        report = StepReport(self.engine_id, started_ns, elapsed, fill_tokens, batch_tokens, emitted,
                            finished, failed, fill_completed)
        self.reports.append(report)
        if snapshot is not None:
            positions = [int(self._pos_buf[i]) for i in range(len(running))]
            self.history.append(self._history_record(running, snapshot, batch_tokens, positions))
        if _PHASES:  # per-step host microseconds of each phase (the plan includes its GPU wait)
            tm.append(time.perf_counter())
            self.__dict__.setdefault("phase_steps", []).append(
                {k: (tm[i + 1] - tm[i]) * 1e6 for i, k in enumerate(("pre", "plan", "attention", "grow_append", "post"))})
        return report

    def _running_rows(self) -> List[GenerationTask]:
        """Started, not done, in gens order (engine.py:416) -- cached until the
        set changes.  A generation's first decode iteration fixes where it
        finishes on the decode counter (one token per iteration)."""
        run = self._running
        if run is None:
            run = [g for g in self.gens.values() if g.started and not g.done]
            t = self._dclock[0]
            for g in run:
                if g._t0 < 0:
                    g._t0 = t
                    self._finish_at.setdefault(t + len(g.token_ids) - g._base, []).append(g)
            self._running = run
            self._running_rids = [g.request_id for g in run]
        return run

    def _grow_rows(self, running: List[GenerationTask], finished: List[str],
                   failed: List[Tuple[str, str]]) -> Dict[str, int]:
        """One token per running generation, gens order, sequential OOM rule
        (engine.py:431-443), in one C call; returns StepReport.emitted.  Token
        counts and block ids live in the pool, emitted counts derive from the
        decode counter: only failing and finishing rows are touched here."""
        nf = self._nfail
        _lib.check(_lib.lib.fk_step_grow(self._pool.handle, self._pos_buf, self._id_buf, ctypes.byref(nf)))
        t = self._dclock[0]
        if nf.value:
            for i, g in enumerate(running):
                if self._pos_buf[i] < 0:  # OutOfMemory: only this request fails (PagedKvStore.grow message)
                    ctx = self.contexts[g.context_id]
                    need = self.store.blocks_for(ctx.token_count + 1) - len(ctx.block_ids)
                    g.done = True
                    g._t_end = t
                    failed.append((g.request_id, f"engine {ctx.engine_id}: need {need} blocks, "
                                                 f"{self.store.free_blocks} free"))
            emitted = {g.request_id: 1 for g in running if g._t_end < 0}
            self._running = None
        else:
            emitted = dict.fromkeys(self._running_rids, 1)
        self._dclock[0] = t + 1
        fin = self._finish_at.pop(t + 1, None)
        if fin:
            live = [g for g in fin if not g.done and self.gens.get(g.request_id) is g]
            if len(live) > 1:
                order = {id(g): i for i, g in enumerate(running)}
                live.sort(key=lambda g: order.get(id(g), len(order)))
            for g in live:
                g.done = True
                g._t_end = t + 1
                finished.append(g.request_id)
            if live:
                self._running = None
        return emitted

    def _history_record(self, running, snapshot, batch_tokens, positions) -> Dict[str, Any]:
        """Snapshot for the parity tests: the outputs are copied to the host on
        the engine stream, i.e. after this step's kernels."""
        def host(t):
            if t is None:
                return None
            with self._torch.cuda.stream(self._stream):
                return t.detach().to("cpu", copy=True)

        return {
            "rows": [g.request_id for g in running],
            "chains": snapshot,
            "leaf_uid": [self.contexts[g.context_id].uid if g.context_id in self.contexts else -1
                         for g in running],
            "batch_tokens": batch_tokens,
            "streamed_tokens": int(self.last_plan.streamed_tokens),
            # leaf tokens before this step's growth: the synthetic query key
            "qpos": [int(self._leaf_pos0[i]) for i in range(len(running))],
            "output": host(self.last_output),
            "output_f32": host(self.last_output_f32),
            "positions": positions,
        }

    # -- request lifecycle (engine.py:488-538) -------------------------------------

    def _forget(self, g: GenerationTask) -> None:
        """A generation leaves gens: freeze its emitted count, drop it from
        the running rows."""
        if g._t0 >= 0 and g._t_end < 0:
            g._t_end = self._dclock[0]
        self._running = None

    def finish_generation(self, request_id: str) -> Optional[int]:
        g = self.gens.pop(request_id, None)
        if g is None:
            return None
        self._forget(g)
        for d in (self.pending_fills, self.charges, self.holder_class, self.request_leaf):
            d.pop(request_id, None)
        ctx = self.contexts.get(g.context_id)
        if ctx is None:
            return None
        ctx.refcount -= 1
        if ctx.refcount == 0 and ctx.dropped:
            self._discard_context(ctx)
            return None
        if not g.token_ids:
            return None
        seed = ctx.chain_hashes[-1] if ctx.chain_hashes else FNV64_EMPTY
        end_hash = hash_token_ids(g.token_ids[: g.emitted], seed)
        ctx.chain_hashes.append(end_hash)
        if end_hash not in self.registry:
            self.registry[end_hash] = ctx.context_id
            ctx.registered_hashes.append(end_hash)
        return end_hash

    def cancel_request(self, request_id: str) -> None:
        self.fill_queue = deque(t for t in self.fill_queue if t.request_id != request_id)
        for d in (self.pending_fills, self.charges, self.holder_class, self.request_leaf):
            d.pop(request_id, None)
        g = self.gens.pop(request_id, None)
        if g is None:
            return
        self._forget(g)
        ctx = self.contexts.get(g.context_id)
        if ctx is not None:
            ctx.refcount -= 1
            ctx.dropped = True
            if ctx.refcount == 0:
                self._discard_context(ctx)

# Alias so a maintainer can rebind `semflow.engine.Engine = Engine`.
Engine = GpuEngine


def engine_factory(geometry: ModelGeometry = LLAMA_13B, devices: Optional[Sequence[int]] = None,
                   migrate_prefixes: bool = False, **kw):
    """A constructor with `Engine`'s signature for SemanticManager's one
    construction site (manager.py:130-139: `Engine(eid, cost, kv_tokens=...,
    token_capacity=...)` for eid = e0 .. e{engines-1}), mapping engine eI to
    GPU devices[I mod len(devices)] (default: every visible GPU), so
    `Config(engines=N)` spreads the prefix-affinity scheduler's groups
    (scheduler.py:198-222) over the GPUs of one process.  Extra keyword
    arguments (model, capture_f32, keep_history, ...) go to every GpuEngine;
    devices=[] builds host-only engines (the integer twin).
    migrate_prefixes=True: the engines fill a prefix another engine of the
    process already holds by copying its K/V (GpuEngine._peer_prefix) --
    the `shared-ctx` fallback of the scheduler then costs an NVLink copy
    instead of a prefill.

        import semflow.manager
        semflow.manager.Engine = engine_factory(LLAMA_13B)
    """
    if devices is None:
        import torch

        devices = list(range(torch.cuda.device_count()))
    devices = list(devices)

    peers: Optional[List[GpuEngine]] = [] if migrate_prefixes else None

    def make(engine_id: str, cost: Any, kv_tokens: int = 120_000, token_capacity: int = 64_000) -> GpuEngine:
        digits = engine_id.lstrip("e")
        idx = int(digits) if digits.isdigit() else 0
        dev = devices[idx % len(devices)] if devices else None
        eng = GpuEngine(engine_id, cost, kv_tokens, token_capacity, device=dev, geometry=geometry, peers=peers, **kw)
        if peers is not None:
            peers.append(eng)
        return eng

    make.devices = devices
    make.peers = peers
    return make
