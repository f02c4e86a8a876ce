/*
 * forkattn.h — C-ABI of the B200 shared-prefix ("fork") decode-attention path.
 *
 * This is the drop-in boundary below the reference engine's Python surface
 * (semflow.engine.Engine, /root/reference/pkg/src/semflow/engine.py).  A
 * reference maintainer binds it with ctypes; the host
 * mirror in paper_2405_19888_b200/engine.py is exactly that binding.
 *
 * Ownership: one fk_pool per engine / per GPU owns the device KV arena, the
 * physical page free list, the logical block-id counter, the context forest
 * topology and the per-step plan.  Q / K / V / output buffers are caller
 * owned device pointers; `stream` is a cudaStream_t passed as void*.
 *
 * Threading: not thread-safe per pool; the caller serialises (the reference
 * manager holds its RLock around every engine call, manager.py:99-109).
 *
 * Every entry point returns an fk_status; on failure no state changed
 * (allocation is atomic like PagedKvStore.grow, engine.py:87-100) and
 * fk_last_error() holds a message.
 */
#ifndef FORKATTN_H
#define FORKATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The Python shim maps 1..4 onto semflow.errors
 * OutOfMemory / UnknownContext / UnknownParentContext / ContextBusy
 * (errors.py:71-84), whose .code feeds the HTTP map (api.py:37-56). */
typedef enum {
  FK_OK = 0,
  FK_OUT_OF_MEMORY = 1,
  FK_UNKNOWN_CONTEXT = 2,
  FK_UNKNOWN_PARENT_CONTEXT = 3,
  FK_CONTEXT_BUSY = 4,
  FK_INVALID_ARGUMENT = 5,
  FK_CUDA_ERROR = 6,
  FK_NO_DEVICE = 7 /* compute entry point called on a host-only pool */
} fk_status;

typedef struct fk_pool fk_pool;

typedef struct {
  int32_t num_layers;   /* L */
  int32_t num_heads;    /* H (KV heads == query heads; MHA like LLaMA-7B/13B) */
  int32_t head_dim;     /* D; the kernels are specialised for 128 */
  int32_t block_size;   /* tokens per page; Config.block_size (config.py:21), must be 16 */
  int64_t total_blocks; /* logical capacity = PagedKvStore.total_blocks (engine.py:71) */
  int64_t num_pages;    /* physical pages in the device arena (>= total_blocks for
                           bit-exact OOM behaviour); ignored when device < 0 */
  int32_t device;       /* CUDA ordinal; -1 = host-only accounting (CPU tests) */
  int32_t reserved;
} fk_pool_desc;

typedef struct {
  int64_t used_blocks;  /* PagedKvStore.used_blocks  (engine.py:77-78) */
  int64_t free_blocks;  /* PagedKvStore.free_blocks  (engine.py:81-82) */
  int64_t peak_used;    /* PagedKvStore.peak_used    (engine.py:73,99-100) */
  int64_t total_blocks; /* PagedKvStore.total_blocks (engine.py:71) */
  int64_t next_block;   /* next logical id of itertools.count() (engine.py:74) */
  int64_t num_pages;    /* physical pages in the arena (0 when host-only) */
  int64_t free_pages;   /* physical pages on the free stack */
  int64_t arena_bytes;  /* device bytes of the KV arena */
  int64_t host_wait_ns; /* host time fk_step_plan spent waiting for the GPU to release a plan
                           slot (the host runs at most one step ahead) */
  int64_t graph_replays; /* fk_attn_decode_layers calls that replayed a cached CUDA graph
                            without recording (nothing the launches depend on changed) */
} fk_pool_stats;

/* Per-step plan summary returned by fk_step_plan. */
typedef struct {
  int64_t batch_tokens;    /* == Engine._batch_tokens(running) (engine.py:470-484) */
  int64_t shared_tokens;   /* tokens of contexts with fan-out >= 2 (streamed once) */
  int64_t private_tokens;  /* tokens of contexts with fan-out 1 */
  int32_t num_rows;        /* B, running requests in gens order */
  int32_t num_shared_ctx;  /* unique shared contexts */
  int32_t num_prefix_ctas; /* prefix work items (context x split x query block) */
  int32_t max_slots;       /* partial slots per (row, head) incl. the private one */
  int32_t num_tc_items;    /* prefix items routed to the tcgen05 kernel */
  int32_t num_mma_items;   /* prefix items routed to the warp-level mma.sync kernel */
  int32_t fused_merge;     /* always 0 since round 2 (the fused merge was removed: every
                              launch merges with fk_merge_kernel) */
  int64_t streamed_tokens; /* KV tokens the kernels stream per layer: batch_tokens, plus the
                              step's new tokens under FK_OPT_APPEND_FIRST */
} fk_plan_info;

/* ---- pool ---------------------------------------------------------------- */
/* Replaces PagedKvStore.__init__ (engine.py:69-74) + the device KV arena.
 * A process holds at most 64 device pools at a time (each owns two
 * __constant__ plan slots); the 65th fails with FK_INVALID_ARGUMENT until
 * one is destroyed.  Host-only pools (device -1) are unlimited. */
int fk_pool_create(const fk_pool_desc* desc, fk_pool** out);
int fk_pool_destroy(fk_pool* pool);
/* manager.py:138 writes store.total_blocks after construction. */
int fk_pool_set_total_blocks(fk_pool* pool, int64_t total_blocks);
/* Grow the physical arena (copies live pages); never shrinks. */
int fk_pool_reserve_pages(fk_pool* pool, int64_t num_pages);
int fk_pool_stats_get(const fk_pool* pool, fk_pool_stats* out);
/* Tuning knobs: FK_OPT_* below. */
int fk_pool_set_option(fk_pool* pool, int32_t option, int64_t value);
const char* fk_last_error(void);

enum {
  FK_OPT_TC_MIN_FANOUT = 1,   /* fan-out at/above which prefix items use tcgen05 (0 = never) */
  FK_OPT_PREFIX_TARGET_CTAS = 2, /* prefix split target (default: 1 wave of SMs) */
  FK_OPT_LAUNCH_ORDER = 3,    /* 0 prefix->private (default), 1 private->prefix (tests merge paths) */
  FK_OPT_MIN_SPLIT_PAGES = 4, /* minimum pages per prefix split */
  FK_OPT_CORUN = 5,           /* 1 (default): tcgen05 prefix CTAs and the private stream split the
                                 SMs and run concurrently; 0: each kernel gets every SM in turn */
  FK_OPT_PREFIX_RATE_PCT = 6, /* co-run SM split: prefix per-SM KV rate relative to the private
                                 stream's, in percent (default 50) */
  FK_OPT_PDL = 7,             /* programmatic dependent launch: 0 plain stream order; 1 (default)
                                 between one layer's kernels; 2 also lets a layer's first kernel
                                 start under the previous layer's merge -- only when q is not
                                 written by the kernel launched right before fk_attn_decode */
  FK_OPT_PRIV_MIN_CHUNK = 8,  /* smallest chunk (pages) of the private kernel's guided dynamic
                                 schedule, 1..32: the granularity of its tail; 0 (default): 2, or
                                 for plans under 32K (head, page) units with no prefix grid (a
                                 few rows) 4..8, fitted to the last round of chunks */
  FK_OPT_PRIV_STATIC_FIRST = 9, /* 1 (default): the private warps that start at once take their
                                 first chunk by warp index instead of a ticket */
  FK_OPT_PRIV_WARPS = 11,     /* private CTA shape: 10 warps x 2 stages (default), 8 x 3 or 12 x 2 */
  FK_OPT_GRAPH = 12,          /* 1 (default): fk_attn_decode_layers replays its launches as a CUDA
                                 graph (captured once per launch structure, parameters updated in
                                 place afterwards); 0: direct launches */
  FK_OPT_TC_BOUNDARY_COST = 14, /* static split: tiles a piece start mid-range costs a CTA (default 12) */
  /* 10, 13 (tcgen05 dynamic tail) and 15 (fused merge) were removed in round 2:
     measured slower than what they replace; setting them fails */
  FK_OPT_APPEND_FIRST = 16,   /* 1: attend to the step's own token (a real decoder): fk_step_plan does
                                 the step's one-token growth (row order, sequential OOM rule) and
                                 plans spans that include it; the caller then takes the growth from
                                 fk_step_grow, commits and appends the new K/V rows, and only then
                                 runs fk_attn_decode.  fk_plan_info.batch_tokens stays the
                                 reference's pre-growth count.  0 (default): the reference's span
                                 (chain tokens at step start, engine.py:416-434), append after */
  FK_OPT_GROUP_FANOUT = 18,   /* shared contexts read by <= this many rows (0..64, default 8) are
                                 streamed by the private kernel once per group of up to 8 rows -- the
                                 rows are the N of its transposed m16n8 products -- instead of by a
                                 prefix kernel (default CTA shape only); 0 = off */
  FK_OPT_DEBUG_SKIP_MERGE = 90 /* diagnostic only: 1 = do not launch the LSE merge (outputs are NOT
                                 written); bounds the time the merge adds to a layer */
};

/* ---- context forest ------------------------------------------------------ */
/* Engine.create_context (engine.py:201-223): topology only (refcounts, the
 * dropped flag and the hash registry stay in the Python mirror). */
int fk_ctx_create(fk_pool* pool, int64_t ctx, int64_t parent /* -1 = root */);
/* PagedKvStore.grow (engine.py:87-100): extend ctx to new_token_count tokens,
 * need = ceil(new/bs) - len(blocks); atomic FK_OUT_OF_MEMORY if need > free.
 * Writes the new logical ids (itertools.count order) to new_ids[0..n). */
int fk_ctx_grow(fk_pool* pool, int64_t ctx, int64_t new_token_count,
                int64_t* new_ids, int64_t cap, int64_t* n_new);
/* PagedKvStore.release + forest removal (engine.py:102-106, 273-285).
 * FK_CONTEXT_BUSY while the context still has children in the forest. */
int fk_ctx_release(fk_pool* pool, int64_t ctx);
int fk_ctx_info(const fk_pool* pool, int64_t ctx, int64_t* token_count,
                int64_t* num_blocks, int64_t* parent);
/* Token count of ctx (Context.token_count, engine.py:53-63), or -1 if unknown:
 * the pool is authoritative, the Python mirror reads it on demand. */
int64_t fk_ctx_tokens(const fk_pool* pool, int64_t ctx);
/* Parity readback: logical ids and the physical pages backing them. */
int fk_ctx_blocks(const fk_pool* pool, int64_t ctx, int64_t* logical,
                  int32_t* physical, int64_t cap, int64_t* n);

/* ---- decode step --------------------------------------------------------- */
/* Engine.step decode half (engine.py:416-417, 470-484): build the work list
 * for the running leaves (gens order) and upload it on `stream`.  dedup=1 is
 * CostModel.shared_kernel=True (shared contexts streamed once for all their
 * descendants); dedup=0 streams every request's whole chain.
 * Stream order: `stream` must be the stream the plan's attention runs on (or
 * be ordered before it): the upload, and any growth of the partial buffers
 * (stream-ordered allocation, no device sync), are enqueued there.  The host
 * runs at most one plan ahead: the call blocks until the GPU has finished
 * with the plan slot it reuses (two slots, host_wait_ns). */
int fk_step_plan(fk_pool* pool, const int64_t* leaves, int32_t num_rows,
                 int32_t dedup, void* stream, fk_plan_info* info);
/* Decode attention for one layer over the current plan.
 * q   : [num_rows][H][D] bf16 (device)
 * out : [num_rows][H][D] bf16 (device)
 * out_f32 : optional [num_rows][H][D] fp32 pre-cast merge output (NULL = off)
 * Span = chain tokens at plan time (the reference counts batch_tokens before
 * growth, engine.py:416-434). */
int fk_attn_decode(fk_pool* pool, int32_t layer, const void* q, void* out,
                   float* out_f32, void* stream);
/* fk_attn_decode for layers [layer0, layer0 + nlayers) in one call, when the
 * queries of several layers are ready at once (layer i reads
 * q + i * q_layer_stride bytes, writes out + i * out_layer_stride); the
 * kernels and their ordering are exactly those of the per-layer calls.
 * Replayed as a CUDA graph (FK_OPT_GRAPH): a call whose pointers, strides,
 * plan slot and launch shapes repeat relaunches the cached graph without
 * recording; keeping q/out buffers and strides stable from step to step is
 * what makes that happen. */
int fk_attn_decode_layers(fk_pool* pool, int32_t layer0, int32_t nlayers, const void* q,
                          int64_t q_layer_stride, void* out, int64_t out_layer_stride, float* out_f32,
                          int64_t f32_layer_stride, void* stream);
/* The one-token growth of every planned row, in row (gens) order, with the
 * sequential OOM rule of engine.py:431-438: positions[r] = token index of
 * row r's new token, or -1 if its grow failed (OutOfMemory: that request
 * fails, the others continue); new_ids[r] = the logical block id the grow
 * allocated, or -1; *n_failed = rows whose grow failed.  Host-only pools use
 * it too (no device work). */
int fk_step_grow(fk_pool* pool, int64_t* positions, int64_t* new_ids, int32_t* n_failed /* nullable */);
/* After the Python mirror grew each leaf by one token (engine.py:431-438):
 * positions[r] = slot index (token count before the grow) of row r's new
 * token, or -1 when that grow failed (OOM).  Uploads append targets. */
int fk_step_commit(fk_pool* pool, const int64_t* positions, void* stream);
/* Write the step's new K/V rows ([num_rows][H][D] bf16 each) for one layer
 * into their (page, slot) targets; rows with position -1 are skipped. */
int fk_append_kv(fk_pool* pool, int32_t layer, const void* k, const void* v,
                 void* stream);
/* Same for layers [layer0, layer0 + nlayers) in one launch: k/v are
 * [nlayers][num_rows][H][D] bf16. */
int fk_append_kv_layers(fk_pool* pool, int32_t layer0, int32_t nlayers,
                        const void* k, const void* v, void* stream);

/* ---- fill (prefill KV content) ------------------------------------------- */
/* The KV half of Engine.fill (engine.py:225-255; the paper's Fill "calculates
 * and fills the KV cache"): write caller K/V rows for tokens
 * [pos0, pos1) of ctx (already grown by fk_ctx_grow) into its pages, for
 * layers [layer0, layer0 + nlayers).  k, v: [nlayers][pos1 - pos0][H][D] bf16
 * (device).  The copy is stream-ordered; the host pointers may be reused
 * once `stream` has passed it. */
int fk_fill_kv(fk_pool* pool, int64_t ctx, int64_t pos0, int64_t pos1, int32_t layer0, int32_t nlayers,
               const void* k, const void* v, void* stream);

/* ---- prefix migration -------------------------------------- */
/* Copy the KV of tokens [0, ntok) of src_ctx (in pool `src`, possibly on
 * another GPU) into dst_ctx of pool `dst` (already grown to >= ntok tokens),
 * all layers.  Across devices the copy kernel runs on dst's GPU and reads
 * src's arena over NVLink peer access (enabled on first use).  Lets a fork
 * group land on a GPU that does not hold its shared prefix without
 * re-running prefill (scheduler.py:217-221 `shared-ctx` restriction). */
int fk_ctx_copy_kv(fk_pool* dst, int64_t dst_ctx, const fk_pool* src, int64_t src_ctx, int64_t ntok,
                   void* stream);

/* ---- synthetic model (deterministic KV / Q; the oracle restates it) ------ */
/* Fill tokens [pos0, pos1) of ctx for every layer/head with the counter-hash
 * generator.  k_scale multiplies K (stress). */
int fk_synth_fill(fk_pool* pool, int64_t ctx, int64_t pos0, int64_t pos1,
                  uint64_t seed, float k_scale, void* stream);
/* Q rows for the current plan: q_all[L][rows_cap][H][D] bf16 (rows_cap >=
 * num_rows; 0 = num_rows), row r keyed by (leaf uid, leaf tokens at plan
 * time, rank of r among rows on that leaf). */
int fk_synth_queries(fk_pool* pool, uint64_t seed, void* q_all, int32_t rows_cap, void* stream);
/* Append the step's synthetic K/V rows (keyed by (leaf uid, position)) for
 * all layers, using the targets of fk_step_commit. */
int fk_synth_append(fk_pool* pool, uint64_t seed, float k_scale, void* stream);

/* ---- hashing ------------------------------------------------------------- */
/* tokenizer.hash_token_ids (tokenizer.py:47-49): FNV-1a-64 over the
 * little-endian u32 bytes of each id, chained from `seed`. */
uint64_t fk_fnv1a64_u32(const uint32_t* ids, size_t n, uint64_t seed);
/* Chain hashes of consecutive segments (prefix.py:78-85): out[i] = hash of
 * segment i seeded with out[i-1] (seed for i=0). seg_off has nseg+1 entries. */
int fk_fnv1a64_chain(const uint32_t* ids, const int64_t* seg_off, int32_t nseg,
                     uint64_t seed, uint64_t* out);

/* Library identification (for the driver's loaded-.so evidence). */
const char* fk_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* FORKATTN_H */
