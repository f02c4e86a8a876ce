// Host side of the fork-attention pool: logical block accounting (bit-exact
// with PagedKvStore, engine.py:66-106), physical page free stack, context
// forest topology, per-step work-list planning and the C-ABI entry points of
// include/forkattn.h.
#include "forkattn.h"
#include "fk_internal.h"

#include <cuda_bf16.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <mutex>
#include <tuple>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

using namespace fk;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define FK_CUDA(expr)                                                        \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess)                                                   \
      return fail(FK_CUDA_ERROR, "%s: %s (%s:%d)", #expr,                    \
                  cudaGetErrorString(_e), __FILE__, __LINE__);               \
  } while (0)

struct Ctx {
  int64_t parent = -1;
  Ctx* par = nullptr;  // the parent's node (unordered_map nodes never move; a parent outlives its children)
  int64_t tokens = 0;
  int32_t children = 0;
  std::vector<int64_t> logical;  // logical block ids (itertools.count order)
  std::vector<int32_t> phys;     // physical pages backing them
  // planner state, valid while mark == the pool's plan epoch
  uint32_t mark = 0;
  int32_t fan = 0;      // rows whose chain holds this context
  int32_t sidx = -1;    // index among the step's shared contexts, or -1
  int32_t gidx = -1;    // index among the step's grouped (small fan-out) contexts, or -1
  int32_t rank = 0;     // rows planned so far with this context as their leaf
  bool shared = false;  // fan-out >= 2 with tokens (dedup mode)
};

// Planner scratch, reused from step to step (fk_step_plan).
struct PlanItem {
  int sh, split, q0, nq, head, page0, npages, ntok, units;
};
struct PlanShared {
  Ctx* ctx;
  int nrows = 0;   // descendant rows (at srows[row0 ..], row order)
  int row0 = 0;
  int seen = 0;
  bool tc = false;
  int splits = 1;  // mma path: head-independent page splits
  int page_off = 0;
  int q_off = 0;
};
struct PlanScratch {
  std::vector<Ctx*> chain, order;
  std::vector<int32_t> chain_off, srows, pages, page_ntok, qrows, it_unit_off, ch_item, ch_t0, ch_t1, cta_chunk0,
      it_first_chunk, pieces_of, rs_off, rs_sh, rs_qb, row_head_base, base_at, it_qslot_off, qslot, row_priv_off,
      row_priv_np, row_unit_off, page_item, chunk_start, row_head_count, item_chunk0, srow_e, acc, pit_e0, pit_np,
      pit_roff, pit_nrows, pit_rows, grow_cnt, grows, gfill, item_slot, item_pieces;
  std::vector<int64_t> leaf_tokens_pre, cut, cut0, qb_off, row_uid, row_pos;
  int64_t n_chunks = 0;  // chunk_start holds n_chunks + 1 entries in use
  std::vector<PlanShared> shared;
  std::vector<PlanItem> items;
};

// One plan slot: pinned staging + device copy + the event that guards reuse.
struct PlanSlot {
  void* host = nullptr;
  void* dev = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
  bool armed = false;
};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Switches the calling thread to a pool's device and restores the caller's
// device on scope exit, so engines on several GPUs can share a process
// without moving each other's (or torch's) current device.
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};
#define FK_ON_DEVICE(dev)                                                                   \
  DeviceGuard device_guard_(dev);                                                           \
  if (device_guard_.err != cudaSuccess)                                                     \
    return fail(FK_CUDA_ERROR, "cudaSetDevice(%d): %s", (int)(dev), cudaGetErrorString(device_guard_.err))

}  // namespace

// A step's attention launches as one CUDA graph: captured the first time a
// launch structure is seen, afterwards only its kernel-node parameters are
// updated (the structure -- functions, grids, PDL edges -- stays).
// Everything the recorded launches of fk_attn_decode_layers depend on
// (functions, grids, argument bytes): when it repeats, the cached graph is
// replayed without re-recording.  FK_DEBUG_GRAPH_CHECK=1 records anyway and
// fails if the launches differ (tests/test_gpu_manager.py).
struct ReplayKey {
  const void* kv;
  int64_t num_pages;
  const void *part_o, *part_ml, *tick;
  size_t part_cap;
  const void *q, *out, *out_f32;
  int64_t q_stride, out_stride, f32_stride;
  int32_t tc_begin, num_items, tc_grid, tc_ctas, priv_any, priv_wpc, priv_grid, num_sms, pdl, launch_order, plan_slot;
  int32_t wide_merge, grouped;  // (grouped: the private kernel's row-group instantiation)
};
static_assert(sizeof(ReplayKey) % 8 == 0, "ReplayKey is compared bytewise");

struct GraphCache {
  ReplayKey key{};
  bool key_ok = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaGraphNode_t> nodes;   // kernel nodes in launch order
  std::vector<fk::LaunchRec> shape;     // structure of the captured launches (no argument bytes)
  cudaStream_t stream = nullptr;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    nodes.clear();
    shape.clear();
    key_ok = false;
  }
};

struct fk_pool {
  fk_pool_desc desc{};
  bool on_device = false;
  std::unordered_map<int64_t, Ctx> ctxs;
  int64_t next_logical = 0;
  int64_t used = 0;
  int64_t peak = 0;
  int64_t total_blocks = 0;
  std::vector<int32_t> free_pages;  // stack, back() is the next page
  int64_t num_pages = 0;

  // device arena
  __nv_bfloat16* kv = nullptr;
  size_t arena_bytes = 0;
  alignas(64) CUtensorMap tmap;      // box {64 dims, 16 rows}: one page
  alignas(64) CUtensorMap tmap_run;  // box {64 dims, 128 rows}: 8 contiguous pages
  alignas(64) CUtensorMap tmap_half; // box {64 dims, 8 rows}: the first half of a page
  bool tmap_ok = false;
  int num_sms = 148;

  // options
  int64_t tc_min_fanout = 2;  // tcgen05 for every shared context (measured faster than mma.sync at fan-out 2..32)
  int64_t prefix_target_ctas = 0;  // 0 -> num_sms
  int64_t launch_order = 0;
  int64_t priv_min_chunk = 0;  // smallest private chunk (pages), the tail granularity; 0: auto (see the planner)
  int64_t priv_wpc = kPrivWarpsPerCta;  // private CTA shape (warps; stages follow)
  int64_t priv_static_first = 1;  // private warps that start at once take chunk = warp index (no ticket)
  int64_t tc_boundary_cost = 12;  // tiles a piece start mid-range costs a tcgen05 CTA (static split; 12 measured
                                  // +0.5..1.4 % over 4 at 13B/7B x 64 and nested, neutral elsewhere)
  int64_t pdl = 1;  // PDL: 1 between a layer's kernels, 2 also into the next layer's
  int64_t use_graph = 1;  // fk_attn_decode_layers replays a CUDA graph
  std::map<std::tuple<int32_t, int32_t, cudaStream_t, int>, GraphCache> graphs;  // (layer0, nlayers, stream, slot/half)
  fk::RecBuf rec_buf;  // launches recorded by fk_attn_decode_layers (storage reused)
  PlanScratch ps;                   // planner scratch (capacity reused across steps)
  uint32_t plan_epoch = 0;
  int64_t min_split_pages = 8;
  int64_t corun = 1;             // tcgen05 prefix and private stream share the SMs spatially
  int64_t prefix_rate_pct = 50;  // prefix KV bytes/s per SM relative to the private stream's (measured optimum, headline)

  // plan (host mirror + device)
  PlanSlot slots[2];
  int cur = -1;
  PlanDev plan{};
  bool have_plan = false;
  std::vector<int64_t> plan_leaves;
  std::vector<int64_t> plan_leaf_tokens;  // leaf tokens at plan time
  size_t off_app_page = 0, off_app_slot = 0, off_app_pos = 0;
  bool committed = false;

  // scratch
  float* part_o = nullptr;
  float2* part_ml = nullptr;
  size_t part_cap = 0;     // entries (rows*slots*H) per half
  int launch_parity = 0;   // which half of the partials the next fk_attn_decode uses
  int64_t host_wait_ns = 0;  // time fk_step_plan blocked on the GPU (plan slot reuse)
  int64_t graph_replays = 0; // fk_attn_decode_layers calls replayed without recording
  int64_t skip_merge = 0;    // FK_OPT_DEBUG_SKIP_MERGE (diagnostic)
  int64_t append_first = 0;  // FK_OPT_APPEND_FIRST: fk_step_plan grows the rows first (attend own token)
  int64_t group_fanout = 8;  // FK_OPT_GROUP_FANOUT: shared contexts with <= this many rows go to the private kernel
                             // (measured: faster than tcgen05 up to 8 forks, slower at 16)
  bool plan_grew = false;    // the current plan already did the step's growth (fk_step_grow returns it)
  std::vector<int64_t> grow_pos, grow_ids;
  unsigned* tick = nullptr;  // device: private chunk tickets, one counter per partial half
  int plan_base = -1;        // first of this pool's two __constant__ plan slots (fk_plan_c)
  int priv_grid = 0;         // private grid (CTAs) of the current plan
  int tc_grid = 0;           // tcgen05 prefix grid, kept while the plan's CTA count moves a little
  uint64_t plan_digest = 0;  // FK_DEBUG_PLAN_DIGEST: hash of the last plan's arrays

  ArenaDev arena() const {
    ArenaDev a;
    a.kv = kv;
    a.num_pages = num_pages;
    a.num_layers = desc.num_layers;
    a.num_heads = desc.num_heads;
    a.part_o = part_o;
    a.part_ml = part_ml;
    a.tick = tick;
    return a;
  }
};

namespace {

// NVTX ranges around the host entry points of the step (SURVEY §5 tracing):
// `ncu --nvtx --nvtx-include "fk_attn_decode_layers/"` selects one call's
// kernels, a timeline tool shows plan / attention / growth / append per step.
// (Push/pop cost a few ns without a tool attached.)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* name, int64_t payload) {
    nvtxEventAttributes_t e = {};
    e.version = NVTX_VERSION;
    e.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    e.messageType = NVTX_MESSAGE_TYPE_ASCII;
    e.message.ascii = name;
    e.payloadType = NVTX_PAYLOAD_TYPE_INT64;
    e.payload.llValue = payload;
    nvtxRangePushEx(&e);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

int64_t blocks_for(int64_t tokens, int64_t bs) { return (tokens + bs - 1) / bs; }

// FNV-1a over every array and scalar a plan uploads (FK_DEBUG_PLAN_DIGEST=1):
// pins the planner's output across rewrites (tests/test_plan.py).
bool plan_digest_on() {
  static const bool on = getenv("FK_DEBUG_PLAN_DIGEST") != nullptr;
  return on;
}
struct PlanDigest {
  uint64_t h = 0xcbf29ce484222325ull;
  void bytes(const void* d, size_t n) {
    const unsigned char* b = (const unsigned char*)d;
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
  }
  void scalars(std::initializer_list<int64_t> xs) {
    for (int64_t x : xs) bytes(&x, 8);
  }
  template <class T>
  void span(const T* v, int64_t n) {
    bytes(&n, 8);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t y = (int64_t)v[i];
      bytes(&y, 8);
    }
  }
  template <class T>
  void vec(const std::vector<T>& v) { span(v.data(), (int64_t)v.size()); }
};

int encode_tmap(fk_pool* p) {
  p->tmap_ok = false;
  if (!p->kv || p->num_pages == 0) return FK_OK;
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* sym = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &sym, cudaEnableDefault, &q);
    if (e != cudaSuccess || !sym) return fail(FK_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)sym;
  }
  const int D = p->desc.head_dim;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)(p->num_pages * kPage),
                        (cuuint64_t)p->desc.num_layers * 2 * p->desc.num_heads};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)p->num_pages * kPage * D * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)kPage, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(&p->tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p->kv, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FK_CUDA_ERROR, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  cuuint32_t box_run[3] = {64, (cuuint32_t)(kPage * kTcTilePages), 1};
  r = fn(&p->tmap_run, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p->kv, dims, strides, box_run, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FK_CUDA_ERROR, "cuTensorMapEncodeTiled (run) failed (%d)", (int)r);
  cuuint32_t box_half[3] = {64, (cuuint32_t)(kPage / 2), 1};
  r = fn(&p->tmap_half, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p->kv, dims, strides, box_half, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FK_CUDA_ERROR, "cuTensorMapEncodeTiled (half) failed (%d)", (int)r);
  p->tmap_ok = true;
  return FK_OK;
}

// Grow the physical arena to `pages`; live pages keep their ids (plane-wise copy).
int reserve_pages(fk_pool* p, int64_t pages) {
  if (pages <= p->num_pages) return FK_OK;
  if (!p->on_device) return FK_OK;
  FK_ON_DEVICE(p->desc.device);
  const size_t D = p->desc.head_dim;
  const size_t planes = (size_t)p->desc.num_layers * 2 * p->desc.num_heads;
  const size_t new_bytes = planes * (size_t)pages * kPage * D * 2;
  __nv_bfloat16* nkv = nullptr;
  cudaError_t e = cudaMalloc(&nkv, new_bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(FK_CUDA_ERROR, "KV arena of %zu bytes (%lld pages): %s", new_bytes,
                (long long)pages, cudaGetErrorString(e));
  }
  // zero so every byte a kernel may touch is a finite bf16.  cudaMemset runs
  // on the legacy default stream, which the pool's (non-blocking) streams do
  // not wait for: synchronize before any fill can write the new pages.
  FK_CUDA(cudaMemset(nkv, 0, new_bytes));
  FK_CUDA(cudaDeviceSynchronize());
  if (p->kv) {
    const size_t old_plane = (size_t)p->num_pages * kPage * D * 2;
    const size_t new_plane = (size_t)pages * kPage * D * 2;
    FK_CUDA(cudaMemcpy2D(nkv, new_plane, p->kv, old_plane, old_plane, planes,
                         cudaMemcpyDeviceToDevice));
    FK_CUDA(cudaFree(p->kv));
  }
  // new physical pages go under the existing free stack so lower ids pop first
  std::vector<int32_t> fresh;
  fresh.reserve(pages - p->num_pages);
  for (int64_t i = pages - 1; i >= p->num_pages; --i) fresh.push_back((int32_t)i);
  fresh.insert(fresh.end(), p->free_pages.begin(), p->free_pages.end());
  p->free_pages.swap(fresh);
  p->kv = nkv;
  p->arena_bytes = new_bytes;
  p->num_pages = pages;
  return encode_tmap(p);
}

int ensure_scratch(fk_pool* p, int rows, int slots, cudaStream_t st) {
  const size_t H = p->desc.num_heads, D = p->desc.head_dim;
  const size_t need = (size_t)std::max(rows, 1) * std::max(slots, 1) * H;
  if (need > p->part_cap) {
    // headroom: max_slots moves by one as suffixes cross page boundaries.
    // Stream-ordered (re)allocation on the plan's stream -- the stream the
    // step's kernels run on -- so growing the partials never syncs the device
    // (a cudaFree would wait for every engine sharing the GPU).
    // (first allocation: room for 64 rows x 16 slots, so a batch that builds
    // up request by request does not reallocate -- and update every graph
    // node -- at every few rows)
    size_t cap = std::max({need + need / 2, p->part_cap * 2, (size_t)64 * 16 * H});
    if (p->part_o) FK_CUDA(cudaFreeAsync(p->part_o, st));
    if (p->part_ml) FK_CUDA(cudaFreeAsync(p->part_ml, st));
    p->part_o = nullptr;
    p->part_ml = nullptr;
    // two halves: consecutive fk_attn_decode launches alternate, so a layer's
    // kernels may start (PDL) while the previous layer's merge still reads
    FK_CUDA(cudaMallocAsync((void**)&p->part_o, 2 * cap * D * sizeof(float), st));
    FK_CUDA(cudaMallocAsync((void**)&p->part_ml, 2 * cap * sizeof(float2), st));
    p->part_cap = cap;
  }
  return FK_OK;
}

int ensure_slot(fk_pool* p, PlanSlot& s, size_t bytes) {
  if (bytes <= s.cap) return FK_OK;
  // pinned allocations are slow: start at 256 KiB and double
  size_t cap = std::max({bytes + bytes / 2, s.cap * 2, (size_t)256 << 10});
  if (s.armed) FK_CUDA(cudaEventSynchronize(s.done));
  if (s.host) FK_CUDA(cudaFreeHost(s.host));
  if (s.dev) FK_CUDA(cudaFree(s.dev));
  s.host = nullptr;
  s.dev = nullptr;
  FK_CUDA(cudaMallocHost(&s.host, cap));
  FK_CUDA(cudaMalloc(&s.dev, cap));
  s.cap = cap;
  return FK_OK;
}

// Byte layout builder for one plan buffer.
struct Layout {
  size_t size = 0;
  size_t add(size_t bytes) {
    size_t off = align_up(size, 16);
    size = off + bytes;
    return off;
  }
};

// Process-wide allocator of the __constant__ plan slots (fk_plan_c): two
// per device pool.
std::mutex g_slot_mu;
std::vector<bool> g_slot_used(kPlanSlots, false);
int alloc_plan_slots() {
  std::lock_guard<std::mutex> lk(g_slot_mu);
  for (int i = 0; i + 1 < kPlanSlots; i += 2)
    if (!g_slot_used[i]) {
      g_slot_used[i] = g_slot_used[i + 1] = true;
      return i;
    }
  return -1;
}
void free_plan_slots(int base) {
  if (base < 0) return;
  std::lock_guard<std::mutex> lk(g_slot_mu);
  g_slot_used[base] = g_slot_used[base + 1] = false;
}

}  // namespace

extern "C" {

const char* fk_last_error(void) { return g_last_error.c_str(); }

const char* fk_build_info(void) {
  return "forkattn sm_100a (" __DATE__ " " __TIME__ "): tcgen05/TMEM/TMA shared-prefix attention "
         "co-run with a dynamic paged private stream, PDL-chained LSE merge";
}

int fk_pool_create(const fk_pool_desc* desc, fk_pool** out) {
  if (!desc || !out) return fail(FK_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (desc->block_size != kPage)
    return fail(FK_INVALID_ARGUMENT, "block_size must be %d (got %d)", kPage, desc->block_size);
  if (desc->head_dim != kHeadDim)
    return fail(FK_INVALID_ARGUMENT, "head_dim must be %d (got %d)", kHeadDim, desc->head_dim);
  if (desc->num_layers < 1 || desc->num_heads < 1 || desc->total_blocks < 0 || desc->num_pages < 0)
    return fail(FK_INVALID_ARGUMENT, "bad pool geometry");
  fk_pool* p = new fk_pool();
  p->desc = *desc;
  p->total_blocks = desc->total_blocks;
  p->on_device = desc->device >= 0;
  if (p->on_device) {
    DeviceGuard dg(desc->device);
    if (dg.err != cudaSuccess) {
      delete p;
      return fail(FK_CUDA_ERROR, "cudaSetDevice(%d): %s", desc->device, cudaGetErrorString(dg.err));
    }
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, desc->device) == cudaSuccess)
      p->num_sms = sms;
    for (auto& s : p->slots) {
      if (cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) != cudaSuccess) {
        delete p;
        return fail(FK_CUDA_ERROR, "cudaEventCreate failed");
      }
    }
    if (cudaMalloc(&p->tick, 2 * sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(p->tick, 0, 2 * sizeof(unsigned)) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      cudaGetLastError();
      fk_pool_destroy(p);
      return fail(FK_CUDA_ERROR, "ticket counter allocation failed");
    }
    p->plan_base = alloc_plan_slots();
    if (p->plan_base < 0) {
      fk_pool_destroy(p);
      return fail(FK_INVALID_ARGUMENT, "more than %d device pools in one process", kPlanSlots / 2);
    }
    int rc = reserve_pages(p, desc->num_pages);
    if (rc != FK_OK) {
      fk_pool_destroy(p);
      return rc;
    }
  }
  *out = p;
  return FK_OK;
}

int fk_pool_destroy(fk_pool* p) {
  if (!p) return FK_OK;
  if (p->on_device) {
    DeviceGuard dg(p->desc.device);
    cudaDeviceSynchronize();
    for (auto& s : p->slots) {
      if (s.host) cudaFreeHost(s.host);
      if (s.dev) cudaFree(s.dev);
      if (s.done) cudaEventDestroy(s.done);
    }
    if (p->kv) cudaFree(p->kv);
    if (p->part_o) cudaFree(p->part_o);
    if (p->part_ml) cudaFree(p->part_ml);
    if (p->tick) cudaFree(p->tick);
    free_plan_slots(p->plan_base);
    for (auto& kv : p->graphs) kv.second.reset();
  }
  delete p;
  return FK_OK;
}

int fk_pool_set_total_blocks(fk_pool* p, int64_t total) {
  if (!p || total < 0) return fail(FK_INVALID_ARGUMENT, "bad total_blocks");
  p->total_blocks = total;
  return FK_OK;
}

int fk_pool_reserve_pages(fk_pool* p, int64_t pages) {
  if (!p || pages < 0) return fail(FK_INVALID_ARGUMENT, "bad page count");
  return reserve_pages(p, pages);
}

int fk_pool_stats_get(const fk_pool* p, fk_pool_stats* out) {
  if (!p || !out) return fail(FK_INVALID_ARGUMENT, "null argument");
  out->used_blocks = p->used;
  out->free_blocks = p->total_blocks - p->used;
  out->peak_used = p->peak;
  out->total_blocks = p->total_blocks;
  out->next_block = p->next_logical;
  out->num_pages = p->num_pages;
  out->free_pages = (int64_t)p->free_pages.size();
  out->arena_bytes = (int64_t)p->arena_bytes;
  out->host_wait_ns = p->host_wait_ns;
  out->graph_replays = p->graph_replays;
  return FK_OK;
}

int fk_pool_set_option(fk_pool* p, int32_t option, int64_t value) {
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  switch (option) {
    case FK_OPT_TC_MIN_FANOUT: p->tc_min_fanout = value; break;
    case FK_OPT_PREFIX_TARGET_CTAS: p->prefix_target_ctas = value; break;
    case FK_OPT_LAUNCH_ORDER: p->launch_order = value; break;
    case FK_OPT_PDL: p->pdl = value; break;
    case FK_OPT_GRAPH: p->use_graph = value != 0; break;
    case FK_OPT_PRIV_STATIC_FIRST: p->priv_static_first = value != 0; break;
    case FK_OPT_PRIV_WARPS:
      if (value != 8 && value != 10 && value != 12)
        return fail(FK_INVALID_ARGUMENT, "private warps must be 8, 10 or 12");
      p->priv_wpc = value;
      break;
    case FK_OPT_TC_BOUNDARY_COST: p->tc_boundary_cost = std::max<int64_t>(0, value); break;
    case FK_OPT_PRIV_MIN_CHUNK: p->priv_min_chunk = std::min<int64_t>(kPrivMaxChunk, std::max<int64_t>(0, value)); break;
    case FK_OPT_MIN_SPLIT_PAGES: p->min_split_pages = std::max<int64_t>(1, value); break;
    case FK_OPT_CORUN: p->corun = value; break;
    case FK_OPT_PREFIX_RATE_PCT: p->prefix_rate_pct = std::max<int64_t>(1, value); break;
    case FK_OPT_APPEND_FIRST: p->append_first = value != 0; break;
    case FK_OPT_GROUP_FANOUT:
      if (value < 0 || value > 64) return fail(FK_INVALID_ARGUMENT, "group fan-out must be 0..64");
      p->group_fanout = value;
      break;
    case FK_OPT_DEBUG_SKIP_MERGE: p->skip_merge = value != 0; break;
    default: return fail(FK_INVALID_ARGUMENT, "unknown option %d", option);
  }
  return FK_OK;
}

// ---- context forest -------------------------------------------------------

int fk_ctx_create(fk_pool* p, int64_t ctx, int64_t parent) {
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (p->ctxs.count(ctx)) return fail(FK_INVALID_ARGUMENT, "context %lld exists", (long long)ctx);
  if (parent >= 0) {
    auto it = p->ctxs.find(parent);
    if (it == p->ctxs.end())
      return fail(FK_UNKNOWN_PARENT_CONTEXT, "unknown parent %lld", (long long)parent);
    it->second.children += 1;
  }
  Ctx c;
  c.parent = parent >= 0 ? parent : -1;
  c.par = parent >= 0 ? &p->ctxs.find(parent)->second : nullptr;
  p->ctxs.emplace(ctx, std::move(c));
  return FK_OK;
}

int fk_ctx_grow(fk_pool* p, int64_t ctx, int64_t new_tokens, int64_t* new_ids, int64_t cap,
                int64_t* n_new) {
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (n_new) *n_new = 0;
  auto it = p->ctxs.find(ctx);
  if (it == p->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "unknown context %lld", (long long)ctx);
  Ctx& c = it->second;
  if (new_tokens < 0) return fail(FK_INVALID_ARGUMENT, "negative token count");
  // engine.py:89 — need may be <= 0 (shrinking never releases blocks)
  const int64_t need = blocks_for(new_tokens, kPage) - (int64_t)c.logical.size();
  const int64_t free_logical = p->total_blocks - p->used;
  if (need > free_logical)
    return fail(FK_OUT_OF_MEMORY, "need %lld blocks, %lld free", (long long)need,
                (long long)free_logical);
  if (need > 0 && new_ids && cap < need)
    return fail(FK_INVALID_ARGUMENT, "id buffer too small (%lld < %lld)", (long long)cap,
                (long long)need);
  if (need > 0 && p->on_device && need > (int64_t)p->free_pages.size()) {
    // the logical pool admits it: back it with more device pages
    // grow geometrically (x1.5), but fall back to exactly what is needed when
    // the device cannot hold the old and the larger new arena at once
    const int64_t exact = p->num_pages + need - (int64_t)p->free_pages.size();
    const int64_t want = std::max<int64_t>(exact, std::min<int64_t>(p->total_blocks,
                                                                   std::max<int64_t>(64, p->num_pages * 3 / 2)));
    int rc = reserve_pages(p, want);
    if (rc != FK_OK && want > exact) rc = reserve_pages(p, exact);
    if (rc != FK_OK) return fail(FK_OUT_OF_MEMORY, "device arena: %s", g_last_error.c_str());
  }
  for (int64_t i = 0; i < need; ++i) {
    const int64_t bid = p->next_logical++;
    c.logical.push_back(bid);
    if (p->on_device) {
      c.phys.push_back(p->free_pages.back());
      p->free_pages.pop_back();
    } else {
      c.phys.push_back(-1);
    }
    if (new_ids) new_ids[i] = bid;
  }
  if (need > 0) p->used += need;
  c.tokens = new_tokens;
  if (p->used > p->peak) p->peak = p->used;
  if (n_new) *n_new = need > 0 ? need : 0;
  return FK_OK;
}

int fk_ctx_release(fk_pool* p, int64_t ctx) {
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  auto it = p->ctxs.find(ctx);
  if (it == p->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "unknown context %lld", (long long)ctx);
  Ctx& c = it->second;
  if (c.children > 0)
    return fail(FK_CONTEXT_BUSY, "context %lld has %d children", (long long)ctx, c.children);
  // physical pages go back to the free stack; logical ids are retired forever
  for (auto pg = c.phys.rbegin(); pg != c.phys.rend(); ++pg)
    if (*pg >= 0) p->free_pages.push_back(*pg);
  p->used -= (int64_t)c.logical.size();
  if (c.parent >= 0) {
    auto par = p->ctxs.find(c.parent);
    if (par != p->ctxs.end()) par->second.children -= 1;
  }
  p->ctxs.erase(it);
  return FK_OK;
}

int fk_ctx_info(const fk_pool* p, int64_t ctx, int64_t* tokens, int64_t* nblocks,
                int64_t* parent) {
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  auto it = p->ctxs.find(ctx);
  if (it == p->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "unknown context %lld", (long long)ctx);
  if (tokens) *tokens = it->second.tokens;
  if (nblocks) *nblocks = (int64_t)it->second.logical.size();
  if (parent) *parent = it->second.parent;
  return FK_OK;
}

int64_t fk_ctx_tokens(const fk_pool* p, int64_t ctx) {
  if (!p) return -1;
  auto it = p->ctxs.find(ctx);
  return it == p->ctxs.end() ? -1 : it->second.tokens;
}

int fk_ctx_blocks(const fk_pool* p, int64_t ctx, int64_t* logical, int32_t* physical, int64_t cap,
                  int64_t* n) {
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  auto it = p->ctxs.find(ctx);
  if (it == p->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "unknown context %lld", (long long)ctx);
  const Ctx& c = it->second;
  const int64_t k = (int64_t)c.logical.size();
  if (n) *n = k;
  if (cap < k && (logical || physical))
    return fail(FK_INVALID_ARGUMENT, "buffer too small (%lld < %lld)", (long long)cap, (long long)k);
  for (int64_t i = 0; i < k; ++i) {
    if (logical) logical[i] = c.logical[i];
    if (physical) physical[i] = c.phys[i];
  }
  return FK_OK;
}

// ---- decode step plan -----------------------------------------------------

int fk_step_plan(fk_pool* p, const int64_t* leaves, int32_t B, int32_t dedup, void* stream,
                 fk_plan_info* info) {
  NvtxRange nvtx("fk_step_plan", B);
  static const bool plan_timing = getenv("FK_DEBUG_TIMING") != nullptr;
  double pt[8] = {0};
#define PT(n) do { if (plan_timing) pt[#n[1] - '0'] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); } while (0)
  if (!p || (B > 0 && !leaves) || B < 0) return fail(FK_INVALID_ARGUMENT, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t H = p->desc.num_heads;

  PT(T0);
  // Everything below reuses the pool's scratch (no per-step allocation once
  // warm) and reaches contexts through pointers (one hash lookup per leaf);
  // tests/test_plan.py::test_plan_digests_pinned holds the output to the
  // round-1 planner's bit for bit.
  PlanScratch& S = p->ps;
  const uint32_t epoch = ++p->plan_epoch;
  // chains leaf -> root, fan-out per context (engine.py:476-482 walk)
  std::vector<Ctx*>& chain = S.chain;
  std::vector<int32_t>& chain_off = S.chain_off;
  std::vector<Ctx*>& order = S.order;  // unique contexts, first-seen (row order, leaf->root)
  chain.clear();
  order.clear();
  chain_off.resize(B + 1);
  for (int r = 0; r < B; ++r) {
    chain_off[r] = (int32_t)chain.size();
    auto li = p->ctxs.find(leaves[r]);
    if (li == p->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "unknown leaf context %lld", (long long)leaves[r]);
    for (Ctx* c = &li->second; c; c = c->par) {
      chain.push_back(c);
      if (c->mark != epoch) {
        c->mark = epoch;
        c->fan = 1;
        c->sidx = -1;
        c->gidx = -1;
        c->rank = 0;
        order.push_back(c);
      } else {
        c->fan += 1;
      }
    }
  }
  chain_off[B] = (int32_t)chain.size();
  auto count_tokens = [&]() {
    int64_t n = 0;
    if (dedup) {
      for (const Ctx* c : order) n += c->tokens;
    } else {
      for (const Ctx* c : chain) n += c->tokens;
    }
    return n;
  };
  int64_t shared_tokens = 0, private_tokens = 0;
  // the reference's count, before the step's growth (engine.py:416-417)
  const int64_t batch_tokens = count_tokens();
  std::vector<int64_t>& leaf_tokens_pre = S.leaf_tokens_pre;
  leaf_tokens_pre.resize(B);
  for (int r = 0; r < B; ++r) leaf_tokens_pre[r] = chain[chain_off[r]]->tokens;
  // FK_OPT_APPEND_FIRST: the step's one-token growth happens now, in row
  // (gens) order with the sequential OOM rule of fk_step_grow, and the
  // kernels' spans include the new token (a decoder attends to its own key)
  p->plan_grew = false;
  if (p->append_first) {
    p->grow_pos.assign(B, -1);
    p->grow_ids.assign(B, -1);
    for (int r = 0; r < B; ++r) {
      const int64_t pos = chain[chain_off[r]]->tokens;
      int64_t n = 0, id = -1;
      const int rc = fk_ctx_grow(p, leaves[r], pos + 1, &id, 1, &n);
      if (rc == FK_OUT_OF_MEMORY) continue;
      if (rc != FK_OK) return rc;
      p->grow_pos[r] = pos;
      p->grow_ids[r] = n > 0 ? id : -1;
    }
    p->plan_grew = true;
  }
  const int64_t streamed_tokens = p->append_first ? count_tokens() : batch_tokens;
  // (after the growth: a leaf two generations share becomes shared once it has a token)
  // Shared contexts with a small fan-out (<= FK_OPT_GROUP_FANOUT rows) are
  // streamed by the private kernel for groups of up to 8 rows (one K/V read
  // serves the group: the rows are the N of its transposed products); larger
  // ones go to the prefix kernels.
  int n_grouped = 0;
  int64_t grouped_tokens = 0, grouped_tok_heads = 0;
  for (Ctx* c : order) {
    c->shared = dedup && c->fan >= 2 && c->tokens > 0;
    if (c->shared && p->group_fanout > 0 && c->fan <= p->group_fanout && p->priv_wpc == kPrivWarpsPerCta) {
      c->shared = false;
      c->gidx = n_grouped++;
      grouped_tokens += c->tokens;
      grouped_tok_heads += c->tokens * H * ((c->fan + kGroupRows - 1) / kGroupRows);
    }
  }
  shared_tokens += grouped_tokens;  // (streamed once per group: the dedup count holds them once)

  PT(T1);
  // ---- shared contexts (K2 work) --------------------------------------------
  std::vector<PlanShared>& shared = S.shared;
  shared.clear();
  for (Ctx* c : order) {
    if (!c->shared) continue;
    c->sidx = (int32_t)shared.size();
    PlanShared s;
    s.ctx = c;
    s.tc = p->tc_min_fanout > 0 && c->fan >= p->tc_min_fanout;
    s.nrows = 0;
    shared.push_back(s);
    shared_tokens += c->tokens;
  }
  const int nsh_real = (int)shared.size();
  // descendant rows of each shared context, row order (counted, then placed)
  std::vector<int32_t>& srows = S.srows;
  for (const Ctx* c : chain)
    if (c->sidx >= 0) shared[c->sidx].nrows += 1;
  {
    int32_t acc = 0;
    for (auto& s : shared) {
      s.row0 = acc;
      acc += s.nrows;
      s.nrows = 0;
    }
    srows.resize(acc);
  }
  for (int r = 0; r < B; ++r)
    for (int32_t k = chain_off[r]; k < chain_off[r + 1]; ++k) {
      const int32_t si = chain[k]->sidx;
      if (si >= 0) srows[shared[si].row0 + shared[si].nrows++] = r;
    }
  std::vector<int32_t>& pages = S.pages;
  std::vector<int32_t>& page_ntok = S.page_ntok;
  std::vector<int32_t>& qrows = S.qrows;
  pages.clear();
  page_ntok.clear();
  qrows.clear();
  for (auto& s : shared) {
    const Ctx& c = *s.ctx;
    s.page_off = (int)pages.size();
    for (size_t k = 0; k < c.phys.size(); ++k) {
      pages.push_back(c.phys[k]);
      page_ntok.push_back((int32_t)std::min<int64_t>(kPage, c.tokens - (int64_t)k * kPage));
    }
    s.q_off = (int)qrows.size();
    qrows.insert(qrows.end(), srows.begin() + s.row0, srows.begin() + s.row0 + s.nrows);
  }
  // mma split policy: ~one wave of CTAs over the mma-class prefix work
  {
    int64_t total = 0;
    for (auto& s : shared)
      if (!s.tc) total += (int64_t)s.ctx->phys.size() * ((s.nrows + kMmaQBlock - 1) / kMmaQBlock) * H;
    const int64_t target = p->prefix_target_ctas > 0 ? p->prefix_target_ctas : p->num_sms;
    const int64_t per = std::max<int64_t>(p->min_split_pages, (total + target - 1) / std::max<int64_t>(target, 1));
    const int64_t ps = (per + kMmaTilePages - 1) / kMmaTilePages * kMmaTilePages;
    for (auto& s : shared) {
      const int64_t np = (int64_t)s.ctx->phys.size();
      s.splits = s.tc ? 1 : (int)std::max<int64_t>(1, (np + ps - 1) / ps);
    }
  }
  // items: mma (ctx, split, qblock, head) then tcgen05 (ctx, qblock, head)
  std::vector<PlanItem>& items = S.items;
  items.clear();
  int num_mma = 0, num_tc = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int si = 0; si < nsh_real; ++si) {
      const PlanShared& s = shared[si];
      if ((int)s.tc != pass) continue;
      const Ctx& c = *s.ctx;
      const int np = (int)c.phys.size();
      const int qb = s.tc ? kTcQBlock : kMmaQBlock;
      const int nq = s.nrows;
      const int psr = s.tc ? np : ((np + s.splits - 1) / s.splits + kMmaTilePages - 1) / kMmaTilePages * kMmaTilePages;
      // items are (query block, head) with the head innermost: with more than
      // one query block (> 128 forks) the unit list is k identical groups,
      // which the static split below mirrors so that the k CTAs reading a
      // tile read it together (the later reads hit L2)
      for (int sp = 0; sp < s.splits; ++sp) {
        const int p0 = sp * psr, p1 = std::min(np, p0 + psr);
        const int64_t t1 = std::min<int64_t>(c.tokens, (int64_t)p1 * kPage);
        for (int q0 = 0; q0 < nq; q0 += qb)
          for (int h = 0; h < H; ++h) {
            PlanItem it;
            it.sh = si;
            it.split = sp;
            it.q0 = q0;
            it.nq = std::min(qb, nq - q0);
            it.head = h;
            it.page0 = p0;
            it.npages = std::max(0, p1 - p0);
            it.ntok = (int)std::max<int64_t>(0, t1 - (int64_t)p0 * kPage);
            it.units = (it.npages + kTcTilePages - 1) / kTcTilePages;
            items.push_back(it);
            (s.tc ? num_tc : num_mma) += 1;
          }
      }
    }
  PT(T2);
  // tcgen05 stream-K: tile units of all tc items over <= one wave of CTAs
  std::vector<int32_t>& it_unit_off = S.it_unit_off;
  it_unit_off.assign(items.size(), 0);
  int64_t tc_units = 0;
  for (size_t i = num_mma; i < items.size(); ++i) {
    it_unit_off[i] = (int32_t)tc_units;
    tc_units += items[i].units;
  }
  // Spatial co-run: when every shared context is on the tcgen05 path, its
  // persistent CTAs take X SMs and the private stream-K grid the other
  // S - X, launched back to back (PDL) so both stream HBM at once.  X splits
  // the SMs in proportion to each side's bytes over its per-SM rate.
  int64_t priv_tok_heads = 0;
  for (const Ctx* c : chain)
    if (!c->shared && c->gidx < 0) priv_tok_heads += c->tokens * H;
  priv_tok_heads += grouped_tok_heads;
  // a 128-query block costs the softmax ~4/3 of a <= 64-query block per tile
  // (the 16-lane layout only covers fan-outs <= 64; measured 2.5 vs 1.9 us)
  double tc_tok_heads = 0.0;
  for (size_t i = num_mma; i < items.size(); ++i) tc_tok_heads += items[i].ntok * (items[i].nq > 64 ? 4.0 / 3.0 : 1.0);
  const bool corun = p->corun && num_mma == 0 && tc_units > 0 && priv_tok_heads > 0 && p->num_sms > 1;
  int64_t tc_target = p->prefix_target_ctas > 0 ? p->prefix_target_ctas : p->num_sms;
  if (corun && p->prefix_target_ctas <= 0) {
    const double wp = tc_tok_heads * 100.0 / (double)p->prefix_rate_pct;
    const double wv = (double)priv_tok_heads;
    tc_target = std::min<int64_t>(p->num_sms - 1, std::max<int64_t>(1, std::llround(p->num_sms * wp / (wp + wv))));
  }
  // tcgen05 schedule: the tile units are split into one cost-balanced range
  // per CTA (a piece start mid-range costs tc_boundary_cost tiles).  (A
  // ticketed dynamic tail of small chunks was measured in round 1: an
  // epilogue per chunk costs more than the balance gains -- removed.)
  // Chunks never cross an item and are listed in unit order (an item's
  // chunks are contiguous: chunk - it_first_chunk = piece index).
  std::vector<int32_t>& ch_item = S.ch_item;
  std::vector<int32_t>& ch_t0 = S.ch_t0;
  std::vector<int32_t>& ch_t1 = S.ch_t1;
  std::vector<int32_t>& cta_chunk0 = S.cta_chunk0;
  std::vector<int32_t>& it_first_chunk = S.it_first_chunk;
  ch_item.clear();
  ch_t0.clear();
  ch_t1.clear();
  cta_chunk0.clear();
  it_first_chunk.assign(items.size(), 0);
  int64_t tc_ctas = 0;
  bool tc_l2_share = false;
  if (tc_units > 0) {
    // at least ~4 tiles per CTA unless FK_OPT_PREFIX_TARGET_CTAS says
    // otherwise: a CTA's start-up (TMEM, barriers, first loads) costs about that
    const int64_t cap = p->prefix_target_ctas > 0 ? tc_units : (tc_units + 3) / 4;
    const int64_t X = std::max<int64_t>(1, std::min<int64_t>(tc_target, cap));
    // item of each unit boundary
    auto emit = [&](int64_t a, int64_t b) {  // chunks for units [a, b), split at items
      size_t i = num_mma;
      while (i + 1 < items.size() && it_unit_off[i + 1] <= a) ++i;
      while (a < b) {
        const int64_t end = std::min<int64_t>(b, it_unit_off[i] + items[i].units);
        ch_item.push_back((int32_t)i);
        ch_t0.push_back((int32_t)(a - it_unit_off[i]));
        ch_t1.push_back((int32_t)(end - it_unit_off[i]));
        a = end;
        ++i;
      }
    };
    // cost-balanced static ranges over [lo, hi) for nx CTAs -> cut points
    const double bc = (double)p->tc_boundary_cost;
    auto split = [&](int64_t lo, int64_t hi, int64_t nx, std::vector<int64_t>& cut) {
      size_t nxt_item = num_mma;
      while (nxt_item < items.size() && it_unit_off[nxt_item] <= lo) ++nxt_item;
      int64_t n_bound = 0;  // item starts strictly inside (lo, hi)
      for (size_t i = nxt_item; i < items.size(); ++i) n_bound += it_unit_off[i] < hi;
      double rest = (double)(hi - lo) + bc * (double)n_bound;
      const size_t first = cut.size();
      cut.push_back(lo);
      double cost = 0.0;
      int64_t u = lo;
      while (u < hi) {
        const int64_t b = (int64_t)(cut.size() - first) - 1;  // current CTA
        const double target = rest / (double)std::max<int64_t>(1, nx - b);
        const int64_t item_end = nxt_item < items.size() ? std::min<int64_t>(hi, it_unit_off[nxt_item]) : hi;
        const bool last = (int64_t)(cut.size() - first) == nx;
        int64_t take = last ? item_end - u
                            : std::min<int64_t>(item_end - u, std::max<int64_t>(1, std::llround(target - cost)));
        u += take;
        cost += (double)take;
        if (u == item_end && nxt_item < items.size() && it_unit_off[nxt_item] == u && u < hi) {
          ++nxt_item;
          if (!last && target - cost < 0.5) {  // close the CTA at the item boundary
            rest -= cost + bc;
            cut.push_back(u);
            cost = 0.0;
          } else {
            cost += bc;  // this CTA starts another piece
          }
        } else if (!last && u < hi && target - cost < 0.5) {
          rest -= cost;
          cut.push_back(u);
          cost = 0.0;
        }
      }
    };
    // One shared context with k >= 2 query blocks (> 128 forks): its unit
    // list is k identical groups (block-major item order above).  Split
    // group 0 over X / k CTAs and give group g the same ranges on CTAs
    // b + g X / k, so the k CTAs reading a tile read it at about the same
    // time and all but the first hit L2 (the loads then keep the default
    // L2 policy: PlanDev::tc_l2_share).
    int64_t mirror_k = 0;
    if (nsh_real == 1 && shared[0].tc && shared[0].splits == 1) {
      const int64_t k = ((int64_t)shared[0].nrows + kTcQBlock - 1) / kTcQBlock;
      if (k >= 2 && X >= 2 * k && (int64_t)(items.size() - num_mma) == k * H && tc_units % k == 0) mirror_k = k;
    }
    std::vector<int64_t>& cut = S.cut;
    cut.clear();
    if (mirror_k) {
      const int64_t ug = tc_units / mirror_k, xg = X / mirror_k;
      std::vector<int64_t>& c0 = S.cut0;
      c0.clear();
      split(0, ug, xg, c0);
      c0.push_back(ug);
      for (int64_t g = 0; g < mirror_k; ++g)
        for (size_t j = 0; j + 1 < c0.size(); ++j) cut.push_back(c0[j] + g * ug);
      cut.push_back(tc_units);
    } else {
      split(0, tc_units, X, cut);
      cut.push_back(tc_units);
    }
    tc_l2_share = mirror_k > 0;
    tc_ctas = (int64_t)cut.size() - 1;
    for (int64_t b = 0; b < tc_ctas; ++b) {
      cta_chunk0.push_back((int32_t)ch_item.size());
      emit(cut[b], cut[b + 1]);
    }
    cta_chunk0.push_back((int32_t)ch_item.size());
    for (size_t i = num_mma, k = 0; i < items.size(); ++i) {
      while (k < ch_item.size() && ch_item[k] != (int32_t)i) ++k;
      it_first_chunk[i] = (int32_t)k;
    }
  }
  const int64_t tc_nchunks = (int64_t)ch_item.size();
  if (getenv("FK_DEBUG_PLAN")) {
    fprintf(stderr, "fk plan: %lld tc units, %lld CTAs, %lld chunks:", (long long)tc_units, (long long)tc_ctas,
            (long long)tc_nchunks);
    for (size_t k = 0; k < ch_item.size(); ++k) fprintf(stderr, " %d:%d-%d", ch_item[k], ch_t0[k], ch_t1[k]);
    fprintf(stderr, "\n");
  }
  auto item_pieces = [&](size_t i) -> int {
    if ((int)i < num_mma) return 1;
    const int64_t next = (i + 1 < items.size()) ? it_first_chunk[i + 1] : tc_nchunks;
    return items[i].units == 0 ? 1 : (int)(next - it_first_chunk[i]);
  };
  PT(T3);
  // per (shared ctx, qblock, head): pieces contributed to each of its rows
  // (dense tables: this runs every step on the host)
  std::vector<int64_t>& qb_off = S.qb_off;  // first (qblock, head) slot of each shared ctx
  qb_off.assign(shared.size() + 1, 0);
  for (size_t si = 0; si < shared.size(); ++si) {
    const int qbs = shared[si].tc ? kTcQBlock : kMmaQBlock;
    qb_off[si + 1] = qb_off[si] + (int64_t)((shared[si].nrows + qbs - 1) / qbs) * H;
  }
  std::vector<int32_t>& pieces_of = S.pieces_of;
  pieces_of.assign(std::max<int64_t>(qb_off.back(), 1), 0);
  for (size_t i = 0; i < items.size(); ++i) {
    const PlanItem& it = items[i];
    const int qb = it.q0 / (shared[it.sh].tc ? kTcQBlock : kMmaQBlock);
    pieces_of[qb_off[it.sh] + (int64_t)qb * H + it.head] += item_pieces(i);
  }
  // each row's shared contexts root -> leaf with its query block in each
  // (rs[rs_off[r] ..]), and the slot base of each at every head
  std::vector<int32_t>& rs_off = S.rs_off;
  std::vector<int32_t>& rs_sh = S.rs_sh;
  std::vector<int32_t>& rs_qb = S.rs_qb;
  std::vector<int32_t>& srow_e = S.srow_e;  // rs entry of each (shared ctx, row) in srows order
  rs_off.resize(B + 1);
  rs_sh.clear();
  rs_qb.clear();
  {
    // position of each row among a shared context's rows: the rows are
    // placed in row order, so a running counter per context gives it
    for (auto& s : shared) s.seen = 0;
    srow_e.resize(srows.size());
    for (int r = 0; r < B; ++r) {
      rs_off[r] = (int32_t)rs_sh.size();
      for (int32_t k = chain_off[r + 1] - 1; k >= chain_off[r]; --k) {  // root -> leaf
        const int32_t si = chain[k]->sidx;
        if (si < 0) continue;
        PlanShared& sc = shared[si];
        srow_e[sc.row0 + sc.seen] = (int32_t)rs_sh.size();
        rs_sh.push_back(si);
        rs_qb.push_back(sc.seen++ / (sc.tc ? kTcQBlock : kMmaQBlock));
      }
    }
    rs_off[B] = (int32_t)rs_sh.size();
  }
  // slot bases: per (row, head) walk the shared chain root -> leaf
  std::vector<int32_t>& row_head_base = S.row_head_base;
  std::vector<int32_t>& base_at = S.base_at;  // [rs entry][H]
  row_head_base.assign(std::max<int64_t>((int64_t)B * H, 1), 0);
  base_at.resize(std::max<size_t>(rs_sh.size() * (size_t)H, 1));
  std::vector<int32_t>& acc = S.acc;
  acc.resize(H);
  for (int r = 0; r < B; ++r) {
    std::fill(acc.begin(), acc.end(), 0);
    for (int32_t e = rs_off[r]; e < rs_off[r + 1]; ++e) {
      const int32_t* po = pieces_of.data() + qb_off[rs_sh[e]] + (int64_t)rs_qb[e] * H;
      int32_t* ba = base_at.data() + (size_t)e * H;
      for (int h = 0; h < H; ++h) {
        ba[h] = acc[h];
        acc[h] += po[h];
      }
    }
    std::copy(acc.begin(), acc.end(), row_head_base.begin() + (int64_t)r * H);
  }
  std::vector<int32_t>& it_qslot_off = S.it_qslot_off;
  std::vector<int32_t>& qslot = S.qslot;
  it_qslot_off.resize(items.size());
  {
    size_t nq_all = 0;
    for (const PlanItem& it : items) nq_all += it.nq;
    qslot.resize(nq_all);
  }
  for (size_t i = 0, o = 0; i < items.size(); ++i) {
    const PlanItem& it = items[i];
    const int32_t* re = srow_e.data() + shared[it.sh].row0 + it.q0;
    const int32_t* ba = base_at.data() + it.head;
    it_qslot_off[i] = (int32_t)o;
    const int add = (int)i < num_mma ? it.split : 0;
    for (int j = 0; j < it.nq; ++j) qslot[o + j] = ba[(size_t)re[j] * H] + add;
    o += it.nq;
  }

  PT(T4);
  // ---- private-kernel items (K3 work) -------------------------------------------
  // An item is a run of page entries streamed once for a group of rows: the
  // pages of a small-fan-out shared context (FK_OPT_GROUP_FANOUT, up to 8 rows
  // per item; a context with more rows gets one item per 8) or one row's
  // private chain (root -> leaf, contexts with fan-out 1).  Grouped items come
  // first, then one item per row in row order (item B_g + r = row r).
  std::vector<int32_t>& it_e0 = S.pit_e0;      // first entry (relative to the private base)
  std::vector<int32_t>& it_np = S.pit_np;      // entries
  std::vector<int32_t>& it_roff = S.pit_roff;  // rows at it_rows[it_roff ..]
  std::vector<int32_t>& it_nrows = S.pit_nrows;
  std::vector<int32_t>& it_rows = S.pit_rows;
  it_e0.clear();
  it_np.clear();
  it_roff.clear();
  it_nrows.clear();
  it_rows.clear();
  const int64_t priv_base = (int64_t)pages.size();
  if (n_grouped > 0) {
    // rows of each grouped context, row order
    std::vector<int32_t>& grow_cnt = S.grow_cnt;
    std::vector<int32_t>& grows = S.grows;
    grow_cnt.assign(n_grouped + 1, 0);
    for (const Ctx* c : chain)
      if (c->gidx >= 0) grow_cnt[c->gidx + 1] += 1;
    for (int gi = 0; gi < n_grouped; ++gi) grow_cnt[gi + 1] += grow_cnt[gi];
    grows.resize(grow_cnt[n_grouped]);
    std::vector<int32_t>& gfill = S.gfill;
    gfill.assign(grow_cnt.begin(), grow_cnt.end() - 1);
    for (int r = 0; r < B; ++r)
      for (int32_t k = chain_off[r]; k < chain_off[r + 1]; ++k) {
        const int32_t gi = chain[k]->gidx;
        if (gi >= 0) grows[gfill[gi]++] = r;
      }
    for (const Ctx* c : order) {
      if (c->gidx < 0) continue;
      const int32_t r0 = grow_cnt[c->gidx], r1 = grow_cnt[c->gidx + 1];
      const int32_t e0 = (int32_t)(pages.size() - priv_base);
      for (size_t j = 0; j < c->phys.size(); ++j) {
        const int64_t nt = std::min<int64_t>(kPage, c->tokens - (int64_t)j * kPage);
        if (nt <= 0) break;
        pages.push_back(c->phys[j]);
        page_ntok.push_back((int32_t)nt);
      }
      const int32_t np = (int32_t)(pages.size() - priv_base) - e0;
      for (int32_t a = r0; a < r1; a += kGroupRows) {
        if (a > r0) {  // the next group streams the same pages again (L2)
          for (int32_t j = 0; j < np; ++j) {
            pages.push_back(pages[priv_base + e0 + j]);
            page_ntok.push_back(page_ntok[priv_base + e0 + j]);
          }
        }
        it_e0.push_back(a > r0 ? (int32_t)(pages.size() - priv_base) - np : e0);
        it_np.push_back(np);
        it_roff.push_back((int32_t)it_rows.size());
        it_nrows.push_back(std::min<int32_t>(kGroupRows, r1 - a));
        for (int32_t b = a; b < std::min<int32_t>(r1, a + kGroupRows); ++b) it_rows.push_back(grows[b]);
      }
    }
  }
  for (int r = 0; r < B; ++r) {
    const int32_t e0 = (int32_t)(pages.size() - priv_base);
    for (int32_t k = chain_off[r + 1] - 1; k >= chain_off[r]; --k) {  // root -> leaf
      const Ctx& c = *chain[k];
      if (c.shared || c.gidx >= 0 || c.tokens <= 0) continue;
      private_tokens += c.tokens;
      for (size_t j = 0; j < c.phys.size(); ++j) {
        const int64_t nt = std::min<int64_t>(kPage, c.tokens - (int64_t)j * kPage);
        if (nt <= 0) break;
        pages.push_back(c.phys[j]);
        page_ntok.push_back((int32_t)nt);
      }
    }
    it_e0.push_back(e0);
    it_np.push_back((int32_t)(pages.size() - priv_base) - e0);
    it_roff.push_back((int32_t)it_rows.size());
    it_nrows.push_back(1);
    it_rows.push_back(r);
  }
  const int32_t n_pitems = (int32_t)it_e0.size();
  // private units (head, flat private entry), head-major
  const int64_t NPT = (int64_t)pages.size() - priv_base;
  std::vector<int32_t>& page_item = S.page_item;
  page_item.resize(std::max<int64_t>(NPT, 1));
  page_item[0] = 0;
  for (int32_t k = 0; k < n_pitems; ++k) std::fill_n(page_item.begin() + it_e0[k], it_np[k], k);
  const int64_t U = NPT * H;
  if (U > INT32_MAX) return fail(FK_INVALID_ARGUMENT, "private work too large (%lld units)", (long long)U);
  PT(T5);
  // Guided dynamic schedule: chunks shrink from ~U / (2 W) pages to mc as the
  // list drains (W = warps that start at once), warps grab them from a ticket
  // counter.  The grid covers every SM: in co-run the CTAs beyond the free
  // SMs start when tcgen05 prefix CTAs retire and take the leftovers.
  const int64_t priv_sms = corun ? std::max<int64_t>(1, p->num_sms - tc_ctas) : p->num_sms;
  const int64_t wpc = p->priv_wpc;
  const int64_t w_active = priv_sms * wpc;
  // size(pos) = clamp(ceil((U - pos) / 2W), min_chunk, 32), generated run by
  // run: one division per distinct size, then plain stores (this runs every step)
  std::vector<int32_t>& chunk_start = S.chunk_start;
  {
    const int64_t w2 = 2 * w_active;
    // chunk count of the guided schedule for a minimum size (the generator
    // below without its stores)
    auto count_chunks = [&](int64_t mc) {
      int64_t n = 0, pos = 0;
      while (pos < U) {
        const int64_t R = U - pos;
        const int64_t sz = std::min<int64_t>(std::max<int64_t>((R + w2 - 1) / w2, mc), kPrivMaxChunk);
        const int64_t floor_r = sz > mc ? (sz - 1) * w2 : 0;
        int64_t k = sz > mc ? (R - floor_r + sz - 1) / sz : (R + sz - 1) / sz;
        k = std::min<int64_t>(k, (R + sz - 1) / sz);
        n += k;
        pos = std::min<int64_t>(U, pos + k * sz);
      }
      return n;
    };
    // Minimum chunk (auto): 2 pages beside a prefix grid (the private CTAs
    // past the free SMs start as prefix CTAs retire, so there is no last
    // round to fit; 2 measured best from 16 to 64 forks, profiles/r02/tune/).
    // Small plans without one (under 32K units: a few rows, every (item, head)
    // run cut into ~U / W pieces) start every warp at once and take ~n / W
    // chunks: the last round leaves ceil(n/W) - n/W of the warps idle for one
    // chunk of mc pages, and each chunk costs about two pages of time (ticket,
    // metadata, pipeline refill, one more partial to merge), so mc in 4..8
    // minimises idle * mc + 2 n / W (fan-outs 1-8: +2.8..6.9 % over a fixed 4,
    // profiles/r02/min_chunk/).
    int64_t mc = p->priv_min_chunk > 0 ? p->priv_min_chunk : kPrivMinChunk;
    if (p->priv_min_chunk == 0 && U < 32768 && tc_ctas == 0 && U > 0) {
      double best = 1e300;
      for (int64_t m = 8; m >= 4; --m) {  // (ties keep the larger chunk)
        const double f = (double)count_chunks(m) / (double)w_active;
        const double cost = (std::ceil(f - 1e-9) - f) * (double)m + 2.0 * f;
        if (cost < best - 1e-9) {
          best = cost;
          mc = m;
        }
      }
    }
    // upper bound of the chunk count: every chunk but the last has >= mc
    // units (grown only: a resize down and up again would zero-fill)
    const size_t bound = (size_t)(U / std::max<int64_t>(mc, 1) + 2);
    if (chunk_start.size() < bound) chunk_start.resize(bound);
    int32_t* cs = chunk_start.data();
    int64_t n = 0, pos = 0;
    while (pos < U) {
      const int64_t R = U - pos;
      int64_t sz = std::min<int64_t>(std::max<int64_t>((R + w2 - 1) / w2, mc), kPrivMaxChunk);
      // the size holds while ceil(R / 2W) stays >= sz (capped) or == sz
      const int64_t floor_r = sz > mc ? (sz - 1) * w2 : 0;  // R must stay above this
      int64_t k = sz > mc ? (R - floor_r + sz - 1) / sz : (R + sz - 1) / sz;
      // k chunks of sz units from pos, the last one cut at U
      k = std::min<int64_t>(k, (R + sz - 1) / sz);
      const int32_t p0 = (int32_t)pos, s32 = (int32_t)sz;
      for (int32_t j = 0; j < (int32_t)k; ++j) cs[n + j] = p0 + j * s32;
      n += k;
      pos = std::min<int64_t>(U, pos + k * sz);
    }
    cs[n] = (int32_t)U;
    S.n_chunks = n;
  }
  const int64_t nchunks = S.n_chunks;
  // launched first (order 1) the private grid must leave the prefix its SMs
  // The grid is the SM count whatever the work (warps without a chunk exit at
  // once), so its launch stays the same from step to step.
  const int64_t grid_ctas = (corun && p->launch_order == 1) ? priv_sms : p->num_sms;
  const int64_t G = grid_ctas * wpc;
  // (item, head) runs are contiguous unit ranges in unit order (head-major,
  // items in entry order), so one forward sweep finds every run's chunks; each
  // row of an item gets that run's pieces as consecutive partial slots, after
  // its tcgen05 / mma prefix pieces and its earlier items' pieces
  std::vector<int32_t>& row_head_count = S.row_head_count;
  std::vector<int32_t>& item_chunk0 = S.item_chunk0;
  std::vector<int32_t>& item_slot = S.item_slot;  // [(it_roff[k] + j) * H + h]
  std::vector<int32_t>& run_pieces = S.item_pieces;  // [item][H]
  row_head_count.assign(row_head_base.begin(), row_head_base.end());
  item_chunk0.assign(std::max<int64_t>((int64_t)n_pitems * H, 1), 0);
  run_pieces.assign(std::max<int64_t>((int64_t)n_pitems * H, 1), 0);
  item_slot.resize(std::max<size_t>(it_rows.size() * (size_t)H, 1));
  {
    const int32_t* cs = chunk_start.data();
    int64_t c = 0;  // chunk holding the current unit
    for (int64_t h = 0; h < H; ++h)
      for (int32_t k = 0; k < n_pitems; ++k) {
        const int64_t np = it_np[k];
        if (np > 0) {
          const int64_t a0 = h * NPT + it_e0[k], b0 = a0 + np;
          while (cs[c + 1] <= a0) ++c;
          const int64_t c0 = c;
          while (cs[c + 1] <= b0 - 1) ++c;
          item_chunk0[k * H + h] = (int32_t)c0;
          run_pieces[k * H + h] = (int32_t)(c - c0 + 1);
        }
      }
    // slots, item by item in entry order (each row's runs follow one another)
    for (int32_t k = 0; k < n_pitems; ++k) {
      const int32_t* pc = run_pieces.data() + (size_t)k * H;
      for (int32_t j = 0; j < it_nrows[k]; ++j) {
        int32_t* cnt = row_head_count.data() + (size_t)it_rows[it_roff[k] + j] * H;
        int32_t* sl = item_slot.data() + (size_t)(it_roff[k] + j) * H;
        for (int64_t h = 0; h < H; ++h) {
          sl[h] = cnt[h];
          cnt[h] += pc[h];
        }
      }
    }
  }
  int max_slots = 1;
  for (int32_t v : row_head_count) max_slots = std::max(max_slots, v);
  PT(T6);
  // synthetic keys: (leaf uid, leaf tokens at plan time + rank << 40)
  std::vector<int64_t>& row_uid = S.row_uid;
  std::vector<int64_t>& row_pos = S.row_pos;
  row_uid.resize(B);
  row_pos.resize(B);
  p->plan_leaves.assign(leaves, leaves + B);
  p->plan_leaf_tokens.resize(B);
  for (int r = 0; r < B; ++r) {
    const int k = chain[chain_off[r]]->rank++;
    row_uid[r] = leaves[r];
    p->plan_leaf_tokens[r] = leaf_tokens_pre[r];
    row_pos[r] = leaf_tokens_pre[r] + ((int64_t)k << 40);
  }

  // the work-list invariant: the KV tokens the kernels stream
  // per layer -- shared contexts once, private contexts per row -- are exactly
  // Engine._batch_tokens(running) (engine.py:470-484)
  if (shared_tokens + private_tokens != streamed_tokens)
    return fail(FK_INVALID_ARGUMENT, "work-list invariant violated: %lld shared + %lld private != %lld batch tokens",
                (long long)shared_tokens, (long long)private_tokens, (long long)streamed_tokens);
  const int n_items = (int)items.size();
  if (info) {
    info->batch_tokens = batch_tokens;
    info->shared_tokens = shared_tokens;
    info->private_tokens = private_tokens;
    info->num_rows = B;
    info->num_shared_ctx = (int32_t)shared.size() + n_grouped;  // (grouped: streamed by the private kernel)
    info->num_prefix_ctas = (int32_t)(num_mma + tc_ctas);
    info->max_slots = max_slots;
    info->num_tc_items = num_tc;
    info->num_mma_items = num_mma;
    info->fused_merge = 0;  // (the fused form was removed in round 2: always the merge kernel)
    info->streamed_tokens = streamed_tokens;
  }
  p->committed = false;
  if (plan_timing) {
    PT(T7);
    fprintf(stderr, "fk plan us: walk %.0f shared %.0f tc %.0f slots %.0f priv %.0f sched %.0f keys %.0f\n",
            pt[1] - pt[0], pt[2] - pt[1], pt[3] - pt[2], pt[4] - pt[3], pt[5] - pt[4], pt[6] - pt[5], pt[7] - pt[6]);
  }
  static const bool plan_debug = getenv("FK_DEBUG_PLAN") != nullptr;
  if (plan_debug) {
    int64_t parts = 0, priv_parts = 0;
    for (int64_t k = 0; k < B * H; ++k) parts += row_head_count[k];
    for (int64_t k = 0; k < B * H; ++k) priv_parts += row_head_count[k] - row_head_base[k];
    fprintf(stderr, "fk plan: %d rows, %lld private units, %lld chunks, partials %lld (private %lld), max slots %d\n",
            B, (long long)U, (long long)nchunks, (long long)parts, (long long)priv_parts, max_slots);
  }
  if (plan_digest_on()) {
    PlanDigest dg;
    dg.scalars({batch_tokens, shared_tokens, private_tokens, streamed_tokens, (int64_t)shared.size(), num_mma, num_tc,
                tc_units, tc_ctas, tc_nchunks, (int64_t)tc_l2_share, priv_base, NPT, U, nchunks, wpc, G, grid_ctas,
                (int64_t)max_slots, (int64_t)n_items, w_active});
    for (int i = 0; i < n_items; ++i) {
      const PlanItem& it = items[i];
      const PlanShared& sh = shared[it.sh];
      dg.scalars({sh.page_off + it.page0, it.npages, it.ntok, sh.q_off + it.q0, it.nq, it.head, it_unit_off[i],
                  it_qslot_off[i], it.units});
    }
    // (the round-1 per-row private layout, from the private items)
    std::vector<int32_t>& row_priv_off = S.row_priv_off;
    std::vector<int32_t>& row_priv_np = S.row_priv_np;
    std::vector<int32_t>& row_unit_off = S.row_unit_off;
    row_priv_off.resize(B);
    row_priv_np.resize(B);
    row_unit_off.assign(std::max(B, 1), 0);
    for (int r = 0; r < B; ++r) {
      const int32_t k = n_pitems - B + r;
      row_priv_off[r] = (int32_t)priv_base + it_e0[k];
      row_priv_np[r] = it_np[k];
      row_unit_off[r] = it_e0[k];
    }
    dg.vec(qrows); dg.vec(qslot); dg.vec(row_priv_off); dg.vec(row_priv_np); dg.vec(row_unit_off);
    dg.vec(row_head_base); dg.vec(row_head_count); dg.vec(pages); dg.vec(page_ntok); dg.vec(row_uid); dg.vec(row_pos);
    dg.vec(page_item); dg.span(chunk_start.data(), nchunks + 1); dg.vec(item_chunk0);
    if (n_pitems > B) {  // grouped items (not in the round-1 planner)
      dg.vec(it_e0); dg.vec(it_np); dg.vec(it_nrows); dg.vec(it_rows); dg.vec(item_slot);
    } dg.vec(ch_item); dg.vec(ch_t0); dg.vec(ch_t1);
    dg.vec(it_first_chunk); dg.vec(cta_chunk0);
    p->plan_digest = dg.h;
  }
  if (!p->on_device) {
    p->have_plan = true;
    return FK_OK;
  }

  PT(T7);
  // ---- upload ---------------------------------------------------------------
  FK_ON_DEVICE(p->desc.device);
  int rc = ensure_scratch(p, B, max_slots, st);
  if (rc != FK_OK) return rc;
  const size_t ni = (size_t)std::max(n_items, 1);
  const size_t nb = (size_t)std::max(B, 1);
  const size_t nbh = (size_t)std::max<int64_t>(B * H, 1);
  Layout L;
  const size_t o_it = L.add(sizeof(int32_t) * 9 * ni);
  const size_t o_q = L.add(sizeof(int32_t) * std::max<size_t>(qrows.size(), 1));
  const size_t o_qs = L.add(sizeof(int32_t) * std::max<size_t>(qslot.size(), 1));
  const size_t o_rh = L.add(sizeof(int32_t) * 2 * nbh);
  const size_t o_pages = L.add(sizeof(int32_t) * std::max<size_t>(pages.size(), 1));
  const size_t o_pnt = L.add(sizeof(int32_t) * std::max<size_t>(pages.size(), 1));
  const size_t o_uid = L.add(sizeof(int64_t) * nb);
  const size_t o_pos = L.add(sizeof(int64_t) * nb);
  const size_t o_app = L.add(sizeof(int32_t) * 2 * nb);
  const size_t o_apos = L.add(sizeof(int64_t) * nb);
  const size_t o_prow = L.add(sizeof(int32_t) * page_item.size());
  const size_t o_cs = L.add(sizeof(int32_t) * (size_t)(nchunks + 1));
  const size_t o_rhc = L.add(sizeof(int32_t) * item_chunk0.size());
  const size_t npi = (size_t)std::max(n_pitems, 1);
  const size_t o_pit = L.add(sizeof(int32_t) * 2 * npi);  // nrows, roff
  const size_t o_pir = L.add(sizeof(int32_t) * std::max<size_t>(it_rows.size(), 1));
  const size_t o_pis = L.add(sizeof(int32_t) * item_slot.size());
  const size_t nchb = sizeof(int32_t) * std::max<size_t>(ch_item.size(), 1);
  const size_t o_chi = L.add(nchb);
  const size_t o_ch0 = L.add(nchb);
  const size_t o_ch1 = L.add(nchb);
  const size_t o_ifc = L.add(sizeof(int32_t) * ni);
  const size_t o_cc0 = L.add(sizeof(int32_t) * std::max<size_t>(cta_chunk0.size(), 1));
  const size_t o_pd = L.add(sizeof(PlanDev));  // the plan struct itself (pinned source of the constant upload)
  // rotate slots; wait until the GPU finished with the one we reuse
  if (p->cur >= 0 && p->slots[p->cur].dev) {
    FK_CUDA(cudaEventRecord(p->slots[p->cur].done, st));
    p->slots[p->cur].armed = true;
  }
  p->cur = (p->cur + 1) & 1;
  PlanSlot& slot = p->slots[p->cur];
  if (slot.armed) {
    const auto w0 = std::chrono::steady_clock::now();
    FK_CUDA(cudaEventSynchronize(slot.done));
    p->host_wait_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - w0).count();
  }
  rc = ensure_slot(p, slot, L.size);
  if (rc != FK_OK) return rc;
  char* h = (char*)slot.host;
  auto put = [&](size_t off, const void* src, size_t bytes) {
    if (bytes) memcpy(h + off, src, bytes);
  };
  int32_t* itb = (int32_t*)(h + o_it);
  for (int i = 0; i < n_items; ++i) {
    const PlanItem& it = items[i];
    const PlanShared& sh = shared[it.sh];
    itb[0 * ni + i] = sh.page_off + it.page0;
    itb[1 * ni + i] = it.npages;
    itb[2 * ni + i] = it.ntok;
    itb[3 * ni + i] = sh.q_off + it.q0;
    itb[4 * ni + i] = it.nq;
    itb[5 * ni + i] = it.head;
    itb[6 * ni + i] = it_unit_off[i];
    itb[7 * ni + i] = it_qslot_off[i];
    itb[8 * ni + i] = it.units;
  }
  put(o_q, qrows.data(), qrows.size() * 4);
  put(o_qs, qslot.data(), qslot.size() * 4);
  put(o_rh, row_head_base.data(), row_head_base.size() * 4);
  put(o_rh + nbh * 4, row_head_count.data(), row_head_count.size() * 4);
  put(o_pages, pages.data(), pages.size() * 4);
  put(o_pnt, page_ntok.data(), page_ntok.size() * 4);
  put(o_uid, row_uid.data(), (size_t)B * 8);
  put(o_pos, row_pos.data(), (size_t)B * 8);
  int32_t* ab = (int32_t*)(h + o_app);
  for (int r = 0; r < B; ++r) {
    ab[r] = -1;
    ab[nb + r] = 0;
  }
  memset(h + o_apos, 0, nb * 8);
  put(o_prow, page_item.data(), page_item.size() * 4);
  put(o_cs, chunk_start.data(), (size_t)(nchunks + 1) * 4);
  put(o_rhc, item_chunk0.data(), item_chunk0.size() * 4);
  put(o_pit, it_nrows.data(), (size_t)n_pitems * 4);
  put(o_pit + npi * 4, it_roff.data(), (size_t)n_pitems * 4);
  put(o_pir, it_rows.data(), it_rows.size() * 4);
  put(o_pis, item_slot.data(), item_slot.size() * 4);
  put(o_chi, ch_item.data(), ch_item.size() * 4);
  put(o_ch0, ch_t0.data(), ch_t0.size() * 4);
  put(o_ch1, ch_t1.data(), ch_t1.size() * 4);
  put(o_ifc, it_first_chunk.data(), it_first_chunk.size() * 4);
  put(o_cc0, cta_chunk0.data(), cta_chunk0.size() * 4);
  FK_CUDA(cudaMemcpyAsync(slot.dev, slot.host, L.size, cudaMemcpyHostToDevice, st));

  const char* d = (const char*)slot.dev;
  PlanDev& pd = p->plan;
  pd.num_rows = B;
  pd.max_slots = max_slots;
  pd.num_items = n_items;
  pd.tc_begin = num_mma;
  const int32_t* ditb = (const int32_t*)(d + o_it);
  pd.it_page_off = ditb + 0 * ni;
  pd.it_npages = ditb + 1 * ni;
  pd.it_ntok = ditb + 2 * ni;
  pd.it_q_off = ditb + 3 * ni;
  pd.it_nq = ditb + 4 * ni;
  pd.it_head = ditb + 5 * ni;
  pd.it_unit_off = ditb + 6 * ni;
  pd.it_qslot_off = ditb + 7 * ni;
  pd.it_units = ditb + 8 * ni;
  pd.qrows = (const int32_t*)(d + o_q);
  pd.qslot = (const int32_t*)(d + o_qs);
  pd.tc_units = (int)tc_units;
  pd.tc_ctas = (int)tc_ctas;
  // The launched prefix grid only changes when the plan's CTA count leaves
  // [grid - 16, grid]: CTAs past tc_ctas exit at once, and a step whose
  // launches repeat the previous ones replays its CUDA graph without node
  // updates (the running set, and with it tc_ctas, moves every step under
  // a serving load).
  if (tc_ctas > 0 && (tc_ctas > p->tc_grid || tc_ctas + 16 < p->tc_grid))
    p->tc_grid = (int)std::min<int64_t>(std::max<int64_t>(p->num_sms, tc_ctas), (tc_ctas + 7) / 8 * 8);
  pd.tc_grid = p->tc_grid;
  pd.tc_nchunks = (int)tc_nchunks;
  pd.tc_chunk_item = (const int32_t*)(d + o_chi);
  pd.tc_chunk_tile0 = (const int32_t*)(d + o_ch0);
  pd.tc_chunk_tile1 = (const int32_t*)(d + o_ch1);
  pd.it_first_chunk = (const int32_t*)(d + o_ifc);
  pd.tc_cta_chunk0 = (const int32_t*)(d + o_cc0);
  pd.tc_l2_share = tc_l2_share ? 1 : 0;
  pd.row_head_base = (const int32_t*)(d + o_rh);
  pd.row_head_count = (const int32_t*)(d + o_rh) + nbh;
  pd.pages = (const int32_t*)(d + o_pages);
  pd.page_ntok = (const int32_t*)(d + o_pnt);
  pd.row_uid = (const long long*)(d + o_uid);
  pd.row_pos = (const long long*)(d + o_pos);
  pd.app_page = (const int32_t*)(d + o_app);
  pd.app_slot = (const int32_t*)(d + o_app) + nb;
  pd.app_pos = (const long long*)(d + o_apos);
  pd.page_item = (const int32_t*)(d + o_prow);
  pd.item_nrows = (const int32_t*)(d + o_pit);
  pd.item_roff = (const int32_t*)(d + o_pit) + npi;
  pd.item_rows = (const int32_t*)(d + o_pir);
  pd.item_slot = (const int32_t*)(d + o_pis);
  pd.priv_base = (int)priv_base;
  pd.priv_np = (int)NPT;
  pd.priv_units = (int)U;
  pd.priv_nchunks = (int)nchunks;
  pd.priv_wpc = (int)wpc;
  pd.priv_warps = (int)G;
  pd.priv_static = p->priv_static_first ? (int)std::min<int64_t>(std::min<int64_t>(w_active, G), nchunks) : 0;
  pd.priv_chunk_start = (const int32_t*)(d + o_cs);
  pd.item_chunk0 = (const int32_t*)(d + o_rhc);
  pd.n_gitems = n_pitems - B;
  pd.n_grows = (int)it_rows.size() - B;
  p->off_app_page = o_app;
  p->off_app_slot = o_app + nb * 4;
  p->off_app_pos = o_apos;
  p->priv_grid = (int)grid_ctas;
  // the plan struct into this slot's __constant__ entry of both kernel units
  memcpy(h + o_pd, &pd, sizeof(PlanDev));
  const int ps = p->plan_base + p->cur;
  FK_CUDA(upload_plan_main(ps, (const PlanDev*)(h + o_pd), st));
  FK_CUDA(upload_plan_tc(ps, (const PlanDev*)(h + o_pd), st));
  p->have_plan = true;
  return FK_OK;
}

int fk_attn_decode(fk_pool* p, int32_t layer, const void* q, void* out, float* out_f32,
                   void* stream) {
  NvtxRange nvtx("fk_attn_decode", layer);
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (!p->on_device) return fail(FK_NO_DEVICE, "host-only pool has no device arena");
  if (!p->have_plan) return fail(FK_INVALID_ARGUMENT, "no plan: call fk_step_plan first");
  if (layer < 0 || layer >= p->desc.num_layers) return fail(FK_INVALID_ARGUMENT, "bad layer %d", layer);
  if (p->plan.num_rows == 0) return FK_OK;
  if (!q || !out) return fail(FK_INVALID_ARGUMENT, "null q/out");
  FK_ON_DEVICE(p->desc.device);
  cudaStream_t st = (cudaStream_t)stream;
  const float scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)p->desc.head_dim));
  ArenaDev a = p->arena();
  if (p->launch_parity) {
    a.part_o += p->part_cap * p->desc.head_dim;
    a.part_ml += p->part_cap;
    a.tick += 1;
  }
  p->launch_parity ^= 1;
  const int ps = p->plan_base + p->cur;  // the plan's __constant__ slot
  const bool has_mma = p->plan.tc_begin > 0;
  const bool has_tc = p->plan.num_items > p->plan.tc_begin;
  // cross-layer PDL: this layer's first kernel may start while the previous
  // layer's merge runs (it writes the other half of the partials and reads
  // q only after griddepcontrol.wait); never behind the mma prefix kernel
  const bool xl = p->pdl >= 2 && !has_mma;
  if (!p->tmap_ok) return fail(FK_CUDA_ERROR, "tensor map not encoded");
  // K2 (shared prefixes) and K3 (private streams) only write partials, so
  // their order is free; K4 merges every (row, head) afterwards and resets
  // this half's ticket counter.  If a launch fails after others went out,
  // the counter is reset behind them so the half starts clean next time.
  bool launched = false;
  auto bail = [&](cudaError_t e, const char* what) -> int {
    if (launched && !g_launch_rec) cudaMemsetAsync(a.tick, 0, sizeof(unsigned), st);
    return fail(FK_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
  };
#define FK_LAUNCH(expr, what)                          \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return bail(_e, what);      \
    launched = true;                                   \
  } while (0)
  auto run_prefix = [&](bool pdl_tc, bool after_private) -> int {
    if (has_mma) FK_LAUNCH(launch_prefix_mma(a, p->plan, ps, layer, q, scale_log2, &p->tmap, st), "prefix (mma)");
    if (has_tc)
      FK_LAUNCH(launch_prefix_tc(a, p->plan, ps, layer, q, scale_log2, &p->tmap, &p->tmap_run, pdl_tc,
                                 after_private, st), "prefix (tcgen05)");
    return FK_OK;
  };
  // Launch order 0: prefix -> private (PDL: private fills the SMs the prefix
  // grid leaves free; its CTAs wait for the prefix grid on exit).  Order 1:
  // private -> prefix (PDL when the tcgen05 grid is the only prefix grid; its
  // CTAs then wait for the private grid on exit).  Either way the second
  // grid's completion implies the first's, which the merge waits for.
  if (p->launch_order == 0) {
    int rc = run_prefix(xl, false);
    if (rc != FK_OK) return rc;
    FK_LAUNCH(launch_private(a, p->plan, ps, layer, q, scale_log2, &p->tmap, &p->tmap_half, p->priv_grid,
                             (p->pdl && (has_mma || has_tc)) || (xl && !has_tc), st), "private");
  } else {
    FK_LAUNCH(launch_private(a, p->plan, ps, layer, q, scale_log2, &p->tmap, &p->tmap_half, p->priv_grid, xl, st), "private");
    const bool chained = p->pdl && has_tc && !has_mma && p->plan.priv_units > 0;
    int rc = run_prefix(chained, chained);
    if (rc != FK_OK) return rc;
  }
  // fixed merge grid (warps loop over (row, head)): 3 CTAs of 8 warps per SM -- as many as
  // its registers let be resident at once (a 4th wave measured 0.5-0.8 % slower per step, 2
  // per SM slower still)
  if (p->skip_merge) {  // diagnostic: no merge (and the ticket half reset by a memset)
    if (fk::g_launch_rec) return fail(FK_INVALID_ARGUMENT, "FK_OPT_DEBUG_SKIP_MERGE needs FK_OPT_GRAPH=0");
    FK_CUDA(cudaMemsetAsync(a.tick, 0, sizeof(unsigned), st));
    return FK_OK;
  }
  // (plans with many partials per (row, head): one CTA of 8 warps per item;
  // the grid stays fixed either way, so the launch does not change per step)
  const bool wide = wide_merge(p->plan.max_slots, p->plan.num_rows, p->desc.num_heads, p->num_sms);
  FK_LAUNCH(launch_merge(a, ps, out, out_f32, layer, wide ? 2 * p->num_sms : 3 * p->num_sms, p->pdl != 0, wide, st),
            "merge");
#undef FK_LAUNCH
  return FK_OK;
}

int fk_attn_decode_layers(fk_pool* p, int32_t layer0, int32_t nlayers, const void* q, int64_t q_layer_stride,
                          void* out, int64_t out_layer_stride, float* out_f32, int64_t f32_layer_stride,
                          void* stream) {
  NvtxRange nvtx("fk_attn_decode_layers", nlayers);
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (nlayers < 0 || layer0 < 0 || layer0 + nlayers > p->desc.num_layers)
    return fail(FK_INVALID_ARGUMENT, "bad layer range [%d, %d)", layer0, layer0 + nlayers);
  auto run = [&]() -> int {
    for (int32_t i = 0; i < nlayers; ++i) {
      const int rc = fk_attn_decode(p, layer0 + i, (const char*)q + i * q_layer_stride,
                                    (char*)out + i * out_layer_stride,
                                    out_f32 ? (float*)((char*)out_f32 + i * f32_layer_stride) : nullptr, stream);
      if (rc != FK_OK) return rc;
    }
    return FK_OK;
  };
  // (the legacy default stream cannot be captured: direct launches there)
  if (!p->use_graph || !p->on_device || stream == nullptr) return run();
  static const bool timing = getenv("FK_DEBUG_TIMING") != nullptr;
  auto now_us = []() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t0 = timing ? now_us() : 0.0;
  const int par0 = p->launch_parity;
  cudaStream_t st = (cudaStream_t)stream;
  // One graph per (layer range, stream, plan slot, starting partial half):
  // with the plan in __constant__ memory the kernel arguments then repeat
  // from step to step, and a replay needs no parameter update at all.
  GraphCache& G = p->graphs[std::make_tuple(layer0, nlayers, st, p->cur * 2 + par0)];
  // 0. nothing the launches depend on changed: replay as is
  ReplayKey key;
  memset(&key, 0, sizeof(key));
  key.kv = p->kv;
  key.num_pages = p->num_pages;
  key.part_o = p->part_o;
  key.part_ml = p->part_ml;
  key.tick = p->tick;
  key.part_cap = p->part_cap;
  key.q = q;
  key.out = out;
  key.out_f32 = out_f32;
  key.q_stride = q_layer_stride;
  key.out_stride = out_layer_stride;
  key.f32_stride = out_f32 ? f32_layer_stride : 0;  // (no f32 output: the stride is never used)
  key.tc_begin = p->plan.tc_begin;
  key.num_items = p->plan.num_items;
  // (the prefix launch depends on the plan's CTA count only through its grid,
  // max(tc_grid, tc_ctas), and whether there is one: the count itself lives in
  // the __constant__ plan and may move from step to step under a serving load)
  key.tc_grid = p->plan.tc_ctas > 0 ? std::max(p->plan.tc_grid, p->plan.tc_ctas) : 0;
  key.tc_ctas = p->plan.tc_ctas > 0;
  key.priv_any = p->plan.priv_units > 0;
  key.priv_wpc = p->plan.priv_wpc;
  key.priv_grid = p->priv_grid;
  key.num_sms = p->num_sms;
  key.pdl = (int32_t)p->pdl;
  key.launch_order = (int32_t)p->launch_order;
  key.plan_slot = p->plan_base + p->cur;
  key.wide_merge = wide_merge(p->plan.max_slots, p->plan.num_rows, p->desc.num_heads, p->num_sms);
  key.grouped = p->plan.n_gitems > 0;
  const bool check = getenv("FK_DEBUG_GRAPH_CHECK") != nullptr;  // (read per call: tests set it)
  const bool key_hit = G.exec && G.key_ok && G.stream == st && p->have_plan && p->plan.num_rows > 0 &&
                       !p->skip_merge && memcmp(&G.key, &key, sizeof(key)) == 0;
  static const bool key_debug = getenv("FK_DEBUG_GRAPH_KEY") != nullptr;
  if (key_debug && G.exec && G.key_ok && !key_hit) {  // which 8-byte word of the key moved
    const uint64_t *a = (const uint64_t*)&G.key, *b = (const uint64_t*)&key;
    fprintf(stderr, "fk graph key miss: words");
    for (size_t w = 0; w < sizeof(key) / 8; ++w)
      if (a[w] != b[w]) fprintf(stderr, " %zu", w);
    fprintf(stderr, "\n");
  }
  if (key_hit && !check) {
    FK_CUDA(cudaGraphLaunch(G.exec, st));
    p->launch_parity = par0 ^ (nlayers & 1);  // as the recorded run would have left it
    p->graph_replays += 1;
    if (timing) fprintf(stderr, "fk graph: replay %.1f us\n", now_us() - t0);
    return FK_OK;
  }
  // 1. record the launches (same code path; the partial-half parity advances
  // before anything runs, and goes back if the graph is not launched)
  struct Rollback {
    fk_pool* p;
    int par;
    bool armed = true;
    ~Rollback() {
      if (armed) p->launch_parity = par;
    }
  } rollback{p, par0};
  fk::RecBuf& recs = p->rec_buf;
  recs.n = 0;
  fk::g_launch_rec = &recs;
  const int rc = run();
  fk::g_launch_rec = nullptr;
  if (rc != FK_OK) return rc;
  if (recs.n == 0) {
    rollback.armed = false;
    return FK_OK;
  }
  bool same = G.exec && G.stream == st && G.shape.size() == recs.n;
  for (size_t i = 0; same && i < recs.n; ++i) {
    const fk::LaunchRec &a = G.shape[i], &b = recs.v[i];
    same = a.func == b.func && a.pdl == b.pdl && a.offs == b.offs;
  }
  if (key_hit) {  // FK_DEBUG_GRAPH_CHECK: the key said "unchanged" -- so must the launches
    for (size_t i = 0; same && i < recs.n; ++i) {
      const fk::LaunchRec &a = G.shape[i], &b = recs.v[i];
      same = a.grid.x == b.grid.x && a.grid.y == b.grid.y && a.block.x == b.block.x && a.smem == b.smem &&
             a.bytes == b.bytes;
    }
    if (!same) return fail(FK_INVALID_ARGUMENT, "graph replay key missed a launch change");
    p->graph_replays += 1;  // (checked: counted as the replay it would have been)
  }
  const double t1 = timing ? now_us() : 0.0;
  int updated = 0;
  if (same) {
    // 2a. known structure: refresh only the nodes whose grid or arguments
    // changed (a grid may change in place; the function and PDL edges not)
    for (size_t i = 0; i < recs.n; ++i) {
      fk::LaunchRec& r = recs.v[i];
      fk::LaunchRec& c = G.shape[i];
      if (c.grid.x == r.grid.x && c.grid.y == r.grid.y && c.block.x == r.block.x && c.smem == r.smem &&
          c.bytes == r.bytes)
        continue;
      r.finalize();
      cudaKernelNodeParams kp = {};
      kp.func = const_cast<void*>(r.func);
      kp.gridDim = r.grid;
      kp.blockDim = r.block;
      kp.sharedMemBytes = (unsigned)r.smem;
      kp.kernelParams = r.args.data();
      FK_CUDA(cudaGraphExecKernelNodeSetParams(G.exec, G.nodes[i], &kp));
      c.grid = r.grid;
      c.block = r.block;
      c.smem = r.smem;
      c.bytes = r.bytes;
      ++updated;
    }
  } else {
    // 2b. new structure: capture the launches (PDL attributes become
    // programmatic edges) and instantiate
    G.reset();
    FK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    for (size_t k = 0; k < recs.n; ++k) {
      fk::LaunchRec& r = recs.v[k];
      r.finalize();
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = r.grid;
      cfg.blockDim = r.block;
      cfg.dynamicSmemBytes = r.smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = r.pdl ? 1 : 0;
      cudaError_t e = cudaLaunchKernelExC(&cfg, r.func, r.args.data());
      cudaStreamCaptureStatus cs;
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      if (e == cudaSuccess) e = cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd);
      if (e != cudaSuccess || nd != 1) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        G.reset();
        return fail(FK_CUDA_ERROR, "graph capture: %s (%zu dependencies)", cudaGetErrorString(e), nd);
      }
      G.nodes.push_back(deps[0]);
    }
    cudaError_t e = cudaStreamEndCapture(st, &G.graph);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&G.exec, G.graph, 0);
    if (e != cudaSuccess) {
      G.reset();
      return fail(FK_CUDA_ERROR, "graph instantiate: %s", cudaGetErrorString(e));
    }
    G.stream = st;
    G.shape.assign(recs.v.begin(), recs.v.begin() + recs.n);
    updated = (int)recs.n;
  }
  const double t2 = timing ? now_us() : 0.0;
  FK_CUDA(cudaGraphLaunch(G.exec, st));
  rollback.armed = false;
  G.key = key;
  G.key_ok = true;
  if (timing)
    fprintf(stderr, "fk graph: %zu launches, record %.1f us, %s %.1f us (%d nodes), launch %.1f us\n", recs.n,
            t1 - t0, same ? "update" : "capture", t2 - t1, updated, now_us() - t2);
  return FK_OK;
}

int fk_step_grow(fk_pool* p, int64_t* positions, int64_t* new_ids, int32_t* n_failed) {
  NvtxRange nvtx("fk_step_grow");
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (!p->have_plan) return fail(FK_INVALID_ARGUMENT, "no plan");
  const int B = (int)p->plan_leaves.size();
  if (B > 0 && (!positions || !new_ids)) return fail(FK_INVALID_ARGUMENT, "null output");
  int32_t nf = 0;
  if (p->plan_grew) {  // FK_OPT_APPEND_FIRST: the plan did this step's growth
    for (int r = 0; r < B; ++r) {
      positions[r] = p->grow_pos[r];
      new_ids[r] = p->grow_ids[r];
      nf += positions[r] < 0;
    }
    p->plan_grew = false;
    if (n_failed) *n_failed = nf;
    return FK_OK;
  }
  for (int r = 0; r < B; ++r) {  // gens order, one token each (engine.py:431-443)
    auto it = p->ctxs.find(p->plan_leaves[r]);
    if (it == p->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "leaf of row %d vanished", r);
    const int64_t pos = it->second.tokens;
    int64_t n = 0;
    const int rc = fk_ctx_grow(p, p->plan_leaves[r], pos + 1, &new_ids[r], 1, &n);
    if (rc == FK_OUT_OF_MEMORY) {
      positions[r] = -1;
      new_ids[r] = -1;
      ++nf;
      continue;
    }
    if (rc != FK_OK) return rc;
    positions[r] = pos;
    if (n == 0) new_ids[r] = -1;
  }
  if (n_failed) *n_failed = nf;
  return FK_OK;
}

int fk_step_commit(fk_pool* p, const int64_t* positions, void* stream) {
  NvtxRange nvtx("fk_step_commit");
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (!p->have_plan) return fail(FK_INVALID_ARGUMENT, "no plan");
  const int B = (int)p->plan_leaves.size();
  if (B > 0 && !positions) return fail(FK_INVALID_ARGUMENT, "null positions");
  // validate against the forest first (no partial effects)
  std::vector<int32_t> pg(B, -1), sl(B, 0);
  std::vector<int64_t> ps(B, 0);
  for (int r = 0; r < B; ++r) {
    if (positions[r] < 0) continue;
    auto it = p->ctxs.find(p->plan_leaves[r]);
    if (it == p->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "leaf of row %d vanished", r);
    const Ctx& c = it->second;
    const int64_t pos = positions[r];
    if (pos >= c.tokens || pos / kPage >= (int64_t)c.phys.size())
      return fail(FK_INVALID_ARGUMENT, "row %d position %lld outside leaf (%lld tokens)", r,
                  (long long)pos, (long long)c.tokens);
    pg[r] = c.phys[pos / kPage];
    sl[r] = (int32_t)(pos % kPage);
    ps[r] = pos;
  }
  p->committed = true;
  if (!p->on_device || B == 0) return FK_OK;
  FK_ON_DEVICE(p->desc.device);
  PlanSlot& slot = p->slots[p->cur];
  char* h = (char*)slot.host;
  const size_t nb = (size_t)std::max(B, 1);
  int32_t* ab = (int32_t*)(h + p->off_app_page);
  memcpy(ab, pg.data(), B * 4);
  memcpy(ab + nb, sl.data(), B * 4);
  memcpy(h + p->off_app_pos, ps.data(), B * 8);
  cudaStream_t st = (cudaStream_t)stream;
  FK_CUDA(cudaMemcpyAsync((char*)slot.dev + p->off_app_page, h + p->off_app_page, nb * 8,
                          cudaMemcpyHostToDevice, st));
  FK_CUDA(cudaMemcpyAsync((char*)slot.dev + p->off_app_pos, h + p->off_app_pos, nb * 8,
                          cudaMemcpyHostToDevice, st));
  return FK_OK;
}

int fk_append_kv(fk_pool* p, int32_t layer, const void* k, const void* v, void* stream) {
  return fk_append_kv_layers(p, layer, 1, k, v, stream);
}

int fk_append_kv_layers(fk_pool* p, int32_t layer0, int32_t nlayers, const void* k, const void* v,
                        void* stream) {
  NvtxRange nvtx("fk_append_kv_layers", nlayers);
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (!p->on_device) return fail(FK_NO_DEVICE, "host-only pool has no device arena");
  if (!p->committed) return fail(FK_INVALID_ARGUMENT, "fk_step_commit not called for this plan");
  if (layer0 < 0 || nlayers < 1 || layer0 + nlayers > p->desc.num_layers)
    return fail(FK_INVALID_ARGUMENT, "bad layer range [%d, %d)", layer0, layer0 + nlayers);
  if (p->plan.num_rows == 0) return FK_OK;
  if (!k || !v) return fail(FK_INVALID_ARGUMENT, "null k/v");
  FK_ON_DEVICE(p->desc.device);
  FK_CUDA(launch_append(p->arena(), p->plan, p->plan_base + p->cur, layer0, nlayers, k, v, (cudaStream_t)stream));
  return FK_OK;
}

int fk_synth_fill(fk_pool* p, int64_t ctx, int64_t pos0, int64_t pos1, uint64_t seed,
                  float k_scale, void* stream) {
  NvtxRange nvtx("fk_synth_fill", pos1 - pos0);
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (!p->on_device) return fail(FK_NO_DEVICE, "host-only pool has no device arena");
  auto it = p->ctxs.find(ctx);
  if (it == p->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "unknown context %lld", (long long)ctx);
  const Ctx& c = it->second;
  if (pos0 < 0 || pos1 < pos0 || pos1 > c.tokens)
    return fail(FK_INVALID_ARGUMENT, "bad range [%lld, %lld) of %lld", (long long)pos0,
                (long long)pos1, (long long)c.tokens);
  if (pos1 == pos0) return FK_OK;
  FK_ON_DEVICE(p->desc.device);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t first = pos0 / kPage, last = (pos1 - 1) / kPage;
  const int n = (int)(last - first + 1);
  int* dpages = nullptr;
  FK_CUDA(cudaMallocAsync(&dpages, sizeof(int) * n, st));
  FK_CUDA(cudaMemcpyAsync(dpages, c.phys.data() + first, sizeof(int) * n, cudaMemcpyHostToDevice, st));
  FK_CUDA(launch_synth_fill(p->arena(), dpages, (int)first, ctx, pos0, pos1, seed, k_scale, st));
  FK_CUDA(cudaFreeAsync(dpages, st));
  return FK_OK;
}

int fk_fill_kv(fk_pool* p, int64_t ctx, int64_t pos0, int64_t pos1, int32_t layer0, int32_t nlayers,
               const void* k, const void* v, void* stream) {
  NvtxRange nvtx("fk_fill_kv", pos1 - pos0);
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (!p->on_device) return fail(FK_NO_DEVICE, "host-only pool has no device arena");
  auto it = p->ctxs.find(ctx);
  if (it == p->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "unknown context %lld", (long long)ctx);
  const Ctx& c = it->second;
  if (pos0 < 0 || pos1 < pos0 || pos1 > c.tokens)
    return fail(FK_INVALID_ARGUMENT, "bad range [%lld, %lld) of %lld", (long long)pos0, (long long)pos1,
                (long long)c.tokens);
  if (layer0 < 0 || nlayers < 1 || layer0 + nlayers > p->desc.num_layers)
    return fail(FK_INVALID_ARGUMENT, "bad layer range [%d, %d)", layer0, layer0 + nlayers);
  if (pos1 == pos0) return FK_OK;
  if (!k || !v) return fail(FK_INVALID_ARGUMENT, "null k/v");
  if (pos1 - pos0 > INT32_MAX / p->desc.num_heads) return fail(FK_INVALID_ARGUMENT, "fill too large");
  FK_ON_DEVICE(p->desc.device);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t first = pos0 / kPage, last = (pos1 - 1) / kPage;
  const int n = (int)(last - first + 1);
  int* dpages = nullptr;
  FK_CUDA(cudaMallocAsync(&dpages, sizeof(int) * n, st));
  FK_CUDA(cudaMemcpyAsync(dpages, c.phys.data() + first, sizeof(int) * n, cudaMemcpyHostToDevice, st));
  FK_CUDA(launch_fill_kv(p->arena(), dpages, (int)first, pos0, (int)(pos1 - pos0), layer0, nlayers, k, v, st));
  FK_CUDA(cudaFreeAsync(dpages, st));
  return FK_OK;
}

int fk_ctx_copy_kv(fk_pool* dst, int64_t dst_ctx, const fk_pool* src, int64_t src_ctx, int64_t ntok,
                   void* stream) {
  NvtxRange nvtx("fk_ctx_copy_kv", ntok);
  if (!dst || !src) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (!dst->on_device || !src->on_device) return fail(FK_NO_DEVICE, "host-only pool has no device arena");
  if (dst->desc.num_layers != src->desc.num_layers || dst->desc.num_heads != src->desc.num_heads ||
      dst->desc.head_dim != src->desc.head_dim)
    return fail(FK_INVALID_ARGUMENT, "pools have different model geometry");
  auto di = dst->ctxs.find(dst_ctx);
  if (di == dst->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "unknown context %lld", (long long)dst_ctx);
  auto si = src->ctxs.find(src_ctx);
  if (si == src->ctxs.end()) return fail(FK_UNKNOWN_CONTEXT, "unknown source context %lld", (long long)src_ctx);
  if (ntok < 0 || ntok > si->second.tokens || ntok > di->second.tokens)
    return fail(FK_INVALID_ARGUMENT, "copy of %lld tokens exceeds a context (%lld -> %lld)", (long long)ntok,
                (long long)si->second.tokens, (long long)di->second.tokens);
  if (ntok == 0) return FK_OK;
  FK_ON_DEVICE(dst->desc.device);
  if (src->desc.device != dst->desc.device) {
    int can = 0;
    FK_CUDA(cudaDeviceCanAccessPeer(&can, dst->desc.device, src->desc.device));
    if (!can) return fail(FK_CUDA_ERROR, "device %d cannot access device %d", dst->desc.device, src->desc.device);
    cudaError_t e = cudaDeviceEnablePeerAccess(src->desc.device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (e != cudaSuccess) return fail(FK_CUDA_ERROR, "peer access: %s", cudaGetErrorString(e));
  }
  const int n = (int)((ntok + kPage - 1) / kPage);
  std::vector<int32_t> pairs(2 * (size_t)n);
  for (int j = 0; j < n; ++j) {
    pairs[j] = si->second.phys[j];
    pairs[n + j] = di->second.phys[j];
  }
  cudaStream_t st = (cudaStream_t)stream;
  int* dpages = nullptr;
  FK_CUDA(cudaMallocAsync(&dpages, sizeof(int) * 2 * n, st));
  FK_CUDA(cudaMemcpyAsync(dpages, pairs.data(), sizeof(int) * 2 * n, cudaMemcpyHostToDevice, st));
  FK_CUDA(launch_copy_pages(dst->arena(), src->kv, src->num_pages, dpages, n, st));
  FK_CUDA(cudaFreeAsync(dpages, st));
  // pairs (pageable) was staged by the H2D copy before this call returns
  return FK_OK;
}

int fk_synth_queries(fk_pool* p, uint64_t seed, void* q_all, int32_t rows_cap, void* stream) {
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (!p->on_device) return fail(FK_NO_DEVICE, "host-only pool has no device arena");
  if (!p->have_plan) return fail(FK_INVALID_ARGUMENT, "no plan");
  if (p->plan.num_rows == 0) return FK_OK;
  FK_ON_DEVICE(p->desc.device);
  if (rows_cap != 0 && rows_cap < p->plan.num_rows) return fail(FK_INVALID_ARGUMENT, "rows_cap %d < %d rows", rows_cap, p->plan.num_rows);
  FK_CUDA(launch_synth_queries(p->arena(), p->plan, p->plan_base + p->cur, seed, q_all,
                               rows_cap ? rows_cap : p->plan.num_rows, (cudaStream_t)stream));
  return FK_OK;
}

int fk_synth_append(fk_pool* p, uint64_t seed, float k_scale, void* stream) {
  if (!p) return fail(FK_INVALID_ARGUMENT, "null pool");
  if (!p->on_device) return fail(FK_NO_DEVICE, "host-only pool has no device arena");
  if (!p->committed) return fail(FK_INVALID_ARGUMENT, "fk_step_commit not called for this plan");
  if (p->plan.num_rows == 0) return FK_OK;
  FK_ON_DEVICE(p->desc.device);
  FK_CUDA(launch_synth_append(p->arena(), p->plan, p->plan_base + p->cur, seed, k_scale, (cudaStream_t)stream));
  return FK_OK;
}

uint64_t fk_debug_plan_digest(const fk_pool* p) { return p ? p->plan_digest : 0; }

// ---- hashing (tokenizer.py:36-49) -------------------------------------------

uint64_t fk_fnv1a64_u32(const uint32_t* ids, size_t n, uint64_t seed) {
  uint64_t h = seed;
  for (size_t i = 0; i < n; ++i) {
    uint32_t t = ids[i];
    for (int b = 0; b < 4; ++b) {
      h ^= (uint64_t)((t >> (8 * b)) & 0xFFu);
      h *= 0x00000100000001B3ULL;
    }
  }
  return h;
}

int fk_fnv1a64_chain(const uint32_t* ids, const int64_t* seg_off, int32_t nseg, uint64_t seed,
                     uint64_t* out) {
  if (nseg < 0 || (nseg > 0 && (!seg_off || !out))) return fail(FK_INVALID_ARGUMENT, "bad arguments");
  uint64_t h = seed;
  for (int32_t i = 0; i < nseg; ++i) {
    const int64_t a = seg_off[i], b = seg_off[i + 1];
    if (b < a) return fail(FK_INVALID_ARGUMENT, "segment %d has negative length", i);
    h = fk_fnv1a64_u32(ids + a, (size_t)(b - a), h);
    out[i] = h;
  }
  return FK_OK;
}

}  // extern "C"
