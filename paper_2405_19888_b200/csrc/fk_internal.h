// Internal structures shared by the host pool (fk_pool.cpp) and the sm_100a
// kernels (fk_*.cu).  Not part of the C-ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <vector>

namespace fk {

constexpr int kPage = 16;      // tokens per page (Config.block_size, config.py:21)
constexpr int kHeadDim = 128;  // D; LLaMA-7B/13B
constexpr int kMmaQBlock = 64; // queries per mma.sync prefix CTA (4 warps x 16 rows)
constexpr int kTcQBlock = 128; // queries per tcgen05 prefix CTA (M = 128 rows)
constexpr int kMmaTilePages = 4;  // 64-token KV tile for the mma.sync path
constexpr int kTcTilePages = 8;   // 128-token KV tile for the tcgen05 path
constexpr int kTcMaxChunk = 24;   // largest tcgen05 chunk (tiles)
constexpr int kPrivWarpsPerCta = 10;  // private kernel default shape: 10 warps per CTA x 2 stages (measured best)
constexpr int kPrivMinChunk = 2;     // private guided schedule: smallest chunk (pages), default
constexpr int kPrivMaxChunk = 32;    // largest chunk (one lane-parallel metadata load)
constexpr int kWideSlots = 32;       // plans with more partials per (row, head) and few (row, head) items
                                     // merge with a CTA per item (fk_merge_wide_kernel)
constexpr int kNarrowMaxSlots = 128; // the warp-per-item merge's register rounds
// The merge kernel for a plan: a CTA per (row, head) when items are many
// partials each and few (a few rows: ~200 pieces per head), a warp per item
// otherwise -- thousands of items (map-reduce: 2560 with ~40 pieces) keep all
// of the fixed grid's warps busy in one pass.
inline bool wide_merge(int max_slots, int rows, int heads, int num_sms) {
  return max_slots > kNarrowMaxSlots || (max_slots > kWideSlots && rows * heads <= 4 * num_sms);
}
constexpr int kGroupRows = 8;        // rows per private-kernel item (the N of its m16n8 products)

// Device view of one step plan.  All arrays live in one device buffer.
// Partials of (row, head) live at slots [0, row_head_count): shared-prefix
// pieces first (root -> leaf), then the private pieces from row_head_base.
struct PlanDev {
  int num_rows;
  int max_slots;
  int num_items;        // prefix items; each is (context, split|-, query block, head)
  int tc_begin;         // items [0, tc_begin) -> mma.sync kernel, [tc_begin, num_items) -> tcgen05
  // prefix items (SoA)
  const int* it_page_off;  // offset into pages[] of the item's first page
  const int* it_npages;
  const int* it_ntok;      // valid tokens in the item (contiguous from its first page)
  const int* it_q_off;     // offset into qrows[]
  const int* it_nq;
  const int* it_head;
  const int* it_unit_off;  // tcgen05 stream-K: first tile unit of the item
  const int* it_qslot_off; // offset into qslot[]
  const int* it_units;     // 128-token tiles of the item
  const int* qrows;        // request rows
  const int* qslot;        // slot of piece 0 for each (item, query)
  // tcgen05 schedule: chunks of consecutive tiles of one item, in unit
  // order; CTA b streams chunks [tc_cta_chunk0[b], tc_cta_chunk0[b + 1]).
  int tc_units, tc_ctas, tc_nchunks;
  int tc_grid;                    // launched CTAs (>= tc_ctas, kept across steps: the extra CTAs exit at once)
  const int* tc_chunk_item;       // [tc_nchunks]
  const int* tc_chunk_tile0;      // [tc_nchunks] first tile within the item
  const int* tc_chunk_tile1;      // [tc_nchunks] end tile (exclusive)
  const int* it_first_chunk;      // per item: its first chunk (piece 0)
  const int* tc_cta_chunk0;       // [tc_ctas + 1]
  int tc_l2_share;                // CTAs b, b + X/k stream the same tiles together: default L2 policy
  // rows
  const int* row_head_base;    // [rows][H] first slot after the row's prefix-kernel pieces
  const int* row_head_count;   // [rows][H] partials the merge combines
  const int* pages;            // physical page ids
  const int* page_ntok;        // valid tokens per page entry
  // private schedule: units u in [0, H * priv_np) = (head, flat private page
  // entry e): head = u / priv_np, entry = priv_base + u % priv_np, cut into
  // chunks [priv_chunk_start[c], priv_chunk_start[c + 1]) that warps grab
  // from a ticket counter.  Entries belong to items: a run of pages streamed
  // once for up to kGroupRows rows (a small-fan-out shared context, or one
  // row's private chain).
  const int* page_item;        // item of each flat private entry
  const int* item_nrows;       // rows of each item (1..kGroupRows)
  const int* item_roff;        // its rows at item_rows[item_roff[k] ..]
  const int* item_rows;
  const int* item_slot;        // [(item_roff[k] + j) * H + head]: slot of the (item, head) run's first piece for row j
  const int* item_chunk0;      // [item][H] first chunk of the (item, head) run
  int n_gitems;                // items [0, n_gitems) are grouped; item n_gitems + r is row r's private chain
  int n_grows;                 // rows listed by the grouped items (row r's private item lists its row at n_grows + r)
  int priv_base;               // offset of the private entries in pages[]
  int priv_np;                 // number of private page entries (NPT)
  int priv_units;              // U = H * NPT
  int priv_nchunks;
  int priv_wpc;                // warps per private CTA (ring shape: 10 -> 2 stages, 8/9 -> 3, 6/7 -> 4, 12/14 -> 2)
  int priv_warps;              // grid warps (grid = priv_warps / priv_wpc)
  int priv_static;             // warps that start on chunk = warp index (the ones that start at once)
  const int* priv_chunk_start; // [priv_nchunks + 1]
  // synthetic keys per row
  const long long* row_uid;    // leaf context uid
  const long long* row_pos;    // leaf tokens at plan time + (rank << 40)
  // append targets (written by fk_step_commit)
  const int* app_page;         // physical page or -1
  const int* app_slot;
  const long long* app_pos;    // position in the leaf (synthetic key)
};

// Device view of the KV arena and scratch.
struct ArenaDev {
  __nv_bfloat16* kv;      // [L][2][H][num_pages][16][D]
  long long num_pages;
  int num_layers;
  int num_heads;
  float* part_o;          // [rows][max_slots][H][D]  (this launch's half)
  float2* part_ml;        // [rows][max_slots][H]  (m in log2 domain, l)
  // private chunk ticket counter of this launch's half: counts from 0, and
  // the launch's merge kernel zeroes it once every CTA of the launch is done
  // (the next launch on this half is two launches later and cannot start
  // before that merge completed: see fk_merge_kernel)
  unsigned* tick;
};

// The step plan lives in __constant__ memory (one entry per pool plan slot,
// uploaded with the plan, fk_common.cuh), so a layer's kernel parameters are
// the same from step to step and the step's CUDA graph replays without
// parameter updates.
constexpr int kPlanSlots = 128;  // 64 device pools per process x 2 plan slots

inline __host__ __device__ long long plane_index(int layer, int kv, int head, int H) {
  return ((long long)layer * 2 + kv) * H + head;
}

// A launch captured as data (function, geometry, PDL flag, argument bytes):
// fk_attn_decode_layers records a step's launches and replays them as a CUDA
// graph (first time: stream capture; afterwards: kernel-node parameter
// updates), instead of issuing ~120 launches from the host every step.
struct LaunchRec {
  const void* func = nullptr;
  dim3 grid, block;
  size_t smem = 0;
  bool pdl = false;
  std::vector<unsigned char> bytes;  // argument values, each at offs[i]
  std::vector<size_t> offs;
  std::vector<void*> args;           // pointers into bytes (rebuilt by finalize())
  void finalize() {
    args.resize(offs.size());
    for (size_t i = 0; i < offs.size(); ++i) args[i] = bytes.data() + offs[i];
  }
};
// Recorded launches; entries are reused across calls (their vectors keep
// their capacity), n = how many are valid.
struct RecBuf {
  std::vector<LaunchRec> v;
  size_t n = 0;
  LaunchRec& push() {
    if (n == v.size()) v.emplace_back();
    LaunchRec& r = v[n++];
    r.bytes.clear();
    r.offs.clear();
    return r;
  }
};
// Non-null while fk_attn_decode_layers records: launch_k appends instead of launching.
extern thread_local RecBuf* g_launch_rec;


// Launchers (fk_kernels.cu, fk_prefix_tc.cu).  All return cudaError_t of the
// launch.  `ps` is the plan's constant-memory slot; `p` the host copy of the
// same plan (grid sizes).
// the plan's constant-memory copy in each translation unit that reads it
cudaError_t upload_plan_main(int ps, const PlanDev* host_pinned, cudaStream_t s);  // fk_kernels.cu
cudaError_t upload_plan_tc(int ps, const PlanDev* host_pinned, cudaStream_t s);    // fk_prefix_tc.cu
cudaError_t launch_private(const ArenaDev& a, const PlanDev& p, int ps, int layer, const void* q,
                           float scale_log2, const CUtensorMap* tmap, const CUtensorMap* tmap_half, int grid, bool pdl,
                           cudaStream_t s);
cudaError_t launch_prefix_mma(const ArenaDev& a, const PlanDev& p, int ps, int layer, const void* q,
                              float scale_log2, const CUtensorMap* tmap, cudaStream_t s);
cudaError_t launch_prefix_tc(const ArenaDev& a, const PlanDev& p, int ps, int layer, const void* q,
                             float scale_log2, const CUtensorMap* tmap, const CUtensorMap* tmap_run,
                             bool pdl, bool after_private, cudaStream_t s);
cudaError_t launch_merge(const ArenaDev& a, int ps, void* out, float* out_f32, int layer, int grid, bool pdl,
                         bool wide, cudaStream_t s);
cudaError_t launch_append(const ArenaDev& a, const PlanDev& p, int ps, int layer0, int nlayers,
                          const void* k, const void* v, cudaStream_t s);
cudaError_t launch_synth_fill(const ArenaDev& a, const int* pages_dev, int npages_first,
                              long long uid, long long pos0, long long pos1,
                              unsigned long long seed, float k_scale, cudaStream_t s);
cudaError_t launch_fill_kv(const ArenaDev& a, const int* pages_dev, int first_page, long long pos0, int ntok,
                           int layer0, int nlayers, const void* k, const void* v, cudaStream_t s);
cudaError_t launch_copy_pages(const ArenaDev& dst, const void* src_kv, long long src_num_pages, const int* pages_dev,
                              int npages, cudaStream_t s);
cudaError_t launch_synth_queries(const ArenaDev& a, const PlanDev& p, int ps, unsigned long long seed, void* q_all,
                                 int rows_cap, cudaStream_t s);
cudaError_t launch_synth_append(const ArenaDev& a, const PlanDev& p, int ps,
                                unsigned long long seed, float k_scale, cudaStream_t s);

}  // namespace fk
