// K2 on the 5th-generation tensor cores: shared-prefix decode attention for
// large fan-out (engine.py:473-483 dedup made real).
//
// Persistent CTAs (one per SM of the prefix share), stream-K over 128-token
// tile units of all tcgen05-class items (shared context x 128-query block x
// head), so every CTA streams the same number of prefix bytes.  Warp roles:
//   warp 0     TMA producer: K and V page boxes (SWIZZLE_128B) into split
//              rings -- K 3 x 32 KiB (freed as soon as S is computed), V
//              4 x 32 KiB (held through softmax and P.V); a partial last tile
//              is padded with copies of a valid page (masked later)
//   warp 1     TMEM owner + single-thread MMA issuer:
//                S[128 q x 128 tok]  = Q . K^T      (TS: Q from TMEM,
//                                                    K K-major from smem)
//                O[128 q x 128 dim] += P . V        (TS: P from TMEM,
//                                                    V MN-major from smem)
//              P is split hi + lo in bf16 (two MMAs) for ~16-bit accuracy;
//              O accumulates in TMEM across the whole piece.
//   warps 2-9  softmax: tile max (pair exchange through smem), P written
//              back over S with tcgen05.st, lazy rescale: the running max only
//              moves when a tile exceeds it by > 8 (log2), and only then is
//              the row of O in TMEM rescaled -- P <= 2^8 keeps fp32 safe.
//              Fan-out <= 64 uses the 16-lane layout (4 threads per row).
// TMEM columns: S/P buffers at 0 and 128, O at 256, Q at 384.
// Keeping Q in TMEM frees its 32 KiB of shared memory for a 4th V stage.
#include "fk_tcgen05.cuh"

#include <cstdio>

namespace fk {

constexpr int kTcSoftmaxWarps = 8;
constexpr int kTcThreads = (2 + kTcSoftmaxWarps) * 32;
constexpr int kTcKStages = 3;                      // K ring (released right after S = Q.K^T)
constexpr int kTcVStages = 4;                      // V ring (held through softmax and P.V)
constexpr int kTcHalf = 128 * 128;                 // 128 rows x 128 B
constexpr int kTcTileBytes = 2 * kTcHalf;          // one K or V tile (32 KiB)
constexpr int kTcChunkQ = 16;                      // chunk queue entries (producer lead <= ~6 chunks)
struct TcMisc {
  uint64_t k_full[kTcKStages], k_empty[kTcKStages], v_full[kTcVStages], v_empty[kTcVStages];
  uint64_t s_full[2], p_full[2], q_full;
  uint64_t cq_full[kTcChunkQ];  // chunk queue: the producer posts each chunk id it streams
  int cq[kTcChunkQ];
  uint32_t tmem_base;
  float s_max[2][2][128];  // [tile parity][half][row]
  float s_l[128];
};
constexpr int kTcSmem = (kTcKStages + kTcVStages) * kTcTileBytes + (int)sizeof(TcMisc);
static_assert(kTcSmem <= 232448, "prefix kernel exceeds the 227 KB opt-in shared memory");
constexpr uint32_t kTmemQ = 384;                   // TMEM columns of Q (A operand of S = Q.K^T):
                                                   // two 64-column buffers, piece k uses k & 1
constexpr float kRescaleThreshold = 8.0f;          // log2 units
template <bool B>
struct BoolC {
  static constexpr bool value = B;
};

#ifdef FK_TIMELINE
__device__ unsigned long long fk_tl[256];
#define TL(i) do { if (blockIdx.x == 0 && (i) < 256) fk_tl[(i)] = global_ns(); } while (0)
#else
#define TL(i) do { } while (0)
#endif

CTA_TL_DECL(fk_tl_cta_prefix);

// Tile cursor over a CTA's dynamic chunk sequence.  Chunk c covers tiles
// [tc_chunk_tile0[c], tc_chunk_tile1[c]) of item tc_chunk_item[c]; the i-th
// chunk a CTA streams is posted by its producer in queue entry i.
struct TcCursor {
  int qi;     // queue index of the current chunk
  int chunk;  // chunk id, or -1 once the counter ran dry
  int item, tile, tile1;
};
__device__ __forceinline__ void tc_load_chunk(const PlanDev& p, TcCursor& c, int chunk) {
  c.chunk = chunk;
  if (chunk >= 0) {
    c.item = p.tc_chunk_item[chunk];
    c.tile = p.tc_chunk_tile0[chunk];
    c.tile1 = p.tc_chunk_tile1[chunk];
  }
}
// consumers: read queue entry i (posted by this CTA's producer)
__device__ __forceinline__ int tc_read_queue(uint64_t* cq_full, const int* cq, int i) {
  mbar_wait(&cq_full[i % kTcChunkQ], (i / kTcChunkQ) & 1);
  return ((volatile const int*)cq)[i % kTcChunkQ];
}

__global__ void __launch_bounds__(kTcThreads, 1) fk_prefix_tc_kernel(ArenaDev a, int ps, int layer,
                                                                     const __nv_bfloat16* __restrict__ q,
                                                                     float scale_log2,
                                                                     const __grid_constant__ CUtensorMap tmap,
                                                                     const __grid_constant__ CUtensorMap tmap_run,
                                                                     int after_private) {
  const PlanDev& p = fk_plan_c[ps];
  // all shared state is dynamic (no static smem), so the buffer starts at
  // the 1 KiB-aligned base SWIZZLE_128B needs
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem;
  uint8_t* sV = smem + kTcKStages * kTcTileBytes;
  TcMisc& ms = *reinterpret_cast<TcMisc*>(smem + (kTcKStages + kTcVStages) * kTcTileBytes);
  uint64_t* k_full = ms.k_full;
  uint64_t* k_empty = ms.k_empty;
  uint64_t* v_full = ms.v_full;
  uint64_t* v_empty = ms.v_empty;
  uint64_t* s_full = ms.s_full;
  uint64_t* p_full = ms.p_full;
  uint64_t& q_full = ms.q_full;
  uint32_t& tmem_base_sh = ms.tmem_base;
  auto& s_max = ms.s_max;
  auto& s_l = ms.s_l;
  if ((smem_u32(smem) & 1023u) != 0) __trap();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.num_heads;
  // the private grid may start at once on the SMs this grid leaves free
  pdl_launch_dependents();
  // Launched behind the private grid (launch order 1), this grid's completion
  // must imply that grid's: thread 0 waits for it on exit.
  if ((int)blockIdx.x >= p.tc_ctas || p.tc_cta_chunk0[blockIdx.x] == p.tc_cta_chunk0[blockIdx.x + 1]) {
    // (exit triggers the dependents)
    if (after_private && threadIdx.x == 0) pdl_wait_primary();
    return;
  }
  TL(160);
  CTA_TL_START(fk_tl_cta_prefix, layer);

  // The producer's first chunk metadata and page window (three dependent
  // global loads) are fetched while warps 1 and 2 set up TMEM and the
  // barriers, so the first TMA load goes out right after the CTA barrier.
  int sidx = 0, send = 0, f_item = 0, f_tile0 = 0, f_tile1 = 0, f_head = 0, f_npi = 0, f_poff = 0, f_win = 0, f_nwin = 0;
  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmap);
      prefetch_tmap(&tmap_run);
    }
    sidx = p.tc_cta_chunk0[blockIdx.x];
    send = p.tc_cta_chunk0[blockIdx.x + 1];
    f_item = p.tc_chunk_item[sidx];
    f_tile0 = p.tc_chunk_tile0[sidx];
    f_tile1 = p.tc_chunk_tile1[sidx];
    f_head = p.it_head[f_item];
    f_npi = p.it_npages[f_item];
    f_poff = p.it_page_off[f_item];
    const int wb = f_tile0 * kTcTilePages;
    f_win = wb + lane < f_npi ? p.pages[f_poff + wb + lane] : 0;
    f_nwin = wb + 32 + lane < f_npi ? p.pages[f_poff + wb + 32 + lane] : 0;
  }
  if (threadIdx.x == 64) {  // (warp 2: warp 0 is busy with the loads above)
    for (int s = 0; s < kTcKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kTcVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], kTcSoftmaxWarps);
    }
    mbar_init(&q_full, kTcSoftmaxWarps);
    for (int i = 0; i < kTcChunkQ; ++i) mbar_init(&ms.cq_full[i], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base_sh;
  uint64_t* cq_full = ms.cq_full;
  int* cq = ms.cq;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // Chunks: the CTA's range of the plan's chunk list; lane 0 posts each
    // chunk id in the queue one chunk ahead of streaming it.  Page ids are prefetched lane-parallel
    // into a 2 x 32-entry register window; the next chunk's item metadata and
    // first window are fetched over the following two tiles, so a chunk
    // switch never waits on a dependent global load.  Lane 0 issues the TMA.
    auto grab = [&]() -> int { return sidx < send ? sidx++ : -1; };
    auto post = [&](int i, int chunk) {
      if (lane == 0) {
        ((volatile int*)cq)[i % kTcChunkQ] = chunk;
        mbar_arrive(&cq_full[i % kTcChunkQ]);
      }
    };
    TcCursor c;
    c.qi = 0;
    c.chunk = grab();  // every CTA has at least one static chunk (prefetched above)
    c.item = f_item;
    c.tile = f_tile0;
    c.tile1 = f_tile1;
    post(0, c.chunk);
    int nxt = grab();  // the chunk after the current one, posted right away
    post(1, nxt);
    int head = f_head, npi = f_npi, poff = f_poff;
    int wbase = c.tile * kTcTilePages;
    int win = f_win, nwin = f_nwin;
    int n_item = 0, n_tile0 = 0, n_tile1 = 0, n_head = 0, n_npi = 0, n_poff = 0, n_win = 0, n_nwin = 0;
    int n_stage = 0;  // 0 nothing, 1 metadata, 2 metadata + first window of chunk `nxt`
    for (int t = 0;; ++t) {
      if (c.tile == c.tile1) {  // current chunk done: switch to `nxt`
        if (nxt < 0) break;
        if (n_stage < 1) {
          n_item = p.tc_chunk_item[nxt];
          n_tile0 = p.tc_chunk_tile0[nxt];
          n_tile1 = p.tc_chunk_tile1[nxt];
          n_head = p.it_head[n_item];
          n_npi = p.it_npages[n_item];
          n_poff = p.it_page_off[n_item];
        }
        if (n_stage < 2) {
          const int wb = n_tile0 * kTcTilePages;
          n_win = wb + lane < n_npi ? p.pages[n_poff + wb + lane] : 0;
          n_nwin = wb + 32 + lane < n_npi ? p.pages[n_poff + wb + 32 + lane] : 0;
        }
        ++c.qi;
        c.chunk = nxt;
        c.item = n_item;
        c.tile = n_tile0;
        c.tile1 = n_tile1;
        head = n_head;
        npi = n_npi;
        poff = n_poff;
        wbase = n_tile0 * kTcTilePages;
        win = n_win;
        nwin = n_nwin;
        n_stage = 0;
        nxt = grab();
        post(c.qi + 1, nxt);
      } else if (nxt >= 0) {
        if (n_stage == 1) {
          const int wb = n_tile0 * kTcTilePages;
          n_win = wb + lane < n_npi ? p.pages[n_poff + wb + lane] : 0;
          n_nwin = wb + 32 + lane < n_npi ? p.pages[n_poff + wb + 32 + lane] : 0;
          n_stage = 2;
        } else if (n_stage == 0) {
          n_item = p.tc_chunk_item[nxt];
          n_tile0 = p.tc_chunk_tile0[nxt];
          n_tile1 = p.tc_chunk_tile1[nxt];
          n_head = p.it_head[n_item];
          n_npi = p.it_npages[n_item];
          n_poff = p.it_page_off[n_item];
          n_stage = 1;
        }
      }
      const int pg0 = c.tile * kTcTilePages;
      if (pg0 >= wbase + 32) {  // slide the window
        wbase += 32;
        win = nwin;
        nwin = wbase + 32 + lane < npi ? p.pages[poff + wbase + 32 + lane] : 0;
      }
      const int np = min(kTcTilePages, npi - pg0);
      int pl[kTcTilePages];
#pragma unroll
      for (int j = 0; j < kTcTilePages; ++j) pl[j] = __shfl_sync(0xffffffffu, win, pg0 - wbase + (j < np ? j : 0));
      if (lane == 0) {
        const int planeK = (int)plane_index(layer, 0, head, H), planeV = (int)plane_index(layer, 1, head, H);
        // 8 physically consecutive pages -> one 128-row box per half (the
        // common case: a context's pages come from one allocation);
        // otherwise one 16-row box per page, a partial tile padded with a
        // valid (masked) page
        bool run = np == kTcTilePages;
#pragma unroll
        for (int j = 1; j < kTcTilePages; ++j) run = run && pl[j] == pl[0] + j;
        auto load_tile = [&](uint8_t* st, int plane, uint64_t* bar) {
          mbar_expect_tx(bar, kTcTilePages * 2 * 2048);
          // evict-first: a tile is read once per layer (measured +3-4 % per
          // step); with mirrored query-block CTAs (tc_l2_share) the default
          // policy, so the partner CTA's read of the tile hits L2
          const uint64_t pol = p.tc_l2_share ? l2_policy_evict_normal() : l2_policy_evict_first();
          if (run) {
            tma_load_3d_hint(st, &tmap_run, 0, pl[0] * kPage, plane, bar, pol);
            tma_load_3d_hint(st + kTcHalf, &tmap_run, 64, pl[0] * kPage, plane, bar, pol);
          } else {
#pragma unroll
            for (int j = 0; j < kTcTilePages; ++j) {
              tma_load_3d_hint(st + j * 2048, &tmap, 0, pl[j] * kPage, plane, bar, pol);
              tma_load_3d_hint(st + kTcHalf + j * 2048, &tmap, 64, pl[j] * kPage, plane, bar, pol);
            }
          }
        };
        const int sk = t % kTcKStages, sv = t % kTcVStages;
        if (t >= kTcKStages) mbar_wait(&k_empty[sk], ((t / kTcKStages) - 1) & 1);
        if (t < 16) TL(128 + t);
        load_tile(sK + sk * kTcTileBytes, planeK, &k_full[sk]);
        if (t >= kTcVStages) mbar_wait(&v_empty[sv], ((t / kTcVStages) - 1) & 1);
        load_tile(sV + sv * kTcTileBytes, planeV, &v_full[sv]);
      }
      __syncwarp();
      ++c.tile;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Two in-order streams polled by one thread: S(t) = Q.K^T as soon as K(t)
    // lands (and, at a chunk start, its Q is staged), PV(t) as soon as P(t)
    // and V(t) are ready.  S(t) reuses the TMEM buffer of P(t-2), so it is
    // only issued after PV(t-2) (the tensor pipe executes in issue order).
    // Every chunk is a piece: P.V restarts its accumulator at a chunk start.
    if (lane == 0) {
      TcCursor cs, cp;
      cs.qi = cp.qi = 0;
      tc_load_chunk(p, cs, tc_read_queue(cq_full, cq, 0));
      cp = cs;
      bool s_new = true, p_new = true;  // the next S / PV is a chunk's first tile
      int ts = 0, tp = 0;
      while (cp.chunk >= 0) {
        if (cs.chunk >= 0 && ts <= tp + 1) {
          const int s = ts % kTcKStages;
          if ((!s_new || mbar_try_wait(&q_full, cs.qi & 1)) && mbar_try_wait(&k_full[s], (ts / kTcKStages) & 1)) {
            const uint32_t q_tm = tm + kTmemQ + (uint32_t)((cs.qi & 1) * 64);
            if (ts < 16) TL(ts);
            tc_fence_after();
            const uint32_t kaddr = smem_u32(sK + s * kTcTileBytes);
            const int sb = ts & 1;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t off = (kk >> 2) * kTcHalf + (kk & 3) * 32;
              mma_ts(tm + sb * 128, q_tm + kk * 8, sdesc(kaddr + off, 16, 1024), kIdescQK, kk > 0);
            }
            mma_commit(&s_full[sb]);
            mma_commit(&k_empty[s]);
            if (ts < 16) TL(16 + ts);
            ++ts;
            s_new = false;
            if (++cs.tile == cs.tile1) {
              ++cs.qi;
              tc_load_chunk(p, cs, tc_read_queue(cq_full, cq, cs.qi));
              s_new = true;
            }
            continue;
          }
        }
        {
          const int sb = tp & 1, s = tp % kTcVStages;
          if (tp < ts && mbar_try_wait(&p_full[sb], (tp >> 1) & 1) && mbar_try_wait(&v_full[s], (tp / kTcVStages) & 1)) {
            if (tp < 16) TL(32 + tp);
            tc_fence_after();
            const uint32_t vaddr = smem_u32(sV + s * kTcTileBytes);
            const uint32_t p_tm = tm + sb * 128;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint64_t bdesc = sdesc(vaddr + kk * 2048, kTcHalf, 1024);
              mma_ts(tm + 256, p_tm + kk * 16, bdesc, kIdescPV, (!p_new || kk > 0) ? 1u : 0u);
              mma_ts(tm + 256, p_tm + kk * 16 + 8, bdesc, kIdescPV, 1u);
            }
            mma_commit(&v_empty[s]);  // also "O includes PV(tp)" for the softmax warps
            if (tp < 16) TL(48 + tp);
            ++tp;
            p_new = false;
            if (++cp.tile == cp.tile1) {
              ++cp.qi;
              tc_load_chunk(p, cp, tc_read_queue(cq_full, cq, cp.qi));
              p_new = true;
            }
          }
        }
      }
    }
  } else {
    // ------------------------------------------------- softmax / epilogue
    // Two thread->score layouts, chosen per piece:
    //  * 32-lane (fan-out > 64): thread = one TMEM lane (query row) of its
    //    warp's quarter, 64 score columns (half = which 64);
    //  * 16-lane (fan-out <= 64): only lanes 0-15 of each quarter hold real
    //    rows, so the warp reads them with the 16x32bx2 shape and each thread
    //    owns 32 columns (sub = lane / 16 picks which 32 of its half's 64):
    //    half the TMEM reads, exp2s and conversions per thread.
    const int quarter = warp & 3;               // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;           // which 64 score columns / 64 O columns
    const int row = quarter * 32 + lane;        // Q staging row (32-lane view)
    // query j sits in TMEM lane 32*(j%4) + j/4: a partial block spreads its
    // rows over all four lane quarters, i.e. over all four SM sub-partitions
    const int qj = 4 * lane + quarter;
    const int sub = lane >> 4;
    const int row16 = quarter * 32 + (lane & 15);
    const int qj16 = 4 * (lane & 15) + quarter;
    const uint32_t lane_tm = tm + ((uint32_t)(quarter * 32) << 16);
    const int bar_id = 1 + quarter;             // named barrier of the two warps sharing these rows
    float m = -INFINITY, l = 0.f;
    int nq = 0, head = 0, ntok = 0;
    bool active = false, r16 = false;
    // Q of the chunk at queue index k -> TMEM buffer k & 1 (this thread's half
    // of its row; the A operand layout of S = Q.K^T: row = lane, 2 bf16 per
    // 32-bit column).  The next chunk's Q is staged while this chunk's last
    // P.V runs, so S of the next chunk does not wait for the epilogue.
    // (a chunk's last tile prefetches the next chunk's Q lines into L1 --
    // prefetch_q, no registers held -- and its piece end loads and stages them)
    auto q_line = [&](int it) -> const uint4* {
      return qj < p.it_nq[it] ? reinterpret_cast<const uint4*>(
                                    q + ((long long)p.qrows[p.it_q_off[it] + qj] * H + p.it_head[it]) * kHeadDim) +
                                    half * 8
                              : nullptr;
    };
    auto prefetch_q = [&](int it) {
      const uint4* src = q_line(it);
      if (src) asm volatile("prefetch.global.L1 [%0];" ::"l"(src));
    };
    auto stage_q = [&](int it, int k) {
      const uint4* src = q_line(it);
      uint32_t qr[32];
#pragma unroll
      for (int k8 = 0; k8 < 8; ++k8) {
        const uint4 v = src ? src[k8] : make_uint4(0u, 0u, 0u, 0u);
        qr[4 * k8] = v.x;
        qr[4 * k8 + 1] = v.y;
        qr[4 * k8 + 2] = v.z;
        qr[4 * k8 + 3] = v.w;
      }
      tmem_st32(lane_tm + kTmemQ + (uint32_t)((k & 1) * 64) + half * 32, qr);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_full);
    };
    // under cross-layer PDL the previous layer's merge may still be running:
    // q and the partials are touched only after it has completed
    if (!after_private) pdl_wait_primary();
    TcCursor c;
    c.qi = 0;
    tc_load_chunk(p, c, tc_read_queue(cq_full, cq, 0));
    stage_q(c.item, 0);
    bool chunk_start = true;
    int t = 0;
    for (; c.chunk >= 0; ++t) {
      const int item = c.item;
      if (chunk_start) {
        nq = p.it_nq[item];
        head = p.it_head[item];
        ntok = p.it_ntok[item];
        active = quarter < nq;
        r16 = nq <= 64;
        m = -INFINITY;
        l = 0.f;
      }
      // the last tile of a chunk: the next chunk's Q loads go out now and
      // land while this tile's scores are processed
      const bool piece_end = c.tile + 1 == c.tile1;  // every chunk is one piece
      const int next = piece_end ? tc_read_queue(cq_full, cq, c.qi + 1) : -1;
      if (next >= 0) prefetch_q(p.tc_chunk_item[next]);
      const int sb = t & 1;
      mbar_wait(&s_full[sb], (t >> 1) & 1);
      if (warp == 4 && lane == 0 && t < 16) TL(64 + t);
      tc_fence_after();
      // "O includes PV(u)" is v_empty[u % kTcVStages] completing its phase
      // u / kTcVStages (committed right after PV(u); the producer waits for
      // every phase before it reuses the stage, so no phase goes unobserved).
      // s_full(t) implies PV(t-2) is done (issued before S(t), in-order
      // pipe), so the phases before the awaited one have completed and the
      // next one cannot (it needs P(u + kTcVStages)): the parity waits for
      // PV(t-1) here and PV(t) at a piece end are unambiguous.
      if (active) {
        auto tile = [&](auto mode) {
          constexpr bool R16 = decltype(mode)::value;
          constexpr int NCH = R16 ? 1 : 2;  // 32-column chunks per thread
          const int my_row = R16 ? row16 : row;
          const int col0 = half * 64 + (R16 ? sub * 32 : 0);
          const int valid = ntok - c.tile * 128 - col0;  // valid columns among this thread's
          const uint32_t s_tm = lane_tm + sb * 128 + half * 64;
          uint32_t r[NCH][32];
#pragma unroll
          for (int cc = 0; cc < NCH; ++cc) {
            if (R16) tmem_ld16x2(s_tm, r[cc]);
            else tmem_ld32(s_tm + cc * 32, r[cc]);
          }
          tmem_wait_ld();
          if (warp == 4 && lane == 0 && t < 16) TL(176 + t);
          float mx = -INFINITY;
          if (valid >= 32 * NCH) {  // full: tree max, no masking
#pragma unroll
            for (int cc = 0; cc < NCH; ++cc) {
              float t8[8];
#pragma unroll
              for (int k = 0; k < 8; ++k)
                t8[k] = fmaxf(fmaxf(__uint_as_float(r[cc][4 * k]), __uint_as_float(r[cc][4 * k + 1])),
                              fmaxf(__uint_as_float(r[cc][4 * k + 2]), __uint_as_float(r[cc][4 * k + 3])));
              mx = fmaxf(mx, fmaxf(fmaxf(fmaxf(t8[0], t8[1]), fmaxf(t8[2], t8[3])),
                                   fmaxf(fmaxf(t8[4], t8[5]), fmaxf(t8[6], t8[7]))));
            }
          } else {
#pragma unroll
            for (int cc = 0; cc < NCH; ++cc)
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (cc * 32 + e < valid) mx = fmaxf(mx, __uint_as_float(r[cc][e]));
          }
          if (R16) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
          s_max[sb][half][my_row] = mx;
          asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
          if (warp == 4 && lane == 0 && t < 16) TL(192 + t);
          const float tile_max = fmaxf(mx, s_max[sb][half ^ 1][my_row]) * scale_log2;
          // lazy rescale: a row keeps its running max unless the tile exceeds
          // it by > 8.  tcgen05.ld/st are warp-collective (.sync.aligned), so
          // the O rescale runs for the whole warp when any of its rows needs
          // it (alpha = 1 for the others).
          const bool rescale = tile_max > m + kRescaleThreshold;
          const bool warp_rescale = __any_sync(0xffffffffu, rescale) && !chunk_start;
          if (t > 0 && (warp_rescale || piece_end))
            mbar_wait(&v_empty[(t - 1) % kTcVStages], ((t - 1) / kTcVStages) & 1);
          if (warp_rescale) {
            const float alpha = rescale ? ex2(m - tile_max) : 1.f;
            l *= alpha;
            tc_fence_after();
            const uint32_t o_tm = lane_tm + 256 + half * 64;
#pragma unroll
            for (int cc = 0; cc < NCH; ++cc) {
              uint32_t o[32];
              if (R16) tmem_ld16x2(o_tm, o);
              else tmem_ld32(o_tm + cc * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              if (R16) tmem_st16x2(o_tm, o);
              else tmem_st32(o_tm + cc * 32, o);
            }
          }
          if (rescale) m = tile_max;
          float sum4[4] = {0.f, 0.f, 0.f, 0.f};
          const bool full = valid >= 32 * NCH;
#pragma unroll
          for (int cc = 0; cc < NCH; ++cc) {
            // per 16-token k-step: 8 columns of bf16x2 P_hi then 8 of P_lo.
            // hi = p truncated to bf16, lo = (p - hi) truncated: ~16 mantissa
            // bits from two byte-permutes and one subtract (no F2F converts)
            uint32_t pk[32];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int c2 = cc * 32 + 2 * e;
              float p0 = ex2(fmaf(__uint_as_float(r[cc][2 * e]), scale_log2, -m));
              float p1 = ex2(fmaf(__uint_as_float(r[cc][2 * e + 1]), scale_log2, -m));
              if (!full) {
                p0 = c2 < valid ? p0 : 0.f;
                p1 = c2 + 1 < valid ? p1 : 0.f;
              }
              sum4[e & 3] += p0 + p1;
              const uint32_t u0 = __float_as_uint(p0), u1 = __float_as_uint(p1);
              pk[(e >> 3) * 16 + (e & 7)] = __byte_perm(u0, u1, 0x7632);
              const float l0 = p0 - __uint_as_float(u0 & 0xFFFF0000u);
              const float l1 = p1 - __uint_as_float(u1 & 0xFFFF0000u);
              pk[(e >> 3) * 16 + 8 + (e & 7)] = __byte_perm(__float_as_uint(l0), __float_as_uint(l1), 0x7632);
            }
            if (R16) tmem_st16x2(s_tm, pk);
            else tmem_st32(s_tm + cc * 32, pk);
          }
          l += (sum4[0] + sum4[1]) + (sum4[2] + sum4[3]);
          if (warp == 4 && lane == 0 && t < 16) TL(208 + t);
          tmem_wait_st();
          if (warp == 4 && lane == 0 && t < 16) TL(224 + t);
        };
        if (r16) tile(BoolC<true>{});
        else tile(BoolC<false>{});
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[sb]);
      if (warp == 4 && lane == 0 && t < 16) TL(80 + t);
      const int chunk = c.chunk;
      chunk_start = false;
      if (piece_end) {
        // next chunk's Q first (S of its first tile can then run under this
        // epilogue), then O (unnormalised, running max m) -> partial slot
        if (warp == 4 && lane == 0) TL(243 + min(c.qi, 3) * 4);
        if (next >= 0) stage_q(p.tc_chunk_item[next], c.qi + 1);
        if (warp == 2 && lane == 0) CTA_TL_NOTE(fk_tl_cta_prefix, layer, 3, c.qi + 1);
        mbar_wait(&v_empty[t % kTcVStages], (t / kTcVStages) & 1);
        if (warp == 4 && lane == 0 && t < 16) TL(96 + t);
        tc_fence_after();
        if (active) {
          auto epilogue = [&](auto mode) {
            constexpr bool R16 = decltype(mode)::value;
            constexpr int NCH = R16 ? 1 : 2;
            const int my_row = R16 ? row16 : row;
            const int my_q = R16 ? qj16 : qj;
            const int col0 = half * 64 + (R16 ? sub * 32 : 0);
            const int piece = chunk - p.it_first_chunk[item];
            const bool real = my_q < nq;
            long long pi = 0;
            int r = 0;
            if (real) {
              r = p.qrows[p.it_q_off[item] + my_q];
              const int k = p.qslot[p.it_qslot_off[item] + my_q] + piece;
              pi = part_index(p, H, r, k, head);
            }
            const uint32_t o_tm = lane_tm + 256 + half * 64;
#pragma unroll
            for (int cc = 0; cc < NCH; ++cc) {
              uint32_t o[32];
              if (R16) tmem_ld16x2(o_tm, o);
              else tmem_ld32(o_tm + cc * 32, o);
              tmem_wait_ld();
              if (warp == 4 && lane == 0 && cc == 0) TL(240 + min(c.qi, 3) * 4);
              if (real) {
                float4* po = reinterpret_cast<float4*>(a.part_o + pi * kHeadDim + col0 + cc * 32);
#pragma unroll
                for (int i4 = 0; i4 < 8; ++i4)
                  po[i4] = make_float4(__uint_as_float(o[4 * i4]), __uint_as_float(o[4 * i4 + 1]),
                                       __uint_as_float(o[4 * i4 + 2]), __uint_as_float(o[4 * i4 + 3]));
              }
            }
            if (warp == 4 && lane == 0) TL(241 + min(c.qi, 3) * 4);
            float lr = l;
            if (R16) lr += __shfl_xor_sync(0xffffffffu, lr, 16);
            const bool lead = !R16 || sub == 0;
            if (half == 1 && lead) s_l[my_row] = lr;
            asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
            if (warp == 4 && lane == 0) TL(242 + min(c.qi, 3) * 4);
            if (half == 0 && lead && real) a.part_ml[pi] = make_float2(m, lr + s_l[my_row]);
          };
          if (r16) epilogue(BoolC<true>{});
          else epilogue(BoolC<false>{});
        }
        tc_fence_before();
        if (warp == 4 && lane == 0 && t < 16) TL(112 + t);
        ++c.qi;
        tc_load_chunk(p, c, next);
        chunk_start = true;
      } else {
        ++c.tile;
      }
    }
    if (warp == 2 && lane == 0) CTA_TL_NOTE(fk_tl_cta_prefix, layer, 2, t);
  }
  tc_fence_before();
  __syncthreads();
  CTA_TL_END(fk_tl_cta_prefix, layer);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
  }
  if (after_private && threadIdx.x == 0) pdl_wait_primary();
}

extern "C" int fk_debug_cta_timeline_prefix(unsigned long long* out, int n) {
#ifdef FK_TIMELINE
  if (cudaDeviceSynchronize() != cudaSuccess) return 6;
  return cudaMemcpyFromSymbol(out, fk_tl_cta_prefix, sizeof(unsigned long long) * 8 * (n < 1024 ? n : 1024)) == cudaSuccess ? 0 : 6;
#else
  (void)out;
  (void)n;
  return 5;
#endif
}

extern "C" int fk_debug_timeline(unsigned long long* out, int n) {
#ifdef FK_TIMELINE
  if (cudaDeviceSynchronize() != cudaSuccess) return 6;
  return cudaMemcpyFromSymbol(out, fk_tl, sizeof(unsigned long long) * (n < 256 ? n : 256)) == cudaSuccess ? 0 : 6;
#else
  (void)out;
  (void)n;
  return 5;
#endif
}

cudaError_t upload_plan_tc(int ps, const PlanDev* host_pinned, cudaStream_t s) {
  return cudaMemcpyToSymbolAsync(fk_plan_c, host_pinned, sizeof(PlanDev), (size_t)ps * sizeof(PlanDev),
                                 cudaMemcpyHostToDevice, s);
}

cudaError_t launch_prefix_tc(const ArenaDev& a, const PlanDev& p, int ps, int layer, const void* q, float scale_log2,
                             const CUtensorMap* tmap, const CUtensorMap* tmap_run, bool pdl, bool after_private,
                             cudaStream_t s) {
  static unsigned long long attr_devices = 0;
  if (!attr_set_on_device(attr_devices)) {
    cudaError_t e = cudaFuncSetAttribute(fk_prefix_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
    if (e != cudaSuccess) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, fk_prefix_tc_kernel);
      int optin = 0, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      fprintf(stderr, "fk_prefix_tc smem attr: %s (static %zu, dyn %d, optin %d, regs %d, local %zu)\n",
              cudaGetErrorString(e), fa.sharedSizeBytes, kTcSmem, optin, fa.numRegs, fa.localSizeBytes);
      return e;
    }
  }
  if (p.tc_ctas == 0) return cudaSuccess;
  return launch_k(fk_prefix_tc_kernel, dim3(p.tc_grid > p.tc_ctas ? p.tc_grid : p.tc_ctas), dim3(kTcThreads), kTcSmem, s, pdl, a, ps, layer,
                  (const __nv_bfloat16*)q, scale_log2, *tmap, *tmap_run, after_private ? 1 : 0);
}

}  // namespace fk
