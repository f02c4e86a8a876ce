// sm_100a decode-attention kernels for shared-prefix ("fork") batches.
//
//  K3  fk_private_kernel    fan-out-1 contexts (the per-request suffix,
//                           engine.py:484 per-request chain cost): warps take
//                           guided chunks of (head, page) units from a ticket
//                           counter, TMA page boxes into per-warp 3-stage smem
//                           rings, q.K^T and P.V on mma.sync, one partial per
//                           (row, head, chunk) piece.
//  K2  fk_prefix_mma_kernel shared contexts on the warp-level path (opt-in,
//                           FK_OPT_TC_MIN_FANOUT): per (context split, 64-query
//                           block, head), TMA (SWIZZLE_128B) page tiles, mma.sync.
//                           The default K2 is fk_prefix_tc_kernel (tcgen05).
//  K4  fk_merge_kernel      LSE merge of every (row, head)'s partials
//                           ("amalgamating ... interim results").
//  K1  fk_append_kernel     new K/V rows -> (page, slot); fk_fill_kv_kernel and
//                           fk_copy_pages_kernel fill / migrate context KV.
//      fk_synth_*           deterministic synthetic KV / Q (oracle restates).
#include "fk_common.cuh"

namespace fk {

thread_local RecBuf* g_launch_rec = nullptr;

// =========================================================== private (n_c=1)
// Units u = (head, flat private page entry e), head-major.  The plan cuts the
// unit list into chunks of decreasing size (guided: big first, 4-unit ones
// at the end) and every warp grabs chunk after chunk from a ticket counter,
// streaming each chunk's pages through its own 3-stage smem ring (TMA,
// SWIZZLE_128B boxes {64 dims, 16 tokens}: K lo/hi, V lo/hi = 8 KiB per
// page).  Slow SMs simply take fewer chunks, and CTAs that only get an SM
// when the tcgen05 prefix CTAs retire take the leftovers -- no static tail.
// Per page, transposed so that M = 16 is the page's tokens / a 16-dim slice:
// S^T = K.q^T (8 mma.sync m16n8k16, the K tile as stored is the A operand)
// and o^T += V^T.[p_hi p_lo]^T (8, V^T through ldmatrix.trans; P split hi +
// lo into B columns 0 and 1, summed at the end): 16 MMAs per page against
// 48 in the q-in-row-0 form (measured +2 to +3 %, and +0.6 % for the column
// trick).
// A chunk always ends a piece: (row, head, chunk) -> one partial slot
// row_head_base + (chunk - first chunk of the item), fixed by the plan.
constexpr int kPwStageBytes = 8192;
template <int STAGES, int WARPS>
constexpr int priv_smem() { return WARPS * STAGES * kPwStageBytes + 1024; }

// byte offset of (token row 0..15, 16-byte chunk 0..15) in one K or V page
// held as two SWIZZLE_128B boxes of 16 rows x 128 B
__device__ __forceinline__ uint32_t sw_page(int row, int c16) {
  return (uint32_t)((c16 >> 3) * 2048 + row * 128 + (((c16 & 7) ^ (row & 7)) << 4));
}

struct UnitMeta {
  int pg, ntok, item, head, nr;  // nr: rows of the item (1 = a private chain)
};

CTA_TL_DECL(fk_tl_cta_priv);

// Streaming warps only write partials; fk_merge_kernel combines them.
// With PDL this grid can start while the prefix grid of the same layer is
// still running (disjoint partial slots); thread 0 of each CTA waits for that
// grid before exiting so "private grid complete" implies "prefix complete".
struct PdlTail {
  __device__ ~PdlTail() {
    if (threadIdx.x == 0) pdl_wait_primary();
  }
};
// GROUPED: the plan has row-group items (small-fan-out shared contexts);
// without them the single-row path is the whole kernel.
template <int STAGES, int WARPS, bool GROUPED>
__global__ void __launch_bounds__(WARPS * 32, 1) fk_private_kernel(ArenaDev a, int ps, int layer,
                                                                   const __nv_bfloat16* __restrict__ q,
                                                                   float scale_log2,
                                                                   const __grid_constant__ CUtensorMap tmap,
                                                                   const __grid_constant__ CUtensorMap tmap_h) {
  const PlanDev& p = fk_plan_c[ps];
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[WARPS][STAGES];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.num_heads;
  CTA_TL_START(fk_tl_cta_priv, layer);
#ifdef FK_TIMELINE
  if (threadIdx.x == 0 && blockIdx.x < 1024) fk_tl_cta_priv[layer & 1][blockIdx.x][3] = 0;
#endif
  pdl_launch_dependents();  // the merge kernel may launch now (it waits for us)
  PdlTail tail;             // on exit: this grid completes only after the prefix grid

  const int g = lane >> 2, t4 = lane & 3;
  const int NPT = p.priv_np, nch = p.priv_nchunks;
  // The warps of the CTAs that start at once (the first priv_static of the
  // grid) begin on chunk = their global warp index, with no ticket round trip
  // before their first loads; every later chunk comes from a ticket:
  // chunk = priv_static + ticket, the counter (this launch's half) starting
  // at 0 and reset by the launch's merge kernel.  Each warp stops after its
  // first failing ticket.
  const int gw = blockIdx.x * WARPS + warp;
  auto grab = [&]() -> int {
    int c = 0;
    if (lane == 0) c = p.priv_static + (int)atomicAdd(a.tick, 1u);
    return __shfl_sync(0xffffffffu, c, 0);
  };
  int ca = gw < p.priv_static ? gw : grab();
  if (ca >= nch) return;

  uint8_t* ring = smem + warp * STAGES * kPwStageBytes;
  if (lane == 0) {
    prefetch_tmap(&tmap);
    prefetch_tmap(&tmap_h);
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[warp][s], 1);
    fence_mbar_init();
  }
  // A chain's last page with <= 8 tokens loads only its first 8 rows; rows
  // 8..15 of the stage keep an earlier page's (finite) bytes, which meet
  // p = 0.  Zero them once so the first use of a stage sees no NaN bits.
#pragma unroll
  for (int s = 0; s < STAGES; ++s)
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      uint4* z = reinterpret_cast<uint4*>(ring + s * kPwStageBytes + x * 2048 + 1024);
      z[lane] = z[lane + 32] = make_uint4(0u, 0u, 0u, 0u);
    }
  fence_proxy_async();  // before the TMA (async proxy) writes the same stages
  __syncwarp();

  // unit metadata of a chunk (<= 32 units) held lane-parallel in registers
  auto load_chunk = [&](int c, int& len) {
    UnitMeta m{0, 0, 0, 0, 1};
    len = 0;
    if (c < nch) {
      const int u0 = p.priv_chunk_start[c];
      len = p.priv_chunk_start[c + 1] - u0;
      if (lane < len) {
        const int u = u0 + lane;
        const int e = u % NPT;
        m.head = u / NPT;
        m.pg = p.pages[p.priv_base + e];
        m.ntok = p.page_ntok[p.priv_base + e];
        m.item = p.page_item[e];
        m.nr = (!GROUPED || m.item >= p.n_gitems) ? 1 : p.item_nrows[m.item];
      }
    }
    return m;
  };
  auto sh = [&](const UnitMeta& m, int i) {
    UnitMeta r;
    r.pg = __shfl_sync(0xffffffffu, m.pg, i);
    r.ntok = __shfl_sync(0xffffffffu, m.ntok, i);
    r.item = __shfl_sync(0xffffffffu, m.item, i);
    r.head = __shfl_sync(0xffffffffu, m.head, i);
    r.nr = __shfl_sync(0xffffffffu, m.nr, i);
    return r;
  };
  auto issue = [&](int s, const UnitMeta& m) {  // lane 0 only
    uint8_t* st = ring + s * kPwStageBytes;
    const int pk = (int)plane_index(layer, 0, m.head, H), pv = (int)plane_index(layer, 1, m.head, H);
    // every private page is read once per layer: evict-first keeps L2 for the
    // partials and the prefix tiles
    const uint64_t pol = l2_policy_evict_first();
    if (m.ntok <= kPage / 2) {  // a chain's short last page: its first 8 rows only
      mbar_expect_tx(&full[warp][s], kPwStageBytes / 2);
      tma_load_3d_hint(st, &tmap_h, 0, m.pg * kPage, pk, &full[warp][s], pol);
      tma_load_3d_hint(st + 2048, &tmap_h, 64, m.pg * kPage, pk, &full[warp][s], pol);
      tma_load_3d_hint(st + 4096, &tmap_h, 0, m.pg * kPage, pv, &full[warp][s], pol);
      tma_load_3d_hint(st + 6144, &tmap_h, 64, m.pg * kPage, pv, &full[warp][s], pol);
      return;
    }
    mbar_expect_tx(&full[warp][s], kPwStageBytes);
    tma_load_3d_hint(st, &tmap, 0, m.pg * kPage, pk, &full[warp][s], pol);
    tma_load_3d_hint(st + 2048, &tmap, 64, m.pg * kPage, pk, &full[warp][s], pol);
    tma_load_3d_hint(st + 4096, &tmap, 0, m.pg * kPage, pv, &full[warp][s], pol);
    tma_load_3d_hint(st + 6144, &tmap, 64, m.pg * kPage, pv, &full[warp][s], pol);
  };

  int la = 0, lb = 0;
  UnitMeta ma = load_chunk(ca, la);
  int cb = grab();
  UnitMeta mb = load_chunk(cb, lb);
  // consumer index i in chunk A; issue index ia relative to A's start (may
  // run into chunk B); seq = units consumed by this warp (ring position)
  int i = 0, ia = 0;
  unsigned seq = 0;
  auto issue_ahead = [&]() {
    while (ia - i < STAGES && ia < la + lb) {
      const UnitMeta m = ia < la ? sh(ma, ia) : sh(mb, ia - la);
      if (lane == 0) {
        if (ia - i > 0 || seq > 0) fence_proxy_async();
        issue((int)((seq + (unsigned)(ia - i)) % STAGES), m);
      }
      ++ia;
    }
  };
  issue_ahead();

  // row j of an item: a private item's row follows from its index, a grouped
  // item lists its rows
  auto item_row = [&](int item, int j) -> int {
    return item >= p.n_gitems ? item - p.n_gitems : p.item_rows[p.item_roff[item] + j];
  };
  // q^T as the B operand of S^T = K . q^T: column n of the 128 x 8 tile is the
  // item's row n (lanes 4n .. 4n + 3 hold it; a private item has column 0
  // only); the next piece's q is prefetched one page ahead into qn
  uint32_t qa[8][2], qn[8][2];
  auto fetch_q = [&](uint32_t (&dst)[8][2], int item, int nr, int head) {
    const int row = g < nr ? item_row(item, g) : -1;
    const uint32_t* Q = reinterpret_cast<const uint32_t*>(q + ((long long)max(row, 0) * H + head) * kHeadDim);
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
      dst[kt][0] = row >= 0 ? Q[kt * 8 + t4] : 0u;
      dst[kt][1] = row >= 0 ? Q[kt * 8 + 4 + t4] : 0u;
    }
  };
  UnitMeta cur = sh(ma, 0);
  fetch_q(qa, cur.item, cur.nr, cur.head);
  // o^T tiles: dims 16 mt + g (c0, c1) and 16 mt + g + 8 (c2, c3) x columns
  // 2 t4, 2 t4 + 1.  Private item: lanes t4 == 0, column 0 = P hi, column 1 =
  // P lo.  Grouped item: the columns are its rows (P hi and lo in two MMAs).
  float o[8][4];
#pragma unroll
  for (int k = 0; k < 8; ++k) o[k][0] = o[k][1] = o[k][2] = o[k][3] = 0.f;
  float m = -INFINITY, l = 0.f;    // private: the row; grouped: column 2 t4
  float m2 = -INFINITY, l2 = 0.f;  // grouped: column 2 t4 + 1
  const int mi = lane >> 3, ri = lane & 7;

  while (true) {
    // the unit after this one (next in A, else first of B) decides the piece end
    const bool chunk_last = i + 1 == la;
    const bool have_next = !chunk_last || lb > 0;
    const UnitMeta nxt = !chunk_last ? sh(ma, i + 1) : (lb > 0 ? sh(mb, 0) : cur);
    const bool piece_end = chunk_last || nxt.item != cur.item || nxt.head != cur.head;
    if (piece_end && have_next) fetch_q(qn, nxt.item, nxt.nr, nxt.head);
    const int s = (int)(seq % STAGES);
    mbar_wait(&full[warp][s], (seq / STAGES) & 1);
    const uint32_t Ks = smem_u32(ring + s * kPwStageBytes);
    const uint32_t Vs = Ks + 4096;
    // transposed products, M = the page's 16 tokens / 16 head dims:
    // S^T = K . q^T (8 MMAs; the K tile is the A operand as stored) and
    // o^T += V^T . [p_hi p_lo]^T (8 MMAs; V^T by ldmatrix.trans).  Lanes
    // t4 == 0 hold the real columns: token / dim g and g + 8.
    float st[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
      uint32_t r0, r1, r2, r3;
      ldsm_x4(Ks + sw_page((mi >> 1) * 8 + ri, 2 * kt + (mi & 1)), r0, r1, r2, r3);
      const uint32_t af[4] = {r0, r2, r1, r3};
      mma_bf16(st, af, qa[kt][0], qa[kt][1]);
    }
    if (!GROUPED || cur.nr == 1) {
      const bool real = t4 == 0;
      const float v0 = real && g < cur.ntok ? st[0] * scale_log2 : -INFINITY;
      const float v1 = real && g + 8 < cur.ntok ? st[2] * scale_log2 : -INFINITY;
      float mx = fmaxf(v0, v1);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      mx = __shfl_sync(0xffffffffu, mx, 0);
      const float m_new = fmaxf(m, mx);
      const float alpha = ex2(m - m_new);
      m = m_new;
      const float p0 = real ? ex2(v0 - m_new) : 0.f, p1 = real ? ex2(v1 - m_new) : 0.f;
      l = l * alpha + (p0 + p1);
      // p^T as the B operand: lane (g, t4) takes tokens 2 t4, 2 t4 + 1 (b0) and
      // 2 t4 + 8, 2 t4 + 9 (b1); token t sits in lane 4 (t & 7)
      const float x0 = __shfl_sync(0xffffffffu, p0, 8 * t4), x1 = __shfl_sync(0xffffffffu, p0, 8 * t4 + 4);
      const float y0 = __shfl_sync(0xffffffffu, p1, 8 * t4), y1 = __shfl_sync(0xffffffffu, p1, 8 * t4 + 4);
      const uint32_t ph0 = pack_bf16(x0, x1), ph1 = pack_bf16(y0, y1);
      const uint32_t pl0 = pack_bf16(x0 - bf_lo(ph0), x1 - bf_hi(ph0));
      const uint32_t pl1 = pack_bf16(y0 - bf_lo(ph1), y1 - bf_hi(ph1));
      // P hi in column 0 and P lo in column 1 of one B operand (lanes g = 0 and
      // g = 1): one MMA per 16-dim slice; o = column 0 + column 1 at the end
      const uint32_t pb0 = g == 1 ? pl0 : ph0, pb1 = g == 1 ? pl1 : ph1;
  #pragma unroll
      for (int k = 0; k < 8; ++k) {
        o[k][0] *= alpha;
        o[k][1] *= alpha;
        o[k][2] *= alpha;
        o[k][3] *= alpha;
      }
  #pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t r0, r1, r2, r3;
        ldsm_x4_t(Vs + sw_page((mi >> 1) * 8 + ri, 2 * mt + (mi & 1)), r0, r1, r2, r3);
        const uint32_t af[4] = {r0, r1, r2, r3};
        mma_bf16(o[mt], af, pb0, pb1);
      }
    } else {
      // grouped item: columns a = 2 t4 and b = 2 t4 + 1 of S^T are rows of the
      // item (the columns past its rows hold q = 0 and are never written)
      const float sa0 = g < cur.ntok ? st[0] * scale_log2 : -INFINITY;
      const float sb0 = g < cur.ntok ? st[1] * scale_log2 : -INFINITY;
      const float sa1 = g + 8 < cur.ntok ? st[2] * scale_log2 : -INFINITY;
      const float sb1 = g + 8 < cur.ntok ? st[3] * scale_log2 : -INFINITY;
      float mxa = fmaxf(sa0, sa1), mxb = fmaxf(sb0, sb1);
#pragma unroll
      for (int x = 4; x < 32; x <<= 1) {
        mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, x));
        mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, x));
      }
      const float mna = fmaxf(m, mxa), mnb = fmaxf(m2, mxb);
      const float ala = ex2(m - mna), alb = ex2(m2 - mnb);
      m = mna;
      m2 = mnb;
      const float pa0 = ex2(sa0 - mna), pb0 = ex2(sb0 - mnb), pa1 = ex2(sa1 - mna), pb1 = ex2(sb1 - mnb);
      l = l * ala + (pa0 + pa1);
      l2 = l2 * alb + (pb0 + pb1);
      // P^T as the B operand: lane (g, t4) needs P(token 2 t4 [+1] [+8], row g);
      // P(token j, row c) sits in lane 4 (j & 7) + (c >> 1), half c & 1 of
      // the (a, b) pair of its token row j (< 8: X, >= 8: Y)
      const uint32_t X = pack_bf16(pa0, pb0), Y = pack_bf16(pa1, pb1);
      const uint32_t Xl = pack_bf16(pa0 - bf_lo(X), pb0 - bf_hi(X));
      const uint32_t Yl = pack_bf16(pa1 - bf_lo(Y), pb1 - bf_hi(Y));
      const int srcA = 8 * t4 + (g >> 1), srcB = srcA + 4;
      const int hs = (g & 1) * 16;
      auto pair = [&](uint32_t v) {
        const uint32_t lo = (__shfl_sync(0xffffffffu, v, srcA) >> hs) & 0xFFFFu;
        const uint32_t hi = (__shfl_sync(0xffffffffu, v, srcB) >> hs) & 0xFFFFu;
        return lo | (hi << 16);
      };
      const uint32_t bh0 = pair(X), bh1 = pair(Y), bl0 = pair(Xl), bl1 = pair(Yl);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        o[k][0] *= ala;
        o[k][1] *= alb;
        o[k][2] *= ala;
        o[k][3] *= alb;
      }
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t r0, r1, r2, r3;
        ldsm_x4_t(Vs + sw_page((mi >> 1) * 8 + ri, 2 * mt + (mi & 1)), r0, r1, r2, r3);
        const uint32_t af[4] = {r0, r1, r2, r3};
        mma_bf16(o[mt], af, bh0, bh1);
        mma_bf16(o[mt], af, bl0, bl1);
      }
    }
    __syncwarp();  // every lane is done reading stage s
    ++i;
    ++seq;
    issue_ahead();
    if (piece_end) {
      // partial of each of the item's rows at this head from this chunk: slot
      // = the (item, head) run's first slot for the row + its piece index
      const int item = cur.item, head = cur.head;
      const int piece = ca - p.item_chunk0[item * H + head];
      auto slot_of = [&](int j) {
        const int roff = item >= p.n_gitems ? p.n_grows + item - p.n_gitems : p.item_roff[item];
        return p.item_slot[(roff + j) * H + head] + piece;
      };
      float lsum = l;
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 4);
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 8);
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 16);
      if (!GROUPED || cur.nr == 1) {
        if (t4 == 0) {
          const int row = item_row(item, 0);
          const long long pi = part_index(p, H, row, slot_of(0), head);
          float* po = a.part_o + pi * kHeadDim;
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            po[mt * 16 + g] = o[mt][0] + o[mt][1];
            po[mt * 16 + g + 8] = o[mt][2] + o[mt][3];
          }
          if (g == 0) a.part_ml[pi] = make_float2(m, lsum);
        }
      } else {
        float lsum2 = l2;
        lsum2 += __shfl_xor_sync(0xffffffffu, lsum2, 4);
        lsum2 += __shfl_xor_sync(0xffffffffu, lsum2, 8);
        lsum2 += __shfl_xor_sync(0xffffffffu, lsum2, 16);
#pragma unroll
        for (int cb2 = 0; cb2 < 2; ++cb2) {
          const int col = 2 * t4 + cb2;
          if (col < cur.nr) {
            const long long pi = part_index(p, H, item_row(item, col), slot_of(col), head);
            float* po = a.part_o + pi * kHeadDim;
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
              po[mt * 16 + g] = o[mt][cb2];
              po[mt * 16 + g + 8] = o[mt][2 + cb2];
            }
            if (g == 0) a.part_ml[pi] = cb2 ? make_float2(m2, lsum2) : make_float2(m, lsum);
          }
        }
      }
      m = -INFINITY;
      l = 0.f;
      m2 = -INFINITY;
      l2 = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k][0] = o[k][1] = o[k][2] = o[k][3] = 0.f;
#pragma unroll
      for (int kt = 0; kt < 8; ++kt) {
        qa[kt][0] = qn[kt][0];
        qa[kt][1] = qn[kt][1];
      }
    }
    if (chunk_last) {
      if (lb == 0) break;  // the ticket counter ran dry
      // B becomes A; grab the chunk after it
      ia -= la;
      i = 0;
      ca = cb;
      ma = mb;
      la = lb;
      cb = grab();
      mb = load_chunk(cb, lb);
      issue_ahead();
    }
    cur = nxt;
  }
#ifdef FK_TIMELINE
  if (lane == 0) CTA_TL_NOTE(fk_tl_cta_priv, layer, 2, global_ns());
#endif
  CTA_TL_END(fk_tl_cta_priv, layer);
}

extern "C" int fk_debug_cta_timeline_priv(unsigned long long* out, int n) {
#ifdef FK_TIMELINE
  if (cudaDeviceSynchronize() != cudaSuccess) return 6;
  return cudaMemcpyFromSymbol(out, fk_tl_cta_priv, sizeof(unsigned long long) * 8 * (n < 1024 ? n : 1024)) == cudaSuccess ? 0 : 6;
#else
  (void)out;
  (void)n;
  return 5;
#endif
}

// ======================================================= prefix (mma.sync)
constexpr int kPmThreads = 128;
constexpr int kPmStages = 3;
constexpr int kPmTileTok = kMmaTilePages * kPage;    // 64
constexpr int kPmHalfBytes = kPmTileTok * 128;       // 64 rows x 128 B (64 head-dim elems)
constexpr int kPmKBytes = 2 * kPmHalfBytes;          // 16 KiB
constexpr int kPmStageBytes = 2 * kPmKBytes;         // K + V
constexpr int kPmSmem = kPmStages * kPmStageBytes + 1024;

// smem byte offset of (row, 16-byte chunk c in [0,16)) in a SWIZZLE_128B
// [2 halves][rows][128 B] tile as written by the TMA box {64, 16}.
__device__ __forceinline__ uint32_t sw128(int row, int c16) {
  return (uint32_t)((c16 >> 3) * kPmHalfBytes + row * 128 + (((c16 & 7) ^ (row & 7)) << 4));
}

__global__ void __launch_bounds__(kPmThreads) fk_prefix_mma_kernel(
    ArenaDev a, int ps, int layer, const __nv_bfloat16* __restrict__ q, float scale_log2,
    const __grid_constant__ CUtensorMap tmap) {
  const PlanDev& p = fk_plan_c[ps];
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kPmStages];
  __shared__ int s_rows[kMmaQBlock];

  pdl_launch_dependents();
  const int item = blockIdx.x, tid = threadIdx.x;
  const int head = p.it_head[item];
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int H = a.num_heads;
  const int npages = p.it_npages[item], ntok = p.it_ntok[item], poff = p.it_page_off[item];
  const int nq = p.it_nq[item], qoff = p.it_q_off[item];
  const int* qslot = p.qslot + p.it_qslot_off[item];
  const int ntiles = (npages + kMmaTilePages - 1) / kMmaTilePages;
  const int planeK = (int)plane_index(layer, 0, head, H), planeV = (int)plane_index(layer, 1, head, H);

  if (tid < kMmaQBlock) s_rows[tid] = tid < nq ? p.qrows[qoff + tid] : -1;
  if (tid == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < kPmStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  // zero the ring once so rows of partial tiles never hold NaN bit patterns
  for (int i = tid; i < kPmStages * kPmStageBytes / 16; i += kPmThreads)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  __syncthreads();

  auto issue = [&](int tile, int s) {
    const int pg0 = tile * kMmaTilePages;
    const int np = min(kMmaTilePages, npages - pg0);
    uint8_t* st = smem + s * kPmStageBytes;
    mbar_expect_tx(&full[s], np * 4 * 2048);
    for (int j = 0; j < np; ++j) {
      const int pg = p.pages[poff + pg0 + j];
      for (int hf = 0; hf < 2; ++hf) {
        tma_load_3d(st + hf * kPmHalfBytes + j * 2048, &tmap, hf * 64, pg * kPage, planeK, &full[s]);
        tma_load_3d(st + kPmKBytes + hf * kPmHalfBytes + j * 2048, &tmap, hf * 64, pg * kPage, planeV,
                    &full[s]);
      }
    }
  };
  if (tid == 0)
    for (int j = 0; j < kPmStages && j < ntiles; ++j) issue(j, j);

  // Q fragments (A operand, row-major 16 x 128 per warp)
  const int r0 = warp * 16 + g, r1 = r0 + 8;
  const bool active = warp * 16 < nq;
  uint32_t qa[8][4];
  {
    const int q0 = s_rows[r0 < kMmaQBlock ? r0 : 0], q1 = s_rows[r1 < kMmaQBlock ? r1 : 0];
    const uint32_t* Q0 = reinterpret_cast<const uint32_t*>(q + ((long long)max(q0, 0) * H + head) * kHeadDim);
    const uint32_t* Q1 = reinterpret_cast<const uint32_t*>(q + ((long long)max(q1, 0) * H + head) * kHeadDim);
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
      qa[kt][0] = (r0 < nq) ? Q0[kt * 8 + t4] : 0u;
      qa[kt][1] = (r1 < nq) ? Q1[kt * 8 + t4] : 0u;
      qa[kt][2] = (r0 < nq) ? Q0[kt * 8 + 4 + t4] : 0u;
      qa[kt][3] = (r1 < nq) ? Q1[kt * 8 + 4 + t4] : 0u;
    }
  }
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int mi = lane >> 3, ri = lane & 7;

  for (int j = 0; j < ntiles; ++j) {
    const int s = j % kPmStages;
    mbar_wait(&full[s], (j / kPmStages) & 1);
    if (active) {
      const uint32_t Kb = smem_u32(smem + s * kPmStageBytes);
      const uint32_t Vb = Kb + kPmKBytes;
      float sc[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
      for (int kt = 0; kt < 8; ++kt) {
#pragma unroll
        for (int np2 = 0; np2 < 4; ++np2) {
          const int tok = np2 * 16 + (mi >> 1) * 8 + ri;
          uint32_t b0, b1, b2, b3;
          ldsm_x4(Kb + sw128(tok, 2 * kt + (mi & 1)), b0, b1, b2, b3);
          mma_bf16(sc[2 * np2], qa[kt], b0, b1);
          mma_bf16(sc[2 * np2 + 1], qa[kt], b2, b3);
        }
      }
      const int valid = ntok - j * kPmTileTok;
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int tok = nt * 8 + 2 * t4 + (e & 1);
          sc[nt][e] = tok < valid ? sc[nt][e] * scale_log2 : -INFINITY;
        }
        mx0 = fmaxf(mx0, fmaxf(sc[nt][0], sc[nt][1]));
        mx1 = fmaxf(mx1, fmaxf(sc[nt][2], sc[nt][3]));
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float al0 = ex2(m0 - mn0), al1 = ex2(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      // P = hi + lo, both bf16: the P.V product keeps ~16 mantissa bits
      // (a single bf16 P costs ~1.3e-3 mean-rel, above the 1e-3 bound)
      uint32_t pa[4][4], pl[4][4];
      float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float p0 = ex2(sc[nt][0] - mn0), p1 = ex2(sc[nt][1] - mn0);
        const float p2 = ex2(sc[nt][2] - mn1), p3 = ex2(sc[nt][3] - mn1);
        ps0 += p0 + p1;
        ps1 += p2 + p3;
        const uint32_t h01 = pack_bf16(p0, p1), h23 = pack_bf16(p2, p3);
        pa[nt >> 1][(nt & 1) * 2 + 0] = h01;
        pa[nt >> 1][(nt & 1) * 2 + 1] = h23;
        pl[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0 - bf_lo(h01), p1 - bf_hi(h01));
        pl[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2 - bf_lo(h23), p3 - bf_hi(h23));
      }
      l0 = l0 * al0 + ps0;
      l1 = l1 * al1 + ps1;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        o[i][0] *= al0;
        o[i][1] *= al0;
        o[i][2] *= al1;
        o[i][3] *= al1;
      }
#pragma unroll
      for (int kt2 = 0; kt2 < 4; ++kt2) {
#pragma unroll
        for (int dp = 0; dp < 8; ++dp) {
          const int tok = kt2 * 16 + (mi & 1) * 8 + ri;
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(Vb + sw128(tok, 2 * dp + (mi >> 1)), b0, b1, b2, b3);
          mma_bf16(o[2 * dp], pa[kt2], b0, b1);
          mma_bf16(o[2 * dp + 1], pa[kt2], b2, b3);
          mma_bf16(o[2 * dp], pl[kt2], b0, b1);
          mma_bf16(o[2 * dp + 1], pl[kt2], b2, b3);
        }
      }
    }
    __syncthreads();
    if (tid == 0 && j + kPmStages < ntiles) {
      fence_proxy_async();
      issue(j + kPmStages, s);
    }
  }

  // partials: m (log2 domain), l, unnormalised o
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  if (active) {
    if (r0 < nq) {
      const long long pi = part_index(p, H, s_rows[r0], qslot[r0], head);
      float2* po = reinterpret_cast<float2*>(a.part_o + pi * kHeadDim);
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) po[nt * 4 + t4] = make_float2(o[nt][0], o[nt][1]);
      if (t4 == 0) a.part_ml[pi] = make_float2(m0, l0);
    }
    if (r1 < nq) {
      const long long pi = part_index(p, H, s_rows[r1], qslot[r1], head);
      float2* po = reinterpret_cast<float2*>(a.part_o + pi * kHeadDim);
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) po[nt * 4 + t4] = make_float2(o[nt][2], o[nt][3]);
      if (t4 == 0) a.part_ml[pi] = make_float2(m1, l1);
    }
  }
}

// ================================================================== merge
// K4: one warp per (row, head) combines every partial (shared-prefix splits
// + private pieces) in log2 space and writes the bf16 row (fp32 optional).
// The grid is fixed (a multiple of the SM count, warps loop over (row,
// head)), so its launch does not change with the batch.
CTA_TL_DECL(fk_tl_cta_merge);

__global__ void __launch_bounds__(256) fk_merge_kernel(ArenaDev a, int ps, __nv_bfloat16* __restrict__ out,
                                                      float* __restrict__ out_f32, int layer) {
  const PlanDev& p = fk_plan_c[ps];
  CTA_TL_START(fk_tl_cta_merge, layer);  // (timeline builds: [0] = after the wait)
  const int lane = threadIdx.x & 31;
  const int H = a.num_heads, nrh = p.num_rows * H, stride = gridDim.x * 8;
  int w = blockIdx.x * 8 + (threadIdx.x >> 5);
  // plan data, read before the wait: the partial counts of this warp's first
  // two (row, head) items (more rows than warps: x 128 / x 256 forks)
  const int ns = w < nrh ? partial_count(p, H, w / H, w % H) : 0;
  const int ns2 = w + stride < nrh ? partial_count(p, H, (w + stride) / H, (w + stride) % H) : 0;
  pdl_wait_primary();       // partials of the prefix and private grids are complete
  pdl_launch_dependents();  // the next layer's first kernel may start (other partial half)
  // Every CTA of this launch's prefix and private grids has finished, so
  // nobody takes a ticket from this half any more: reset it for the launch
  // after next (which cannot start before this grid completes -- its first
  // kernel waits, directly or through the kernels in between, for this one).
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.tick = 0u;
#ifdef FK_TIMELINE
  if (threadIdx.x == 0 && blockIdx.x < 1024) fk_tl_cta_merge[layer & 1][blockIdx.x][0] = global_ns();
#endif
  if (w < nrh) merge_row_head_warp(a, p, w / H, w % H, out, out_f32, lane, ns);  // (8 early slots: 12 / 16 measured slower)
  w += stride;
  if (w < nrh) merge_row_head_warp(a, p, w / H, w % H, out, out_f32, lane, ns2);
  for (w += stride; w < nrh; w += stride) merge_row_head_warp(a, p, w / H, w % H, out, out_f32, lane);
  CTA_TL_END(fk_tl_cta_merge, layer);
}

// K4 for plans with many partials per (row, head) -- small batches, where the
// private stream of one row is cut into ~U / W chunks (a single 6k-token
// request has ~100 pieces per head) -- one CTA per (row, head): warp w
// combines slots w, w + 8, ...: the first kWidePre of them (128 slots per
// item) with their (m, l) and o all loaded in one memory round trip, any
// further ones 32 (m, l) / 8 o at a time; then warp 0 combines the 8 warp
// results through shared memory.  A warp per item would walk ~100 slots one
// load round after another.
constexpr int kWideWarps = 8;
constexpr int kWidePre = 16;
__global__ void __launch_bounds__(kWideWarps * 32) fk_merge_wide_kernel(ArenaDev a, int ps,
                                                                       __nv_bfloat16* __restrict__ out,
                                                                       float* __restrict__ out_f32, int layer) {
  const PlanDev& p = fk_plan_c[ps];
  __shared__ float s_m[kWideWarps], s_l[kWideWarps];
  __shared__ float4 s_o[kWideWarps][32];
  CTA_TL_START(fk_tl_cta_merge, layer);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.num_heads, nrh = p.num_rows * H;
  pdl_wait_primary();       // partials of the prefix and private grids are complete
  pdl_launch_dependents();  // the next layer's first kernel may start (other partial half)
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.tick = 0u;  // (as fk_merge_kernel)
  for (int w = blockIdx.x; w < nrh; w += gridDim.x) {
    const int row = w / H, head = w % H;
    const int ns = partial_count(p, H, row, head);
    const long long base = part_index(p, H, row, 0, head);  // slot stride is H
    float M = -INFINITY, L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    {  // slots warp + kWideWarps * j, j < kWidePre: o and (m, l) loads issued together
      float4 v[kWidePre];
#pragma unroll
      for (int j = 0; j < kWidePre; ++j) {
        const int kk = warp + kWideWarps * j;
        v[j] = kk < ns ? __ldcg(reinterpret_cast<const float4*>(a.part_o + (base + (long long)kk * H) * kHeadDim) + lane)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      const int kl = warp + kWideWarps * lane;
      const bool mine = lane < kWidePre && kl < ns;
      const float2 ml = mine ? __ldcg(&a.part_ml[base + (long long)kl * H]) : make_float2(-INFINITY, 0.f);
      M = ml.x;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      const float wl = mine && M != -INFINITY ? ex2(ml.x - M) : 0.f;
      L = ml.y * wl;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
#pragma unroll
      for (int j = 0; j < kWidePre; ++j) {
        const float wk = __shfl_sync(0xffffffffu, wl, j);
        acc.x = fmaf(v[j].x, wk, acc.x);
        acc.y = fmaf(v[j].y, wk, acc.y);
        acc.z = fmaf(v[j].z, wk, acc.z);
        acc.w = fmaf(v[j].w, wk, acc.w);
      }
    }
    // any further slots, 32 per round (online across rounds)
    for (int j0 = kWidePre; warp + kWideWarps * j0 < ns; j0 += 32) {
      const int kl = warp + kWideWarps * (j0 + lane);
      const float2 ml = kl < ns ? __ldcg(&a.part_ml[base + (long long)kl * H]) : make_float2(-INFINITY, 0.f);
      float mr = ml.x;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, o));
      const float mn = fmaxf(M, mr);
      if (mn == -INFINITY) continue;
      const float sc = ex2(M - mn);  // (M == -inf: 0, nothing accumulated yet)
      acc.x *= sc;
      acc.y *= sc;
      acc.z *= sc;
      acc.w *= sc;
      L *= sc;
      M = mn;
      const float wl = kl < ns ? ex2(ml.x - M) : 0.f;
      float lsum = ml.y * wl;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
      L += lsum;
      const int cnt = min(32, (ns - warp + kWideWarps - 1) / kWideWarps - j0);
      for (int g0 = 0; g0 < cnt; g0 += 8) {
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int kk = warp + kWideWarps * (j0 + g0 + k);
          v[k] = g0 + k < cnt ? __ldcg(reinterpret_cast<const float4*>(a.part_o + (base + (long long)kk * H) * kHeadDim) + lane)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float wk = __shfl_sync(0xffffffffu, wl, (g0 + k) & 31);
          acc.x = fmaf(v[k].x, wk, acc.x);
          acc.y = fmaf(v[k].y, wk, acc.y);
          acc.z = fmaf(v[k].z, wk, acc.z);
          acc.w = fmaf(v[k].w, wk, acc.w);
        }
      }
    }
    if (lane == 0) {
      s_m[warp] = M;
      s_l[warp] = L;
    }
    s_o[warp][lane] = acc;
    __syncthreads();
    if (warp == 0) {
      float Mc = -INFINITY;
#pragma unroll
      for (int k = 0; k < kWideWarps; ++k) Mc = fmaxf(Mc, s_m[k]);
      float Lc = 0.f;
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      if (Mc != -INFINITY) {
#pragma unroll
        for (int k = 0; k < kWideWarps; ++k) {
          const float wk = s_m[k] == -INFINITY ? 0.f : ex2(s_m[k] - Mc);
          Lc = fmaf(s_l[k], wk, Lc);
          const float4 v = s_o[k][lane];
          r.x = fmaf(v.x, wk, r.x);
          r.y = fmaf(v.y, wk, r.y);
          r.z = fmaf(v.z, wk, r.z);
          r.w = fmaf(v.w, wk, r.w);
        }
      }
      const float inv = Lc > 0.f ? 1.f / Lc : 0.f;
      r = make_float4(r.x * inv, r.y * inv, r.z * inv, r.w * inv);
      const long long oi = ((long long)row * H + head) * kHeadDim + lane * 4;
      *reinterpret_cast<uint2*>(out + oi) = make_uint2(pack_bf16(r.x, r.y), pack_bf16(r.z, r.w));
      if (out_f32) *reinterpret_cast<float4*>(out_f32 + oi) = r;
    }
    __syncthreads();
  }
  CTA_TL_END(fk_tl_cta_merge, layer);
}

extern "C" int fk_debug_cta_timeline_merge(unsigned long long* out, int n) {
#ifdef FK_TIMELINE
  if (cudaDeviceSynchronize() != cudaSuccess) return 6;
  return cudaMemcpyFromSymbol(out, fk_tl_cta_merge, sizeof(unsigned long long) * 8 * (n < 1024 ? n : 1024)) == cudaSuccess ? 0 : 6;
#else
  (void)out;
  (void)n;
  return 5;
#endif
}

// ================================================================= append
// K1: the step's new K/V rows -> (page, slot) of each row's leaf, for
// layers [layer0, layer0 + nlayers).  One warp per (row, head) and group of
// kAppendLayers layers: lanes 0-15 move K, 16-31 V, 16 B each; all of a
// warp's loads are issued before its stores.
constexpr int kAppendLayers = 8;
__global__ void __launch_bounds__(256) fk_append_kernel(ArenaDev a, int ps, int layer0, int nlayers,
                                                       const uint4* __restrict__ k, const uint4* __restrict__ v) {
  const PlanDev& p = fk_plan_c[ps];
  const int H = a.num_heads;
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= p.num_rows * H) return;
  const int row = w / H, h = w % H;
  const int pg = p.app_page[row];
  if (pg < 0) return;
  const int slot = p.app_slot[row];
  const int l0 = blockIdx.y * kAppendLayers;
  const long long plane_elems = a.num_pages * kPage * kHeadDim;
  const int kv = lane >> 4, c = lane & 15;
  const uint4* src = kv == 0 ? k : v;
  uint4 val[kAppendLayers];
#pragma unroll
  for (int i = 0; i < kAppendLayers; ++i)
    if (l0 + i < nlayers) val[i] = __ldcs(&src[(((long long)(l0 + i) * p.num_rows + row) * H + h) * 16 + c]);
#pragma unroll
  for (int i = 0; i < kAppendLayers; ++i)
    if (l0 + i < nlayers) {
      uint4* dst = reinterpret_cast<uint4*>(a.kv + plane_index(layer0 + l0 + i, kv, h, H) * plane_elems +
                                            ((long long)pg * kPage + slot) * kHeadDim);
      dst[c] = val[i];
    }
}

// ================================================================== fill
// Caller K/V rows for tokens [pos0, pos0 + ntok) of one context -> pages,
// for layers [layer0, layer0 + gridDim.y).  One warp per (token, head):
// lanes 0-15 move the 256 B K row, lanes 16-31 the V row, 16 B each.
// src k/v: [nlayers][ntok][H][D] bf16.
__global__ void __launch_bounds__(256) fk_fill_kv_kernel(ArenaDev a, const int* __restrict__ pages, int first_page,
                                                        long long pos0, int ntok, int layer0,
                                                        const uint4* __restrict__ k, const uint4* __restrict__ v) {
  const int H = a.num_heads;
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= ntok * H) return;
  const int t = w / H, h = w % H;
  const int li = blockIdx.y, layer = layer0 + li;
  const long long pos = pos0 + t;
  const int pg = pages[pos / kPage - first_page];
  const int slot = (int)(pos % kPage);
  const long long plane_elems = a.num_pages * kPage * kHeadDim;
  const int kv = lane >> 4, c = lane & 15;
  const uint4* src = kv == 0 ? k : v;
  const uint4 val = src[(((long long)li * ntok + t) * H + h) * 16 + c];
  uint4* dst = reinterpret_cast<uint4*>(a.kv + plane_index(layer, kv, h, H) * plane_elems +
                                        ((long long)pg * kPage + slot) * kHeadDim);
  dst[c] = val;
}

// ============================================================ migration
// Context KV pages from another pool (another GPU over NVLink peer access, or
// the same GPU) into this pool: one CTA per (page pair, plane chunk), each
// thread moves 16 B of a 4 KiB (layer, kv, head, page) block.  src_kv is a
// peer-mapped pointer when the pools live on different devices.
__global__ void __launch_bounds__(256) fk_copy_pages_kernel(ArenaDev dst, const __nv_bfloat16* __restrict__ src_kv,
                                                           long long src_num_pages, const int* __restrict__ pages,
                                                           int npages) {
  const int j = blockIdx.x;  // page pair
  const int planes = dst.num_layers * 2 * dst.num_heads;
  const int sp = pages[j], dp = pages[npages + j];
  const long long dplane = dst.num_pages * kPage * kHeadDim, splane = src_num_pages * kPage * kHeadDim;
  for (int pl = blockIdx.y; pl < planes; pl += gridDim.y) {
    const uint4* s = reinterpret_cast<const uint4*>(src_kv + pl * splane + (long long)sp * kPage * kHeadDim);
    uint4* d = reinterpret_cast<uint4*>(dst.kv + pl * dplane + (long long)dp * kPage * kHeadDim);
    d[threadIdx.x] = __ldg(s + threadIdx.x);  // 256 x 16 B = one 4 KiB page block
  }
}

cudaError_t launch_copy_pages(const ArenaDev& dst, const void* src_kv, long long src_num_pages, const int* pages_dev,
                              int npages, cudaStream_t s) {
  const int planes = dst.num_layers * 2 * dst.num_heads;
  dim3 grid(npages, planes < 64 ? planes : 64);
  fk_copy_pages_kernel<<<grid, 256, 0, s>>>(dst, (const __nv_bfloat16*)src_kv, src_num_pages, pages_dev, npages);
  return cudaGetLastError();
}

// ============================================================== synthetic
__global__ void fk_synth_fill_kernel(ArenaDev a, const int* __restrict__ pages, int first_page, long long uid,
                                     long long pos0, unsigned long long seed, float k_scale) {
  const long long pos = pos0 + blockIdx.x;
  const int layer = blockIdx.y;
  const int H = a.num_heads;
  const int pg = pages[pos / kPage - first_page];
  const int slot = (int)(pos % kPage);
  const long long plane_elems = a.num_pages * kPage * kHeadDim;
  for (int i = threadIdx.x; i < 2 * H * 32; i += blockDim.x) {
    const int kv = i / (H * 32);
    const int h = (i / 32) % H, j = i % 32;
    const unsigned long long key = synth_key(seed, kv == 0 ? kTagK : kTagV, uid, pos, layer, h);
    const uint2 w = synth_chunk(key, j, kv == 0 ? k_scale : 1.f);
    uint2* dst = reinterpret_cast<uint2*>(a.kv + plane_index(layer, kv, h, H) * plane_elems +
                                          ((long long)pg * kPage + slot) * kHeadDim);
    dst[j] = w;
  }
}

__global__ void fk_synth_queries_kernel(ArenaDev a, int ps, unsigned long long seed, uint2* q_all, int B) {
  const PlanDev& p = fk_plan_c[ps];
  const int row = blockIdx.x, layer = blockIdx.y;
  const int H = a.num_heads;  // q_all: [layers][B (>= rows)][H][D]
  for (int i = threadIdx.x; i < H * 32; i += blockDim.x) {
    const int h = i / 32, j = i % 32;
    const unsigned long long key = synth_key(seed, kTagQ, p.row_uid[row], p.row_pos[row], layer, h);
    q_all[(((long long)layer * B + row) * H + h) * 32 + j] = synth_chunk(key, j, 1.f);
  }
}

__global__ void fk_synth_append_kernel(ArenaDev a, int ps, unsigned long long seed, float k_scale) {
  const PlanDev& p = fk_plan_c[ps];
  const int row = blockIdx.x, layer = blockIdx.y;
  const int pg = p.app_page[row];
  if (pg < 0) return;
  const int slot = p.app_slot[row];
  const int H = a.num_heads;
  const long long plane_elems = a.num_pages * kPage * kHeadDim;
  for (int i = threadIdx.x; i < 2 * H * 32; i += blockDim.x) {
    const int kv = i / (H * 32);
    const int h = (i / 32) % H, j = i % 32;
    const unsigned long long key =
        synth_key(seed, kv == 0 ? kTagK : kTagV, p.row_uid[row], p.app_pos[row], layer, h);
    const uint2 w = synth_chunk(key, j, kv == 0 ? k_scale : 1.f);
    uint2* dst = reinterpret_cast<uint2*>(a.kv + plane_index(layer, kv, h, H) * plane_elems +
                                          ((long long)pg * kPage + slot) * kHeadDim);
    dst[j] = w;
  }
}

// ============================================================== launchers
cudaError_t upload_plan_main(int ps, const PlanDev* host_pinned, cudaStream_t s) {
  return cudaMemcpyToSymbolAsync(fk_plan_c, host_pinned, sizeof(PlanDev), (size_t)ps * sizeof(PlanDev),
                                 cudaMemcpyHostToDevice, s);
}

template <int STAGES, int WARPS, bool GROUPED>
static cudaError_t launch_private_shape(const ArenaDev& a, int ps, int layer, const void* q, float scale_log2,
                                       const CUtensorMap* tmap, const CUtensorMap* tmap_h, int grid_ctas, bool pdl,
                                       cudaStream_t s) {
  static unsigned long long attr_devices = 0;
  constexpr int smem = priv_smem<STAGES, WARPS>();
  if (!attr_set_on_device(attr_devices)) {
    cudaError_t e = cudaFuncSetAttribute(fk_private_kernel<STAGES, WARPS, GROUPED>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  return launch_k(fk_private_kernel<STAGES, WARPS, GROUPED>, dim3(grid_ctas), dim3(WARPS * 32), smem, s, pdl, a, ps, layer,
                  (const __nv_bfloat16*)q, scale_log2, *tmap, *tmap_h);
}

cudaError_t launch_private(const ArenaDev& a, const PlanDev& p, int ps, int layer, const void* q, float scale_log2,
                           const CUtensorMap* tmap, const CUtensorMap* tmap_h, int grid, bool pdl, cudaStream_t s) {
  if (p.priv_units == 0) return cudaSuccess;
  // ring shapes: per-warp stages x warps per CTA (8 KiB stages): 10 x 2 = 160 KiB
  // (the default, measured best), 8 x 3 and 12 x 2 = 192 KiB
  switch (p.priv_wpc) {
    case 8: return launch_private_shape<3, 8, false>(a, ps, layer, q, scale_log2, tmap, tmap_h, grid, pdl, s);
    case 12: return launch_private_shape<2, 12, false>(a, ps, layer, q, scale_log2, tmap, tmap_h, grid, pdl, s);
    default:
      // (row groups: the default shape only -- the planner keeps them off for the others)
      if (p.n_gitems > 0) return launch_private_shape<2, 10, true>(a, ps, layer, q, scale_log2, tmap, tmap_h, grid, pdl, s);
      return launch_private_shape<2, 10, false>(a, ps, layer, q, scale_log2, tmap, tmap_h, grid, pdl, s);
  }
}

cudaError_t launch_merge(const ArenaDev& a, int ps, void* out, float* out_f32, int layer, int grid, bool pdl,
                         bool wide, cudaStream_t s) {
  if (wide)
    return launch_k(fk_merge_wide_kernel, dim3(grid), dim3(kWideWarps * 32), 0, s, pdl, a, ps, (__nv_bfloat16*)out,
                    out_f32, layer);
  return launch_k(fk_merge_kernel, dim3(grid), dim3(256), 0, s, pdl, a, ps, (__nv_bfloat16*)out, out_f32, layer);
}

cudaError_t launch_prefix_mma(const ArenaDev& a, const PlanDev& p, int ps, int layer, const void* q,
                              float scale_log2, const CUtensorMap* tmap, cudaStream_t s) {
  static unsigned long long attr_devices = 0;
  if (!attr_set_on_device(attr_devices)) {
    cudaError_t e = cudaFuncSetAttribute(fk_prefix_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPmSmem);
    if (e != cudaSuccess) return e;
  }
  return launch_k(fk_prefix_mma_kernel, dim3(p.tc_begin), dim3(kPmThreads), kPmSmem, s, false, a, ps, layer,
                  (const __nv_bfloat16*)q, scale_log2, *tmap);
}

cudaError_t launch_append(const ArenaDev& a, const PlanDev& p, int ps, int layer0, int nlayers, const void* k,
                          const void* v, cudaStream_t s) {
  dim3 grid((p.num_rows * a.num_heads + 7) / 8, (nlayers + kAppendLayers - 1) / kAppendLayers);
  fk_append_kernel<<<grid, 256, 0, s>>>(a, ps, layer0, nlayers, (const uint4*)k, (const uint4*)v);
  return cudaGetLastError();
}

cudaError_t launch_synth_fill(const ArenaDev& a, const int* pages_dev, int first_page, long long uid,
                              long long pos0, long long pos1, unsigned long long seed, float k_scale,
                              cudaStream_t s) {
  dim3 grid((unsigned)(pos1 - pos0), a.num_layers);
  fk_synth_fill_kernel<<<grid, 256, 0, s>>>(a, pages_dev, first_page, uid, pos0, seed, k_scale);
  return cudaGetLastError();
}

cudaError_t launch_fill_kv(const ArenaDev& a, const int* pages_dev, int first_page, long long pos0, int ntok,
                           int layer0, int nlayers, const void* k, const void* v, cudaStream_t s) {
  dim3 grid((unsigned)((ntok * a.num_heads + 7) / 8), nlayers);
  fk_fill_kv_kernel<<<grid, 256, 0, s>>>(a, pages_dev, first_page, pos0, ntok, layer0, (const uint4*)k,
                                          (const uint4*)v);
  return cudaGetLastError();
}

cudaError_t launch_synth_queries(const ArenaDev& a, const PlanDev& p, int ps, unsigned long long seed, void* q_all,
                                 int rows_cap, cudaStream_t s) {
  dim3 grid(p.num_rows, a.num_layers);
  fk_synth_queries_kernel<<<grid, 256, 0, s>>>(a, ps, seed, (uint2*)q_all, rows_cap);
  return cudaGetLastError();
}

cudaError_t launch_synth_append(const ArenaDev& a, const PlanDev& p, int ps, unsigned long long seed, float k_scale,
                                cudaStream_t s) {
  dim3 grid(p.num_rows, a.num_layers);
  fk_synth_append_kernel<<<grid, 256, 0, s>>>(a, ps, seed, k_scale);
  return cudaGetLastError();
}

}  // namespace fk
