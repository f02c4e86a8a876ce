// sm_100a decode-attention kernels for shared-prefix ("fork") batches.
//
//  K3+K4  fk_private_kernel   per (row, head): streams the row's private pages
//                             (fan-out 1 contexts, engine.py:484 per-request
//                             chain cost) with 1-D bulk copies into a 4-stage
//                             smem ring, CUDA-core online softmax, then arrives
//                             on the (row, head) counter and, if last, merges
//                             every partial ("amalgamating").
//  K2     fk_prefix_mma_kernel per (shared context split, 64-query block,
//                             head): TMA (SWIZZLE_128B) page tiles, Q.K^T and
//                             P.V on mma.sync m16n8k16 — the warp-level path
//                             for small fan-out (engine.py:473-483 dedup).
//  K1     fk_append_kernel     new K/V row -> (page, slot).
//         fk_synth_*           deterministic synthetic KV / Q (oracle restates).
#include "fk_common.cuh"

namespace fk {

// =========================================================== private (n_c=1)
// Warp-granular stream-K: the private work is the unit list (row, head, page)
// in row-major order; global warp w streams units [w*per, (w+1)*per) through
// its own 3-stage smem ring (1-D bulk copies, 8 KiB per page: K then V), so
// every warp moves the same number of bytes and no block barrier is needed.
// A (row, head) item cut by a range boundary yields one partial per piece.
constexpr int kPageBytes = kPage * kHeadDim * 2;  // 4 KiB per (page, head, K|V)
constexpr int kPwThreads = kPrivWarpsPerCta * 32;
constexpr int kPwStageBytes = 2 * kPageBytes;
constexpr int kPwSmem = kPrivWarpsPerCta * kPrivStages * kPwStageBytes;

struct UnitCursor {
  int row, head, page;
};

__device__ __forceinline__ UnitCursor locate_unit(const PlanDev& p, int H, int u) {
  int lo = 0, hi = p.num_rows - 1;  // largest row with row_unit_off <= u (has pages)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.row_unit_off[mid] <= u) lo = mid; else hi = mid - 1;
  }
  const int np = p.row_priv_npages[lo];
  const int rel = u - p.row_unit_off[lo];
  return UnitCursor{lo, rel / np, rel % np};
}

__device__ __forceinline__ void advance_unit(const PlanDev& p, int H, UnitCursor& c) {
  if (++c.page < p.row_priv_npages[c.row]) return;
  c.page = 0;
  if (++c.head < H) return;
  c.head = 0;
  do {
    ++c.row;
  } while (c.row < p.num_rows && p.row_priv_npages[c.row] == 0);
}

__global__ void __launch_bounds__(kPwThreads, 1) fk_private_kernel(ArenaDev a, PlanDev p, int layer,
                                                                   const __nv_bfloat16* __restrict__ q,
                                                                   __nv_bfloat16* __restrict__ out,
                                                                   float* __restrict__ out_f32,
                                                                   float scale_log2) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kPrivWarpsPerCta][kPrivStages];
  __shared__ int s_ntok[kPrivWarpsPerCta][kPrivStages];
  __shared__ __align__(16) float s_p[kPrivWarpsPerCta][kPage];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kPrivWarpsPerCta + warp;
  const int H = a.num_heads;

  // rows with no tokens at all (no private pages, no shared slot): output 0
  for (int r = gw; r < p.num_rows; r += gridDim.x * kPrivWarpsPerCta) {
    if (p.row_priv_npages[r] == 0 && p.row_nslots[r] == 0) {
      for (int h = 0; h < H; ++h) {
        const long long oi = ((long long)r * H + h) * kHeadDim + lane * 4;
        *reinterpret_cast<uint2*>(out + oi) = make_uint2(0u, 0u);
        if (out_f32) *reinterpret_cast<float4*>(out_f32 + oi) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  const int u0 = gw * p.priv_per;
  const int u1 = min(p.priv_units, u0 + p.priv_per);
  if (u0 >= u1) return;

  uint8_t* ring = smem + warp * kPrivStages * kPwStageBytes;
  const long long plane_elems = a.num_pages * kPage * kHeadDim;
  if (lane == 0) {
    for (int s = 0; s < kPrivStages; ++s) mbar_init(&full[warp][s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  UnitCursor pc = locate_unit(p, H, u0);
  int pu = u0;
  auto issue = [&](int s) {  // lane 0 only
    const int e = p.row_priv_off[pc.row] + pc.page;
    const int pg = p.pages[e];
    s_ntok[warp][s] = p.page_ntok[e];
    const __nv_bfloat16* kp = a.kv + plane_index(layer, 0, pc.head, H) * plane_elems + (long long)pg * kPage * kHeadDim;
    const __nv_bfloat16* vp = a.kv + plane_index(layer, 1, pc.head, H) * plane_elems + (long long)pg * kPage * kHeadDim;
    uint8_t* st = ring + s * kPwStageBytes;
    mbar_expect_tx(&full[warp][s], kPwStageBytes);
    bulk_g2s(st, kp, kPageBytes, &full[warp][s]);
    bulk_g2s(st + kPageBytes, vp, kPageBytes, &full[warp][s]);
  };
  if (lane == 0) {
    for (int s = 0; s < kPrivStages && pu < u1; ++s, ++pu) {
      issue(s);
      advance_unit(p, H, pc);
    }
  }

  // q . k mapping: token t = lane/2, head-dim half hh = lane%2, chunk order
  // rotated per lane so a quarter-warp's 16-byte smem reads hit 8 distinct
  // bank groups.
  const int t = lane >> 1, hh = lane & 1;
  const int rot = (t & 3) + 4 * hh;
  float qr[64];
  UnitCursor cc = locate_unit(p, H, u0);
  auto load_q = [&](int row, int head) {
    const uint4* qs = reinterpret_cast<const uint4*>(q + ((long long)row * H + head) * kHeadDim + hh * 64);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 w4 = qs[(i + rot) & 7];
      const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        qr[i * 8 + 2 * j] = bf_lo(w[j]) * scale_log2;
        qr[i * 8 + 2 * j + 1] = bf_hi(w[j]) * scale_log2;
      }
    }
  };
  load_q(cc.row, cc.head);
  float m = -INFINITY, l = 0.f;
  float4 o = make_float4(0.f, 0.f, 0.f, 0.f);

  for (int u = u0; u < u1; ++u) {
    const int s = (u - u0) % kPrivStages;
    mbar_wait(&full[warp][s], ((u - u0) / kPrivStages) & 1);
    const int ntok = s_ntok[warp][s];
    const uint8_t* Ks = ring + s * kPwStageBytes;
    const uint8_t* Vs = Ks + kPageBytes;
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 k4 = *reinterpret_cast<const uint4*>(Ks + t * 256 + hh * 128 + ((i + rot) & 7) * 16);
      const uint32_t w[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        dot = fmaf(qr[i * 8 + 2 * j], bf_lo(w[j]), dot);
        dot = fmaf(qr[i * 8 + 2 * j + 1], bf_hi(w[j]), dot);
      }
    }
    dot += __shfl_xor_sync(0xffffffffu, dot, 1);
    const float sc = t < ntok ? dot : -INFINITY;
    float mx = sc;
#pragma unroll
    for (int off = 2; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float m_new = fmaxf(m, mx);  // finite: every listed page holds >= 1 token
    const float alpha = ex2(m - m_new);
    const float pt = ex2(sc - m_new);
    float ps = pt;
#pragma unroll
    for (int off = 2; off < 32; off <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
    l = l * alpha + ps;
    m = m_new;
    if (hh == 0) s_p[warp][t] = pt;
    __syncwarp();
    o.x *= alpha;
    o.y *= alpha;
    o.z *= alpha;
    o.w *= alpha;
#pragma unroll
    for (int t4 = 0; t4 < 4; ++t4) {
      const float4 p4 = *reinterpret_cast<const float4*>(&s_p[warp][t4 * 4]);
      const float pv[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint2 v = *reinterpret_cast<const uint2*>(Vs + (t4 * 4 + e) * 256 + lane * 8);
        o.x = fmaf(pv[e], bf_lo(v.x), o.x);
        o.y = fmaf(pv[e], bf_hi(v.x), o.y);
        o.z = fmaf(pv[e], bf_lo(v.y), o.z);
        o.w = fmaf(pv[e], bf_hi(v.y), o.w);
      }
    }
    __syncwarp();  // stage s and s_p are free again
    if (lane == 0 && pu < u1) {  // producer state lives in lane 0 only
      fence_proxy_async();
      issue(s);
      advance_unit(p, H, pc);
      ++pu;
    }
    // piece boundary: last unit of this warp or of this (row, head) item
    const int row = cc.row, head = cc.head;
    advance_unit(p, H, cc);
    if (u + 1 == u1 || cc.page == 0) {
      const int np = p.row_priv_npages[row];
      const int first = (p.row_unit_off[row] + head * np) / p.priv_per;
      const int slot = p.row_nslots[row] + (gw - first);
      const long long pi = part_index(p, H, row, slot, head);
      reinterpret_cast<float4*>(a.part_o + pi * kHeadDim)[lane] = o;
      if (lane == 0) a.part_ml[pi] = make_float2(m, l);
      if (arrive_last_warp(a, p, row, head, lane)) {
        merge_row_head_warp(a, p, row, head, out, out_f32, lane);
        if (lane == 0) a.counters[row * H + head] = 0;
      }
      m = -INFINITY;
      l = 0.f;
      o = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u + 1 < u1) load_q(cc.row, cc.head);
    }
  }
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
    ArenaDev a, PlanDev p, int layer, const __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ out,
    float* __restrict__ out_f32, float scale_log2, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kPmStages];
  __shared__ int s_rows[kMmaQBlock];
  __shared__ int s_merge[kMmaQBlock];
  __shared__ int s_nmerge;

  const int item = blockIdx.x, head = blockIdx.y, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int H = a.num_heads;
  const int npages = p.it_npages[item], ntok = p.it_ntok[item], poff = p.it_page_off[item];
  const int nq = p.it_nq[item], qoff = p.it_q_off[item], slot = p.it_slot[item];
  const int ntiles = (npages + kMmaTilePages - 1) / kMmaTilePages;
  const int planeK = (int)plane_index(layer, 0, head, H), planeV = (int)plane_index(layer, 1, head, H);

  if (tid < kMmaQBlock) s_rows[tid] = tid < nq ? p.qrows[qoff + tid] : -1;
  if (tid == 0) {
    prefetch_tmap(&tmap);
    for (int s = 0; s < kPmStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    s_nmerge = 0;
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
      const long long pi = part_index(p, H, s_rows[r0], slot, head);
      float2* po = reinterpret_cast<float2*>(a.part_o + pi * kHeadDim);
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) po[nt * 4 + t4] = make_float2(o[nt][0], o[nt][1]);
      if (t4 == 0) a.part_ml[pi] = make_float2(m0, l0);
    }
    if (r1 < nq) {
      const long long pi = part_index(p, H, s_rows[r1], slot, head);
      float2* po = reinterpret_cast<float2*>(a.part_o + pi * kHeadDim);
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) po[nt * 4 + t4] = make_float2(o[nt][2], o[nt][3]);
      if (t4 == 0) a.part_ml[pi] = make_float2(m1, l1);
    }
  }
  __threadfence();
  __syncthreads();
  if (tid < nq) {
    const int row = s_rows[tid];
    const int prev = atomicAdd(&a.counters[row * H + head], 1);
    if (prev == expected_arrivals(p, row, head) - 1) s_merge[atomicAdd(&s_nmerge, 1)] = row;
  }
  __syncthreads();
  const int nm = s_nmerge;
  if (nm > 0) {
    __threadfence();
    for (int k = warp; k < nm; k += kPmThreads / 32) {
      const int row = s_merge[k];
      merge_row_head_warp(a, p, row, head, out, out_f32, lane);
      if (lane == 0) a.counters[row * H + head] = 0;
    }
  }
}

// ================================================================= append
__global__ void fk_append_kernel(ArenaDev a, PlanDev p, int layer, const uint4* __restrict__ k,
                                 const uint4* __restrict__ v) {
  const int row = blockIdx.x;
  const int pg = p.app_page[row];
  if (pg < 0) return;
  const int slot = p.app_slot[row];
  const int H = a.num_heads;
  const long long plane_elems = a.num_pages * kPage * kHeadDim;
  const int per_head = kHeadDim / 8;  // uint4 per head row
  for (int i = threadIdx.x; i < 2 * H * per_head; i += blockDim.x) {
    const int kv = i / (H * per_head);
    const int rem = i % (H * per_head);
    const int h = rem / per_head, c = rem % per_head;
    const uint4* src = kv == 0 ? k : v;
    uint4* dst = reinterpret_cast<uint4*>(a.kv + plane_index(layer, kv, h, H) * plane_elems +
                                          ((long long)pg * kPage + slot) * kHeadDim);
    dst[c] = src[((long long)row * H + h) * per_head + c];
  }
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

__global__ void fk_synth_queries_kernel(ArenaDev a, PlanDev p, unsigned long long seed, uint2* q_all) {
  const int row = blockIdx.x, layer = blockIdx.y;
  const int H = a.num_heads, B = p.num_rows;
  for (int i = threadIdx.x; i < H * 32; i += blockDim.x) {
    const int h = i / 32, j = i % 32;
    const unsigned long long key = synth_key(seed, kTagQ, p.row_uid[row], p.row_pos[row], layer, h);
    q_all[(((long long)layer * B + row) * H + h) * 32 + j] = synth_chunk(key, j, 1.f);
  }
}

__global__ void fk_synth_append_kernel(ArenaDev a, PlanDev p, unsigned long long seed, float k_scale) {
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
cudaError_t launch_private(const ArenaDev& a, const PlanDev& p, int layer, const void* q, void* out,
                           float* out_f32, float scale_log2, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fk_private_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPwSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = (p.priv_warps + kPrivWarpsPerCta - 1) / kPrivWarpsPerCta;
  fk_private_kernel<<<grid, kPwThreads, kPwSmem, s>>>(a, p, layer, (const __nv_bfloat16*)q, (__nv_bfloat16*)out,
                                                      out_f32, scale_log2);
  return cudaGetLastError();
}

cudaError_t launch_prefix_mma(const ArenaDev& a, const PlanDev& p, int layer, const void* q, void* out,
                              float* out_f32, float scale_log2, const CUtensorMap* tmap, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fk_prefix_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPmSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(p.tc_begin, a.num_heads);
  fk_prefix_mma_kernel<<<grid, kPmThreads, kPmSmem, s>>>(a, p, layer, (const __nv_bfloat16*)q,
                                                         (__nv_bfloat16*)out, out_f32, scale_log2, *tmap);
  return cudaGetLastError();
}

cudaError_t launch_append(const ArenaDev& a, const PlanDev& p, int layer, const void* k, const void* v,
                          cudaStream_t s) {
  fk_append_kernel<<<p.num_rows, 256, 0, s>>>(a, p, layer, (const uint4*)k, (const uint4*)v);
  return cudaGetLastError();
}

cudaError_t launch_synth_fill(const ArenaDev& a, const int* pages_dev, int first_page, long long uid,
                              long long pos0, long long pos1, unsigned long long seed, float k_scale,
                              cudaStream_t s) {
  dim3 grid((unsigned)(pos1 - pos0), a.num_layers);
  fk_synth_fill_kernel<<<grid, 256, 0, s>>>(a, pages_dev, first_page, uid, pos0, seed, k_scale);
  return cudaGetLastError();
}

cudaError_t launch_synth_queries(const ArenaDev& a, const PlanDev& p, unsigned long long seed, void* q_all,
                                 cudaStream_t s) {
  dim3 grid(p.num_rows, a.num_layers);
  fk_synth_queries_kernel<<<grid, 256, 0, s>>>(a, p, seed, (uint2*)q_all);
  return cudaGetLastError();
}

cudaError_t launch_synth_append(const ArenaDev& a, const PlanDev& p, unsigned long long seed, float k_scale,
                                cudaStream_t s) {
  dim3 grid(p.num_rows, a.num_layers);
  fk_synth_append_kernel<<<grid, 256, 0, s>>>(a, p, seed, k_scale);
  return cudaGetLastError();
}

}  // namespace fk
