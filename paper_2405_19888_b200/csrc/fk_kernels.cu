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
constexpr int kPrivThreads = 128;
constexpr int kPrivStages = 4;
constexpr int kPageBytes = kPage * kHeadDim * 2;  // 4 KiB per (page, head, K|V)

__global__ void __launch_bounds__(kPrivThreads) fk_private_kernel(ArenaDev a, PlanDev p, int layer,
                                                                  const __nv_bfloat16* __restrict__ q,
                                                                  __nv_bfloat16* __restrict__ out,
                                                                  float* __restrict__ out_f32,
                                                                  float scale_log2) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kPrivStages];
  __shared__ float s_scores[kPage];
  __shared__ float s_comb[64][3];
  __shared__ int s_last;

  const int row = blockIdx.x, head = blockIdx.y, tid = threadIdx.x;
  const int H = a.num_heads;
  const int npages = p.row_priv_npages[row];
  const int poff = p.row_priv_off[row];
  const long long plane_elems = a.num_pages * kPage * kHeadDim;
  const __nv_bfloat16* Kp = a.kv + plane_index(layer, 0, head, H) * plane_elems;
  const __nv_bfloat16* Vp = a.kv + plane_index(layer, 1, head, H) * plane_elems;

  if (tid == 0) {
    for (int s = 0; s < kPrivStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < kPrivStages && i < npages; ++i) {
      const int pg = p.pages[poff + i];
      uint8_t* st = smem + i * 2 * kPageBytes;
      mbar_expect_tx(&full[i], 2 * kPageBytes);
      bulk_g2s(st, Kp + (long long)pg * kPage * kHeadDim, kPageBytes, &full[i]);
      bulk_g2s(st + kPageBytes, Vp + (long long)pg * kPage * kHeadDim, kPageBytes, &full[i]);
    }
  }

  // q . k mapping: token = tid/8, 16-wide head-dim chunk = tid%8
  const int qk_tok = tid >> 3, qk_c = tid & 7;
  float qv[16];
  {
    const uint4* qs = reinterpret_cast<const uint4*>(q + ((long long)row * H + head) * kHeadDim + qk_c * 16);
    const uint4 a0 = qs[0], a1 = qs[1];
    const uint32_t w[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      qv[2 * i] = bf_lo(w[i]) * scale_log2;
      qv[2 * i + 1] = bf_hi(w[i]) * scale_log2;
    }
  }
  // p . v mapping: head-dim pair = tid%64, token half = tid/64
  const int pv_pair = tid & 63, pv_half = tid >> 6;
  float o0 = 0.f, o1 = 0.f, m = -INFINITY, l = 0.f;

  for (int i = 0; i < npages; ++i) {
    const int s = i % kPrivStages;
    mbar_wait(&full[s], (i / kPrivStages) & 1);
    const int ntok = p.page_ntok[poff + i];
    const uint8_t* Ks = smem + s * 2 * kPageBytes;
    const uint8_t* Vs = Ks + kPageBytes;
    {
      const uint4* kr = reinterpret_cast<const uint4*>(Ks + qk_tok * 256 + qk_c * 32);
      const uint4 k0 = kr[0], k1 = kr[1];
      const uint32_t w[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
      float dot = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        dot = fmaf(qv[2 * j], bf_lo(w[j]), dot);
        dot = fmaf(qv[2 * j + 1], bf_hi(w[j]), dot);
      }
      dot += __shfl_xor_sync(0xffffffffu, dot, 4);
      dot += __shfl_xor_sync(0xffffffffu, dot, 2);
      dot += __shfl_xor_sync(0xffffffffu, dot, 1);
      if (qk_c == 0) s_scores[qk_tok] = qk_tok < ntok ? dot : -INFINITY;
    }
    __syncthreads();
    float mx = -INFINITY;
#pragma unroll
    for (int t = 0; t < kPage; ++t) mx = fmaxf(mx, s_scores[t]);
    const float m_new = fmaxf(m, mx);  // finite: every listed page holds >= 1 token
    const float alpha = ex2(m - m_new);
    m = m_new;
    float ps = 0.f, a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int tok = pv_half * 8 + t;
      const float pt = ex2(s_scores[tok] - m_new);
      ps += pt;
      const uint32_t v = *reinterpret_cast<const uint32_t*>(Vs + tok * 256 + pv_pair * 4);
      a0 = fmaf(pt, bf_lo(v), a0);
      a1 = fmaf(pt, bf_hi(v), a1);
    }
    l = l * alpha + ps;
    o0 = o0 * alpha + a0;
    o1 = o1 * alpha + a1;
    __syncthreads();  // stage s and s_scores free
    if (tid == 0 && i + kPrivStages < npages) {
      const int pg = p.pages[poff + i + kPrivStages];
      uint8_t* st = smem + s * 2 * kPageBytes;
      fence_proxy_async();
      mbar_expect_tx(&full[s], 2 * kPageBytes);
      bulk_g2s(st, Kp + (long long)pg * kPage * kHeadDim, kPageBytes, &full[s]);
      bulk_g2s(st + kPageBytes, Vp + (long long)pg * kPage * kHeadDim, kPageBytes, &full[s]);
    }
  }
  // combine the two token halves (same running max on every thread)
  if (pv_half == 1) {
    s_comb[pv_pair][0] = o0;
    s_comb[pv_pair][1] = o1;
    s_comb[pv_pair][2] = l;
  }
  __syncthreads();
  const int slot = p.row_nslots[row];
  const long long pi = part_index(p, H, row, slot, head);
  if (pv_half == 0) {
    o0 += s_comb[pv_pair][0];
    o1 += s_comb[pv_pair][1];
    l += s_comb[pv_pair][2];
    reinterpret_cast<float2*>(a.part_o + pi * kHeadDim)[pv_pair] = make_float2(o0, o1);
    if (pv_pair == 0) a.part_ml[pi] = make_float2(m, l);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int prev = atomicAdd(&a.counters[row * H + head], 1);
    s_last = prev == p.row_nslots[row];  // expected arrivals = nslots + 1
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    merge_row_head(a, p, row, head, out, out_f32, tid);
    if (tid == 0) a.counters[row * H + head] = 0;
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
      uint32_t pa[4][4];
      float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const float p0 = ex2(sc[nt][0] - mn0), p1 = ex2(sc[nt][1] - mn0);
        const float p2 = ex2(sc[nt][2] - mn1), p3 = ex2(sc[nt][3] - mn1);
        ps0 += p0 + p1;
        ps1 += p2 + p3;
        pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
        pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
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
    if (prev == p.row_nslots[row]) s_merge[atomicAdd(&s_nmerge, 1)] = row;
  }
  __syncthreads();
  const int nm = s_nmerge;
  if (nm > 0) {
    __threadfence();
    for (int k = 0; k < nm; ++k) {
      const int row = s_merge[k];
      merge_row_head(a, p, row, head, out, out_f32, tid);
      if (tid == 0) a.counters[row * H + head] = 0;
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
  dim3 grid(p.num_rows, a.num_heads);
  fk_private_kernel<<<grid, kPrivThreads, kPrivStages * 2 * kPageBytes, s>>>(
      a, p, layer, (const __nv_bfloat16*)q, (__nv_bfloat16*)out, out_f32, scale_log2);
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
