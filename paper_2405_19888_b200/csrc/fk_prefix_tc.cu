// K2 on the 5th-generation tensor cores: shared-prefix decode attention for
// large fan-out (engine.py:473-483 dedup made real).
//
// One CTA per SM, stream-K over 128-token tile units of all tcgen05-class
// items (shared context x 128-query block x head), so every SM streams the
// same number of prefix bytes.  Warp roles:
//   warp 0     TMA producer: K and V page boxes (SWIZZLE_128B) into a
//              3-stage 64 KiB ring (mbarrier complete_tx)
//   warp 1     TMEM owner + single-thread MMA issuer:
//                S[128 q x 128 tok]  = Q . K^T      (SS, K-major A and B)
//                O[128 q x 128 dim]  = P . V        (TS: P from TMEM,
//                                                    V MN-major from smem)
//              P is split hi + lo in bf16 (two MMAs) for ~16-bit accuracy.
//   warps 2-5  softmax + epilogue, thread = query row = TMEM lane: S is
//              read with tcgen05.ld, P written back over S with tcgen05.st,
//              the PV tile is accumulated into registers with the running
//              rescale (O_reg = O_reg * alpha + O_tile).
// TMEM: S/P buffers at columns 0 and 128 (P written over the S columns
// already read: per 16-token k-step 8 columns P_hi + 8 columns P_lo), O
// tiles at 256 and 384.
#include "fk_tcgen05.cuh"

namespace fk {

constexpr int kTcThreads = 192;
constexpr int kTcStages = 3;
constexpr int kTcHalf = 128 * 128;                 // 128 rows x 128 B
constexpr int kTcTileBytes = 2 * kTcHalf;          // one K or V tile (32 KiB)
constexpr int kTcStageBytes = 2 * kTcTileBytes;    // K + V
constexpr int kTcQBytes = 2 * kTcHalf;
constexpr int kTcSmem = kTcQBytes + kTcStages * kTcStageBytes + 1024;

// unit cursor over the tcgen05 items of the plan
struct TcCursor {
  int item, tile;
};
__device__ __forceinline__ TcCursor tc_locate(const PlanDev& p, int u) {
  int lo = p.tc_begin, hi = p.num_items - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.it_unit_off[mid] <= u) lo = mid; else hi = mid - 1;
  }
  return TcCursor{lo, u - p.it_unit_off[lo]};
}
__device__ __forceinline__ void tc_advance(const PlanDev& p, TcCursor& c) {
  if (++c.tile == p.it_units[c.item]) {
    ++c.item;
    c.tile = 0;
  }
}

__global__ void __launch_bounds__(kTcThreads, 1) fk_prefix_tc_kernel(ArenaDev a, PlanDev p, int layer,
                                                                     const __nv_bfloat16* __restrict__ q,
                                                                     float scale_log2,
                                                                     const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + kTcQBytes;
  __shared__ uint64_t kv_full[kTcStages], kv_empty[kTcStages];
  __shared__ uint64_t s_full[2], p_full[2], o_full[2], o_free[2], q_full;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.num_heads;
  const int u0 = blockIdx.x * p.tc_per;
  const int u1 = min(p.tc_units, u0 + p.tc_per);
  if (u0 >= u1) return;
  const int T = u1 - u0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_free[b], 128);
    }
    mbar_init(&q_full, 128);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // zero the K/V ring once: rows of partial tiles then hold finite values
  for (int i = threadIdx.x; i < kTcStages * kTcStageBytes / 16; i += kTcThreads)
    reinterpret_cast<uint4*>(sKV)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&tmap);
      TcCursor c = tc_locate(p, u0);
      for (int t = 0; t < T; ++t) {
        const int s = t % kTcStages;
        if (t >= kTcStages) mbar_wait(&kv_empty[s], ((t / kTcStages) - 1) & 1);
        const int head = p.it_head[c.item];
        const int planeK = (int)plane_index(layer, 0, head, H), planeV = (int)plane_index(layer, 1, head, H);
        const int pg0 = c.tile * kTcTilePages;
        const int np = min(kTcTilePages, p.it_npages[c.item] - pg0);
        uint8_t* st = sKV + s * kTcStageBytes;
        mbar_expect_tx(&kv_full[s], np * 4 * 2048);
        for (int j = 0; j < np; ++j) {
          const int pg = p.pages[p.it_page_off[c.item] + pg0 + j];
          for (int hf = 0; hf < 2; ++hf) {
            tma_load_3d(st + hf * kTcHalf + j * 2048, &tmap, hf * 64, pg * kPage, planeK, &kv_full[s]);
            tma_load_3d(st + kTcTileBytes + hf * kTcHalf + j * 2048, &tmap, hf * 64, pg * kPage, planeV,
                        &kv_full[s]);
          }
        }
        tc_advance(p, c);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      TcCursor c = tc_locate(p, u0);
      int nitem = 0;
      const uint32_t qaddr = smem_u32(sQ);
      auto issue_pv = [&](int t) {
        const int sb = t & 1, s = t % kTcStages;
        mbar_wait(&p_full[sb], (t >> 1) & 1);
        if (t >= 2) mbar_wait(&o_free[sb], ((t >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t vaddr = smem_u32(sKV + s * kTcStageBytes + kTcTileBytes);
        const uint32_t o_tm = tm + 256 + sb * 128;
        const uint32_t p_tm = tm + sb * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bdesc = sdesc(vaddr + kk * 2048, kTcHalf, 1024);
          mma_ts(o_tm, p_tm + kk * 16, bdesc, kIdescPV, kk > 0);
          mma_ts(o_tm, p_tm + kk * 16 + 8, bdesc, kIdescPV, 1);
        }
        mma_commit(&o_full[sb]);
        mma_commit(&kv_empty[s]);
      };
      bool pv_pending = false;  // PV(t-1) not yet issued
      for (int t = 0; t < T; ++t) {
        if (t == 0 || c.tile == 0) {
          // item boundary: the softmax warps drain PV(t-1) before staging the
          // next Q, so flush it before waiting for that Q
          if (pv_pending) {
            issue_pv(t - 1);
            pv_pending = false;
          }
          mbar_wait(&q_full, nitem & 1);
          ++nitem;
        }
        const int s = t % kTcStages, sb = t & 1;
        mbar_wait(&kv_full[s], (t / kTcStages) & 1);
        tc_fence_after();
        const uint32_t kaddr = smem_u32(sKV + s * kTcStageBytes);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * kTcHalf + (kk & 3) * 32;
          mma_ss(tm + sb * 128, sdesc(qaddr + off, 16, 1024), sdesc(kaddr + off, 16, 1024), kIdescQK, kk > 0);
        }
        mma_commit(&s_full[sb]);
        if (pv_pending) issue_pv(t - 1);
        pv_pending = true;
        tc_advance(p, c);
      }
      issue_pv(T - 1);
    }
  } else {
    // ------------------------------------------------- softmax / epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_tm = tm + ((uint32_t)(quarter * 32) << 16);
    TcCursor c = tc_locate(p, u0);
    float O[128];
    float m = -INFINITY, l = 0.f, alpha_prev = 1.f;
    int nq = 0, head = 0, ntok = 0, seg_start = 0;
    bool active = false;
    auto acc_o = [&](int t, float al) {
      const int ob = t & 1;
      mbar_wait(&o_full[ob], (t >> 1) & 1);
      tc_fence_after();
      if (active) {
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t r[32];
          tmem_ld32(lane_tm + 256 + ob * 128 + cc * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) O[cc * 32 + e] = fmaf(O[cc * 32 + e], al, __uint_as_float(r[e]));
        }
      }
      tc_fence_before();
      mbar_arrive(&o_free[ob]);
    };
    for (int t = 0; t < T; ++t) {
      const int item = c.item;
      if (t == 0 || c.tile == 0) {
        // new item: stage Q (row-major, SWIZZLE_128B K-major) and reset state
        seg_start = t;  // this CTA's piece of the item starts here (maybe mid-item)
        nq = p.it_nq[item];
        head = p.it_head[item];
        ntok = p.it_ntok[item];
        active = quarter * 32 < nq;
        const bool real = row < nq;
        const uint4* src = real ? reinterpret_cast<const uint4*>(
                                      q + ((long long)p.qrows[p.it_q_off[item] + row] * H + head) * kHeadDim)
                                : nullptr;
#pragma unroll
        for (int cch = 0; cch < 16; ++cch) {
          const uint4 v = real ? src[cch] : make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(sQ + (cch >> 3) * kTcHalf + row * 128 + (((cch & 7) ^ (row & 7)) << 4)) = v;
        }
        fence_proxy_async();
        mbar_arrive(&q_full);
        m = -INFINITY;
        l = 0.f;
#pragma unroll
        for (int i = 0; i < 128; ++i) O[i] = 0.f;
      }
      const int sb = t & 1;
      mbar_wait(&s_full[sb], (t >> 1) & 1);
      tc_fence_after();
      float alpha = 1.f;
      if (active) {
        const int valid = ntok - c.tile * 128;
        const uint32_t s_tm = lane_tm + sb * 128;
        float mx = -INFINITY;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t r[32];
          tmem_ld32(s_tm + cc * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (cc * 32 + e < valid) mx = fmaxf(mx, __uint_as_float(r[e]));
        }
        const float m_new = fmaxf(m, mx * scale_log2);
        alpha = ex2(m - m_new);
        m = m_new;
        float sum = 0.f;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t r[32];
          tmem_ld32(s_tm + cc * 32, r);
          tmem_wait_ld();
          // P over the S columns just read: per 16-token k-step, 8 columns
          // of bf16x2 P_hi then 8 columns of P_lo
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int c0 = cc * 32 + 2 * e;
            const float p0 = c0 < valid ? ex2(fmaf(__uint_as_float(r[2 * e]), scale_log2, -m_new)) : 0.f;
            const float p1 = c0 + 1 < valid ? ex2(fmaf(__uint_as_float(r[2 * e + 1]), scale_log2, -m_new)) : 0.f;
            sum += p0 + p1;
            const uint32_t h = pack_bf16(p0, p1);
            pk[(e >> 3) * 16 + (e & 7)] = h;
            pk[(e >> 3) * 16 + 8 + (e & 7)] = pack_bf16(p0 - bf_lo(h), p1 - bf_hi(h));
          }
          tmem_st32(s_tm + cc * 32, pk);
        }
        tmem_wait_st();
        l = l * alpha + sum;
      }
      tc_fence_before();
      mbar_arrive(&p_full[sb]);
      if (t > seg_start) acc_o(t - 1, alpha_prev);
      alpha_prev = alpha;
      const bool last = c.tile + 1 == p.it_units[item];
      if (last || t == T - 1) {
        acc_o(t, alpha);
        if (row < nq) {
          const int piece = blockIdx.x - p.it_unit_off[item] / p.tc_per;
          const int r = p.qrows[p.it_q_off[item] + row];
          const int k = p.qslot[p.it_qslot_off[item] + row] + piece;
          const long long pi = part_index(p, H, r, k, head);
          float4* po = reinterpret_cast<float4*>(a.part_o + pi * kHeadDim);
#pragma unroll
          for (int i = 0; i < 32; ++i) po[i] = make_float4(O[4 * i], O[4 * i + 1], O[4 * i + 2], O[4 * i + 3]);
          a.part_ml[pi] = make_float2(m, l);
        }
      }
      tc_advance(p, c);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
  }
}

cudaError_t launch_prefix_tc(const ArenaDev& a, const PlanDev& p, int layer, const void* q, float scale_log2,
                             const CUtensorMap* tmap, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fk_prefix_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (p.tc_ctas == 0) return cudaSuccess;
  fk_prefix_tc_kernel<<<p.tc_ctas, kTcThreads, kTcSmem, s>>>(a, p, layer, (const __nv_bfloat16*)q, scale_log2,
                                                             *tmap);
  return cudaGetLastError();
}

}  // namespace fk
