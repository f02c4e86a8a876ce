// K2 on the 5th-generation tensor cores: shared-prefix decode attention for
// large fan-out (engine.py:473-483 dedup made real).
//
// One CTA per SM, stream-K over 128-token tile units of all tcgen05-class
// items (shared context x 128-query block x head), so every SM streams the
// same number of prefix bytes.  Warp roles:
//   warp 0     TMA producer: K and V page boxes (SWIZZLE_128B) into a
//              3-stage 64 KiB ring (mbarrier complete_tx); a partial last
//              tile is padded with copies of a valid page (masked later)
//   warp 1     TMEM owner + single-thread MMA issuer:
//                S[128 q x 128 tok]  = Q . K^T      (SS, K-major A and B)
//                O[128 q x 128 dim] += P . V        (TS: P from TMEM,
//                                                    V MN-major from smem)
//              P is split hi + lo in bf16 (two MMAs) for ~16-bit accuracy;
//              O accumulates in TMEM across the whole piece.
//   warps 2-9  softmax, two threads per query row (TMEM lane), 64 score
//              columns each: tile max (pair exchange through smem), P written
//              back over S with tcgen05.st, lazy rescale: the running max only
//              moves when a tile exceeds it by > 8 (log2), and only then is
//              the row of O in TMEM rescaled -- P <= 2^8 keeps fp32 safe.
// TMEM: S/P buffers at columns 0 and 128, O at 256.
#include "fk_tcgen05.cuh"

#include <cstdio>

namespace fk {

constexpr int kTcSoftmaxWarps = 8;
constexpr int kTcThreads = (2 + kTcSoftmaxWarps) * 32;
constexpr int kTcStages = 3;
constexpr int kTcHalf = 128 * 128;                 // 128 rows x 128 B
constexpr int kTcTileBytes = 2 * kTcHalf;          // one K or V tile (32 KiB)
constexpr int kTcStageBytes = 2 * kTcTileBytes;    // K + V
constexpr int kTcQBytes = 2 * kTcHalf;
struct TcMisc {
  uint64_t k_full[kTcStages], k_empty[kTcStages], v_full[kTcStages], v_empty[kTcStages];
  uint64_t s_full[2], p_full[2], o_done, q_full;
  uint32_t tmem_base;
  float s_max[2][2][128];  // [tile parity][half][row]
  float s_l[128];
};
constexpr int kTcSmem = kTcQBytes + kTcStages * kTcStageBytes + (int)sizeof(TcMisc);
constexpr float kRescaleThreshold = 8.0f;          // log2 units

#ifdef FK_TIMELINE
__device__ unsigned long long fk_tl[256];
#define TL(i) do { if (blockIdx.x == 0 && (i) < 256) fk_tl[(i)] = global_ns(); } while (0)
#else
#define TL(i) do { } while (0)
#endif

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
                                                                     const __grid_constant__ CUtensorMap tmap,
                                                                     const __grid_constant__ CUtensorMap tmap_run) {
  // all shared state is dynamic (no static smem), so the buffer starts at
  // the 1 KiB-aligned base SWIZZLE_128B needs
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + kTcQBytes;
  TcMisc& ms = *reinterpret_cast<TcMisc*>(smem + kTcQBytes + kTcStages * kTcStageBytes);
  uint64_t* k_full = ms.k_full;
  uint64_t* k_empty = ms.k_empty;
  uint64_t* v_full = ms.v_full;
  uint64_t* v_empty = ms.v_empty;
  uint64_t* s_full = ms.s_full;
  uint64_t* p_full = ms.p_full;
  uint64_t& o_done = ms.o_done;
  uint64_t& q_full = ms.q_full;
  uint32_t& tmem_base_sh = ms.tmem_base;
  auto& s_max = ms.s_max;
  auto& s_l = ms.s_l;
  if ((smem_u32(smem) & 1023u) != 0) __trap();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.num_heads;
  const int u0 = blockIdx.x * p.tc_per;
  const int u1 = min(p.tc_units, u0 + p.tc_per);
  pdl_launch_dependents();  // the private grid may start on SMs we release
  if (u0 >= u1) return;
  const int T = u1 - u0;
  TL(160);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], kTcSoftmaxWarps);
    }
    mbar_init(&o_done, 1);
    mbar_init(&q_full, kTcSoftmaxWarps);
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
  const int start_item = p.tc_start_item[blockIdx.x];
  const TcCursor c0{start_item, u0 - p.it_unit_off[start_item]};

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // The whole warp walks the tiles; page ids are prefetched lane-parallel
    // into a 2 x 32-entry register window (4 tiles ahead), so no dependent
    // global load sits between two tiles' TMA issues.  Lane 0 issues.
    if (lane == 0) {
      prefetch_tmap(&tmap);
      prefetch_tmap(&tmap_run);
    }
    TcCursor c = c0;
    int cur_item = -1, head = 0, npi = 0, poff = 0;
    int wbase = 0, win = 0, nwin = 0;
    for (int t = 0; t < T; ++t) {
      if (c.item != cur_item) {
        cur_item = c.item;
        head = p.it_head[cur_item];
        npi = p.it_npages[cur_item];
        poff = p.it_page_off[cur_item];
        wbase = c.tile * kTcTilePages;
        win = wbase + lane < npi ? p.pages[poff + wbase + lane] : 0;
        nwin = wbase + 32 + lane < npi ? p.pages[poff + wbase + 32 + lane] : 0;
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
        const int s = t % kTcStages;
        const int planeK = (int)plane_index(layer, 0, head, H), planeV = (int)plane_index(layer, 1, head, H);
        uint8_t* st = sKV + s * kTcStageBytes;
        // 8 physically consecutive pages -> one 128-row box per half (the
        // common case: a context's pages come from one allocation);
        // otherwise one 16-row box per page, a partial tile padded with a
        // valid (masked) page
        bool run = np == kTcTilePages;
#pragma unroll
        for (int j = 1; j < kTcTilePages; ++j) run = run && pl[j] == pl[0] + j;
        if (t >= kTcStages) mbar_wait(&k_empty[s], ((t / kTcStages) - 1) & 1);
        if (t < 16) TL(128 + t);
        mbar_expect_tx(&k_full[s], kTcTilePages * 2 * 2048);
        if (run) {
          tma_load_3d(st, &tmap_run, 0, pl[0] * kPage, planeK, &k_full[s]);
          tma_load_3d(st + kTcHalf, &tmap_run, 64, pl[0] * kPage, planeK, &k_full[s]);
        } else {
#pragma unroll
          for (int j = 0; j < kTcTilePages; ++j) {
            tma_load_3d(st + j * 2048, &tmap, 0, pl[j] * kPage, planeK, &k_full[s]);
            tma_load_3d(st + kTcHalf + j * 2048, &tmap, 64, pl[j] * kPage, planeK, &k_full[s]);
          }
        }
        if (t >= kTcStages) mbar_wait(&v_empty[s], ((t / kTcStages) - 1) & 1);
        mbar_expect_tx(&v_full[s], kTcTilePages * 2 * 2048);
        if (run) {
          tma_load_3d(st + kTcTileBytes, &tmap_run, 0, pl[0] * kPage, planeV, &v_full[s]);
          tma_load_3d(st + kTcTileBytes + kTcHalf, &tmap_run, 64, pl[0] * kPage, planeV, &v_full[s]);
        } else {
#pragma unroll
          for (int j = 0; j < kTcTilePages; ++j) {
            tma_load_3d(st + kTcTileBytes + j * 2048, &tmap, 0, pl[j] * kPage, planeV, &v_full[s]);
            tma_load_3d(st + kTcTileBytes + kTcHalf + j * 2048, &tmap, 64, pl[j] * kPage, planeV, &v_full[s]);
          }
        }
      }
      __syncwarp();
      tc_advance(p, c);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Two in-order streams polled by one thread: S(t) = Q.K^T as soon as K(t)
    // lands (and, at a piece start, its Q is staged), PV(t) as soon as P(t)
    // and V(t) are ready.  S(t) reuses the TMEM buffer of P(t-2), so it is
    // only issued after PV(t-2) (the tensor pipe executes in issue order).
    if (lane == 0) {
      TcCursor cs = c0, cp = c0;
      int nitem = 0, ts = 0, tp = 0, pv_seg = 0;
      const uint32_t qaddr = smem_u32(sQ);
      while (tp < T) {
        if (ts < T && ts <= tp + 1) {
          const bool starts = ts == 0 || cs.tile == 0;
          const int s = ts % kTcStages;
          if ((!starts || mbar_try_wait(&q_full, nitem & 1)) && mbar_try_wait(&k_full[s], (ts / kTcStages) & 1)) {
            if (starts) ++nitem;
            if (ts < 16) TL(ts);
            tc_fence_after();
            const uint32_t kaddr = smem_u32(sKV + s * kTcStageBytes);
            const int sb = ts & 1;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t off = (kk >> 2) * kTcHalf + (kk & 3) * 32;
              mma_ss(tm + sb * 128, sdesc(qaddr + off, 16, 1024), sdesc(kaddr + off, 16, 1024), kIdescQK, kk > 0);
            }
            mma_commit(&s_full[sb]);
            mma_commit(&k_empty[s]);
            if (ts < 16) TL(16 + ts);
            tc_advance(p, cs);
            ++ts;
            continue;
          }
        }
        {
          const int sb = tp & 1, s = tp % kTcStages;
          if (tp < ts && mbar_try_wait(&p_full[sb], (tp >> 1) & 1) && mbar_try_wait(&v_full[s], (tp / kTcStages) & 1)) {
            if (tp == 0 || cp.tile == 0) pv_seg = tp;
            if (tp < 16) TL(32 + tp);
            tc_fence_after();
            const uint32_t vaddr = smem_u32(sKV + s * kTcStageBytes + kTcTileBytes);
            const uint32_t p_tm = tm + sb * 128;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint64_t bdesc = sdesc(vaddr + kk * 2048, kTcHalf, 1024);
              mma_ts(tm + 256, p_tm + kk * 16, bdesc, kIdescPV, (tp > pv_seg || kk > 0) ? 1u : 0u);
              mma_ts(tm + 256, p_tm + kk * 16 + 8, bdesc, kIdescPV, 1u);
            }
            mma_commit(&o_done);
            mma_commit(&v_empty[s]);
            if (tp < 16) TL(48 + tp);
            tc_advance(p, cp);
            ++tp;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------- softmax / epilogue
    const int quarter = warp & 3;               // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;           // which 64 score columns / 64 O columns
    const int row = quarter * 32 + lane;
    // query j sits in TMEM lane 32*(j%4) + j/4: a partial block spreads its
    // rows over all four lane quarters, i.e. over all four SM sub-partitions
    const int qj = 4 * lane + quarter;
    const uint32_t lane_tm = tm + ((uint32_t)(quarter * 32) << 16);
    const int bar_id = 1 + quarter;             // named barrier of the two warps sharing these rows
    TcCursor c = c0;
    float m = -INFINITY, l = 0.f;
    int nq = 0, head = 0, ntok = 0, seg_start = 0;
    bool active = false;
    for (int t = 0; t < T; ++t) {
      const int item = c.item;
      if (t == 0 || c.tile == 0) {
        // new piece: stage this thread's half of its Q row (SW128 K-major)
        seg_start = t;
        nq = p.it_nq[item];
        head = p.it_head[item];
        ntok = p.it_ntok[item];
        active = quarter < nq;
        const bool real = qj < nq;
        const uint4* src = real ? reinterpret_cast<const uint4*>(
                                      q + ((long long)p.qrows[p.it_q_off[item] + qj] * H + head) * kHeadDim)
                                : nullptr;
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) {
          const int cch = half * 8 + k8;
          const uint4 v = real ? src[cch] : make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(sQ + half * kTcHalf + row * 128 + ((k8 ^ (row & 7)) << 4)) = v;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&q_full);
        m = -INFINITY;
        l = 0.f;
      }
      const int sb = t & 1;
      mbar_wait(&s_full[sb], (t >> 1) & 1);
      if (warp == 4 && lane == 0 && t < 16) TL(64 + t);
      tc_fence_after();
      if (active) {
        const int valid = ntok - c.tile * 128 - half * 64;  // valid columns among this thread's 64
        const uint32_t s_tm = lane_tm + sb * 128 + half * 64;
        uint32_t r0[32], r1[32];
        tmem_ld32(s_tm, r0);
        tmem_ld32(s_tm + 32, r1);
        tmem_wait_ld();
        if (warp == 4 && lane == 0 && t < 16) TL(176 + t);
        float mx;
        if (valid >= 64) {  // full tile: tree max, no masking
          float t8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            t8[k] = fmaxf(fmaxf(__uint_as_float(r0[4 * k]), __uint_as_float(r0[4 * k + 1])),
                          fmaxf(__uint_as_float(r0[4 * k + 2]), __uint_as_float(r0[4 * k + 3])));
            t8[k] = fmaxf(t8[k], fmaxf(fmaxf(__uint_as_float(r1[4 * k]), __uint_as_float(r1[4 * k + 1])),
                                       fmaxf(__uint_as_float(r1[4 * k + 2]), __uint_as_float(r1[4 * k + 3]))));
          }
          mx = fmaxf(fmaxf(fmaxf(t8[0], t8[1]), fmaxf(t8[2], t8[3])), fmaxf(fmaxf(t8[4], t8[5]), fmaxf(t8[6], t8[7])));
        } else {
          mx = -INFINITY;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (e < valid) mx = fmaxf(mx, __uint_as_float(r0[e]));
            if (e + 32 < valid) mx = fmaxf(mx, __uint_as_float(r1[e]));
          }
        }
        s_max[sb][half][row] = mx;
        asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
        if (warp == 4 && lane == 0 && t < 16) TL(192 + t);
        const float tile_max = fmaxf(mx, s_max[sb][half ^ 1][row]) * scale_log2;
        // lazy rescale: keep the running max unless the tile exceeds it by > 8
        if (tile_max > m + kRescaleThreshold) {
          const float m_new = tile_max;
          if (t > seg_start) {
            const float alpha = ex2(m - m_new);
            l *= alpha;
            mbar_wait(&o_done, (t - 1) & 1);  // PV(t-1) has landed in O
            tc_fence_after();
            const uint32_t o_tm = lane_tm + 256 + half * 64;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              uint32_t o[32];
              tmem_ld32(o_tm + cc * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st32(o_tm + cc * 32, o);
            }
          }
          m = m_new;
        }
        float sum4[4] = {0.f, 0.f, 0.f, 0.f};
        const bool full = valid >= 64;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const uint32_t* r = cc == 0 ? r0 : r1;
          // per 16-token k-step: 8 columns of bf16x2 P_hi then 8 of P_lo
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int c2 = cc * 32 + 2 * e;
            float p0 = ex2(fmaf(__uint_as_float(r[2 * e]), scale_log2, -m));
            float p1 = ex2(fmaf(__uint_as_float(r[2 * e + 1]), scale_log2, -m));
            if (!full) {
              p0 = c2 < valid ? p0 : 0.f;
              p1 = c2 + 1 < valid ? p1 : 0.f;
            }
            sum4[e & 3] += p0 + p1;
            const uint32_t hpk = pack_bf16(p0, p1);
            pk[(e >> 3) * 16 + (e & 7)] = hpk;
            pk[(e >> 3) * 16 + 8 + (e & 7)] = pack_bf16(p0 - bf_lo(hpk), p1 - bf_hi(hpk));
          }
          tmem_st32(s_tm + cc * 32, pk);
        }
        const float sum = (sum4[0] + sum4[1]) + (sum4[2] + sum4[3]);
        if (warp == 4 && lane == 0 && t < 16) TL(208 + t);
        tmem_wait_st();
        if (warp == 4 && lane == 0 && t < 16) TL(224 + t);
        l += sum;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[sb]);
      if (warp == 4 && lane == 0 && t < 16) TL(80 + t);
      const bool last = c.tile + 1 == p.it_units[item];
      if (last || t == T - 1) {
        // piece end: O (unnormalised, running max m) -> partial slot
        mbar_wait(&o_done, t & 1);
        if (warp == 4 && lane == 0 && t < 16) TL(96 + t);
        tc_fence_after();
        if (active) {
          const int piece = blockIdx.x - p.it_unit_off[item] / p.tc_per;
          const bool real = qj < nq;
          long long pi = 0;
          if (real) {
            const int r = p.qrows[p.it_q_off[item] + qj];
            const int k = p.qslot[p.it_qslot_off[item] + qj] + piece;
            pi = part_index(p, H, r, k, head);
          }
          const uint32_t o_tm = lane_tm + 256 + half * 64;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            uint32_t o[32];
            tmem_ld32(o_tm + cc * 32, o);
            tmem_wait_ld();
            if (real) {
              float4* po = reinterpret_cast<float4*>(a.part_o + pi * kHeadDim + half * 64 + cc * 32);
#pragma unroll
              for (int i4 = 0; i4 < 8; ++i4)
                po[i4] = make_float4(__uint_as_float(o[4 * i4]), __uint_as_float(o[4 * i4 + 1]),
                                     __uint_as_float(o[4 * i4 + 2]), __uint_as_float(o[4 * i4 + 3]));
            }
          }
          if (half == 1) s_l[row] = l;
          asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
          if (half == 0 && real) a.part_ml[pi] = make_float2(m, l + s_l[row]);
        }
        tc_fence_before();
        if (warp == 4 && lane == 0 && t < 16) TL(112 + t);
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

cudaError_t launch_prefix_tc(const ArenaDev& a, const PlanDev& p, int layer, const void* q, float scale_log2,
                             const CUtensorMap* tmap, const CUtensorMap* tmap_run, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
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
    attr = true;
  }
  if (p.tc_ctas == 0) return cudaSuccess;
  fk_prefix_tc_kernel<<<p.tc_ctas, kTcThreads, kTcSmem, s>>>(a, p, layer, (const __nv_bfloat16*)q, scale_log2,
                                                             *tmap, *tmap_run);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, fk_prefix_tc_kernel);
    int optin = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    fprintf(stderr, "fk_prefix_tc launch: %s (static smem %zu, dyn %d, max dyn attr %d, optin %d, regs %d, threads %d)\n",
            cudaGetErrorString(e), fa.sharedSizeBytes, kTcSmem, fa.maxDynamicSharedSizeBytes, optin, fa.numRegs,
            fa.maxThreadsPerBlock);
  }
  return e;
}

}  // namespace fk
