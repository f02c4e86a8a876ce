// Device helpers shared by the sm_100a kernels: mbarrier / bulk-copy / TMA
// PTX wrappers, warp MMA wrappers, the synthetic counter-hash generator and
// the log-sum-exp merge of per-(row, head) partials.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>
#include <vector>
#include "fk_internal.h"

namespace fk {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Watchdog: a pipeline bug must fail the launch, not hang the GPU.
constexpr uint64_t kWaitLimitNs = 10ull * 1000 * 1000 * 1000;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = global_ns();
  uint32_t n = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++n & 1023u) == 0 && global_ns() - t0 > kWaitLimitNs) __trap();
  }
}
// 1-D bulk copy global -> shared, completion on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 3-D TMA tile load (SASS: UTMALDG).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// same with an L2 cache policy (createpolicy: evict_first for streams read once)
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// Debug builds (-DFK_TIMELINE): per-CTA start/end stamps of the attention
// kernels, read back with fk_debug_cta_timeline (profiles/cta_timeline.py).
#ifdef FK_TIMELINE
#define CTA_TL_DECL(name) __device__ unsigned long long name[2][1024][4]
#define CTA_TL_START(name, layer) do { if (threadIdx.x == 0 && blockIdx.x < 1024) name[(layer) & 1][blockIdx.x][0] = global_ns(); } while (0)
#define CTA_TL_END(name, layer) do { if ((threadIdx.x & 31) == 0 && blockIdx.x < 1024) name[(layer) & 1][blockIdx.x][1] = global_ns(); } while (0)  // last writer ~ last warp
#define CTA_TL_NOTE(name, layer, k, v) do { if (blockIdx.x < 1024) name[(layer) & 1][blockIdx.x][k] = (v); } while (0)
#else
#define CTA_TL_DECL(name) static_assert(true, "")
#define CTA_TL_START(name, layer) do { } while (0)
#define CTA_TL_END(name, layer) do { } while (0)
#define CTA_TL_NOTE(name, layer, k, v) do { } while (0)
#endif

// Launch with optional programmatic dependent launch (PDL): the kernel may
// start while its stream predecessor is still running; it must call
// pdl_wait_primary() before touching the predecessor's results.
// cudaFuncSetAttribute is per device: remember which devices a kernel's
// dynamic shared-memory opt-in was set on (engines may share a process).
inline bool attr_set_on_device(unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask & bit) return true;
  mask |= bit;
  return false;
}

template <typename T>
inline void rec_push_arg(LaunchRec& r, const T& v) {
  const size_t al = alignof(T) < 16 ? alignof(T) : 16;
  size_t off = (r.bytes.size() + al - 1) / al * al;
  r.bytes.resize(off + sizeof(T));
  memcpy(r.bytes.data() + off, &v, sizeof(T));
  r.offs.push_back(off);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                            Args&&... args) {
  if (g_launch_rec) {
    LaunchRec& r = g_launch_rec->push();
    r.func = (const void*)kernel;
    r.grid = grid;
    r.block = block;
    r.smem = smem;
    r.pdl = pdl;
    (rec_push_arg<KArgs>(r, static_cast<KArgs>(args)), ...);
    return cudaSuccess;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// programmatic dependent launch (PDL) controls
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_primary() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// ------------------------------------------------- synthetic data generator
// Counter-hash generator restated by oracle/forkattn_oracle.py (synth_*):
//   key = MIX(seed ^ tag<<56); key = MIX(key ^ uid); key = MIX(key ^ pos);
//   key = MIX(key ^ layer); key = MIX(key ^ head); w_j = MIX(key ^ j)
//   element 4j+i = bf16_rne(((w_j >> 16i) & 0xFFFF) - 32768) * 1.75/32768 [* k_scale])
constexpr unsigned long long kTagK = 1, kTagV = 2, kTagQ = 3;
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}
__device__ __forceinline__ unsigned long long synth_key(unsigned long long seed, unsigned long long tag,
                                                        long long uid, long long pos, int layer, int head) {
  unsigned long long k = mix64(seed ^ (tag << 56));
  k = mix64(k ^ (unsigned long long)uid);
  k = mix64(k ^ (unsigned long long)pos);
  k = mix64(k ^ (unsigned long long)layer);
  k = mix64(k ^ (unsigned long long)head);
  return k;
}
// four bf16 values of chunk j packed as uint2
__device__ __forceinline__ uint2 synth_chunk(unsigned long long key, int j, float scale) {
  const unsigned long long w = mix64(key ^ (unsigned long long)j);
  float v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int u = (int)((w >> (16 * i)) & 0xFFFFull);
    v[i] = (float)(u - 32768) * 5.340576171875e-05f * scale;
  }
  return make_uint2(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]));
}

// ------------------------------------------------------------ the plan
// Per translation unit (static): uploaded by upload_plan_main / _tc.
static __constant__ PlanDev fk_plan_c[kPlanSlots];

// ------------------------------------------------------ partial bookkeeping
__device__ __forceinline__ long long part_index(const PlanDev& p, int H, int row, int slot, int head) {
  return ((long long)row * p.max_slots + slot) * H + head;
}

// Partials the merge of (row, head) combines (shared pieces + private pieces).
__device__ __forceinline__ int partial_count(const PlanDev& p, int H, int row, int head) {
  return p.row_head_count[(long long)row * H + head];
}

// Merge all partials of (row, head) into the bf16 (and optional fp32)
// output; one warp, 4 head-dim elements per lane.  Rows with no token at
// all (no partial) produce zeros.
template <int kMergeEarly = 8>
__device__ __forceinline__ void merge_row_head_warp(const ArenaDev& a, const PlanDev& p, int row, int head,
                                                    __nv_bfloat16* out, float* out_f32, int lane, int ns) {
  // (m, l) of every slot lane-parallel (slot k in lane k % 32 of round k /
  // 32, up to kMergeRounds rounds in registers) and the o (4 dims per lane)
  // of the first kMergeEarly slots in one memory round trip; any further
  // slots' o 8 at a time
  constexpr int kMergeRounds = 4;  // up to 128 partials per (row, head)
  const int H = a.num_heads;
  const long long base = part_index(p, H, row, 0, head);  // slot stride is H
  float4 v0[kMergeEarly];
#pragma unroll
  for (int k = 0; k < kMergeEarly; ++k)
    v0[k] = k < ns ? __ldcg(reinterpret_cast<const float4*>(a.part_o + (base + (long long)k * H) * kHeadDim) + lane)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
  float2 ml[kMergeRounds];
  float M = -INFINITY;
#pragma unroll
  for (int r = 0; r < kMergeRounds; ++r) {
    const int k = r * 32 + lane;
    ml[r] = k < ns ? __ldcg(&a.part_ml[base + (long long)k * H]) : make_float2(-INFINITY, 0.f);
    M = fmaxf(M, ml[r].x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float w[kMergeRounds];
  float L = 0.f;
#pragma unroll
  for (int r = 0; r < kMergeRounds; ++r) {
    w[r] = (M == -INFINITY || r * 32 + lane >= ns) ? 0.f : ex2(ml[r].x - M);
    L = fmaf(ml[r].y, w[r], L);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int nsm = min(ns, 32 * kMergeRounds);
  // (the first kMergeEarly partials' o were loaded together with the (m, l)
  // round above: one memory round trip for the common case)
#pragma unroll
  for (int k = 0; k < kMergeEarly; ++k) {
    const float wk = __shfl_sync(0xffffffffu, w[0], k);
    acc.x = fmaf(v0[k].x, wk, acc.x);
    acc.y = fmaf(v0[k].y, wk, acc.y);
    acc.z = fmaf(v0[k].z, wk, acc.z);
    acc.w = fmaf(v0[k].w, wk, acc.w);
  }
  for (int k0 = kMergeEarly; k0 < nsm; k0 += 8) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      v[k] = k0 + k < nsm ? __ldcg(reinterpret_cast<const float4*>(a.part_o + (base + (long long)(k0 + k) * H) * kHeadDim) + lane)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
    const int r = k0 >> 5;  // the 8 slots of this group share one round
    float wr = w[0];
#pragma unroll
    for (int rr = 1; rr < kMergeRounds; ++rr) wr = r == rr ? w[rr] : wr;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float wk = __shfl_sync(0xffffffffu, wr, (k0 + k) & 31);
      acc.x = fmaf(v[k].x, wk, acc.x);
      acc.y = fmaf(v[k].y, wk, acc.y);
      acc.z = fmaf(v[k].z, wk, acc.z);
      acc.w = fmaf(v[k].w, wk, acc.w);
    }
  }
  if (ns > 32 * kMergeRounds && M != -INFINITY) {  // beyond the register rounds: one slot at a time
    // (the planner keeps far fewer partials; this only guards correctness)
    for (int k = 32 * kMergeRounds; k < ns; ++k) M = fmaxf(M, __ldcg(&a.part_ml[base + (long long)k * H]).x);
    acc = make_float4(0.f, 0.f, 0.f, 0.f);  // start over with the max of every slot
    L = 0.f;
    for (int k = 0; k < ns; ++k) {
      const float2 mk = __ldcg(&a.part_ml[base + (long long)k * H]);
      const float wk = ex2(mk.x - M);
      L = fmaf(mk.y, wk, L);
      const float4 v = __ldcg(reinterpret_cast<const float4*>(a.part_o + (base + (long long)k * H) * kHeadDim) + lane);
      acc.x = fmaf(v.x, wk, acc.x);
      acc.y = fmaf(v.y, wk, acc.y);
      acc.z = fmaf(v.z, wk, acc.z);
      acc.w = fmaf(v.w, wk, acc.w);
    }
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  const long long oi = ((long long)row * H + head) * kHeadDim + lane * 4;
  const float4 r = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  *reinterpret_cast<uint2*>(out + oi) = make_uint2(pack_bf16(r.x, r.y), pack_bf16(r.z, r.w));
  if (out_f32) *reinterpret_cast<float4*>(out_f32 + oi) = r;
}
__device__ __forceinline__ void merge_row_head_warp(const ArenaDev& a, const PlanDev& p, int row, int head,
                                                    __nv_bfloat16* out, float* out_f32, int lane) {
  merge_row_head_warp<8>(a, p, row, head, out, out_f32, lane, partial_count(p, a.num_heads, row, head));
}

}  // namespace fk
