// HBM read-ceiling probe for the private-stream access pattern (not product
// code; run by hand under gpurun to size the design).  Streams 8 KiB "pages"
// (two 4 KiB halves in different planes, like K and V) into per-warp smem
// rings with 1-D bulk copies and no compute, for several layouts / depths,
// and a plain coalesced LDG.128 read for reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mem_probe mem_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) stream_kernel(const char* base, const long long* off_k,
                                                                const long long* off_v, int units, int per,
                                                                float* sink) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t full[WARPS][STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * WARPS + warp;
  const int u0 = gw * per, u1 = min(units, u0 + per);
  if (u0 >= u1) return;
  char* ring = smem + warp * STAGES * 8192;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  auto issue = [&](int s, int u) {
    uint32_t bar = smem_u32(&full[warp][s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(8192));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                     smem_u32(ring + s * 8192)), "l"(base + off_k[u]), "r"(bar) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                     smem_u32(ring + s * 8192 + 4096)), "l"(base + off_v[u]), "r"(bar) : "memory");
  };
  int pu = u0;
  if (lane == 0)
    for (int s = 0; s < STAGES && pu < u1; ++s, ++pu) issue(s, pu);
  pu = __shfl_sync(0xffffffffu, pu, 0);
  float acc = 0.f;
  for (int u = u0; u < u1; ++u) {
    const int s = (u - u0) % STAGES;
    const uint32_t par = ((u - u0) / STAGES) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(ok) : "r"(smem_u32(&full[warp][s])), "r"(par) : "memory");
    acc += *reinterpret_cast<const float*>(ring + s * 8192 + lane * 4);
    __syncwarp();
    if (lane == 0 && pu < u1) {
      asm volatile("fence.proxy.async.shared::cta;");
      issue(s, pu);
    }
    ++pu;
  }
  if (acc == 12345.f) sink[gw] = acc;
}

__global__ void ldg_kernel(const int4* p, long long n, float* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int4 v = __ldg(p + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 12345) sink[0] = acc.y;
}

template <int STAGES, int WARPS>
float run(const char* base, const std::vector<long long>& k, const std::vector<long long>& v, float* sink) {
  long long *dk, *dv;
  cudaMalloc(&dk, k.size() * 8);
  cudaMalloc(&dv, v.size() * 8);
  cudaMemcpy(dk, k.data(), k.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, v.data(), v.size() * 8, cudaMemcpyHostToDevice);
  int units = (int)k.size();
  int warps = 148 * WARPS;
  int per = (units + warps - 1) / warps;
  int smem = WARPS * STAGES * 8192;
  cudaFuncSetAttribute(stream_kernel<STAGES, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) stream_kernel<STAGES, WARPS><<<148, WARPS * 32, smem>>>(base, dk, dv, units, per, sink);
  cudaEventRecord(a);
  const int R = 20;
  for (int i = 0; i < R; ++i) stream_kernel<STAGES, WARPS><<<148, WARPS * 32, smem>>>(base, dk, dv, units, per, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(dk);
  cudaFree(dv);
  return (double)units * 8192 * R / (ms * 1e-3) / 1e9;
}

int main() {
  const int H = 40, P = 2048;                   // planes x pages like the 13B arena
  const long long plane = (long long)P * 4096;  // bytes per plane
  const long long L = 8;                        // layers allocated (span beyond L2)
  const size_t bytes = (size_t)L * 2 * H * plane;
  char* base;
  cudaMalloc(&base, bytes);
  cudaMemset(base, 1, bytes);
  float* sink;
  cudaMalloc(&sink, 1 << 20);
  std::mt19937 rng(1);
  // private pages: 64 rows x 16 pages, pages 375.. (like the headline), unit order (head, entry)
  std::vector<int> rowpages;
  for (int i = 0; i < 1024; ++i) rowpages.push_back(375 + i);
  auto make = [&](int layer, bool shuffle_pages, bool page_major) {
    std::vector<long long> k, v;
    std::vector<int> pg = rowpages;
    if (shuffle_pages) std::shuffle(pg.begin(), pg.end(), rng);
    for (int h = 0; h < H; ++h)
      for (int e = 0; e < (int)pg.size(); ++e) {
        if (page_major) {  // [L][P][2][H][16][128]
          long long pb = ((long long)layer * P + pg[e]) * 2 * H * 4096;
          k.push_back(pb + (0LL * H + h) * 4096);
          v.push_back(pb + (1LL * H + h) * 4096);
        } else {  // [L][2][H][P][16][128]
          k.push_back(((long long)(layer * 2 + 0) * H + h) * plane + (long long)pg[e] * 4096);
          v.push_back(((long long)(layer * 2 + 1) * H + h) * plane + (long long)pg[e] * 4096);
        }
      }
    return std::make_pair(k, v);
  };
  for (int pm = 0; pm < 2; ++pm)
    for (int sh = 0; sh < 2; ++sh) {
      auto kv = make(3, sh, pm);
      printf("layout=%s pages=%s  S3W8 %.0f  S4W6 %.0f  S2W12 %.0f  S6W4 %.0f GB/s\n", pm ? "page-major" : "plane-major",
             sh ? "shuffled" : "sorted", run<3, 8>(base, kv.first, kv.second, sink),
             run<4, 6>(base, kv.first, kv.second, sink), run<2, 12>(base, kv.first, kv.second, sink),
             run<6, 4>(base, kv.first, kv.second, sink));
    }
  // coalesced read of 335 MB
  long long n = 335LL * 1024 * 1024 / 16;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) ldg_kernel<<<148 * 8, 512>>>((const int4*)base, n, sink);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) ldg_kernel<<<148 * 8, 512>>>((const int4*)(base + (i % 4) * n * 16), n, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("LDG.128 coalesced read: %.0f GB/s\n", n * 16.0 * 20 / (ms * 1e-3) / 1e9);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
