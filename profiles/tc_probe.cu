// Descriptor / layout probe for the tcgen05 prefix kernel (not product code).
// Checks, on one CTA, the exact operand layouts fk_prefix_tc_kernel uses:
//   (1) S = Q.K^T   SS MMA, Q and K K-major SWIZZLE_128B in smem
//   (2) O = P.V     TS MMA, P (bf16x2 packed) in TMEM, V MN-major SW128 smem
// against a CPU reference, for a few descriptor variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2405_19888_b200/csrc -I../include \
//        -o build/tc_probe tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "fk_tcgen05.cuh"

using namespace fk;

__device__ __forceinline__ uint32_t swz(int row, int c16) {
  return (uint32_t)((c16 >> 3) * 16384 + row * 128 + (((c16 & 7) ^ (row & 7)) << 4));
}

// mode 0: QK test; mode 1: PV test.  variant selects descriptor options.
__global__ void __launch_bounds__(128, 1) probe(int mode, int variant, const __nv_bfloat16* A, const __nv_bfloat16* Bm,
                                                float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;          // 32 KiB
  uint8_t* sB = sm + 32768;  // 32 KiB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  // row t of each 128x128 bf16 operand -> swizzled smem
  for (int c = 0; c < 16; ++c) {
    *reinterpret_cast<uint4*>(sA + swz(t, c)) = reinterpret_cast<const uint4*>(A + t * 128)[c];
    *reinterpret_cast<uint4*>(sB + swz(t, c)) = reinterpret_cast<const uint4*>(Bm + t * 128)[c];
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t lane_tm = tm + ((uint32_t)(warp * 32) << 16);
  if (mode == 1) {
    // P row t (from A): tokens 0..127 packed 2 per column at columns 0..63
    uint32_t pk[16];
    for (int cc = 0; cc < 4; ++cc) {
      for (int e = 0; e < 16; ++e) {
        const __nv_bfloat16* src = A + t * 128 + cc * 32 + 2 * e;
        pk[e] = (uint32_t)(*reinterpret_cast<const unsigned short*>(src)) |
                ((uint32_t)(*reinterpret_cast<const unsigned short*>(src + 1)) << 16);
      }
      tmem_st16(lane_tm + 128 + cc * 16, pk);
    }
    tmem_wait_st();
    tc_fence_before();
  }
  __syncthreads();
  if (t == 0) {
    tc_fence_after();
    const uint32_t a = smem_u32(sA), b = smem_u32(sB);
    if (mode == 0) {
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        const uint32_t lbo = variant == 1 ? 0 : 16;
        mma_ss(tm, sdesc(a + off, lbo, 1024), sdesc(b + off, lbo, 1024), kIdescQK, kk > 0);
      }
    } else {
      for (int kk = 0; kk < 8; ++kk) {
        uint64_t bd;
        if (variant == 0) bd = sdesc(b + kk * 2048, 16384, 1024);
        else bd = sdesc(b + kk * 2048, 1024, 16384);  // LBO/SBO swapped
        mma_ts(tm, tm + 128 + kk * 8, bd, kIdescPV, kk > 0);
      }
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int cc = 0; cc < 4; ++cc) {
    uint32_t r[32];
    tmem_ld32(lane_tm + cc * 32, r);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) out[t * 128 + cc * 32 + e] = __uint_as_float(r[e]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

static float bf(unsigned short h) {
  unsigned int u = (unsigned int)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main() {
  const int N = 128 * 128;
  std::vector<unsigned short> ha(N), hb(N);
  srand(1);
  for (int i = 0; i < N; ++i) {
    float x = (rand() / (float)RAND_MAX - 0.5f) * 2, y = (rand() / (float)RAND_MAX - 0.5f) * 2;
    unsigned int ux, uy;
    memcpy(&ux, &x, 4);
    memcpy(&uy, &y, 4);
    ha[i] = ux >> 16;
    hb[i] = uy >> 16;
  }
  __nv_bfloat16 *da, *db;
  float* dout;
  cudaMalloc(&da, N * 2);
  cudaMalloc(&db, N * 2);
  cudaMalloc(&dout, N * 4);
  cudaMemcpy(da, ha.data(), N * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), N * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  std::vector<float> out(N);
  for (int mode = 0; mode < 2; ++mode)
    for (int variant = 0; variant < 2; ++variant) {
      cudaMemset(dout, 0, N * 4);
      probe<<<1, 128, 70000>>>(mode, variant, da, db, dout);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(out.data(), dout, N * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0, maxref = 0;
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < 128; ++j) {
          double ref = 0;
          for (int k = 0; k < 128; ++k)
            ref += mode == 0 ? (double)bf(ha[i * 128 + k]) * bf(hb[j * 128 + k])   // Q.K^T
                             : (double)bf(ha[i * 128 + k]) * bf(hb[k * 128 + j]);  // P.V
          maxerr = fmax(maxerr, fabs(ref - out[i * 128 + j]));
          maxref = fmax(maxref, fabs(ref));
        }
      printf("mode=%s variant=%d err=%s max_abs_err=%.3e (max |ref| %.2f) out[0..3]=%.3f %.3f %.3f %.3f\n",
             mode ? "PV" : "QK", variant, cudaGetErrorString(e), maxerr, maxref, out[0], out[1], out[2], out[3]);
    }
  return 0;
}
