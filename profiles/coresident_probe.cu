// Can a small CTA of a PDL-dependent kernel start on an SM while a big-smem
// CTA of its primary still runs there?  (diagnostic for the streaming merge)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cop profiles/coresident_probe.cu && /tmp/cop
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long tA[1024][2], tB[1024][2];
__device__ __forceinline__ unsigned long long gns() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void kA(int us, int trigger) {
  extern __shared__ char sm[];
  if (trigger) asm volatile("griddepcontrol.launch_dependents;");
  unsigned long long t0 = gns();
  if (threadIdx.x == 0) tA[blockIdx.x][0] = t0;
  sm[threadIdx.x] = 1;
  while (gns() - t0 < (unsigned long long)us * 1000) { }
  if (threadIdx.x == 0) tA[blockIdx.x][1] = gns();
}
__global__ void __launch_bounds__(128) kB() {
  if (threadIdx.x == 0) tB[blockIdx.x][0] = gns();
  asm volatile("griddepcontrol.wait;");
  if (threadIdx.x == 0) tB[blockIdx.x][1] = gns();
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int configs[][3] = {{160 * 1024, 320, 0}, {160 * 1024, 320, 1}, {100 * 1024, 320, 1}, {192 * 1024, 256, 1}, {32 * 1024, 320, 1}};
  for (auto& c : configs) for (int carve = 0; carve < 2; ++carve) {
    int smem = c[0], thr = c[1], pdl = c[2];
    cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (carve) cudaFuncSetAttribute(kB, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    kA<<<sms, thr, smem, s>>>(50, 1);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = sms; cfg.blockDim = 128; cfg.stream = s;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = pdl;
    cudaLaunchKernelEx(&cfg, kB);
    cudaError_t e = cudaStreamSynchronize(s);
    unsigned long long a[1024][2], b[1024][2];
    cudaMemcpyFromSymbol(a, tA, sizeof(a)); cudaMemcpyFromSymbol(b, tB, sizeof(b));
    unsigned long long a0 = ~0ull, aend = 0, bmin = ~0ull, bmax = 0;
    for (int i = 0; i < sms; ++i) { a0 = a[i][0] < a0 ? a[i][0] : a0; aend = a[i][1] > aend ? a[i][1] : aend;
      bmin = b[i][0] < bmin ? b[i][0] : bmin; bmax = b[i][0] > bmax ? b[i][0] : bmax; }
    printf("A smem %3d KB thr %d | B pdl %d carve %d: B start %.1f..%.1f us, A end %.1f us (%s)\n", smem / 1024, thr, pdl,
           carve, (bmin - a0) / 1e3, (bmax - a0) / 1e3, (aend - a0) / 1e3, cudaGetErrorString(e));
    cudaStreamDestroy(s);
  }
  return 0;
}
