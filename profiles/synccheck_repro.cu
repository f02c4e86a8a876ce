// Minimal repro: compute-sanitizer synccheck reports "Barrier error detected.
// Missing wait" when an mbarrier completes a phase that no thread waits for
// and is then arrived on again -- legal per the PTX mbarrier model (a phase
// needs no observer; parity waits only need the awaited phase to be at most
// one behind).  Round 1's fk_prefix_tc_kernel committed an "O done" barrier
// after every P.V tile and waited on it only at piece ends and rescales,
// which synccheck reported at mma_commit; round 2 signals "O includes PV(u)"
// through the V-stage "empty" barrier instead, whose every phase the TMA
// producer waits for, and synccheck is clean on the kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/sc profiles/synccheck_repro.cu
//   compute-sanitizer --tool synccheck /tmp/sc 0   # skipped phase: reported
//   compute-sanitizer --tool synccheck /tmp/sc 1   # every phase waited: clean
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void wait_parity(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
}

__global__ void phases(int wait_every, int* out) {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)) : "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k) {
      arrive(&bar);                        // completes phase k
      if (wait_every) wait_parity(&bar, k & 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 32) {
    wait_parity(&bar, 1);                  // phase 3 completed (current phase 4, parity 0)
    out[0] = 1;
  }
}

int main(int argc, char** argv) {
  const int wait_every = argc > 1 ? atoi(argv[1]) : 0;
  int* d = nullptr;
  cudaMalloc(&d, sizeof(int));
  phases<<<1, 64>>>(wait_every, d);
  const cudaError_t e = cudaDeviceSynchronize();
  int h = 0;
  cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost);
  printf("wait_every=%d: %s, out=%d\n", wait_every, cudaGetErrorString(e), h);
  return e == cudaSuccess ? 0 : 1;
}
