// Minimal probe: does compute-sanitizer racecheck flag shared-memory reads that follow an
// mbarrier wait on a cp.async.bulk global->shared copy (the textbook TMA pattern)?
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const uint4* src, uint4* dst, uint4* gmem, int S) {
  __shared__ __align__(16) uint4 buf[64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(1024));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(buf)), "l"(src), "r"(1024), "r"(sa(&bar)) : "memory");
  }
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(sa(&bar)) : "memory");
  } while (!ok);
  // the replay kernel's d_ptr pattern: a generic pointer that is shared below S, global above
  const uint4* p = (int)threadIdx.x < S ? buf + threadIdx.x : gmem + threadIdx.x;
  dst[threadIdx.x] = *p;
}
int main() {
  uint4 *s, *d;
  cudaMalloc(&s, 1024); cudaMalloc(&d, 1024);
  cudaMemset(s, 7, 1024);
  uint4* g;
  cudaMalloc(&g, 1024);
  k<<<1, 64>>>(s, d, g, 64);
  uint4 h[64];
  cudaMemcpy(h, d, 1024, cudaMemcpyDeviceToHost);
  printf("probe done: %u (expect %u)\n", h[63].w, 0x07070707u);
  return 0;
}
