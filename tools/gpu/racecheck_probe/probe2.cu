// Probe 2: one warp reuses its shared buffer for two bulk copies (parity 0 then 1), reading
// it between them (lane-distributed reads) -- the replay kernel's chain-after-chain pattern.
// SYNC selects what separates the reads of copy 1 from the async writes of copy 2.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ void wait(uint64_t* bar, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(sa(bar)), "r"(ph) : "memory");
  } while (!ok);
}
__global__ void k(const uint4* src, uint4* dst, int mode) {
  __shared__ __align__(16) uint4 buf[32];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < 2; it++) {
    if (mode == 1) __syncwarp();
    if (mode == 2) __syncthreads();
    if (mode == 3) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(512));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(buf)), "l"(src + 32 * it), "r"(512), "r"(sa(&bar)) : "memory");
    }
    wait(&bar, it & 1);
    acc.x += buf[(lane + it) & 31].x;  // lane-distributed reads of the copied data
    __syncwarp();
  }
  dst[lane] = acc;
}
int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  uint4 *s, *d;
  cudaMalloc(&s, 2048); cudaMalloc(&d, 512);
  cudaMemset(s, 1, 2048);
  k<<<1, 32>>>(s, d, mode);
  uint4 h[32];
  cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
  printf("mode %d done: %u\n", mode, h[0].x);
  return 0;
}
