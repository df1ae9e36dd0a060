#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int* out) {
  __shared__ uint64_t bar[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(&bar[i])), "r"(8));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // bar0: warp 0 arrives with count 8
  if (w == 0 && lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar[0])), "r"(8) : "memory");
  // bar1: warps 0..3 arrive with count 2
  if (w < 4 && lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar[1])), "r"(2) : "memory");
  // bar2: all 8 warps count 1 (no count operand)
  if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(sa(&bar[2])) : "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) {
      uint32_t ok;
      asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(sa(&bar[i])), "r"(0) : "memory");
      out[i] = ok;
    }
  }
}
int main() {
  int* d; cudaMalloc(&d, 16); cudaMemset(d, 0xff, 16);
  k<<<1, 256>>>(d);
  int h[4]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("count8 %d count2x4 %d count1x8 %d err %s\n", h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
}
