// TMA 1-D bulk-copy streaming microbenchmark: one CTA per SM streams a private slice of a
// large buffer through a ring of D chunks of C bytes (one elected producer thread, consumer
// warps wait on the full barrier and release the chunk).  Reports aggregate GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_stream tools/tma_stream.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mexp(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void marr(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ bool mtry(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
               : "=r"(ok) : "r"(su(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) { while (!mtry(b, ph)) {} }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s),
               "r"(n), "r"(su(b)) : "memory");
}

// NCW consumer warps + 1 producer warp
template <int NCW>
__global__ void k(const unsigned char* src, size_t per_cta, int C, int D, float* out, int nprod) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)C * D);
  uint64_t* empty = full + D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < D; ++i) {
      minit(&full[i], 1);
      minit(&empty[i], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned char* base = src + per_cta * blockIdx.x;
  const int64_t n = per_cta / C;
  if (warp == NCW) {
    if (lane < nprod)
      for (int64_t i = lane; i < n; i += nprod) {
        const int s = (int)(i % D);
        if (i >= D) mwait(&empty[s], (uint32_t)(((i / D) - 1) & 1));
        mexp(&full[s], C);
        bulk(sm + (size_t)s * C, base + i * C, C, &full[s]);
      }
    return;
  }
  float acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int s = (int)(i % D);
    mwait(&full[s], (uint32_t)((i / D) & 1));
    acc += reinterpret_cast<const float*>(sm + (size_t)s * C)[lane * 8 + warp];
    __syncwarp();
    if (lane == 0) marr(&empty[s]);
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)4 << 30;
  unsigned char* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  float* out;
  cudaMalloc(&out, 64);
  const size_t per_cta = (total / sms) & ~(size_t)65535;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int nprod : {1, 2, 4, 8})
  for (int C : {4096, 8192, 16384, 32768}) {
    for (int D : {4, 8, 12, 16}) {
      if (D % nprod) continue;
      const size_t smem = (size_t)C * D + 2 * D * 8;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(k<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k<8><<<sms, 9 * 32, smem>>>(src, per_cta, C, D, out, nprod);
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      k<8><<<sms, 9 * 32, smem>>>(src, per_cta, C, D, out, nprod);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("producers %d chunk %6d B x depth %2d (%6zu KB in flight): %7.1f GB/s  %s\n", nprod, C, D, (size_t)C * D / 1024,
             per_cta * sms / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
