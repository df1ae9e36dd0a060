// Microtest of the tcgen05 kind::tf32 path used by the complex64 window pass (csrc/fast_tc.cu):
// one CTA computes D (M x N, fp32, TMEM) = A (M x K) * B^T (B: N x K), both K-major in shared
// memory with no swizzle, and writes D back.  Establishes (on the B200) the canonical layout /
// descriptor conventions and the TMEM accumulator layout for M = 64 and 128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_tf32_test tools/umma_tf32_test.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cmath>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: element (r, k) at (r / 8) * SBO + (k / 4) * LBO + (r % 8) * 16 + (k % 4) * 4
__host__ __device__ inline uint32_t kmaj_off(int r, int k, uint32_t lbo, uint32_t sbo) {
  return (r / 8) * sbo + (k / 4) * lbo + (r % 8) * 16 + (k % 4) * 4;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

template <int M, int N>
__device__ __forceinline__ uint32_t idesc_tf32() {
  uint32_t d = 0;
  d |= 1u << 4;          // c_format F32
  d |= 2u << 7;          // a_format TF32
  d |= 2u << 10;         // b_format TF32
  // a_major = b_major = 0 (K-major)
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(M >> 4) << 24;
  return d;
}

template <int M, int N, int K>
__global__ void k_test(const float* A, const float* B, float* D, int swap, int* lanes_out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* sA = sm;
  unsigned char* sB = sm + M * K * 4;
  const uint32_t lboA = swap ? (M / 8) * 128 : 128, sboA = swap ? 128 : (K / 4) * 128;
  const uint32_t lboB = swap ? (N / 8) * 128 : 128, sboB = swap ? 128 : (K / 4) * 128;
  // NOTE: with swap, the layout itself stays "K contiguous in 16-byte core rows", only which of the
  // two strides is called LBO changes; the data placement below follows (lbo = K step, sbo = MN step)
  const uint32_t kstepA = swap ? sboA : lboA, mnstepA = swap ? lboA : sboA;
  const uint32_t kstepB = swap ? sboB : lboB, mnstepB = swap ? lboB : sboB;
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<float*>(sA + (r / 8) * mnstepA + (k / 4) * kstepA + (r % 8) * 16 + (k % 4) * 4) = A[r * K + k];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<float*>(sB + (r / 8) * mnstepB + (k / 4) * kstepB + (r % 8) * 16 + (k % 4) * 4) = B[r * K + k];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32<M, N>();
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint64_t da = make_desc(smem_u32(sA) + kk * 2 * kstepA, lboA, sboA);
      const uint64_t db = make_desc(smem_u32(sB) + kk * 2 * kstepB, lboB, sboB);
      const uint32_t acc = kk > 0;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  // wait for the MMAs
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(ok)
          : "r"(smem_u32(&bar)), "r"(0u)
          : "memory");
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // every warp reads its lane quadrant: lanes 32 (warp % 4) .., N columns
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      const uint32_t addr = tm + ((uint32_t)(32 * warp) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 8; ++j) D[(32 * warp + lane) * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "n"(128));
  (void)lanes_out;
}

template <int M, int N, int K>
static void run(int swap) {
  std::vector<float> A(M * K), B(N * K), D(128 * N, -999.f);
  for (int r = 0; r < M; ++r)
    for (int k = 0; k < K; ++k) A[r * K + k] = (float)(((r * 7 + k * 3) % 9) - 4) + (k == 0 ? (float)r : 0.f);
  for (int r = 0; r < N; ++r)
    for (int k = 0; k < K; ++k) B[r * K + k] = (float)(((r * 5 + k * 11) % 7) - 3);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dD, D.data(), D.size() * 4, cudaMemcpyHostToDevice);
  const int smem = (M + N) * K * 4;
  cudaFuncSetAttribute(k_test<M, N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_test<M, N, K><<<1, 128, smem>>>(dA, dB, dD, swap, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("M=%d N=%d K=%d swap=%d: CUDA error %s\n", M, N, K, swap, cudaGetErrorString(e));
    exit(1);
  }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  // reference and the lane map: for every TMEM lane, which row of D (if any) it holds
  std::vector<float> R(M * N);
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < N; ++c) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[r * K + k] * B[c * K + k];
      R[r * N + c] = (float)s;
    }
  int ok_rows = 0;
  printf("M=%d N=%d K=%d swap=%d: lane -> row:", M, N, K, swap);
  for (int ln = 0; ln < 128; ++ln) {
    int found = -1;
    for (int r = 0; r < M && found < 0; ++r) {
      bool eq = true;
      for (int c = 0; c < N && eq; ++c) eq = fabsf(D[ln * N + c] - R[r * N + c]) < 1e-3f;
      if (eq) found = r;
    }
    if (found >= 0) ++ok_rows;
    printf(" %d", found);
  }
  printf("\n  rows matched: %d of %d\n", ok_rows, M);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
}

int main() {
  run<128, 32, 32>(0);
  run<64, 32, 32>(0);
  run<64, 16, 64>(0);
  run<64, 64, 64>(0);
  return 0;
}
