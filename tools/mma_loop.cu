// Inner-loop microbenchmark for the c128 window-pass k-step: per step a warp loads its A
// fragment (2 x 16 B / lane) and B fragments (NT x 16 B / lane) from shared memory and issues
// 3 x 2 x NT DMMAs (3M complex product).  Measures DMMA-pipe throughput for:
//   mode 0: load, then the 24 DMMAs (no pipelining)
//   mode 1: software-pipelined (next step's loads between the two DMMA halves)
//   mode 2: 4M product (no 3M sums): 32 DMMAs per step, pipelined
//   mode 3: mode 1 with 16 steps unrolled (compile-time trip count)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_loop tools/mma_loop.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int NT = 4;
struct Fr {
  double2 a[2];
  double as[2];
  double2 b[NT];
  double bs[NT];
};

__device__ __forceinline__ void load(Fr& f, const double2* sA, const double2* sB, int step, int lane, const int (&bo)[NT]) {
  const double2* pa = sA + (step & 7) * 64;
  f.a[0] = pa[lane];
  f.a[1] = pa[32 + lane];
  f.as[0] = f.a[0].x + f.a[0].y;
  f.as[1] = f.a[1].x + f.a[1].y;
  const double2* pb = sB + (step & 3) * 128;
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) {
    f.b[ni] = pb[bo[ni]];
    f.bs[ni] = f.b[ni].x + f.b[ni].y;
  }
}

template <int MI>
__device__ __forceinline__ void part(double (&p)[3][2][NT][2], const Fr& f) {
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) {
    mma(p[0][MI][ni][0], p[0][MI][ni][1], f.a[MI].x, f.b[ni].x);
    mma(p[1][MI][ni][0], p[1][MI][ni][1], f.a[MI].y, f.b[ni].y);
    mma(p[2][MI][ni][0], p[2][MI][ni][1], f.as[MI], f.bs[ni]);
  }
}
template <int MI>
__device__ __forceinline__ void part4(double (&p)[3][2][NT][2], const Fr& f) {
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) {
    mma(p[0][MI][ni][0], p[0][MI][ni][1], f.a[MI].x, f.b[ni].x);
    mma(p[1][MI][ni][0], p[1][MI][ni][1], f.a[MI].y, f.b[ni].y);
    mma(p[2][MI][ni][0], p[2][MI][ni][1], f.a[MI].x, f.b[ni].y);
    mma(p[2][MI][ni][0], p[2][MI][ni][1], f.a[MI].y, f.b[ni].x);
  }
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_loop(double* out, int steps) {
  __shared__ double2 sA[8 * 64];
  __shared__ double2 sB[4 * 128 + 64];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) sA[i] = make_double2(1e-3 * i, 2e-3 * i);
  for (int i = threadIdx.x; i < 4 * 128 + 64; i += blockDim.x) sB[i] = make_double2(3e-3 * i, -1e-3 * i);
  __syncthreads();
  int bo[NT];
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) bo[ni] = t * 32 + ((8 * ni + g) ^ (((t & 3) << 1) | (t & 1)));
  double p[3][2][NT][2];
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) p[q][mi][ni][0] = p[q][mi][ni][1] = 0;
  if constexpr (MODE == 0) {
    for (int s = 0; s < steps; ++s) {
      Fr f;
      load(f, sA, sB, s, lane, bo);
      part<0>(p, f);
      part<1>(p, f);
    }
  } else if constexpr (MODE == 1 || MODE == 2) {
    Fr f0, f1;
    load(f0, sA, sB, 0, lane, bo);
    for (int s = 0; s < steps; s += 2) {
      if (MODE == 1) part<0>(p, f0); else part4<0>(p, f0);
      load(f1, sA, sB, s + 1, lane, bo);
      if (MODE == 1) part<1>(p, f0); else part4<1>(p, f0);
      if (MODE == 1) part<0>(p, f1); else part4<0>(p, f1);
      load(f0, sA, sB, s + 2, lane, bo);
      if (MODE == 1) part<1>(p, f1); else part4<1>(p, f1);
    }
  } else if constexpr (MODE == 4) {
    // slot-owner op structure: 8 pipelined k-steps, barrier, 3M epilogue to smem, barrier
    extern __shared__ double2 sO[];  // 8 warps x 512
    const int w = threadIdx.x >> 5;
    for (int s0 = 0; s0 < steps; s0 += 8) {
      Fr f[2];
      load(f[0], sA, sB, s0, lane, bo);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        part<0>(p, f[s & 1]);
        if (s + 1 < 8) load(f[(s + 1) & 1], sA, sB, s0 + s + 1, lane, bo);
        part<1>(p, f[s & 1]);
      }
      __syncthreads();
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double p1 = p[0][mi][ni][e], p2 = p[1][mi][ni][e], p3 = p[2][mi][ni][e];
            sO[w * 512 + (8 * mi + g) * 32 + ((8 * ni + 2 * t + e) ^ g)] = make_double2(p1 - p2, p3 - p1 - p2);
            p[0][mi][ni][e] = p[1][mi][ni][e] = p[2][mi][ni][e] = 0;
          }
      __syncthreads();
    }
    for (int k = threadIdx.x; k < 8 * 512; k += 256) p[0][0][0][0] += sO[k].x;
  } else {
    for (int s0 = 0; s0 < steps; s0 += 16) {
      Fr f[2];
      load(f[0], sA, sB, s0, lane, bo);
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        part<0>(p, f[s & 1]);
        if (s + 1 < 16) load(f[(s + 1) & 1], sA, sB, s0 + s + 1, lane, bo);
        part<1>(p, f[s & 1]);
      }
    }
  }
  double r = 0;
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) r += p[q][mi][ni][0] + p[q][mi][ni][1];
  if (r == 12345.678) out[0] = r;
}

template <int MODE>
static void run(int sms, double* d, const char* name, int dmma_per_step) {
  const int steps = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(k_loop<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k_loop<MODE><<<sms, 256, 65536>>>(d, steps);
  cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    k_loop<MODE><<<sms, 256, 65536>>>(d, steps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double dmma = (double)sms * 8 * steps * dmma_per_step;
  printf("%-34s %.1f TF (DMMA-equivalent, 512 flop each), %.3f ms\n", name, dmma * 512 / (best * 1e-3) / 1e12, best);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 64);
  run<0>(sms, d, "3M, load then MMA", 24);
  run<1>(sms, d, "3M, pipelined", 24);
  run<2>(sms, d, "4M, pipelined", 32);
  run<3>(sms, d, "3M, pipelined, 16 steps unrolled", 24);
  run<4>(sms, d, "3M, slot-owner op: 8 steps + 2 barriers + epilogue", 24);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
