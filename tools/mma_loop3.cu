// DMMA k-step microbenchmark, round 2: how the warp layout of the window-pass kernel maps onto
// the FP64 tensor pipe.  Each warp runs k-steps of the 3M complex product (load A: 2 x 16 B/lane,
// B: NT x 16 B/lane from shared memory, 2 + NT DADDs, 6 NT DMMAs), software-pipelined.
//   L(NT, W):    pure loop, W warps per CTA (1 CTA per SM)
//   OP(NT, W):   op structure: 8 k-steps, 3M epilogue to shared memory, one named barrier per
//                group of W/2 warps (two independent column groups)
//   OPB(NT, W):  as OP, plus a group barrier before the epilogue (two barriers per op)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_loop3 tools/mma_loop3.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NT>
struct Fr {
  double2 a[2];
  double as[2];
  double2 b[NT];
  double bs[NT];
};

template <int NT>
__device__ __forceinline__ void load(Fr<NT>& f, const double2* sA, const double2* sB, int step, int lane,
                                     const int (&bo)[NT]) {
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

template <int NT>
__device__ __forceinline__ void mac(double (&p)[3][2][NT][2], const Fr<NT>& f) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      mma(p[0][mi][ni][0], p[0][mi][ni][1], f.a[mi].x, f.b[ni].x);
      mma(p[1][mi][ni][0], p[1][mi][ni][1], f.a[mi].y, f.b[ni].y);
      mma(p[2][mi][ni][0], p[2][mi][ni][1], f.as[mi], f.bs[ni]);
    }
}

template <int NT, int W, int MODE>
__global__ void __launch_bounds__(W * 32, 1) k_loop(double* out, int steps) {
  extern __shared__ double2 sm[];
  double2* sA = sm;             // 8 x 64
  double2* sB = sm + 512;       // 4 x 128 + 64
  double2* sO = sm + 512 + 576; // W x 256
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) sA[i] = make_double2(1e-3 * i, 2e-3 * i);
  for (int i = threadIdx.x; i < 576; i += blockDim.x) sB[i] = make_double2(3e-3 * i, -1e-3 * i);
  __syncthreads();
  int bo[NT];
  const int c0w = (w & 1) * 8 * NT % 32;
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) bo[ni] = t * 32 + ((c0w + 8 * ni + g) ^ (((t & 3) << 1) | (t & 1)));
  double p[3][2][NT][2];
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) p[q][mi][ni][0] = p[q][mi][ni][1] = 0;
  const int grp = w / (W / 2);
  for (int s0 = 0; s0 < steps; s0 += 8) {
    Fr<NT> f[2];
    load(f[0], sA, sB, s0, lane, bo);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (s + 1 < 8) load(f[(s + 1) & 1], sA, sB, s0 + s + 1, lane, bo);
      mac(p, f[s & 1]);
    }
    if (MODE >= 1) {
      if (MODE == 2) asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(W * 16) : "memory");
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double p1 = p[0][mi][ni][e], p2 = p[1][mi][ni][e], p3 = p[2][mi][ni][e];
            sO[w * 256 + ((8 * mi + g) * 16 + ((8 * ni + 2 * t + e) ^ g)) % 256] = make_double2(p1 - p2, p3 - p1 - p2);
            p[0][mi][ni][e] = p[1][mi][ni][e] = p[2][mi][ni][e] = 0;
          }
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(W * 16) : "memory");
    }
  }
  double r = 0;
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) r += p[q][mi][ni][0] + p[q][mi][ni][1];
  if (MODE >= 1) r += sO[(threadIdx.x * 7) % (W * 256)].x;
  if (r == 12345.678) out[0] = r;
}

template <int NT, int W, int MODE>
static void run(int sms, double* d, const char* name) {
  const int steps = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int smem = (512 + 576 + W * 256) * 16;
  cudaFuncSetAttribute(k_loop<NT, W, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_loop<NT, W, MODE><<<sms, W * 32, smem>>>(d, steps);
  cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    k_loop<NT, W, MODE><<<sms, W * 32, smem>>>(d, steps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double dmma = (double)sms * W * steps * 6 * NT;
  printf("%-44s %.1f TF (DMMA flops), %.3f ms\n", name, dmma * 512 / (best * 1e-3) / 1e12, best);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 64);
  run<4, 8, 0>(sms, d, "loop NT=4 W=8");
  run<2, 8, 0>(sms, d, "loop NT=2 W=8");
  run<2, 16, 0>(sms, d, "loop NT=2 W=16");
  run<1, 16, 0>(sms, d, "loop NT=1 W=16");
  run<4, 8, 1>(sms, d, "op NT=4 W=8 (1 barrier)");
  run<2, 16, 1>(sms, d, "op NT=2 W=16 (1 barrier)");
  run<2, 16, 2>(sms, d, "op NT=2 W=16 (2 barriers)");
  run<1, 16, 1>(sms, d, "op NT=1 W=16 (1 barrier)");
  run<4, 8, 2>(sms, d, "op NT=4 W=8 (2 barriers)");
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
