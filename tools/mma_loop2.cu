// Microbenchmark for a "column-owner" decomposition of the c128 window pass: 4 warps per SM
// (one per sub-partition), each warp computes all 8 slots of a window for its own 8 of the 32
// right-hand-side columns, slot by slot: per slot 8 k-steps of (A: 2 x LDS.128, B: 1 x LDS.128,
// 3M sums, 6 DMMA), then a 16 x 8 epilogue to shared memory.  No cross-warp barriers.
// Reports DMMA-equivalent TF/s (512 flop per DMMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_loop2 tools/mma_loop2.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
struct Fr {
  double2 a[2];
  double as[2];
  double2 b;
  double bs;
};
__device__ __forceinline__ void ld(Fr& f, const double2* A, const double2* B, int lane) {
  f.a[0] = A[lane];
  f.a[1] = A[32 + lane];
  f.b = B[lane];
  f.as[0] = f.a[0].x + f.a[0].y;
  f.as[1] = f.a[1].x + f.a[1].y;
  f.bs = f.b.x + f.b.y;
}
template <int MI>
__device__ __forceinline__ void half(double (&p)[3][2][2], const Fr& f) {
  mma(p[0][MI][0], p[0][MI][1], f.a[MI].x, f.b.x);
  mma(p[1][MI][0], p[1][MI][1], f.a[MI].y, f.b.y);
  mma(p[2][MI][0], p[2][MI][1], f.as[MI], f.bs);
}

// MODE 0: one slot at a time; MODE 1: two slots interleaved (more independent DMMA chains)
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(double* out, int items) {
  extern __shared__ double2 sm[];
  double2* sA = sm;                 // 8 slots x 8 steps x 64
  double2* sB = sm + 8 * 8 * 64;    // per warp: 8 slots x 16 rows x 8 cols
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (int i = threadIdx.x; i < 8 * 8 * 64 + 4 * 8 * 128 * 2; i += blockDim.x) sm[i] = make_double2(1e-3 * (i & 255), 1e-4 * i);
  __syncthreads();
  double2* in = sB + warp * 2 * 8 * 128;
  double2* outb = in + 8 * 128;
  double r = 0;
  for (int it = 0; it < items; ++it) {
    for (int op = 0; op < 3; ++op) {
      if (MODE == 0) {
        for (int o = 0; o < 8; ++o) {
          double p[3][2][2] = {};
          const double2* A = sA + o * 8 * 64;
          const double2* B = in + ((o ^ op) & 7) * 128;
          Fr f[2];
          ld(f[0], A, B, lane);
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            half<0>(p, f[s & 1]);
            if (s + 1 < 8) ld(f[(s + 1) & 1], A + (s + 1) * 64, B + ((s + 1) & 3) * 32, lane);
            half<1>(p, f[s & 1]);
          }
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              outb[o * 128 + (8 * mi + g) * 8 + 2 * t + e] =
                  make_double2(p[0][mi][e] - p[1][mi][e], p[2][mi][e] - p[0][mi][e] - p[1][mi][e]);
        }
      } else {
        for (int o = 0; o < 8; o += 2) {
          double p[3][2][2] = {}, q[3][2][2] = {};
          const double2* A0 = sA + o * 8 * 64;
          const double2* A1 = A0 + 8 * 64;
          const double2* B0 = in + ((o ^ op) & 7) * 128;
          const double2* B1 = in + (((o + 1) ^ op) & 7) * 128;
          Fr f[2], h[2];
          ld(f[0], A0, B0, lane);
          ld(h[0], A1, B1, lane);
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            half<0>(p, f[s & 1]);
            half<0>(q, h[s & 1]);
            if (s + 1 < 8) {
              ld(f[(s + 1) & 1], A0 + (s + 1) * 64, B0 + ((s + 1) & 3) * 32, lane);
              ld(h[(s + 1) & 1], A1 + (s + 1) * 64, B1 + ((s + 1) & 3) * 32, lane);
            }
            half<1>(p, f[s & 1]);
            half<1>(q, h[s & 1]);
          }
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              outb[o * 128 + (8 * mi + g) * 8 + 2 * t + e] =
                  make_double2(p[0][mi][e] - p[1][mi][e], p[2][mi][e] - p[0][mi][e] - p[1][mi][e]);
              outb[(o + 1) * 128 + (8 * mi + g) * 8 + 2 * t + e] =
                  make_double2(q[0][mi][e] - q[1][mi][e], q[2][mi][e] - q[0][mi][e] - q[1][mi][e]);
            }
        }
      }
      __syncwarp();
      double2* tmp = in;
      in = outb;
      outb = tmp;
    }
  }
  r = in[lane].x;
  if (r == 12345.678) out[0] = r;
}

template <int MODE>
static void run(int sms, double* d, const char* name) {
  const int items = 64;
  const size_t smem = (8 * 8 * 64 + 4 * 8 * 128 * 2) * 16;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<MODE><<<sms, 128, smem>>>(d, items);
  cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    k<MODE><<<sms, 128, smem>>>(d, items);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double dmma = (double)sms * 4 * items * 3 * 8 * 8 * 6;
  printf("%-40s %.1f TF, %.3f ms  (%s)\n", name, dmma * 512 / (best * 1e-3) / 1e12, best,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 64);
  run<0>(sms, d, "column-owner, one slot at a time");
  run<1>(sms, d, "column-owner, two slots interleaved");
}
