// Pipe microbenchmarks, round 2: which mma.sync shapes reach the FP64 / TF32 tensor peak on
// B200 (sm_100a), and whether the DMMA and DFMA pipes (or TF32-MMA and FFMA) add up when
// warps of one CTA use both.  Prints one line per case: TFLOP/s (2 flops per FMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipes2 tools/pipes2.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define ITERS 1024
#define CH 12

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma1684(double (&c)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void dmma1688(double (&c)[4], double a0, double a1, double a2, double a3, double b0,
                                         double b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}
__device__ __forceinline__ void dmma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]),
        "d"(b[2]), "d"(b[3]));
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], uint32_t a, uint32_t b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a), "r"(a), "r"(a), "r"(a), "r"(b), "r"(b));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a, uint32_t b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a), "r"(a), "r"(a), "r"(a), "r"(b), "r"(b));
}
__device__ __forceinline__ void mma_i8(int (&c)[4], uint32_t a, uint32_t b) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3]) : "r"(a), "r"(a), "r"(a), "r"(a), "r"(b), "r"(b));
}

// mode: 0 dmma884, 1 dmma1684, 2 dmma1688, 3 dmma16816, 4 dfma, 5 tf32, 6 ffma, 7 bf16, 8 int8
template <int MODE>
__device__ void body(double* out, double s) {
  if constexpr (MODE == 0) {
    double acc[CH][2];
    const double a = s + threadIdx.x * 1e-9, b = s * 0.5;
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int c = 0; c < CH; ++c) dmma884(acc[c][0], acc[c][1], a, b);
    double r = 0;
    for (int c = 0; c < CH; ++c) r += acc[c][0] + acc[c][1];
    if (r == 12345.678) out[0] = r;
  } else if constexpr (MODE == 1 || MODE == 2 || MODE == 3) {
    double acc[CH][4];
    double a[8], b[4];
    for (int i = 0; i < 8; ++i) a[i] = s + threadIdx.x * 1e-9 + i;
    for (int i = 0; i < 4; ++i) b[i] = s * 0.5 + i;
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if constexpr (MODE == 1) dmma1684(acc[c], a[0], a[1], b[0]);
        if constexpr (MODE == 2) dmma1688(acc[c], a[0], a[1], a[2], a[3], b[0], b[1]);
        if constexpr (MODE == 3) dmma16816(acc[c], a, b);
      }
    double r = 0;
    for (int c = 0; c < CH; ++c) r += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    if (r == 12345.678) out[0] = r;
  } else if constexpr (MODE == 4) {
    double x[16];
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < ITERS * 4; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fma(x[i], s, 1e-12);
    double r = 0;
    for (int i = 0; i < 16; ++i) r += x[i];
    if (r == 12345.678) out[0] = r;
  } else if constexpr (MODE == 5 || MODE == 7) {
    float acc[CH][4];
    const uint32_t a = __float_as_uint((float)s + threadIdx.x * 1e-9f), b = __float_as_uint((float)s * 0.5f);
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if constexpr (MODE == 5) mma_tf32(acc[c], a, b);
        else mma_bf16(acc[c], a, b);
      }
    float r = 0;
    for (int c = 0; c < CH; ++c) r += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    if (r == 12345.678f) out[0] = r;
  } else if constexpr (MODE == 6) {
    float x[16];
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9f + i;
    const float sf = (float)s;
    for (int it = 0; it < ITERS * 8; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], sf, 1e-12f);
    float r = 0;
    for (int i = 0; i < 16; ++i) r += x[i];
    if (r == 12345.678f) out[0] = r;
  } else if constexpr (MODE == 8) {
    int acc[CH][4];
    const uint32_t a = 0x01020304u + threadIdx.x, b = 0x01010101u;
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int c = 0; c < CH; ++c) mma_i8(acc[c], a, b);
    int r = 0;
    for (int c = 0; c < CH; ++c) r += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    if (r == 12345) out[0] = r;
  }
}

// warps [0, split) run mode A, the rest mode B
template <int A, int B>
__global__ void k_mix(double* out, double s, int split) {
  if ((int)(threadIdx.x >> 5) < split)
    body<A>(out, s);
  else
    body<B>(out, s);
}

// flops per warp of one body<MODE>()
static double warp_flops(int mode) {
  switch (mode) {
    case 0: return 2.0 * 8 * 8 * 4 * CH * ITERS;
    case 1: return 2.0 * 16 * 8 * 4 * CH * ITERS;
    case 2: return 2.0 * 16 * 8 * 8 * CH * ITERS;
    case 3: return 2.0 * 16 * 8 * 16 * CH * ITERS;
    case 4: return 2.0 * 32 * 16 * ITERS * 4;
    case 5: return 2.0 * 16 * 8 * 8 * CH * ITERS;
    case 6: return 2.0 * 32 * 16 * ITERS * 8;
    case 7: return 2.0 * 16 * 8 * 16 * CH * ITERS;
    case 8: return 2.0 * 16 * 8 * 32 * CH * ITERS;
  }
  return 0;
}

template <typename F>
static float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

template <int A, int B>
static void run(const char* name, int warps, int split, int sms, double* d) {
  const float ms = timeit([&] { k_mix<A, B><<<sms, warps * 32>>>(d, 1.0000001, split); });
  const double fa = warp_flops(A) * split * sms, fb = warp_flops(B) * (warps - split) * sms;
  printf("%-28s warps/SM %2d (%2d A + %2d B): A %.1f TF  B %.1f TF  total %.1f TF  (%.3f ms)\n", name, warps, split,
         warps - split, fa / (ms * 1e-3) / 1e12, fb / (ms * 1e-3) / 1e12, (fa + fb) / (ms * 1e-3) / 1e12, ms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 64);
  for (int w : {4, 8, 16}) {
    run<0, 0>("dmma m8n8k4", w, w, sms, d);
    run<1, 1>("dmma m16n8k4", w, w, sms, d);
    run<2, 2>("dmma m16n8k8", w, w, sms, d);
    run<3, 3>("dmma m16n8k16", w, w, sms, d);
    run<4, 4>("dfma", w, w, sms, d);
    run<5, 5>("tf32 m16n8k8", w, w, sms, d);
    run<7, 7>("bf16 m16n8k16", w, w, sms, d);
    run<8, 8>("s8 m16n8k32", w, w, sms, d);
    run<6, 6>("ffma", w, w, sms, d);
  }
  run<0, 4>("mix dmma884 + dfma", 8, 4, sms, d);
  run<0, 4>("mix dmma884 + dfma", 16, 8, sms, d);
  run<3, 4>("mix dmma16816 + dfma", 8, 4, sms, d);
  run<3, 4>("mix dmma16816 + dfma", 16, 8, sms, d);
  run<5, 6>("mix tf32 + ffma", 8, 4, sms, d);
  run<5, 6>("mix tf32 + ffma", 16, 8, sms, d);
  run<0, 5>("mix dmma884 + tf32", 8, 4, sms, d);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
