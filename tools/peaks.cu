// Pipe-peak microbenchmarks on B200 (sm_100a): DFMA, FFMA, DMMA (mma.sync f64) and
// TF32 mma.sync.  Prints one JSON object.  Used as the arithmetic roofline denominators
// (MEASURED_PEAKS.json has only HBM and bf16 GEMM).
#include <cuda_runtime.h>
#include <cstdio>

#define ITERS 2048

__global__ void k_dfma(double* out, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1e-12);
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 12345.678) out[0] = r;
}

__global__ void k_ffma(float* out, float s) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 1e-12f);
  float r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 12345.678f) out[0] = r;
}

__global__ void k_dmma(double* out, double s) {
  double acc[4][2];
  double a = s + threadIdx.x * 1e-9, b = s * 0.5;
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = 0;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  double r = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) r += acc[c][0] + acc[c][1];
  if (r == 12345.678) out[0] = r;
}

__global__ void k_tf32(float* out, float s) {
  float acc[4][4];
  unsigned a0 = __float_as_uint(s + threadIdx.x * 1e-9f), b0 = __float_as_uint(s * 0.5f);
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[c][q] = 0;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                   : "r"(a0), "r"(a0), "r"(a0), "r"(a0), "r"(b0), "r"(b0));
  float r = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int q = 0; q < 4; ++q) r += acc[c][q];
  if (r == 12345.678f) out[0] = r;
}

template <typename F>
static float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
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

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* dout;
  cudaMalloc(&dout, 64);
  const int blocks = sms * 8, threads = 256;
  const double nthr = double(blocks) * threads;
  float t_dfma = timeit([&] { k_dfma<<<blocks, threads>>>(dout, 1.0000001); });
  float t_ffma = timeit([&] { k_ffma<<<blocks, threads>>>((float*)dout, 1.0000001f); });
  float t_dmma = timeit([&] { k_dmma<<<blocks, threads>>>(dout, 1.0000001); });
  float t_tf32 = timeit([&] { k_tf32<<<blocks, threads>>>((float*)dout, 1.0000001f); });
  const double warps = nthr / 32;
  double dfma = 2.0 * 8 * ITERS * nthr / (t_dfma * 1e-3) / 1e12;
  double ffma = 2.0 * 16 * ITERS * nthr / (t_ffma * 1e-3) / 1e12;
  double dmma = 2.0 * 8 * 8 * 4 * 4 * ITERS * warps / (t_dmma * 1e-3) / 1e12;
  double tf32 = 2.0 * 16 * 8 * 8 * 4 * ITERS * warps / (t_tf32 * 1e-3) / 1e12;
  cudaError_t e = cudaGetLastError();
  printf("{\"dfma_tflops\": %.2f, \"ffma_tflops\": %.2f, \"dmma_sync_tflops\": %.2f, \"tf32_mma_sync_tflops\": %.2f, \"sms\": %d, \"err\": \"%s\"}\n",
         dfma, ffma, dmma, tf32, sms, cudaGetErrorString(e));
  return 0;
}
