// DMMA / TF32-mma.sync throughput vs warps per SM and independent chains per warp.
#include <cstdio>
#define ITERS 1024
template <int CH>
__global__ void k_dmma(double* out, double s) {
  double acc[CH][2];
  double a = s + threadIdx.x * 1e-9, b = s * 0.5;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  double r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r += acc[c][0] + acc[c][1];
  if (r == 12345.678) out[0] = r;
}
template <int CH>
__global__ void k_tf32(float* out, float s) {
  float acc[CH][4];
  unsigned a0 = __float_as_uint(s + threadIdx.x * 1e-9f), b0 = __float_as_uint(s * 0.5f);
#pragma unroll
  for (int c = 0; c < CH; ++c) for (int q = 0; q < 4; ++q) acc[c][q] = 0;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                   : "r"(a0), "r"(a0), "r"(a0), "r"(a0), "r"(b0), "r"(b0));
  float r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) for (int q = 0; q < 4; ++q) r += acc[c][q];
  if (r == 12345.678f) out[0] = r;
}
template <typename F> float tm(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize(); float best = 1e9;
  for (int r = 0; r < 3; ++r) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  return best;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 16, 32}) {
    int th = warps * 32;
    float t4 = tm([&] { k_dmma<4><<<sms, th>>>(d, 1.0000001); });
    float t24 = tm([&] { k_dmma<24><<<sms, th>>>(d, 1.0000001); });
    double w = (double)sms * warps;
    printf("DMMA warps/SM %2d: chains4 %.1f TF, chains24 %.1f TF\n", warps, 512.0 * 4 * ITERS * w / (t4 * 1e-3) / 1e12,
           512.0 * 24 * ITERS * w / (t24 * 1e-3) / 1e12);
    float u4 = tm([&] { k_tf32<4><<<sms, th>>>((float*)d, 1.0000001f); });
    float u16 = tm([&] { k_tf32<16><<<sms, th>>>((float*)d, 1.0000001f); });
    printf("TF32 warps/SM %2d: chains4 %.1f TF, chains16 %.1f TF\n", warps, 2048.0 * 4 * ITERS * w / (u4 * 1e-3) / 1e12,
           2048.0 * 16 * ITERS * w / (u16 * 1e-3) / 1e12);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
