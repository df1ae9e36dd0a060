// complex64 k-step microbenchmark: the 3M product on the 3xTF32 split (m16n8k8 mma.sync), as
// the c64 window pass runs it, against variants with other shared-memory operand layouts.
// 16 warps per CTA, one CTA per SM, each warp 16 rows x 16 columns (NT = 2) unless noted.
//   V0  HMMA only (operands pre-split in registers): the pipe ceiling of 9 HMMA per n-tile
//   V1  current layouts: A record (re, im) pairs -> LDS.128 x 2; B (re, im) float2 per (k, n)
//   V2  planar A record (re quad | im quad); B paired rows (re_t, re_t+4, im_t, im_t+4) float4
//   V3  V2 with 4M (12 HMMA per n-tile, no sum splits)
//   V4  V2 with A pre-split in shared memory (hi / lo of re, im, re + im)
//   V5  V2, two m-tiles per warp (32 rows x 16 columns, B splits reused), 8 warps
// Prints useful complex-MAC throughput (8 flops per complex MAC) and the HMMA-pipe TF.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_loop tools/tf32_loop.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void split(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}

template <int MT, int NT>
struct Acc {
  float p[3][MT][NT][4];
  __device__ void zero() {
    for (int q = 0; q < 3; ++q)
      for (int m = 0; m < MT; ++m)
        for (int n = 0; n < NT; ++n)
          for (int e = 0; e < 4; ++e) p[q][m][n][e] = 0.f;
  }
  __device__ float sum() const {
    float r = 0;
    for (int q = 0; q < 3; ++q)
      for (int m = 0; m < MT; ++m)
        for (int n = 0; n < NT; ++n)
          for (int e = 0; e < 4; ++e) r += p[q][m][n][e];
    return r;
  }
};

struct FA {  // split A of one m-tile
  uint32_t h[3][4], l[3][4];
};
struct FB {  // split B of one n-tile
  uint32_t h[3][2], l[3][2];
};

__device__ __forceinline__ void fa_from(FA& f, const float (&re)[4], const float (&im)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    split(re[e], f.h[0][e], f.l[0][e]);
    split(im[e], f.h[1][e], f.l[1][e]);
    split(re[e] + im[e], f.h[2][e], f.l[2][e]);
  }
}
__device__ __forceinline__ void fb_from(FB& f, const float (&re)[2], const float (&im)[2]) {
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    split(re[e], f.h[0][e], f.l[0][e]);
    split(im[e], f.h[1][e], f.l[1][e]);
    split(re[e] + im[e], f.h[2][e], f.l[2][e]);
  }
}
__device__ __forceinline__ void mac3(float (&p)[3][4], const FA& a, const FB& b) {
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    mma(p[q], a.h[q], b.l[q]);
    mma(p[q], a.l[q], b.h[q]);
    mma(p[q], a.h[q], b.h[q]);
  }
}
__device__ __forceinline__ void mac4(float (&p)[3][4], const FA& a, const FB& b) {
  // 4M: p0 += ar br - ai bi (sign folded into a copy of ai), p1 += ar bi + ai br
  uint32_t nh[4], nl[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    nh[e] = a.h[1][e] ^ 0x80000000u;
    nl[e] = a.l[1][e] ^ 0x80000000u;
  }
  mma(p[0], a.h[0], b.l[0]);
  mma(p[0], a.l[0], b.h[0]);
  mma(p[0], a.h[0], b.h[0]);
  mma(p[0], nh, b.l[1]);
  mma(p[0], nl, b.h[1]);
  mma(p[0], nh, b.h[1]);
  mma(p[1], a.h[0], b.l[1]);
  mma(p[1], a.l[0], b.h[1]);
  mma(p[1], a.h[0], b.h[1]);
  mma(p[1], a.h[1], b.l[0]);
  mma(p[1], a.l[1], b.h[0]);
  mma(p[1], a.h[1], b.h[0]);
}
__device__ __forceinline__ void fa_re_im(FA& f, const float (&re)[4], const float (&im)[4]) {  // no sum split (4M)
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    split(re[e], f.h[0][e], f.l[0][e]);
    split(im[e], f.h[1][e], f.l[1][e]);
  }
}
__device__ __forceinline__ void fb_re_im(FB& f, const float (&re)[2], const float (&im)[2]) {
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    split(re[e], f.h[0][e], f.l[0][e]);
    split(im[e], f.h[1][e], f.l[1][e]);
  }
}

// shared memory: A records 8 x 1 KB (per m-tile record: 32 lanes x 32 B), B 4 x 16 rows x 16 cols
template <int V, int MT, int NT>
__device__ __forceinline__ void step(Acc<MT, NT>& acc, const unsigned char* sA, const unsigned char* sB, int s,
                                     int lane, const int (&bo)[NT]) {
  const int t = lane & 3;
  (void)t;
  FA fa[MT];
  FB fb[NT];
  const unsigned char* ra = sA + (s & 7) * 1024 * MT;
  const unsigned char* rb = sB + (s & 3) * 2048;
  if (V == 1) {
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const float4* p = reinterpret_cast<const float4*>(ra + m * 1024);
      const float4 x = p[lane], y = p[32 + lane];
      const float re[4] = {x.x, x.z, y.x, y.z}, im[4] = {x.y, x.w, y.y, y.w};
      fa_from(fa[m], re, im);
    }
    const float2* b = reinterpret_cast<const float2*>(rb);
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const float2 v0 = b[bo[n]], v1 = b[bo[n] + 64];
      const float re[2] = {v0.x, v1.x}, im[2] = {v0.y, v1.y};
      fb_from(fb[n], re, im);
    }
  } else {
    if (V == 4) {
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const uint4* p = reinterpret_cast<const uint4*>(ra + m * 1024);  // 6 quads, reuse 2 KB region
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const uint4 h = p[(2 * q) * 32 % 64 + lane], l = p[(2 * q + 1) * 32 % 64 + lane];
          fa[m].h[q][0] = h.x, fa[m].h[q][1] = h.y, fa[m].h[q][2] = h.z, fa[m].h[q][3] = h.w;
          fa[m].l[q][0] = l.x ^ q, fa[m].l[q][1] = l.y, fa[m].l[q][2] = l.z, fa[m].l[q][3] = l.w;
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const float4* p = reinterpret_cast<const float4*>(ra + m * 1024);
        const float4 x = p[lane], y = p[32 + lane];
        const float re[4] = {x.x, x.y, x.z, x.w}, im[4] = {y.x, y.y, y.z, y.w};
        if (V == 3) fa_re_im(fa[m], re, im);
        else fa_from(fa[m], re, im);
      }
    }
    const float4* b = reinterpret_cast<const float4*>(rb);
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const float4 v = b[bo[n]];
      const float re[2] = {v.x, v.y}, im[2] = {v.z, v.w};
      if (V == 3) fb_re_im(fb[n], re, im);
      else fb_from(fb[n], re, im);
    }
  }
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      float(&p)[3][4] = *reinterpret_cast<float(*)[3][4]>(&acc.p[0][m][n][0]);
      // acc.p is [q][m][n][e]; gather a [q][e] view through copies
      float c[3][4];
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) c[q][e] = acc.p[q][m][n][e];
      if (V == 3) mac4(c, fa[m], fb[n]);
      else mac3(c, fa[m], fb[n]);
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc.p[q][m][n][e] = c[q][e];
      (void)p;
    }
}

template <int V, int MT, int NT, int W>
__global__ void __launch_bounds__(W * 32, 1) k_loop(float* out, int steps) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned char* sA = sm;               // 16 KB
  unsigned char* sB = sm + 16384;       // 8 KB
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 6144; i += blockDim.x)
    reinterpret_cast<float*>(sm)[i] = 1e-3f * (i % 97) - 0.04f;
  __syncthreads();
  int bo[NT];
  const int c0w = (w & 1) * 8 * NT % 16;
#pragma unroll
  for (int n = 0; n < NT; ++n) bo[n] = V == 1 ? t * 16 + ((c0w + 8 * n + g) ^ (t << 2)) : t * 16 + ((c0w + 8 * n + g) ^ (t << 2));
  Acc<MT, NT> acc;
  acc.zero();
  if (V == 0) {
    FA fa[MT];
    FB fb[NT];
    for (int m = 0; m < MT; ++m)
      for (int q = 0; q < 3; ++q)
        for (int e = 0; e < 4; ++e) fa[m].h[q][e] = fa[m].l[q][e] = __float_as_uint(sm[lane + q + e] * 1.f);
    for (int n = 0; n < NT; ++n)
      for (int q = 0; q < 3; ++q)
        for (int e = 0; e < 2; ++e) fb[n].h[q][e] = fb[n].l[q][e] = lane + q + e;
    for (int s = 0; s < steps; ++s) {
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          float c[3][4];
#pragma unroll
          for (int q = 0; q < 3; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) c[q][e] = acc.p[q][m][n][e];
          mac3(c, fa[m], fb[n]);
#pragma unroll
          for (int q = 0; q < 3; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc.p[q][m][n][e] = c[q][e];
        }
    }
  } else {
    for (int s0 = 0; s0 < steps; s0 += 4) {
#pragma unroll
      for (int s = 0; s < 4; ++s) step<V, MT, NT>(acc, sA, sB, s0 + s + w, lane, bo);
    }
  }
  const float r = acc.sum();
  if (r == 12345.678f) out[0] = r;
}

template <int V, int MT, int NT, int W>
static void run(int sms, float* d, const char* name) {
  const int steps = 8192;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int smem = 24576;
  cudaFuncSetAttribute(k_loop<V, MT, NT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_loop<V, MT, NT, W><<<sms, W * 32, smem>>>(d, steps);
  cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    k_loop<V, MT, NT, W><<<sms, W * 32, smem>>>(d, steps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double cmac = (double)sms * W * steps * MT * NT * 16 * 8 * 8;  // complex MACs
  const double hmma = (double)sms * W * steps * MT * NT * (V == 3 ? 12 : 9);
  printf("%-50s useful %.1f TF (8 flop/cMAC), HMMA pipe %.1f TF, %.3f ms\n", name, cmac * 8 / (best * 1e-3) / 1e12,
         hmma * 2048 / (best * 1e-3) / 1e12, best);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d;
  cudaMalloc(&d, 64);
  run<0, 1, 2, 16>(sms, d, "V0 HMMA only, 16 warps NT=2");
  run<1, 1, 2, 16>(sms, d, "V1 current layouts, 16 warps NT=2");
  run<2, 1, 2, 16>(sms, d, "V2 planar A, paired-row B, 16 warps NT=2");
  run<3, 1, 2, 16>(sms, d, "V3 planar, 4M, 16 warps NT=2");
  run<4, 1, 2, 16>(sms, d, "V4 planar, A pre-split, 16 warps NT=2");
  run<2, 2, 2, 8>(sms, d, "V5 planar, 2 m-tiles, 8 warps NT=2");
  run<2, 2, 2, 16>(sms, d, "V5b planar, 2 m-tiles, 16 warps NT=2");
  run<1, 2, 2, 8>(sms, d, "V1 current, 2 m-tiles, 8 warps NT=2");
  run<2, 1, 4, 8>(sms, d, "V2 planar, NT=4, 8 warps");
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
