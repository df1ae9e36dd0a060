// Device building blocks shared by the fast-path kernels (fast.cu: window passes, leaf.cu: leaf
// products): mbarrier / TMA helpers and the two tensor-pipe complex-product policies.
//
// complex128 (PolC128): mma.sync.m8n8k4.f64 ("DMMA") with the 3-multiplication product
//     P1 = Ar Br,  P2 = Ai Bi,  P3 = (Ar + Ai)(Br + Bi);   Re = P1 - P2,  Im = P3 - P1 - P2.
// (DMMA and DFMA share one FP64 budget on B200 -- profiles/r01_pipes2.txt -- so fewer
// multiplications is the lever.)
// complex64 (PolC64): the same 3M product on mma.sync.m16n8k8.tf32 with the 3xTF32 split
// x = hi + lo, a*b ~ ah*bh + ah*bl + al*bh: FP32-level accuracy at tensor-pipe rate (plain TF32,
// ~1e-3, would fail the 1e-5 bar -- SURVEY 7.3).
//
// A operands (factor blocks) arrive as 1 KB k-step records in MMA fragment order (written once
// at bf_create, plan.cu fill_step).  B operands come from
//   * a half slab in shared memory: 16 rows x 16 columns, element (row, col) at
//     row*16 + (col ^ swz(row)) (bank-conflict free for C-fragment stores and B-fragment loads);
//   * a column-major box of user rows in shared memory (TMA 2-D tile of X);
//   * global memory through a row permutation (gather fallback).
#pragma once

#include <cuda.h>
#include <cstdio>

#include "fast.cuh"

namespace bfa {

// ---- mbarrier / TMA helpers -----------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// 1-D bulk copy global -> shared (TMA), completion counted on `bar` (complete_tx)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// bulk prefetch of a global range into L2 (no shared memory, no completion): the operand stream
// warms L2 a few pages ahead of the ring so that the page's own bulk copy is an L2 hit
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
// 2-D tensor tile load (TMA) into shared memory, completion counted on `bar`
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait for the phase of `bar` with the given parity.  A watchdog turns a protocol deadlock into
// a trapped launch (BF_ERR_CUDA on the next call) instead of a hung device.
static __device__ __noinline__ void mbar_wait_slow(uint64_t* bar, uint32_t parity, int tag) {
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > (1ll << 34)) {
      printf("bfapply: mbarrier watchdog block %d thread %d tag %d parity %u\n", blockIdx.x, threadIdx.x, tag, parity);
      __trap();
    }
  }
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, int tag = 0) {
  if (!mbar_try(bar, parity)) mbar_wait_slow(bar, parity, tag);
}
// shared-memory counter increment with acquire-release semantics (the last arriver of a release
// count re-arms a buffer with TMA: every arriver's reads of it happen before)
__device__ __forceinline__ int atom_add_acqrel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;\n" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}
// Page-release counter increment without the acquire-release fence (SASS: MEMBAR.ALL.CTA before
// the ATOMS, which also waits for the thread's in-flight global stores).  Sufficient for the
// ring pages: a warp releases a page only after the DMMAs / HMMAs of its last k-step on that page
// have issued, and those read the registers its LDS wrote, so every shared-memory read of the
// page is complete when the counter moves; the last arriver's TMA then overwrites it.
// (-DBF_RELEASE_ACQREL=1 restores the fenced form, for the A/B.)
#ifndef BF_RELEASE_ACQREL
#define BF_RELEASE_ACQREL 0
#endif
__device__ __forceinline__ int atom_add_release_page(int* p, int v) {
#if BF_RELEASE_ACQREL
  return atom_add_acqrel(p, v);
#else
  int old;
  asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], %2;\n" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
#endif
}
// conditional negation by flipping the sign bit on the integer pipe (a select of -x would cost
// an FP64-pipe DADD next to the DMMAs)
__device__ __forceinline__ double conj_im(double x, bool cj) {
  return __longlong_as_double(__double_as_longlong(x) ^ ((long long)cj << 63));
}
__device__ __forceinline__ float conj_im(float x, bool cj) {
  return __int_as_float(__float_as_int(x) ^ ((int)cj << 31));
}
// Programmatic dependent launch (PDL): the fused-path kernels are launched with programmatic
// stream serialization, so the next launch's CTAs start (barrier init, factor prefetch) on SMs
// this grid's tail frees.  pdl_wait() returns once every earlier grid on the stream has completed
// and its memory is visible -- no thread touches memory earlier stream work may write or read
// (slabs, X, Y) before it; factor records are immutable after create and may be read before.
// Both are no-ops for a launch without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
// named barrier over `nthreads` threads (ids >= 1; 0 is __syncthreads)
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// ======================================================================================
// complex128 policy: DMMA m8n8k4, fragments (lane = 4g + t):
//   A (8x4): A[g][t];  B (4x8): B[t][g];  C (8x8): C[g][2t+e].
// One k-step record (1 KB): [mi][lane] double2 for the 16 x 4 block.
// With KS = 4 the slab swizzle of row k0 + t depends only on t, so every B-fragment address is
// slab + k0 * 16 + (a lane constant).
// ======================================================================================
template <int NT_>
struct PolC128 {
  using E = double2;
  static constexpr int KS = 4;
  static constexpr int NT = NT_;  // 8-column n-tiles per warp
  __host__ __device__ static __forceinline__ int swz(int row) { return ((row & 3) << 1) | (row & 1); }
  __device__ static __forceinline__ void mma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
  }
  // operands of one k-step, with the 3M sums precomputed
  struct Frags {
    double2 a[2];
    double as[2];
    double2 b[NT];
    double bs[NT];
  };
  static constexpr bool LEAF_OPS = true;  // the pass kernel may run the fused leaf ops
  static constexpr bool PAIR_SHARE = false;  // see PolC64T
  // lane-constant element offset of B row t, n-tile ni (k0 = 0) inside a half slab
  __device__ static __forceinline__ int boff(int t, int g, int c0w, int ni) {
    return t * FAST_HC + ((c0w + 8 * ni + g) ^ swz(t));
  }
  // leaf kernels: n-tile ni of the 32-column tile = [half ni / 2][columns 8 (ni & 1) ..]
  __device__ static __forceinline__ int leaf_boff(int ni, int t, int g) {
    return (ni >> 1) * FAST_HSLAB + boff(t, g, 8 * (ni & 1), 0);
  }
  // byte offset of the warp's part of a factor record (all of it)
  __device__ static __forceinline__ int rec_off(int) { return 0; }
  // half-slab element (r, c): r * 16 + (c ^ swz(r))
  __device__ static __forceinline__ void slab_put(E* hs, int r, int c, E v) { hs[r * FAST_HC + (c ^ swz(r))] = v; }
  template <class Ac>
  __device__ static __forceinline__ void store_slab(const Ac& acc, E* hs, int c0w, int g, int t, int) {
    acc.each(g, t, [&](int r, int c, E v) { slab_put(hs, r, c0w + c, v); });
  }
  __device__ static __forceinline__ void load_a(Frags& f, const unsigned char* rec, int lane) {
    const E* p = reinterpret_cast<const E*>(rec);
    f.a[0] = p[lane];
    f.a[1] = p[32 + lane];
    f.as[0] = f.a[0].x + f.a[0].y;
    f.as[1] = f.a[1].x + f.a[1].y;
  }
  __device__ static __forceinline__ void set_b(Frags& f, int ni, E v) {
    f.b[ni] = v;
    f.bs[ni] = v.x + v.y;
  }
  __device__ static __forceinline__ void load_b(Frags& f, const E* slab_k0, const int (&bo)[NT]) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) set_b(f, ni, slab_k0[bo[ni]]);
  }
  // from a column-major box (element (k, c) at c * ldb + k) in shared memory, rows k0..
  __device__ static __forceinline__ void load_b_col(Frags& f, const E* box, int ldb, int k0, int c0w, int g, int t,
                                                    bool cj) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      E v = box[(c0w + 8 * ni + g) * ldb + k0 + t];
      v.y = conj_im(v.y, cj);
      set_b(f, ni, v);
    }
  }
  static constexpr int XROWS = 1;
  __device__ static __forceinline__ void x_rows(int64_t (&p)[XROWS], int64_t k0, int t) { p[0] = k0 + t; }
  // from global memory: user rows rows[] (already permuted), columns col0 + 8 ni + g
  __device__ static __forceinline__ void load_b_x(Frags& f, const E* __restrict__ X, const int64_t (&rows)[XROWS],
                                                  int64_t ldx, int col0, int g, int nrhs, bool cj) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const int col = col0 + 8 * ni + g;
      E v = col < nrhs ? __ldg(X + rows[0] + (int64_t)col * ldx) : make_double2(0.0, 0.0);
      v.y = conj_im(v.y, cj);
      set_b(f, ni, v);
    }
  }
  // the product the fused kernels run: 3M (FP64 pipe is the bound; the 3M sums are cheap)
  struct Acc;
  using FFrags = Frags;
  using FAcc = Acc;
  __device__ static __forceinline__ void load_fa(Frags& f, const unsigned char* rec, int lane) { load_a(f, rec, lane); }
  struct Acc {
    double p[3][2][NT][2];
    __device__ __forceinline__ void zero() {
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) p[q][mi][ni][0] = p[q][mi][ni][1] = 0.0;
    }
    // one k-step: 3 x 2 x NT DMMAs
    __device__ __forceinline__ void mac(const Frags& f) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
          mma(p[0][mi][ni][0], p[0][mi][ni][1], f.a[mi].x, f.b[ni].x);
          mma(p[1][mi][ni][0], p[1][mi][ni][1], f.a[mi].y, f.b[ni].y);
          mma(p[2][mi][ni][0], p[2][mi][ni][1], f.as[mi], f.bs[ni]);
        }
    }
    // visit every output element: fn(row, col_in_warp_tile, value); rows 0..15, cols 0..8NT-1
    template <typename Fn>
    __device__ __forceinline__ void each(int g, int t, Fn fn) const {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double p1 = p[0][mi][ni][e], p2 = p[1][mi][ni][e], p3 = p[2][mi][ni][e];
            fn(8 * mi + g, 8 * ni + 2 * t + e, make_double2(p1 - p2, p3 - p1 - p2));
          }
    }
  };
  // 4M product (4 real MMAs per complex MMA, no 3M sums): re += ar br + (-ai) bi,
  // im += ar bi + ai br.  Exact whenever the factor entries are 0 / +-1 / +-i (selection
  // blocks, identity pins), which the 3M combination is not.
  struct Acc4 {
    double p[2][2][NT][2];
    __device__ __forceinline__ void zero() {
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) p[q][mi][ni][0] = p[q][mi][ni][1] = 0.0;
    }
    __device__ __forceinline__ void mac(const Frags& f) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
          mma(p[0][mi][ni][0], p[0][mi][ni][1], f.a[mi].x, f.b[ni].x);
          mma(p[0][mi][ni][0], p[0][mi][ni][1], -f.a[mi].y, f.b[ni].y);
          mma(p[1][mi][ni][0], p[1][mi][ni][1], f.a[mi].x, f.b[ni].y);
          mma(p[1][mi][ni][0], p[1][mi][ni][1], f.a[mi].y, f.b[ni].x);
        }
    }
    template <typename Fn>
    __device__ __forceinline__ void each(int g, int t, Fn fn) const {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) fn(8 * mi + g, 8 * ni + 2 * t + e, make_double2(p[0][mi][ni][e], p[1][mi][ni][e]));
    }
  };
};

// ======================================================================================
// complex64 policy (leaf kernels): 3xTF32 mma.sync m16n8k8, fragments (lane = 4g + t):
//   A (16x8): a0 = A[g][t], a1 = A[g+8][t], a2 = A[g][t+4], a3 = A[g+8][t+4]
//   B (8x8):  b0 = B[t][g], b1 = B[t+4][g];   C (16x8): c0,c1 = C[g][2t+e], c2,c3 = C[g+8][2t+e]
// One k-step record (1 KB): [re | im][lane][a0..a3] floats (planar: each plane one lane-
// contiguous 16-byte load straight into the MMA's A registers).  Column-leaf records (B = X)
// use the natural K order; row-leaf records (B = a slab) the slab's K order kappa = t <-> row
// 2t, kappa = t + 4 <-> row 2t + 1 (see PolC64T for the complex64 half-slab layout).
// ======================================================================================
template <int NT_>
struct PolC64 {
  using E = float2;
  static constexpr int KS = 8;
  static constexpr int NT = NT_;
  __host__ __device__ static __forceinline__ int swz(int row) { return ((row & 1) << 3) | (((row >> 1) & 1) << 2); }
  __device__ static __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  __device__ static __forceinline__ void split(float x, uint32_t& hi, uint32_t& lo) {
    hi = __float_as_uint(x) & 0xffffe000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
  }
  struct Frags {
    uint32_t ah[3][4], al[3][4];  // (re, im, re + im) x fragment registers
    float2 b[NT][2];
  };
  // The product the fused kernels run on complex64: 3M on the 3xTF32 split.  (A 4M variant --
  // 2 splits per operand element, no sums, 12 instead of 9 HMMAs -- measured slower on B200:
  // 0.143 vs 0.129 ms per 3-level pass, tools/gpurun_scripts/gpu_r2q.sh.)
  struct Acc;
  using FFrags = Frags;
  using FAcc = Acc;
  __device__ static __forceinline__ void load_fa(Frags& f, const unsigned char* rec, int lane) { load_a(f, rec, lane); }
  __device__ static __forceinline__ int boff(int t, int g, int c0w, int ni) {
    return t * FAST_HC + ((c0w + 8 * ni + g) ^ swz(t));  // row t + 4 is +4*16 (same swizzle)
  }
  static constexpr bool LEAF_OPS = true;
  __device__ static __forceinline__ void load_a(Frags& f, const unsigned char* rec, int lane) {
    const float4* p = reinterpret_cast<const float4*>(rec);
    const float4 x = p[lane], y = p[32 + lane];  // re / im planes
    const float re[4] = {x.x, x.y, x.z, x.w}, im[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      split(re[e], f.ah[0][e], f.al[0][e]);
      split(im[e], f.ah[1][e], f.al[1][e]);
      split(re[e] + im[e], f.ah[2][e], f.al[2][e]);
    }
  }
  // leaf kernels: float offset of n-tile ni's B values in the two half slabs (PolC64T layout):
  // lane (g, t)'s own fragment, component (ni & 1) = column g / g + 8, rows 2t (+0) / 2t+1 (+2)
  __device__ static __forceinline__ int leaf_boff(int ni, int t, int g) {
    return 2 * (ni >> 1) * FAST_HSLAB + 4 * (4 * g + t) + (ni & 1);
  }
  template <class F>
  __device__ static __forceinline__ void load_b(F& f, const E* slab_k0, const int (&bo)[NT]) {
    const float* s = reinterpret_cast<const float*>(slab_k0);
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      f.b[ni][0] = make_float2(s[bo[ni]], s[bo[ni] + 128]);
      f.b[ni][1] = make_float2(s[bo[ni] + 2], s[bo[ni] + 130]);
    }
  }
  // half-slab element (r, c) in the PolC64T layout
  __device__ static __forceinline__ void slab_put(E* hs, int r, int c, E v) {
    const int kb = r >> 3, t = (r & 7) >> 1, lane = 4 * (c & 7) + t, comp = (c >> 3) + 2 * (r & 1);
    float* f = reinterpret_cast<float*>(hs) + kb * 256 + 4 * lane + comp;
    f[0] = v.x;
    f[128] = v.y;
  }
  template <class F>
  __device__ static __forceinline__ void load_b_col(F& f, const E* box, int ldb, int k0, int c0w, int g, int t,
                                                    bool cj) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const E* col = box + (c0w + 8 * ni + g) * ldb + k0 + t;
      float2 v0 = col[0], v1 = col[4];
      v0.y = conj_im(v0.y, cj);
      v1.y = conj_im(v1.y, cj);
      f.b[ni][0] = v0;
      f.b[ni][1] = v1;
    }
  }
  static constexpr int XROWS = 2;
  __device__ static __forceinline__ void x_rows(int64_t (&p)[XROWS], int64_t k0, int t) {
    p[0] = k0 + t;
    p[1] = k0 + t + 4;
  }
  template <class F>
  __device__ static __forceinline__ void load_b_x(F& f, const E* __restrict__ X, const int64_t (&rows)[XROWS],
                                                  int64_t ldx, int col0, int g, int nrhs, bool cj) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const int col = col0 + 8 * ni + g;
      float2 v0 = make_float2(0.f, 0.f), v1 = v0;
      if (col < nrhs) {
        v0 = __ldg(X + rows[0] + (int64_t)col * ldx);
        v1 = __ldg(X + rows[1] + (int64_t)col * ldx);
      }
      v0.y = conj_im(v0.y, cj);
      v1.y = conj_im(v1.y, cj);
      f.b[ni][0] = v0;
      f.b[ni][1] = v1;
    }
  }
  struct Acc {
    float p[3][NT][4];
    __device__ __forceinline__ void zero() {
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 4; ++e) p[q][ni][e] = 0.f;
    }
    __device__ __forceinline__ void mac(const Frags& f) {
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        uint32_t bh[3][2], bl[3][2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          split(f.b[ni][e].x, bh[0][e], bl[0][e]);
          split(f.b[ni][e].y, bh[1][e], bl[1][e]);
          split(f.b[ni][e].x + f.b[ni][e].y, bh[2][e], bl[2][e]);
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          mma(p[q][ni], f.ah[q], bl[q]);
          mma(p[q][ni], f.al[q], bh[q]);
          mma(p[q][ni], f.ah[q], bh[q]);
        }
      }
    }
    template <typename Fn>
    __device__ __forceinline__ void each(int g, int t, Fn fn) const {
#pragma unroll
      for (int ni = 0; ni < NT; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p1 = p[0][ni][e], p2 = p[1][ni][e], p3 = p[2][ni][e];
          fn(g + 8 * (e >> 1), 8 * ni + 2 * t + (e & 1), make_float2(p1 - p2, p3 - p1 - p2));
        }
    }
  };
  // 4M product on the 3xTF32 split (see PolC128::Acc4); uses f.ah/al[0] (re) and [1] (im) only
  struct Acc4 {
    float p[2][NT][4];
    __device__ __forceinline__ void zero() {
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 4; ++e) p[q][ni][e] = 0.f;
    }
    __device__ __forceinline__ void mac(const Frags& f) {
      uint32_t nh[4], nl[4];  // -ai (sign flip is exact on both split parts)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        nh[e] = f.ah[1][e] ^ 0x80000000u;
        nl[e] = f.al[1][e] ^ 0x80000000u;
      }
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        uint32_t bh[2][2], bl[2][2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          split(f.b[ni][e].x, bh[0][e], bl[0][e]);
          split(f.b[ni][e].y, bh[1][e], bl[1][e]);
        }
        // re += ar br - ai bi
        mma(p[0][ni], f.ah[0], bl[0]);
        mma(p[0][ni], f.al[0], bh[0]);
        mma(p[0][ni], f.ah[0], bh[0]);
        mma(p[0][ni], nh, bl[1]);
        mma(p[0][ni], nl, bh[1]);
        mma(p[0][ni], nh, bh[1]);
        // im += ar bi + ai br
        mma(p[1][ni], f.ah[0], bl[1]);
        mma(p[1][ni], f.al[0], bh[1]);
        mma(p[1][ni], f.ah[0], bh[1]);
        mma(p[1][ni], f.ah[1], bl[0]);
        mma(p[1][ni], f.al[1], bh[0]);
        mma(p[1][ni], f.ah[1], bh[0]);
      }
    }
    template <typename Fn>
    __device__ __forceinline__ void each(int g, int t, Fn fn) const {
#pragma unroll
      for (int ni = 0; ni < NT; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) fn(g + 8 * (e >> 1), 8 * ni + 2 * t + (e & 1), make_float2(p[0][ni][e], p[1][ni][e]));
    }
  };
};

// ======================================================================================
// complex64 window-pass policy, transposed product: out^T (16 columns x 8NT rows) =
// slab^T (16 columns x K) * F^T (K x 8NT rows), i.e. M = the 16 rhs columns of a half slab,
// N = output rows, K = input rows.  Both operands then load straight into their MMA registers
// (the slab's re / im planes: one lane-contiguous 16-byte load each; the factor: one per n-tile)
// and the accumulator tile of lane (g, t) is exactly the slab fragment lane (g, t) loads in the
// next op, so the epilogue is two 16-byte stores per n-tile.  (The row-major formulation needed
// ~50 % more instructions per HMMA: register moves to assemble re / im operand pairs from
// interleaved complex loads, tools/tf32_loop.cu: 168 vs 201 TF of HMMA issue.)
// K order inside a k-step: kappa = t <-> row 2t, kappa = t + 4 <-> row 2t + 1.
// complex64 half slab (HBM and shared memory, 2 KB): [kb = row / 8][re | im][lane][4] floats,
//   lane (g, t): (row 8kb + 2t, col g), (8kb + 2t, g + 8), (8kb + 2t + 1, g), (8kb + 2t + 1, g + 8).
// Factor record (1 KB per k-step and slot): [j = output row / 8][lane][re b0, re b1, im b0, im b1],
//   b0 = F(8j + g, 8ki + 2t), b1 = F(8j + g, 8ki + 2t + 1).
// ======================================================================================
template <int NT_>
struct PolC64T {
  using E = float2;
  static constexpr int KS = 8;
  static constexpr int NT = NT_;  // 8-row n-tiles per warp (NT = 1: the warp's c0w / 8 selects which)
  static constexpr bool LEAF_OPS = false;
  // a warp may run the two output slots that share an input pair in one k-loop, splitting the
  // slab fragment (A role) once for both (fast.cu, 4-level windows)
  static constexpr bool PAIR_SHARE = true;
  __device__ static __forceinline__ void split(float x, uint32_t& hi, uint32_t& lo) { PolC64<1>::split(x, hi, lo); }
  __device__ static __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    PolC64<1>::mma(c, a, b);
  }
  struct Frags {
    float4 sr, si;   // slab fragment (A role): re, im
    float4 f[NT];    // factor fragments (B role): re b0, re b1, im b0, im b1
  };
  struct Acc;
  using FFrags = Frags;
  using FAcc = Acc;
  __device__ static __forceinline__ int boff(int t, int g, int, int) { return 4 * g + t; }  // = lane
  __device__ static __forceinline__ int rec_off(int c0w) { return (c0w >> 3) * 512; }
  __device__ static __forceinline__ void load_fa(Frags& f, const unsigned char* rec, int lane) {
    const float4* p = reinterpret_cast<const float4*>(rec);
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) f.f[ni] = p[ni * 32 + lane];
  }
  __device__ static __forceinline__ void load_b(Frags& f, const E* slab_k0, const int (&bo)[NT]) {
    const float4* p = reinterpret_cast<const float4*>(slab_k0);
    f.sr = p[bo[0]];
    f.si = p[32 + bo[0]];
  }
  // the 3xTF32 split of a slab fragment (A role): (re, im, re + im) x (hi, lo)
  struct ASplit {
    uint32_t h[3][4], l[3][4];
  };
  __device__ static __forceinline__ void split_a(const Frags& f, ASplit& s) {
    const float re[4] = {f.sr.x, f.sr.y, f.sr.z, f.sr.w}, im[4] = {f.si.x, f.si.y, f.si.z, f.si.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      split(re[e], s.h[0][e], s.l[0][e]);
      split(im[e], s.h[1][e], s.l[1][e]);
      split(re[e] + im[e], s.h[2][e], s.l[2][e]);
    }
  }
  // the factor fragments of a second output slot (pair-shared ops, fast.cu PAIRW)
  __device__ static __forceinline__ void load_fa2(float4 (&g)[NT], const unsigned char* rec, int lane) {
    const float4* p = reinterpret_cast<const float4*>(rec);
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) g[ni] = p[ni * 32 + lane];
  }
  struct Acc {
    float p[3][NT][4];
    __device__ __forceinline__ void zero() {
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 4; ++e) p[q][ni][e] = 0.f;
    }
    // one k-step on an already split slab fragment with the factor fragments fb
    __device__ __forceinline__ void mac_split(const ASplit& s, const float4 (&fb)[NT]) {
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        uint32_t bh[3][2], bl[3][2];
        const float br[2] = {fb[ni].x, fb[ni].y}, bi[2] = {fb[ni].z, fb[ni].w};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          split(br[e], bh[0][e], bl[0][e]);
          split(bi[e], bh[1][e], bl[1][e]);
          split(br[e] + bi[e], bh[2][e], bl[2][e]);
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          mma(p[q][ni], s.h[q], bl[q]);
          mma(p[q][ni], s.l[q], bh[q]);
          mma(p[q][ni], s.h[q], bh[q]);
        }
      }
    }
    __device__ __forceinline__ void mac(const Frags& f) {
      ASplit s;
      split_a(f, s);
      mac_split(s, f.f);
    }
    // every output element: fn(row of the warp's n-tiles, column in the half, value)
    template <typename Fn>
    __device__ __forceinline__ void each(int g, int t, Fn fn) const {
#pragma unroll
      for (int ni = 0; ni < NT; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p1 = p[0][ni][e], p2 = p[1][ni][e], p3 = p[2][ni][e];
          fn(8 * ni + 2 * t + (e & 1), g + 8 * (e >> 1), make_float2(p1 - p2, p3 - p1 - p2));
        }
    }
  };
  // the warp's output rows 8 (c0w / 8 + ni) .. of the half slab: two 16-byte stores per n-tile
  __device__ static __forceinline__ void store_slab(const Acc& acc, E* hs, int c0w, int, int, int lane) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      float re[4], im[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p1 = acc.p[0][ni][e], p2 = acc.p[1][ni][e], p3 = acc.p[2][ni][e];
        re[e] = p1 - p2;
        im[e] = p3 - p1 - p2;
      }
      float4* d = reinterpret_cast<float4*>(hs + ((c0w >> 3) + ni) * 128);
      d[lane] = make_float4(re[0], re[2], re[1], re[3]);
      d[32 + lane] = make_float4(im[0], im[2], im[1], im[3]);
    }
  }
};

}  // namespace bfa
