// Fused window-pass kernels (see fast.cuh for windows, slots and the operand stream).
//
// Persistent, warp-specialised CTA (one per SM).  The producer warp streams, per work item
// (window, rhs tile):
//   * the window's input slabs (one 1-D TMA bulk copy per slot) into one of two window
//     buffers, one item ahead of the consumers;
//   * every op's factor stream, page by page, into a ring of 8 KB pages (1-D TMA bulk copies,
//     mbarrier complete_tx), as far ahead as the ring allows;
//   * for the X-reading leaf op, the X rows of each (k-step, slot) by 2-D TMA tensor loads.
// The 8 consumer warps walk the pages in the same order, run the block products on the tensor
// pipe and release each page right after its k-steps, so HBM streaming overlaps the MMAs at
// page granularity.  For d = 3 each warp owns one slot (16 x 32 output); for d = 2 / 1 two /
// four warps share a slot and split its 32 columns (template NT = 8-column tiles per warp).
//
// complex128 (PolC128): mma.sync.m8n8k4.f64 ("DMMA") with the 3-multiplication product
//     P1 = Ar Br,  P2 = Ai Bi,  P3 = (Ar + Ai)(Br + Bi);   Re = P1 - P2,  Im = P3 - P1 - P2.
// (DMMA and DFMA share one FP64 budget on B200 -- profiles/r01_pipes2.txt -- so fewer
// multiplications is the lever.)
// complex64 (PolC64): the same 3M product on mma.sync.m16n8k8.tf32 with the 3xTF32 split
// x = hi + lo, a*b ~ ah*bh + ah*bl + al*bh: FP32-level accuracy at tensor-pipe rate (plain TF32,
// ~1e-3, would fail the 1e-5 bar -- SURVEY 7.3).
//
// Slab layout (window buffers and HBM ping-pong buffers): 16 rows x 32 complex, element
// (row, col) at  row * 32 + (col ^ swz(row)); swz is chosen per element size so that MMA
// C-fragment stores and B-fragment loads are shared-memory bank-conflict free.
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait for the phase of `bar` with the given parity.  A watchdog turns a protocol deadlock into
// a trapped launch (BF_ERR_CUDA on the next call) instead of a hung device.
__device__ __noinline__ void mbar_wait_slow(uint64_t* bar, uint32_t parity, int tag) {
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

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(FAST_NCONS * 32) : "memory"); }

// window slot -> canonical block index at window level s
__device__ __forceinline__ int64_t canon(const FastPass& P, int64_t a, int64_t b, int s, int slot) {
  const int ds = P.d - s;
  const int64_t tau = (a << s) + (slot >> ds);
  const int64_t nu = (b << ds) + (slot & ((1 << ds) - 1));
  return (tau << (P.L - (P.l0 + s))) + nu;
}

// ======================================================================================
// complex128 policy: DMMA m8n8k4, fragments (lane = 4g + t):
//   A (8x4): A[g][t];  B (4x8): B[t][g];  C (8x8): C[g][2t+e].
// One k-step record (1 KB): [mi][lane] double2 for the 16 x 4 block.
// With KS = 4 the slab swizzle of row k0 + t depends only on t, so every B-fragment address is
// slab + k0 * 32 + (a lane constant).
// ======================================================================================
template <int NT_>
struct PolC128 {
  using E = double2;
  static constexpr int KS = 4;
  static constexpr int NT = NT_;
  static constexpr int NPAGES = 6;   // 16 KB pages: 2 x 64 KB windows (the 2nd = X staging) + 96 KB ring
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
  // lane-constant element offset of B row t, n-tile ni (k0 = 0)
  __device__ static __forceinline__ int boff(int t, int g, int c0w, int ni) {
    return t * 32 + ((c0w + 8 * ni + g) ^ swz(t));
  }
  __device__ static __forceinline__ void load_a(Frags& f, const unsigned char* rec, int lane) {
    const E* p = reinterpret_cast<const E*>(rec);
    f.a[0] = p[lane];
    f.a[1] = p[32 + lane];
    f.as[0] = f.a[0].x + f.a[0].y;
    f.as[1] = f.a[1].x + f.a[1].y;
  }
  __device__ static __forceinline__ void load_b(Frags& f, const E* slab_k0, const int (&bo)[NT]) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      f.b[ni] = slab_k0[bo[ni]];
      f.bs[ni] = f.b[ni].x + f.b[ni].y;
    }
  }
  // from an X box in shared memory (TMA SWIZZLE_64B; box = 4 rows x 32 columns, 64 B per column)
  __device__ static __forceinline__ void load_b_box(Frags& f, const unsigned char* box, int c0, int g, int t, bool cj) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const int c = c0 + 8 * ni + g;
      E v = *reinterpret_cast<const E*>(box + c * 64 + ((t ^ ((c >> 1) & 3)) << 4));
      if (cj) v.y = -v.y;
      f.b[ni] = v;
      f.bs[ni] = v.x + v.y;
    }
  }
  static constexpr int XROWS = 1;
  __device__ static __forceinline__ void x_rows(int64_t (&p)[XROWS], int64_t k0, int t) { p[0] = k0 + t; }
  __device__ static __forceinline__ void load_b_x(Frags& f, const E* __restrict__ X, const int64_t (&rows)[XROWS],
                                                  int64_t ldx, int col0, int g, int nrhs, bool cj) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const int col = col0 + 8 * ni + g;
      E v = col < nrhs ? __ldg(X + rows[0] + (int64_t)col * ldx) : make_double2(0.0, 0.0);
      if (cj) v.y = -v.y;
      f.b[ni] = v;
      f.bs[ni] = v.x + v.y;
    }
  }
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
    // half PART of one k-step: row group mi = PART (3 x NT DMMAs)
    template <int PART>
    __device__ __forceinline__ void part(const Frags& f) {
      constexpr int mi = PART;
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        mma(p[0][mi][ni][0], p[0][mi][ni][1], f.a[mi].x, f.b[ni].x);
        mma(p[1][mi][ni][0], p[1][mi][ni][1], f.a[mi].y, f.b[ni].y);
        mma(p[2][mi][ni][0], p[2][mi][ni][1], f.as[mi], f.bs[ni]);
      }
    }
    // visit every output element: f(row, col_in_warp_tile, value); rows 0..15, cols 0..8NT-1
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
};

// ======================================================================================
// complex64 policy: 3xTF32 mma.sync m16n8k8, fragments (lane = 4g + t):
//   A (16x8): a0 = A[g][t], a1 = A[g+8][t], a2 = A[g][t+4], a3 = A[g+8][t+4]
//   B (8x8):  b0 = B[t][g], b1 = B[t+4][g];   C (16x8): c0,c1 = C[g][2t+e], c2,c3 = C[g+8][2t+e]
// One k-step record (1 KB): [lane][4] float2 for the 16 x 8 block.  The A operand is split
// into TF32 hi / lo parts once per k-step (load_a); B per n-tile inside part().
// ======================================================================================
template <int NT_>
struct PolC64 {
  using E = float2;
  static constexpr int KS = 8;
  static constexpr int NT = NT_;
  static constexpr int NPAGES = 8;   // 32 KB window + 64 KB window / X staging + 128 KB ring
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
  __device__ static __forceinline__ int boff(int t, int g, int c0w, int ni) {
    return t * 32 + ((c0w + 8 * ni + g) ^ swz(t));  // row t + 4 is +128 (same swizzle)
  }
  __device__ static __forceinline__ void load_a(Frags& f, const unsigned char* rec, int lane) {
    const float4* p = reinterpret_cast<const float4*>(rec) + 2 * lane;
    const float4 x = p[0], y = p[1];
    const float2 v[4] = {make_float2(x.x, x.y), make_float2(x.z, x.w), make_float2(y.x, y.y), make_float2(y.z, y.w)};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      split(v[e].x, f.ah[0][e], f.al[0][e]);
      split(v[e].y, f.ah[1][e], f.al[1][e]);
      split(v[e].x + v[e].y, f.ah[2][e], f.al[2][e]);
    }
  }
  __device__ static __forceinline__ void load_b(Frags& f, const E* slab_k0, const int (&bo)[NT]) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      f.b[ni][0] = slab_k0[bo[ni]];
      f.b[ni][1] = slab_k0[bo[ni] + 128];
    }
  }
  // X box: 8 rows x 32 columns, 64 B per column, TMA SWIZZLE_64B
  __device__ static __forceinline__ void load_b_box(Frags& f, const unsigned char* box, int c0, int g, int t, bool cj) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const int c = c0 + 8 * ni + g;
      const int sw = (c >> 1) & 3;
      const unsigned char* col = box + c * 64;
      float2 v0 = *reinterpret_cast<const E*>(col + (((t >> 1) ^ sw) << 4) + ((t & 1) << 3));
      float2 v1 = *reinterpret_cast<const E*>(col + ((((t + 4) >> 1) ^ sw) << 4) + ((t & 1) << 3));
      if (cj) {
        v0.y = -v0.y;
        v1.y = -v1.y;
      }
      f.b[ni][0] = v0;
      f.b[ni][1] = v1;
    }
  }
  static constexpr int XROWS = 2;
  __device__ static __forceinline__ void x_rows(int64_t (&p)[XROWS], int64_t k0, int t) {
    p[0] = k0 + t;
    p[1] = k0 + t + 4;
  }
  __device__ static __forceinline__ void load_b_x(Frags& f, const E* __restrict__ X, const int64_t (&rows)[XROWS],
                                                  int64_t ldx, int col0, int g, int nrhs, bool cj) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const int col = col0 + 8 * ni + g;
      float2 v0 = make_float2(0.f, 0.f), v1 = v0;
      if (col < nrhs) {
        v0 = __ldg(X + rows[0] + (int64_t)col * ldx);
        v1 = __ldg(X + rows[1] + (int64_t)col * ldx);
      }
      if (cj) {
        v0.y = -v0.y;
        v1.y = -v1.y;
      }
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
    // PART 0 / 1: the first / second half of the n-tiles (all of them in part 0 when NT = 1)
    template <int PART>
    __device__ __forceinline__ void part(const Frags& f) {
      constexpr int lo = NT == 1 ? (PART == 0 ? 0 : 1) : PART * (NT / 2);
      constexpr int hi = NT == 1 ? 1 : (PART + 1) * (NT / 2);
#pragma unroll
      for (int ni = lo; ni < hi; ++ni) {
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
};


// cp.async (16 B, L2 only) into shared memory, completion tracked by an mbarrier arrival
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_zero(void* dst, const void* any) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;\n" ::"r"(smem_u32(dst)), "l"(any) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// slab index of block (tau, nu) at level l in the HBM ping-pong buffers: tau-major for op N,
// nu-major for op C / T, so that the S slabs a window reads at its input level are contiguous
// (one bulk copy) in both directions.
__device__ __forceinline__ int64_t slab_index(const FastPass& P, int64_t a, int64_t b, int s, int slot) {
  const int ds = P.d - s, l = P.l0 + s;
  const int64_t tau = (a << s) + (slot >> ds);
  const int64_t nu = (b << ds) + (slot & ((1 << ds) - 1));
  return P.numaj ? (nu << l) + tau : (tau << (P.L - l)) + nu;
}

// ======================================================================================
// The persistent pass kernel: 8 consumer warps + 1 producer warp.
//
// Producer warp, per work item (window, 32-column tile): the window's S input slabs (one bulk
// copy, one item ahead, into window buffer i & 1); then per op and per group of SPP k-steps one
// 16 KB A page (bulk copy; 16 KB copies stream at ~7 TB/s chip-wide where 8 KB copies stall at
// ~3.8 -- tools/tma_stream.cu) and, for the X-reading leaf op, the X rows of those k-steps,
// gathered by all 32 lanes with 16-byte cp.async into swizzled column-major boxes.  Every ring
// page has one barrier with 32 arrivals (bulk page: lane 0's expect_tx + 31 plain arrivals; X
// page: one cp.async completion arrival per lane).
// Consumers: a pair op reads two slabs of other slots -> barrier before the in-place write and
// after it; everything else is warp-local.  (9 warps cap threads at 168 registers, so the k-step
// is load-then-MMA, which tools/mma_loop.cu measures at 94 % of the DMMA peak.)
// ======================================================================================
template <class Pol>
__global__ void __launch_bounds__(FAST_THREADS, 1) k_bf_pass(const __grid_constant__ FastArgs A) {
  using E = typename Pol::E;
  constexpr int NT = Pol::NT;
  constexpr int S = 2 * NT;                          // slots of the window (2^d)
  constexpr int WPS = FAST_NCONS / S;                // warps per slot
  constexpr int SPP = FAST_PAGE / (S * FAST_FRAG);   // k-steps per A page
  constexpr int NP = Pol::NPAGES;
  constexpr int WIN = (1 << FAST_DMAX) * FAST_SLAB;  // window buffer (elements)
  constexpr int KPS = FAST_RANK / Pol::KS;           // k-steps per 16-row slab / U row group
  constexpr int XST = FAST_XSTAGES;                  // X staging depth (k-steps) of the leaf op
  static_assert(WPS * NT * 8 == FAST_NB, "warp tiling must cover the slab columns");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  E* winbuf = reinterpret_cast<E*>(smem_raw);  // window 0, then window 1 / X staging
  unsigned char* ring = smem_raw + fast_win_region<E>();
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + NP * FAST_PAGE);
  uint64_t* winF = bars;
  uint64_t* winE = bars + 2;
  uint64_t* full = bars + 4;
  uint64_t* empty = bars + 4 + NP;

  const FastPass& P = A.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nitems = P.nwin * ((A.nrhs + FAST_NB - 1) / FAST_NB);
  const int nwin_log = P.L - P.d;
  const int64_t bmask = (int64_t(1) << P.bbits) - 1;
  const bool xp = P.xpage != 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&winF[i], 1);
      mbar_init(&winE[i], 1);
    }
    for (int i = 0; i < NP; ++i) {
      mbar_init(&full[i], 32);
      mbar_init(&empty[i], FAST_NCONS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int diag = A.diag;
  if (warp == FAST_NCONS) {
    // ---------------------------------------------------------------- producer warp
    if (diag & 1) {
      __syncthreads();
      return;
    }
    const unsigned char* Fb = static_cast<const unsigned char*>(A.F) + P.fbase;
    const E* Sin = static_cast<const E*>(A.Sin);
    int slot = 0;
    uint32_t ph = 0;
    int64_t issued = 0;
    auto acquire = [&]() {  // wait until the next ring slot is free
      if (lane == 0 && issued >= NP) mbar_wait(&empty[slot], ph ^ 1, 1);
      __syncwarp();
    };
    auto advance = [&]() {
      ++issued;
      if (++slot == NP) {
        slot = 0;
        ph ^= 1;
      }
    };
    int i = 0;
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++i) {
      const int64_t w = item & ((int64_t(1) << nwin_log) - 1), jt = item >> nwin_log;
      const int64_t a = w >> P.bbits, b = w & bmask;
      if (P.in_s >= 0 && lane == 0) {  // (passes without a window input use buffer 0 only)
        const int wb = i & 1;
        if (i >= 2) mbar_wait(&winE[wb], ((i - 2) >> 1) & 1, 2);
        const uint32_t bytes = (uint32_t)(S * FAST_SLAB * sizeof(E));
        mbar_expect_tx(&winF[wb], bytes);
        bulk_g2s(winbuf + wb * WIN, Sin + (jt * A.nlev + slab_index(P, a, b, P.in_s, 0)) * FAST_SLAB, bytes, &winF[wb]);
      }
      const unsigned char* Fw = Fb + w * P.win_bytes;
      for (int q = 0; q < P.nops; ++q) {
        const FastOp& op = P.ops[q];
        for (int s0 = 0; s0 < op.nsteps; s0 += SPP) {
          const int nst = min(SPP, op.nsteps - s0);
          // A page: one bulk copy
          acquire();
          if (lane == 0) {
            const uint32_t ab = (uint32_t)(nst * S * FAST_FRAG);
            mbar_expect_tx(&full[slot], ab);
            bulk_g2s(ring + (size_t)slot * FAST_PAGE, Fw + op.off + (int64_t)s0 * S * FAST_FRAG, ab, &full[slot]);
          } else {
            mbar_arrive(&full[slot]);
          }
          advance();
        }
      }
    }
    // stay resident until the consumers are done (an exited warp must not take part in their
    // named-barrier accounting), and until this warp's async copies have landed
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    __syncthreads();
    return;
  }

  // ------------------------------------------------------------------ consumers
  const int g = lane >> 2, t = lane & 3;
  const int o = warp / WPS;
  const int c0w = 8 * NT * (warp % WPS);  // first column (inside the 32-column tile) of this warp
  int bo[NT];                             // lane-constant B-fragment offsets inside a slab
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) bo[ni] = Pol::boff(t, g, c0w, ni);
  E* __restrict__ Sout = static_cast<E*>(A.Sout);
  const bool cj = A.conj_io != 0;
  int slot = 0;
  uint32_t ph = 0;
  auto wait_pg = [&](int sl, uint32_t p) {
    if (!(diag & 1)) mbar_wait(&full[sl], p, 4);
  };
  auto next_pg = [&]() {
    if (lane == 0 && !(diag & 1)) mbar_arrive(&empty[slot]);
    if (++slot == NP) {
      slot = 0;
      ph ^= 1;
    }
  };
  int i = 0;
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++i) {
    const int64_t w = item & ((int64_t(1) << nwin_log) - 1), jt = item >> nwin_log;
    const int64_t a = w >> P.bbits, b = w & bmask;
    const int wb = P.in_s >= 0 ? (i & 1) : 0;  // no window input: buffer 1 holds the X staging
    E* win = winbuf + wb * WIN;
    const int j0 = (int)jt * FAST_NB + c0w;  // first rhs column of this warp
    if (P.in_s >= 0 && !(diag & 1)) mbar_wait(&winF[wb], (i >> 1) & 1, 3);
    for (int q = 0; q < P.nops; ++q) {
      const FastOp op = P.ops[q];
      const bool last = q == P.nops - 1;
      typename Pol::Acc acc;
      acc.zero();
      const E* own = win + o * FAST_SLAB;
      if (op.kind == FK_PAIR_DOWN || op.kind == FK_PAIR_UP || op.kind == FK_DIAG) {
        const E* sp0 = own;
        const E* sp1 = own;
        const int ds = P.d - op.s;
        if (op.kind == FK_PAIR_DOWN) {  // output level s+1 from input level s
          const int tp = o >> (ds - 1), up = o & ((1 << (ds - 1)) - 1);
          sp0 = win + (((tp >> 1) << ds) + 2 * up) * FAST_SLAB;
          sp1 = sp0 + FAST_SLAB;
        } else if (op.kind == FK_PAIR_UP) {  // output level s from input level s+1
          const int tt = o >> ds, u = o & ((1 << ds) - 1);
          sp0 = win + (((2 * tt) << (ds - 1)) + (u >> 1)) * FAST_SLAB;
          sp1 = win + (((2 * tt + 1) << (ds - 1)) + (u >> 1)) * FAST_SLAB;
        }
        const int n = op.nsteps;
#pragma unroll 1
        for (int s0 = 0; s0 < n; s0 += SPP) {
          wait_pg(slot, ph);
          const unsigned char* pg = ring + (size_t)slot * FAST_PAGE;
#pragma unroll
          for (int st = 0; st < SPP; ++st) {
            const int s = s0 + st;
            if (s < n) {
              typename Pol::Frags f;
              Pol::load_a(f, pg + (st * S + o) * FAST_FRAG, lane);
              Pol::load_b(f, (s < KPS ? sp0 : sp1) + (s & (KPS - 1)) * Pol::KS * 32, bo);
              acc.template part<0>(f);
              acc.template part<1>(f);
            }
          }
          __syncwarp();
          next_pg();
        }
      } else if (op.kind == FK_LEAF_IN) {
        // B operand = X rows of this slot's leaf.  Each warp prefetches its own rows XST k-steps
        // ahead with 16-byte cp.async (lane = column) into a private staging ring in the
        // otherwise unused second window buffer: box = KS rows x 32 columns, 64 B per column,
        // 16-byte units swizzled by (column >> 1) & 3.
        const int64_t row0 = canon(P, a, b, op.s, o) * op.leaf;
        const int n = op.nsteps;
        unsigned char* xst = reinterpret_cast<unsigned char*>(winbuf + WIN) + warp * XST * FAST_XBOX;
        const E* X = static_cast<const E*>(A.X);
        const int colg = (int)jt * FAST_NB + lane;  // this lane's column
        const int sw = (lane >> 1) & 3;
        const int64_t base = A.xperm && xp ? A.xperm[row0] : row0;  // contiguous leaf: user row of row0
        auto fetch = [&](int s) {  // issue the copies of k-step s (always commits one group)
          if (s < n) {
            unsigned char* box = xst + (s % XST) * FAST_XBOX + lane * 64;
            if (colg < A.nrhs) {
              if (xp) {
                const unsigned char* src =
                    reinterpret_cast<const unsigned char*>(X + base + (int64_t)s * Pol::KS + (int64_t)colg * A.ldx);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  if (A.xalign16) cp_async16(box + ((u ^ sw) << 4), src + u * 16);
                  else {
                    cp_async8(box + ((u ^ sw) << 4), src + u * 16);
                    cp_async8(box + ((u ^ sw) << 4) + 8, src + u * 16 + 8);
                  }
                }
              } else {  // permuted leaf: one user row per element
                constexpr int PER = 16 / (int)sizeof(E);  // elements per 16-byte unit
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                  for (int e = 0; e < PER; ++e) {
                    const int64_t row = A.xperm[row0 + (int64_t)s * Pol::KS + u * PER + e];
                    const unsigned char* src = reinterpret_cast<const unsigned char*>(X + row + (int64_t)colg * A.ldx);
                    if (PER == 1) cp_async16(box + ((u ^ sw) << 4), src);
                    else cp_async8(box + ((u ^ sw) << 4) + e * 8, src);
                  }
              }
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u) cp_async16_zero(box + (u << 4), X);
            }
          }
          asm volatile("cp.async.commit_group;\n" ::: "memory");
        };
#pragma unroll
        for (int k = 0; k < XST - 1; ++k) fetch(k);
#pragma unroll 1
        for (int s0 = 0; s0 < n; s0 += SPP) {
          wait_pg(slot, ph);
          const unsigned char* pg = ring + (size_t)slot * FAST_PAGE;
#pragma unroll
          for (int st = 0; st < SPP; ++st) {
            const int s = s0 + st;
            if (s < n) {
              fetch(s + XST - 1);
              asm volatile("cp.async.wait_group %0;\n" ::"n"(XST - 1) : "memory");
              __syncwarp();
              typename Pol::Frags f;
              Pol::load_a(f, pg + (st * S + o) * FAST_FRAG, lane);
              Pol::load_b_box(f, xst + (s % XST) * FAST_XBOX, c0w, g, t, cj);
              acc.template part<0>(f);
              acc.template part<1>(f);
              __syncwarp();  // the box is reused XST steps later
            }
          }
          __syncwarp();
          next_pg();
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
      } else {  // FK_LEAF_OUT: U_tau y (op N) / conj(Vt_nu)^T y (op C) into Y, 16 rows at a time
        E* __restrict__ Y = static_cast<E*>(A.Y);
        const int64_t row0 = canon(P, a, b, op.s, o) * op.leaf;
        const int n = op.nsteps;
#pragma unroll 1
        for (int s0 = 0; s0 < n; s0 += SPP) {
          wait_pg(slot, ph);
          const unsigned char* pg = ring + (size_t)slot * FAST_PAGE;
#pragma unroll
          for (int st = 0; st < SPP; ++st) {
            const int s = s0 + st;
            if (s < n) {
              typename Pol::Frags f;
              Pol::load_a(f, pg + (st * S + o) * FAST_FRAG, lane);
              Pol::load_b(f, own + (s & (KPS - 1)) * Pol::KS * 32, bo);
              acc.template part<0>(f);
              acc.template part<1>(f);
              if ((s & (KPS - 1)) == KPS - 1) {
                const int64_t rb = row0 + (s / KPS) * 16;
                acc.each(g, t, [&](int r, int c, E v) {
                  const int col = j0 + c;
                  if (col < A.nrhs) {
                    const int64_t pr = rb + r;
                    const int64_t row = A.yperm ? A.yperm[pr] : pr;
                    if (cj) v.y = -v.y;
                    Y[row + (int64_t)col * A.ldy] = v;
                  }
                });
                acc.zero();
              }
            }
          }
          __syncwarp();
          next_pg();
        }
        continue;  // written to Y
      }
      // in-place update: a pair op reads other slots' slabs, so all warps must be done reading
      if (op.kind == FK_PAIR_DOWN || op.kind == FK_PAIR_UP) consumer_sync();
      else __syncwarp();
      if (last && P.out_s >= 0 && !(diag & 2)) {
        E* dst = Sout + (jt * A.nlev + slab_index(P, a, b, P.out_s, o)) * FAST_SLAB;
        acc.each(g, t, [&](int r, int c, E v) { dst[r * 32 + ((c0w + c) ^ Pol::swz(r))] = v; });
      } else {
        E* dst = win + o * FAST_SLAB;
        acc.each(g, t, [&](int r, int c, E v) { dst[r * 32 + ((c0w + c) ^ Pol::swz(r))] = v; });
      }
      // the next op reads other slots only if it is a pair op
      if (!last) {
        const int nk = P.ops[q + 1].kind;
        if (nk == FK_PAIR_DOWN || nk == FK_PAIR_UP) consumer_sync();
        else __syncwarp();
      }
    }
    consumer_sync();  // every warp is done with this window buffer
    if (threadIdx.x == 0 && !(diag & 1)) mbar_arrive(&winE[wb]);
  }
  __syncthreads();  // joins the producer warp
}

const char* fast_kernel_name(int dtype) { return dtype == BF_C128 ? "k_bf_pass<c128>" : "k_bf_pass<c64>"; }

template <class Pol>
static size_t smem_of() {
  constexpr int NP = Pol::NPAGES;
  return fast_win_region<typename Pol::E>() + (size_t)NP * FAST_PAGE + (4 + 2 * NP) * 8;
}

size_t fast_smem_bytes(int dtype) { return dtype == BF_C128 ? smem_of<PolC128<4>>() : smem_of<PolC64<4>>(); }

template <class Pol>
static void launch_one(const FastArgs& a, unsigned grid, cudaStream_t st) {
  static bool attr = false;
  const size_t smem = smem_of<Pol>();
  if (!attr) {
    cudaFuncSetAttribute(k_bf_pass<Pol>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_bf_pass<Pol><<<grid, FAST_THREADS, smem, st>>>(a);
}

void launch_fast_pass(int dtype, const FastArgs& a, cudaStream_t st) {
  static int nsm = 0;
  if (nsm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t items = a.p.nwin * ((a.nrhs + FAST_NB - 1) / FAST_NB);
  const unsigned grid = (unsigned)(items < nsm ? items : nsm);
  const int d = a.p.d;
  if (dtype == BF_C128) {
    if (d == 3) launch_one<PolC128<4>>(a, grid, st);
    else if (d == 2) launch_one<PolC128<2>>(a, grid, st);
    else launch_one<PolC128<1>>(a, grid, st);
  } else {
    if (d == 3) launch_one<PolC64<4>>(a, grid, st);
    else if (d == 2) launch_one<PolC64<2>>(a, grid, st);
    else launch_one<PolC64<1>>(a, grid, st);
  }
}

}  // namespace bfa
