// Fused window-pass kernels (see fast.cuh for the window / slot definitions).
//
// Persistent, warp-specialised CTA (one per SM): a producer warp streams, with TMA 1-D bulk
// copies (cp.async.bulk + mbarrier complete_tx), each work item's window input slabs into one
// of two window buffers and the item's fragment-ordered factor data into a ring of 16 KB
// chunks; 16 consumer warps run the block products on tensor cores and hand buffers back
// through mbarriers, so HBM streaming of item i+1 overlaps the math of item i.
//
// complex128 (PolC128): mma.sync.m8n8k4.f64 ("DMMA") with the 3-multiplication complex product
//     P1 = Ar Br,  P2 = Ai Bi,  P3 = (Ar + Ai)(Br + Bi);   Re = P1 - P2,  Im = P3 - P1 - P2
// (3 real MMAs per complex MMA instead of 4; on B200 DMMA and DFMA have the same measured peak,
// profiles/pipe_peaks.json, so fewer multiplications is the lever).
// complex64 (PolC64): the same 3M product on mma.sync.m16n8k8.tf32 with the 3xTF32 split
// x = hi + lo (hi = x with the low 13 mantissa bits cleared), a*b ~ ah*bh + ah*bl + al*bh:
// FP32-level accuracy (~1e-6 relative) at tensor-core rate (plain TF32 would give ~1e-3,
// failing the 1e-5 bar -- SURVEY 7.3).
//
// Slab layout (shared memory and the HBM ping-pong buffers): 16 rows x 32 complex; the
// element (row, col) lives at  row * 32 + (col ^ swz(row)).  swz is chosen per element size
// so that MMA C-fragment stores and B-fragment loads are shared-memory bank-conflict free.
#include <cstdio>

#include "fast.cuh"

#ifndef BF_C128_3M
#define BF_C128_3M 1
#endif
#ifndef BF_USE_RING
#define BF_USE_RING 1
#endif

namespace bfa {

// ---- mbarrier / bulk-copy (TMA 1-D) helpers --------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
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
// Wait for the phase of `bar` with the given parity to complete.  A watchdog turns a
// protocol deadlock into a trapped launch (BF_ERR_CUDA) instead of a hung device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, int tag = 0, long long info = 0) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  const long long lim = tag == 2 ? (1ll << 35) : (1ll << 33);  // producer waits longest
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > lim) {
      printf("bfapply: mbarrier watchdog block %d thread %d tag %d parity %u info %lld\n", blockIdx.x, threadIdx.x, tag,
             parity, info);
      __trap();
    }
  }
}
// Ring ops (transfer and centre stages) stream their operands through the factor ring.  Every
// ring op has at most FAST_NBUF chunks, so a consumer never waits on a ring phase more than one
// ahead of the barrier (an mbarrier parity wait aliases beyond that).  Leaf ops read their
// operand directly with coalesced loads.
__device__ __forceinline__ bool ring_op(int kind) { return BF_USE_RING && kind != FK_LEAF_IN && kind != FK_LEAF_OUT; }

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
// A data per 16-row x 4-col k-step: [mi][lane] (64 entries).
// ======================================================================================
struct PolC128 {
  using E = double2;
  static constexpr int KS = 4;
  static constexpr int A_KSTEP = 64;
  static constexpr int NT = 4;  // n-tiles (8 columns each) per warp: the whole slab
  __device__ static __forceinline__ int swz(int row) { return ((row & 3) << 1) | (row & 1); }
  __device__ static __forceinline__ void mma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
  }
  struct AFrag {
    double2 v[2];
  };
  struct BFrag {
    double2 v;
  };
  __device__ static __forceinline__ void load_a(AFrag& f, const E* Ak, int lane) {
    f.v[0] = Ak[lane];
    f.v[1] = Ak[32 + lane];
  }
  __device__ static __forceinline__ void load_a_g(AFrag& f, const E* __restrict__ Ak, int lane) {
    f.v[0] = __ldg(Ak + lane);
    f.v[1] = __ldg(Ak + 32 + lane);
  }
  // B fragment for the n-tile at column c0 of rows k0.. of a slab in shared memory
  __device__ static __forceinline__ void load_b(BFrag& f, const E* slab, int k0, int c0, int g, int t) {
    const int row = k0 + t;
    f.v = slab[row * 32 + ((c0 + g) ^ swz(row))];
  }
  __device__ static __forceinline__ void load_b_x(BFrag& f, const E* __restrict__ X, int64_t row, int64_t ldx, int col,
                                                  int nrhs, bool cj) {
    f.v = col < nrhs ? __ldg(X + row + (int64_t)col * ldx) : make_double2(0.0, 0.0);
    if (cj) f.v.y = -f.v.y;
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
#if BF_C128_3M
    // 3M: P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi)
    __device__ __forceinline__ void step(const AFrag& a, const BFrag (&b)[NT]) {
      double bs[NT];
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) bs[ni] = b[ni].v.x + b[ni].v.y;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const double as = a.v[mi].x + a.v[mi].y;
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
          mma(p[0][mi][ni][0], p[0][mi][ni][1], a.v[mi].x, b[ni].v.x);
          mma(p[1][mi][ni][0], p[1][mi][ni][1], a.v[mi].y, b[ni].v.y);
          mma(p[2][mi][ni][0], p[2][mi][ni][1], as, bs[ni]);
        }
      }
    }
#else
    // 4M without in-loop FP64 adds: P1 = Ar Br, P2 = Ai Bi, P3 = Ar Bi + Ai Br.  On B200 the
    // DADDs that 3M needs share the FP64 pipe with DMMA and stall its issue stream (ncu:
    // math-pipe-throttle at the DADDs, DMMA pipe ~50% active), so 4 DMMAs per complex
    // product run faster than 3 DMMAs + 2 dependent DADDs.
    __device__ __forceinline__ void step(const AFrag& a, const BFrag (&b)[NT]) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
          mma(p[0][mi][ni][0], p[0][mi][ni][1], a.v[mi].x, b[ni].v.x);
          mma(p[1][mi][ni][0], p[1][mi][ni][1], a.v[mi].y, b[ni].v.y);
          mma(p[2][mi][ni][0], p[2][mi][ni][1], a.v[mi].x, b[ni].v.y);
          mma(p[2][mi][ni][0], p[2][mi][ni][1], a.v[mi].y, b[ni].v.x);
        }
    }
#endif
    // visit every output element: f(row, col_in_warp_tile, value); rows 0..15, cols 0..8NT-1
    template <typename Fn>
    __device__ __forceinline__ void each(int g, int t, Fn f) const {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double p1 = p[0][mi][ni][e], p2 = p[1][mi][ni][e], p3 = p[2][mi][ni][e];
#if BF_C128_3M
            f(8 * mi + g, 8 * ni + 2 * t + e, make_double2(p1 - p2, p3 - p1 - p2));
#else
            f(8 * mi + g, 8 * ni + 2 * t + e, make_double2(p1 - p2, p3));
#endif
          }
    }
  };
};

// ======================================================================================
// complex64 policy: 3xTF32 mma.sync m16n8k8, fragments (lane = 4g + t):
//   A (16x8): a0 = A[g][t], a1 = A[g+8][t], a2 = A[g][t+4], a3 = A[g+8][t+4]
//   B (8x8):  b0 = B[t][g], b1 = B[t+4][g];   C (16x8): c0,c1 = C[g][2t+e], c2,c3 = C[g+8][2t+e]
// A data per 16-row x 8-col k-step: [lane][4] (128 entries).
// ======================================================================================
struct PolC64 {
  using E = float2;
  static constexpr int KS = 8;
  static constexpr int A_KSTEP = 128;
  static constexpr int NT = 4;
  __device__ static __forceinline__ int swz(int row) { return ((row & 1) << 3) | (((row >> 1) & 1) << 2); }
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
  struct AFrag {
    float2 v[4];
  };
  struct BFrag {
    float2 v[2];
  };
  __device__ static __forceinline__ void load_a_g(AFrag& f, const E* __restrict__ Ak, int lane) {
    const float4* p = reinterpret_cast<const float4*>(Ak + 4 * lane);
    const float4 x = __ldg(p), y = __ldg(p + 1);
    f.v[0] = make_float2(x.x, x.y);
    f.v[1] = make_float2(x.z, x.w);
    f.v[2] = make_float2(y.x, y.y);
    f.v[3] = make_float2(y.z, y.w);
  }
  __device__ static __forceinline__ void load_a(AFrag& f, const E* Ak, int lane) {
    const float4* p = reinterpret_cast<const float4*>(Ak + 4 * lane);
    const float4 x = p[0], y = p[1];
    f.v[0] = make_float2(x.x, x.y);
    f.v[1] = make_float2(x.z, x.w);
    f.v[2] = make_float2(y.x, y.y);
    f.v[3] = make_float2(y.z, y.w);
  }
  __device__ static __forceinline__ void load_b(BFrag& f, const E* slab, int k0, int c0, int g, int t) {
    const int r0 = k0 + t, r1 = k0 + t + 4;
    f.v[0] = slab[r0 * 32 + ((c0 + g) ^ swz(r0))];
    f.v[1] = slab[r1 * 32 + ((c0 + g) ^ swz(r1))];
  }
  __device__ static __forceinline__ void load_b_x2(BFrag& f, const E* __restrict__ X, int64_t row0, int64_t row1,
                                                   int64_t ldx, int col, int nrhs, bool cj) {
    if (col < nrhs) {
      f.v[0] = __ldg(X + row0 + (int64_t)col * ldx);
      f.v[1] = __ldg(X + row1 + (int64_t)col * ldx);
    } else {
      f.v[0] = f.v[1] = make_float2(0.f, 0.f);
    }
    if (cj) {
      f.v[0].y = -f.v[0].y;
      f.v[1].y = -f.v[1].y;
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
    __device__ __forceinline__ void step(const AFrag& a, const BFrag (&b)[NT]) {
      uint32_t ah[3][4], al[3][4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        split(a.v[e].x, ah[0][e], al[0][e]);
        split(a.v[e].y, ah[1][e], al[1][e]);
        split(a.v[e].x + a.v[e].y, ah[2][e], al[2][e]);
      }
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        uint32_t bh[3][2], bl[3][2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          split(b[ni].v[e].x, bh[0][e], bl[0][e]);
          split(b[ni].v[e].y, bh[1][e], bl[1][e]);
          split(b[ni].v[e].x + b[ni].v[e].y, bh[2][e], bl[2][e]);
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          mma(p[q][ni], ah[q], bl[q]);
          mma(p[q][ni], al[q], bh[q]);
          mma(p[q][ni], ah[q], bh[q]);
        }
      }
    }
    template <typename Fn>
    __device__ __forceinline__ void each(int g, int t, Fn f) const {
#pragma unroll
      for (int ni = 0; ni < NT; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p1 = p[0][ni][e], p2 = p[1][ni][e], p3 = p[2][ni][e];
          f(g + 8 * (e >> 1), 8 * ni + 2 * t + (e & 1), make_float2(p1 - p2, p3 - p1 - p2));
        }
    }
  };
};

// ======================================================================================
// the persistent pass kernel
// ======================================================================================
template <class Pol>
__global__ void __launch_bounds__(FAST_THREADS, 1) k_bf_pass(const __grid_constant__ FastArgs A) {
  using E = typename Pol::E;
  constexpr int SLOTS = 1 << FAST_DMAX;
  constexpr int WPS = FAST_NCONS / SLOTS;  // warps per slot
  constexpr int NT = Pol::NT;
  static_assert(WPS * NT * 8 == FAST_NB, "warp tiling must cover the slab columns");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  E* winbuf = reinterpret_cast<E*>(smem_raw);  // 2 x SLOTS x FAST_SLAB
  unsigned char* ring = smem_raw + 2 * SLOTS * FAST_SLAB * sizeof(E);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + FAST_NBUF * FAST_CHUNK);
  uint64_t* winF = bars;
  uint64_t* winE = bars + 2;
  uint64_t* full = bars + 4;
  uint64_t* empty = bars + 4 + FAST_NBUF;

  const FastPass& P = A.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nslot = 1 << P.d;
  const int64_t ntile = (A.nrhs + FAST_NB - 1) / FAST_NB;
  const int64_t nitems = P.nwin * ntile;
  const int64_t bmask = (int64_t(1) << P.bbits) - 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&winF[i], 1);
      mbar_init(&winE[i], 1);
    }
    for (int i = 0; i < FAST_NBUF; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], FAST_NCONS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == FAST_NCONS) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      const E* Fb = static_cast<const E*>(A.F) + P.fbase;
      const E* Sin = static_cast<const E*>(A.Sin);
      int64_t rc = 0;
      int i = 0;
      for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++i) {
        const int64_t w = item % P.nwin, jt = item / P.nwin;
        const int64_t a = w >> P.bbits, b = w & bmask;
        const int wb = i & 1;
        if (P.in_s >= 0) {
          if (i >= 2) mbar_wait(&winE[wb], ((i - 2) >> 1) & 1, 1);
          mbar_expect_tx(&winF[wb], (uint32_t)(nslot * FAST_SLAB * sizeof(E)));
          E* dst = winbuf + wb * SLOTS * FAST_SLAB;
          for (int s = 0; s < nslot; ++s)
            bulk_g2s(dst + s * FAST_SLAB, Sin + (jt * A.nlev + canon(P, a, b, P.in_s, s)) * FAST_SLAB,
                     FAST_SLAB * sizeof(E), &winF[wb]);
        }
        const unsigned char* Fw = reinterpret_cast<const unsigned char*>(Fb + w * P.win_size);
        for (int q = 0; q < P.nops; ++q) {
          if (!ring_op(P.ops[q].kind)) continue;
          const int64_t sb = fast_slot_size(P.ops[q]) * sizeof(E);
          const int per = (int)(FAST_CHUNK / sb);
          const int nch = (nslot + per - 1) / per;
          for (int c = 0; c < nch; ++c, ++rc) {
            const int bi = (int)(rc % FAST_NBUF);
            if (rc >= FAST_NBUF) mbar_wait(&empty[bi], (uint32_t)(((rc / FAST_NBUF) - 1) & 1), 2, rc);
            const uint32_t bytes = (uint32_t)(min(per, nslot - c * per) * sb);
            mbar_expect_tx(&full[bi], bytes);
            bulk_g2s(ring + bi * FAST_CHUNK, Fw + P.ops[q].off * sizeof(E) + (int64_t)c * per * sb, bytes, &full[bi]);
          }
        }
      }
    }
    // The producer warp stays resident until the consumers are done: an exited warp must not
    // take part in the consumers' named-barrier (bar.sync 1) accounting.
    __syncwarp();
    __syncthreads();
    return;
  }

  // ------------------------------------------------------------------ consumers
  const int g = lane >> 2, t = lane & 3;
  const int o = warp / WPS, h = warp % WPS;
  const bool active = o < nslot;
  const E* __restrict__ X = static_cast<const E*>(A.X);
  E* __restrict__ Y = static_cast<E*>(A.Y);
  E* __restrict__ Sout = static_cast<E*>(A.Sout);
  const bool cj = A.conj_io != 0;
  int64_t rc = 0;
  int i = 0;
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++i) {
    const int64_t w = item % P.nwin, jt = item / P.nwin;
    const int64_t a = w >> P.bbits, b = w & bmask;
    const int wb = i & 1;
    E* win = winbuf + wb * SLOTS * FAST_SLAB;
    const int j0 = (int)jt * FAST_NB + 8 * NT * h;  // first rhs column of this warp
    if (P.in_s >= 0) mbar_wait(&winF[wb], (i >> 1) & 1, 3);
    for (int q = 0; q < P.nops; ++q) {
      const FastOp op = P.ops[q];
      const bool inring = ring_op(op.kind);
      const int64_t sb = fast_slot_size(op) * sizeof(E);
      const int per = (int)(FAST_CHUNK / sb);
      const int nch = inring ? (nslot + per - 1) / per : 0;
      const int64_t cidx = rc + o / per;
      const int bi = (int)(cidx % FAST_NBUF);
      const int users = min(per, nslot - (o / per) * per) * WPS;
      // ring ops read their operand from the ring chunk; leaf ops straight from HBM/L2
      const E* Aslot = inring ? reinterpret_cast<const E*>(ring + bi * FAST_CHUNK + (o % per) * sb)
                              : static_cast<const E*>(A.F) + P.fbase + w * P.win_size + op.off + o * fast_slot_size(op);
      rc += nch;
      const bool last = q == P.nops - 1;
      if (active && inring) mbar_wait(&full[bi], (uint32_t)((cidx / FAST_NBUF) & 1), 4, cidx * 100 + q);

      if (op.kind == FK_LEAF_OUT) {
        if (active) {
          const int64_t row0 = canon(P, a, b, op.s, o) * op.leaf;
          const E* src = win + o * FAST_SLAB;
          for (int mg = 0; mg < op.leaf / 16; ++mg) {
            typename Pol::Acc acc;
            acc.zero();
#pragma unroll
            for (int ki = 0; ki < FAST_RANK / Pol::KS; ++ki) {
              typename Pol::AFrag af;
              typename Pol::BFrag bf[NT];
              Pol::load_a_g(af, Aslot + (mg * (FAST_RANK / Pol::KS) + ki) * Pol::A_KSTEP, lane);
#pragma unroll
              for (int ni = 0; ni < NT; ++ni) Pol::load_b(bf[ni], src, ki * Pol::KS, 8 * NT * h + 8 * ni, g, t);
              acc.step(af, bf);
            }
            acc.each(g, t, [&](int r, int c, E v) {
              const int col = j0 + c;
              if (col < A.nrhs) {
                const int64_t p = row0 + mg * 16 + r;
                const int64_t row = A.yperm ? A.yperm[p] : p;
                if (cj) v.y = -v.y;
                Y[row + (int64_t)col * A.ldy] = v;
              }
            });
          }
        }
        continue;
      }

      typename Pol::Acc acc;
      acc.zero();
      if (active) {
        if (op.kind == FK_LEAF_IN) {
          const int64_t row0 = canon(P, a, b, op.s, o) * op.leaf;
          const int nk = op.leaf / Pol::KS;
#pragma unroll 2
          for (int ki = 0; ki < nk; ++ki) {
            typename Pol::AFrag af;
            typename Pol::BFrag bf[NT];
            Pol::load_a_g(af, Aslot + ki * Pol::A_KSTEP, lane);
            if constexpr (Pol::KS == 4) {
              const int64_t p = row0 + 4 * ki + t;
              const int64_t row = A.xperm ? A.xperm[p] : p;
#pragma unroll
              for (int ni = 0; ni < NT; ++ni) Pol::load_b_x(bf[ni], X, row, A.ldx, j0 + 8 * ni + g, A.nrhs, cj);
            } else {
              const int64_t p0 = row0 + 8 * ki + t, p1 = p0 + 4;
              const int64_t r0 = A.xperm ? A.xperm[p0] : p0, r1 = A.xperm ? A.xperm[p1] : p1;
#pragma unroll
              for (int ni = 0; ni < NT; ++ni) Pol::load_b_x2(bf[ni], X, r0, r1, A.ldx, j0 + 8 * ni + g, A.nrhs, cj);
            }
            acc.step(af, bf);
          }
        } else {
          int src[2];
          int nsrc = 2;
          const int ds = P.d - op.s;
          if (op.kind == FK_PAIR_DOWN) {  // output level s+1 from input level s
            const int tp = o >> (ds - 1), up = o & ((1 << (ds - 1)) - 1);
            src[0] = ((tp >> 1) << ds) + 2 * up;
            src[1] = src[0] + 1;
          } else if (op.kind == FK_PAIR_UP) {  // output level s from input level s+1
            const int tt = o >> ds, u = o & ((1 << ds) - 1);
            src[0] = ((2 * tt) << (ds - 1)) + (u >> 1);
            src[1] = ((2 * tt + 1) << (ds - 1)) + (u >> 1);
          } else {
            src[0] = o;
            nsrc = 1;
          }
          constexpr int KPS = FAST_RANK / Pol::KS;  // k-steps per source slab
#pragma unroll
          for (int sidx = 0; sidx < 2; ++sidx) {
            if (sidx < nsrc) {
              const E* sl = win + src[sidx] * FAST_SLAB;
#pragma unroll
              for (int ki = 0; ki < KPS; ++ki) {
                typename Pol::AFrag af;
                typename Pol::BFrag bf[NT];
                if (inring)
                  Pol::load_a(af, Aslot + (sidx * KPS + ki) * Pol::A_KSTEP, lane);
                else
                  Pol::load_a_g(af, Aslot + (sidx * KPS + ki) * Pol::A_KSTEP, lane);
#pragma unroll
                for (int ni = 0; ni < NT; ++ni) Pol::load_b(bf[ni], sl, ki * Pol::KS, 8 * NT * h + 8 * ni, g, t);
                acc.step(af, bf);
              }
            }
          }
        }
        if (inring) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[bi], FAST_NCONS / users);
        }
      }
      consumer_sync();  // every warp has finished reading this op's input slabs
      if (active) {
        if (last && P.out_s >= 0) {
          E* dst = Sout + (jt * A.nlev + canon(P, a, b, P.out_s, o)) * FAST_SLAB;
          acc.each(g, t, [&](int r, int c, E v) { dst[r * 32 + ((8 * NT * h + c) ^ Pol::swz(r))] = v; });
        } else {
          E* dst = win + o * FAST_SLAB;
          acc.each(g, t, [&](int r, int c, E v) { dst[r * 32 + ((8 * NT * h + c) ^ Pol::swz(r))] = v; });
        }
      }
      if (!(last && P.out_s >= 0)) consumer_sync();
    }
    consumer_sync();
    if (threadIdx.x == 0) mbar_arrive(&winE[wb], 1);
  }
  __syncthreads();  // joins the producer warp
}

const char* fast_kernel_name(int dtype) { return dtype == BF_C128 ? "k_bf_pass<c128>" : "k_bf_pass<c64>"; }

size_t fast_smem_bytes(int dtype) {
  const size_t es = dtype == BF_C128 ? 16 : 8;
  return 2 * (size_t)(1 << FAST_DMAX) * FAST_SLAB * es + (size_t)FAST_NBUF * FAST_CHUNK + (4 + 2 * FAST_NBUF) * 8;
}

void launch_fast_pass(int dtype, const FastArgs& a, cudaStream_t st) {
  static int nsm = 0;
  static bool attr[2] = {false, false};
  if (nsm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = fast_smem_bytes(dtype);
  const int64_t items = a.p.nwin * ((a.nrhs + FAST_NB - 1) / FAST_NB);
  const unsigned grid = (unsigned)(items < nsm ? items : nsm);
  if (dtype == BF_C128) {
    if (!attr[0]) {
      cudaFuncSetAttribute(k_bf_pass<PolC128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr[0] = true;
    }
    k_bf_pass<PolC128><<<grid, FAST_THREADS, smem, st>>>(a);
  } else {
    if (!attr[1]) {
      cudaFuncSetAttribute(k_bf_pass<PolC64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr[1] = true;
    }
    k_bf_pass<PolC64><<<grid, FAST_THREADS, smem, st>>>(a);
  }
}

}  // namespace bfa
