// Fused window-pass kernels (see fast.cuh for the window / slot definitions).
//
// complex128: every block product out(16 x 32) = sum_s A_s(16 x 16 or 16 x leaf) in_s
// runs on the FP64 tensor pipe (mma.sync.m8n8k4.f64, "DMMA") with the 3-multiplication
// complex product:
//     P1 = Ar Br,  P2 = Ai Bi,  P3 = (Ar + Ai)(Br + Bi);   Re = P1 - P2,  Im = P3 - P1 - P2,
// i.e. 3 real DMMAs per complex MMA instead of 4.  (B200 DMMA throughput measured equal to
// DFMA -- profiles/pipe_peaks.json -- so the 25% saving is the lever; operands come from
// registers, which keeps issue slots and the shared-memory port free.)
//
// Fragment layouts (PTX ISA, m8n8k4 .f64): lane = 4 g + t,
//   A (8 x 4, row): a = A[g][t];   B (4 x 8, col): b = B[t][g];   C (8 x 8): c_e = C[g][2t + e].
// A slab in shared memory (and in the HBM ping-pong buffers) is 16 rows x 32 complex with
// the 16-byte unit of (row, col) at  row * 32 + (col ^ swz(row)),  swz(r) = ((r&3)<<1)|(r&1):
// both the C-fragment stores and the B-fragment loads hit 8 distinct 16-byte bank groups per
// quarter-warp phase (conflict free).
#include "fast.cuh"

namespace bfa {

__device__ __forceinline__ int swz(int row) { return ((row & 3) << 1) | (row & 1); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// window slot -> canonical block index at window level s
__device__ __forceinline__ int64_t canon(const FastPass& P, int64_t a, int64_t b, int s, int slot) {
  const int ds = P.d - s;
  const int64_t tau = (a << s) + (slot >> ds);
  const int64_t nu = (b << ds) + (slot & ((1 << ds) - 1));
  return (tau << (P.L - (P.l0 + s))) + nu;
}

struct Acc3 {
  double p[3][2][4][2];  // [product][mi][ni][e]
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) p[q][mi][ni][0] = p[q][mi][ni][1] = 0.0;
  }
  // one k-step of 4: A fragments for 2 m-tiles, B fragments for 4 n-tiles
  __device__ __forceinline__ void step(const double2 (&a)[2], const double2 (&bf)[4]) {
    double bs[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) bs[ni] = bf[ni].x + bf[ni].y;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const double as = a[mi].x + a[mi].y;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        dmma(p[0][mi][ni][0], p[0][mi][ni][1], a[mi].x, bf[ni].x);
        dmma(p[1][mi][ni][0], p[1][mi][ni][1], a[mi].y, bf[ni].y);
        dmma(p[2][mi][ni][0], p[2][mi][ni][1], as, bs[ni]);
      }
    }
  }
  // combine into complex results: res[mi][ni][e]
  __device__ __forceinline__ void result(double2 (&res)[2][4][2]) const {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double p1 = p[0][mi][ni][e], p2 = p[1][mi][ni][e], p3 = p[2][mi][ni][e];
          res[mi][ni][e] = make_double2(p1 - p2, p3 - p1 - p2);
        }
  }
};

// B fragments (2 n-tiles of half h) of k-step ki (rows 4ki..4ki+3) of window slot `slot`
__device__ __forceinline__ void load_b_smem(double2 (&bf)[2], const double2* win, int slot, int ki, int h, int g,
                                            int t) {
  const double2* base = win + slot * FAST_SLAB + (4 * ki + t) * 32 + 16 * h + (g ^ swz(t));
  bf[0] = base[0];
  bf[1] = base[8];
}

// A fragments (2 m-tiles) of k-chunk `chunk` from fragment-ordered data (global or shared)
__device__ __forceinline__ void load_a(double2 (&a)[2], const double2* A, int chunk, int lane) {
  a[0] = A[(chunk * 2 + 0) * 32 + lane];
  a[1] = A[(chunk * 2 + 1) * 32 + lane];
}
__device__ __forceinline__ void load_a_g(double2 (&a)[2], const double2* __restrict__ A, int chunk, int lane) {
  a[0] = __ldg(A + (chunk * 2 + 0) * 32 + lane);
  a[1] = __ldg(A + (chunk * 2 + 1) * 32 + lane);
}

// ---- mbarrier / bulk-copy (TMA 1-D) helpers --------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct Acc3h {  // 3M accumulators for a 16 x 16 (2 m-tiles x 2 n-tiles) output
  double p[3][2][2][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) p[q][mi][ni][0] = p[q][mi][ni][1] = 0.0;
  }
  __device__ __forceinline__ void step(const double2 (&a)[2], const double2 (&bf)[2]) {
    double bs[2];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) bs[ni] = bf[ni].x + bf[ni].y;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const double as = a[mi].x + a[mi].y;
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) {
        dmma(p[0][mi][ni][0], p[0][mi][ni][1], a[mi].x, bf[ni].x);
        dmma(p[1][mi][ni][0], p[1][mi][ni][1], a[mi].y, bf[ni].y);
        dmma(p[2][mi][ni][0], p[2][mi][ni][1], as, bs[ni]);
      }
    }
  }
  __device__ __forceinline__ void result(double2 (&res)[2][2][2]) const {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double p1 = p[0][mi][ni][e], p2 = p[1][mi][ni][e], p3 = p[2][mi][ni][e];
          res[mi][ni][e] = make_double2(p1 - p2, p3 - p1 - p2);
        }
  }
};

__device__ __forceinline__ bool uses_ring(int kind) { return kind != FK_LEAF_IN && kind != FK_LEAF_OUT; }

// 16 warps: warp w computes the half (columns 16h..16h+15, h = w & 1) of window slot o = w >> 1.
__global__ void __launch_bounds__(FAST_THREADS, 1) k_bf_pass_c128(const __grid_constant__ FastArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* win = reinterpret_cast<double2*>(smem_raw);
  double2* fbuf = win + (1 << FAST_DMAX) * FAST_SLAB;  // 2 x FAST_OPBUF complex
  uint64_t* bars = reinterpret_cast<uint64_t*>(fbuf + 2 * FAST_OPBUF);
  const FastPass& P = A.p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int o = warp >> 1, h = warp & 1;
  const int d = P.d, nslot = 1 << d;
  const int64_t w = blockIdx.x;
  const int jt = blockIdx.y;
  const int j0 = jt * FAST_NB;
  const int64_t a = w >> P.bbits, b = w & ((int64_t(1) << P.bbits) - 1);
  const double2* __restrict__ F = static_cast<const double2*>(A.F) + P.fbase + w * P.win_size;
  const double2* __restrict__ X = static_cast<const double2*>(A.X);
  double2* __restrict__ Y = static_cast<double2*>(A.Y);
  const double2* __restrict__ Sin = static_cast<const double2*>(A.Sin) + (int64_t)jt * A.nlev * FAST_SLAB;
  double2* __restrict__ Sout = static_cast<double2*>(A.Sout) + (int64_t)jt * A.nlev * FAST_SLAB;

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // producer (thread 0): stream op q's factors for this window into ring buffer q & 1
  auto issue = [&](int q) {
    if (threadIdx.x == 0 && q < P.nops && uses_ring(P.ops[q].kind)) {
      const uint32_t bytes = (uint32_t)(nslot * fast_slot_size(P.ops[q]) * sizeof(double2));
      mbar_expect_tx(&bars[q & 1], bytes);
      bulk_g2s(fbuf + (q & 1) * FAST_OPBUF, F + P.ops[q].off, bytes, &bars[q & 1]);
    }
  };
  issue(0);
  if (P.in_s >= 0) {
    for (int e = threadIdx.x; e < nslot * FAST_SLAB; e += blockDim.x) {
      const int slot = e / FAST_SLAB, u = e % FAST_SLAB;
      win[e] = Sin[canon(P, a, b, P.in_s, slot) * FAST_SLAB + u];
    }
  }
  __syncthreads();
  uint32_t phase[2] = {0, 0};

  for (int q = 0; q < P.nops; ++q) {
    issue(q + 1);
    const FastOp op = P.ops[q];
    const bool active = o < nslot;
    if (op.kind == FK_LEAF_OUT) {
      if (active) {
        const double2* __restrict__ Fo = F + op.off + (int64_t)o * fast_slot_size(op);
        const int64_t row0 = canon(P, a, b, op.s, o) * op.leaf;
        for (int mg = 0; mg < op.leaf / 16; ++mg) {
          Acc3h acc;
          acc.zero();
#pragma unroll
          for (int ki = 0; ki < 4; ++ki) {
            double2 af[2], bf[2];
            load_a_g(af, Fo, mg * 4 + ki, lane);
            load_b_smem(bf, win, o, ki, h, g, t);
            acc.step(af, bf);
          }
          double2 res[2][2][2];
          acc.result(res);
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) {
            const int64_t p = row0 + mg * 16 + mi * 8 + g;
            const int64_t row = A.yperm ? A.yperm[p] : p;
#pragma unroll
            for (int ni = 0; ni < 2; ++ni)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int col = j0 + 16 * h + 8 * ni + 2 * t + e;
                if (col < A.nrhs) {
                  double2 v = res[mi][ni][e];
                  if (A.conj_io) v.y = -v.y;
                  Y[row + (int64_t)col * A.ldy] = v;
                }
              }
          }
        }
      }
      continue;
    }
    double2 res[2][2][2];
    if (uses_ring(op.kind)) {
      mbar_wait(&bars[q & 1], phase[q & 1]);
      phase[q & 1] ^= 1;
    }
    if (active) {
      Acc3h acc;
      acc.zero();
      if (op.kind == FK_LEAF_IN) {
        const double2* __restrict__ Fo = F + op.off + (int64_t)o * fast_slot_size(op);
        const int64_t row0 = canon(P, a, b, op.s, o) * op.leaf;
        for (int ki = 0; ki < op.leaf / 4; ++ki) {
          double2 af[2], bf[2];
          load_a_g(af, Fo, ki, lane);
          const int64_t p = row0 + 4 * ki + t;
          const int64_t row = A.xperm ? A.xperm[p] : p;
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            const int col = j0 + 16 * h + 8 * ni + g;
            bf[ni] = col < A.nrhs ? __ldg(X + row + (int64_t)col * A.ldx) : make_double2(0.0, 0.0);
            if (A.conj_io) bf[ni].y = -bf[ni].y;
          }
          acc.step(af, bf);
        }
      } else {
        const double2* Fo = fbuf + (q & 1) * FAST_OPBUF + o * fast_slot_size(op);
        int src[2];
        int nsrc = 2;
        const int ds = d - op.s;
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
#pragma unroll
        for (int sidx = 0; sidx < 2; ++sidx) {
          if (sidx < nsrc) {
#pragma unroll
            for (int ki = 0; ki < 4; ++ki) {
              double2 af[2], bf[2];
              load_a(af, Fo, sidx * 4 + ki, lane);
              load_b_smem(bf, win, src[sidx], ki, h, g, t);
              acc.step(af, bf);
            }
          }
        }
      }
      acc.result(res);
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int row = mi * 8 + g;
        double2* dst = win + o * FAST_SLAB + row * 32 + 16 * h;
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) dst[8 * ni + ((2 * t + e) ^ swz(row))] = res[mi][ni][e];
      }
    }
    __syncthreads();
  }

  if (P.out_s >= 0) {
    for (int e = threadIdx.x; e < nslot * FAST_SLAB; e += blockDim.x) {
      const int slot = e / FAST_SLAB, u = e % FAST_SLAB;
      Sout[canon(P, a, b, P.out_s, slot) * FAST_SLAB + u] = win[e];
    }
  }
}

const char* fast_kernel_name(int dtype) { return dtype == BF_C128 ? "k_bf_pass_c128" : "k_bf_pass_c64"; }

void launch_fast_pass(int dtype, const FastArgs& a, cudaStream_t st) {
  const int nslot = 1 << a.p.d;
  (void)nslot;
  const size_t smem = ((size_t)(1 << FAST_DMAX) * FAST_SLAB + 2 * FAST_OPBUF) * 16 + 64;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(k_bf_pass_c128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_done = true;
  }
  dim3 grid((unsigned)a.p.nwin, (a.nrhs + FAST_NB - 1) / FAST_NB);
  k_bf_pass_c128<<<grid, FAST_THREADS, smem, st>>>(a);
}

}  // namespace bfa
