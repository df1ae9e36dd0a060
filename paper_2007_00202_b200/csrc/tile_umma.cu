// complex64 generic gather-sum on the 5th-generation tensor cores (tcgen05.mma kind::tf32, TMEM
// accumulators) -- the HOD-BF / ragged-rank / NEXT-2..4 rounds of kernels.cu (SURVEY 8(a) a1-a7 on
// the generic plan; the HOD-BF apply) for complex64 with nrhs >= 64:
//
//   out^T (rhs x m) = sum_t In_t^T (rhs x k) A_t^T (k x m)
//
// Used for the rounds between slab levels (In and out in the slab space; the leaf rounds reading X
// or writing Y keep the row-tile kernel).  One CTA (4 warps, 44 KB: 5 per SM) per (unit = task x
// 32-row block, 128-column rhs tile): MMA M = 128 right-hand sides (TMEM lane = rhs), N = 64 =
// [re | im] of the 32 output rows, K streamed in chunks of 8 (one MMA step).  The complex product is the real embedding with the imaginary sign folded
// into the factor planes:
//   D[:, 0:32]  = Xr Ar^T - Xi Ai^T = re,   D[:, 32:64] = Xr Ai^T + Xi Ar^T = im
//   i.e. D += Xr [Ar; Ai]^T + Xi [-Ai; Ar]^T,
// with the factor rows stored once as three planes [-Ai | Ar | Ai] (the N = 64 operand [Ar; Ai]
// starts at plane 1, [-Ai; Ar] at plane 0).  Accuracy: 3xTF32 -- every operand split into hi and
// lo (x = hi + lo to ~2^-22, both rounded to nearest TF32), D += Ahi Bhi + Ahi Blo + Alo Bhi (6
// MMAs per chunk).  Operands: K-major, no swizzle, canonical core matrices (8 rows x 16 bytes), built
// in shared memory by all threads from coalesced global loads (split + scatter) in two stages; the
// loads of chunk c + 1 are in flight while chunk c is converted and multiplied; one thread issues
// the MMAs and commits them to the stage's mbarrier.  Conventions (descriptor LBO / SBO, instruction descriptor, TMEM lane =
// row for M = 128) measured on the B200 with tools/umma_tf32_test.cu.
#include <cstdio>

#include "mma.cuh"

namespace bfa {

namespace {
constexpr int UM_M = 128;                       // right-hand sides per CTA tile (MMA M, TMEM lanes)
constexpr int UM_TR = 32;                       // task rows per unit (the plan's 32-row blocks)
constexpr int UM_N = 64;                        // MMA N: [re | im] x 32 rows
constexpr int UM_KC = 8;                        // K per chunk (one MMA step)
constexpr int UM_APL = UM_M * UM_KC * 4;        // 4 KB: one real plane of In^T (128 x 8 fp32)
constexpr int UM_BPL = UM_TR * UM_KC * 4;       // 1 KB: one real plane of factor rows (32 x 8)
constexpr int UM_STAGE = 4 * UM_APL + 6 * UM_BPL;  // A: Xr hi, lo, Xi hi, lo; B: hi [-Ai|Ar|Ai], lo [...]
constexpr int UM_NST = 2;
constexpr int UM_SMEM = UM_NST * UM_STAGE;      // 44 KB: 5 CTAs per SM
constexpr int UM_THREADS = 128;
constexpr uint32_t UM_TMEM_COLS = 64;

// byte offset of element (row, k) of a K-major no-swizzle operand with K = 8 per row group:
// core matrices of 8 rows x 4 K (16 B rows, 128 B), the two K-adjacent ones contiguous
// (LBO = 128), 8-row groups 256 B apart (SBO = 256)
__device__ __forceinline__ uint32_t um_off(int row, int k) {
  return (uint32_t)((row >> 3) * 256 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t um_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(128 >> 4) << 16;  // LBO: K-direction core-matrix step
  d |= (uint64_t)(256 >> 4) << 32;  // SBO: M/N-direction 8-row step
  d |= (uint64_t)1 << 46;           // descriptor version (sm_100)
  return d;                         // base offset 0, SWIZZLE_NONE
}
// kind::tf32, D = F32, A = B = TF32, both K-major, N = 64, M = 128
constexpr uint32_t UM_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(UM_N >> 3) << 17) |
                              ((uint32_t)(UM_M >> 4) << 24);

__device__ __forceinline__ void um_mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(UM_IDESC), "r"(acc));
}
__device__ __forceinline__ void um_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
// 3xTF32 split with round-to-nearest TF32 parts (hi = rn(x), lo = rn(x - hi), x - hi exact in
// FP32): the tensor core reads only the top 19 bits of each operand, so a raw FP32 lo would be
// truncated toward zero -- a bias that accumulates over K (measured 1.0e-5 vs 3e-6 relative error
// on a ragged rank-70 butterfly)
__device__ __forceinline__ float um_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void um_split(float x, float& hi, float& lo) {
  hi = um_rna(x);
  lo = um_rna(x - hi);
}
__device__ __forceinline__ void um_ld32(uint32_t addr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
}  // namespace

__global__ void __launch_bounds__(UM_THREADS) k_stage_umma(StageArgs a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar[UM_NST];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 un = a.units[blockIdx.x];  // plan tables: immutable, read before the PDL wait
  const Task tk = a.tasks[un.x];
  if (tid == 0) {
    for (int s = 0; s < UM_NST; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_slot)),
                 "n"(UM_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_slot;
  pdl_wait();  // slabs / X / Y of the previous rounds

  const int r0 = un.y * UM_TR;
  const int j0 = blockIdx.y * UM_M;
  const float2* __restrict__ pool = static_cast<const float2*>(a.pool);
  const float2* __restrict__ S = static_cast<const float2*>(a.S);
  const float2* __restrict__ X = static_cast<const float2*>(a.X);
  const uint32_t sbase = smem_u32(sm);
  const int m = tid;                         // A part: this thread's rhs row
  const int bn = tid >> 2, bg = (tid & 3) * 2;  // B part: factor row, first k of its 2
  const bool mok = j0 + m < a.nrhs;
  const bool nok = r0 + bn < tk.m;

  // chunk sequence: (term q, rows kc..kc+7 of its K); the operands of chunk c + 1 are loaded into
  // registers before chunk c is converted and issued, so their latency overlaps the MMAs
  int lq = 0, lkc = 0;  // next chunk to load
  Term ltm{};
  if (tk.nterm > 0) ltm = a.terms[tk.term0];
  float2 xv[UM_KC], fv[2];
  auto load = [&]() {
    const bool cj = (ltm.conj != 0) != (a.conj_flip != 0);
#pragma unroll
    for (int k = 0; k < UM_KC; ++k) {
      xv[k] = make_float2(0.f, 0.f);
      if (mok && lkc + k < ltm.k) {
        const int64_t p = ltm.in_row + lkc + k;
        xv[k] = ltm.in_kind == 0 ? S[p * a.ldS + j0 + m] : X[(a.xperm ? a.xperm[p] : p) + (int64_t)(j0 + m) * a.ldx];
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      fv[e] = make_float2(0.f, 0.f);
      if (nok && lkc + bg + e < ltm.k)
        fv[e] = pool[ltm.a_off + (int64_t)(r0 + bn) * ltm.a_rs + (int64_t)(lkc + bg + e) * ltm.a_cs];
      fv[e].y = conj_im(fv[e].y, cj);
    }
    lkc += UM_KC;
    if (lkc >= ltm.k) {
      lkc = 0;
      if (++lq < tk.nterm) ltm = a.terms[tk.term0 + lq];
    }
  };
  int nch = 0;
  for (int q = 0; q < tk.nterm; ++q) nch += (a.terms[tk.term0 + q].k + UM_KC - 1) / UM_KC;
  if (nch > 0) load();
  int c = 0;  // chunks issued
  for (; c < nch; ++c) {
    const int st = c & 1;
    float2 cx[UM_KC], cf[2];
#pragma unroll
    for (int k = 0; k < UM_KC; ++k) cx[k] = xv[k];
    cf[0] = fv[0];
    cf[1] = fv[1];
    if (c + 1 < nch) load();
    // the stage is free once the MMAs of chunk c - 2 are done
    if (c >= 2) mbar_wait(&mbar[st], (uint32_t)(((c - 2) >> 1) & 1), 21);
    unsigned char* sa = sm + st * UM_STAGE;
    unsigned char* sb = sa + 4 * UM_APL;
#pragma unroll
    for (int g = 0; g < UM_KC / 4; ++g) {
      float rh[4], rl[4], ih[4], il[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        um_split(cx[4 * g + e].x, rh[e], rl[e]);
        um_split(cx[4 * g + e].y, ih[e], il[e]);
      }
      const uint32_t o = um_off(m, 4 * g);
      *reinterpret_cast<float4*>(sa + 0 * UM_APL + o) = make_float4(rh[0], rh[1], rh[2], rh[3]);
      *reinterpret_cast<float4*>(sa + 1 * UM_APL + o) = make_float4(rl[0], rl[1], rl[2], rl[3]);
      *reinterpret_cast<float4*>(sa + 2 * UM_APL + o) = make_float4(ih[0], ih[1], ih[2], ih[3]);
      *reinterpret_cast<float4*>(sa + 3 * UM_APL + o) = make_float4(il[0], il[1], il[2], il[3]);
    }
    {
      float rh[2], rl[2], ih[2], il[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        um_split(cf[e].x, rh[e], rl[e]);
        um_split(cf[e].y, ih[e], il[e]);
      }
      const uint32_t o = um_off(bn, bg);
      // hi planes [-Ai | Ar | Ai], then lo planes
      *reinterpret_cast<float2*>(sb + 0 * UM_BPL + o) = make_float2(-ih[0], -ih[1]);
      *reinterpret_cast<float2*>(sb + 1 * UM_BPL + o) = make_float2(rh[0], rh[1]);
      *reinterpret_cast<float2*>(sb + 2 * UM_BPL + o) = make_float2(ih[0], ih[1]);
      *reinterpret_cast<float2*>(sb + 3 * UM_BPL + o) = make_float2(-il[0], -il[1]);
      *reinterpret_cast<float2*>(sb + 4 * UM_BPL + o) = make_float2(rl[0], rl[1]);
      *reinterpret_cast<float2*>(sb + 5 * UM_BPL + o) = make_float2(il[0], il[1]);
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t A0 = sbase + st * UM_STAGE, B0 = A0 + 4 * UM_APL;
#pragma unroll
      for (int x = 0; x < 2; ++x) {  // x = 0: Xr with [Ar; Ai], x = 1: Xi with [-Ai; Ar]
        const uint32_t ah = A0 + (2 * x) * UM_APL, al = A0 + (2 * x + 1) * UM_APL;
        const uint32_t bh = B0 + (x == 0 ? 1 : 0) * UM_BPL, bl = B0 + (x == 0 ? 4 : 3) * UM_BPL;
        um_mma(tmem, um_desc(ah), um_desc(bh), (c > 0 || x > 0) ? 1u : 0u);
        um_mma(tmem, um_desc(ah), um_desc(bl), 1u);
        um_mma(tmem, um_desc(al), um_desc(bh), 1u);
      }
      um_commit(&mbar[st]);
    }
  }
  // epilogue: warp w owns TMEM lanes 32w.. = rhs 32w + lane; columns 0..31 re, 32..63 im
  const int col = j0 + 32 * warp + lane;
  float re[32], im[32];
  if (c > 0) {
    mbar_wait(&mbar[(c - 1) & 1], (uint32_t)(((c - 1) >> 1) & 1), 22);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16);
    um_ld32(ta, re);
    um_ld32(ta + 32, im);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  } else {
#pragma unroll
    for (int n = 0; n < 32; ++n) re[n] = im[n] = 0.f;
  }
  pdl_trigger();
  if (col < a.nrhs) {
#pragma unroll
    for (int n = 0; n < 32; ++n) {
      const int r = r0 + n;
      if (r >= tk.m) break;
      const float2 v = make_float2(re[n], im[n]);
      if (a.out_kind == 0) {
        static_cast<float2*>(a.S)[(tk.out_row + r) * a.ldS + col] = v;
      } else {
        const int64_t p = tk.out_row + r;
        static_cast<float2*>(a.Y)[(a.yperm ? a.yperm[p] : p) + (int64_t)col * a.ldy] = v;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(UM_TMEM_COLS));
}

void launch_tile_umma(const StageArgs& a, cudaStream_t st) {
  static std::atomic<size_t> attr[BF_MAX_DEVICES];
  ensure_smem_attr(attr, (const void*)k_stage_umma, UM_SMEM);
  launch_pdl(k_stage_umma, (unsigned)a.nunits, (unsigned)((a.nrhs + UM_M - 1) / UM_M), UM_THREADS, UM_SMEM, st, a);
}

}  // namespace bfa
