// Fused "window pass" path for uniform-rank butterflies (rank 16, leaves multiple of 16).
//
// A pass covers d <= 3 consecutive levels l0..l1 of Eq. (3.3).  One CTA owns a closed
// window (SURVEY 7.3 hard part 3): T_O node a at level l0 and T_S node b at level L-l1.
// At window level s (0..d) the window holds the 2^d slabs (tau, nu) with
//     tau = a 2^s + (slot >> (d-s)),   nu = b 2^(d-s) + (slot & (2^(d-s)-1)),
// so every stage inside the pass reads and writes only slabs of the same window, which
// stay in shared memory.  Between passes, slabs go through two ping-pong HBM buffers
// in canonical order.  Factor blocks are re-laid out at create time into the exact
// fragment order the tensor-core MMA consumes, window-major, so each warp streams its
// operands with fully coalesced 512-byte loads.
#pragma once
#include "common.cuh"

namespace bfa {

enum FastKind : int32_t { FK_LEAF_IN = 0, FK_PAIR_DOWN = 1, FK_PAIR_UP = 2, FK_DIAG = 3, FK_LEAF_OUT = 4 };
constexpr int FAST_RANK = 16;      // r: slab rows
constexpr int FAST_NB = 32;        // right-hand sides per CTA (slab columns)
constexpr int FAST_DMAX = 3;       // window levels per pass
constexpr int FAST_MAXOPS = 8;
constexpr int FAST_SLAB = FAST_RANK * FAST_NB;  // complex entries per slab (512)
constexpr int FAST_NCONS = 8;                       // consumer warps (one per window slot; 17 warps would cap registers at 96)
constexpr int FAST_THREADS = (FAST_NCONS + 1) * 32;  // + one producer warp
constexpr int FAST_CHUNK = 16384;                    // bytes per factor-ring chunk
constexpr int FAST_NBUF = 6;                         // factor-ring depth

struct FastOp {
  int32_t kind;
  int32_t s;      // window level: input level of PAIR_DOWN, output level of PAIR_UP, level of DIAG / leaves
  int32_t leaf;   // leaf size (LEAF_IN: K; LEAF_OUT: M)
  int32_t pad;
  int64_t off;    // complex offset of this op's factors inside a window chunk
  int64_t flops;  // real flops of this op per window per 32 rhs (accounting)
};

struct FastPass {
  int32_t d, L, l0, bbits;  // window levels, tree depth, first level, log2(#b values) = L - l1
  int32_t nops, in_s, out_s, pad;
  int64_t fbase, win_size;  // factor offset of window 0, complex entries per window
  int64_t nwin;
  int64_t factor_entries, user_in, user_out;  // accounting
  FastOp ops[FAST_MAXOPS];
};

struct FastArgs {
  FastPass p;
  const void* F;
  const void* X;
  int64_t ldx;
  const int64_t* xperm;
  void* Y;
  int64_t ldy;
  const int64_t* yperm;
  const void* Sin;
  void* Sout;
  int64_t nlev;  // slabs per level (2^L)
  int32_t nrhs;
  int32_t conj_io;  // op T: conjugate X on load and Y on store (K^T X = conj(K^H conj X))
};

void launch_fast_pass(int dtype, const FastArgs& a, cudaStream_t st);
size_t fast_smem_bytes(int dtype);
const char* fast_kernel_name(int dtype);

// per-slot complex entries of an op's factor data
__host__ __device__ inline int64_t fast_slot_size(const FastOp& op) {
  switch (op.kind) {
    case FK_LEAF_IN:
    case FK_LEAF_OUT: return int64_t(FAST_RANK) * op.leaf;
    case FK_PAIR_DOWN:
    case FK_PAIR_UP: return 2 * FAST_RANK * FAST_RANK;
    default: return FAST_RANK * FAST_RANK;
  }
}

}  // namespace bfa
