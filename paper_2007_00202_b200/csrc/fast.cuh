// Fused "window pass" path for uniform-rank butterflies (rank 16, power-of-two leaves that
// are multiples of 16).
//
// A pass covers d <= 3 consecutive levels l0..l1 of Eq. (3.3).  One work item is a closed
// window (SURVEY 7.3 hard part 3): T_O node a at level l0 and T_S node b at level L-l1.  At
// window level s (0..d) the window holds the S = 2^d slabs (tau, nu) with
//     tau = a 2^s + (slot >> (d-s)),   nu = b 2^(d-s) + (slot & (2^(d-s)-1)),
// so every stage inside the pass reads and writes only slabs of the same window, which stay
// in shared memory.  Between passes, slabs go through two ping-pong HBM buffers in canonical
// order.
//
// Operand stream.  Every op of a pass is a sequence of MMA k-steps; the A operand (the factor
// block) of one k-step of one slot is one 1 KB fragment-ordered record.  At create time each
// op's factors are laid out window-major as [step][slot][1 KB], so any run of consecutive
// k-steps of all slots is one contiguous byte range: the producer warp streams it into 8 KB
// pages of a shared-memory ring with TMA bulk copies, and all consumer warps walk the pages in
// order, releasing each page as soon as they have used it.  For the leaf op that reads the
// user block X, the X rows of each (k-step, slot) are brought in by TMA tensor loads (2-D map
// over X) into two more pages per A page.
#pragma once

#include "common.cuh"

namespace bfa {

enum FastKind : int32_t { FK_LEAF_IN = 0, FK_PAIR_DOWN = 1, FK_PAIR_UP = 2, FK_DIAG = 3, FK_LEAF_OUT = 4 };
constexpr int FAST_RANK = 16;                   // r: slab rows
constexpr int FAST_NB = 32;                     // right-hand sides per work item (slab columns)
constexpr int FAST_DMAX = 3;                    // window levels per pass
constexpr int FAST_MAXOPS = 8;
constexpr int FAST_SLAB = FAST_RANK * FAST_NB;  // complex entries per slab (512)
constexpr int FAST_NCONS = 8;                   // consumer warps
constexpr int FAST_THREADS = (FAST_NCONS + 1) * 32;  // + one producer warp
constexpr int FAST_FRAG = 1024;                 // bytes of A operand per (k-step, slot)
constexpr int FAST_PAGE = 16384;                // bytes per ring page
constexpr int FAST_XBOX = 2048;                 // bytes of X per (k-step, slot): KS rows x 32 rhs
constexpr int FAST_XSTAGES = 4;                 // X staging depth per consumer warp (k-steps)
// bytes of the two window buffers; the second doubles as the per-warp X staging of the leaf op
template <typename E>
__host__ __device__ constexpr size_t fast_win_region() {
  constexpr size_t win = (size_t)(1 << FAST_DMAX) * FAST_SLAB * sizeof(E);
  constexpr size_t xst = (size_t)FAST_NCONS * FAST_XSTAGES * FAST_XBOX;
  return win + (win > xst ? win : xst);
}

struct FastOp {
  int32_t kind;
  int32_t s;       // window level: input level of PAIR_DOWN, output level of PAIR_UP, level of DIAG / leaves
  int32_t leaf;    // leaf size (LEAF_IN: K; LEAF_OUT: M)
  int32_t nsteps;  // MMA k-steps (LEAF_OUT: (leaf/16) x (16/KS), row-group major)
  int64_t off;     // byte offset of this op's factor stream inside a window record
};

struct FastPass {
  int32_t d, L, l0, bbits;  // window levels, tree depth, first level, log2(#b values) = L - l1
  int32_t nops, in_s, out_s, xpage;  // xpage: LEAF_IN X rows are gathered into ring pages
  int32_t numaj, pad;                // HBM slab order: 0 tau-major (op N), 1 nu-major (op C / T)
  int64_t fbase, win_bytes;  // byte offset of window 0's record, bytes per window record
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
  int32_t xalign16; // X rows of one leaf start on 16-byte boundaries (else 8-byte cp.async)
  int32_t diag;     // profiling only (env BF_FAST_DIAG, results are garbage): bit 0 = no operand
                    // streaming (compute only), bit 1 = inter-pass slabs not written to HBM
};

void launch_fast_pass(int dtype, const FastArgs& a, cudaStream_t st);
size_t fast_smem_bytes(int dtype);
const char* fast_kernel_name(int dtype);

// k-steps per MMA along K: complex128 DMMA m8n8k4 -> 4, complex64 TF32 m16n8k8 -> 8
__host__ __device__ inline int fast_ks(int csize) { return csize == 16 ? 4 : 8; }

__host__ __device__ inline int fast_nsteps(int kind, int leaf, int ks) {
  switch (kind) {
    case FK_LEAF_IN: return leaf / ks;
    case FK_LEAF_OUT: return (leaf / 16) * (16 / ks);
    case FK_PAIR_DOWN:
    case FK_PAIR_UP: return 2 * FAST_RANK / ks;
    default: return FAST_RANK / ks;
  }
}


}  // namespace bfa
