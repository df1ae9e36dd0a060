// Fast path for rank-16 butterflies (power-of-two leaves that are multiples of 16, at most 256;
// ranks <= 16 are zero-padded to 16 at create, plan.cu pad_rank16): one apply = a leaf launch, a
// few window passes, a leaf launch.
//
// Leaf launches (leaf.cu): every leaf product of Eq. (3.3)'s outer factors
// (V^0 = blkdiag(Vt_nu) on the input side, U^L = blkdiag(U_tau) on the output side)
// in one HBM-bound launch that streams the user block X in / Y out once.
//
// Window passes (fast.cu; a2 - a4): a pass covers d <= 3 consecutive levels l0..l1 of
// Eq. (3.3).  One work item is a closed window (SURVEY 7.3 hard part 3): T_O node a at level l0
// and T_S node b at level L-l1.  At window level s (0..d) the window holds the S = 2^d slabs
// (tau, nu) with
//     tau = a 2^s + (slot >> (d-s)),   nu = b 2^(d-s) + (slot & (2^(d-s)-1)),
// so every stage inside the pass reads and writes only slabs of the same window, which stay in
// shared memory.  Between launches slabs go through two ping-pong HBM buffers in canonical order.
//
// Operand stream.  Every op is a sequence of MMA k-steps; the A operand (factor block) of one
// k-step of one slot is one 1 KB fragment-ordered record.  At create time each op's factors are
// laid out window-major as [step][slot][1 KB], so any run of consecutive k-steps of all slots
// is one contiguous byte range, streamed into the 32 KB pages of a shared-memory ring with TMA
// bulk copies.  There is no producer warp: whichever compute warp releases a page last re-arms it
// with the page NP ahead (fast.cu).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace bfa {

enum FastKind : int32_t { FK_LEAF_IN = 0, FK_PAIR_DOWN = 1, FK_PAIR_UP = 2, FK_DIAG = 3, FK_LEAF_OUT = 4 };
constexpr int FAST_RANK = 16;                   // r: slab rows
constexpr int FAST_NB = 32;                     // right-hand sides per work item (slab columns)
constexpr int FAST_DMAX = 3;                    // window levels per pass (complex128)
constexpr int FAST_DMAX_C64 = 4;                // complex64: 16-slot windows fit next to the ring
constexpr int FAST_MAXOPS = 8;
constexpr int FAST_MAXPEER = 8;                 // ranks the fused peer-memory exchange addresses
constexpr int FAST_SLAB = FAST_RANK * FAST_NB;  // complex entries per slab (512)
constexpr int FAST_HC = 16;                     // rhs columns per half slab (one pass CTA's share)
constexpr int FAST_HSLAB = FAST_RANK * FAST_HC; // complex entries per half slab (256)
constexpr int FAST_NCONS = 16;                  // warps of the pass kernel (no producer warp)
constexpr int FAST_NCONS_HALF = 8;              // ... per 16-column half
constexpr int FAST_THREADS = FAST_NCONS * 32;
constexpr int FAST_FRAG = 1024;                 // bytes of A operand per (k-step, slot)
constexpr int LEAF_NCONS = 8;                   // warps of the leaf kernels (each owns whole items)
constexpr int LEAF_THREADS = LEAF_NCONS * 32;

struct FastOp {
  int32_t kind;
  int32_t s;       // window level: input level of PAIR_DOWN, output level of PAIR_UP, level of DIAG / leaves
  int32_t leaf;    // leaf size (LEAF_IN: K; LEAF_OUT: M)
  int32_t nsteps;  // MMA k-steps (LEAF_OUT: (leaf/16) x (16/KS), row-group major)
  int64_t off;     // byte offset of this op's factor stream inside a window record
};

struct FastPass {
  int32_t d, L, l0, bbits;  // window levels, tree depth, first level, log2(#b values) = L - l1
  int32_t nops, in_s, out_s, leaf;  // leaf: 0 window pass, 1 leaf-in launch, 2 leaf-out launch
  int32_t numaj, xin;               // HBM slab order: 0 tau-major (op N), 1 nu-major (op C / T);
                                    // xin / xout: 0 slab buffer, 1 / 2 exchange layout whose
  int32_t xout, xleaf;              // peer is the owner of tau / of nu (multi-GPU split);
                                    // xleaf: op 0 is the column leaf reading X (no window input)
  int32_t a_log, b_log;  // the pass's windows: a = a_lo + (w >> b_log), b = b_lo + (w & (2^b_log - 1))
  int32_t wt_log, wn_log;  // exchange: centre tau / nu per peer = 2^(lc - p) / 2^(L - lc - p)
  int64_t a_lo, b_lo;
  int64_t yleaf_lo;          // fused leaf-out: global index of the first leaf of the local Y rows
  int64_t fbase, win_bytes;  // byte offset of window 0's record, bytes per window record
  int64_t nwin;              // 2^(a_log + b_log)
  int64_t factor_entries, user_in, user_out;  // accounting
  FastOp ops[FAST_MAXOPS];
};

struct FastArgs {
  CUtensorMap xmap;       // xleaf pass: 2-D map over X, box = SPL*KS rows x 32 columns
  FastPass p;
  const void* X;          // xleaf pass: user block read
  const int64_t* xperm;   // tree position -> user row (contiguous leaves: only the first row used)
  const void* F;
  const void* Sin;
  void* Sout;
  void* Y;                // fused leaf-out op (last op FK_LEAF_OUT): user block written
  int64_t ldy;
  const int64_t* yperm;   // tree position -> user row (NULL = identity)
  int32_t conj_io;        // op T: conjugate Y on store
  int32_t ycontig;        // every leaf is a run of consecutive user rows
  int64_t nlev;  // slabs per level (2^L)
  int32_t nrhs;
  int32_t ntiles;  // 32-column rhs tiles (exchange layout stride)
  int32_t skew;  // ns the second column half starts late (tuning knob, env BF_FAST_SKEW)
  int32_t halves;  // column halves with work: 2; 1 when nrhs <= 16; 0 = one 8-column tile (nrhs <= 8)
  int32_t p2p;   // xout pass: write each slab straight into its receiver's recv region
  int32_t myrank;
  void* peer[FAST_MAXPEER];  // p2p: every rank's recv-region base (peer memory over NVLink)
  int32_t no_pairw;  // 4-level complex64 passes: one slot per k-loop (env BF_NO_PAIRW, A/B of PAIRW)
  int32_t diag;  // profiling only (env BF_FAST_DIAG, results are garbage): bit 0 = no operand
                 // streaming (compute only), bit 1 = output slabs not written to HBM, bit 2 = no
                 // intermediate epilogue / barriers, bit 3 (with 2) = epilogue stores, no barriers
};

// Leaf launch: item = (leaf, 32-column tile).  Slab `leaf` of the HBM slab buffer is the leaf's
// intermediate (both directions: the leaf level's canonical index equals the leaf index).
struct LeafArgs {
  CUtensorMap map;       // TMA map over X (mode 0) when tma != 0
  const void* F;         // leaf records: leaf i at F + i * nsteps KB
  const void* X;         // mode 0: user block read
  int64_t ldx;
  const int64_t* xperm;  // tree position -> user row (NULL = identity)
  void* Y;               // mode 1: user block written
  int64_t ldy;
  const int64_t* yperm;
  const void* Sin;       // mode 1: slabs read
  void* Sout;            // mode 0: slabs written
  int64_t nleaf, nlev;
  int64_t leaf_lo;       // global index of local leaf 0 (its slab index); X / Y rows are local
  int32_t leaf, nsteps;  // leaf size, k-steps per leaf record
  int32_t nrhs, conj_io; // conj_io: op T conjugates X on load and Y on store
  int32_t mode, tma;     // mode 0 = IN, 1 = OUT; tma: X rows by 2-D TMA (contiguous leaves)
  int32_t npairs, nst;   // concurrent items (item-owning warps), smem stages (npairs x depth)
  int32_t brows, diag;   // chunk rows (IN: leaf rows per stage = TMA box rows; OUT: output rows)
  int64_t stage_bytes, a_bytes;
};

void launch_fast_pass(int dtype, const FastArgs& a, cudaStream_t st);
const char* fast_kernel_name(int dtype);
// returns false when the leaf launch cannot be configured (shared memory)
void launch_leaf(int dtype, LeafArgs& a, cudaStream_t st);
// 2-D TMA map over a column-major (rows x nrhs, ld) complex block, box = brows x 32 (false when
// the block's base / stride are not 16-byte aligned)
bool fast_make_xmap(int dtype, const void* X, int64_t rows, int64_t nrhs, int64_t ld, int brows, CUtensorMap* map);
const char* leaf_kernel_name(int dtype, int mode);

// k-steps per MMA along K: complex128 DMMA m8n8k4 -> 4, complex64 TF32 m16n8k8 -> 8
__host__ __device__ inline int fast_ks(int csize) { return csize == 16 ? 4 : 8; }

// k-steps per ring page of the fused column-leaf op: each step carries S A records and the S
// slots' X rows (KS rows x 32 columns each) of a 32 KB page
__host__ __device__ constexpr int fast_spl(int csize, int S) { return 32768 / (S * (1024 + (csize == 16 ? 4 : 8) * 32 * csize)); }

__host__ __device__ inline int fast_nsteps(int kind, int leaf, int ks) {
  switch (kind) {
    case FK_LEAF_IN: return leaf / ks;
    case FK_LEAF_OUT: return (leaf / 16) * (16 / ks);
    case FK_PAIR_DOWN:
    case FK_PAIR_UP: return 2 * FAST_RANK / ks;
    default: return FAST_RANK / ks;
  }
}

// HBM ping-pong slab buffers: [rhs tile jt][column half][slab index][16 rows x 16 columns], each
// half slab laid out like the shared-memory copies (complex128: element (r, c) at
// r * 16 + (c ^ swz(r)); complex64: the MMA-fragment order of mma.cuh PolC64T).
__host__ __device__ inline int64_t half_slab_off(int64_t jt, int half, int64_t nlev, int64_t idx) {
  return ((jt * 2 + half) * nlev + idx) * FAST_HSLAB;
}

// slab index of block (tau, nu) at level l in the HBM ping-pong buffers: tau-major for op N,
// nu-major for op C / T, so that the S slabs a window reads at its input level are contiguous
// (one bulk copy) in both directions.
__host__ __device__ inline int64_t slab_index(const FastPass& P, int64_t a, int64_t b, int s, int slot) {
  const int ds = P.d - s, l = P.l0 + s;
  const int64_t tau = (a << s) + (slot >> ds);
  const int64_t nu = (b << ds) + (slot & ((1 << ds) - 1));
  return P.numaj ? (nu << l) + tau : (tau << (P.L - l)) + nu;
}

// element offset of the half slab (jt, half) of window (a, b)'s slot at window level s, in
// the slab buffer (mode 0) or in the exchange layout of the centre level (mode 1 / 2: peer =
// owner of tau / of nu): [peer][jt][half][tau_l][nu_l] for op N, [peer][jt][half][nu_l][tau_l]
// for op C, so the 2^d slabs a receiving window reads are contiguous again.
// With chunk >= 0 the chunk index is given (the sender's rank when it writes straight into a
// receiver's recv region) instead of the peer; *peer_out returns the peer.
__host__ __device__ inline int64_t pass_slab_off(const FastPass& P, int mode, int64_t jt, int half, int64_t nlev,
                                                 int64_t ntiles, int64_t a, int64_t b, int s, int slot,
                                                 int chunk = -1, int* peer_out = nullptr) {
  if (mode == 0) return half_slab_off(jt, half, nlev, slab_index(P, a, b, s, slot));
  const int ds = P.d - s;
  const int64_t tau = (a << s) + (slot >> ds);
  const int64_t nu = (b << ds) + (slot & ((1 << ds) - 1));
  const int64_t wt = int64_t(1) << P.wt_log, wn = int64_t(1) << P.wn_log;
  const int64_t tl = tau & (wt - 1), nl = nu & (wn - 1);
  int64_t peer = mode == 1 ? (tau >> P.wt_log) : (nu >> P.wn_log);
  if (peer_out) *peer_out = (int)peer;
  if (chunk >= 0) peer = chunk;
  const int64_t inner = P.numaj ? nl * wt + tl : tl * wn + nl;
  return (((peer * ntiles + jt) * 2 + half) * (wt * wn) + inner) * FAST_HSLAB;
}

}  // namespace bfa
