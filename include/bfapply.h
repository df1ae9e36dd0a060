/*
 * bfapply.h -- C-ABI of libbfapply: multi-RHS application of butterfly and HOD-BF
 * compressed matrices on NVIDIA B200 (sm_100a).
 *
 * What is applied (PAPER.md = arxiv 2007.00202, cited as P:<line>):
 *   * a butterfly K(O,S) in the factored ("hybrid") form of Eq. (3.3)
 *         K = (U^L R^{L-1} ... R^{lc}) B^{lc} (W^{lc} ... W^1 V^0),
 *     with the block structure of P:322-354 and the nested bases of Eq. (3.2)
 *     (P:302-317); "storage and application costs ... scale as O(n log n)";
 *   * an HOD-BF matrix: dense leaf diagonal blocks D_tau plus, for every
 *     pair of siblings tau1, tau2 of T_H, the butterflies A(T_tau1, T_tau2) and
 *     A(T_tau2, T_tau1); O(n log^2 n) to apply.
 * to a block of nrhs right-hand sides, forward (K X) or conjugate-transposed (K^H X).
 *
 * Indexing (same as bfinputs/factors.py and DESIGN.md):
 *   level l in [0, L]; block (tau, nu) pairs tau, a level-l node of T_O, with nu, a
 *   level-(L-l) node of T_S, both numbered left to right; children of x are 2x, 2x+1.
 *   Canonical block order within a level: idx = tau * 2^(L-l) + nu.
 *   Row ranks  r^l_{tau,nu}, l = lc..L   (r^L_{tau,0} = columns of U_tau)
 *   Col ranks  c^l_{tau,nu}, l = 0..lc   (c^0_{0,nu} = rows of Vt_nu)
 *   Factor block shapes (ranks may differ per block, B may be rectangular):
 *     U_tau      : m_tau x r^L_{tau,0}
 *     R_{tau,nu} : (r^{l+1}_{2tau,nu>>1} + r^{l+1}_{2tau+1,nu>>1}) x r^l_{tau,nu}, l = lc..L-1
 *     B_{tau,nu} : r^{lc}_{tau,nu} x c^{lc}_{tau,nu}
 *     W_{tau,nu} : c^l_{tau,nu} x (c^{l-1}_{tau>>1,2nu} + c^{l-1}_{tau>>1,2nu+1}), l = 1..lc
 *     Vt_nu      : c^0_{0,nu} x n_nu        (stored as it multiplies; never conjugated)
 *   Each factor array holds its blocks column-major, back to back, levels ascending and
 *   blocks in canonical order within a level.  Complex numbers are interleaved
 *   (re, im) -- the layout of torch.complex64 / complex128 and numpy complex64/128.
 *
 * Right-hand sides / results are column-major with a leading dimension (BLAS
 * convention): element (i, j) of X is X[i + j*ldx].  A C-contiguous torch tensor of
 * shape (nrhs, n) is exactly that layout with ldx = n.
 *
 * Ownership: *_create deep-copies every host array to the device (the caller may
 * free them on return); the handle owns that device memory until *_destroy.  X, Y and
 * the workspace of *_apply are caller-owned DEVICE buffers; the apply makes no
 * allocation, no host synchronisation and launches only on the given stream.
 * Handles are immutable after create: concurrent applies on different streams with
 * distinct workspaces are legal.  A handle is bound to one device.
 *
 * Errors: every entry point returns a bf_status; no exception crosses the ABI.  A
 * thread-local message is available from bf_last_error().  Asynchronous CUDA faults
 * surface as BF_ERR_CUDA on a later call.  There is no CPU fallback: without a CUDA
 * device every create/apply returns BF_ERR_DEVICE.
 */
#ifndef BFAPPLY_H
#define BFAPPLY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bf_s* bf_handle;
typedef struct hodbf_s* hodbf_handle;
typedef void* bf_stream_t; /* a cudaStream_t; NULL = legacy default stream */

typedef enum { BF_C64 = 1, BF_C128 = 2 } bf_dtype;

/* N: Y = K X.  C: Y = K^H X (conjugate transpose, the north-star "adjoint").
 * T: Y = K^T X (plain transpose, SPEC's A^T X). */
typedef enum { BF_OP_N = 0, BF_OP_T = 1, BF_OP_C = 2 } bf_op;

typedef enum {
  BF_OK = 0,
  BF_ERR_ARG = -1,    /* NULL / negative argument, X and Y overlap, workspace too small   */
  BF_ERR_SHAPE = -2,  /* leaf offsets not monotone / not summing to m, n; L out of range  */
  BF_ERR_RANK = -3,   /* negative rank, or factor lengths inconsistent with the ranks     */
  BF_ERR_PERM = -4,   /* a permutation is not a bijection                                 */
  BF_ERR_CUDA = -5,   /* a CUDA runtime error (including earlier asynchronous faults)     */
  BF_ERR_OOM = -6,    /* device allocation failed                                         */
  BF_ERR_NCCL = -7,   /* distributed layout not supported for this rank count             */
  BF_ERR_DEVICE = -8  /* no CUDA device / wrong device / not an sm_100 device             */
} bf_status;

/* bf_desc.flags.  BF_CREATE_FUSED_ONLY: when the butterfly runs on the fused kernels (uniform
 * power-of-two leaves of 16-256, ranks <= 16), keep only their per-op factor records and release
 * the generic factor pool after create -- two copies of the factors on the device instead of
 * three (config 5 complex128: 4.96 instead of 7.45 GB).  bf_extract / bf_extract_list and
 * bf_export's factor copies then return BF_ERR_ARG.  No effect on other butterflies. */
typedef enum { BF_CREATE_FUSED_ONLY = 1 } bf_create_flags;

/* Butterfly descriptor.  All pointers are HOST pointers. */
typedef struct {
  int32_t dtype;                 /* bf_dtype                                                  */
  int32_t L;                     /* number of levels, 0 <= L <= 30                           */
  int32_t lc;                    /* centre level, 0 <= lc <= L; pass -1 for floor(L/2) (A2)  */
  int32_t flags;                 /* bf_create_flags (0 = default)                            */
  int64_t m, n;                  /* rows (|O|) and columns (|S|)                             */
  const int64_t* row_leaf_ptr;   /* 2^L + 1 offsets of T_O leaves in tree order              */
  const int64_t* col_leaf_ptr;   /* 2^L + 1 offsets of T_S leaves                            */
  const int64_t* row_perm;       /* m: tree position -> user row; NULL = identity           */
  const int64_t* col_perm;       /* n: tree position -> user column; NULL = identity        */
  const int32_t* rank_row;       /* (L-lc+1) * 2^L: r^l_{tau,nu}, l = lc..L, canonical order  */
  const int32_t* rank_col;       /* (lc+1) * 2^L:   c^l_{tau,nu}, l = 0..lc                   */
  const void *U, *R, *B, *W, *Vt;/* packed factor arrays (see above)                          */
  int64_t len_U, len_R, len_B, len_W, len_Vt; /* element counts of the five arrays; must equal
                                                the counts implied by the ranks (BF_ERR_RANK) */
  /* Optional non-canonical block orderings ("level-by-level index permutations", north star;
   * SURVEY 8(b)).  NULL = every level canonical.  Otherwise L + 1 pointers; entry l (NULL =
   * canonical) is a 2^L int32 bijection  storage slot s -> canonical index tau * 2^(L-l) + nu
   * of level l.  It orders everything stored per level-l block: the level-l ranks (rank_row
   * if l >= lc, rank_col if l <= lc) and the level-l factor blocks (U at l = L, R at
   * lc <= l < L, B at l = lc, W at 1 <= l <= lc, Vt at l = 0), which are then packed in slot
   * order.  Leaf offsets and perms are unaffected.  Not a bijection: BF_ERR_PERM.  The
   * library re-packs to canonical order at create (host copy; the apply is unchanged). */
  const int32_t* const* level_maps;
} bf_desc;

/* HOD-BF descriptor.  offdiag has sum_{l=1..LH} 2^l entries, level-major:
 * entry (l, tau) at index 2^l - 2 + tau is the butterfly of A(T_tau, T_{tau^1}) with
 * L = LH - l levels, tree-local (NULL) perms, and leaf offsets equal to leaf_ptr's
 * slices for T_tau (rows) and T_{tau^1} (columns), rebased to 0. */
typedef struct {
  int32_t dtype;
  int32_t LH;                    /* HOD-BF levels, 0 <= LH <= 20                             */
  int64_t n;
  const int64_t* leaf_ptr;       /* 2^LH + 1 offsets of T_H leaves (tree order)              */
  const int64_t* perm;           /* n: tree position -> user index; NULL = identity          */
  const void* D;                 /* 2^LH dense leaf blocks, column-major, back to back       */
  int64_t len_D;
  const bf_desc* offdiag;
} hodbf_desc;

/* Run-time information about a handle (for benchmarks / roofline accounting). */
typedef struct {
  int64_t factor_entries;        /* stored complex factor entries (algorithmic)               */
  int64_t device_bytes;          /* device memory owned by the handle                        */
  int32_t launches_n;            /* kernel launches per apply, op N                          */
  int32_t launches_c;            /* kernel launches per apply, op C / T                      */
  int64_t rows_in, rows_out;     /* rows of X and Y for op N (n, m)                          */
} bf_info_t;

/* ---- butterfly --------------------------------------------------------------------- */
int bf_create(const bf_desc* desc, int device, bf_handle* out);
int bf_destroy(bf_handle h);
int bf_info(bf_handle h, bf_info_t* info);
/* Bytes of device workspace one apply with `nrhs` columns needs (any op). */
int bf_workspace_size(bf_handle h, int64_t nrhs, size_t* bytes);
/* Y (m x nrhs) <- K X (X: n x nrhs).  The byte ranges of X and Y (first to last element) must
 * not overlap (BF_ERR_ARG); Y is overwritten (beta = 0). */
int bf_apply(bf_handle h, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
             void* work, size_t work_bytes, bf_stream_t stream);
/* Y (n x nrhs) <- K^H X (X: m x nrhs). */
int bf_apply_adj(bf_handle h, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
                 void* work, size_t work_bytes, bf_stream_t stream);
/* General form; bf_apply / bf_apply_adj are op N / op C. */
int bf_apply_op(bf_handle h, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y,
                int64_t ldy, void* work, size_t work_bytes, bf_stream_t stream);
/* End-to-end form with HOST X / Y (pinned for full speed): H2D copy of X, apply, D2H copy
 * of Y.  Y_host is complete once the caller synchronises `stream`; X_host must stay unchanged
 * until then.  The copies and the apply run on three streams owned by the handle and
 * consecutive calls alternate between two sets of device X / Y copies, so call k+1's H2D and
 * apply overlap call k's D2H (the two PCIe directions are independent); calls on one handle are
 * serialised (internal lock); on the first call, and when op, nrhs or the workspace change, the
 * pipeline also waits for the caller's earlier work on `stream`.  The workspace must be at least bf_workspace_size_host bytes (it also holds the two
 * sets of device copies) and the same workspace must be passed to consecutive calls. */
int bf_workspace_size_host(bf_handle h, int op, int64_t nrhs, size_t* bytes);
int bf_apply_host(bf_handle h, int op, int64_t nrhs, const void* X_host, int64_t ldx,
                  void* Y_host, int64_t ldy, void* work, size_t work_bytes, bf_stream_t stream);

/* ---- HOD-BF ------------------------------------------------------------------------ */
int hodbf_create(const hodbf_desc* desc, int device, hodbf_handle* out);
int hodbf_destroy(hodbf_handle h);
int hodbf_info(hodbf_handle h, bf_info_t* info);
int hodbf_workspace_size(hodbf_handle h, int64_t nrhs, size_t* bytes);
/* Y (n x nrhs) <- A X, A^T X or A^H X. */
int hodbf_apply(hodbf_handle h, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y,
                int64_t ldy, void* work, size_t work_bytes, bf_stream_t stream);
/* hodbf_apply_host: as bf_apply_host (same three-stream pipeline; workspace from
 * hodbf_workspace_size_host, the same one passed to consecutive calls). */
int hodbf_workspace_size_host(hodbf_handle h, int64_t nrhs, size_t* bytes);
int hodbf_apply_host(hodbf_handle h, int op, int64_t nrhs, const void* X_host, int64_t ldx,
                     void* Y_host, int64_t ldy, void* work, size_t work_bytes,
                     bf_stream_t stream);

/* ---- distributed butterfly (one process per GPU) ------------------------
 * P = nranks = 2^p GPUs, p <= min(lc, L - lc).  Rank g owns the column subtree nu_g at
 * level p of T_S (its V leaves, W stages and B blocks) and the row subtree tau_g at level p
 * of T_O (its R stages and U leaves).  Forward: X_loc = rows of X in S_{nu_g}, Y_loc = rows
 * of Y in O_{tau_g}; adjoint: the other way round.  Local rows are in user order restricted
 * to the subtree, which must map to a contiguous user range (else BF_ERR_PERM).
 * An apply is  pre -> all-to-all of the centre slabs -> post:
 *   bf_dist_apply_pre  writes the send region of `work` (slabs grouped by destination);
 *   the caller exchanges send -> recv with an all-to-all (NCCL) using bf_dist_layout;
 *   bf_dist_apply_post reads the recv region and writes Y_loc.
 * `desc` is the FULL descriptor (every rank passes the same); only the rank's blocks are
 * uploaded.  nranks = 1 runs the same path with a self exchange.
 * device < 0 builds a HOST-ONLY plan: layouts, local rows and the exchange block maps can be
 * queried (multi-process CPU tests of the exchange logic), nothing is uploaded, and
 * bf_dist_apply_pre / _post return BF_ERR_DEVICE. */
int bf_dist_create(const bf_desc* desc, int rank, int nranks, int device, bf_handle* out);
/* Workspace bytes, and the send/recv regions: byte offsets into work plus per-peer
 * ELEMENT counts (complex entries) -- arrays of length nranks.  Op selects N or C/T. */
int bf_dist_layout(bf_handle h, int op, int64_t nrhs, size_t* work_bytes, size_t* send_off,
                   size_t* recv_off, int64_t* send_counts, int64_t* recv_counts);
/* The centre blocks (canonical index tau * 2^(L-lc) + nu at level lc) in the
 * order their slabs occupy the send and the recv region (grouped by peer, peers ascending).
 * Each block occupies rank x nrhs elements (op N: r^lc, op C / T: c^lc).  Pass NULL arrays to
 * query only the counts. */
int bf_dist_exchange_blocks(bf_handle h, int op, int64_t* n_send, int64_t* send_blocks, int64_t* n_recv,
                            int64_t* recv_blocks);
/* Element layout of the send / recv regions.  0: every centre block occupies rank x nrhs
 * consecutive elements (row-major, nrhs fastest) in bf_dist_exchange_blocks order.  1 (uniform
 * rank-16 butterflies, fused kernels): each peer's chunk is [rhs tile of 32][column half of 16]
 * [block, in bf_dist_exchange_blocks order][16 rows][16 columns], the 16 x 16 half slab stored
 * in the kernels' half-slab layout (complex128: element (r, c) at r*16 + (c ^ swz(r)); complex64:
 * MMA-fragment order [r/8][re | im][lane][4] floats, see mma.cuh PolC64T); nrhs is padded to a
 * multiple of 32.  Either way the regions are moved as opaque bytes by the all-to-all. */
int bf_dist_slab_format(bf_handle h, int32_t* fmt);
/* The level whose slabs the split exchanges: lc for the generic split; for the fused split the
 * level in [log2 nranks, L - log2 nranks] that minimises the window passes (plan.cu
 * split_exchange_level; config 5 complex128: 6).  bf_dist_exchange_blocks' block indices are
 * canonical indices at this level. */
int bf_dist_exchange_level(bf_handle h, int op, int32_t* level);

int bf_dist_local_rows(bf_handle h, int op, int64_t* rows_in, int64_t* rows_out,
                       int64_t* user_off_in, int64_t* user_off_out);
int bf_dist_apply_pre(bf_handle h, int op, int64_t nrhs, const void* X_loc, int64_t ldx,
                      void* work, size_t work_bytes, bf_stream_t stream);
/* Fused exchange (bf_dist_slab_format 1 only): like bf_dist_apply_pre, but the pass that
 * ends at the centre level stores each slab straight into its receiver's recv region over peer
 * memory (NVLink / NVSwitch) while it computes -- no send region, no all-to-all.  peer_recv[q]
 * (host array of nranks device pointers) is rank q's recv-region base as mapped in this
 * process (e.g. torch symmetric memory, CUDA IPC); this rank's chunk in it is at the offset
 * its own bf_dist_layout recv region has for source `rank`.  The caller then synchronises the
 * ranks (every sender done) before bf_dist_apply_post, and again before the next pre writes
 * into the recv regions. */
int bf_dist_apply_pre_p2p(bf_handle h, int op, int64_t nrhs, const void* X_loc, int64_t ldx,
                          void* work, size_t work_bytes, void* const* peer_recv, bf_stream_t stream);
int bf_dist_apply_post(bf_handle h, int op, int64_t nrhs, void* Y_loc, int64_t ldy,
                       void* work, size_t work_bytes, bf_stream_t stream);

/* ---- distributed apply with a library-owned NCCL communicator (SURVEY 8(b) stretch goal;
 * north star: "the middle-level redistribution is an NCCL all-to-all over NVLink") ----------
 * NCCL is loaded at run time (dlopen "libnccl.so.2", env BF_NCCL_LIB overrides; inside a
 * PyTorch process that is the NCCL torch already loaded); when it cannot be loaded these calls
 * return BF_ERR_NCCL.
 *   bf_nccl_available     1 when NCCL is loadable, else 0.
 *   bf_nccl_get_unique_id writes the 128-byte ncclUniqueId (call on one rank, send the bytes to
 *                         every rank by any means, e.g. torch.distributed.broadcast).
 *   bf_nccl_comm_init     ncclCommInitRank on `device` (collective over the nranks processes);
 *                         *comm is an ncclComm_t owned by the caller: free it with
 *                         bf_nccl_comm_destroy after every handle using it is destroyed.
 *   bf_create_dist        bf_dist_create plus the communicator (checked: its size / rank /
 *                         device equal nranks / rank / device; NULL only when nranks == 1 or
 *                         device < 0).  The handle does not own the communicator.
 *   bf_apply_dist         one whole distributed apply on `stream`: bf_dist_apply_pre, the
 *                         exchange of the send region's per-peer chunks into every peer's
 *                         recv region (grouped ncclSend / ncclRecv; one rank: a device copy),
 *                         bf_dist_apply_post.  Arguments as bf_dist_apply_pre / _post (X_loc,
 *                         Y_loc and work are device buffers; work >= bf_dist_layout's
 *                         work_bytes).  Every rank must call it with the same op and nrhs. */
int bf_nccl_available(void);
int bf_nccl_get_unique_id(void* id);
int bf_nccl_comm_init(int nranks, const void* id, int rank, int device, void** comm);
int bf_nccl_comm_destroy(void* comm);
int bf_create_dist(const bf_desc* desc, int rank, int nranks, void* nccl_comm, int device, bf_handle* out);
int bf_apply_dist(bf_handle h, int op, int64_t nrhs, const void* X_loc, int64_t ldx, void* Y_loc, int64_t ldy,
                  void* work, size_t work_bytes, bf_stream_t stream);

/* Sub-matrix extraction (Alg. 3 extract_BF): out(i, j) =
 * K(rows[i], cols[j]) for user row / column indices (HOST arrays of nI / nJ int64, any order,
 * repeats allowed), out a DEVICE column-major nI x nJ block with ldo >= nI.  Computed as a
 * partial matvec: K E_J on the blocks (l, tau, nu) whose tau is an ancestor of a requested
 * row's leaf and whose nu is an ancestor of a requested column's leaf, then the requested rows.
 * Each touched block's slab holds only the requested columns under its column node (the columns
 * in tree order form one range per node), so a W / R block is one product per touched child at
 * that child's width: every block multiplied once.  Single-device handles only
 * (BF_ERR_ARG for a bf_dist handle).  Synchronous: uses a grow-only scratch of the handle and
 * returns after the work on `stream` completed.  BF_ERR_ARG on out-of-range indices or NULL
 * arguments. */
int bf_extract(bf_handle h, int64_t nI, const int64_t* rows, int64_t nJ, const int64_t* cols, void* out,
               int64_t ldo, bf_stream_t stream);

/* Alg. 3's list form: K(I_k, J_k) for every request k of a list, evaluated together
 * (one launch per stage for all requests; each request's touched blocks multiplied once, at the
 * width of its columns under the block's column node).  Request k: nI[k] rows rows[k][...] and
 * nJ[k] columns cols[k][...] (HOST user indices), result into the DEVICE block out[k] (column-major,
 * leading dimension ldo[k] >= nI[k]).  Synchronous on `stream`.  Errors as bf_extract. */
int bf_extract_list(bf_handle h, int64_t npairs, const int64_t* nI, const int64_t* const* rows, const int64_t* nJ,
                    const int64_t* const* cols, void* const* out, const int64_t* ldo, bf_stream_t stream);

/* HOD-BF sub-matrix extraction (extract_HODBF): out(i, j) =
 * A(rows[i], cols[j]) for user indices, as bf_extract: the entries inside one leaf from D_t,
 * every other one from the sibling butterfly of the level where the row's and the column's
 * tree nodes split, each butterfly's share as a partial matvec over its touched blocks.
 * Same arguments, errors and synchronous behaviour as bf_extract. */
int hodbf_extract(hodbf_handle h, int64_t nI, const int64_t* rows, int64_t nJ, const int64_t* cols, void* out,
                  int64_t ldo, bf_stream_t stream);

/* Y += A on a column-major rows x nrhs complex block (device pointers, ld >= rows): the sum of
 * the HOD-BF contributions of a tree-partitioned apply ("Y(T_tau) += B_tau X(...)"; the
 * row-side posts of the off-diagonal butterflies at the distributed levels write a scratch block
 * that this adds into the rank's local result).  A and Y must not overlap.  BF_ERR_ARG on NULL
 * pointers, a negative size, ld < rows or an unknown dtype; an asynchronous launch on `stream`. */
int bf_accumulate(int dtype, int64_t rows, int64_t nrhs, const void* A, int64_t lda, void* Y, int64_t ldy,
                  bf_stream_t stream);

/* ---- introspection / in-situ timing ------------------------------------------------------
 * An apply is a fixed sequence of kernel launches ("rounds").  bf_round_info describes round
 * `round` of op `op`: the kernel variant, the number of independent block products, and the
 * algorithmic traffic of that round (factor entries read once; user rows of X read / of Y
 * written; slab rows produced).  *_apply_events records events[i] on `stream` right before
 * round i and events[nrounds] after the last one (nevents must be >= nrounds + 1; the events
 * are caller-created cudaEvent_t handles), so a caller can time every round inside its own
 * timed region. */
typedef struct {
  int32_t kernel;                /* kernel variant id (see name)                             */
  int32_t ntasks;                /* independent output slabs in the launch                   */
  int64_t factor_entries;        /* factor entries the round reads                           */
  int64_t user_rows_in;          /* rows of X read (leaf rounds)                             */
  int64_t user_rows_out;         /* rows of Y written (leaf rounds)                          */
  int64_t slab_rows_in;          /* intermediate slab rows read                              */
  int64_t slab_rows_out;         /* intermediate slab rows written                           */
  char name[48];
} bf_round_info_t;
int bf_rounds(bf_handle h, int op, int32_t* nrounds);
int bf_round_info(bf_handle h, int op, int32_t round, bf_round_info_t* info);
int bf_apply_op_events(bf_handle h, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y,
                       int64_t ldy, void* work, size_t work_bytes, bf_stream_t stream,
                       void* const* events, int32_t nevents);
int hodbf_rounds(hodbf_handle h, int op, int32_t* nrounds);
int hodbf_round_info(hodbf_handle h, int op, int32_t round, bf_round_info_t* info);
int hodbf_apply_events(hodbf_handle h, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y,
                       int64_t ldy, void* work, size_t work_bytes, bf_stream_t stream,
                       void* const* events, int32_t nevents);

/* ---- misc ---------------------------------------------------------------------------- */
/* Copy a single-GPU handle's factors back to HOST arrays in the bf_desc layout (levels and blocks in
 * canonical order, column-major blocks).  lens[5] receives the element counts of U, R, B, W, Vt;
 * rank_row ((L-lc+1) 2^L) and rank_col ((lc+1) 2^L) the ranks; any pointer may be NULL.  The
 * trees (leaf offsets, perms) are the ones the handle was created with.  Synchronous. */
int bf_export(bf_handle h, int64_t* lens, int32_t* rank_row, int32_t* rank_col, void* U, void* R, void* B,
              void* W, void* Vt);

/* ---- randomized matrix-free construction (BF_random_matvec) ------------------------------
 * PAPER.md Sec. 3.3: a butterfly built from multi-RHS products with an operator A that
 * is available only as a matvec; O(sqrt(n)) sketch columns of an O(n log n) matvec.  Its consumer
 * is the Schur-complement construction of Alg. 5 and the HOD-BF inversion of Alg. 4
 * (P:576-612).  The trees (leaf offsets and perms) of the result are the caller's; ranks come from
 * interpolative decompositions of Gaussian sketches, truncated at relative tolerance
 * eps, capped at rank_max (the sketch width is rank_max + oversample per block).  The algorithm
 * (level-by-level peeling) runs on the device: sketch generation, the
 * gathers, a batched column-pivoted QR per block and the centre least-squares solves are library
 * kernels; only the small per-block results (ranks, pivots, interpolation matrices) pass through
 * the host to be packed into the result's descriptor, which is then bf_create'd on `device`.
 *
 * The operator is a callback: fn(ctx, op, nrhs, X, ldx, Y, ldy, stream) must write
 * Y = A X (op BF_OP_N: X n x nrhs, Y m x nrhs) or Y = A^H X (op BF_OP_C: X m x nrhs, Y n x nrhs),
 * column-major DEVICE blocks in user order, ordered on `stream`, and return BF_OK.  bf_operator_apply
 * below is such a callback for sums of products of library handles.  Synchronous: the call
 * returns with the result built (it synchronises `stream`).  Errors: BF_ERR_ARG (bad descriptor,
 * callback failure), BF_ERR_SHAPE / BF_ERR_PERM (trees), BF_ERR_CUDA, BF_ERR_OOM. */
typedef int (*bf_matvec_fn)(void* ctx, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
                            bf_stream_t stream);
typedef struct {
  int32_t dtype;                 /* bf_dtype of the result and of the sketches                   */
  int32_t L, lc;                 /* levels and centre level of the result (lc < 0: floor(L/2))   */
  int32_t rank_max;              /* rank cap per block                                           */
  int64_t m, n;                  /* A is m x n                                                   */
  const int64_t* row_leaf_ptr;   /* 2^L + 1 offsets of T_O leaves (tree order)                   */
  const int64_t* col_leaf_ptr;   /* 2^L + 1 offsets of T_S leaves                                */
  const int64_t* row_perm;       /* tree position -> user row; NULL = identity                  */
  const int64_t* col_perm;       /* tree position -> user column; NULL = identity               */
  double eps;                    /* relative ID truncation |R_jj| <= eps |R_11|                  */
  int32_t oversample;            /* extra sketch columns per block (>= 0; 8-16 typical)          */
  int32_t reserved;
  uint64_t seed;                 /* counter-based Gaussian sketches: same seed, same result      */
  size_t chunk_bytes;            /* device budget of one sketch block + its product (0: 1 GiB)   */
} bf_rmv_desc;
typedef struct {
  int64_t matvec_cols_n;         /* columns applied through A (op N)                             */
  int64_t matvec_cols_c;         /* columns applied through A^H (op C)                           */
  int32_t max_rank;              /* largest block rank of the result                             */
  int32_t saturated;             /* blocks whose rank reached rank_max (sketch possibly too thin) */
  double t_matvec_ms;            /* device time inside the callback (CUDA events)                */
  double t_total_ms;             /* wall time of the whole construction                          */
} bf_rmv_stats;
int bf_random_matvec(const bf_rmv_desc* desc, bf_matvec_fn fn, void* ctx, int device, bf_stream_t stream,
                     bf_handle* out, bf_rmv_stats* stats);

/* The batched interpolative decomposition bf_random_matvec runs, exposed for reuse and testing:
 * nmat complex matrices, matrix i k x pcnt[i] column-major (ld k), packed back to back in the
 * DEVICE buffer M.  Each is factored in place by Householder QR with column pivoting (largest
 * remaining column norm, ties to the lowest index), stopped at rank r where |R_rr| <= eps |R_00|
 * or r = rmax.  Outputs (DEVICE): rank[i]; perm[sum_{j<i} pcnt[j] ..]
 * the column order (the first r are the skeleton columns); and, in rows 0..r-1 of the columns
 * r..pcnt[i]-1 of matrix i, T = R11^{-1} R12, so M(:, perm[r + j]) ~= sum_q M(:, perm[q]) T(q, j).
 * Synchronous. */
int bf_batched_id(int dtype, int64_t nmat, int32_t k, const int64_t* pcnt, void* M, double eps, int32_t rmax,
                  int32_t* rank, int32_t* perm, bf_stream_t stream);

/* Composite operators: A = sum_s alpha_s P_s, each product P_s = fac[nfac-1] ... fac[0] (fac[0]
 * applied first) mapping X rows [col_off, col_off + fac[0].cols) to Y rows [row_off, row_off +
 * fac[nfac-1].rows) of the m x n operator (block placement).  A factor is a butterfly or HOD-BF
 * handle with op BF_OP_N or BF_OP_C, or the identity; rows x cols is its shape as it appears.
 * bf_operator_apply(ctx = const bf_operator*) has the bf_matvec_fn signature: Y = A X (op N) or
 * A^H X (op C) on device blocks; it allocates its temporaries and synchronises `stream`. */
typedef enum {
  BF_FACTOR_BF = 0,              /* a butterfly handle, op N or C                                 */
  BF_FACTOR_HODBF = 1,           /* an HOD-BF handle                                              */
  BF_FACTOR_IDENTITY = 2,        /* I (rows == cols)                                              */
  BF_FACTOR_BF_PLUS_I = 3,       /* I + K for a square butterfly handle K                         */
  BF_FACTOR_SELECT = 4,          /* rows < cols: rows [aux0, aux0 + rows) of X; rows > cols: X     *
                                  * embedded at rows [aux0, aux0 + cols) of a zero block          */
  BF_FACTOR_HODBF_INV = 5,       /* A^{-1} of an HOD-BF inverse handle (user order)               */
  BF_FACTOR_HODBF_INV_NODE = 6   /* D_tau^{-1} of node (l = aux0, tau = aux1), tree order          */
} bf_factor_kind;
typedef struct {
  int32_t kind, op;
  void* handle;                  /* bf_handle / hodbf_handle / hodbf_inv_handle; NULL otherwise   */
  int64_t rows, cols;
  int64_t aux0, aux1;
} bf_factor;
typedef struct {
  double alpha_re, alpha_im;
  int32_t nfac, reserved;
  const bf_factor* fac;
  int64_t row_off, col_off;
} bf_product;
typedef struct {
  int32_t dtype, nprod;
  int64_t m, n;
  const bf_product* prod;
} bf_operator;
int bf_operator_apply(void* op, int opn, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
                      bf_stream_t stream);

/* ---- HOD-BF inversion (Alg. 4 HODBF_invert with BF_SMW) -------------------------
 * Builds A^{-1} of an HOD-BF matrix in the multiplicative form of Alg. 4 line 9: dense leaf inverses
 * (line 3) and, for every internal node tau of T_H, a butterfly K_tau over T_tau x T_tau with
 * (I + K_tau) = BF_SMW([I, B'_tau1; B'_tau2, I]) where B'_tau_i = BF_random_matvec(D_tau_i^{-1} B_tau_i)
 * (lines 7-8).  BF_SMW follows Alg. 4 on the node's child split (readings in DESIGN.md section 3);
 * nodes of at most dense_max rows are inverted densely (the low-rank / dense SMW base case).
 * Every compression is bf_random_matvec with (eps, rank_max, oversample).  The descriptor is the
 * hodbf_create one (host arrays, caller-owned).  Synchronous.  stats accumulates the constructions'
 * sketch columns and ranks.  Errors: as bf_random_matvec; BF_ERR_ARG for a singular leaf. */
typedef struct hodbf_inv_s* hodbf_inv_handle;
typedef struct {
  double eps;                    /* relative ID tolerance of every compression                     */
  int32_t rank_max, oversample;
  uint64_t seed;
  int64_t dense_max;             /* nodes with at most this many rows: dense inverse (0: leaves only) */
} bf_inv_opts;
int hodbf_invert(const hodbf_desc* desc, const bf_inv_opts* opts, int device, bf_stream_t stream,
                 hodbf_inv_handle* out, bf_rmv_stats* stats);
int hodbf_inv_destroy(hodbf_inv_handle h);
/* Y = A^{-1} X (op N) or A^{-H} X (op C); X, Y n x nrhs column-major DEVICE blocks in user order,
 * non-overlapping; work: hodbf_inv_workspace_size bytes of device memory.  Asynchronous on
 * `stream` (the product of the inverse's factors: one blocked dense-leaf launch and the node
 * butterflies' applies, level by level). */
int hodbf_inv_workspace_size(hodbf_inv_handle h, int64_t nrhs, size_t* bytes);
int hodbf_inv_apply(hodbf_inv_handle h, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
                    void* work, size_t work_bytes, bf_stream_t stream);
/* stored entries (dense leaf inverses + every K_tau's factors) and number of K_tau butterflies */
int hodbf_inv_info(hodbf_inv_handle h, int64_t* factor_entries, int32_t* nbutterflies);

/* ---- multifrontal solve-phase sweep (Alg. 1 line precGMRES) ---------------------------
 * An assembly tree of compressed fronts: front i has separator unknowns [s_off, s_off + s_len) of
 * the global N-vector (disjoint ranges), update unknowns u_idx (u_len distinct global indices held
 * by its ancestors), F11^{-1} as an HOD-BF inverse (s x s, its own user order = the separator's local
 * order), and F12 (s x u) / F21 (u x s) as butterflies.  Fronts are listed in topological order:
 * every front before its parent.  The handles are BORROWED: they must outlive the bf_mf handle.
 *   forward (children first): z_s = F11^{-1} y_s; y_u -= F21 z_s   (y starts as B)
 *   backward (root first):    x_s = z_s - F11^{-1} F12 x_u
 * bf_mf_solve writes X = M^{-1} B (N x nrhs, column-major DEVICE blocks, non-overlapping) with a
 * workspace of bf_mf_workspace_size bytes; asynchronous on `stream`, no allocation.  The fronts of
 * one height (forward) / depth (backward) run concurrently on streams owned by the handle, forked
 * from and joined back into `stream` (so the call is stream-ordered and graph-capturable);
 * concurrent solves on one handle are serialised (internal lock).  Results are deterministic. */
typedef struct bf_mf_s* bf_mf_handle;
typedef struct {
  int32_t parent, reserved;      /* parent front (-1: a root)                                      */
  int64_t s_off, s_len;
  int64_t u_len;
  const int64_t* u_idx;          /* host array, copied at create                                   */
  hodbf_inv_handle F11inv;
  bf_handle F12, F21;
} bf_front;
int bf_mf_create(int dtype, int64_t N, int32_t nfront, const bf_front* fronts, int device, bf_mf_handle* out);
int bf_mf_destroy(bf_mf_handle h);
int bf_mf_workspace_size(bf_mf_handle h, int64_t nrhs, size_t* bytes);
int bf_mf_solve(bf_mf_handle h, int64_t nrhs, const void* B, int64_t ldb, void* X, int64_t ldx, void* work,
                size_t work_bytes, bf_stream_t stream);

const char* bf_status_string(int status);
const char* bf_last_error(void);
/* Library version and the compile target, e.g. "bfapply 0.1 sm_100a". */
const char* bf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BFAPPLY_H */
