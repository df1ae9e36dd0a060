// Shared definitions of libbfapply (host + device).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdlib>
#include <stdint.h>

#include <string>
#include <vector>

#include "bfapply.h"

namespace bfa {

// error carried from deep inside the host logic to the C-ABI boundary
struct Err {
  int code;
  std::string msg;
};

// One product A * In that contributes to a task's output rows.
//   A(i, k) = pool[a_off + i * a_rs + k * a_cs]   (conjugated if conj ^ conj_flip)
//   In(k, :) = slab-space row (in_row + k)        when in_kind == 0
//            = X row perm[in_row + k]             when in_kind == 1 (user X, column-major)
struct Term {
  int64_t a_off;
  int64_t in_row;
  int32_t a_rs, a_cs;
  int32_t k;
  int16_t conj, in_kind;
};

// One output slab: rows [out_row, out_row + m) of the slab space (out_kind 0) or the user
// rows perm[out_row + i] of Y (out_kind 1) receive sum_t A_t In_t.
struct Task {
  int64_t out_row;
  int32_t m;
  int32_t term0;
  int32_t nterm;
  int32_t pad;
};

// One kernel launch of a plan (a "round": every task in it is independent).
struct Round {
  const Task* tasks;   // device
  const Term* terms;   // device
  const int2* units;   // device: (task, 32-row block) work units of the tensor-core kernel
  int32_t nunits;
  int32_t pad0;
  int32_t ntasks;
  int32_t out_kind;    // 0 slab space, 1 user Y
  int32_t max_m;
  int32_t max_k;
  int32_t fast;        // specialised kernel id (0 = generic)
  int32_t pad;
  const int2* cols;    // device, optional (bf_extract): per task the rhs-column range [x, y) it must
                       // produce -- column tiles outside it are skipped (they stay zero)
  // algorithmic accounting (host only)
  int64_t factor_entries, user_in, user_out, slab_in, slab_out;
};

struct StageArgs {
  const Task* tasks;
  const Term* terms;
  const void* pool;
  const void* X;
  int64_t ldx;
  const int64_t* xperm;
  void* S;
  int64_t ldS;
  void* Y;
  int64_t ldy;
  const int64_t* yperm;
  const int2* units;
  int32_t nunits;
  int32_t out_kind;
  int32_t conj_flip;
  int32_t nrhs;
  int32_t m3;  // 3M complex products (0: 4M, exact on selection factors)
  const int2* cols;  // Round::cols of the launched round (nullptr: every column tile)
};

void launch_round(int dtype, const Round& r, StageArgs a, cudaStream_t st);
// complex64 rounds on tcgen05 (tile_umma.cu): one CTA per (unit, 128-column rhs tile)
void launch_tile_umma(const StageArgs& a, cudaStream_t st);
// One product of the compact extraction (bf_extract, Alg. 3): out[out_off + i out_ld + j] (+ if acc)=
// sum_k pool[a_off + i a_rs + k a_cs] in[in_off + k in_ld + j], i < m, j < w, k < kk (row-major
// compact slabs, rmatvec.cu k_xprod)
struct XProd {
  int64_t a_off, in_off, out_off;
  int32_t a_rs, a_cs, m, kk, w, in_ld, out_ld, acc;
};
void launch_xprod(int dtype, int64_t np, const void* P, const void* pool, const void* S, void* O, cudaStream_t st);

// One butterfly's share of a level-wise extraction (extract.cu k_xlevel; bf_extract / hodbf_extract,
// Alg. 3): the handle's device geometry tables, the request's blob section and its two slab
// buffers.  Slabs of level l are [pos of tau among the touched T_O nodes][rank row < Rl][request
// column j], so every output element of every stage is one independent dot product.
struct XLPart {
  const int32_t* rr;    // row ranks, levels lc..L: rr[(l - lc) nb + idx]
  const int32_t* rc;    // column ranks, levels 0..lc: rc[l nb + idx]
  const int64_t* roff;  // R block offsets (pool, from fr), levels lc..L-1
  const int64_t* woff;  // W block offsets (from fw), levels 1..lc: woff[(l - 1) nb + idx]
  const int64_t* boff;  // B block offsets (from fb), level lc
  int64_t fr, fb, fw;   // pool bases of the part's R / B / W sections
  int32_t L, lc, nI, nJ;
  void* out;            // out[orow[i] + ocol[j] ldo]
  int64_t ldo;
  int64_t slab[2];      // element offsets of the part's ping-pong slab buffers
  // int64 offsets into the query blob: per column tj (leaf), vtoff, ocol; per row ti (leaf), uoff,
  // ustr, orow, ypos (position of the row's leaf among the touched level-L nodes); per level l
  // tau_off[l] (start of level l in taus / ppos), taus (touched T_O nodes, ascending), ppos (each
  // one's parent position in level l - 1's list); Rz[l] (l <= lc) / Ry[l - lc] rows per slab
  int64_t o_tj, o_vtoff, o_ocol, o_ti, o_uoff, o_ustr, o_orow, o_ypos, o_toff, o_taus, o_ppos, o_rz, o_ry;
};
// stage s of every part (0 = Vt gather, 1..lc W, lc+1 B, lc+2..L+1 R, L+2 U rows, scattered to out);
// wpre: nparts + 1 prefix sums of the parts' work items (output elements) at stage s
void launch_xlevel(int dtype, int s, int nparts, const XLPart* P, const int64_t* wpre, int64_t total,
                   const int64_t* blob, const void* pool, void* S, cudaStream_t st);
void launch_xgather_vt(int dtype, int64_t n, const int64_t* e, const void* pool, void* S, cudaStream_t st);
void launch_xscatter(int dtype, int64_t nI, int64_t nJ, const int64_t* orow, const int64_t* ocol, const void* T, void* out,
                     int64_t ldo, cudaStream_t st);

void launch_accumulate(int dtype, int64_t rows, int64_t nrhs, const void* A, int64_t lda, void* Y, int64_t ldy,
                       cudaStream_t st);
void launch_extract_vt_cols(int dtype, int64_t nJ, const int64_t* jmap, const void* pool, void* S, int64_t ldS,
                            cudaStream_t st);
void launch_extract_u_rows(int dtype, int64_t nE, const int64_t* imap, const int64_t* ocol, const void* pool,
                           const void* S, int64_t ldS, void* out, int64_t ldo, cudaStream_t st);
void launch_extract_gather(int dtype, int64_t n, const int64_t* pairs, const void* pool, void* out, cudaStream_t st);

// Per-device launch attributes.  A process may hold handles on several GPUs (a handle is bound to
// the device it was created on and launches with that device current), so everything cached about
// "the device" is cached per device id, lock-free and thread-safe.
constexpr int BF_MAX_DEVICES = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
// streaming multiprocessors of the current device
inline int device_sm_count() {
  static std::atomic<int> cache[BF_MAX_DEVICES];
  const int d = current_device();
  if (d < 0 || d >= BF_MAX_DEVICES) throw Err{BF_ERR_DEVICE, "device id out of range"};
  int v = cache[d].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    if (e != cudaSuccess || v <= 0) throw Err{BF_ERR_CUDA, std::string("SM count: ") + cudaGetErrorString(e)};
    cache[d].store(v, std::memory_order_relaxed);
  }
  return v;
}
// cudaFuncAttributeMaxDynamicSharedMemorySize of `kernel` on the current device, set once per
// device and raised when a larger launch needs it; `state` is the caller's per-kernel static
// (one slot per device: the largest size set so far).  Failures surface as BF_ERR_CUDA.
inline void ensure_smem_attr(std::atomic<size_t> (&state)[BF_MAX_DEVICES], const void* kernel, size_t smem) {
  const int d = current_device();
  if (d < 0 || d >= BF_MAX_DEVICES) throw Err{BF_ERR_DEVICE, "device id out of range"};
  if (state[d].load(std::memory_order_acquire) >= smem) return;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) throw Err{BF_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e)};
  size_t cur = state[d].load(std::memory_order_relaxed);
  while (cur < smem && !state[d].compare_exchange_weak(cur, smem, std::memory_order_release)) {
  }
}

// Launch with programmatic stream serialization (PDL, see mma.cuh pdl_wait) unless env BF_NO_PDL
// is set; the kernel must call pdl_wait() before touching stream-ordered memory.
inline bool pdl_enabled() {
  static const bool on = getenv("BF_NO_PDL") == nullptr;
  return on;
}
template <typename Arg>
inline void launch_pdl(void (*kernel)(Arg), unsigned grid, unsigned grid_y, unsigned block, size_t smem,
                       cudaStream_t st, const Arg& a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, grid_y);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, a);
}
template <typename Arg>
inline void launch_pdl(void (*kernel)(Arg), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       const Arg& a) {
  launch_pdl(kernel, grid, 1u, block, smem, st, a);
}
const char* round_kernel_name(int dtype, const Round& r, int* id);

}  // namespace bfa
