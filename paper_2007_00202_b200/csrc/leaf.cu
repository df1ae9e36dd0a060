// Leaf kernels of the fast path (SURVEY 8(a) rows a1 and a5, and their adjoints in a6):
//   IN : z_i = A_i X(rows of leaf i, :)     A_i = Vt_nu (op N) or U_tau^H (op C)    (V^0; U^L)
//   OUT: Y(rows of leaf i, :) = A_i y_i     A_i = U_tau (op N) or conj(Vt_nu)^T (op C)
// One item = (leaf, 32-column rhs tile).  Each leaf product is (16 x leaf)(leaf x 32) or
// (leaf x 16)(16 x 32): the user block is read / written once and the factor once.
//   * every warp owns whole items (k = warp, warp + 8, ... of the CTA's items) and all 32
//     columns (NT = 4: A fragments loaded once per k-step, 24 independent MMAs per k-step);
//   * an item is processed in chunks (IN: KC rows of the leaf, OUT: MC output rows), each chunk
//     one shared-memory stage of the warp: the chunk's A records (one 1-D bulk copy) plus, for
//     IN, the chunk's X rows as one 2-D TMA tile (KC rows x 32 columns, column-major; columns
//     beyond nrhs arrive as zeros), for OUT the leaf's two half slabs (bulk copies);
//   * lane 0 of the warp keeps DEP chunks in flight in the warp's own stages and re-arms a stage
//     as soon as the warp is done with it: no producer warp, no barrier between warps.
//   IN writes the output slab to HBM; OUT writes Y rows straight from the accumulators (each store
//   instruction covers 8 consecutive rows x 4 columns: full sectors).
// Leaves whose user rows are not contiguous runs (general permutations) read X through the
// permutation with plain loads (correct, not fast).
#include <cstdio>
#include <cstdlib>

#include "mma.cuh"

namespace bfa {

template <class Pol, int MODE, int NW = LEAF_NCONS>
__global__ void __launch_bounds__(NW * 32, 1) k_leaf(const __grid_constant__ LeafArgs A) {
  using E = typename Pol::E;
  constexpr int KS = Pol::KS;
  constexpr int NT = Pol::NT;
  // NT = 4: a leaf warp covers the 32-column tile; NT = 2 (nrhs <= 16): its first half only (the
  // second is padding: the next window pass skips it, the row leaf writes only valid columns)
  static_assert(NT == 4 || NT == 2 || NT == 1, "a leaf warp covers the tile, its first half or 8 columns");
  constexpr int KPS = FAST_RANK / KS;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Lf = A.leaf;
  const int64_t nitems = A.nleaf * ((A.nrhs + FAST_NB - 1) / FAST_NB);
  const int nw = A.npairs;                    // item-owning warps
  const int dep = A.nst / nw;
  const int chunk = A.brows;                  // IN: KC leaf rows; OUT: MC output rows
  const int nch = Lf / chunk;                 // chunks per item
  const size_t stage = (size_t)A.stage_bytes;
  const size_t a_item = (size_t)A.nsteps * FAST_FRAG;          // A bytes of one leaf
  const size_t a_chunk = a_item / nch;                          // A bytes of one chunk
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + A.nst * stage);
  if (threadIdx.x == 0) {
    for (int i = 0; i < A.nst; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  pdl_wait();  // X / slabs are written by earlier stream work
  pdl_trigger();
  __syncthreads();
  if (warp >= nw) return;
  unsigned char* mystages = smem + (size_t)warp * dep * stage;
  uint64_t* myfull = full + warp * dep;
  // chunk sequence of this warp: c -> item k = warp + (c / nch) * nw, chunk c % nch
  auto issue = [&](int64_t c) {
    const int64_t item = blockIdx.x + (warp + (c / nch) * nw) * (int64_t)gridDim.x;
    if (item >= nitems) return;
    const int ch = (int)(c % nch);
    const int64_t leaf = item % A.nleaf, jt = item / A.nleaf;
    const int st = (int)(c % dep);
    unsigned char* sb = mystages + st * stage;
    uint32_t bytes = (uint32_t)a_chunk;
    if (MODE == 0 && A.tma) bytes += (uint32_t)(chunk * FAST_NB * sizeof(E));
    if (MODE == 1) bytes += (uint32_t)(2 * FAST_HSLAB * sizeof(E));
    mbar_expect_tx(&myfull[st], bytes);
    bulk_g2s(sb, static_cast<const unsigned char*>(A.F) + leaf * a_item + ch * a_chunk, (uint32_t)a_chunk, &myfull[st]);
    if (MODE == 0 && A.tma) {
      const int64_t r0 = (A.xperm ? A.xperm[leaf * Lf] : leaf * Lf) + (int64_t)ch * chunk;
      tma_load_2d(sb + a_chunk, &A.map, (int)(r0 * (int64_t)(sizeof(E) / 8)), (int)(jt * FAST_NB), &myfull[st]);
    }
    if (MODE == 1)
      for (int hh = 0; hh < 2; ++hh)
        bulk_g2s(sb + a_chunk + hh * FAST_HSLAB * sizeof(E),
                 static_cast<const E*>(A.Sin) + half_slab_off(jt, hh, A.nlev, A.leaf_lo + leaf),
                 (uint32_t)(FAST_HSLAB * sizeof(E)), &myfull[st]);
  };
  if (lane == 0) {
    if (A.tma && MODE == 0) asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&A.map)) : "memory");
    for (int c = 0; c < dep; ++c) issue(c);
  }

  const int g = lane >> 2, t = lane & 3;
  const bool cj = A.conj_io != 0;
  int bo[NT];  // B-fragment offsets in the two half slabs [half][16 x 16] (OUT)
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) bo[ni] = Pol::leaf_boff(ni, t, g);
  int64_t c = 0;  // chunk sequence number
  for (int64_t item = blockIdx.x + (int64_t)warp * gridDim.x; item < nitems; item += (int64_t)nw * gridDim.x) {
    const int64_t leaf = item % A.nleaf, jt = item / A.nleaf;
    const int j0 = (int)jt * FAST_NB;  // first rhs column of the tile
    typename Pol::FAcc acc;
    acc.zero();
    for (int ch = 0; ch < nch; ++ch, ++c) {
      const int st = (int)(c % dep);
      const unsigned char* sb = mystages + st * stage;
      mbar_wait(&myfull[st], (uint32_t)((c / dep) & 1), 12);
      if (MODE == 0) {
        // z += A_leaf(:, chunk rows) * X(chunk rows, tile)
        const E* xb = reinterpret_cast<const E*>(sb + a_chunk);
        const int nks = chunk / KS;
#pragma unroll 2
        for (int s = 0; s < nks; ++s) {
          typename Pol::FFrags f;
          Pol::load_fa(f, sb + (size_t)s * FAST_FRAG, lane);
          if (A.tma) {
            Pol::load_b_col(f, xb, chunk, s * KS, 0, g, t, cj);
          } else {
            int64_t p[Pol::XROWS], rows[Pol::XROWS];
            Pol::x_rows(p, leaf * Lf + (int64_t)ch * chunk + s * KS, t);
#pragma unroll
            for (int e = 0; e < Pol::XROWS; ++e) rows[e] = A.xperm ? A.xperm[p[e]] : p[e];
            Pol::load_b_x(f, static_cast<const E*>(A.X), rows, A.ldx, j0, g, A.nrhs, cj);
          }
          acc.mac(f);
        }
      } else {
        // Y(chunk rows of leaf, tile) = A_leaf(chunk rows, :) (MC x 16) * y (16 x 32), 16 rows at a time
        const E* ys = reinterpret_cast<const E*>(sb + a_chunk);
        E* __restrict__ Y = static_cast<E*>(A.Y);
        const int64_t base = A.tma ? (A.yperm ? A.yperm[leaf * Lf] : leaf * Lf) : 0;
        for (int mgl = 0; mgl < chunk / 16; ++mgl) {
          acc.zero();
#pragma unroll
          for (int ki = 0; ki < KPS; ++ki) {
            typename Pol::FFrags f;
            Pol::load_fa(f, sb + (size_t)(mgl * KPS + ki) * FAST_FRAG, lane);
            Pol::load_b(f, ys + ki * KS * FAST_HC, bo);
            acc.mac(f);
          }
          const int64_t rr = (int64_t)ch * chunk + mgl * 16;  // first leaf row of this group
          acc.each(g, t, [&](int r, int cc, E v) {
            const int col = j0 + cc;
            if (col < A.nrhs) {
              const int64_t row = A.tma ? base + rr + r : (A.yperm ? A.yperm[leaf * Lf + rr + r] : leaf * Lf + rr + r);
              v.y = conj_im(v.y, cj);
              Y[row + (int64_t)col * A.ldy] = v;
            }
          });
        }
      }
      // the warp is done with the stage: re-arm it DEP chunks ahead
      __syncwarp();
      if (lane == 0) issue(c + dep);
    }
    if (MODE == 0) {
      E* dst0 = static_cast<E*>(A.Sout) + half_slab_off(jt, 0, A.nlev, A.leaf_lo + leaf);
      E* dst1 = static_cast<E*>(A.Sout) + half_slab_off(jt, 1, A.nlev, A.leaf_lo + leaf);
      acc.each(g, t, [&](int r, int cc, E v) {
        Pol::slab_put(cc < FAST_HC ? dst0 : dst1, r, cc & (FAST_HC - 1), v);
      });
    }
  }
}

// ---- host side ----------------------------------------------------------------------------------
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// resolved once, thread-safely (function-local static initialisation: applies on several host
// threads may reach their first TMA map at the same time)
static EncodeTiled encode_fn() {
  static const EncodeTiled fn = []() -> EncodeTiled {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiled>(p);
    return nullptr;
  }();
  return fn;
}

// 2-D map over a column-major (rows x nrhs, ld) complex block in 8-byte units; box = brows x 32
static bool make_map(int dtype, const void* base, int64_t rows, int64_t nrhs, int64_t ld, int brows, CUtensorMap* map) {
  const int64_t cs = dtype == BF_C128 ? 16 : 8, w = cs / 8;
  if (((uintptr_t)base & 15) || (ld * cs) % 16 || rows * w >= (int64_t(1) << 31) || nrhs >= (int64_t(1) << 31))
    return false;
  if (brows * w > 256) return false;
  EncodeTiled fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)(rows * w), (cuuint64_t)nrhs};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * cs)};
  const cuuint32_t box[2] = {(cuuint32_t)(brows * w), (cuuint32_t)FAST_NB};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool fast_make_xmap(int dtype, const void* X, int64_t rows, int64_t nrhs, int64_t ld, int brows, CUtensorMap* map) {
  return make_map(dtype, X, rows, nrhs, ld, brows, map);
}

constexpr size_t LEAF_SMEM = 227 * 1024;

template <class Pol, int MODE, int NW = LEAF_NCONS>
static void launch_leaf_t(LeafArgs& a, cudaStream_t st) {
  const int nsm = device_sm_count();
  using E = typename Pol::E;
  const int nch = a.leaf / a.brows;
  const size_t a_chunk = (size_t)a.nsteps * FAST_FRAG / nch;
  const size_t b_bytes = MODE == 0 ? (a.tma ? (size_t)a.brows * FAST_NB * sizeof(E) : 0) : 2 * FAST_HSLAB * sizeof(E);
  a.stage_bytes = (int64_t)((a_chunk + b_bytes + 1023) & ~size_t(1023));
  const size_t avail = LEAF_SMEM - 64 * 8;  // barriers
  const size_t stg = (size_t)a.stage_bytes;
  const int np = NW;  // item-owning warps
  int dep = (int)(avail / ((size_t)np * stg));
  int maxdep = 4;
  if (const char* e = getenv("BF_LEAF_DEP")) maxdep = atoi(e);  // tuning knob
  if (dep > maxdep) dep = maxdep;
  if (dep < 1) throw Err{BF_ERR_ARG, "leaf chunk too large for the leaf kernel's shared memory"};
  a.npairs = np;
  a.nst = np * dep;
  const size_t smem = (size_t)a.nst * stg + (size_t)a.nst * 8;
  static std::atomic<size_t> attr[BF_MAX_DEVICES];
  ensure_smem_attr(attr, (const void*)k_leaf<Pol, MODE, NW>, smem);
  const int64_t items = a.nleaf * ((a.nrhs + FAST_NB - 1) / FAST_NB);
  const unsigned grid = (unsigned)(items < nsm ? items : nsm);
  launch_pdl(k_leaf<Pol, MODE, NW>, grid, NW * 32, smem, st, a);
}

// full 32-column tiles: item-owning warps per CTA (8 by default; env BF_LEAF_NW_IN / BF_LEAF_NW_OUT
// = 12 or 16 for the A/B of more warps against the register cap and the stage depth they leave)
template <class Pol, int MODE>
static void launch_leaf_nw(LeafArgs& a, cudaStream_t st) {
  static const int nw = []() {
    const char* e = getenv(MODE == 0 ? "BF_LEAF_NW_IN" : "BF_LEAF_NW_OUT");
    return e ? atoi(e) : LEAF_NCONS;
  }();
  if (nw == 16) launch_leaf_t<Pol, MODE, 16>(a, st);
  else if (nw == 12) launch_leaf_t<Pol, MODE, 12>(a, st);
  else launch_leaf_t<Pol, MODE, LEAF_NCONS>(a, st);
}

void launch_leaf(int dtype, LeafArgs& a, cudaStream_t st) {
  const int w = dtype == BF_C128 ? 2 : 1;
  // chunk rows (measured best on B200, tools/gpurun_scripts/gpu_r2h.sh): IN 16 (c128) / 32 (c64) leaf rows,
  // OUT 16 (c128) / 64 (c64) output rows; depth 2-4 stages per warp
  int kc = a.mode == 0 ? (dtype == BF_C128 ? 16 : 32) : (dtype == BF_C128 ? 16 : 64);
  if (const char* e = getenv(a.mode == 0 ? "BF_LEAF_KC" : "BF_LEAF_MC")) kc = atoi(e);  // tuning knob
  a.brows = a.leaf < kc ? a.leaf : kc;
  // X by TMA when the leaves are contiguous runs of user rows and the block is aligned
  if (a.tma && a.mode == 0)
    a.tma = make_map(dtype, a.X, a.nleaf * a.leaf, a.nrhs, a.ldx, a.brows, &a.map) ? 1 : 0;
  (void)w;
  const bool narrow = a.nrhs <= FAST_HC && !getenv("BF_NO_HALF_SKIP");  // the tile's second half is padding
  const bool eight = narrow && a.nrhs <= 8 && !getenv("BF_NO_NARROW");   // and columns 8..15 too
  if (dtype == BF_C128) {
    if (eight) {
      if (a.mode == 0) launch_leaf_t<PolC128<1>, 0>(a, st);
      else launch_leaf_t<PolC128<1>, 1>(a, st);
    } else if (narrow) {
      if (a.mode == 0) launch_leaf_t<PolC128<2>, 0>(a, st);
      else launch_leaf_t<PolC128<2>, 1>(a, st);
    } else {
      if (a.mode == 0) launch_leaf_nw<PolC128<4>, 0>(a, st);
      else launch_leaf_nw<PolC128<4>, 1>(a, st);
    }
  } else {
    if (eight) {
      if (a.mode == 0) launch_leaf_t<PolC64<1>, 0>(a, st);
      else launch_leaf_t<PolC64<1>, 1>(a, st);
    } else if (narrow) {
      if (a.mode == 0) launch_leaf_t<PolC64<2>, 0>(a, st);
      else launch_leaf_t<PolC64<2>, 1>(a, st);
    } else {
      if (a.mode == 0) launch_leaf_nw<PolC64<4>, 0>(a, st);
      else launch_leaf_nw<PolC64<4>, 1>(a, st);
    }
  }
}

const char* leaf_kernel_name(int dtype, int mode) {
  static const char* nm[2][2] = {{"k_leaf<c64,in>", "k_leaf<c64,out>"}, {"k_leaf<c128,in>", "k_leaf<c128,out>"}};
  return nm[dtype == BF_C128][mode];
}

}  // namespace bfa
