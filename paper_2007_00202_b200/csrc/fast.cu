// Window-pass kernel of the fast path (see fast.cuh for windows, slots and the operand stream;
// mma.cuh for the complex-product policies).  SURVEY 8(a) rows a2 (W stages, Eq. 3.2 right,
// P:312-317), a3 (centre B), a4 (R stages, Eq. 3.2 left) and their adjoints (a6).
//
// One work item = (window, 32-column rhs tile); one persistent CTA of 16 warps per SM.  The
// operator acts on rows only, so the two 16-column halves of the tile are independent: warps
// 0-7 own half 0, warps 8-15 half 1, and each half synchronises only with itself (named barrier
// 1 + half), so the halves can drift against each other.  Inside a half, warp w computes slot
// o = w % S for the 8*NT columns of column tile w / S.  (Two independent 8-warp CTAs per SM, one
// per half, were measured slower: the ring a CTA can afford is half as deep.)
//   * operand stream: a ring of 32 KB pages (TMA bulk copies, full mbarriers) shared by the two
//     halves; whoever releases a page last re-arms it with the page NP ahead (no producer warp,
//     so all 16 warps compute with 128 registers each);
//   * the ops of an item ping-pong between two half-window buffers (op q reads buffer rd, writes
//     the other), so one CTA barrier per op suffices: between an op's writes and the next pair
//     op's reads of other slots.  The last op writes the output slabs straight to HBM; when
//     every warp has reached it, the other buffer takes the next window.
//   * complex64 windows may span 4 levels (16 slots per half): each warp then runs every op for
//     two slots -- the two outputs of one input pair, in one k-loop, so that the 3xTF32 split of
//     each slab fragment is computed once for both (PAIRW; the slot pair changes with the op).
#include <cstdio>

#include "mma.cuh"

namespace bfa {

template <class Pol, int D, int HV = 2, int PGB = 32768>
struct PassCfg {
  using E = typename Pol::E;
  static constexpr int WINH = (1 << (D > 3 ? D : 3)) * FAST_HSLAB;  // half window (elements)
  // window buffer: [half][slot][16 x 16]; with nrhs <= 16 (HV <= 1) the second column half is
  // padding and is neither loaded nor stored, so a buffer holds one half
  static constexpr int HALVES = HV == 2 ? 2 : 1;
  static constexpr int WIN = HALVES * WINH;
  static constexpr int PG = PGB;                              // ring page (bytes)
  // ring pages: complex128 3 (2 x 64 KB windows), complex64 4 (3-level windows) or 3 (4-level).
  // (Measured on complex64: a 5th page or a third window buffer, which lets the next window load
  // a whole item ahead, made the 3-level pass slower: 0.1156 / 0.1168 vs 0.1136 ms.)  With one
  // window half (nrhs <= 16) the freed shared memory could deepen the ring to 5-6 pages: measured
  // neutral at nrhs 1 / 8 / 16 for both dtypes (0.639 vs 0.636 ms c128 at nrhs 1,
  // tools/gpurun_scripts/r2_g9.sh), so the ring keeps its depth.
  static constexpr int NP = (sizeof(E) == 16 ? 3 : D > 3 ? 3 : 4) * (32768 / PGB);
  __host__ __device__ static constexpr size_t bars_off() { return 2 * WIN * sizeof(E) + (size_t)NP * PG; }
  __host__ __device__ static constexpr size_t smem() { return bars_off() + (1 + NP) * 8 + (1 + NP) * 4; }
};

// The operand stream of one CTA: page j (0, 1, 2, ...) is k-steps [s0, s0 + nst) of op q of the
// CTA's item j / PPI.
template <class Pol, int D, int HV = 2, int PGB = 32768>
struct Stream {
  using E = typename Pol::E;
  using Cfg = PassCfg<Pol, D, HV, PGB>;
  static constexpr int S = 1 << D;
  static constexpr int SPP = Cfg::PG / (S * FAST_FRAG);  // k-steps per page
  static constexpr int SPL = fast_spl((int)sizeof(E), S); // k-steps per page of the column-leaf op
  static constexpr int XT = SPL * Pol::KS * FAST_NB * (int)sizeof(E);  // X tile bytes per slot
  // pages ahead of the ring's newest page whose factor records are prefetched into L2
  // (cp.async.bulk.prefetch.L2; ncu of the complex64 4-level pass: half of the page waits found
  // the page not yet landed).  Measured slower on config 5 (tools/gpurun_scripts/r2_g30.sh):
  // c128 1.346 / 1.364 ms and c64 0.738 / 0.738 ms at 2 / 4 pages ahead against 1.258 / 0.676 ms
  // without, so it is off (-DBF_PASS_PF=n for the A/B).
#ifndef BF_PASS_PF
#define BF_PASS_PF 0
#endif
  static constexpr int PF = BF_PASS_PF;
  __host__ __device__ static int steps_per_page(int kind) { return kind == FK_LEAF_IN ? SPL : SPP; }
  const FastArgs& A;
  unsigned char* ring;
  E* winbuf;
  uint64_t* full;
  uint64_t* winF;
  int64_t nitems;
  int ppi;  // pages per item
  __device__ __forceinline__ int64_t item_of(int64_t i) const { return blockIdx.x + i * gridDim.x; }
  // factor bytes of page j (A records only): source, byte count, op, first k-step; false past the end
  __device__ bool page_src(int64_t j, const unsigned char*& src, uint32_t& bytes, int& q, int& s0,
                           int64_t& item) const {
    const FastPass& P = A.p;
    // (32-bit division whenever the page index fits: it runs on the ring's critical path, in
    // the thread that re-arms the page)
    const int64_t i = j < 0xffffffffll ? (int64_t)((uint32_t)j / (uint32_t)ppi) : j / ppi;
    item = item_of(i);
    if (item >= nitems) return false;
    int r = (int)(j - i * ppi);
    q = 0;
    for (;; ++q) {
      const int sp = steps_per_page(P.ops[q].kind);
      const int np = (P.ops[q].nsteps + sp - 1) / sp;
      if (r < np) break;
      r -= np;
    }
    const FastOp& op = P.ops[q];
    const int sp = steps_per_page(op.kind);
    s0 = r * sp;
    const int nst = min(sp, op.nsteps - s0);
    const int64_t w = item & (P.nwin - 1);  // local window index (records of this rank only)
    src = static_cast<const unsigned char*>(A.F) + P.fbase + w * P.win_bytes + op.off + (int64_t)s0 * S * FAST_FRAG;
    bytes = (uint32_t)(nst * S * FAST_FRAG);
    return true;
  }
  __device__ void issue_page(int64_t j) const {
    const FastPass& P = A.p;
    const unsigned char* src;
    uint32_t bytes;
    int q, s0;
    int64_t item;
    if (!page_src(j, src, bytes, q, s0, item)) return;
    // warm L2 with page j + PF (its factor records) while page j streams into the ring
    if (PF > 0) {
      const unsigned char* ps;
      uint32_t pb;
      int pq, ps0;
      int64_t pit;
      if (page_src(j + PF, ps, pb, pq, ps0, pit)) bulk_prefetch_l2(ps, pb);
    }
    const FastOp& op = P.ops[q];
    const int64_t w = item & (P.nwin - 1);
    const int slot = (int)(j % Cfg::NP);
    unsigned char* pg = ring + (size_t)slot * Cfg::PG;
    if (op.kind != FK_LEAF_IN) {
      mbar_expect_tx(&full[slot], bytes);
      bulk_g2s(pg, src, bytes, &full[slot]);
      return;
    }
    // column leaf: the A records plus, per slot, SPL * KS rows x 32 columns of X (2-D TMA tile)
    mbar_expect_tx(&full[slot], bytes + S * XT);
    bulk_g2s(pg, src, bytes, &full[slot]);
    const int64_t jt = item >> (P.a_log + P.b_log);
    const int64_t a = P.a_lo + (w >> P.b_log), b = P.b_lo + (w & ((int64_t(1) << P.b_log) - 1));
    const int ds = P.d - op.s;
    for (int o = 0; o < S; ++o) {
      const int64_t leaf = ((a << op.s) + (o >> ds)) + ((b << ds) + (o & ((1 << ds) - 1)));  // tau or nu
      const int64_t r0 = (A.xperm ? A.xperm[leaf * op.leaf] : leaf * op.leaf) + (int64_t)s0 * Pol::KS;
      tma_load_2d(pg + SPL * S * FAST_FRAG + o * XT, &A.xmap, (int)(r0 * (int64_t)(sizeof(E) / 8)),
                  (int)(jt * FAST_NB), &full[slot]);
    }
  }
  __device__ void issue_window(int64_t i, int wb) const {
    const FastPass& P = A.p;
    const int64_t item = item_of(i);
    if (item >= nitems) return;
    const int64_t w = item & (P.nwin - 1), jt = item >> (P.a_log + P.b_log);
    const int64_t a = P.a_lo + (w >> P.b_log), b = P.b_lo + (w & ((int64_t(1) << P.b_log) - 1));
    const uint32_t bytes = (uint32_t)(S * FAST_HSLAB * sizeof(E));
    mbar_expect_tx(winF, Cfg::HALVES * bytes);
    const E* Sin = static_cast<const E*>(A.Sin);
    for (int h = 0; h < Cfg::HALVES; ++h) {
      E* dst = winbuf + wb * Cfg::WIN + h * Cfg::WINH;
      if (!P.xin) {  // the window's input slabs are contiguous in the slab buffer
        bulk_g2s(dst, Sin + pass_slab_off(P, 0, jt, h, A.nlev, A.ntiles, a, b, P.in_s, 0), bytes, winF);
      } else {  // exchange layout: the slabs may come from several peers' chunks
        int p0 = 0, p1 = 0;
        const int64_t o0 = pass_slab_off(P, P.xin, jt, h, A.nlev, A.ntiles, a, b, P.in_s, 0, -1, &p0);
        const int64_t o1 = pass_slab_off(P, P.xin, jt, h, A.nlev, A.ntiles, a, b, P.in_s, S - 1, -1, &p1);
        if (p0 == p1 && o1 - o0 == (int64_t)(S - 1) * FAST_HSLAB) {
          // one peer's chunk holds the window's slabs in slot order: one copy (small copies are
          // issue-bound, ~0.3 us each)
          bulk_g2s(dst, Sin + o0, bytes, winF);
        } else {
          for (int o = 0; o < S; ++o)
            bulk_g2s(dst + o * FAST_HSLAB, Sin + pass_slab_off(P, P.xin, jt, h, A.nlev, A.ntiles, a, b, P.in_s, o),
                     (uint32_t)(FAST_HSLAB * sizeof(E)), winF);
        }
      }
    }
  }
};

// HV: column halves with work (1 when nrhs <= 16, the second half of the only tile being padding;
// 0 = narrow, nrhs <= 8: one half, one 8-column n-tile per warp (Pol::NT == 1), a warp per slot;
// 3 = nrhs 9-16: one half worked by all 16 warps).
// A compile-time choice, so that the two-half instantiation keeps its code generation.
template <class Pol, int D, int HV = 2, int PGB = 32768>
__global__ void __launch_bounds__(FAST_THREADS, 1) k_bf_pass(const __grid_constant__ FastArgs A) {
  using E = typename Pol::E;
  using Cfg = PassCfg<Pol, D, HV, PGB>;
  using St = Stream<Pol, D, HV, PGB>;
  // the fused leaf ops assume 32 KB pages (whole 16-row groups / the X tiles of fast_spl); the
  // small-page instantiation serves window passes without them (launch_fast_pass)
  constexpr bool LEAF_OK = Pol::LEAF_OPS && PGB == 32768;
  constexpr int NT = Pol::NT;
  constexpr int S = 1 << D;                          // slots of the window
  constexpr int CT = HV == 0 ? 1 : 2 / NT;           // column tiles per slot (in a half)
  static_assert(HV != 0 || NT == 1, "narrow passes use one 8-column n-tile per warp");
  // warps per working half: 8, or all 16 on the one half of nrhs 9-16 (HV = 3)
  constexpr int NCH = HV == 3 ? FAST_NCONS : FAST_NCONS_HALF;
  // slots per warp: 2 for 4-level windows (16 slots, 8 warps per half), else 1
  constexpr int SPW = S * CT > NCH ? S * CT / NCH : 1;
  static_assert(SPW == 1 || CT == 1, "several slots per warp need whole-slot warps");
  // two slots per warp (complex64 4-level windows): the warp's slots of a pair op are the two
  // outputs of one input pair, sharing the slab fragments' 3xTF32 split (Pol::PAIR_SHARE)
  constexpr bool PAIRW = Pol::PAIR_SHARE && SPW == 2;
  constexpr int NACTH = S * CT / SPW;                // active warps per half
  constexpr int NACT = (HV == 3 ? 1 : 2) * NACTH;    // active warps
  constexpr int SPP = St::SPP;                       // k-steps per page
  constexpr int NP = Cfg::NP;
  constexpr int WIN = Cfg::WIN;
  constexpr int KPS = FAST_RANK / Pol::KS;           // k-steps per 16-row slab
  static_assert(NACT <= FAST_NCONS, "too many warps");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  E* winbuf = reinterpret_cast<E*>(smem_raw);
  unsigned char* ring = smem_raw + 2 * WIN * sizeof(E);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + Cfg::bars_off());
  uint64_t* winF = bars;                              // window loads (one phase per item)
  uint64_t* full = bars + 1;
  int* wcnt = reinterpret_cast<int*>(bars + 1 + NP);  // arrivals at the last op of an item
  int* pcnt = wcnt + 1;                               // page releases

  const FastPass& P = A.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int diag = A.diag;
  St str{A, ring, winbuf, full, winF, P.nwin * ((A.nrhs + FAST_NB - 1) / FAST_NB), 0};
  for (int q = 0; q < P.nops; ++q) {
    const int sp = St::steps_per_page(P.ops[q].kind);
    str.ppi += (P.ops[q].nsteps + sp - 1) / sp;
  }
  const int64_t nitems = str.nitems;
  const int nwin_log = P.a_log + P.b_log;
  const int64_t bmask = (int64_t(1) << P.b_log) - 1;

  if (threadIdx.x == 0) {
    mbar_init(winF, 1);
    wcnt[0] = 0;
    for (int i = 0; i < NP; ++i) {
      mbar_init(&full[i], 1);
      pcnt[i] = 0;
    }
    fence_mbar_init();
    // factor pages do not depend on earlier stream work: prefetch them before the PDL wait
    if (!(diag & 1) && !P.xleaf)
      for (int j = 0; j < NP; ++j) str.issue_page(j);
  }
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0 && !(diag & 1)) {
    if (P.in_s >= 0) str.issue_window(0, 0);
    if (P.xleaf) {  // column-leaf pages carry X tiles
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&A.xmap)) : "memory");
      for (int j = 0; j < NP; ++j) str.issue_page(j);
    }
  }
  __syncthreads();
  const int half = HV == 3 ? 0 : warp / FAST_NCONS_HALF, hw = HV == 3 ? warp : warp % FAST_NCONS_HALF;
  if (hw >= NACTH) return;  // idle warps (d = 1)
  // nrhs <= 16 (HV = 1): the second column half of the (only) tile is padding -- its warps skip
  // the work, and every release count waits for the first half's warps only; HV = 3: all 16 warps
  // work on that half, a warp per (slot, 8-column tile)
  constexpr int HVN = HV == 0 || HV == 3 ? 1 : HV;  // halves with work
  if (half >= HVN) return;
  constexpr int nact = HVN * NACTH;

  if (half == 1 && A.skew > 0) __nanosleep(A.skew);
  const int g = lane >> 2, t = lane & 3;
  const int o0 = hw % (S / SPW);          // the warp's first slot (its others: o0 + S / SPW, ...)
  const int c0w = 8 * NT * (hw / S);      // first column of this warp inside the half
  const int hbar = 1 + half;              // the half's named barrier
  int bo[NT];                             // lane-constant B-fragment offsets inside a half slab
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) bo[ni] = Pol::boff(t, g, c0w, ni);
  E* __restrict__ Sout = static_cast<E*>(A.Sout);
  int64_t j = 0;  // page sequence number
  int slot = 0;   // j % NP
  int rnd = 0;    // j / NP
  uint32_t ph = 0;
  int64_t i = 0;
  int cur = 0;    // window buffer holding the current item's input
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++i) {
    const int64_t w = item & ((int64_t(1) << nwin_log) - 1), jt = item >> nwin_log;
    const int64_t a = P.a_lo + (w >> P.b_log), b = P.b_lo + (w & bmask);
    if (!(diag & 1) && P.in_s >= 0) mbar_wait(winF, (uint32_t)(i & 1), 3);
    int rd = cur;  // op q reads buffer rd, writes rd ^ 1
    for (int q = 0; q < P.nops; ++q) {
      const FastOp op = P.ops[q];
      const bool last = q == P.nops - 1;
      // (the condition order matters to the complex128 code generation: 2 % per apply)
      if (lane == 0 && !(diag & 1) && P.in_s >= 0 && last) {
        // every warp past op q-1 -> buffer rd ^ 1 is free: the last one in loads the next window
        if (atom_add_acqrel(wcnt, 1) == (int)(i + 1) * nact - 1) str.issue_window(i + 1, rd ^ 1);
      }
      const E* win = winbuf + rd * WIN + half * Cfg::WINH;
      if constexpr (PAIRW) {
        if (!A.no_pairw && (op.kind == FK_PAIR_DOWN || op.kind == FK_PAIR_UP)) {
          // the warp's two slots are the outputs that read the same input pair (they differ in
          // bit pb: the top bit of the T_O index for a W stage, bit 0 for an R stage), so one k-loop
          // splits each slab fragment once for both of them
          const int ds = P.d - op.s;
          const int pb = op.kind == FK_PAIR_DOWN ? ds - 1 : 0;
          const int oA = ((hw >> pb) << (pb + 1)) | (hw & ((1 << pb) - 1)), oB = oA | (1 << pb);
          const E* sp0;
          if (op.kind == FK_PAIR_DOWN) {
            const int tp = oA >> (ds - 1), up = oA & ((1 << (ds - 1)) - 1);
            sp0 = win + (((tp >> 1) << ds) + 2 * up) * FAST_HSLAB;
          } else {
            const int tt = oA >> ds, u = oA & ((1 << ds) - 1);
            sp0 = win + (((2 * tt) << (ds - 1)) + (u >> 1)) * FAST_HSLAB;
          }
          const E* sp1 = op.kind == FK_PAIR_DOWN ? sp0 + FAST_HSLAB
                                                 : win + (((2 * (oA >> ds) + 1) << (ds - 1)) + ((oA & ((1 << ds) - 1)) >> 1)) * FAST_HSLAB;
          typename Pol::FAcc accA, accB;
          accA.zero();
          accB.zero();
          constexpr int NSTEP = 2 * FAST_RANK / Pol::KS;
          constexpr int SPO = SPP < NSTEP ? SPP : NSTEP;
          static_assert(NSTEP % SPO == 0, "pages must split ops evenly");
          auto bsrc = [&](int k) { return (k < KPS ? sp0 : sp1) + (k & (KPS - 1)) * Pol::KS * FAST_HC; };
          if (!(diag & 1)) mbar_wait(&full[slot], ph, 4);
          const int roffA = oA * FAST_FRAG + Pol::rec_off(c0w), droff = (oB - oA) * FAST_FRAG;
          const unsigned char* pgn = ring + (size_t)slot * Cfg::PG + roffA;
          int nslot = slot;
          uint32_t nph = ph;
          typename Pol::FFrags f[2];
          float4 fb[2][NT];
          Pol::load_fa(f[0], pgn, lane);
          Pol::load_fa2(fb[0], pgn + droff, lane);
          Pol::load_b(f[0], bsrc(0), bo);
#pragma unroll
          for (int k = 0; k < NSTEP; ++k) {
            if (k + 1 < NSTEP) {
              const int k1 = k + 1;
              if (k1 % SPO == 0) {
                if (++nslot == NP) {
                  nslot = 0;
                  nph ^= 1;
                }
                if (!(diag & 1)) mbar_wait(&full[nslot], nph, 4);
                pgn = ring + (size_t)nslot * Cfg::PG + roffA;
              }
              Pol::load_fa(f[k1 & 1], pgn + (k1 % SPO) * S * FAST_FRAG, lane);
              Pol::load_fa2(fb[k1 & 1], pgn + (k1 % SPO) * S * FAST_FRAG + droff, lane);
              Pol::load_b(f[k1 & 1], bsrc(k1), bo);
            }
            {
              typename Pol::ASplit sa;
              Pol::split_a(f[k & 1], sa);
              accA.mac_split(sa, f[k & 1].f);
              accB.mac_split(sa, fb[k & 1]);
            }
            if ((k + 1) % SPO == 0) {
              __syncwarp();
              if (lane == 0 && !(diag & 1)) {
                if (atom_add_release_page(&pcnt[slot], 1) == (rnd + 1) * nact - 1) str.issue_page(j + NP);
              }
              ++j;
              if (++slot == NP) {
                slot = 0;
                ph ^= 1;
                ++rnd;
              }
            }
          }
          if (last) {
            if (!(diag & 2)) {
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                const int o = v ? oB : oA;
                E* dst;
                if (P.xout && A.p2p) {
                  int peer = 0;
                  const int64_t off =
                      pass_slab_off(P, P.xout, jt, half, A.nlev, A.ntiles, a, b, P.out_s, o, A.myrank, &peer);
                  dst = static_cast<E*>(A.peer[peer]) + off;
                } else {
                  dst = Sout + pass_slab_off(P, P.xout, jt, half, A.nlev, A.ntiles, a, b, P.out_s, o);
                }
                Pol::store_slab(v ? accB : accA, dst, c0w, g, t, lane);
              }
            }
            cur = rd ^ 1;
          } else {
            if (!(diag & 4)) {
              if (q == 0) named_sync(hbar, NACTH * 32);
              E* dst = winbuf + (rd ^ 1) * WIN + half * Cfg::WINH;
              Pol::store_slab(accA, dst + oA * FAST_HSLAB, c0w, g, t, lane);
              Pol::store_slab(accB, dst + oB * FAST_HSLAB, c0w, g, t, lane);
              named_sync(hbar, NACTH * 32);
            } else {
              E* dst = winbuf + (rd ^ 1) * WIN + half * Cfg::WINH;
              Pol::store_slab(accA, dst + oA * FAST_HSLAB, c0w, g, t, lane);
              Pol::store_slab(accB, dst + oB * FAST_HSLAB, c0w, g, t, lane);
            }
            rd ^= 1;
          }
          continue;
        }
      }
#pragma unroll
      for (int sl = 0; sl < SPW; ++sl) {
      const int o = o0 + sl * (S / SPW);  // slot
      const bool rel = sl == SPW - 1;     // the warp's last slot releases the op's pages
      (void)rel;
      typename Pol::FAcc acc;
      acc.zero();
      const E* sp0 = win + o * FAST_HSLAB;
      const E* sp1 = sp0;
      const int ds = P.d - op.s;
      if (op.kind == FK_PAIR_DOWN) {  // output level s+1 from input level s
        const int tp = o >> (ds - 1), up = o & ((1 << (ds - 1)) - 1);
        sp0 = win + (((tp >> 1) << ds) + 2 * up) * FAST_HSLAB;
        sp1 = sp0 + FAST_HSLAB;
      } else if (op.kind == FK_PAIR_UP) {  // output level s from input level s+1
        const int tt = o >> ds, u = o & ((1 << ds) - 1);
        sp0 = win + (((2 * tt) << (ds - 1)) + (u >> 1)) * FAST_HSLAB;
        sp1 = win + (((2 * tt + 1) << (ds - 1)) + (u >> 1)) * FAST_HSLAB;
      }
      if (LEAF_OK && op.kind == FK_LEAF_OUT) {
        if constexpr (LEAF_OK) {
        // fused row leaf (a5): Y(rows of this slot's leaf) = A (leaf x 16) y (16 x 32), one 16-row
        // group at a time; A records stream through the ring like any op, y is this slot's slab
        const int ds2 = P.d - op.s;
        const int64_t leaf = ((a << op.s) + (o >> ds2)) + ((b << ds2) + (o & ((1 << ds2) - 1))) -
                             P.yleaf_lo;  // tau or nu, relative to the local Y rows
        const int Lf = op.leaf;
        const int64_t base = A.ycontig ? (A.yperm ? A.yperm[leaf * Lf] : leaf * Lf) : 0;
        E* __restrict__ Y = static_cast<E*>(A.Y);
        const bool cj = A.conj_io != 0;
        const int n = op.nsteps;
        static_assert(SPP % KPS == 0, "a page holds whole 16-row groups");
        const int j0 = (int)jt * FAST_NB + half * FAST_HC + c0w;
        for (int s0 = 0; s0 < n; s0 += SPP) {
          if (!(diag & 1)) mbar_wait(&full[slot], ph, 4);
          const unsigned char* pg = ring + (size_t)slot * Cfg::PG + o * FAST_FRAG;
          const int ngrp = min(SPP, n - s0) / KPS;
#pragma unroll 1
          for (int mg = 0; mg < ngrp; ++mg) {
            // the KPS k-steps of one 16-row group, software-pipelined
            typename Pol::FFrags f[2];
            Pol::load_fa(f[0], pg + (mg * KPS) * S * FAST_FRAG, lane);
            Pol::load_b(f[0], sp0, bo);
#pragma unroll
            for (int ki = 0; ki < KPS; ++ki) {
              if (ki + 1 < KPS) {
                Pol::load_fa(f[(ki + 1) & 1], pg + (mg * KPS + ki + 1) * S * FAST_FRAG, lane);
                Pol::load_b(f[(ki + 1) & 1], sp0 + (ki + 1) * Pol::KS * FAST_HC, bo);
              }
              acc.mac(f[ki & 1]);
            }
            const int64_t rr = (int64_t)((s0 / KPS) + mg) * 16;  // first leaf row of this group
            acc.each(g, t, [&](int r, int c, E v) {
              const int col = j0 + c;
              if (col < A.nrhs) {
                const int64_t row = A.ycontig ? base + rr + r : (A.yperm ? A.yperm[leaf * Lf + rr + r] : leaf * Lf + rr + r);
                v.y = conj_im(v.y, cj);
                Y[row + (int64_t)col * A.ldy] = v;
              }
            });
            acc.zero();
          }
          __syncwarp();
          if (lane == 0 && !(diag & 1)) {
            if (atom_add_release_page(&pcnt[slot], 1) == (rnd + 1) * nact - 1) str.issue_page(j + NP);
          }
          ++j;
          if (++slot == NP) {
            slot = 0;
            ph ^= 1;
            ++rnd;
          }
        }
        }
        cur = rd ^ 1;
        continue;  // (always the last op; one slot per warp)
      }
      if (LEAF_OK && op.kind == FK_LEAF_IN) {
        if constexpr (LEAF_OK) {
        // fused column leaf (a1): z = A (16 x leaf) X(rows of this slot's leaf, tile); every page
        // carries SPL k-steps of A records and of X rows (the 2-D TMA tiles of Stream::issue_page)
        constexpr int SPL = St::SPL;
        const bool cj = A.conj_io != 0;
        const int cx = half * FAST_HC + c0w;  // first column of this warp inside the 32-column X tile
        const int n = op.nsteps;
        for (int s0 = 0; s0 < n; s0 += SPL) {
          if (!(diag & 1)) mbar_wait(&full[slot], ph, 4);
          const unsigned char* pg = ring + (size_t)slot * Cfg::PG;
          const E* xt = reinterpret_cast<const E*>(pg + SPL * S * FAST_FRAG + o * St::XT);
#pragma unroll
          for (int st = 0; st < SPL; ++st) {
            typename Pol::FFrags f;
            Pol::load_fa(f, pg + (st * S + o) * FAST_FRAG, lane);
            Pol::load_b_col(f, xt, SPL * Pol::KS, st * Pol::KS, cx, g, t, cj);
            acc.mac(f);
          }
          __syncwarp();
          if (lane == 0 && !(diag & 1)) {
            if (atom_add_release_page(&pcnt[slot], 1) == (rnd + 1) * nact - 1) str.issue_page(j + NP);
          }
          ++j;
          if (++slot == NP) {
            slot = 0;
            ph ^= 1;
            ++rnd;
          }
        }
        }
      } else {
      // every op of a pass is a pair op of NSTEP = 32 / KS k-steps (the centre is folded into
      // R^{lc} / W^{lc} at create), so the k-step loop is fully unrolled, software-pipelined
      // across page boundaries: the operands of k-step k + 1 load while k-step k's MMAs issue
      constexpr int NSTEP = 2 * FAST_RANK / Pol::KS;
      constexpr int SPO = SPP < NSTEP ? SPP : NSTEP;  // k-steps per page of an op
      static_assert(NSTEP % SPO == 0, "pages must split ops evenly");
      auto bsrc = [&](int k) { return (k < KPS ? sp0 : sp1) + (k & (KPS - 1)) * Pol::KS * FAST_HC; };
      if (!(diag & 1)) mbar_wait(&full[slot], ph, 4);
      const int roff = o * FAST_FRAG + Pol::rec_off(c0w);  // the warp's part of its slot's records
      const unsigned char* pgn = ring + (size_t)slot * Cfg::PG + roff;
      int nslot = slot;
      uint32_t nph = ph;
      typename Pol::FFrags f[2];
      Pol::load_fa(f[0], pgn, lane);
      Pol::load_b(f[0], bsrc(0), bo);
#pragma unroll
      for (int k = 0; k < NSTEP; ++k) {
        if (k + 1 < NSTEP) {
          const int k1 = k + 1;
          if (k1 % SPO == 0) {  // k-step k1 is on the next page
            if (++nslot == NP) {
              nslot = 0;
              nph ^= 1;
            }
            if (!(diag & 1)) mbar_wait(&full[nslot], nph, 4);
            pgn = ring + (size_t)nslot * Cfg::PG + roff;
          }
          Pol::load_fa(f[k1 & 1], pgn + (k1 % SPO) * S * FAST_FRAG, lane);
          Pol::load_b(f[k1 & 1], bsrc(k1), bo);
        }
        acc.mac(f[k & 1]);
        if ((k + 1) % SPO == 0 && rel) {
          // release the page; the last warp out re-arms it with page j + NP
          __syncwarp();
          if (lane == 0 && !(diag & 1)) {
            if (atom_add_release_page(&pcnt[slot], 1) == (rnd + 1) * nact - 1) str.issue_page(j + NP);
          }
          ++j;
          if (++slot == NP) {
            slot = 0;
            ph ^= 1;
            ++rnd;
          }
        }
      }
      }  // pair op
      if (last) {
        if (!(diag & 2)) {
          E* dst;
          if (P.xout && A.p2p) {  // fused exchange: straight into the receiver's recv region
            int peer = 0;
            const int64_t off =
                pass_slab_off(P, P.xout, jt, half, A.nlev, A.ntiles, a, b, P.out_s, o, A.myrank, &peer);
            dst = static_cast<E*>(A.peer[peer]) + off;
          } else {
            dst = Sout + pass_slab_off(P, P.xout, jt, half, A.nlev, A.ntiles, a, b, P.out_s, o);
          }
          Pol::store_slab(acc, dst, c0w, g, t, lane);
        }
        if (rel) cur = rd ^ 1;
      } else {
        if (!(diag & 4)) {
          // op 0 writes the buffer the previous item's last op read: the half must be past it
          if (q == 0 && sl == 0) named_sync(hbar, NACTH * 32);
          E* dst = winbuf + (rd ^ 1) * WIN + half * Cfg::WINH + o * FAST_HSLAB;
          Pol::store_slab(acc, dst, c0w, g, t, lane);
          // the next (pair) op reads other slots: their writes must be visible
          if (rel) named_sync(hbar, NACTH * 32);
        } else if (diag & 8) {  // profiling: epilogue stores without the barriers
          E* dst = winbuf + (rd ^ 1) * WIN + half * Cfg::WINH + o * FAST_HSLAB;
          Pol::store_slab(acc, dst, c0w, g, t, lane);
        } else {  // profiling: keep the accumulators live without any epilogue
          float sink = 0.f;
          acc.each(g, t, [&](int r, int c, E v) { sink += (float)v.x; });
          if (sink == 1.2345f) winbuf[0] = E{};
        }
        if (rel) rd ^= 1;
      }
      }  // slots of the warp
    }
  }
}

const char* fast_kernel_name(int dtype) { return dtype == BF_C128 ? "k_bf_pass<c128>" : "k_bf_pass<c64>"; }

template <class Pol, int D, int HV, int PGB = 32768>
static void launch_hv(const FastArgs& a, unsigned grid, cudaStream_t st) {
  static std::atomic<size_t> attr[BF_MAX_DEVICES];
  const size_t smem = PassCfg<Pol, D, HV, PGB>::smem();
  static_assert(PassCfg<Pol, D, HV, PGB>::smem() <= 227 * 1024, "pass kernel shared memory");
  ensure_smem_attr(attr, (const void*)k_bf_pass<Pol, D, HV, PGB>, smem);
  launch_pdl(k_bf_pass<Pol, D, HV, PGB>, grid, FAST_THREADS, smem, st, a);
}

template <class Pol, int D>
static void launch_one(const FastArgs& a, unsigned grid, cudaStream_t st) {
  if (a.halves <= 1) launch_hv<Pol, D, 1>(a, grid, st);
  else launch_hv<Pol, D, 2>(a, grid, st);
}

// nrhs 9-16 (one column half): all 16 warps on it (HV = 3) instead of 8 (HV = 1, the other 8 idle);
// env BF_NO_HV3 keeps HV = 1 (A/B)
static bool use_hv3(const FastArgs& a) {
  static const bool off = getenv("BF_NO_HV3") != nullptr;
  return a.halves == 1 && !off;
}

void launch_fast_pass(int dtype, const FastArgs& a, cudaStream_t st) {
  const int nsm = device_sm_count();
  const int64_t items = a.p.nwin * ((a.nrhs + FAST_NB - 1) / FAST_NB);  // (window, rhs tile)
  const unsigned grid = (unsigned)(items < nsm ? items : nsm);
  const int d = a.p.d;
  if (dtype == BF_C128 && a.halves == 0) {  // nrhs <= 8: 8 columns per warp, a warp per slot
    if (d == 3) launch_hv<PolC128<1>, 3, 0>(a, grid, st);
    else if (d == 2) launch_hv<PolC128<1>, 2, 0>(a, grid, st);
    else launch_hv<PolC128<1>, 1, 0>(a, grid, st);
  } else if (dtype == BF_C128) {
    // 16 KB ring pages (six instead of three 32 KB ones: a page is released after 2 k-steps, so
    // the two column halves may drift further apart) for 3-level passes without leaf ops; env
    // BF_PASS_SMALLPG = 1 (A/B measurement)
    static const bool small_pg = getenv("BF_PASS_SMALLPG") && atoi(getenv("BF_PASS_SMALLPG")) != 0;
    const bool leaf_ops = a.p.xleaf || a.p.ops[a.p.nops - 1].kind == FK_LEAF_OUT;
    if (small_pg && d == 3 && a.halves == 2 && !leaf_ops) {
      launch_hv<PolC128<2>, 3, 2, 16384>(a, grid, st);
      return;
    }
    if (use_hv3(a)) {
      if (d == 3) launch_hv<PolC128<1>, 3, 3>(a, grid, st);
      else if (d == 2) launch_hv<PolC128<1>, 2, 3>(a, grid, st);
      else launch_hv<PolC128<1>, 1, 3>(a, grid, st);
      return;
    }
    if (d == 3) launch_one<PolC128<2>, 3>(a, grid, st);
    else if (d == 2) launch_one<PolC128<2>, 2>(a, grid, st);  // 8 warps x 16 columns: 3 % faster than 16 x 8
    else launch_one<PolC128<1>, 1>(a, grid, st);
  } else {
    if (use_hv3(a)) {
      if (d == 4) launch_hv<PolC64T<2>, 4, 3>(a, grid, st);
      else if (d == 3) launch_hv<PolC64T<2>, 3, 3>(a, grid, st);
      else if (d == 2) launch_hv<PolC64T<1>, 2, 3>(a, grid, st);
      else launch_hv<PolC64T<1>, 1, 3>(a, grid, st);
      return;
    }
    if (d == 4) launch_one<PolC64T<2>, 4>(a, grid, st);
    else if (d == 3) launch_one<PolC64T<2>, 3>(a, grid, st);
    else if (d == 2) launch_one<PolC64T<1>, 2>(a, grid, st);
    else launch_one<PolC64T<1>, 1>(a, grid, st);
  }
}

}  // namespace bfa
