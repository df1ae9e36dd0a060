// Device kernels of libbfapply (sm_100a).
//
// Every stage of the butterfly apply -- the V^0 leaf products, the W^l transfer stages,
// the centre B^{lc}, the R^l transfer stages and the U^L leaf products (Eq. 3.3,
// P:318-354), forward or conjugate-transposed -- and every HOD-BF round is a
// batch of independent small complex products
//        out_task = sum_t A_t In_t            (A_t: m x k_t factor block or view)
// described by Task / Term tables built once at create time (plan.cu).  This generic path
// serves ragged ranks (kernel-compressed butterflies, HOD-BF, the distributed split); the
// uniform rank-16 case has its own fused kernels (fast.cu, leaf.cu).
#include <algorithm>
#include <type_traits>

#include "mma.cuh"

namespace bfa {

// ------------------------------------------------------------------------------------
// tensor-core gather-sum kernel (the same Task / Term tables).  One CTA (8 warps) computes a
// 32-row x 64-column tile of one task's output: per term, K is streamed in chunks of 16 through
// two shared-memory stages (cp.async, zero-filled outside the task's rows, the term's K and
// nrhs), so every A element is read once per 64 columns and every input row once per 32 output
// rows (the L2 traffic of per-warp direct loads bound the previous version at ~10 TF).  Warp w
// computes rows 16 (w & 1).. and columns 16 (w >> 1).. with the 3M complex product (DMMA for
// complex128, 3xTF32 for complex64), or 4M when every factor entry is 0 / +-1 / +-i (selection
// blocks: the 4M product keeps those applies exact; StageArgs::m3).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async_el(void* dst, const void* src, bool ok, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}

template <class Pol>
struct TileCfg {
  using E = typename Pol::E;
  static constexpr int TR = 32, TC = 64, KC = 16;       // tile rows (64: slower), columns, K chunk (8 / 32: slower)
  static constexpr int SA = sizeof(E) == 16 ? 34 : 36;  // padded strides (bank-conflict free
  static constexpr int SB = sizeof(E) == 16 ? 66 : 68;  //   fragment reads)
  static constexpr int STAGE = KC * (SA + SB);          // elements per stage
  static constexpr int NST = 2;                         // cp.async stages (3 measured no faster)
};

// fragments of k-step k0 of a staged chunk: A tile [k][row] (stride SA), B tile [k][col] (SB)
// (M3: also the 3M sums re + im of both operands)
template <bool M3, int NT>
__device__ __forceinline__ void tile_frags(PolC128<NT>, typename PolC128<NT>::Frags& f, const double2* sA, const double2* sB, int wr,
                                           int wc, int k0, int g, int t, bool cj) {
  using C = TileCfg<PolC128<NT>>;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    double2 v = sA[(k0 + t) * C::SA + wr + 8 * mi + g];
    v.y = conj_im(v.y, cj);
    f.a[mi] = v;
    if (M3) f.as[mi] = v.x + v.y;
  }
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) {
    f.b[ni] = sB[(k0 + t) * C::SB + wc + 8 * ni + g];
    if (M3) f.bs[ni] = f.b[ni].x + f.b[ni].y;
  }
}
template <bool M3, int NT>
__device__ __forceinline__ void tile_frags(PolC64<NT>, typename PolC64<NT>::Frags& f, const float2* sA, const float2* sB, int wr,
                                           int wc, int k0, int g, int t, bool cj) {
  using P = PolC64<NT>;
  using C = TileCfg<P>;
  float2 v[4];
  v[0] = sA[(k0 + t) * C::SA + wr + g];
  v[1] = sA[(k0 + t) * C::SA + wr + g + 8];
  v[2] = sA[(k0 + t + 4) * C::SA + wr + g];
  v[3] = sA[(k0 + t + 4) * C::SA + wr + g + 8];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    v[e].y = conj_im(v[e].y, cj);
    P::split(v[e].x, f.ah[0][e], f.al[0][e]);
    P::split(v[e].y, f.ah[1][e], f.al[1][e]);
    if (M3) P::split(v[e].x + v[e].y, f.ah[2][e], f.al[2][e]);
  }
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) {
    f.b[ni][0] = sB[(k0 + t) * C::SB + wc + 8 * ni + g];
    f.b[ni][1] = sB[(k0 + t + 4) * C::SB + wc + 8 * ni + g];
  }
}

// A/B knob (build with -DBF_TILE_KSKIP=0): run every k-step of a K chunk, including the zero-filled
// rows past a term's K
#ifndef BF_TILE_KSKIP
#define BF_TILE_KSKIP 1
#endif
__device__ __forceinline__ constexpr bool tile_kskip() { return BF_TILE_KSKIP != 0; }

template <class Pol, bool M3, int MINB = 2>
__global__ void __launch_bounds__(256, MINB) k_stage_tile(StageArgs a) {
  using E = typename Pol::E;
  using C = TileCfg<Pol>;
  constexpr int KS = Pol::KS, TR = C::TR, TC = C::TC, KC = C::KC, SA = C::SA, SB = C::SB;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  E* sm = reinterpret_cast<E*>(sm_raw);  // C::NST stages of [A: KC x SA][B: KC x SB]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int2 un = a.units[blockIdx.x];  // plan tables: immutable, read before the PDL wait
  const Task tk = a.tasks[un.x];
  pdl_wait();  // slabs / X / Y of the previous rounds (programmatic dependent launch)
  const int r0 = un.y * TR;
  const int j0 = blockIdx.y * TC;
  if (a.cols) {  // bf_extract: only the column tiles the task's output has nonzeros in
    const int2 cr = a.cols[un.x];
    if (j0 >= cr.y || j0 + TC <= cr.x) return;
  }
  const int g = lane >> 2, t = lane & 3;
  const int wr = 16 * (w & 1), wc = 16 * (w >> 1);  // warp tile origin inside the CTA tile
  const E* __restrict__ pool = static_cast<const E*>(a.pool);
  const E* __restrict__ S = static_cast<const E*>(a.S);
  const E* __restrict__ X = static_cast<const E*>(a.X);

  // chunk c of the flattened (term, K chunk) sequence -> stage c % NST
  int q_ld = 0, kc_ld = 0;  // next chunk to load
  auto load = [&](int stg) {
    if (q_ld >= tk.nterm) return;
    const Term tm = a.terms[tk.term0 + q_ld];
    E* sA = sm + stg * C::STAGE;
    E* sB = sA + KC * SA;
    // A: TR x KC at (r0, kc_ld); lanes along the contiguous dimension of the factor view
#pragma unroll
    for (int e = 0; e < TR * KC / 256; ++e) {
      const int x = tid + 256 * e;
      int i, k;
      if (tm.a_rs == 1) {
        i = x % TR;
        k = x / TR;
      } else {
        k = x % KC;
        i = x / KC;
      }
      const bool ok = r0 + i < tk.m && kc_ld + k < tm.k;
      const E* src = pool + (ok ? tm.a_off + (int64_t)(r0 + i) * tm.a_rs + (int64_t)(kc_ld + k) * tm.a_cs : 0);
      cp_async_el(sA + k * SA + i, src, ok, (int)sizeof(E));
    }
    // B: KC x TC input rows (kc_ld..) x columns (j0..)
#pragma unroll
    for (int e = 0; e < KC * TC / 256; ++e) {
      const int x = tid + 256 * e;
      int k, j;
      if (tm.in_kind == 0) {  // slab rows: columns contiguous
        j = x % TC;
        k = x / TC;
      } else {  // user X (column-major): rows contiguous
        k = x % KC;
        j = x / KC;
      }
      const bool ok = kc_ld + k < tm.k && j0 + j < a.nrhs;
      const E* src = S;
      if (ok) {
        const int64_t p = tm.in_row + kc_ld + k;
        src = tm.in_kind == 0 ? S + p * a.ldS + j0 + j : X + (a.xperm ? a.xperm[p] : p) + (int64_t)(j0 + j) * a.ldx;
      }
      cp_async_el(sB + k * SB + j, src, ok, (int)sizeof(E));
    }
    kc_ld += KC;
    if (kc_ld >= tm.k) {
      kc_ld = 0;
      ++q_ld;
    }
  };

  std::conditional_t<M3, typename Pol::Acc, typename Pol::Acc4> acc;
  acc.zero();
#pragma unroll
  for (int st = 0; st < C::NST - 1; ++st) {
    load(st);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  int c = 0;
  for (int q = 0; q < tk.nterm; ++q) {
    const Term tm = a.terms[tk.term0 + q];
    const bool cj = (tm.conj != 0) != (a.conj_flip != 0);
    for (int kc = 0; kc < tm.k; kc += KC, ++c) {
      load((c + C::NST - 1) % C::NST);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group %0;\n" ::"n"(C::NST - 1) : "memory");
      __syncthreads();
      const E* sA = sm + (c % C::NST) * C::STAGE;
      const E* sB = sA + KC * SA;
      const int kvalid = tile_kskip() ? tm.k - kc : KC;  // k-steps past the term's K only add zeros
#pragma unroll
      for (int k0 = 0; k0 < KC; k0 += KS) {
        if (k0 >= kvalid) break;
        typename Pol::Frags f;
        tile_frags<M3>(Pol{}, f, sA, sB, wr, wc, k0, g, t, cj);
        acc.mac(f);
      }
      __syncthreads();
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  pdl_trigger();  // the next round's CTAs may launch once every CTA of this one is storing
  const int rb = r0 + wr, cb = j0 + wc;
  if (a.out_kind == 0) {
    E* Sd = static_cast<E*>(a.S);
    acc.each(g, t, [&](int r, int cc, E v) {
      if (rb + r < tk.m && cb + cc < a.nrhs) Sd[(tk.out_row + rb + r) * a.ldS + cb + cc] = v;
    });
  } else {
    E* Y = static_cast<E*>(a.Y);
    acc.each(g, t, [&](int r, int cc, E v) {
      if (rb + r < tk.m && cb + cc < a.nrhs) {
        const int64_t p = tk.out_row + rb + r;
        Y[(a.yperm ? a.yperm[p] : p) + (int64_t)(cb + cc) * a.ldy] = v;
      }
    });
  }
}

// ------------------------------------------------------------------------------------
// Persistent, transposed-orientation gather-sum (complex128; SURVEY 7.3 hard part 2, VERDICT r1
// item 3):   out^T (nrhs x m) = sum_t In_t^T (nrhs x k) A_t^T (k x m)
// * M of the MMA is the right-hand sides (a multiple of 8) and N the task's output rows, padded
//   only to 8 (runtime n-tile count) instead of to the 32-row tile: the ragged small ranks of the
//   kernel-compressed butterflies and HOD-BF (configs 2-4, ranks ~6-70) waste far fewer DMMAs.
// * Persistent: a grid of 2 CTAs per SM walks the round's items (unit = (task, 32-row block)) x
//   64-column tile) with a cp.async ring of NST K-chunks whose loader runs NST - 1 chunks ahead
//   ACROSS item boundaries, so the first loads of the next item overlap the current item's MMAs
//   and epilogue (the one-item-per-CTA version paid a full load latency per item: each item is
//   only ~2-5 chunks of 16).
// Warp w owns the 8 columns 8w.. of the item's tile and every 8-row n-tile holding task rows:
//   A frag (8 x 4, [nrhs][k]) of lane (g, t) = In(k0 + t, 8w + g)
//   B frag (4 x 8, [k][row])  of lane (g, t) = A(8 nt + g, k0 + t)
//   C (8 x 8)  c[g][2t + e]   = out(row 8 nt + 2t + e, column 8w + g)
// ------------------------------------------------------------------------------------
// A/B knob (build with -DBF_TILE_BRANCHY=1): the round-2 first-cut k-loop with a per-n-tile branch
#ifndef BF_TILE_BRANCHY
#define BF_TILE_BRANCHY 0
#endif
__device__ __forceinline__ constexpr bool tile_branchy() { return BF_TILE_BRANCHY != 0; }

template <bool M3, int NST, int MINB = 2>
__global__ void __launch_bounds__(256, MINB) k_stage_tileT(StageArgs a) {
  using E = double2;
  using C = TileCfg<PolC128<2>>;
  constexpr int TR = C::TR, TC = C::TC, KC = C::KC, SA = C::SA, SB = C::SB, STAGE = C::STAGE;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  E* sm = reinterpret_cast<E*>(sm_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ctiles = (a.nrhs + TC - 1) / TC;
  const int64_t nitems = (int64_t)a.nunits * ctiles;
  // the CTA's items: one unit with all its column tiles (grid = units; the loader runs ahead across
  // the column tiles), or a persistent stride over every item (grid < units x tiles)
  const bool per_unit = gridDim.x == (unsigned)a.nunits;
  const int64_t i0 = per_unit ? (int64_t)blockIdx.x * ctiles : blockIdx.x;
  const int64_t i1 = per_unit ? i0 + ctiles : nitems;
  const int64_t istep = per_unit ? 1 : gridDim.x;
  const E* __restrict__ pool = static_cast<const E*>(a.pool);
  const E* __restrict__ S = static_cast<const E*>(a.S);
  const E* __restrict__ X = static_cast<const E*>(a.X);
  pdl_wait();  // slabs / X / Y of the previous rounds
  // ---- loader: its own walk over (item, term, K chunk), NST - 1 chunks ahead of the consumer
  int64_t l_item = i0;
  int l_q = 0, l_kc = 0;
  Task l_tk{};
  int l_r0 = 0, l_j0 = 0;
  auto l_fetch = [&]() {  // task of l_item; skips items without terms (they consume no chunk)
    for (; l_item < i1; l_item += istep) {
      const int2 un = a.units[l_item / ctiles];
      l_tk = a.tasks[un.x];
      l_r0 = un.y * TR;
      l_j0 = (int)(l_item % ctiles) * TC;
      bool skip = l_tk.nterm == 0;
      if (!skip && a.cols) {
        const int2 cr = a.cols[un.x];
        skip = l_j0 >= cr.y || l_j0 + TC <= cr.x;
      }
      if (!skip) return;
    }
  };
  l_fetch();
  auto load = [&](int stg) {
    if (l_item >= i1) return;
    const Term tm = a.terms[l_tk.term0 + l_q];
    E* sA = sm + stg * STAGE;
    E* sB = sA + KC * SA;
#pragma unroll
    for (int e = 0; e < TR * KC / 256; ++e) {
      const int x = tid + 256 * e;
      int i, k;
      if (tm.a_rs == 1) {
        i = x % TR;
        k = x / TR;
      } else {
        k = x % KC;
        i = x / KC;
      }
      const bool ok = l_r0 + i < l_tk.m && l_kc + k < tm.k;
      const E* src = pool + (ok ? tm.a_off + (int64_t)(l_r0 + i) * tm.a_rs + (int64_t)(l_kc + k) * tm.a_cs : 0);
      cp_async_el(sA + k * SA + i, src, ok, 16);
    }
#pragma unroll
    for (int e = 0; e < KC * TC / 256; ++e) {
      const int x = tid + 256 * e;
      int k, j;
      if (tm.in_kind == 0) {
        j = x % TC;
        k = x / TC;
      } else {
        k = x % KC;
        j = x / KC;
      }
      const bool ok = l_kc + k < tm.k && l_j0 + j < a.nrhs;
      const E* src = S;
      if (ok) {
        const int64_t p = tm.in_row + l_kc + k;
        src = tm.in_kind == 0 ? S + p * a.ldS + l_j0 + j : X + (a.xperm ? a.xperm[p] : p) + (int64_t)(l_j0 + j) * a.ldx;
      }
      cp_async_el(sB + k * SB + j, src, ok, 16);
    }
    l_kc += KC;
    if (l_kc >= tm.k) {
      l_kc = 0;
      if (++l_q >= l_tk.nterm) {
        l_q = 0;
        l_item += istep;
        l_fetch();
      }
    }
  };
#pragma unroll
  for (int st = 0; st < NST - 1; ++st) {
    load(st);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  const int cw = 8 * w;
  int c = 0;  // consumed chunks
  for (int64_t item = i0; item < i1; item += istep) {
    const int2 un = a.units[item / ctiles];
    const Task tk = a.tasks[un.x];
    const int r0 = un.y * TR, j0 = (int)(item % ctiles) * TC;
    if (a.cols) {
      const int2 cr = a.cols[un.x];
      if (j0 >= cr.y || j0 + TC <= cr.x) continue;  // bf_extract: column tile outside the task's range
    }
    const int ntiles = min(4, (tk.m - r0 + 7) >> 3);  // 8-row n-tiles holding task rows
    double acc[3][4][2];
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) acc[q][nt][0] = acc[q][nt][1] = 0.0;
    for (int q = 0; q < tk.nterm; ++q) {
      const Term tm = a.terms[tk.term0 + q];
      const bool cj = (tm.conj != 0) != (a.conj_flip != 0);
      for (int kc = 0; kc < tm.k; kc += KC, ++c) {
        load((c + NST - 1) % NST);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group %0;\n" ::"n"(NST - 1) : "memory");
        __syncthreads();
        const E* sA = sm + (c % NST) * STAGE;
        const E* sB = sA + KC * SA;
        // one chunk with the n-tile count a compile-time constant: every fragment of a k-step
        // is loaded (and its 3M sum formed) before its DMMAs issue, with no per-n-tile branch
        // between them (the branchy form left the DMMAs waiting on each load / DADD in turn --
        // ncu: "wait" and short-scoreboard stalls led, DMMA 45 % active)
        // k-steps holding term rows: the chunk's tail beyond tm.k is zero-filled shared memory, whose
        // DMMAs would only add zeros (ragged K = r1 + r2 pads up to 15 rows per term otherwise)
        const int kvalid = tile_kskip() ? tm.k - kc : KC;
        auto chunk = [&](auto ntc) {
          constexpr int NTL = decltype(ntc)::value;
#pragma unroll
          for (int k0 = 0; k0 < KC; k0 += 4) {
            if (k0 >= kvalid) break;
            const E x = sB[(k0 + t) * SB + cw + g];  // In^T fragment
            E f[NTL];
            double fs[NTL];
#pragma unroll
            for (int nt = 0; nt < NTL; ++nt) {
              f[nt] = sA[(k0 + t) * SA + 8 * nt + g];  // A^T fragment
              f[nt].y = conj_im(f[nt].y, cj);
              fs[nt] = f[nt].x + f[nt].y;
            }
            const double xs = x.x + x.y;
#pragma unroll
            for (int nt = 0; nt < NTL; ++nt) {
              if (M3) {
                PolC128<1>::mma(acc[0][nt][0], acc[0][nt][1], x.x, f[nt].x);
                PolC128<1>::mma(acc[1][nt][0], acc[1][nt][1], x.y, f[nt].y);
              } else {  // 4M: re += xr fr - xi fi, im += xr fi + xi fr (exact on selection factors)
                PolC128<1>::mma(acc[0][nt][0], acc[0][nt][1], x.x, f[nt].x);
                PolC128<1>::mma(acc[0][nt][0], acc[0][nt][1], -x.y, f[nt].y);
                PolC128<1>::mma(acc[1][nt][0], acc[1][nt][1], x.x, f[nt].y);
                PolC128<1>::mma(acc[1][nt][0], acc[1][nt][1], x.y, f[nt].x);
              }
            }
            if (M3) {
#pragma unroll
              for (int nt = 0; nt < NTL; ++nt) PolC128<1>::mma(acc[2][nt][0], acc[2][nt][1], xs, fs[nt]);
            }
          }
        };
        if (!tile_branchy()) {
          switch (ntiles) {
            case 1: chunk(std::integral_constant<int, 1>{}); break;
            case 2: chunk(std::integral_constant<int, 2>{}); break;
            case 3: chunk(std::integral_constant<int, 3>{}); break;
            default: chunk(std::integral_constant<int, 4>{}); break;
          }
        } else {
#pragma unroll
        for (int k0 = 0; k0 < KC; k0 += 4) {
          const E x = sB[(k0 + t) * SB + cw + g];  // In^T fragment
          const double xs = x.x + x.y;
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            if (nt < ntiles) {
              E f = sA[(k0 + t) * SA + 8 * nt + g];  // A^T fragment
              f.y = conj_im(f.y, cj);
              if (M3) {
                PolC128<1>::mma(acc[0][nt][0], acc[0][nt][1], x.x, f.x);
                PolC128<1>::mma(acc[1][nt][0], acc[1][nt][1], x.y, f.y);
                PolC128<1>::mma(acc[2][nt][0], acc[2][nt][1], xs, f.x + f.y);
              } else {
                PolC128<1>::mma(acc[0][nt][0], acc[0][nt][1], x.x, f.x);
                PolC128<1>::mma(acc[0][nt][0], acc[0][nt][1], -x.y, f.y);
                PolC128<1>::mma(acc[1][nt][0], acc[1][nt][1], x.x, f.y);
                PolC128<1>::mma(acc[1][nt][0], acc[1][nt][1], x.y, f.x);
              }
            }
          }
        }
        }
        __syncthreads();
      }
    }
    const int col = j0 + cw + g;
    if (col < a.nrhs) {
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        if (nt >= ntiles) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = r0 + 8 * nt + 2 * t + e;
          if (r >= tk.m) continue;
          E v;
          if (M3) {
            const double p1 = acc[0][nt][e], p2 = acc[1][nt][e], p3 = acc[2][nt][e];
            v = make_double2(p1 - p2, p3 - p1 - p2);
          } else {
            v = make_double2(acc[0][nt][e], acc[1][nt][e]);
          }
          if (a.out_kind == 0) {
            static_cast<E*>(a.S)[(tk.out_row + r) * a.ldS + col] = v;
          } else {
            const int64_t p = tk.out_row + r;
            static_cast<E*>(a.Y)[(a.yperm ? a.yperm[p] : p) + (int64_t)col * a.ldy] = v;
          }
        }
      }
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  pdl_trigger();
}

template <bool M3, int NST, int MINB = 2>
static void launch_tileT_t(const StageArgs& a, cudaStream_t st) {
  using C = TileCfg<PolC128<2>>;
  constexpr size_t smem = NST * C::STAGE * sizeof(double2);
  static std::atomic<size_t> attr[BF_MAX_DEVICES];
  ensure_smem_attr(attr, (const void*)k_stage_tileT<M3, NST, MINB>, smem);
  // grid: one CTA per unit walking all its column tiles (the loader runs ahead across them) when
  // the round has enough units to fill the SMs (>= 4 per SM), else one CTA per (unit, column tile)
  // -- config 4: 18.7 vs 19.6 ms, config 3's small late rounds: per-item is faster.  BF_TILE_GRID
  // = 0 / 1 forces either, 2 = a persistent stride (2 CTAs per SM; config 3 1.67 vs 1.48 ms: a static
  // stride balances the uneven items worse than the hardware scheduler).
  static const int gm = getenv("BF_TILE_GRID") ? atoi(getenv("BF_TILE_GRID")) : -1;
  const int64_t ct = (a.nrhs + C::TC - 1) / C::TC;
  const int64_t items = (int64_t)a.nunits * ct;
  const int nsm = device_sm_count();
  const int mode = gm >= 0 ? gm : (a.nunits >= 4LL * nsm ? 1 : 0);
  int64_t grid = mode == 1 ? a.nunits : mode == 0 ? items : std::min<int64_t>(items, 2LL * nsm);
  if (mode != 1 && ct > 1 && grid == a.nunits) grid = std::max<int64_t>(1, grid - 1);  // stride mode, not per-unit
  launch_pdl(k_stage_tileT<M3, NST, MINB>, (unsigned)grid, 1u, 256, smem, st, a);
}

// ------------------------------------------------------------------------------------
// Narrow right-hand-side blocks (nrhs <= 4, the solve regime of P:697): the round's products
// are matrix-vector products, bound by reading the factor entries once.  CUDA-core FMAs, one
// warp per unit (task, 32-row block), lane = output row, persistent grid-stride over units;
// per k the lanes read one factor column (coalesced for op N, a_rs = 1) and broadcast-read the
// k-th input row.
// ------------------------------------------------------------------------------------
template <typename V, int NR>
__global__ void __launch_bounds__(256) k_stage_gemv(StageArgs a) {
  using T = decltype(V{}.x);
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const V* __restrict__ pool = static_cast<const V*>(a.pool);
  const V* __restrict__ S = static_cast<const V*>(a.S);
  const V* __restrict__ X = static_cast<const V*>(a.X);
  pdl_wait();
  for (int64_t u = wid; u < a.nunits; u += nw) {
    const int2 un = a.units[u];
    const Task tk = a.tasks[un.x];
    const int r = un.y * 32 + lane;
    const bool act = r < tk.m;
    T re[NR], im[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) re[j] = im[j] = 0;
    for (int q = 0; q < tk.nterm; ++q) {
      const Term tm = a.terms[tk.term0 + q];
      const bool cj = (tm.conj != 0) != (a.conj_flip != 0);
      const V* Ar = pool + tm.a_off + (int64_t)(act ? r : 0) * tm.a_rs;
#pragma unroll 4
      for (int k = 0; k < tm.k; ++k) {
        V f = act ? __ldg(Ar + (int64_t)k * tm.a_cs) : V{};
        f.y = conj_im(f.y, cj);
        const int64_t p = tm.in_row + k;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          V x = V{};
          if (j < a.nrhs) x = tm.in_kind == 0 ? S[p * a.ldS + j] : X[(a.xperm ? a.xperm[p] : p) + (int64_t)j * a.ldx];
          re[j] = fma(f.x, x.x, re[j]);
          re[j] = fma(-f.y, x.y, re[j]);
          im[j] = fma(f.x, x.y, im[j]);
          im[j] = fma(f.y, x.x, im[j]);
        }
      }
    }
    if (!act) continue;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j >= a.nrhs) break;
      V v;
      v.x = re[j];
      v.y = im[j];
      if (a.out_kind == 0) {
        static_cast<V*>(a.S)[(tk.out_row + r) * a.ldS + j] = v;
      } else {
        const int64_t p = tk.out_row + r;
        static_cast<V*>(a.Y)[(a.yperm ? a.yperm[p] : p) + (int64_t)j * a.ldy] = v;
      }
    }
  }
  pdl_trigger();
}

template <typename V, int NR>
static void launch_gemv_t(const StageArgs& a, cudaStream_t st) {
  const int64_t warps = a.nunits;
  const int64_t cap = 16LL * device_sm_count() * 8;  // 16 CTAs of 8 warps per SM
  const int64_t w = warps < cap ? warps : cap;
  launch_pdl(k_stage_gemv<V, NR>, (unsigned)((w + 7) / 8), 1u, 256, 0, st, a);
}

template <class Pol, bool M3, int MINB>
static void launch_tile_t(dim3 grid, const StageArgs& a, cudaStream_t st) {
  constexpr size_t smem = TileCfg<Pol>::NST * TileCfg<Pol>::STAGE * sizeof(typename Pol::E);
  static std::atomic<size_t> attr[BF_MAX_DEVICES];
  ensure_smem_attr(attr, (const void*)k_stage_tile<Pol, M3, MINB>, smem);
  launch_pdl(k_stage_tile<Pol, M3, MINB>, grid.x, grid.y, 256, smem, st, a);
}
// BF_TILE_MINB: CTAs per SM the tile kernels are compiled for (register cap): 3 (72-80 registers,
// no spills; 3 x 51 KB of shared memory), measured on configs 2-4 against 2
static int tile_minb() {
  static const int v = getenv("BF_TILE_MINB") ? atoi(getenv("BF_TILE_MINB")) : 3;
  return v;
}
template <class Pol>
static void launch_tile(dim3 grid, const StageArgs& a, cudaStream_t st) {
  if (tile_minb() >= 3) {
    if (a.m3) launch_tile_t<Pol, true, 3>(grid, a, st);
    else launch_tile_t<Pol, false, 3>(grid, a, st);
    return;
  }
  if (a.m3) launch_tile_t<Pol, true, 2>(grid, a, st);
  else launch_tile_t<Pol, false, 2>(grid, a, st);
}

template <typename V>
static void launch_generic(const Round& r, StageArgs a, cudaStream_t st) {
  a.tasks = r.tasks;
  a.terms = r.terms;
  a.units = r.units;
  a.nunits = r.nunits;
  a.out_kind = r.out_kind;
  a.cols = r.cols;
  dim3 grid(r.nunits, (a.nrhs + 63) / 64);  // CTA tile: 32 rows x 64 columns
  // kernel choice: nrhs <= 4 -> matrix-vector kernel; complex128 with nrhs > 8 -> the persistent
  // transposed-orientation kernel; otherwise the row-tile kernel.  (env BF_TILE = 0 forces the
  // row-tile kernel everywhere, for A/B measurements)
  // (the matrix-vector kernel k_stage_gemv measured 3.3x slower than the tile kernels on the
  // nrhs = 1 solve sweep -- one warp per small task leaves most lanes idle -- and is only
  // selected by BF_TILE = 2, for measurements)
  static const int mode = getenv("BF_TILE") ? atoi(getenv("BF_TILE")) : 1;
  if (mode == 2 && a.nrhs <= 4 && !a.cols) {
    if (a.nrhs == 1) launch_gemv_t<V, 1>(a, st);
    else if (a.nrhs == 2) launch_gemv_t<V, 2>(a, st);
    else launch_gemv_t<V, 4>(a, st);
    return;
  }
  // rounds into the slab space (leaf V, W, centre and R stages: ranks as output rows) run
  // transposed; the rounds that write user rows (leaf U blocks, HOD-BF diagonal blocks: leaf-size
  // outputs) keep the row tiles (config 3: 1.48 ms all-transposed, 1.58 row tiles; the last round
  // 0.279 vs 0.259 ms)
  if (mode && sizeof(V) == 16 && a.nrhs > 8 && r.out_kind == 0) {
    if (tile_minb() >= 3) {  // 78 registers, 3 CTAs / SM: config 3 1.47 vs 1.56 ms, config 4 17.2 vs 18.7
                              // (config 2 0.247 vs 0.237)
      if (a.m3) launch_tileT_t<true, 2, 3>(a, st);
      else launch_tileT_t<false, 2, 3>(a, st);
    } else {
      if (a.m3) launch_tileT_t<true, 2>(a, st);
      else launch_tileT_t<false, 2>(a, st);
    }
    return;
  }
  // complex64 with >= 64 right-hand sides, rounds between slab levels: the tcgen05 kernel (M = 128
  // rhs per CTA tile; env BF_UMMA = 0 keeps the mma.sync row tiles, for A/B measurements)
  static const int umma = getenv("BF_UMMA") ? atoi(getenv("BF_UMMA")) : 1;
  if (sizeof(V) == 8 && umma && mode && a.nrhs >= 64 && !a.cols &&
      (umma == 2 || (r.out_kind == 0 && r.user_in == 0))) {
    launch_tile_umma(a, st);
    return;
  }
  if (sizeof(V) == 16)
    launch_tile<PolC128<2>>(grid, a, st);
  else
    launch_tile<PolC64<2>>(grid, a, st);
}

// Y += A, column-major rows x nrhs (bf_accumulate): grid-stride over the block, one complex
// element per thread and step (HBM-bound elementwise work; coalesced along the rows)
template <typename V>
__global__ void k_accumulate(int64_t rows, int64_t nrhs, const V* __restrict__ A, int64_t lda, V* __restrict__ Y,
                             int64_t ldy) {
  const int64_t total = rows * nrhs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / rows, r = i - c * rows;
    const V a = A[r + c * lda];
    V y = Y[r + c * ldy];
    y.x += a.x;
    y.y += a.y;
    Y[r + c * ldy] = y;
  }
}

// Y += alpha A (bf_operator_apply's accumulation of one product into the sum)
template <typename V>
__global__ void k_axpy(int64_t rows, int64_t nrhs, double are, double aim, const V* __restrict__ A, int64_t lda,
                       V* __restrict__ Y, int64_t ldy) {
  const int64_t total = rows * nrhs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / rows, r = i - c * rows;
    const V a = A[r + c * lda];
    V y = Y[r + c * ldy];
    y.x += (are * a.x - aim * a.y);
    y.y += (are * a.y + aim * a.x);
    Y[r + c * ldy] = y;
  }
}

void launch_axpy(int dtype, int64_t rows, int64_t nrhs, double are, double aim, const void* A, int64_t lda, void* Y,
                 int64_t ldy, cudaStream_t st) {
  const int64_t total = rows * nrhs;
  if (total == 0) return;
  const int nsm = device_sm_count();
  const int64_t want = (total + 255) / 256;
  const unsigned grid = (unsigned)(want < 8LL * nsm ? want : 8LL * nsm);
  if (dtype == BF_C128)
    k_axpy<double2><<<grid, 256, 0, st>>>(rows, nrhs, are, aim, static_cast<const double2*>(A), lda,
                                          static_cast<double2*>(Y), ldy);
  else
    k_axpy<float2><<<grid, 256, 0, st>>>(rows, nrhs, are, aim, static_cast<const float2*>(A), lda,
                                         static_cast<float2*>(Y), ldy);
}

void launch_accumulate(int dtype, int64_t rows, int64_t nrhs, const void* A, int64_t lda, void* Y, int64_t ldy,
                       cudaStream_t st) {
  const int nsm = device_sm_count();
  const int64_t total = rows * nrhs;
  if (total == 0) return;
  const int64_t want = (total + 255) / 256;
  const unsigned grid = (unsigned)(want < 8LL * nsm ? want : 8LL * nsm);
  if (dtype == BF_C128)
    k_accumulate<double2><<<grid, 256, 0, st>>>(rows, nrhs, static_cast<const double2*>(A), lda,
                                                static_cast<double2*>(Y), ldy);
  else
    k_accumulate<float2><<<grid, 256, 0, st>>>(rows, nrhs, static_cast<const float2*>(A), lda,
                                               static_cast<float2*>(Y), ldy);
}

// bf_extract, first round (the column leaves on unit vectors, Eq. 3.3's V^0 applied to E_J):
// z^0 slab column of request j = the Vt column of that request.  jmap[j] = {slab row of the
// leaf's z^0, rank c, pool offset of the Vt column, slab column}; the slabs were zeroed before.
template <typename V>
__global__ void k_extract_vt_cols(int64_t nJ, const int64_t* __restrict__ jmap, const V* __restrict__ pool,
                                  V* __restrict__ S, int64_t ldS) {
  for (int64_t j = blockIdx.x; j < nJ; j += gridDim.x) {
    const int64_t row0 = jmap[4 * j], c = jmap[4 * j + 1], off = jmap[4 * j + 2], col = jmap[4 * j + 3];
    for (int64_t r = threadIdx.x; r < c; r += blockDim.x) S[(row0 + r) * ldS + col] = pool[off + r];
  }
}

// bf_extract, last round (Eq. 3.3's U^L restricted to the requested rows): for request-row entry
// e = {pool offset of the U row, its stride, rank r, slab row of y^L, output row, first slab
// column, column count}: out(orow, ocol[c]) = U(row, :) y^L(:, c) for its slab columns c.
template <typename V>
__global__ void k_extract_u_rows(int64_t nE, const int64_t* __restrict__ imap, const int64_t* __restrict__ ocol,
                                 const V* __restrict__ pool, const V* __restrict__ S, int64_t ldS,
                                 V* __restrict__ out, int64_t ldo) {
  for (int64_t e = blockIdx.x; e < nE; e += gridDim.x) {
    const int64_t* m = imap + 7 * e;
    const int64_t off = m[0], mt = m[1], r = m[2], row0 = m[3], orow = m[4], c0 = m[5], nc = m[6];
    for (int64_t jj = threadIdx.x; jj < nc; jj += blockDim.x) {
      const int64_t c = c0 + jj;
      decltype(V::x) re = 0, im = 0;
      for (int64_t k = 0; k < r; ++k) {
        const V u = pool[off + k * mt], y = S[(row0 + k) * ldS + c];
        re += u.x * y.x - u.y * y.y;
        im += u.x * y.y + u.y * y.x;
      }
      V o;
      o.x = re;
      o.y = im;
      out[orow + ocol[c] * ldo] = o;
    }
  }
}

// hodbf_extract: the dense-leaf entries, out[pairs[2q]] = pool[pairs[2q + 1]]
template <typename V>
__global__ void k_extract_gather(int64_t n, const int64_t* __restrict__ pairs, const V* __restrict__ pool,
                                 V* __restrict__ out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    out[pairs[2 * q]] = pool[pairs[2 * q + 1]];
}


void launch_extract_vt_cols(int dtype, int64_t nJ, const int64_t* jmap, const void* pool, void* S, int64_t ldS,
                            cudaStream_t st) {
  if (nJ == 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(nJ, 65535);
  if (dtype == BF_C128)
    k_extract_vt_cols<double2><<<grid, 64, 0, st>>>(nJ, jmap, static_cast<const double2*>(pool),
                                                    static_cast<double2*>(S), ldS);
  else
    k_extract_vt_cols<float2><<<grid, 64, 0, st>>>(nJ, jmap, static_cast<const float2*>(pool),
                                                   static_cast<float2*>(S), ldS);
}

void launch_extract_u_rows(int dtype, int64_t nE, const int64_t* imap, const int64_t* ocol, const void* pool,
                           const void* S, int64_t ldS, void* out, int64_t ldo, cudaStream_t st) {
  if (nE == 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(nE, 65535);
  if (dtype == BF_C128)
    k_extract_u_rows<double2><<<grid, 128, 0, st>>>(nE, imap, ocol, static_cast<const double2*>(pool),
                                                    static_cast<const double2*>(S), ldS, static_cast<double2*>(out), ldo);
  else
    k_extract_u_rows<float2><<<grid, 128, 0, st>>>(nE, imap, ocol, static_cast<const float2*>(pool),
                                                   static_cast<const float2*>(S), ldS, static_cast<float2*>(out), ldo);
}

void launch_extract_gather(int dtype, int64_t n, const int64_t* pairs, const void* pool, void* out, cudaStream_t st) {
  if (n == 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 4096);
  if (dtype == BF_C128)
    k_extract_gather<double2><<<grid, 256, 0, st>>>(n, pairs, static_cast<const double2*>(pool), static_cast<double2*>(out));
  else
    k_extract_gather<float2><<<grid, 256, 0, st>>>(n, pairs, static_cast<const float2*>(pool), static_cast<float2*>(out));
}

const char* round_kernel_name(int dtype, const Round& r, int* id) {
  (void)r;
  if (id) *id = 3;
  return dtype == BF_C128 ? "k_stage_tile<c128>" : "k_stage_tile<c64>";
}

void launch_round(int dtype, const Round& r, StageArgs a, cudaStream_t st) {
  if (r.ntasks == 0) return;
  if (dtype == BF_C128)
    launch_generic<double2>(r, a, st);
  else
    launch_generic<float2>(r, a, st);
}

}  // namespace bfa
