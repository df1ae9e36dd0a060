// Device kernels of libbfapply (sm_100a).
//
// Every stage of the butterfly apply -- the V^0 leaf products, the W^l transfer stages,
// the centre B^{lc}, the R^l transfer stages and the U^L leaf products (Eq. 3.3,
// P:318-354), forward or conjugate-transposed -- and every HOD-BF round is a
// batch of independent small complex products
//        out_task = sum_t A_t In_t            (A_t: m x k_t factor block or view)
// described by Task / Term tables built once at create time (plan.cu).  The generic
// kernel below runs one task x 32 right-hand sides per CTA:
//   * lanes map to right-hand sides, so every slab read/write is a coalesced row of
//     nrhs complex values (the slab space stores each slab rank x nrhs, nrhs fastest);
//   * factor chunks and input chunks are staged in shared memory; factor entries are
//     read back as warp-wide broadcasts;
//   * user X / Y (column-major, leaf rows gathered / scattered through the tree
//     permutation) are staged through shared memory so global accesses run along rows.
#include "common.cuh"

namespace bfa {

template <typename V>
struct Scalar;
template <>
struct Scalar<double2> {
  using R = double;
};
template <>
struct Scalar<float2> {
  using R = float;
};

template <typename V>
__device__ __forceinline__ V vzero() {
  V v;
  v.x = 0;
  v.y = 0;
  return v;
}

// ------------------------------------------------------------------------------------
// generic gather-sum product kernel
// ------------------------------------------------------------------------------------
template <typename V, int RPT>
__global__ void __launch_bounds__(128) k_stage_generic(StageArgs a) {
  using R = typename Scalar<V>::R;
  constexpr int NT = 128, KC = 32, NR = 4 * RPT;
  __shared__ V sA[KC][NR];
  __shared__ V sIn[KC][33];
  const Task t = a.tasks[blockIdx.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j0 = blockIdx.y * 32;
  const int jn = min(32, a.nrhs - j0);
  const V* __restrict__ pool = static_cast<const V*>(a.pool);
  const V* __restrict__ X = static_cast<const V*>(a.X);
  V* __restrict__ S = static_cast<V*>(a.S);
  V* __restrict__ Y = static_cast<V*>(a.Y);

  for (int r0 = 0; r0 < t.m; r0 += NR) {
    const int rn = min(NR, t.m - r0);
    R ax[RPT], ay[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) ax[q] = ay[q] = R(0);
    for (int q = 0; q < t.nterm; ++q) {
      const Term tm = a.terms[t.term0 + q];
      const bool cj = (tm.conj != 0) != (a.conj_flip != 0);
      for (int kc = 0; kc < tm.k; kc += KC) {
        const int kn = min(KC, tm.k - kc);
        __syncthreads();
        if (tm.in_kind == 0) {
          const V* src = S + (tm.in_row + kc) * a.ldS + j0;
          for (int e = threadIdx.x; e < KC * 32; e += NT) {
            const int kk = e >> 5, jj = e & 31;
            sIn[kk][jj] = (kk < kn && jj < jn) ? src[(int64_t)kk * a.ldS + jj] : vzero<V>();
          }
        } else {
          for (int e = threadIdx.x; e < KC * 32; e += NT) {
            const int kk = e & 31, jj = e >> 5;
            V v = vzero<V>();
            if (kk < kn && jj < jn) {
              const int64_t p = tm.in_row + kc + kk;
              const int64_t row = a.xperm ? a.xperm[p] : p;
              v = X[row + (int64_t)(j0 + jj) * a.ldx];
            }
            sIn[kk][jj] = v;
          }
        }
        for (int e = threadIdx.x; e < KC * NR; e += NT) {
          int ii, kk;
          if (tm.a_rs == 1) {
            ii = e % NR;
            kk = e / NR;
          } else {
            kk = e % KC;
            ii = e / KC;
          }
          V v = vzero<V>();
          if (ii < rn && kk < kn) {
            v = pool[tm.a_off + (int64_t)(r0 + ii) * tm.a_rs + (int64_t)(kc + kk) * tm.a_cs];
            if (cj) v.y = -v.y;
          }
          sA[kk][ii] = v;
        }
        __syncthreads();
        for (int kk = 0; kk < kn; ++kk) {
          const V x = sIn[kk][lane];
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const V av = sA[kk][w * RPT + q];
            ax[q] = fma(av.x, x.x, ax[q]);
            ax[q] = fma(-av.y, x.y, ax[q]);
            ay[q] = fma(av.x, x.y, ay[q]);
            ay[q] = fma(av.y, x.x, ay[q]);
          }
        }
      }
    }
    if (a.out_kind == 0) {
      if (lane < jn) {
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const int i = w * RPT + q;
          if (i < rn) {
            V v;
            v.x = ax[q];
            v.y = ay[q];
            S[(t.out_row + r0 + i) * a.ldS + j0 + lane] = v;
          }
        }
      }
    } else {
      __syncthreads();
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        V v;
        v.x = ax[q];
        v.y = ay[q];
        sIn[w * RPT + q][lane] = v;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < NR * 32; e += NT) {
        const int ii = e % NR, jj = e / NR;
        if (ii < rn && jj < jn) {
          const int64_t p = t.out_row + r0 + ii;
          const int64_t row = a.yperm ? a.yperm[p] : p;
          Y[row + (int64_t)(j0 + jj) * a.ldy] = sIn[ii][jj];
        }
      }
    }
  }
}

template <typename V>
static void launch_generic(const Round& r, StageArgs a, cudaStream_t st) {
  a.tasks = r.tasks;
  a.terms = r.terms;
  a.out_kind = r.out_kind;
  dim3 grid(r.ntasks, (a.nrhs + 31) / 32);
  if (r.max_m <= 16)
    k_stage_generic<V, 4><<<grid, 128, 0, st>>>(a);
  else
    k_stage_generic<V, 8><<<grid, 128, 0, st>>>(a);
}

const char* round_kernel_name(int dtype, const Round& r, int* id) {
  const bool big = r.max_m > 16;
  if (id) *id = big ? 2 : 1;
  if (dtype == BF_C128) return big ? "k_stage_generic<double2,8>" : "k_stage_generic<double2,4>";
  return big ? "k_stage_generic<float2,8>" : "k_stage_generic<float2,4>";
}

void launch_round(int dtype, const Round& r, StageArgs a, cudaStream_t st) {
  if (r.ntasks == 0) return;
  if (dtype == BF_C128)
    launch_generic<double2>(r, a, st);
  else
    launch_generic<float2>(r, a, st);
}

}  // namespace bfa
