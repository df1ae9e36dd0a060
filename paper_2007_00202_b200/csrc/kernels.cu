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
#include "mma.cuh"

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
// tensor-core gather-sum kernel (the same Task / Term tables): one warp per work unit =
// (task, 16-row group) x 16 right-hand sides, 4M complex products on the tensor pipe
// (mma.cuh policies: DMMA for complex128, 3xTF32 for complex64).  Operands are read straight
// from global memory / L2 (factor blocks with arbitrary row / column strides and conjugation,
// slab rows or permuted user rows), zero-padded outside the task's rows, the term's K and nrhs.
// ------------------------------------------------------------------------------------
template <class Pol>
__device__ __forceinline__ typename Pol::E ldA(const StageArgs& a, const Term& tm, int row, int k, int m, bool cj) {
  using E = typename Pol::E;
  E v{};
  if (row < m && k < tm.k) {
    v = __ldg(static_cast<const E*>(a.pool) + tm.a_off + (int64_t)row * tm.a_rs + (int64_t)k * tm.a_cs);
    v.y = conj_im(v.y, cj);
  }
  return v;
}
template <class Pol>
__device__ __forceinline__ typename Pol::E ldB(const StageArgs& a, const Term& tm, int k, int col) {
  using E = typename Pol::E;
  E v{};
  if (k < tm.k && col < a.nrhs) {
    const int64_t p = tm.in_row + k;
    if (tm.in_kind == 0)
      v = __ldg(static_cast<const E*>(a.S) + p * a.ldS + col);
    else
      v = __ldg(static_cast<const E*>(a.X) + (a.xperm ? a.xperm[p] : p) + (int64_t)col * a.ldx);
  }
  return v;
}

// fill the fragments of k-step k0 (c128: DMMA m8n8k4 layout; c64: TF32 m16n8k8 layout)
template <int NT>
__device__ __forceinline__ void frags(PolC128<NT>& /*tag*/, typename PolC128<NT>::Frags& f, const StageArgs& a,
                                      const Term& tm, int r0, int m, int k0, int j0, int g, int t, bool cj) {
  using P = PolC128<NT>;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    f.a[mi] = ldA<P>(a, tm, r0 + 8 * mi + g, k0 + t, m, cj);
    f.as[mi] = f.a[mi].x + f.a[mi].y;
  }
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) P::set_b(f, ni, ldB<P>(a, tm, k0 + t, j0 + 8 * ni + g));
}
template <int NT>
__device__ __forceinline__ void frags(PolC64<NT>& /*tag*/, typename PolC64<NT>::Frags& f, const StageArgs& a,
                                      const Term& tm, int r0, int m, int k0, int j0, int g, int t, bool cj) {
  using P = PolC64<NT>;
  float2 v[4];
  v[0] = ldA<P>(a, tm, r0 + g, k0 + t, m, cj);
  v[1] = ldA<P>(a, tm, r0 + g + 8, k0 + t, m, cj);
  v[2] = ldA<P>(a, tm, r0 + g, k0 + t + 4, m, cj);
  v[3] = ldA<P>(a, tm, r0 + g + 8, k0 + t + 4, m, cj);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    P::split(v[e].x, f.ah[0][e], f.al[0][e]);
    P::split(v[e].y, f.ah[1][e], f.al[1][e]);
    P::split(v[e].x + v[e].y, f.ah[2][e], f.al[2][e]);
  }
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) {
    f.b[ni][0] = ldB<P>(a, tm, k0 + t, j0 + 8 * ni + g);
    f.b[ni][1] = ldB<P>(a, tm, k0 + t + 4, j0 + 8 * ni + g);
  }
}

template <class Pol>
__global__ void __launch_bounds__(256, 2) k_stage_mma(StageArgs a) {
  using E = typename Pol::E;
  constexpr int KS = Pol::KS;
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= a.nunits) return;
  const int2 un = a.units[u];
  const Task tk = a.tasks[un.x];
  const int r0 = un.y * 16;
  const int j0 = blockIdx.y * 8 * Pol::NT;
  const int g = lane >> 2, t = lane & 3;
  Pol tag;
  typename Pol::Acc4 acc;  // 4M: exact on selection / identity factors
  acc.zero();
  for (int q = 0; q < tk.nterm; ++q) {
    const Term tm = a.terms[tk.term0 + q];
    const bool cj = (tm.conj != 0) != (a.conj_flip != 0);
    typename Pol::Frags f[2];
    frags(tag, f[0], a, tm, r0, tk.m, 0, j0, g, t, cj);
    int k0 = 0;
    for (; k0 + KS < tm.k; k0 += 2 * KS) {
      frags(tag, f[1], a, tm, r0, tk.m, k0 + KS, j0, g, t, cj);
      acc.mac(f[0]);
      if (k0 + 2 * KS < tm.k) frags(tag, f[0], a, tm, r0, tk.m, k0 + 2 * KS, j0, g, t, cj);
      acc.mac(f[1]);
    }
    if (k0 < tm.k) acc.mac(f[0]);
  }
  if (a.out_kind == 0) {
    E* S = static_cast<E*>(a.S);
    acc.each(g, t, [&](int r, int c, E v) {
      if (r0 + r < tk.m && j0 + c < a.nrhs) S[(tk.out_row + r0 + r) * a.ldS + j0 + c] = v;
    });
  } else {
    E* Y = static_cast<E*>(a.Y);
    acc.each(g, t, [&](int r, int c, E v) {
      if (r0 + r < tk.m && j0 + c < a.nrhs) {
        const int64_t p = tk.out_row + r0 + r;
        Y[(a.yperm ? a.yperm[p] : p) + (int64_t)(j0 + c) * a.ldy] = v;
      }
    });
  }
}

template <typename V>
static void launch_generic(const Round& r, StageArgs a, cudaStream_t st) {
  a.tasks = r.tasks;
  a.terms = r.terms;
  a.units = r.units;
  a.nunits = r.nunits;
  a.out_kind = r.out_kind;
  dim3 grid((r.nunits + 7) / 8, (a.nrhs + 15) / 16);  // warp tile: 16 rows x 16 columns
  if (sizeof(V) == 16)
    k_stage_mma<PolC128<2>><<<grid, 256, 0, st>>>(a);
  else
    k_stage_mma<PolC64<2>><<<grid, 256, 0, st>>>(a);
}

const char* round_kernel_name(int dtype, const Round& r, int* id) {
  (void)r;
  if (id) *id = 3;
  return dtype == BF_C128 ? "k_stage_mma<c128>" : "k_stage_mma<c64>";
}

void launch_round(int dtype, const Round& r, StageArgs a, cudaStream_t st) {
  if (r.ntasks == 0) return;
  if (dtype == BF_C128)
    launch_generic<double2>(r, a, st);
  else
    launch_generic<float2>(r, a, st);
}

}  // namespace bfa
