// Device kernels of the randomized matrix-free butterfly construction (bf_random_matvec,
// SURVEY 8(f) NEXT-2; Sec. 3.3, "BF_random_matvec": a butterfly built from
// O(n^{1/2}) multi-RHS applies of an O(n log n) matvec; Alg. 5 line S_construction).
// The host driver is rmatvec_host.inc (level-by-level peeling).
//
//   k_sketch_fill   Gaussian sketch blocks with a per-row group support (counter-based RNG:
//                   every entry is a pure function of (seed, level, row, column), so chunking
//                   and launch order never change the sketch)
//   k_gather_t      the sketch rows of each block's candidate skeletons, transposed into one
//                   packed k x p matrix per block (conjugated for the column side)
//   k_batched_id    interpolative decomposition of every packed matrix: Householder QR with
//                   column pivoting, truncated at |R_jj| < eps |R_11| ("U = P[I;
//                   (R11^-1 R12)^T]"), T = R11^-1 R12 written over R12; one CTA per matrix
//   k_batched_lsq   the centre blocks: B = Y Z^+ (least squares through a Householder QR of Z^H)
#include <cstdio>

#include "common.cuh"

namespace bfa {

// ---- complex helpers on double2 / float2 -------------------------------------------------
template <typename V> struct Real;
template <> struct Real<double2> { using T = double; };
template <> struct Real<float2> { using T = float; };

template <typename V> __device__ __forceinline__ V cmk(typename Real<V>::T x, typename Real<V>::T y) {
  V v;
  v.x = x;
  v.y = y;
  return v;
}
template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return cmk<V>(a.x + b.x, a.y + b.y); }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return cmk<V>(a.x - b.x, a.y - b.y); }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  return cmk<V>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
template <typename V> __device__ __forceinline__ V cmulc(V a, V b) {
  return cmk<V>(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
template <typename V> __device__ __forceinline__ V cconj(V a) { return cmk<V>(a.x, -a.y); }
template <typename V> __device__ __forceinline__ typename Real<V>::T cabs2(V a) { return a.x * a.x + a.y * a.y; }
template <typename V> __device__ __forceinline__ V cdiv(V a, V b) {
  const typename Real<V>::T d = cabs2(b);
  return cmk<V>((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
template <typename V> __device__ __forceinline__ V cscale(V a, typename Real<V>::T s) { return cmk<V>(a.x * s, a.y * s); }

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- counter-based Gaussian --------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// one standard complex Gaussian (re, im each N(0, 1)) for the counter (seed, level, row, col)
__device__ __forceinline__ void gauss2(uint64_t seed, int level, int64_t row, int64_t col, double& re, double& im) {
  const uint64_t h0 = splitmix64(seed ^ ((uint64_t)level << 58) ^ splitmix64((uint64_t)row * 0x100000001B3ull + (uint64_t)col));
  const uint64_t h1 = splitmix64(h0);
  const double u1 = ((h0 >> 11) + 1) * (1.0 / 9007199254740992.0);  // (0, 1]
  const double u2 = (h1 >> 11) * (1.0 / 9007199254740992.0);        // [0, 1)
  const double rad = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  re = rad * c;
  im = rad * s;
}

// Om[u + c ld] for user rows u < rows, columns c < ncols.  group[u] is the tree node (at the
// sketch's level) that row u belongs to.  overlay = 0: column c belongs to group g0 + c / k and is
// nonzero only on that group's rows; overlay = 1: column c of every row u is column
// group[u] * k + c of the full (block-diagonal) sketch -- the groups' disjoint supports folded
// into k columns.
template <typename V>
__global__ void k_sketch_fill(V* __restrict__ Om, int64_t ld, int64_t rows, int64_t ncols, const int64_t* __restrict__ group,
                              int64_t g0, int k, uint64_t seed, int level, int overlay) {
  const int64_t total = rows * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / rows, u = e - c * rows;
    const int64_t g = group[u];
    int64_t gc;
    bool on;
    if (overlay) {
      on = g >= 0;
      gc = g * k + c;
    } else {
      on = g == g0 + c / k;
      gc = g0 * k + c;
    }
    double re = 0.0, im = 0.0;
    if (on) gauss2(seed, level, u, gc, re, im);
    Om[u + c * ld] = cmk<V>((typename Real<V>::T)re, (typename Real<V>::T)im);
  }
}

// Packed matrix i (k rows x p_i columns, column-major, ld k) at out + out_off[i]:
//   out[a + b k] = f(Y[rows[moff[i] + b] + (mcol[i] + a) ldy]),  f = conj if cj else identity.
// One CTA per matrix.
template <typename V>
__global__ void k_gather_t(V* __restrict__ out, const V* __restrict__ Y, int64_t ldy, const int64_t* __restrict__ rows,
                           const int64_t* __restrict__ moff, const int64_t* __restrict__ mcol,
                           const int64_t* __restrict__ out_off, int k, int cj) {
  const int64_t i = blockIdx.x;
  const int64_t r0 = moff[i], p = moff[i + 1] - r0, c0 = mcol[i];
  V* o = out + out_off[i];
  for (int64_t e = threadIdx.x; e < p * k; e += blockDim.x) {
    const int64_t b = e / k, a = e - b * k;
    V v = Y[rows[r0 + b] + (c0 + a) * ldy];
    if (cj) v.y = -v.y;
    o[a + b * k] = v;
  }
}

// ---- Householder QR (with optional column pivoting) of one k x p matrix in global memory --
// Reflector for column j: H = I - v v^H * (2 / v^H v), v = x - beta e_0, beta = -e^{i arg x_0} ||x||,
// so that H x = beta e_0.  With pivot != 0 the column of largest remaining norm is moved to
// position j first (ties: the lowest index) and the factorisation stops at rank r when
// |R_rr| <= eps |R_00| (relative truncation) or at rmax.  Columns [ncols_fac, p)
// are only updated (right-hand sides of a least-squares solve).  Returns the rank (number of
// reflectors applied) in *rank_out; perm (p entries) gets the column order.
constexpr int QR_THREADS = 256;
constexpr int QR_WARPS = QR_THREADS / 32;
constexpr int QR_MAXK = 1024;  // rows of a packed matrix (sketch width) held in shared memory

template <typename V>
__device__ int householder_qr(V* A, int k, int p, int ncols_fac, int pivot, double eps, int rmax, int* perm,
                              typename Real<V>::T* cn, V* v) {
  using T = typename Real<V>::T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ T s_vv, s_r00;
  __shared__ int s_piv, s_stop;
  for (int c = threadIdx.x; c < p; c += blockDim.x) perm[c] = c;
  const int jmax = min(min(k, ncols_fac), rmax);
  int j = 0;
  for (; j < jmax; ++j) {
    // pivot: remaining column norms over rows j..k-1 (recomputed: robust, same order of work)
    if (pivot) {
      for (int c = j + warp; c < ncols_fac; c += QR_WARPS) {
        T s = 0;
        for (int r = j + lane; r < k; r += 32) s += cabs2(A[r + (int64_t)c * k]);
        s = warp_sum(s);
        if (lane == 0) cn[c] = s;
      }
      __syncthreads();
      if (warp == 0) {
        T best = -1;
        int bi = ncols_fac;
        for (int c = j + lane; c < ncols_fac; c += 32)
          if (cn[c] > best) {  // strict: the lowest index wins ties within a lane
            best = cn[c];
            bi = c;
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const T ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
          }
        }
        if (lane == 0) {
          s_piv = bi;
          const T nrm = sqrt(max(best, (T)0));
          if (j == 0) s_r00 = nrm;
          s_stop = !(nrm > 0) || (j > 0 && nrm <= (T)eps * s_r00);
        }
      }
      __syncthreads();
      if (s_stop) break;
      const int pv = s_piv;
      if (pv != j) {
        for (int r = threadIdx.x; r < k; r += blockDim.x) {
          const V t = A[r + (int64_t)j * k];
          A[r + (int64_t)j * k] = A[r + (int64_t)pv * k];
          A[r + (int64_t)pv * k] = t;
        }
        if (threadIdx.x == 0) {
          const int t = perm[j];
          perm[j] = perm[pv];
          perm[pv] = t;
        }
      }
      __syncthreads();
    }
    // reflector of column j, rows j..k-1
    if (warp == 0) {
      T s = 0;
      for (int r = j + lane; r < k; r += 32) {
        const V x = A[r + (int64_t)j * k];
        v[r] = x;
        s += cabs2(x);
      }
      s = warp_sum(s);
      if (lane == 0) {
        const V x0 = v[j];
        const T nx = sqrt(s), a0 = sqrt(cabs2(x0));
        // beta = -e^{i arg x0} ||x||
        const V ph = a0 > 0 ? cmk<V>(x0.x / a0, x0.y / a0) : cmk<V>(1, 0);
        const V beta = cmk<V>(-ph.x * nx, -ph.y * nx);
        v[j] = csub(x0, beta);
        s_vv = s - cabs2(x0) + cabs2(v[j]);
        A[j + (int64_t)j * k] = beta;
      }
    }
    __syncthreads();
    const T vv = s_vv;
    // apply H to the trailing columns (and the right-hand-side columns)
    for (int c = j + 1 + warp; c < p; c += QR_WARPS) {
      V* col = A + (int64_t)c * k;
      V d = cmk<V>(0, 0);
      for (int r = j + lane; r < k; r += 32) d = cadd(d, cmulc(v[r], col[r]));
      d.x = warp_sum(d.x);
      d.y = warp_sum(d.y);
      if (vv > 0) {
        const V f = cscale(d, (T)2 / vv);
        for (int r = j + lane; r < k; r += 32) col[r] = csub(col[r], cmul(v[r], f));
      }
    }
    for (int r = j + 1 + threadIdx.x; r < k; r += blockDim.x) A[r + (int64_t)j * k] = cmk<V>(0, 0);
    __syncthreads();
  }
  return j;
}

// Interpolative decomposition of every packed matrix (k x p_i, ld k) in place.  On return:
//   rank[i] = r; perm[poff[i] + 0..p_i) = column order (the first r are the skeleton columns);
//   rows 0..r-1 of columns r..p_i-1 hold T = R11^{-1} R12, so that
//   M(:, perm[r + j]) ~= sum_q M(:, perm[q]) T(q, j)   (the column ID of P:285-288).
template <typename V>
__global__ void __launch_bounds__(QR_THREADS) k_batched_id(V* __restrict__ M, const int64_t* __restrict__ moff,
                                                             const int64_t* __restrict__ pcnt, int k, double eps,
                                                             int rmax, int32_t* __restrict__ rank,
                                                             int32_t* __restrict__ perm, const int64_t* __restrict__ poff) {
  using T = typename Real<V>::T;
  extern __shared__ __align__(16) unsigned char sm[];
  V* v = reinterpret_cast<V*>(sm);                       // k
  T* cn = reinterpret_cast<T*>(sm + sizeof(V) * k);      // p
  const int64_t i = blockIdx.x;
  const int p = (int)pcnt[i];
  V* A = M + moff[i];
  int* pm = perm + poff[i];
  const int r = householder_qr<V>(A, k, p, p, 1, eps, rmax, pm, cn, v);
  __syncthreads();
  // T = R11^{-1} R12 by back substitution, one column of R12 per thread
  for (int c = r + threadIdx.x; c < p; c += blockDim.x) {
    V* col = A + (int64_t)c * k;
    for (int q = r - 1; q >= 0; --q) {
      V s = col[q];
      for (int w = q + 1; w < r; ++w) s = csub(s, cmul(A[q + (int64_t)w * k], col[w]));
      const V d = A[q + (int64_t)q * k];
      col[q] = cabs2(d) > 0 ? cdiv(s, d) : cmk<V>(0, 0);
    }
  }
  if (threadIdx.x == 0) rank[i] = r;
}

// Centre blocks (least squares B Z = Y, Z: c x k full row rank, Y: r x k):
//   work (k x (c + r), ld k) = [Z^H | Y^H]; Householder QR of the first c columns applied to all;
//   B^H = R^{-1} (Q^H Y^H)[0..c);  B (r x c, column-major) written to out + boff[i].
// Z rows come from the slab space (row zrow[i] + q, k contiguous columns: Z(q, a) = S[(zrow + q) k + a]),
// Y rows from the sketch (user row yrows[yoff[i] + q], columns ycol[i] + a).
template <typename V>
__global__ void __launch_bounds__(QR_THREADS) k_batched_lsq(V* __restrict__ work, const int64_t* __restrict__ woff,
                                                              const V* __restrict__ S, const int64_t* __restrict__ zrow,
                                                              const int32_t* __restrict__ cdim, const V* __restrict__ Ysk,
                                                              int64_t ldy, const int64_t* __restrict__ yrows,
                                                              const int64_t* __restrict__ yoff, const int64_t* __restrict__ ycol,
                                                              int k, V* __restrict__ out, const int64_t* __restrict__ boff) {
  using T = typename Real<V>::T;
  extern __shared__ __align__(16) unsigned char sm[];
  V* v = reinterpret_cast<V*>(sm);
  T* cn = reinterpret_cast<T*>(sm + sizeof(V) * k);
  int* pm = reinterpret_cast<int*>(sm + sizeof(V) * k + sizeof(T) * k);
  const int64_t i = blockIdx.x;
  const int c = cdim[i];
  const int r = (int)(yoff[i + 1] - yoff[i]);
  if (r == 0) return;  // B is r x c: nothing to write
  if (c == 0) return;
  V* A = work + woff[i];
  for (int64_t e = threadIdx.x; e < (int64_t)k * (c + r); e += blockDim.x) {
    const int col = (int)(e / k), a = (int)(e - (int64_t)col * k);
    V x;
    if (col < c)
      x = cconj(S[(zrow[i] + col) * (int64_t)k + a]);
    else
      x = cconj(Ysk[yrows[yoff[i] + (col - c)] + (ycol[i] + a) * ldy]);
    A[a + (int64_t)col * k] = x;
  }
  __syncthreads();
  householder_qr<V>(A, k, c + r, c, 0, 0.0, c, pm, cn, v);
  __syncthreads();
  // back substitution: B^H(:, q) = R^{-1} (Q^H Y^H)(0..c, q), one right-hand side per thread
  for (int q = threadIdx.x; q < r; q += blockDim.x) {
    V* col = A + (int64_t)(c + q) * k;
    for (int a = c - 1; a >= 0; --a) {
      V s = col[a];
      for (int w = a + 1; w < c; ++w) s = csub(s, cmul(A[a + (int64_t)w * k], col[w]));
      const V d = A[a + (int64_t)a * k];
      col[a] = cabs2(d) > 0 ? cdiv(s, d) : cmk<V>(0, 0);
    }
    // B(q, a) = conj(B^H(a, q))
    for (int a = 0; a < c; ++a) out[boff[i] + q + (int64_t)a * r] = cconj(col[a]);
  }
}

// ---- launchers ----------------------------------------------------------------------------
void launch_sketch_fill(int dtype, void* Om, int64_t ld, int64_t rows, int64_t ncols, const int64_t* group, int64_t g0,
                        int k, uint64_t seed, int level, int overlay, cudaStream_t st) {
  const int64_t total = rows * ncols;
  if (total == 0) return;
  const int nsm = device_sm_count();
  const int64_t want = (total + 255) / 256;
  const unsigned grid = (unsigned)(want < 16LL * nsm ? want : 16LL * nsm);
  if (dtype == BF_C128)
    k_sketch_fill<double2><<<grid, 256, 0, st>>>(static_cast<double2*>(Om), ld, rows, ncols, group, g0, k, seed, level, overlay);
  else
    k_sketch_fill<float2><<<grid, 256, 0, st>>>(static_cast<float2*>(Om), ld, rows, ncols, group, g0, k, seed, level, overlay);
}

void launch_gather_t(int dtype, int64_t nmat, void* out, const void* Y, int64_t ldy, const int64_t* rows, const int64_t* moff,
                     const int64_t* mcol, const int64_t* out_off, int k, int cj, cudaStream_t st) {
  if (nmat == 0) return;
  if (dtype == BF_C128)
    k_gather_t<double2><<<(unsigned)nmat, 256, 0, st>>>(static_cast<double2*>(out), static_cast<const double2*>(Y), ldy,
                                                         rows, moff, mcol, out_off, k, cj);
  else
    k_gather_t<float2><<<(unsigned)nmat, 256, 0, st>>>(static_cast<float2*>(out), static_cast<const float2*>(Y), ldy,
                                                        rows, moff, mcol, out_off, k, cj);
}

void launch_batched_id(int dtype, int64_t nmat, void* M, const int64_t* moff, const int64_t* pcnt, int k, int pmax,
                       double eps, int rmax, int32_t* rank, int32_t* perm, const int64_t* poff, cudaStream_t st) {
  if (nmat == 0) return;
  if (k > QR_MAXK) throw Err{BF_ERR_ARG, "sketch width above the batched ID's limit (1024)"};
  const size_t cs = dtype == BF_C128 ? 16 : 8;
  const size_t smem = cs * k + (cs / 2) * (size_t)(pmax > 0 ? pmax : 1);
  static std::atomic<size_t> a128[BF_MAX_DEVICES], a64[BF_MAX_DEVICES];
  if (dtype == BF_C128) {
    ensure_smem_attr(a128, (const void*)k_batched_id<double2>, smem);
    k_batched_id<double2><<<(unsigned)nmat, QR_THREADS, smem, st>>>(static_cast<double2*>(M), moff, pcnt, k, eps, rmax,
                                                                    rank, perm, poff);
  } else {
    ensure_smem_attr(a64, (const void*)k_batched_id<float2>, smem);
    k_batched_id<float2><<<(unsigned)nmat, QR_THREADS, smem, st>>>(static_cast<float2*>(M), moff, pcnt, k, eps, rmax,
                                                                   rank, perm, poff);
  }
}

void launch_batched_lsq(int dtype, int64_t nmat, void* work, const int64_t* woff, const void* S, const int64_t* zrow,
                        const int32_t* cdim, const void* Ysk, int64_t ldy, const int64_t* yrows, const int64_t* yoff,
                        const int64_t* ycol, int k, int maxcr, void* out, const int64_t* boff, cudaStream_t st) {
  if (nmat == 0) return;
  const size_t cs = dtype == BF_C128 ? 16 : 8;
  const size_t smem = cs * k + (cs / 2) * (size_t)k + sizeof(int) * (size_t)(maxcr > 0 ? maxcr : 1);
  static std::atomic<size_t> a128[BF_MAX_DEVICES], a64[BF_MAX_DEVICES];
  if (dtype == BF_C128) {
    ensure_smem_attr(a128, (const void*)k_batched_lsq<double2>, smem);
    k_batched_lsq<double2><<<(unsigned)nmat, QR_THREADS, smem, st>>>(
        static_cast<double2*>(work), woff, static_cast<const double2*>(S), zrow, cdim, static_cast<const double2*>(Ysk), ldy,
        yrows, yoff, ycol, k, static_cast<double2*>(out), boff);
  } else {
    ensure_smem_attr(a64, (const void*)k_batched_lsq<float2>, smem);
    k_batched_lsq<float2><<<(unsigned)nmat, QR_THREADS, smem, st>>>(
        static_cast<float2*>(work), woff, static_cast<const float2*>(S), zrow, cdim, static_cast<const float2*>(Ysk), ldy,
        yrows, yoff, ycol, k, static_cast<float2*>(out), boff);
  }
}

}  // namespace bfa

namespace bfa {

// In-place inverse of every square matrix (n_i x n_i, column-major, ld n_i) packed in M
// (Gauss-Jordan elimination with partial pivoting, one CTA per matrix): the dense leaf inverses
// of Alg. 4 line 3 ("Directly compute D_tau^{-1}") and the L = 0 base case of BF_SMW.
// info[i] = 0, or j + 1 when pivot column j was exactly singular.
template <typename V>
__global__ void __launch_bounds__(QR_THREADS) k_batched_inv(V* __restrict__ M, const int64_t* __restrict__ moff,
                                                              const int64_t* __restrict__ dim, int32_t* __restrict__ info) {
  using T = typename Real<V>::T;
  extern __shared__ __align__(16) unsigned char sm[];
  int* piv = reinterpret_cast<int*>(sm);  // n: row order
  __shared__ int s_p, s_bad;
  const int64_t i = blockIdx.x;
  const int n = (int)dim[i];
  V* A = M + moff[i];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_bad = 0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) piv[r] = r;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (warp == 0) {  // partial pivot: largest |A(r, j)|, r >= j (lowest index on ties)
      T best = -1;
      int bi = j;
      for (int r = j + lane; r < n; r += 32) {
        const T a = cabs2(A[r + (int64_t)j * n]);
        if (a > best) {
          best = a;
          bi = r;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const T ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (lane == 0) {
        s_p = bi;
        if (!(best > 0) && s_bad == 0) s_bad = j + 1;
      }
    }
    __syncthreads();
    const int p = s_p;
    if (p != j) {  // swap rows j and p (all columns)
      for (int c = threadIdx.x; c < n; c += blockDim.x) {
        const V t = A[j + (int64_t)c * n];
        A[j + (int64_t)c * n] = A[p + (int64_t)c * n];
        A[p + (int64_t)c * n] = t;
      }
      if (threadIdx.x == 0) {
        const int t = piv[j];
        piv[j] = piv[p];
        piv[p] = t;
      }
    }
    __syncthreads();
    const V d = A[j + (int64_t)j * n];
    const V dinv = cabs2(d) > 0 ? cdiv(cmk<V>(1, 0), d) : cmk<V>(0, 0);
    __syncthreads();
    // scale row j: A(j, c) *= 1/d for c != j; A(j, j) = 1/d
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      if (c == j)
        A[j + (int64_t)c * n] = dinv;
      else
        A[j + (int64_t)c * n] = cmul(A[j + (int64_t)c * n], dinv);
    }
    __syncthreads();
    // eliminate column j from every other row: A(r, c) -= A(r, j) A(j, c); A(r, j) = -A(r, j) / d
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int c = e / n, r = e - c * n;
      if (r == j || c == j) continue;
      A[r + (int64_t)c * n] = csub(A[r + (int64_t)c * n], cmul(A[r + (int64_t)j * n], A[j + (int64_t)c * n]));
    }
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x)
      if (r != j) A[r + (int64_t)j * n] = cmul(cmk<V>(-A[r + (int64_t)j * n].x, -A[r + (int64_t)j * n].y), dinv);
    __syncthreads();
  }
  // A now holds inv(P A_orig) = inv(A_orig) P^T, P the accumulated row interchanges (row j of P A
  // is row piv[j] of A): permute the columns back, inv(A_orig)(:, piv[c]) = A(:, c)
  V* tmp = reinterpret_cast<V*>(sm + ((sizeof(int) * (size_t)n + 15) & ~size_t(15)));
  for (int r = 0; r < n; ++r) {
    for (int c = threadIdx.x; c < n; c += blockDim.x) tmp[piv[c]] = A[r + (int64_t)c * n];
    __syncthreads();
    for (int c = threadIdx.x; c < n; c += blockDim.x) A[r + (int64_t)c * n] = tmp[c];
    __syncthreads();
  }
  if (threadIdx.x == 0) info[i] = s_bad;
}

void launch_batched_inv(int dtype, int64_t nmat, void* M, const int64_t* moff, const int64_t* dim, int nmax,
                        int32_t* info, cudaStream_t st) {
  if (nmat == 0) return;
  const size_t cs = dtype == BF_C128 ? 16 : 8;
  const size_t smem = ((sizeof(int) * (size_t)nmax + 15) & ~size_t(15)) + cs * (size_t)nmax;
  static std::atomic<size_t> a128[BF_MAX_DEVICES], a64[BF_MAX_DEVICES];
  if (dtype == BF_C128) {
    ensure_smem_attr(a128, (const void*)k_batched_inv<double2>, smem);
    k_batched_inv<double2><<<(unsigned)nmat, QR_THREADS, smem, st>>>(static_cast<double2*>(M), moff, dim, info);
  } else {
    ensure_smem_attr(a64, (const void*)k_batched_inv<float2>, smem);
    k_batched_inv<float2><<<(unsigned)nmat, QR_THREADS, smem, st>>>(static_cast<float2*>(M), moff, dim, info);
  }
}

}  // namespace bfa

namespace bfa {

// Y(leaf rows) = D_t X(leaf rows) (op N) or D_t^H X (op C) for the leaves t of one node: the dense
// leaf-inverse factor of the HOD-BF inverse.  lp points at the node's first leaf offset (absolute
// tree positions; r0 = the node's first row), D_t column-major at D + doff[t].  Grid: (leaf,
// 8-column group).
template <typename V>
__global__ void k_blockdiag(const int64_t* __restrict__ lp, int64_t r0, const V* __restrict__ D,
                            const int64_t* __restrict__ doff, int op, int64_t nrhs, const V* __restrict__ X, int64_t ldx,
                            V* __restrict__ Y, int64_t ldy) {
  const int64_t t = blockIdx.x, j0 = (int64_t)blockIdx.y * 8;
  const int64_t a = lp[t] - r0, s = lp[t + 1] - lp[t];
  const V* Dt = D + doff[t];
  const int nj = (int)min((int64_t)8, nrhs - j0);
  for (int64_t e = threadIdx.x; e < s * nj; e += blockDim.x) {
    const int64_t jj = e / s, r = e - jj * s, j = j0 + jj;
    V acc = cmk<V>(0, 0);
    if (op == BF_OP_N) {
      for (int64_t k = 0; k < s; ++k) acc = cadd(acc, cmul(Dt[r + k * s], X[a + k + j * ldx]));
    } else {
      for (int64_t k = 0; k < s; ++k) acc = cadd(acc, cmulc(Dt[k + r * s], X[a + k + j * ldx]));
    }
    Y[a + r + j * ldy] = acc;
  }
}

void launch_blockdiag(int dtype, int64_t nleaf, const int64_t* lp, int64_t r0, const void* D, const int64_t* doff, int op,
                      int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy, int lmax, cudaStream_t st) {
  if (nleaf == 0 || nrhs == 0) return;
  (void)lmax;
  dim3 grid((unsigned)nleaf, (unsigned)((nrhs + 7) / 8));
  if (dtype == BF_C128)
    k_blockdiag<double2><<<grid, 256, 0, st>>>(lp, r0, static_cast<const double2*>(D), doff, op, nrhs,
                                               static_cast<const double2*>(X), ldx, static_cast<double2*>(Y), ldy);
  else
    k_blockdiag<float2><<<grid, 256, 0, st>>>(lp, r0, static_cast<const float2*>(D), doff, op, nrhs,
                                              static_cast<const float2*>(X), ldx, static_cast<float2*>(Y), ldy);
}

// gather (scatter = 0): Y[i] = X[perm[i]]; scatter (1): Y[perm[i]] = X[i]; perm NULL = identity
template <typename V>
__global__ void k_permute_rows(int64_t rows, int64_t nrhs, const int64_t* __restrict__ perm, int scatter,
                               const V* __restrict__ X, int64_t ldx, V* __restrict__ Y, int64_t ldy) {
  const int64_t total = rows * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    const int64_t p = perm ? perm[i] : i;
    if (scatter)
      Y[p + j * ldy] = X[i + j * ldx];
    else
      Y[i + j * ldy] = X[p + j * ldx];
  }
}

void launch_permute_rows(int dtype, int64_t rows, int64_t nrhs, const int64_t* perm, int scatter, const void* X,
                         int64_t ldx, void* Y, int64_t ldy, cudaStream_t st) {
  const int64_t total = rows * nrhs;
  if (total == 0) return;
  const int nsm = device_sm_count();
  const int64_t want = (total + 255) / 256;
  const unsigned grid = (unsigned)(want < 8LL * nsm ? want : 8LL * nsm);
  if (dtype == BF_C128)
    k_permute_rows<double2><<<grid, 256, 0, st>>>(rows, nrhs, perm, scatter, static_cast<const double2*>(X), ldx,
                                                  static_cast<double2*>(Y), ldy);
  else
    k_permute_rows<float2><<<grid, 256, 0, st>>>(rows, nrhs, perm, scatter, static_cast<const float2*>(X), ldx,
                                                 static_cast<float2*>(Y), ldy);
}

}  // namespace bfa

namespace bfa {

// rows[i] of an index list: gather Y[i] = X[idx[i]] (add = 0) or scatter-add Y[idx[i]] += alpha X[i]
// (add = 1; the indices of one call are distinct, so no two threads update the same row): the
// extend-add moves of the multifrontal solve sweep
template <typename V>
__global__ void k_index_rows(int64_t rows, int64_t nrhs, const int64_t* __restrict__ idx, int add, double are,
                             double aim, const V* __restrict__ X, int64_t ldx, V* __restrict__ Y, int64_t ldy) {
  const int64_t total = rows * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    if (add) {
      const V a = X[i + j * ldx];
      V y = Y[idx[i] + j * ldy];
      y.x += (are * a.x - aim * a.y);
      y.y += (are * a.y + aim * a.x);
      Y[idx[i] + j * ldy] = y;
    } else {
      Y[i + j * ldy] = X[idx[i] + j * ldx];
    }
  }
}

void launch_index_rows(int dtype, int64_t rows, int64_t nrhs, const int64_t* idx, int add, double are, double aim,
                       const void* X, int64_t ldx, void* Y, int64_t ldy, cudaStream_t st) {
  const int64_t total = rows * nrhs;
  if (total == 0) return;
  const int nsm = device_sm_count();
  const int64_t want = (total + 255) / 256;
  const unsigned grid = (unsigned)(want < 8LL * nsm ? want : 8LL * nsm);
  if (dtype == BF_C128)
    k_index_rows<double2><<<grid, 256, 0, st>>>(rows, nrhs, idx, add, are, aim, static_cast<const double2*>(X), ldx,
                                                static_cast<double2*>(Y), ldy);
  else
    k_index_rows<float2><<<grid, 256, 0, st>>>(rows, nrhs, idx, add, are, aim, static_cast<const float2*>(X), ldx,
                                               static_cast<float2*>(Y), ldy);
}

}  // namespace bfa

namespace bfa {

// ---- compact sub-matrix extraction (Alg. 3 extract_BF: every touched block is
// multiplied once, at the width of the requested columns under its column node) -------------
// One product: out[out_off + i * out_ld + j] (+)= sum_k A(i, k) in[in_off + k * in_ld + j],
// A(i, k) = pool[a_off + i * a_rs + k * a_cs]; i < m, j < w, k < kk.  Row-major compact slabs.

// one warp per product; lanes over the m x w outputs
template <typename V>
__global__ void k_xprod(int64_t np, const XProd* __restrict__ P, const V* __restrict__ pool, const V* __restrict__ S,
                        V* __restrict__ O) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = wid; p < np; p += nw) {
    const XProd q = P[p];
    const int tot = q.m * q.w;
    for (int e = lane; e < tot; e += 32) {
      const int i = e / q.w, j = e - i * q.w;
      const V* a = pool + q.a_off + (int64_t)i * q.a_rs;
      const V* x = S + q.in_off + j;
      V s = cmk<V>(0, 0);
      for (int k = 0; k < q.kk; ++k) s = cadd(s, cmul(a[(int64_t)k * q.a_cs], x[(int64_t)k * q.in_ld]));
      V* o = O + q.out_off + (int64_t)i * q.out_ld + j;
      if (q.acc) s = cadd(s, *o);
      *o = s;
    }
  }
}

// the level-0 slabs: S[dst + r * w + jj] = pool[src + r] for r < c (the requested Vt columns;
// entry e = {dst slab offset + column, w, rank c, pool offset of the Vt column})
template <typename V>
__global__ void k_xgather_vt(int64_t n, const int64_t* __restrict__ e, const V* __restrict__ pool, V* __restrict__ S) {
  for (int64_t q = blockIdx.x; q < n; q += gridDim.x) {
    const int64_t dst = e[4 * q], w = e[4 * q + 1], c = e[4 * q + 2], src = e[4 * q + 3];
    for (int64_t r = threadIdx.x; r < c; r += blockDim.x) S[dst + r * w] = pool[src + r];
  }
}

// scatter the compact result rows (tree-sorted columns) to the caller's matrix:
// out[orow[i] + ocol[j] * ldo] = T[i * nJ + j]
template <typename V>
__global__ void k_xscatter(int64_t nI, int64_t nJ, const int64_t* __restrict__ orow, const int64_t* __restrict__ ocol,
                           const V* __restrict__ T, V* __restrict__ out, int64_t ldo) {
  const int64_t tot = nI * nJ;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / nJ, j = e - i * nJ;
    out[orow[i] + ocol[j] * ldo] = T[e];
  }
}

// Level-wise extraction (Alg. 3; every touched block multiplied once, at the columns
// that need it): stage s of every part in one launch.  A part's slab at level l is
// [pos][r < Rl][j < nJ]: request column j belongs to exactly one T_S node per level (nu = tj[j] >> l)
// and, one level down, to exactly one of its children, so every slab column of a block is a small
// matrix-vector product with that child's block.  One thread per (pos, 8-row chunk, column j):
// the input column is read once per 8 output rows, the factor rows of a k are 8 consecutive
// entries.  Rows r >= the block's rank are neither written nor read.
constexpr int XL_RC = 8;
template <typename V>
__device__ __forceinline__ void xl_dot(const V* __restrict__ a, int64_t lda, int nr, const V* __restrict__ y, int K,
                                       int64_t ldy, V* __restrict__ o, int64_t ldo) {
  V acc[XL_RC];
#pragma unroll
  for (int q = 0; q < XL_RC; ++q) acc[q] = cmk<V>(0, 0);
  for (int k = 0; k < K; ++k) {
    const V yk = y[k * ldy];
    const V* ak = a + k * lda;
#pragma unroll
    for (int q = 0; q < XL_RC; ++q)
      if (q < nr) acc[q] = cadd(acc[q], cmul(ak[q], yk));
  }
#pragma unroll
  for (int q = 0; q < XL_RC; ++q)
    if (q < nr) o[q * ldo] = acc[q];
}

template <typename V>
__device__ __forceinline__ void xl_stage(int s, int np, const XLPart* __restrict__ P, const int64_t* __restrict__ wpre,
                                         const int64_t* __restrict__ B, const V* __restrict__ pool, V* __restrict__ S) {
  const int64_t tot = wpre[np];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = np - 1;  // the part: last k with wpre[k] <= e
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (wpre[mid] <= e) lo = mid;
      else hi = mid - 1;
    }
    const XLPart& p = P[lo];
    int64_t x = e - wpre[lo];
    const int nJ = p.nJ, L = p.L, lc = p.lc;
    const int64_t nb = int64_t(1) << L;
    const int j = (int)(x % nJ);
    x /= nJ;
    const V* in = S + p.slab[(s - 1) & 1];
    V* o = S + p.slab[s & 1];
    if (s == 0) {  // z^0_nu(r, j) = Vt_nu(r, column j)
      const int64_t t = B[p.o_tj + j];
      const int r = (int)x;
      if (r >= p.rc[t]) continue;
      o[(int64_t)r * nJ + j] = pool[B[p.o_vtoff + j] + r];
    } else if (s <= L + 1) {
      const int64_t t = B[p.o_tj + j];  // the column's leaf (T_S level-0 node)
      const int l = s <= lc ? s : s == lc + 1 ? lc : s - 1;  // output level
      const int64_t* rs = s <= lc ? B + p.o_rz : B + p.o_ry - lc;  // rows per slab, indexed by level
      const int R = (int)rs[l];
      const int nch = (R + XL_RC - 1) / XL_RC;
      const int r0 = (int)(x % nch) * XL_RC;
      const int64_t pos = x / nch;
      const int64_t tau = (l == 0) ? 0 : B[p.o_taus + B[p.o_toff + l] + pos];
      const int64_t nu = t >> l, io = (tau << (L - l)) | nu;
      const V* a;
      const V* y;
      int64_t lda;
      int K, rows;
      if (s <= lc) {  // W stage l: z^l_{tau,nu} = W_{tau,nu} [z^{l-1}_{tau>>1,2nu}; z^{l-1}_{tau>>1,2nu+1}]
        const int c = p.rc[l * nb + io];
        if (r0 >= c) continue;
        rows = c;
        const int sb = (int)((t >> (l - 1)) & 1);
        const int64_t tp = l == 1 ? 0 : tau >> 1, pp = l == 1 ? 0 : B[p.o_ppos + B[p.o_toff + l] + pos];
        const int64_t ic0 = (tp << (L - l + 1)) | (2 * nu);
        const int c0 = p.rc[(l - 1) * nb + ic0];
        K = sb ? p.rc[(l - 1) * nb + ic0 + 1] : c0;
        lda = c;
        a = pool + p.fw + p.woff[(l - 1) * nb + io] + r0 + (int64_t)(sb ? c0 : 0) * c;
        y = in + pp * B[p.o_rz + l - 1] * nJ + j;
      } else if (s == lc + 1) {  // centre: y^lc_{tau,nu} = B_{tau,nu} z^lc_{tau,nu}
        const int ri = p.rr[io];
        if (r0 >= ri) continue;
        rows = ri;
        K = p.rc[lc * nb + io];
        lda = ri;
        a = pool + p.fb + p.boff[io] + r0;
        y = in + pos * B[p.o_rz + lc] * nJ + j;
      } else {  // R stage l - 1 -> l (gather form): y^l_{tau,nu} = R_{tau>>1, 2nu+s}[rows of child tau & 1] y^{l-1}
        const int32_t* rr1 = p.rr + (int64_t)(l - lc) * nb;
        const int ro = rr1[io];
        if (r0 >= ro) continue;
        rows = ro;
        const int64_t a2 = tau >> 1, ch = t >> (l - 1), i = (a2 << (L - l + 1)) | ch;
        const int rt = rr1[((2 * a2) << (L - l)) | nu], rb = rr1[((2 * a2 + 1) << (L - l)) | nu];
        K = p.rr[(int64_t)(l - 1 - lc) * nb + i];
        lda = rt + rb;
        a = pool + p.fr + p.roff[(int64_t)(l - 1 - lc) * nb + i] + ((tau & 1) ? rt : 0) + r0;
        const int64_t pp = B[p.o_ppos + B[p.o_toff + l] + pos];
        y = in + pp * B[p.o_ry + l - 1 - lc] * nJ + j;
      }
      xl_dot(a, lda, min(XL_RC, rows - r0), y, K, (int64_t)nJ, o + (pos * R + r0) * nJ + j, (int64_t)nJ);
    } else {  // U rows: K(row i, column j) = U_tau(row, :) y^L_tau(:, j)
      const int i = (int)x;
      const int64_t tau = B[p.o_ti + i];
      const int kn = p.rr[(int64_t)(L - lc) * nb + tau];
      const V* a = pool + B[p.o_uoff + i];
      const int64_t us = B[p.o_ustr + i];
      const V* y = in + B[p.o_ypos + i] * B[p.o_ry + L - lc] * nJ + j;
      V acc = cmk<V>(0, 0);
      for (int k = 0; k < kn; ++k) acc = cadd(acc, cmul(a[k * us], y[(int64_t)k * nJ]));
      static_cast<V*>(p.out)[B[p.o_orow + i] + B[p.o_ocol + j] * p.ldo] = acc;
    }
  }
}

template <typename V>
__global__ void __launch_bounds__(256) k_xlevel(int s, int np, const XLPart* __restrict__ P,
                                                const int64_t* __restrict__ wpre, const int64_t* __restrict__ B,
                                                const V* __restrict__ pool, V* __restrict__ S) {
  xl_stage(s, np, P, wpre, B, pool, S);
}

void launch_xlevel(int dtype, int s, int nparts, const XLPart* P, const int64_t* wpre, int64_t total,
                   const int64_t* blob, const void* pool, void* S, cudaStream_t st) {
  if (total <= 0 || nparts <= 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (dtype == BF_C128)
    k_xlevel<double2><<<grid, 256, 0, st>>>(s, nparts, P, wpre, blob, static_cast<const double2*>(pool),
                                            static_cast<double2*>(S));
  else
    k_xlevel<float2><<<grid, 256, 0, st>>>(s, nparts, P, wpre, blob, static_cast<const float2*>(pool),
                                           static_cast<float2*>(S));
}

void launch_xprod(int dtype, int64_t np, const void* P, const void* pool, const void* S, void* O, cudaStream_t st) {
  if (np == 0) return;
  const int64_t blocks = std::min<int64_t>((np + 7) / 8, 65535 * 4);
  if (dtype == BF_C128)
    k_xprod<double2><<<(unsigned)blocks, 256, 0, st>>>(np, static_cast<const XProd*>(P), static_cast<const double2*>(pool),
                                                        static_cast<const double2*>(S), static_cast<double2*>(O));
  else
    k_xprod<float2><<<(unsigned)blocks, 256, 0, st>>>(np, static_cast<const XProd*>(P), static_cast<const float2*>(pool),
                                                       static_cast<const float2*>(S), static_cast<float2*>(O));
}

void launch_xgather_vt(int dtype, int64_t n, const int64_t* e, const void* pool, void* S, cudaStream_t st) {
  if (n == 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(n, 65535);
  if (dtype == BF_C128)
    k_xgather_vt<double2><<<grid, 64, 0, st>>>(n, e, static_cast<const double2*>(pool), static_cast<double2*>(S));
  else
    k_xgather_vt<float2><<<grid, 64, 0, st>>>(n, e, static_cast<const float2*>(pool), static_cast<float2*>(S));
}

void launch_xscatter(int dtype, int64_t nI, int64_t nJ, const int64_t* orow, const int64_t* ocol, const void* T, void* out,
                     int64_t ldo, cudaStream_t st) {
  const int64_t tot = nI * nJ;
  if (tot == 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>((tot + 255) / 256, 8192);
  if (dtype == BF_C128)
    k_xscatter<double2><<<grid, 256, 0, st>>>(nI, nJ, orow, ocol, static_cast<const double2*>(T),
                                              static_cast<double2*>(out), ldo);
  else
    k_xscatter<float2><<<grid, 256, 0, st>>>(nI, nJ, orow, ocol, static_cast<const float2*>(T),
                                             static_cast<float2*>(out), ldo);
}

}  // namespace bfa
