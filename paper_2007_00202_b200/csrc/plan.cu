// Host side of libbfapply: descriptor validation, device upload, and the per-op plans
// (Task / Term tables) that turn Eq. (3.3) into a short sequence of batched launches.
//
// Butterfly, op N (Y = K X), one launch ("round") per stage -- SURVEY 8(a) a1-a5:
//   r0            a1  z^0_{0,nu}   = Vt_nu X(col_perm[S_nu])
//   r1 .. r_lc    a2  z^l_{tau,nu} = W_{tau,nu} [z^{l-1}_{tau>>1,2nu}; z^{l-1}_{tau>>1,2nu+1}]
//   r_lc+1        a3  y^lc_{tau,nu} = B_{tau,nu} z^lc_{tau,nu}
//   ...           a4  y^{l+1}_{t',nu'} = sum_s R_{t'>>1,2nu'+s}[rows of child t'&1] y^l_{t'>>1,2nu'+s}
//                     (the gather form of [y_{2tau}; y_{2tau+1}] += R_{tau,nu} y_{tau,nu})
//   r_L+2         a5  Y(row_perm[O_tau]) = U_tau y^L_{tau,0}
// op C (Y = K^H X) runs the same rounds backwards with conjugate-transposed factor views;
// op T reuses the op-C tables with the conjugation flipped.
// Intermediates live in one "slab space" in the workspace: every (space, level, block)
// owns rank x nrhs entries (nrhs fastest), so no stage ever overwrites another stage's
// data and no atomics are needed (each output slab is written by exactly one task).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <type_traits>
#include <vector>
#include <unordered_map>

#include "common.cuh"
#include "fast.cuh"

namespace bfa {

thread_local std::string g_last_error;
// Set while bf_dist_create builds a host-only plan (device < 0): layouts and exchange maps
// are computed, nothing is uploaded, and every apply on the handle fails with BF_ERR_DEVICE.
thread_local bool g_host_only = false;


#define BF_CK(call)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw Err{e_ == cudaErrorMemoryAllocation ? BF_ERR_OOM : BF_ERR_CUDA,               \
                std::string(#call) + ": " + cudaGetErrorString(e_)};                      \
  } while (0)

static void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw Err{code, msg};
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (dev < 0) return;  // host-only plan: no device is touched
    cudaGetDevice(&prev);
    if (prev != dev) BF_CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

static size_t csize(int dtype) { return dtype == BF_C128 ? 16 : 8; }

// --------------------------------------------------------------------------------------
// geometry of one butterfly (ranks, leaves, factor block offsets)
// --------------------------------------------------------------------------------------
struct Geom {
  int L = 0, lc = 0;
  int64_t m = 0, n = 0, nb = 1;
  std::vector<int64_t> rlp, clp;
  std::vector<int32_t> rr, rc;
  std::vector<int64_t> u_off, vt_off, b_off;
  std::vector<std::vector<int64_t>> r_off, w_off;  // indexed by level l
  int64_t len_U = 0, len_R = 0, len_B = 0, len_W = 0, len_Vt = 0;

  int64_t idx(int l, int64_t tau, int64_t nu) const { return (tau << (L - l)) | nu; }
  int r(int l, int64_t i) const { return rr[(size_t)(l - lc) * nb + i]; }
  int c(int l, int64_t i) const { return rc[(size_t)l * nb + i]; }
  int64_t mt(int64_t tau) const { return rlp[tau + 1] - rlp[tau]; }
  int64_t nv(int64_t nu) const { return clp[nu + 1] - clp[nu]; }
  int R_rows(int l, int64_t tau, int64_t nu) const {
    return r(l + 1, idx(l + 1, 2 * tau, nu >> 1)) + r(l + 1, idx(l + 1, 2 * tau + 1, nu >> 1));
  }
  int W_cols(int l, int64_t tau, int64_t nu) const {
    return c(l - 1, idx(l - 1, tau >> 1, 2 * nu)) + c(l - 1, idx(l - 1, tau >> 1, 2 * nu + 1));
  }
};

static void check_leafptr(const int64_t* p, int64_t nb, int64_t total, const char* what) {
  require(p != nullptr, BF_ERR_ARG, std::string(what) + " is NULL");
  require(p[0] == 0, BF_ERR_SHAPE, std::string(what) + "[0] != 0");
  for (int64_t i = 0; i < nb; ++i)
    require(p[i + 1] >= p[i], BF_ERR_SHAPE, std::string(what) + " not monotone");
  require(p[nb] == total, BF_ERR_SHAPE, std::string(what) + " does not end at the dimension");
}

static void check_perm(const int64_t* p, int64_t n, const char* what) {
  if (!p) return;
  std::vector<char> seen((size_t)n, 0);
  for (int64_t i = 0; i < n; ++i) {
    require(p[i] >= 0 && p[i] < n && !seen[(size_t)p[i]], BF_ERR_PERM,
            std::string(what) + " is not a permutation");
    seen[(size_t)p[i]] = 1;
  }
}

static Geom make_geom(const bf_desc& d) {
  Geom g;
  require(d.dtype == BF_C64 || d.dtype == BF_C128, BF_ERR_ARG, "dtype must be BF_C64 or BF_C128");
  require(d.L >= 0 && d.L <= 30, BF_ERR_SHAPE, "L out of range [0, 30]");
  require(d.level_maps == nullptr, BF_ERR_ARG, "internal: level_maps not canonicalised");
  g.L = d.L;
  g.lc = d.lc < 0 ? d.L / 2 : d.lc;
  require(g.lc >= 0 && g.lc <= g.L, BF_ERR_SHAPE, "lc out of range [0, L]");
  require(d.m >= 0 && d.n >= 0, BF_ERR_SHAPE, "negative dimension");
  g.m = d.m;
  g.n = d.n;
  g.nb = int64_t(1) << g.L;
  check_leafptr(d.row_leaf_ptr, g.nb, d.m, "row_leaf_ptr");
  check_leafptr(d.col_leaf_ptr, g.nb, d.n, "col_leaf_ptr");
  g.rlp.assign(d.row_leaf_ptr, d.row_leaf_ptr + g.nb + 1);
  g.clp.assign(d.col_leaf_ptr, d.col_leaf_ptr + g.nb + 1);
  require(d.rank_row && d.rank_col, BF_ERR_ARG, "rank arrays are NULL");
  g.rr.assign(d.rank_row, d.rank_row + (size_t)(g.L - g.lc + 1) * g.nb);
  g.rc.assign(d.rank_col, d.rank_col + (size_t)(g.lc + 1) * g.nb);
  for (int32_t v : g.rr) require(v >= 0, BF_ERR_RANK, "negative row rank");
  for (int32_t v : g.rc) require(v >= 0, BF_ERR_RANK, "negative column rank");
  // rank_row at l = L must be zero for nu != 0 slots? Level L has 2^L tau and one nu:
  // the canonical index tau*2^0 + 0 covers all 2^L entries, so nothing is unused.
  int64_t o = 0;
  g.u_off.resize(g.nb);
  for (int64_t t = 0; t < g.nb; ++t) {
    g.u_off[t] = o;
    o += g.mt(t) * g.r(g.L, t);
  }
  g.len_U = o;
  o = 0;
  g.r_off.assign(g.L + 1, {});
  for (int l = g.lc; l < g.L; ++l) {
    g.r_off[l].resize(g.nb);
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (g.L - l)); ++nu) {
        g.r_off[l][g.idx(l, tau, nu)] = o;
        o += int64_t(g.R_rows(l, tau, nu)) * g.r(l, g.idx(l, tau, nu));
      }
  }
  g.len_R = o;
  o = 0;
  g.b_off.resize(g.nb);
  for (int64_t i = 0; i < g.nb; ++i) {
    g.b_off[i] = o;
    o += int64_t(g.r(g.lc, i)) * g.c(g.lc, i);
  }
  g.len_B = o;
  o = 0;
  g.w_off.assign(g.lc + 1, {});
  for (int l = 1; l <= g.lc; ++l) {
    g.w_off[l].resize(g.nb);
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (g.L - l)); ++nu) {
        g.w_off[l][g.idx(l, tau, nu)] = o;
        o += int64_t(g.c(l, g.idx(l, tau, nu))) * g.W_cols(l, tau, nu);
      }
  }
  g.len_W = o;
  o = 0;
  g.vt_off.resize(g.nb);
  for (int64_t nu = 0; nu < g.nb; ++nu) {
    g.vt_off[nu] = o;
    o += int64_t(g.c(0, nu)) * g.nv(nu);
  }
  g.len_Vt = o;
  require(d.len_U == g.len_U && d.len_R == g.len_R && d.len_B == g.len_B && d.len_W == g.len_W &&
              d.len_Vt == g.len_Vt,
          BF_ERR_RANK, "factor array lengths do not match the rank chains");
  require((g.len_U == 0 || d.U) && (g.len_R == 0 || d.R) && (g.len_B == 0 || d.B) &&
              (g.len_W == 0 || d.W) && (g.len_Vt == 0 || d.Vt),
          BF_ERR_ARG, "factor array is NULL");
  return g;
}

// --------------------------------------------------------------------------------------
// bf_desc.level_maps: per-level block orderings other than the canonical
// idx = tau * 2^(L-l) + nu.  The descriptor is re-packed on the host into canonical order
// (ranks and factor blocks of every mapped level), so everything after create sees only
// canonical descriptors.  Canon owns the re-packed arrays.
// --------------------------------------------------------------------------------------
struct Canon {
  bf_desc d{};
  std::vector<int32_t> rr, rc;
  std::vector<char> f[5];  // U, R, B, W, Vt
};

static const bf_desc& canonical(const bf_desc& in, Canon& cn) {
  if (!in.level_maps) return in;
  require(in.dtype == BF_C64 || in.dtype == BF_C128, BF_ERR_ARG, "dtype must be BF_C64 or BF_C128");
  require(in.L >= 0 && in.L <= 30, BF_ERR_SHAPE, "L out of range [0, 30]");
  const int L = in.L, lc = in.lc < 0 ? in.L / 2 : in.lc;
  require(lc >= 0 && lc <= L, BF_ERR_SHAPE, "lc out of range [0, L]");
  require(in.rank_row && in.rank_col, BF_ERR_ARG, "rank arrays are NULL");
  const int64_t nb = int64_t(1) << L;
  const int32_t* const* M = in.level_maps;
  for (int l = 0; l <= L; ++l) {
    if (!M[l]) continue;
    std::vector<char> seen((size_t)nb, 0);
    for (int64_t s = 0; s < nb; ++s) {
      const int64_t i = M[l][s];
      require(i >= 0 && i < nb && !seen[(size_t)i], BF_ERR_PERM,
              "level_maps[" + std::to_string(l) + "] is not a bijection of [0, 2^L)");
      seen[(size_t)i] = 1;
    }
  }
  auto slot_to = [&](int l, int64_t s) -> int64_t { return M[l] ? M[l][s] : s; };
  cn.rr.assign(in.rank_row, in.rank_row + (size_t)(L - lc + 1) * nb);
  cn.rc.assign(in.rank_col, in.rank_col + (size_t)(lc + 1) * nb);
  for (int l = lc; l <= L; ++l)
    for (int64_t s = 0; s < nb; ++s) cn.rr[(size_t)(l - lc) * nb + slot_to(l, s)] = in.rank_row[(l - lc) * nb + s];
  for (int l = 0; l <= lc; ++l)
    for (int64_t s = 0; s < nb; ++s) cn.rc[(size_t)l * nb + slot_to(l, s)] = in.rank_col[l * nb + s];
  cn.d = in;
  cn.d.level_maps = nullptr;
  cn.d.rank_row = cn.rr.data();
  cn.d.rank_col = cn.rc.data();
  // canonical geometry (validates leaves, ranks and array lengths; the lengths do not depend
  // on the order of the blocks)
  const Geom g = make_geom(cn.d);
  const size_t cs = csize(in.dtype);
  const void* src[5] = {in.U, in.R, in.B, in.W, in.Vt};
  const int64_t len[5] = {g.len_U, g.len_R, g.len_B, g.len_W, g.len_Vt};
  for (int a = 0; a < 5; ++a) cn.f[a].resize((size_t)len[a] * cs);
  // one level of one array: storage slots in order, each copied to its canonical offset
  auto level = [&](int a, int l, const std::vector<int64_t>& coff, auto size_of, int64_t& in_off) {
    for (int64_t s = 0; s < nb; ++s) {
      const int64_t i = slot_to(l, s);
      const int64_t sz = size_of(i);
      if (sz) std::memcpy(cn.f[a].data() + coff[i] * cs, static_cast<const char*>(src[a]) + in_off * cs, sz * cs);
      in_off += sz;
    }
  };
  auto tau_of = [&](int l, int64_t i) { return i >> (L - l); };
  auto nu_of = [&](int l, int64_t i) { return i & ((int64_t(1) << (L - l)) - 1); };
  int64_t o = 0;
  level(0, L, g.u_off, [&](int64_t i) { return g.mt(i) * g.r(L, i); }, o);
  o = 0;
  for (int l = lc; l < L; ++l)
    level(1, l, g.r_off[l], [&](int64_t i) { return int64_t(g.R_rows(l, tau_of(l, i), nu_of(l, i))) * g.r(l, i); }, o);
  o = 0;
  level(2, lc, g.b_off, [&](int64_t i) { return int64_t(g.r(lc, i)) * g.c(lc, i); }, o);
  o = 0;
  for (int l = 1; l <= lc; ++l)
    level(3, l, g.w_off[l], [&](int64_t i) { return int64_t(g.c(l, i)) * g.W_cols(l, tau_of(l, i), nu_of(l, i)); }, o);
  o = 0;
  level(4, 0, g.vt_off, [&](int64_t i) { return int64_t(g.c(0, i)) * g.nv(i); }, o);
  cn.d.U = cn.f[0].data();
  cn.d.R = cn.f[1].data();
  cn.d.B = cn.f[2].data();
  cn.d.W = cn.f[3].data();
  cn.d.Vt = cn.f[4].data();
  return cn.d;
}

// factor-pool base offsets (elements) of one butterfly's five arrays
struct FBase {
  int64_t u = 0, r = 0, b = 0, w = 0, vt = 0;
};

// slab-space row offsets of one butterfly's coefficient slabs
struct Slabs {
  std::vector<int64_t> row;  // (l - lc) * nb + i, l = lc..L
  std::vector<int64_t> col;  // l * nb + i,        l = 0..lc
  int xspace = 0;            // 0 none, 1 row space at lc (op N exchange), 2 col space at lc (op C)
  std::vector<int64_t> xout, xin;
  int64_t row_out(const Geom& g, int l, int64_t i) const {
    return (xspace == 1 && l == g.lc) ? xout[i] : row[(size_t)(l - g.lc) * g.nb + i];
  }
  int64_t row_in(const Geom& g, int l, int64_t i) const {
    return (xspace == 1 && l == g.lc) ? xin[i] : row[(size_t)(l - g.lc) * g.nb + i];
  }
  int64_t col_out(const Geom& g, int l, int64_t i) const {
    return (xspace == 2 && l == g.lc) ? xout[i] : col[(size_t)l * g.nb + i];
  }
  int64_t col_in(const Geom& g, int l, int64_t i) const {
    return (xspace == 2 && l == g.lc) ? xin[i] : col[(size_t)l * g.nb + i];
  }
};

// ownership of blocks for the distributed split; p = log2(ranks)
struct Own {
  int p = 0;
  int64_t g = 0;
  // column side: nu at T_S level L - l lies under nu_g (level p)
  bool col(const Geom& G, int l, int64_t nu) const { return p == 0 || (nu >> (G.L - l - p)) == g; }
  // row side: tau at T_O level l lies under tau_g
  bool row(int l, int64_t tau) const { return p == 0 || (tau >> (l - p)) == g; }
};

struct PlanBuilder {
  std::vector<std::vector<Task>> tasks;
  std::vector<std::vector<Term>> terms;
  std::vector<int> okind;
  bool use_cols = false;                   // bf_extract: per-task column ranges
  std::vector<std::vector<int2>> cols;
  void add(int round, int out_kind, int64_t out_row, int64_t m, const Term* t, int nt,
           int2 colr = make_int2(0, 0)) {
    if (m <= 0) return;
    if ((int)tasks.size() <= round) {
      tasks.resize(round + 1);
      terms.resize(round + 1);
      okind.resize(round + 1, -1);
      cols.resize(round + 1);
    }
    if (use_cols) cols[round].push_back(colr);
    require(okind[round] == -1 || okind[round] == out_kind, BF_ERR_ARG, "internal: mixed out kinds");
    okind[round] = out_kind;
    Task tk{};
    tk.out_row = out_row;
    tk.m = (int32_t)m;
    tk.term0 = (int32_t)terms[round].size();
    tk.nterm = 0;
    for (int q = 0; q < nt; ++q) {
      if (t[q].k <= 0) continue;
      terms[round].push_back(t[q]);
      tk.nterm++;
    }
    tasks[round].push_back(tk);
  }
};

static Term mk(int64_t a_off, int a_rs, int a_cs, int64_t k, int64_t in_row, int in_kind, int conj) {
  Term t{};
  t.a_off = a_off;
  t.in_row = in_row;
  t.a_rs = a_rs;
  t.a_cs = a_cs;
  t.k = (int32_t)k;
  t.conj = (int16_t)conj;
  t.in_kind = (int16_t)in_kind;
  return t;
}

// Blocks an extraction touches (Alg. 3): (l, tau, nu) with tau at T_O level l an
// ancestor of a requested row's leaf and nu at T_S level L - l an ancestor of a requested
// column's leaf.  Every other block of K E_J restricted to the rows I is zero or unused.
struct Touch {
  std::vector<std::vector<uint8_t>> row;  // [l][tau], l = 0..L
  std::vector<std::vector<uint8_t>> col;  // [l][nu],  nu at T_S level L - l
  std::vector<std::vector<int64_t>> rows, cols;  // the same as ascending lists
  std::vector<std::vector<int2>> crange;         // [l][nu]: requested columns (tree-sorted) under nu
  bool r(int l, int64_t tau) const { return row[l][tau] != 0; }
  bool c(int l, int64_t nu) const { return col[l][nu] != 0; }
};

// grow-only device scratch of the extraction calls of one handle
// Device copies of a butterfly geometry's rank and block-offset tables (the level-wise
// extraction, k_xlevel), uploaded on a handle's first extraction.
struct XGeomDev {
  void* buf = nullptr;
  const int32_t *rr = nullptr, *rc = nullptr;
  const int64_t *roff = nullptr, *woff = nullptr, *boff = nullptr;
  std::vector<int64_t> Rz, Ry;  // rows per slab: max column rank at l = 0..lc, max row rank at l = lc..L
};

struct XScratch {
  std::mutex mu;
  void* buf = nullptr;
  size_t bytes = 0;
  std::map<const void*, XGeomDev> geo;  // keyed by the Geom (owned by the handle, never moved)
  void* get(size_t need) {
    if (bytes < need) {
      if (buf) cudaFree(buf);
      buf = nullptr;
      bytes = 0;
      BF_CK(cudaMalloc(&buf, need));
      bytes = need;
    }
    return buf;
  }
  void* hbuf = nullptr;  // pinned staging of the per-request tables (a pageable copy is staged)
  size_t hbytes = 0;
  void* host(size_t need) {
    if (hbytes < need) {
      if (hbuf) cudaFreeHost(hbuf);
      hbuf = nullptr;
      hbytes = 0;
      BF_CK(cudaHostAlloc(&hbuf, need, cudaHostAllocDefault));
      hbytes = need;
    }
    return hbuf;
  }
  ~XScratch() {
    if (buf) cudaFree(buf);
    if (hbuf) cudaFreeHost(hbuf);
    for (auto& g : geo)
      if (g.second.buf) cudaFree(g.second.buf);
  }
};

struct EmitOpts {
  bool leaf_in = true, leaf_out = true;  // emit the V / U leaf stages (HOD-BF fuses them)
  int64_t x_base = 0, y_base = 0;        // tree position of local X / Y row 0
  Own own;
};

// op N rounds: 0 leaf V, 1..lc W, lc+1 B, lc+2.. R, L+2 leaf U
static void emit_N(PlanBuilder& pb, const Geom& G, const FBase& F, const Slabs& S, const EmitOpts& o) {
  const int L = G.L, lc = G.lc;
  if (o.leaf_in)
    for (int64_t nu = 0; nu < G.nb; ++nu) {
      if (!o.own.col(G, 0, nu)) continue;
      const int c = G.c(0, nu);
      Term t = mk(F.vt + G.vt_off[nu], 1, c, G.nv(nu), G.clp[nu] - o.x_base, 1, 0);
      pb.add(0, 0, S.col_out(G, 0, nu), c, &t, 1);
    }
  for (int l = 1; l <= lc; ++l)
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        if (!o.own.col(G, l, nu)) continue;
        const int64_t i = G.idx(l, tau, nu);
        const int64_t i1 = G.idx(l - 1, tau >> 1, 2 * nu), i2 = i1 + 1;
        const int c = G.c(l, i), c1 = G.c(l - 1, i1), c2 = G.c(l - 1, i2);
        Term t[2] = {mk(F.w + G.w_off[l][i], 1, c, c1, S.col_in(G, l - 1, i1), 0, 0),
                     mk(F.w + G.w_off[l][i] + int64_t(c1) * c, 1, c, c2, S.col_in(G, l - 1, i2), 0, 0)};
        if (c1 > 0 && c2 > 0 && t[1].in_row == t[0].in_row + c1) {  // adjacent inputs: one term
          t[0].k = c1 + c2;
          pb.add(l, 0, S.col_out(G, l, i), c, t, 1);
        } else {
          pb.add(l, 0, S.col_out(G, l, i), c, t, 2);
        }
      }
  for (int64_t i = 0; i < G.nb; ++i) {
    const int64_t nu = i & ((int64_t(1) << (L - lc)) - 1);
    if (!o.own.col(G, lc, nu)) continue;
    const int r = G.r(lc, i), c = G.c(lc, i);
    Term t = mk(F.b + G.b_off[i], 1, r, c, S.col_in(G, lc, i), 0, 0);
    pb.add(lc + 1, 0, S.row_out(G, lc, i), r, &t, 1);
  }
  for (int l = lc; l < L; ++l)
    for (int64_t tp = 0; tp < (int64_t(1) << (l + 1)); ++tp)
      for (int64_t np = 0; np < (int64_t(1) << (L - l - 1)); ++np) {
        if (!o.own.row(l + 1, tp)) continue;
        const int64_t a = tp >> 1;
        const int part = (int)(tp & 1);
        const int rt = G.r(l + 1, G.idx(l + 1, 2 * a, np)), rb = G.r(l + 1, G.idx(l + 1, 2 * a + 1, np));
        Term t[2];
        for (int s = 0; s < 2; ++s) {
          const int64_t i = G.idx(l, a, 2 * np + s);
          t[s] = mk(F.r + G.r_off[l][i] + (part ? rt : 0), 1, rt + rb, G.r(l, i), S.row_in(G, l, i), 0, 0);
        }
        const int64_t io = G.idx(l + 1, tp, np);
        pb.add(lc + 2 + (l - lc), 0, S.row_out(G, l + 1, io), G.r(l + 1, io), t, 2);
      }
  if (o.leaf_out)
    for (int64_t tau = 0; tau < G.nb; ++tau) {
      if (!o.own.row(L, tau)) continue;
      Term t = mk(F.u + G.u_off[tau], 1, (int)G.mt(tau), G.r(L, tau), S.row_in(G, L, tau), 0, 0);
      pb.add(L + 2, 1, G.rlp[tau] - o.y_base, G.mt(tau), &t, 1);
    }
}

// bf_extract: the inner op-N rounds of emit_N (W stages, centre, R stages) over the touched
// blocks only (O(touched) work per query); the two leaf rounds are bf_extract's own kernels
// (Vt columns of the requested columns, U rows of the requested rows)
static void emit_N_touched(PlanBuilder& pb, const Geom& G, const FBase& F, const Slabs& S, const Touch& T) {
  const int L = G.L, lc = G.lc;
  // the (tree-sorted) requested columns under nu at T_S level L - l: T.crange[l][nu]
  auto cr = [&](int l, int64_t nu) { return T.crange.empty() ? make_int2(0, 0) : T.crange[l][nu]; };
  for (int l = 1; l <= lc; ++l)
    for (int64_t tau : T.rows[l])
      for (int64_t nu : T.cols[l]) {
        const int64_t i = G.idx(l, tau, nu);
        const int64_t i1 = G.idx(l - 1, tau >> 1, 2 * nu), i2 = i1 + 1;
        const int c = G.c(l, i), c1 = G.c(l - 1, i1), c2 = G.c(l - 1, i2);
        Term t[2] = {mk(F.w + G.w_off[l][i], 1, c, c1, S.col_in(G, l - 1, i1), 0, 0),
                     mk(F.w + G.w_off[l][i] + int64_t(c1) * c, 1, c, c2, S.col_in(G, l - 1, i2), 0, 0)};
        if (!T.c(l - 1, 2 * nu)) t[0].k = 0;
        if (!T.c(l - 1, 2 * nu + 1)) t[1].k = 0;
        pb.add(l, 0, S.col_out(G, l, i), c, t, 2, cr(l, nu));
      }
  for (int64_t tau : T.rows[lc])
    for (int64_t nu : T.cols[lc]) {
      const int64_t i = G.idx(lc, tau, nu);
      const int r = G.r(lc, i), c = G.c(lc, i);
      Term t = mk(F.b + G.b_off[i], 1, r, c, S.col_in(G, lc, i), 0, 0);
      pb.add(lc + 1, 0, S.row_out(G, lc, i), r, &t, 1, cr(lc, nu));
    }
  for (int l = lc; l < L; ++l)
    for (int64_t tp : T.rows[l + 1])
      for (int64_t np : T.cols[l + 1]) {
        const int64_t a = tp >> 1;
        const int part = (int)(tp & 1);
        const int rt = G.r(l + 1, G.idx(l + 1, 2 * a, np)), rb = G.r(l + 1, G.idx(l + 1, 2 * a + 1, np));
        Term t[2];
        for (int s = 0; s < 2; ++s) {
          const int64_t i = G.idx(l, a, 2 * np + s);
          t[s] = mk(F.r + G.r_off[l][i] + (part ? rt : 0), 1, rt + rb, G.r(l, i), S.row_in(G, l, i), 0, 0);
          if (!T.c(l, 2 * np + s)) t[s].k = 0;
        }
        const int64_t io = G.idx(l + 1, tp, np);
        pb.add(lc + 2 + (l - lc), 0, S.row_out(G, l + 1, io), G.r(l + 1, io), t, 2, cr(l + 1, np));
      }
}

// op C rounds: 0 leaf U^H, 1..L-lc R^H, L-lc+1 B^H, .. W^H, L+2 leaf Vt^H
static void emit_C(PlanBuilder& pb, const Geom& G, const FBase& F, const Slabs& S, const EmitOpts& o) {
  const int L = G.L, lc = G.lc;
  if (o.leaf_in)
    for (int64_t tau = 0; tau < G.nb; ++tau) {
      if (!o.own.row(L, tau)) continue;
      const int r = G.r(L, tau);
      Term t = mk(F.u + G.u_off[tau], (int)G.mt(tau), 1, G.mt(tau), G.rlp[tau] - o.x_base, 1, 1);
      pb.add(0, 0, S.row_out(G, L, tau), r, &t, 1);
    }
  for (int l = L - 1; l >= lc; --l)
    for (int64_t a = 0; a < (int64_t(1) << l); ++a)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        if (!o.own.row(l, a)) continue;
        const int64_t i = G.idx(l, a, nu);
        const int64_t it = G.idx(l + 1, 2 * a, nu >> 1), ib = G.idx(l + 1, 2 * a + 1, nu >> 1);
        const int rt = G.r(l + 1, it), rb = G.r(l + 1, ib);
        Term t[2] = {mk(F.r + G.r_off[l][i], rt + rb, 1, rt, S.row_in(G, l + 1, it), 0, 1),
                     mk(F.r + G.r_off[l][i] + rt, rt + rb, 1, rb, S.row_in(G, l + 1, ib), 0, 1)};
        pb.add(1 + (L - 1 - l), 0, S.row_out(G, l, i), G.r(l, i), t, 2);
      }
  for (int64_t i = 0; i < G.nb; ++i) {
    const int64_t tau = i >> (L - lc);
    if (!o.own.row(lc, tau)) continue;
    const int r = G.r(lc, i), c = G.c(lc, i);
    Term t = mk(F.b + G.b_off[i], r, 1, r, S.row_in(G, lc, i), 0, 1);
    pb.add(L - lc + 1, 0, S.col_out(G, lc, i), c, &t, 1);
  }
  for (int l = lc; l >= 1; --l)
    for (int64_t a = 0; a < (int64_t(1) << (l - 1)); ++a)
      for (int64_t mu = 0; mu < (int64_t(1) << (L - l + 1)); ++mu) {
        if (!o.own.col(G, l - 1, mu)) continue;
        const int64_t nu = mu >> 1;
        const int b = (int)(mu & 1);
        const int64_t io = G.idx(l - 1, a, mu);
        const int c1 = G.c(l - 1, G.idx(l - 1, a, 2 * nu));
        Term t[2];
        for (int s = 0; s < 2; ++s) {
          const int64_t i = G.idx(l, 2 * a + s, nu);
          const int cl = G.c(l, i);
          t[s] = mk(F.w + G.w_off[l][i] + int64_t(b ? c1 : 0) * cl, cl, 1, cl, S.col_in(G, l, i), 0, 1);
        }
        pb.add(L - lc + 2 + (lc - l), 0, S.col_out(G, l - 1, io), G.c(l - 1, io), t, 2);
      }
  if (o.leaf_out)
    for (int64_t nu = 0; nu < G.nb; ++nu) {
      if (!o.own.col(G, 0, nu)) continue;
      const int c = G.c(0, nu);
      Term t = mk(F.vt + G.vt_off[nu], c, 1, c, S.col_in(G, 0, nu), 0, 1);
      pb.add(L + 2, 1, G.clp[nu] - o.y_base, G.nv(nu), &t, 1);
    }
}

// --------------------------------------------------------------------------------------
// fused window-pass plan (fast.cuh) for uniform rank-16 butterflies
// --------------------------------------------------------------------------------------
struct FastPlan {
  int lx = 0;  // split: the exchange level (split_exchange_level); lc otherwise
  std::vector<FastPass> passes;
  void* F = nullptr;
  int64_t entries = 0;
  bool contig_in = false;   // every leaf the IN launch reads is a run of consecutive user rows
  bool contig_out = false;  // ... and every leaf the OUT launch writes
  int split = -1;           // multi-GPU split: passes [0, split) before the exchange, the rest after
};

// exact: every rank is 16 (the factors go to the fused kernels as they are); otherwise ranks
// <= 16 are accepted and the factors are zero-padded to rank 16 at create (pad_rank16)
static bool fast_eligible(const Geom& G, int dtype, bool exact = true) {
  (void)dtype;
  if (G.L < 1) return false;
  for (int32_t v : G.rr)
    if (exact ? v != FAST_RANK : v > FAST_RANK) return false;
  for (int32_t v : G.rc)
    if (exact ? v != FAST_RANK : v > FAST_RANK) return false;
  const int64_t lr = G.mt(0), lcn = G.nv(0);
  // power-of-two leaves, multiples of 16 (whole MMA row groups / k-steps), at most 256 rows
  if (lr < 16 || lcn < 16 || lr > 256 || lcn > 256) return false;
  if ((lr & (lr - 1)) || (lcn & (lcn - 1))) return false;
  for (int64_t i = 0; i < G.nb; ++i)
    if (G.mt(i) != lr || G.nv(i) != lcn) return false;
  return true;
}

// Padding ragged ranks <= 16 up to 16 multiplies the streamed entries (a rank-r block of a W / R
// stage by (16 / r)^2): it pays while the padded butterfly streams at most 3x the given entries
// (the fused kernels run at ~3x the generic kernels' rate), or while it is small enough (<= 16 MB
// padded) that the generic plan's launch count, not bytes, sets its time (config 1: 31 vs 45 us).
// Beyond that a ragged butterfly stays on the generic kernels -- also a memory bound: a rank-1
// butterfly would otherwise be stored 256x larger (once per op).
static bool pad_pays(const Geom& G, int64_t entries, size_t cs) {
  if (fast_eligible(G, 0, true)) return true;  // uniform rank 16: nothing to pad
  const int64_t padded = 16 * (G.m + G.n) + G.nb * (int64_t)G.L * 512 + G.nb * 256;
  return padded <= 3 * entries || (double)padded * (double)cs <= 16.0 * (1 << 20);
}

// every leaf of size `leaf` maps to a run of consecutive user rows (so whole rows can be copied)
static bool leaves_contiguous(const int64_t* perm, int64_t n, int64_t leaf) {
  if (!perm) return true;
  for (int64_t s = 0; s < n; s += leaf)
    for (int64_t i = 1; i < leaf; ++i)
      if (perm[s + i] != perm[s] + i) return false;
  return true;
}

template <typename CT>
struct HostFactors {
  const CT *U, *R, *B, *W, *Vt;
};

// A butterfly with ragged ranks <= 16 (and the fused path's uniform power-of-two leaves) as the
// same linear map with every rank 16: each block zero-padded (U_tau and W / R blocks get zero
// columns, Vt_nu / B / W / R zero rows; a W block's columns and an R block's rows keep their two
// child parts at offsets 0 and 16), so the products only add exact zeros (Eq. 3.3 with padded
// factors; ID-compressed butterflies of rank <= 16 on the level-fused kernels).
template <typename CT>
struct Padded16 {
  std::vector<CT> U, R, B, W, Vt;
  std::vector<int32_t> rr, rc;
  bf_desc d{};
  Geom G;
};
template <typename CT>
static void pad_rank16(const bf_desc& d, const Geom& G, Padded16<CT>& P) {
  const int L = G.L, lc = G.lc;
  const int64_t nb = G.nb;
  P.rr.assign((size_t)(L - lc + 1) * nb, FAST_RANK);
  P.rc.assign((size_t)(lc + 1) * nb, FAST_RANK);
  P.U.assign((size_t)G.m * 16, CT{});
  P.R.assign((size_t)(L - lc) * nb * 32 * 16, CT{});
  P.B.assign((size_t)nb * 16 * 16, CT{});
  P.W.assign((size_t)lc * nb * 16 * 32, CT{});
  P.Vt.assign((size_t)G.n * 16, CT{});
  P.d = d;
  P.d.rank_row = P.rr.data();
  P.d.rank_col = P.rc.data();
  P.d.U = P.U.data();
  P.d.R = P.R.data();
  P.d.B = P.B.data();
  P.d.W = P.W.data();
  P.d.Vt = P.Vt.data();
  P.d.len_U = (int64_t)P.U.size();
  P.d.len_R = (int64_t)P.R.size();
  P.d.len_B = (int64_t)P.B.size();
  P.d.len_W = (int64_t)P.W.size();
  P.d.len_Vt = (int64_t)P.Vt.size();
  P.G = make_geom(P.d);
  const Geom& Q = P.G;
  const CT *U = static_cast<const CT*>(d.U), *R = static_cast<const CT*>(d.R), *B = static_cast<const CT*>(d.B),
           *W = static_cast<const CT*>(d.W), *Vt = static_cast<const CT*>(d.Vt);
  for (int64_t t = 0; t < nb; ++t) {  // U_tau: mt x r -> mt x 16
    const int64_t mt = G.mt(t);
    const int r = G.r(L, t);
    for (int k = 0; k < r; ++k)
      for (int64_t i = 0; i < mt; ++i) P.U[Q.u_off[t] + i + k * mt] = U[G.u_off[t] + i + k * mt];
  }
  for (int l = lc; l < L; ++l)  // R^l_{tau,nu}: (rt + rb) x r -> 32 x 16, child rows at 0 / 16
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        const int64_t i = G.idx(l, tau, nu);
        const int rt = G.r(l + 1, G.idx(l + 1, 2 * tau, nu >> 1)), rb = G.r(l + 1, G.idx(l + 1, 2 * tau + 1, nu >> 1));
        const int r = G.r(l, i), ld = rt + rb;
        for (int k = 0; k < r; ++k)
          for (int row = 0; row < ld; ++row)
            P.R[Q.r_off[l][i] + (row < rt ? row : 16 + row - rt) + k * 32] = R[G.r_off[l][i] + row + k * ld];
      }
  for (int64_t i = 0; i < nb; ++i) {  // B: r x c -> 16 x 16
    const int r = G.r(lc, i), c = G.c(lc, i);
    for (int k = 0; k < c; ++k)
      for (int row = 0; row < r; ++row) P.B[Q.b_off[i] + row + k * 16] = B[G.b_off[i] + row + k * r];
  }
  for (int l = 1; l <= lc; ++l)  // W^l_{tau,nu}: c x (cl + cr) -> 16 x 32, child columns at 0 / 16
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        const int64_t i = G.idx(l, tau, nu);
        const int cl = G.c(l - 1, G.idx(l - 1, tau >> 1, 2 * nu)), cr = G.c(l - 1, G.idx(l - 1, tau >> 1, 2 * nu + 1));
        const int c = G.c(l, i);
        for (int col = 0; col < cl + cr; ++col)
          for (int row = 0; row < c; ++row)
            P.W[Q.w_off[l][i] + row + (col < cl ? col : 16 + col - cl) * 16] = W[G.w_off[l][i] + row + col * c];
      }
  for (int64_t nu = 0; nu < nb; ++nu) {  // Vt_nu: c x nv -> 16 x nv
    const int64_t nv = G.nv(nu);
    const int c = G.c(0, nu);
    for (int64_t col = 0; col < nv; ++col)
      for (int row = 0; row < c; ++row) P.Vt[Q.vt_off[nu] + row + col * 16] = Vt[G.vt_off[nu] + row + col * c];
  }
}

template <typename CT>
static inline CT cj(CT v, bool c) {
  if (c) v.y = -v.y;
  return v;
}

// one 1 KB k-step record of an M x K operand: row group mg (16 rows), k-step ki, in the MMA
// fragment order the kernels consume (mma.cuh).
// complex128 (mma m8n8k4, KS = 4): [mi][lane], lane = 4g + t <-> (row 16mg + 8mi + g, col 4ki + t)
// complex64 (mma m16n8k8, KS = 8), `mode`:
//   REC_A_NAT  (column-leaf records, B = X): [re | im][lane][a0..a3], a0..a3 = (g, t), (g+8, t),
//              (g, t+4), (g+8, t+4) of the 16 x 8 block at rows 16mg, cols 8ki
//   REC_A_PAIR (row-leaf records, B = a slab): as REC_A_NAT with K order kappa = t <-> col 2t,
//              kappa = t + 4 <-> col 2t + 1 (the complex64 slab's K order)
//   REC_B_T    (window-pass records, PolC64T: the factor is the B operand of out^T = slab^T F^T):
//              [j][lane][re b0, re b1, im b0, im b1], b0 = (8j + g, 8ki + 2t), b1 = (8j + g, 8ki + 2t + 1)
enum { REC_A_NAT = 0, REC_A_PAIR = 1, REC_B_T = 2 };
template <typename CT, typename Fn>
static void fill_step(CT* dst, int mg, int ki, Fn A, int mode) {
  if (sizeof(CT) == 16) {
    for (int mi = 0; mi < 2; ++mi)
      for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3;
        dst[mi * 32 + lane] = A(16 * mg + 8 * mi + g, 4 * ki + t);
      }
    return;
  }
  auto* f = reinterpret_cast<decltype(dst->x)*>(dst);
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    if (mode == REC_B_T) {
      for (int j = 0; j < 2; ++j) {
        const CT v0 = A(8 * j + g, 8 * ki + 2 * t), v1 = A(8 * j + g, 8 * ki + 2 * t + 1);
        auto* q = f + (j * 32 + lane) * 4;
        q[0] = v0.x;
        q[1] = v1.x;
        q[2] = v0.y;
        q[3] = v1.y;
      }
      continue;
    }
    const int k0 = mode == REC_A_PAIR ? 2 * t : t, k1 = mode == REC_A_PAIR ? 2 * t + 1 : t + 4;
    const CT a[4] = {A(16 * mg + g, 8 * ki + k0), A(16 * mg + g + 8, 8 * ki + k0), A(16 * mg + g, 8 * ki + k1),
                     A(16 * mg + g + 8, 8 * ki + k1)};
    for (int e = 0; e < 4; ++e) {
      f[4 * lane + e] = a[e].x;
      f[128 + 4 * lane + e] = a[e].y;
    }
  }
}

// op 0 = N (forward), 1 = C (adjoint; conjugate-transposed factor views)
// The level at which a fused split exchanges its slabs.  Any level lx in [dp, L - dp] works: a
// block (tau, nu) at level l depends only on X(S_nu) and feeds only Y(O_tau), so every level-l
// block with nu (T_S level L - l >= dp) inside one column subtree can be computed by that
// subtree's rank, and every one with tau (T_O level l >= dp) inside one row subtree by that
// one's -- the paper's centre level lc is just one choice.  The exchange level splits the L
// levels into the two sides' window passes, so it is chosen to minimise the pass count (each
// pass is a slab round trip and a launch ramp): config 5 complex128 at 3-level windows exchanges
// at level 6 (2 + 3 passes, as on one GPU) instead of 7 (3 + 3).  Ties: the level nearest lc.
// Env BF_DIST_LX forces a level (A/B measurements).
static int split_exchange_level(int L, int lc, int dp, int dmax) {
  if (const char* e = getenv("BF_DIST_LX")) {
    const int v = atoi(e);
    if (v >= dp && v <= L - dp) return v;
  }
  int best = lc, bc = 1 << 30;
  for (int lx = dp; lx <= L - dp; ++lx) {
    const int c = (lx + dmax - 1) / dmax + (L - lx + dmax - 1) / dmax;
    if (c < bc || (c == bc && std::abs(lx - lc) < std::abs(best - lc))) {
      bc = c;
      best = lx;
    }
  }
  return best;
}

template <typename CT>
static void build_fast(FastPlan& FP, const Geom& G, const HostFactors<CT>& H, int opk, size_t* acct,
                       int dp = -1, int dg = 0, bool x_contig = false, int lx_req = -1) {
  // dp >= 0: rank dg's share of the split over 2^dp GPUs: the levels below the
  // exchange level lx (W side and, when lx > lc, the first R stages; leaves of T_S) restricted
  // to the column subtree dg at level dp, the levels above it (leaves of T_O) to the row subtree
  // dg; the pass that ends at lx writes the exchange layout and the pass that starts there reads
  // it (split_exchange_level).
  const int L = G.L, lc = G.lc;
  const bool split = dp >= 0;
  const int ks = fast_ks((int)sizeof(CT));
  std::vector<int> lv;  // level boundaries of the window passes
  // window levels per pass: 3 (complex128), 4 (complex64; env BF_C64_DMAX = 3 for A/B)
  int dmax = sizeof(CT) == 16 ? FAST_DMAX : FAST_DMAX_C64;
  if (sizeof(CT) == 8 && getenv("BF_C64_DMAX")) dmax = std::max(1, std::min(FAST_DMAX_C64, atoi(getenv("BF_C64_DMAX"))));
  if (sizeof(CT) == 16 && getenv("BF_C128_DMAX")) dmax = std::max(1, std::min(FAST_DMAX, atoi(getenv("BF_C128_DMAX"))));
  // env BF_PASS_FILL (A/B): 1 = full dmax-level passes with the remainder last, 2 = remainder first
  const int fill = getenv("BF_PASS_FILL") ? atoi(getenv("BF_PASS_FILL")) : 0;
  auto chunk = [&](int lo, int hi) {  // split [lo, hi] into near-equal passes of <= dmax levels
    const int n = hi - lo, k = (n + dmax - 1) / dmax;
    if (fill && n % dmax) {
      int at = lo;
      if (fill == 2) lv.push_back(at += n % dmax);
      while (at + dmax <= hi) lv.push_back(at += dmax);
      if (fill == 1) lv.push_back(hi);
      return;
    }
    for (int p = 0, at = lo; p < k; ++p) {
      at += n / k + (p < n % k ? 1 : 0);
      lv.push_back(at);
    }
  };
  lv.push_back(0);
  const int lx = !split ? lc : (lx_req >= 0 ? lx_req : split_exchange_level(L, lc, dp, dmax));
  FP.lx = lx;
  if (split) {
    chunk(0, lx);
    chunk(lx, L);
  } else {
    chunk(0, L);
    if (opk == 0 && sizeof(CT) == 16) {  // op N: the smaller passes first, so that the last pass
                                         // (which runs the fused row leaf) is a full-width one;
                                         // op C runs the passes top-down
      std::vector<int> r(lv.size());
      for (size_t i = 0; i < lv.size(); ++i) r[i] = L - lv[lv.size() - 1 - i];
      lv = r;
    }
  }
  const int np = (int)lv.size() - 1;
  const int lr = (int)G.mt(0), lcn = (int)G.nv(0);
  const bool adj = opk == 1;
  // The centre factor B^{lc} is folded into its neighbour at create time: R'_{tau,nu} = R_{tau,nu}
  // B_{tau,nu} (32x16, Eq. 3.2 left applied to y = B z) when lc < L, else W'_{tau,nu} = B W
  // (lc = L).  One fewer window op (epilogue + barrier) and 2.7 % fewer entries streamed per
  // apply; the product is formed in complex128 on the host.
  const bool fold_r = lc < L;
  std::vector<CT> fused;
  int64_t fbase0 = 0;
  {
    const std::vector<int64_t>& off = fold_r ? G.r_off[lc] : G.w_off[lc];
    const int64_t nbl = G.nb;
    int64_t lo = INT64_MAX, hi = 0;
    for (int64_t i = 0; i < nbl; ++i) {
      lo = std::min(lo, off[i]);
      hi = std::max(hi, off[i] + 32 * 16);
    }
    fbase0 = lo;
    fused.assign((size_t)(hi - lo), CT{});
    for (int64_t i = 0; i < nbl; ++i) {
      const CT* Bb = H.B + G.b_off[i];
      CT* dst = fused.data() + (off[i] - lo);
      if (fold_r) {  // R (32 x 16, ld 32) * B (16 x 16)
        const CT* Rb = H.R + off[i];
        for (int j = 0; j < 16; ++j)
          for (int r = 0; r < 32; ++r) {
            double re = 0, im = 0;
            for (int k = 0; k < 16; ++k) {
              const CT x = Rb[r + k * 32], y = Bb[k + j * 16];
              re += (double)x.x * y.x - (double)x.y * y.y;
              im += (double)x.x * y.y + (double)x.y * y.x;
            }
            dst[r + j * 32].x = re;
            dst[r + j * 32].y = im;
          }
      } else {  // B (16 x 16) * W (16 x 32, ld 16)
        const CT* Wb = H.W + off[i];
        for (int j = 0; j < 32; ++j)
          for (int r = 0; r < 16; ++r) {
            double re = 0, im = 0;
            for (int k = 0; k < 16; ++k) {
              const CT x = Bb[r + k * 16], y = Wb[k + j * 16];
              re += (double)x.x * y.x - (double)x.y * y.y;
              im += (double)x.x * y.y + (double)x.y * y.x;
            }
            dst[r + j * 16].x = re;
            dst[r + j * 16].y = im;
          }
      }
    }
  }
  auto Rblk = [&](int l, int64_t i) -> const CT* {
    return fold_r && l == lc ? fused.data() + (G.r_off[l][i] - fbase0) : H.R + G.r_off[l][i];
  };
  auto Wblk = [&](int l, int64_t i) -> const CT* {
    return !fold_r && l == lc ? fused.data() + (G.w_off[l][i] - fbase0) : H.W + G.w_off[l][i];
  };
  std::vector<FastPass> passes;
  int64_t total = 0;  // bytes
  // launch k: 0 = leaf-in, 1..np = window passes, np + 1 = leaf-out.  On one GPU the row leaf
  // (a5) is fused into the last window pass as its final op (FK_LEAF_OUT): the pass's output
  // slabs never go to HBM and one launch disappears.
  // (complex128 only: for complex64 the fused op measured no faster than the leaf kernel)
  const bool fuse_out = sizeof(CT) == 16 && !getenv("BF_NO_FUSE_OUT");
  // The column leaf (a1) can likewise run as the first op of the first pass (FK_LEAF_IN, X rows
  // by 2-D TMA tiles in the ring pages; needs every leaf to be a run of consecutive user rows),
  // but measured slower than the separate leaf kernel on config 5 (0.42 vs 0.17 + 0.14 ms: the
  // X stream outruns the 3-page ring of a 2-level pass), so it is opt-in (env BF_FUSE_IN).
  const bool fuse_in = sizeof(CT) == 16 && !split && x_contig && getenv("BF_FUSE_IN");
  for (int k = 0; k < np + 2; ++k) {
    if (k == np + 1 && fuse_out) break;
    if (k == 0 && fuse_in) continue;
    FastPass P{};
    P.L = L;
    std::vector<FastOp> ops;
    auto add = [&](int kind, int s, int leaf) {
      FastOp o{};
      o.kind = kind;
      o.s = s;
      o.leaf = leaf;
      o.nsteps = fast_nsteps(kind, leaf, ks);
      ops.push_back(o);
    };
    int d = 0;
    P.xin = P.xout = 0;
    if (split) {
      P.wt_log = lx - dp;
      P.wn_log = L - lx - dp;
    }
    if (k == 0 || k == np + 1) {
      // leaf launch (d = 0): window w = one leaf at level 0 (T_S leaf nu = b) or L (T_O leaf tau = a)
      const bool in = k == 0;
      const bool at0 = in != adj;  // op N reads X through Vt (level 0); op C through U^H (level L)
      P.leaf = in ? 1 : 2;
      P.l0 = at0 ? 0 : L;
      P.d = 0;
      P.bbits = L - P.l0;
      const int loc = L - (split ? dp : 0);  // log2 of this rank's leaves
      const int64_t lo = split ? int64_t(dg) << loc : 0;
      if (at0) {
        P.a_log = 0;
        P.a_lo = 0;
        P.b_log = loc;
        P.b_lo = lo;
      } else {
        P.a_log = loc;
        P.a_lo = lo;
        P.b_log = 0;
        P.b_lo = 0;
      }
      add(in ? FK_LEAF_IN : FK_LEAF_OUT, 0, at0 ? lcn : lr);
      P.in_s = in ? -1 : 0;
      P.out_s = in ? 0 : -1;
    } else {
      const int p = adj ? np - k : k - 1;
      P.l0 = lv[p];
      P.d = lv[p + 1] - lv[p];
      const int l0 = P.l0, l1 = lv[p + 1];
      d = P.d;
      P.bbits = L - l1;
      // windows: a over T_O level l0, b over T_S level L - l1 (restricted on a split)
      P.a_log = l0;
      P.a_lo = 0;
      P.b_log = L - l1;
      P.b_lo = 0;
      if (split && l1 <= lx) {  // below the exchange: column subtree dg
        P.b_log = L - l1 - dp;
        P.b_lo = int64_t(dg) << P.b_log;
      } else if (split) {  // R side: row subtree dg
        P.a_log = l0 - dp;
        P.a_lo = int64_t(dg) << P.a_log;
      }
      if (fuse_in && k == 1) {
        add(FK_LEAF_IN, adj ? d : 0, adj ? lr : lcn);  // Vt_nu on X (level 0) / U_tau^H on X (level L)
        P.xleaf = 1;                                     // window pass whose input is X, not slabs
      }
      if (!adj) {
        for (int l = l0 + 1; l <= l1 && l <= lc; ++l) add(FK_PAIR_DOWN, l - 1 - l0, 0);  // W_l
        for (int l = std::max(l0, lc); l < l1; ++l) add(FK_PAIR_DOWN, l - l0, 0);      // R_l
        P.in_s = P.xleaf ? -1 : 0;
        P.out_s = d;
        if (split && l1 == lx) P.xout = 1;  // send the level-lx slabs to the owner of tau
        if (split && l0 == lx) P.xin = 2;   // receive from the owner of nu
      } else {
        for (int l = l1 - 1; l >= l0 && l >= lc; --l) add(FK_PAIR_UP, l - l0, 0);        // R^H_l
        for (int l = std::min(l1, lc); l >= l0 + 1; --l) add(FK_PAIR_UP, l - 1 - l0, 0); // W^H_l
        P.in_s = P.xleaf ? -1 : d;
        P.out_s = 0;
        if (split && l0 == lx) P.xout = 2;  // send to the owner of nu
        if (split && l1 == lx) P.xin = 1;   // receive from the owner of tau
      }
      if (P.xout || P.xin) FP.split = (int)passes.size() + (P.xout ? 1 : 0);
      if (fuse_out && k == np) {
        add(FK_LEAF_OUT, adj ? 0 : d, adj ? lcn : lr);  // U_tau (level L) / conj(Vt_nu)^T (level 0)
        P.out_s = -1;
        P.yleaf_lo = split ? int64_t(dg) << (L - dp) : 0;  // Y rows are rank-local on a split
      }
    }
    P.nwin = int64_t(1) << (P.a_log + P.b_log);
    require((int)ops.size() <= FAST_MAXOPS, BF_ERR_ARG, "internal: too many ops in a pass");
    for (const FastOp& o : ops)  // the pass kernel runs pair ops only (the centre is folded)
      require(o.kind != FK_DIAG, BF_ERR_ARG, "internal: centre op on the fast path");
    P.nops = (int)ops.size();
    const int nslot = 1 << d;
    int64_t off = 0;
    for (int q = 0; q < P.nops; ++q) {
      ops[q].off = off;
      off += (int64_t)ops[q].nsteps * nslot * FAST_FRAG;
      P.ops[q] = ops[q];
    }
    P.win_bytes = off;
    P.fbase = total;
    P.numaj = adj ? 1 : 0;
    P.factor_entries = off / (int64_t)sizeof(CT) * P.nwin;
    total += off * P.nwin;
    for (int q = 0; q < P.nops; ++q) {
      if (ops[q].kind == FK_LEAF_IN) P.user_in = P.nwin * ops[q].leaf << P.d;
      if (ops[q].kind == FK_LEAF_OUT) P.user_out = P.nwin * ops[q].leaf << P.d;
    }
    passes.push_back(P);
  }
  std::vector<CT> host((size_t)(total / (int64_t)sizeof(CT)));
  constexpr int REC = FAST_FRAG / (int)sizeof(CT);  // complex entries per k-step record
  for (const FastPass& P : passes) {
    const int d = P.d, nslot = 1 << d;
    for (int64_t w = 0; w < P.nwin; ++w) {
      const int64_t a = P.a_lo + (w >> P.b_log), b = P.b_lo + (w & ((int64_t(1) << P.b_log) - 1));
      for (int q = 0; q < P.nops; ++q) {
        const FastOp& op = P.ops[q];
        CT* base = host.data() + (P.fbase + w * P.win_bytes + op.off) / (int64_t)sizeof(CT);
        for (int o = 0; o < nslot; ++o) {
          // block (tau, nu) of slot o at window level s
          auto blk = [&](int s, int64_t& tau, int64_t& nu) {
            const int ds = d - s;
            tau = (a << s) + (o >> ds);
            nu = (b << ds) + (o & ((1 << ds) - 1));
          };
          // record of k-step `step` of slot o
          auto rec = [&](int step) { return base + ((int64_t)step * nslot + o) * REC; };
          int64_t tau, nu;
          if (op.kind == FK_LEAF_IN) {
            blk(op.s, tau, nu);
            for (int st = 0; st < op.nsteps; ++st) {
              if (!adj) {
                const CT* V = H.Vt + G.vt_off[nu];
                fill_step(rec(st), 0, st, [&](int i, int k) { return V[i + k * 16]; }, REC_A_NAT);
              } else {
                const CT* U = H.U + G.u_off[tau];
                fill_step(rec(st), 0, st, [&](int i, int k) { return cj(U[k + (int64_t)i * lr], true); }, REC_A_NAT);
              }
            }
          } else if (op.kind == FK_LEAF_OUT) {
            blk(op.s, tau, nu);
            const int kpm = 16 / ks;
            for (int st = 0; st < op.nsteps; ++st) {
              const int mg = st / kpm, ki = st % kpm;
              if (!adj) {
                const CT* U = H.U + G.u_off[tau];
                fill_step(rec(st), mg, ki, [&](int i, int k) { return U[i + (int64_t)k * lr]; }, REC_A_PAIR);
              } else {
                const CT* V = H.Vt + G.vt_off[nu];
                fill_step(rec(st), mg, ki, [&](int i, int k) { return cj(V[k + i * 16], true); }, REC_A_PAIR);
              }
            }
          } else if (op.kind == FK_DIAG) {
            blk(op.s, tau, nu);
            const CT* Bb = H.B + G.b_off[G.idx(lc, tau, nu)];
            for (int st = 0; st < op.nsteps; ++st)
              fill_step(rec(st), 0, st, [&](int i, int k) { return adj ? cj(Bb[k + i * 16], true) : Bb[i + k * 16]; }, REC_B_T);
          } else if (op.kind == FK_PAIR_DOWN) {
            blk(op.s + 1, tau, nu);  // output block at level l0 + s + 1
            const int l = P.l0 + op.s + 1;
            if (l <= lc) {  // W_l
              const CT* Wb = Wblk(l, G.idx(l, tau, nu));
              for (int st = 0; st < op.nsteps; ++st)
                fill_step(rec(st), 0, st, [&](int i, int k) { return Wb[i + k * 16]; }, REC_B_T);
            } else {  // R_{l-1}, gather form
              const int lr_ = l - 1;
              const int part = (int)(tau & 1);
              const CT* R0 = Rblk(lr_, G.idx(lr_, tau >> 1, 2 * nu));
              const CT* R1 = Rblk(lr_, G.idx(lr_, tau >> 1, 2 * nu + 1));
              for (int st = 0; st < op.nsteps; ++st)
                fill_step(rec(st), 0, st, [&](int i, int k) {
                  const CT* Rs = k < 16 ? R0 : R1;
                  return Rs[(part * 16 + i) + (k & 15) * 32];
                }, REC_B_T);
            }
          } else {  // FK_PAIR_UP: output block at level l = l0 + s
            blk(op.s, tau, nu);
            const int l = P.l0 + op.s;
            if (l >= lc) {  // R^H_l: inputs (2tau + p, nu >> 1)
              const CT* Rb = Rblk(l, G.idx(l, tau, nu));
              for (int st = 0; st < op.nsteps; ++st)
                fill_step(rec(st), 0, st, [&](int i, int k) {
                  const int pp = k >> 4;
                  return cj(Rb[(pp * 16 + (k & 15)) + i * 32], true);
                }, REC_B_T);
            } else {  // W^H_{l+1}: inputs (2tau + p, nu >> 1) at level l + 1, column part nu & 1
              const int lw = l + 1;
              const CT* W0 = Wblk(lw, G.idx(lw, 2 * tau, nu >> 1));
              const CT* W1 = Wblk(lw, G.idx(lw, 2 * tau + 1, nu >> 1));
              const int cp = (int)(nu & 1);
              for (int st = 0; st < op.nsteps; ++st)
                fill_step(rec(st), 0, st, [&](int i, int k) {
                  const CT* Ws = k < 16 ? W0 : W1;
                  return cj(Ws[(k & 15) + (cp * 16 + i) * 16], true);
                }, REC_B_T);
            }
          }
        }
      }
    }
  }
  FP.passes = std::move(passes);
  FP.entries = total / (int64_t)sizeof(CT);
  if (total && !g_host_only) {
    BF_CK(cudaMalloc(&FP.F, (size_t)total));
    BF_CK(cudaMemcpy(FP.F, host.data(), (size_t)total, cudaMemcpyHostToDevice));
    *acct += (size_t)total;
  }
}

// --------------------------------------------------------------------------------------
// device plan
// --------------------------------------------------------------------------------------
struct Plan {
  std::vector<Round> rounds;
  void* dev = nullptr;
  int launches() const {
    int k = 0;
    for (auto& r : rounds) k += r.ntasks > 0;
    return k;
  }
};

static void upload_plan(Plan& P, PlanBuilder& pb, int round_lo, int round_hi, size_t* bytes) {
  size_t tot = 0;
  std::vector<size_t> toff, xoff, uoff, coff;
  std::vector<std::vector<int2>> units;
  for (int r = round_lo; r < round_hi && r < (int)pb.tasks.size(); ++r) {
    toff.push_back(tot);
    tot += pb.tasks[r].size() * sizeof(Task);
    tot = (tot + 255) & ~size_t(255);
    xoff.push_back(tot);
    tot += pb.terms[r].size() * sizeof(Term);
    tot = (tot + 255) & ~size_t(255);
    // work units of the tensor-core stage kernel: one per (task, 32-row block)
    std::vector<int2> u;
    for (size_t ti = 0; ti < pb.tasks[r].size(); ++ti)
      for (int rg = 0; rg * 32 < pb.tasks[r][ti].m; ++rg) u.push_back(make_int2((int)ti, rg));
    uoff.push_back(tot);
    tot += u.size() * sizeof(int2);
    tot = (tot + 255) & ~size_t(255);
    units.push_back(std::move(u));
    coff.push_back(tot);
    if (pb.use_cols) {
      tot += pb.cols[r].size() * sizeof(int2);
      tot = (tot + 255) & ~size_t(255);
    }
  }
  if (tot == 0) return;
  std::vector<char> host(tot);
  if (g_host_only) tot = 0;
  for (int r = round_lo, q = 0; r < round_hi && r < (int)pb.tasks.size(); ++r, ++q) {
    if (!pb.tasks[r].empty()) memcpy(host.data() + toff[q], pb.tasks[r].data(), pb.tasks[r].size() * sizeof(Task));
    if (!pb.terms[r].empty()) memcpy(host.data() + xoff[q], pb.terms[r].data(), pb.terms[r].size() * sizeof(Term));
    if (!units[q].empty()) memcpy(host.data() + uoff[q], units[q].data(), units[q].size() * sizeof(int2));
    if (pb.use_cols && !pb.cols[r].empty())
      memcpy(host.data() + coff[q], pb.cols[r].data(), pb.cols[r].size() * sizeof(int2));
  }
  if (tot) {
    BF_CK(cudaMalloc(&P.dev, tot));
    BF_CK(cudaMemcpy(P.dev, host.data(), tot, cudaMemcpyHostToDevice));
    *bytes += tot;
  }
  for (int r = round_lo, q = 0; r < round_hi && r < (int)pb.tasks.size(); ++r, ++q) {
    Round R{};
    R.tasks = reinterpret_cast<const Task*>((char*)P.dev + toff[q]);
    R.terms = reinterpret_cast<const Term*>((char*)P.dev + xoff[q]);
    R.units = reinterpret_cast<const int2*>((char*)P.dev + uoff[q]);
    R.cols = pb.use_cols ? reinterpret_cast<const int2*>((char*)P.dev + coff[q]) : nullptr;
    R.nunits = (int32_t)units[q].size();
    R.ntasks = (int32_t)pb.tasks[r].size();
    R.out_kind = pb.okind[r] < 0 ? 0 : pb.okind[r];
    int mm = 0, mk_ = 0;
    for (auto& t : pb.tasks[r]) mm = std::max(mm, t.m);
    for (auto& t : pb.terms[r]) mk_ = std::max(mk_, t.k);
    R.max_m = mm;
    R.max_k = mk_;
    for (auto& t : pb.tasks[r]) {
      if (pb.okind[r] == 1)
        R.user_out += t.m;
      else
        R.slab_out += t.m;
      for (int q = 0; q < t.nterm; ++q) {
        const Term& x = pb.terms[r][t.term0 + q];
        R.factor_entries += int64_t(t.m) * x.k;
        if (x.in_kind == 1)
          R.user_in += x.k;
        else
          R.slab_in += x.k;
      }
    }
    if (R.ntasks > 0) P.rounds.push_back(R);
  }
}

static void free_plan(Plan& P) {
  if (P.dev) cudaFree(P.dev);
  P.dev = nullptr;
  P.rounds.clear();
}

static void run_plan(int dtype, const Plan& P, StageArgs a, cudaStream_t st, void* const* ev = nullptr,
                     int nev = 0) {
  if (ev) require(nev >= (int)P.rounds.size() + 1, BF_ERR_ARG, "need nrounds + 1 events");
  for (size_t i = 0; i < P.rounds.size(); ++i) {
    if (ev) BF_CK(cudaEventRecord(static_cast<cudaEvent_t>(ev[i]), st));
    launch_round(dtype, P.rounds[i], a, st);
  }
  if (ev) BF_CK(cudaEventRecord(static_cast<cudaEvent_t>(ev[P.rounds.size()]), st));
  BF_CK(cudaGetLastError());
}

static void round_info(int dtype, const Plan& P, int round, bf_round_info_t* info) {
  require(info != nullptr && round >= 0 && round < (int)P.rounds.size(), BF_ERR_ARG, "round out of range");
  const Round& r = P.rounds[round];
  memset(info, 0, sizeof(*info));
  int id = 0;
  const char* nm = round_kernel_name(dtype, r, &id);
  info->kernel = id;
  info->ntasks = r.ntasks;
  info->factor_entries = r.factor_entries;
  info->user_rows_in = r.user_in;
  info->user_rows_out = r.user_out;
  info->slab_rows_in = r.slab_in;
  info->slab_rows_out = r.slab_out;
  strncpy(info->name, nm, sizeof(info->name) - 1);
}

}  // namespace bfa

// ======================================================================================
// handles
// ======================================================================================
using namespace bfa;

// The generic kernel's complex product: 3M (three real products, 25 % fewer tensor-core
// instructions) unless every factor entry is 0, +-1, +-i -- selection blocks such as the identity
// pin, for which the 4M product keeps the apply exact (3M's (a_r + a_i)(b_r + b_i)
// - a_r b_r - a_i b_i rounds even when a is a selection).
static bool selection_only(const void* p, int64_t entries, size_t cs) {
  const int64_t n = entries * 2;
  if (cs == 16) {
    const double* v = static_cast<const double*>(p);
    for (int64_t i = 0; i < n; ++i)
      if (v[i] != 0.0 && v[i] != 1.0 && v[i] != -1.0) return false;
  } else {
    const float* v = static_cast<const float*>(p);
    for (int64_t i = 0; i < n; ++i)
      if (v[i] != 0.f && v[i] != 1.f && v[i] != -1.f) return false;
  }
  return true;
}

// bf_apply_host / hodbf_apply_host pipelining: H2D on one handle-owned stream, the apply on a
// second, D2H on a third, with two alternating device X / Y buffer sets inside the workspace, so
// call k+1's H2D and apply overlap call k's D2H (the two PCIe directions are independent).
struct HostPipe {
  std::mutex mu;  // calls on one handle are serialised
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr, s_cmp = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_cmp[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
  cudaEvent_t ev_st = nullptr;  // the caller's stream at the start of a call
  int64_t calls = 0;
  int last_op = -1;              // (op, nrhs, workspace) of the previous call: a change relocates
  int64_t last_nrhs = -1;        // the buffer sets inside the workspace
  const void* last_work = nullptr;
  void release() {
    if (!s_h2d) return;
    cudaStreamSynchronize(s_h2d);
    cudaStreamSynchronize(s_cmp);
    cudaStreamSynchronize(s_d2h);
    cudaStreamDestroy(s_h2d);
    cudaStreamDestroy(s_cmp);
    cudaStreamDestroy(s_d2h);
    cudaEventDestroy(ev_st);
    for (int k = 0; k < 2; ++k) {
      cudaEventDestroy(ev_h2d[k]);
      cudaEventDestroy(ev_cmp[k]);
      cudaEventDestroy(ev_d2h[k]);
    }
    s_h2d = nullptr;
  }
};

struct bf_s {
  int dtype = BF_C128;
  int device = 0;
  Geom G;
  void* pool = nullptr;
  int32_t m3 = 1;  // generic kernel: 3M complex products (0: 4M, every factor entry 0 / +-1 / +-i)
  int64_t* d_rperm = nullptr;
  int64_t* d_cperm = nullptr;
  int64_t slab_rows = 0;
  int64_t factor_entries = 0;
  size_t device_bytes = 0;
  Plan plan[2];  // [0] op N, [1] op C/T
  bool use_fast = false;
  bool fused_only = false;  // BF_CREATE_FUSED_ONLY: the generic pool was released after the fused build
  FastPlan fast[2];
  // distributed
  bool dist = false;
  int rank = 0, nranks = 1;
  void* nccl = nullptr;  // bf_create_dist: the caller's ncclComm_t (not owned)
  Plan pre[2], post[2];
  int64_t send_rows[2] = {0, 0}, recv_rows[2] = {0, 0};
  int64_t send_base[2] = {0, 0}, recv_base[2] = {0, 0};  // slab rows
  std::vector<int64_t> send_cnt[2], recv_cnt[2];         // rows per peer
  std::vector<int64_t> send_blk[2], recv_blk[2];         // centre blocks in exchange-region order
  bool host_only = false;
  int64_t loc_rows_in[2] = {0, 0}, loc_rows_out[2] = {0, 0};
  int64_t loc_user_in[2] = {0, 0}, loc_user_out[2] = {0, 0};
  int64_t* d_lperm_in[2] = {nullptr, nullptr};
  int64_t* d_lperm_out[2] = {nullptr, nullptr};
  // bf_apply_host pipelining: copy streams, per-buffer-set events, call counter
  std::mutex hmu;
  HostPipe hp;
  std::vector<int64_t> h_rinv, h_cinv;  // bf_extract: user index -> tree position (filled on first use)
  XScratch xs;                          // bf_extract's device scratch
  ~bf_s() {
    if (host_only) return;
    cudaSetDevice(device);
    hp.release();
    for (int k = 0; k < 2; ++k) {
      free_plan(plan[k]);
      free_plan(pre[k]);
      free_plan(post[k]);
    }
    if (d_lperm_in[0]) cudaFree(d_lperm_in[0]);  // [1] aliases [0] with in / out swapped
    if (d_lperm_out[0]) cudaFree(d_lperm_out[0]);
    for (int k = 0; k < 2; ++k)
      if (fast[k].F) cudaFree(fast[k].F);
    if (pool) cudaFree(pool);
    if (d_rperm) cudaFree(d_rperm);
    if (d_cperm) cudaFree(d_cperm);
  }
};

struct hodbf_s {
  int dtype = BF_C128;
  int device = 0;
  int64_t n = 0;
  int LH = 0;
  void* pool = nullptr;
  int32_t m3 = 1;  // as bf_s::m3
  // hodbf_extract: tree geometry and pool layout kept from create
  std::vector<int64_t> lp, inv;              // leaf offsets; user index -> tree position
  std::vector<Geom> G;                       // every off-diagonal butterfly (level-major)
  std::vector<FBase> F;                      // their R / B / W pool offsets
  std::vector<int64_t> M_off, SV_off, sumc;  // per leaf: [D | U^(1..LH)] and stacked Vt
  std::vector<int64_t> ustart, vstart;       // [leaf][l]: first U column / Vt row of level l
  XScratch xs;
  int64_t* d_perm = nullptr;
  int64_t slab_rows = 0;
  int64_t factor_entries = 0;
  size_t device_bytes = 0;
  Plan plan[2];
  HostPipe hp;  // hodbf_apply_host
  ~hodbf_s() {
    cudaSetDevice(device);
    hp.release();
    free_plan(plan[0]);
    free_plan(plan[1]);
    if (pool) cudaFree(pool);
    if (d_perm) cudaFree(d_perm);
  }
};

namespace bfa {

static int fail(const Err& e) {
  g_last_error = e.msg;
  return e.code;
}

static void check_device(int device) {
  int cnt = 0;
  cudaError_t e = cudaGetDeviceCount(&cnt);
  require(e == cudaSuccess && cnt > 0, BF_ERR_DEVICE, "no CUDA device available (libbfapply has no CPU path)");
  require(device >= 0 && device < cnt, BF_ERR_DEVICE, "device index out of range");
  int major = 0;
  BF_CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  require(major == 10, BF_ERR_DEVICE, "libbfapply is built for sm_100a (B200); device is not compute capability 10.x");
}

static void* upload(const void* h, size_t bytes, size_t* acct) {
  if (bytes == 0 || g_host_only) return nullptr;
  void* d = nullptr;
  BF_CK(cudaMalloc(&d, bytes));
  BF_CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
  *acct += bytes;
  return d;
}

// canonical slab allocation for a whole (single-GPU) butterfly: col space 0..lc, row space lc..L
static Slabs canonical_slabs(const Geom& G, int64_t& cursor) {
  Slabs S;
  S.col.assign((size_t)(G.lc + 1) * G.nb, -1);
  S.row.assign((size_t)(G.L - G.lc + 1) * G.nb, -1);
  for (int l = 0; l <= G.lc; ++l)
    for (int64_t i = 0; i < G.nb; ++i) {
      S.col[(size_t)l * G.nb + i] = cursor;
      cursor += G.c(l, i);
    }
  for (int l = G.lc; l <= G.L; ++l)
    for (int64_t i = 0; i < G.nb; ++i) {
      S.row[(size_t)(l - G.lc) * G.nb + i] = cursor;
      cursor += G.r(l, i);
    }
  return S;
}

// slab rows of the touched blocks only (bf_extract): untouched blocks get none (no term reads
// them -- emit_N drops their terms)
static Slabs touched_slabs(const Geom& G, const Touch& T, int64_t& cursor) {
  Slabs S;
  S.col.assign((size_t)(G.lc + 1) * G.nb, -1);
  S.row.assign((size_t)(G.L - G.lc + 1) * G.nb, -1);
  for (int l = 0; l <= G.lc; ++l)
    for (int64_t tau : T.rows[l])
      for (int64_t nu : T.cols[l]) {
        const int64_t i = G.idx(l, tau, nu);
        S.col[(size_t)l * G.nb + i] = cursor;
        cursor += G.c(l, i);
      }
  for (int l = G.lc; l <= G.L; ++l)
    for (int64_t tau : T.rows[l])
      for (int64_t nu : T.cols[l]) {
        const int64_t i = G.idx(l, tau, nu);
        S.row[(size_t)(l - G.lc) * G.nb + i] = cursor;
        cursor += G.r(l, i);
      }
  return S;
}

static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

static void validate_apply(int64_t nrhs, const void* X, int64_t ldx, int64_t rows_x, const void* Y,
                           int64_t ldy, int64_t rows_y, size_t work_bytes, size_t need, size_t cs) {
  require(nrhs >= 0, BF_ERR_ARG, "nrhs < 0");
  if (nrhs == 0) return;
  require(X != nullptr && Y != nullptr, BF_ERR_ARG, "X or Y is NULL");
  require(ldx >= std::max<int64_t>(rows_x, 1) && ldy >= std::max<int64_t>(rows_y, 1), BF_ERR_ARG,
          "leading dimension smaller than the number of rows");
  // X and Y must not overlap: compare the byte extents [first element, last element] of the two
  // column-major blocks (the apply reads X after it has started writing Y)
  const uintptr_t x0 = reinterpret_cast<uintptr_t>(X), y0 = reinterpret_cast<uintptr_t>(Y);
  const uintptr_t x1 = x0 + (uintptr_t)(((nrhs - 1) * ldx + std::max<int64_t>(rows_x, 1)) * (int64_t)cs);
  const uintptr_t y1 = y0 + (uintptr_t)(((nrhs - 1) * ldy + std::max<int64_t>(rows_y, 1)) * (int64_t)cs);
  require(x1 <= y0 || y1 <= x0, BF_ERR_ARG, "X and Y must not overlap");
  require(work_bytes >= need, BF_ERR_ARG, "workspace too small");
}

}  // namespace bfa

// ======================================================================================
// C ABI
// ======================================================================================
extern "C" {

const char* bf_status_string(int s) {
  switch (s) {
    case BF_OK: return "BF_OK";
    case BF_ERR_ARG: return "BF_ERR_ARG";
    case BF_ERR_SHAPE: return "BF_ERR_SHAPE";
    case BF_ERR_RANK: return "BF_ERR_RANK";
    case BF_ERR_PERM: return "BF_ERR_PERM";
    case BF_ERR_CUDA: return "BF_ERR_CUDA";
    case BF_ERR_OOM: return "BF_ERR_OOM";
    case BF_ERR_NCCL: return "BF_ERR_NCCL";
    case BF_ERR_DEVICE: return "BF_ERR_DEVICE";
    default: return "BF_ERR_UNKNOWN";
  }
}

const char* bf_last_error(void) { return bfa::g_last_error.c_str(); }

const char* bf_version(void) { return "bfapply 0.1 sm_100a"; }

int bf_create(const bf_desc* d, int device, bf_handle* out) {
  if (!d || !out) return fail(Err{BF_ERR_ARG, "NULL argument"});
  *out = nullptr;
  try {
    Canon cn_;
    d = &canonical(*d, cn_);
    Geom G = make_geom(*d);
    check_perm(d->row_perm, d->m, "row_perm");
    check_perm(d->col_perm, d->n, "col_perm");
    check_device(device);
    DeviceGuard dg(device);
    std::unique_ptr<bf_s> h(new bf_s());
    h->dtype = d->dtype;
    h->device = device;
    const size_t cs = csize(d->dtype);
    const int64_t tot = G.len_U + G.len_R + G.len_B + G.len_W + G.len_Vt;
    h->factor_entries = tot;
    FBase F;
    F.u = 0;
    F.r = G.len_U;
    F.b = F.r + G.len_R;
    F.w = F.b + G.len_B;
    F.vt = F.w + G.len_W;
    if (tot > 0) {
      BF_CK(cudaMalloc(&h->pool, (size_t)tot * cs));
      h->device_bytes += (size_t)tot * cs;
      char* p = static_cast<char*>(h->pool);
      if (G.len_U) BF_CK(cudaMemcpy(p + F.u * cs, d->U, G.len_U * cs, cudaMemcpyHostToDevice));
      if (G.len_R) BF_CK(cudaMemcpy(p + F.r * cs, d->R, G.len_R * cs, cudaMemcpyHostToDevice));
      if (G.len_B) BF_CK(cudaMemcpy(p + F.b * cs, d->B, G.len_B * cs, cudaMemcpyHostToDevice));
      if (G.len_W) BF_CK(cudaMemcpy(p + F.w * cs, d->W, G.len_W * cs, cudaMemcpyHostToDevice));
      if (G.len_Vt) BF_CK(cudaMemcpy(p + F.vt * cs, d->Vt, G.len_Vt * cs, cudaMemcpyHostToDevice));
    }
    h->m3 = !(selection_only(d->U, G.len_U, cs) && selection_only(d->R, G.len_R, cs) &&
              selection_only(d->B, G.len_B, cs) && selection_only(d->W, G.len_W, cs) &&
              selection_only(d->Vt, G.len_Vt, cs));
    // an identity permutation is stored as NULL (no per-row index loads on the device)
    auto is_id = [](const int64_t* p, int64_t n) {
      for (int64_t i = 0; i < n; ++i)
        if (p[i] != i) return false;
      return true;
    };
    if (d->row_perm && !is_id(d->row_perm, d->m)) h->d_rperm = (int64_t*)upload(d->row_perm, d->m * 8, &h->device_bytes);
    if (d->col_perm && !is_id(d->col_perm, d->n)) h->d_cperm = (int64_t*)upload(d->col_perm, d->n * 8, &h->device_bytes);
    int64_t cursor = 0;
    Slabs S = canonical_slabs(G, cursor);
    h->slab_rows = cursor;
    for (int k = 0; k < 2; ++k) {
      PlanBuilder pb;
      EmitOpts o;
      if (k == 0)
        emit_N(pb, G, F, S, o);
      else
        emit_C(pb, G, F, S, o);
      upload_plan(h->plan[k], pb, 0, (int)pb.tasks.size(), &h->device_bytes);
    }
    // the fused kernels use the 3M product; selection factors (every entry 0 / +-1 / +-i, the
    // identity pin) stay on the generic path, whose 4M product keeps their apply exact
    // the fused kernels: uniform rank 16 as given, ranks <= 16 zero-padded to 16 (pad_rank16; env
    // BF_FAST_PAD = 0 keeps ragged ranks on the generic path, for A/B measurements)
    static const bool pad_ok = !getenv("BF_FAST_PAD") || atoi(getenv("BF_FAST_PAD")) != 0;
    if (fast_eligible(G, d->dtype, !pad_ok) && h->m3 && !getenv("BF_DISABLE_FAST") && pad_pays(G, tot, cs)) {
      const bool cc = leaves_contiguous(d->col_perm, d->n, G.nv(0));
      const bool rc = leaves_contiguous(d->row_perm, d->m, G.mt(0));
      const bool exact = fast_eligible(G, d->dtype, true);
      auto build = [&](auto* tag) {
        using CT = std::remove_pointer_t<decltype(tag)>;
        Padded16<CT> P;
        if (!exact) pad_rank16(*d, G, P);
        const HostFactors<CT> HF = exact ? HostFactors<CT>{static_cast<const CT*>(d->U), static_cast<const CT*>(d->R),
                                                           static_cast<const CT*>(d->B), static_cast<const CT*>(d->W),
                                                           static_cast<const CT*>(d->Vt)}
                                         : HostFactors<CT>{P.U.data(), P.R.data(), P.B.data(), P.W.data(), P.Vt.data()};
        const Geom& GF = exact ? G : P.G;
        for (int k = 0; k < 2; ++k) {
          if (sizeof(CT) == 16) build_fast(h->fast[k], GF, HF, k, &h->device_bytes, -1, 0, k == 0 ? cc : rc);
          else build_fast(h->fast[k], GF, HF, k, &h->device_bytes);
        }
      };
      if (d->dtype == BF_C128) build((double2*)nullptr);
      else build((float2*)nullptr);
      h->fast[0].contig_in = cc;
      h->fast[0].contig_out = rc;
      h->fast[1].contig_in = rc;
      h->fast[1].contig_out = cc;
      h->use_fast = true;
      if ((d->flags & BF_CREATE_FUSED_ONLY) && h->pool) {
        // every op now runs on the fused records: release the generic pool (one of the three
        // copies of the factors; extraction and export need it and then return BF_ERR_ARG)
        BF_CK(cudaFree(h->pool));
        h->pool = nullptr;
        h->device_bytes -= (size_t)tot * cs;
        h->fused_only = true;
      }
    }
    h->G = std::move(G);
    *out = h.release();
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  } catch (const std::bad_alloc&) {
    return fail(Err{BF_ERR_OOM, "host allocation failed"});
  }
}

int bf_destroy(bf_handle h) {
  delete h;
  return BF_OK;
}

int bf_info(bf_handle h, bf_info_t* info) {
  if (!h || !info) return fail(Err{BF_ERR_ARG, "NULL argument"});
  info->factor_entries = h->factor_entries;
  info->device_bytes = (int64_t)h->device_bytes;
  if (h->dist && !h->use_fast) {
    info->launches_n = h->pre[0].launches() + h->post[0].launches();
    info->launches_c = h->pre[1].launches() + h->post[1].launches();
  } else if (h->use_fast) {
    info->launches_n = (int32_t)h->fast[0].passes.size();
    info->launches_c = (int32_t)h->fast[1].passes.size();
  } else {
    info->launches_n = h->plan[0].launches();
    info->launches_c = h->plan[1].launches();
  }
  info->rows_in = h->G.n;
  info->rows_out = h->G.m;
  return BF_OK;
}

// Copy a (single-GPU) handle's factors back to host arrays in the bf_desc layout: the five
// packed arrays and the two rank arrays.  lens (5 entries) receives the element counts of U, R,
// B, W, Vt; any output pointer may be NULL (then only lens / ranks are filled).  Used to hand a
// butterfly built on the device (bf_random_matvec) to host tooling and to the CPU oracle.
int bf_export(bf_handle h, int64_t* lens, int32_t* rank_row, int32_t* rank_col, void* U, void* R, void* B, void* W,
              void* Vt) {
  if (!h) return fail(Err{BF_ERR_ARG, "NULL handle"});
  try {
    require(!h->dist, BF_ERR_ARG, "bf_export: distributed handles hold a rank-local part only");
    const Geom& G = h->G;
    const int64_t L5[5] = {G.len_U, G.len_R, G.len_B, G.len_W, G.len_Vt};
    if (lens)
      for (int q = 0; q < 5; ++q) lens[q] = L5[q];
    if (rank_row) std::copy(G.rr.begin(), G.rr.end(), rank_row);
    if (rank_col) std::copy(G.rc.begin(), G.rc.end(), rank_col);
    DeviceGuard dg(h->device);
    const size_t cs = csize(h->dtype);
    void* dst[5] = {U, R, B, W, Vt};
    require(!h->fused_only || !(U || R || B || W || Vt), BF_ERR_ARG,
            "handle created with BF_CREATE_FUSED_ONLY keeps no factor pool to export");
    int64_t off = 0;
    for (int q = 0; q < 5; ++q) {
      if (dst[q] && L5[q]) BF_CK(cudaMemcpy(dst[q], static_cast<char*>(h->pool) + off * cs, L5[q] * cs, cudaMemcpyDeviceToHost));
      off += L5[q];
    }
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

// fast-path workspace: two slab buffers (every slab of a level, [tile][half][slab][16 x 16]) and,
// on a split handle, the send and recv regions of the centre exchange (2^L / P slabs each)
static size_t fast_buf_bytes(bf_handle h, int64_t nrhs) {
  const size_t tiles = (size_t)((nrhs + FAST_NB - 1) / FAST_NB);
  return align256((size_t)h->G.nb * tiles * FAST_SLAB * csize(h->dtype));
}
static size_t fast_x_bytes(bf_handle h, int64_t nrhs) {
  if (!h->dist) return 0;
  return align256(fast_buf_bytes(h, nrhs) / (size_t)h->nranks);
}
static size_t fast_ws(bf_handle h, int64_t nrhs) {
  if (!h->use_fast) return 0;
  return 2 * fast_buf_bytes(h, nrhs) + 2 * fast_x_bytes(h, nrhs);
}

int bf_workspace_size(bf_handle h, int64_t nrhs, size_t* bytes) {
  if (!h || !bytes || nrhs < 0) return fail(Err{BF_ERR_ARG, "bad argument"});
  if (h->use_fast && !h->dist)
    *bytes = fast_ws(h, nrhs);
  else
    *bytes = align256((size_t)h->slab_rows * (size_t)nrhs * csize(h->dtype));
  return BF_OK;
}

// launches [lo, hi) of the fast plan of op slot k.  Workspace: two slab buffers, then (split
// handles only) the send and the recv region of the centre exchange.
static void run_fast(bf_handle h, int k, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
                     void* work, cudaStream_t st, void* const* ev, int nev, int lo = 0, int hi = -1,
                     void* const* peer_recv = nullptr) {
  const FastPlan& FP = h->fast[k];
  if (hi < 0) hi = (int)FP.passes.size();
  if (ev) require(nev >= hi - lo + 1, BF_ERR_ARG, "need nrounds + 1 events");
  const size_t bufb = fast_buf_bytes(h, nrhs), xb = fast_x_bytes(h, nrhs);
  char* buf[2] = {static_cast<char*>(work), static_cast<char*>(work) + bufb};
  char* sendb = static_cast<char*>(work) + 2 * bufb;
  char* recvb = sendb + xb;
  const bool fwd = k == 0;
  const int diag = getenv("BF_FAST_DIAG") ? atoi(getenv("BF_FAST_DIAG")) : 0;
  const int32_t no_pairw = getenv("BF_NO_PAIRW") ? 1 : 0;
  const int32_t ntiles = (int32_t)((nrhs + FAST_NB - 1) / FAST_NB);
  for (int i = lo; i < hi; ++i) {
    const FastPass& P = FP.passes[i];
    if (ev) BF_CK(cudaEventRecord(static_cast<cudaEvent_t>(ev[i - lo]), st));
    if (P.leaf) {
      LeafArgs a{};
      a.mode = P.leaf == 1 ? 0 : 1;
      a.F = static_cast<const char*>(FP.F) + P.fbase;
      a.X = X;
      a.ldx = ldx;
      a.xperm = h->dist ? h->d_lperm_in[k] : fwd ? h->d_cperm : h->d_rperm;
      a.Y = Y;
      a.ldy = ldy;
      a.yperm = h->dist ? h->d_lperm_out[k] : fwd ? h->d_rperm : h->d_cperm;
      a.Sin = buf[i % 2];
      a.Sout = buf[(i + 1) % 2];
      a.nleaf = P.nwin;
      a.leaf_lo = P.a_lo + P.b_lo;  // one of them is 0 (d = 0 windows)
      a.nlev = h->G.nb;
      a.leaf = P.ops[0].leaf;
      a.nsteps = P.ops[0].nsteps;
      a.nrhs = (int32_t)nrhs;
      a.conj_io = op == BF_OP_T ? 1 : 0;
      // user rows of every leaf contiguous: X by TMA tiles (IN) / Y by base + offset (OUT)
      a.tma = (a.mode == 0 ? FP.contig_in : FP.contig_out) && !getenv("BF_DISABLE_TMA") ? 1 : 0;
      a.diag = diag;
      launch_leaf(h->dtype, a, st);
    } else {
      FastArgs a{};
      a.p = P;
      a.diag = diag;
      a.no_pairw = no_pairw;
      a.skew = getenv("BF_FAST_SKEW") ? atoi(getenv("BF_FAST_SKEW")) : 0;
      // column halves with work: 2; 1 when nrhs <= 16; 0 (narrow, 8 columns) when nrhs <= 8
      a.halves = getenv("BF_NO_HALF_SKIP") ? 2 : nrhs <= 8 && !getenv("BF_NO_NARROW") ? 0 : nrhs <= FAST_HC ? 1 : 2;
      if (peer_recv && P.xout) {  // fused peer-memory exchange
        a.p2p = 1;
        a.myrank = h->rank;
        for (int q = 0; q < h->nranks; ++q) a.peer[q] = peer_recv[q];
      }
      a.F = FP.F;
      a.Sin = P.xin ? recvb : buf[i % 2];
      a.Sout = P.xout ? sendb : buf[(i + 1) % 2];
      a.nlev = h->G.nb;
      a.nrhs = (int32_t)nrhs;
      a.ntiles = ntiles;
      if (P.xleaf) {  // fused column leaf: X rows by 2-D TMA tiles
        const int S = 1 << P.d, cs = (int)csize(h->dtype);
        const int64_t rows = P.user_in;
        require(fast_make_xmap(h->dtype, X, rows, nrhs, ldx, fast_spl(cs, S) * fast_ks(cs), &a.xmap), BF_ERR_ARG,
                "X must be 16-byte aligned with a 16-byte multiple column stride");
        a.X = X;
        a.xperm = fwd ? h->d_cperm : h->d_rperm;
      }
      a.Y = Y;  // fused leaf-out (last pass)
      a.ldy = ldy;
      a.yperm = h->dist ? h->d_lperm_out[k] : fwd ? h->d_rperm : h->d_cperm;
      a.conj_io = op == BF_OP_T ? 1 : 0;
      a.ycontig = FP.contig_out ? 1 : 0;
      launch_fast_pass(h->dtype, a, st);
    }
    if (getenv("BF_DEBUG_SYNC")) {
      cudaError_t e = cudaStreamSynchronize(st);
      fprintf(stderr, "bfapply debug: launch %d (leaf=%d d=%d l0=%d nops=%d nwin=%lld) -> %s\n", i, P.leaf, P.d, P.l0,
              P.nops, (long long)P.nwin, cudaGetErrorString(e));
      BF_CK(e);
    }
  }
  if (ev) BF_CK(cudaEventRecord(static_cast<cudaEvent_t>(ev[hi - lo]), st));
  BF_CK(cudaGetLastError());
}

int bf_apply_op_events(bf_handle h, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
                       void* work, size_t work_bytes, bf_stream_t stream, void* const* events, int32_t nevents) {
  if (!h) return fail(Err{BF_ERR_ARG, "NULL handle"});
  try {
    require(op == BF_OP_N || op == BF_OP_C || op == BF_OP_T, BF_ERR_ARG, "bad op");
    require(!h->dist, BF_ERR_ARG, "distributed handle: use bf_dist_apply_pre/post");
    const bool fwd = op == BF_OP_N;
    const int64_t rx = fwd ? h->G.n : h->G.m, ry = fwd ? h->G.m : h->G.n;
    size_t need = 0;
    bf_workspace_size(h, nrhs, &need);
    validate_apply(nrhs, X, ldx, rx, Y, ldy, ry, work_bytes, need, csize(h->dtype));
    if (nrhs == 0 || ry == 0) return BF_OK;
    require(need == 0 || work != nullptr, BF_ERR_ARG, "workspace is NULL");
    DeviceGuard dg(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (rx == 0 || h->plan[fwd ? 0 : 1].rounds.empty()) {
      // K has no columns (or no entries): Y = 0
      for (int64_t j = 0; j < nrhs; ++j)
        BF_CK(cudaMemsetAsync((char*)Y + (size_t)j * ldy * csize(h->dtype), 0, (size_t)ry * csize(h->dtype), st));
    }
    StageArgs a{};
    a.pool = h->pool;
    a.m3 = h->m3;
    a.X = X;
    a.ldx = ldx;
    a.xperm = fwd ? h->d_cperm : h->d_rperm;
    a.S = work;
    a.ldS = nrhs;
    a.Y = Y;
    a.ldy = ldy;
    a.yperm = fwd ? h->d_rperm : h->d_cperm;
    a.conj_flip = (op == BF_OP_T) ? 1 : 0;
    a.nrhs = (int32_t)nrhs;
    require(nrhs <= (int64_t)65535 * 32, BF_ERR_ARG, "nrhs too large for one launch");
    if (h->use_fast) {
      run_fast(h, fwd ? 0 : 1, op, nrhs, X, ldx, Y, ldy, work, st, events, nevents);
      return BF_OK;
    }
    run_plan(h->dtype, h->plan[fwd ? 0 : 1], a, st, events, nevents);
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

int bf_apply_op(bf_handle h, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
                void* work, size_t work_bytes, bf_stream_t stream) {
  return bf_apply_op_events(h, op, nrhs, X, ldx, Y, ldy, work, work_bytes, stream, nullptr, 0);
}

int bf_rounds(bf_handle h, int op, int32_t* n) {
  if (!h || !n) return fail(Err{BF_ERR_ARG, "NULL argument"});
  const int k = op == BF_OP_N ? 0 : 1;
  if (h->use_fast)
    *n = (int32_t)h->fast[k].passes.size();
  else
    *n = h->dist ? (int32_t)(h->pre[k].rounds.size() + h->post[k].rounds.size()) : (int32_t)h->plan[k].rounds.size();
  return BF_OK;
}

int bf_round_info(bf_handle h, int op, int32_t round, bf_round_info_t* info) {
  if (!h) return fail(Err{BF_ERR_ARG, "NULL handle"});
  try {
    const int k = op == BF_OP_N ? 0 : 1;
    if (h->use_fast) {
      require(info && round >= 0 && round < (int)h->fast[k].passes.size(), BF_ERR_ARG, "round out of range");
      const FastPass& P = h->fast[k].passes[round];
      memset(info, 0, sizeof(*info));
      info->kernel = P.leaf ? 10 + P.leaf : 10;  // 10 window pass, 11 leaf in, 12 leaf out
      info->ntasks = (int32_t)P.nwin;
      info->factor_entries = P.factor_entries;
      info->user_rows_in = P.user_in;
      info->user_rows_out = P.user_out;
      info->slab_rows_in = P.in_s >= 0 ? h->G.nb * FAST_RANK : 0;
      info->slab_rows_out = P.out_s >= 0 ? h->G.nb * FAST_RANK : 0;
      strncpy(info->name, P.leaf ? leaf_kernel_name(h->dtype, P.leaf - 1) : fast_kernel_name(h->dtype),
              sizeof(info->name) - 1);
      return BF_OK;
    }
    if (h->dist) {
      const int np = (int)h->pre[k].rounds.size();
      if (round < np)
        round_info(h->dtype, h->pre[k], round, info);
      else
        round_info(h->dtype, h->post[k], round - np, info);
    } else {
      round_info(h->dtype, h->plan[k], round, info);
    }
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

int bf_apply(bf_handle h, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy, void* work,
             size_t work_bytes, bf_stream_t stream) {
  return bf_apply_op(h, BF_OP_N, nrhs, X, ldx, Y, ldy, work, work_bytes, stream);
}

int bf_apply_adj(bf_handle h, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy, void* work,
                 size_t work_bytes, bf_stream_t stream) {
  return bf_apply_op(h, BF_OP_C, nrhs, X, ldx, Y, ldy, work, work_bytes, stream);
}

int bf_workspace_size_host(bf_handle h, int op, int64_t nrhs, size_t* bytes) {
  if (!h || !bytes || nrhs < 0) return fail(Err{BF_ERR_ARG, "bad argument"});
  const bool fwd = op == BF_OP_N;
  const int64_t rx = fwd ? h->G.n : h->G.m, ry = fwd ? h->G.m : h->G.n;
  size_t s = 0;
  bf_workspace_size(h, nrhs, &s);
  const size_t cs = csize(h->dtype);
  // two sets of device X / Y copies: consecutive calls alternate between them
  *bytes = s + 2 * (align256((size_t)rx * nrhs * cs) + align256((size_t)ry * nrhs * cs));
  return BF_OK;
}

}  // extern "C"

namespace bfa {
// One host-to-host apply through the HostPipe: H2D of X into buffer set k & 1 (after call k - 2's
// D2H released it; after a relayout, after both sets' D2H), the apply on the compute stream (after
// this call's H2D only), D2H of Y; the caller's stream waits for the D2H, so Y_host is complete
// in its order.  The workspace belongs to this pipeline between calls; on the first call and
// after a relayout the copies and the apply also wait for the caller's earlier work on `st` (e.g.
// the workspace's allocation).  Layout of `work`: [apply workspace s][set 0: X | Y][set 1: X | Y].
template <class Apply>
static void host_pipeline(HostPipe& hp, int op, int64_t nrhs, const void* Xh, int64_t ldx, int64_t rx, void* Yh,
                          int64_t ldy, int64_t ry, void* work, size_t s, size_t cs, cudaStream_t st, Apply apply) {
  std::lock_guard<std::mutex> lk(hp.mu);
  if (!hp.s_h2d) {
    BF_CK(cudaStreamCreateWithFlags(&hp.s_h2d, cudaStreamNonBlocking));
    BF_CK(cudaStreamCreateWithFlags(&hp.s_cmp, cudaStreamNonBlocking));
    BF_CK(cudaStreamCreateWithFlags(&hp.s_d2h, cudaStreamNonBlocking));
    BF_CK(cudaEventCreateWithFlags(&hp.ev_st, cudaEventDisableTiming));
    for (int k = 0; k < 2; ++k) {
      BF_CK(cudaEventCreateWithFlags(&hp.ev_h2d[k], cudaEventDisableTiming));
      BF_CK(cudaEventCreateWithFlags(&hp.ev_cmp[k], cudaEventDisableTiming));
      BF_CK(cudaEventCreateWithFlags(&hp.ev_d2h[k], cudaEventDisableTiming));
    }
  }
  const size_t bx = align256((size_t)rx * nrhs * cs), by = align256((size_t)ry * nrhs * cs);
  const int set = (int)(hp.calls & 1);
  char* dX = static_cast<char*>(work) + s + set * (bx + by);
  char* dY = dX + bx;
  // The X / Y regions of a set move with (op, nrhs) -- the slab workspace grows with nrhs and rx /
  // ry swap with op -- and with the workspace pointer, so after such a change this call's regions
  // may overlap the other set's: wait for both.
  const bool relayout = hp.calls > 0 && (op != hp.last_op || nrhs != hp.last_nrhs || work != hp.last_work);
  if (hp.calls >= 2) BF_CK(cudaStreamWaitEvent(hp.s_h2d, hp.ev_d2h[set], 0));
  if (relayout) BF_CK(cudaStreamWaitEvent(hp.s_h2d, hp.ev_d2h[set ^ 1], 0));
  if (hp.calls == 0 || relayout) {
    BF_CK(cudaEventRecord(hp.ev_st, st));
    BF_CK(cudaStreamWaitEvent(hp.s_h2d, hp.ev_st, 0));
    BF_CK(cudaStreamWaitEvent(hp.s_cmp, hp.ev_st, 0));
  }
  hp.last_op = op;
  hp.last_nrhs = nrhs;
  hp.last_work = work;
  if (ldx == rx)
    BF_CK(cudaMemcpyAsync(dX, Xh, (size_t)rx * nrhs * cs, cudaMemcpyHostToDevice, hp.s_h2d));
  else
    BF_CK(cudaMemcpy2DAsync(dX, rx * cs, Xh, ldx * cs, rx * cs, nrhs, cudaMemcpyHostToDevice, hp.s_h2d));
  BF_CK(cudaEventRecord(hp.ev_h2d[set], hp.s_h2d));
  BF_CK(cudaStreamWaitEvent(hp.s_cmp, hp.ev_h2d[set], 0));
  const int rc = apply(dX, dY, hp.s_cmp);
  if (rc != BF_OK) throw Err{rc, bf_last_error()};
  BF_CK(cudaEventRecord(hp.ev_cmp[set], hp.s_cmp));
  BF_CK(cudaStreamWaitEvent(hp.s_d2h, hp.ev_cmp[set], 0));
  if (ldy == ry)
    BF_CK(cudaMemcpyAsync(Yh, dY, (size_t)ry * nrhs * cs, cudaMemcpyDeviceToHost, hp.s_d2h));
  else
    BF_CK(cudaMemcpy2DAsync(Yh, ldy * cs, dY, ry * cs, ry * cs, nrhs, cudaMemcpyDeviceToHost, hp.s_d2h));
  BF_CK(cudaEventRecord(hp.ev_d2h[set], hp.s_d2h));
  BF_CK(cudaStreamWaitEvent(st, hp.ev_d2h[set], 0));
  ++hp.calls;
}
}  // namespace bfa

extern "C" {

// Host-memory apply, pipelined across calls (host_pipeline): every call's own copies are inside
// it, and `stream` waits for this call's D2H, so Y_host is complete when the caller synchronises it.
int bf_apply_host(bf_handle h, int op, int64_t nrhs, const void* Xh, int64_t ldx, void* Yh, int64_t ldy,
                  void* work, size_t work_bytes, bf_stream_t stream) {
  if (!h) return fail(Err{BF_ERR_ARG, "NULL handle"});
  try {
    const bool fwd = op == BF_OP_N;
    const int64_t rx = fwd ? h->G.n : h->G.m, ry = fwd ? h->G.m : h->G.n;
    size_t need = 0, s = 0;
    bf_workspace_size_host(h, op, nrhs, &need);
    bf_workspace_size(h, nrhs, &s);
    validate_apply(nrhs, Xh, ldx, rx, Yh, ldy, ry, work_bytes, need, csize(h->dtype));
    if (nrhs == 0) return BF_OK;
    DeviceGuard dg(h->device);
    host_pipeline(h->hp, op, nrhs, Xh, ldx, rx, Yh, ldy, ry, work, s, csize(h->dtype), static_cast<cudaStream_t>(stream),
                  [&](void* dX, void* dY, cudaStream_t sc) {
                    return bf_apply_op(h, op, nrhs, dX, std::max<int64_t>(rx, 1), dY, std::max<int64_t>(ry, 1), work,
                                       s, sc);
                  });
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

// --------------------------------------------------------------------------------------
// HOD-BF
// --------------------------------------------------------------------------------------
int hodbf_create(const hodbf_desc* d, int device, hodbf_handle* out) {
  if (!d || !out) return fail(Err{BF_ERR_ARG, "NULL argument"});
  *out = nullptr;
  try {
    require(d->dtype == BF_C64 || d->dtype == BF_C128, BF_ERR_ARG, "bad dtype");
    require(d->LH >= 0 && d->LH <= 20, BF_ERR_SHAPE, "LH out of range [0, 20]");
    const int LH = d->LH;
    const int64_t nleaf = int64_t(1) << LH;
    check_leafptr(d->leaf_ptr, nleaf, d->n, "leaf_ptr");
    check_perm(d->perm, d->n, "perm");
    const int64_t* lp = d->leaf_ptr;
    int64_t lenD = 0;
    for (int64_t t = 0; t < nleaf; ++t) lenD += (lp[t + 1] - lp[t]) * (lp[t + 1] - lp[t]);
    require(d->len_D == lenD && (lenD == 0 || d->D), BF_ERR_SHAPE, "len_D does not match the leaf sizes");
    const int64_t nbf = 2 * nleaf - 2;
    require(nbf == 0 || d->offdiag, BF_ERR_ARG, "offdiag is NULL");
    // off-diagonal butterflies with level_maps: re-packed to canonical order (the rest of the
    // create reads d->offdiag only)
    std::vector<Canon> cns;
    std::vector<bf_desc> offc;
    hodbf_desc dc;
    for (int64_t k = 0; k < nbf; ++k)
      if (d->offdiag[k].level_maps) {
        cns.resize((size_t)nbf);
        offc.resize((size_t)nbf);
        for (int64_t q = 0; q < nbf; ++q) offc[q] = canonical(d->offdiag[q], cns[q]);
        dc = *d;
        dc.offdiag = offc.data();
        d = &dc;
        break;
      }
    // geometry of every off-diagonal butterfly, checked against the HOD-BF tree
    std::vector<Geom> G(nbf);
    for (int l = 1; l <= LH; ++l)
      for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau) {
        const int64_t k = (int64_t(1) << l) - 2 + tau;
        const bf_desc& b = d->offdiag[k];
        require(b.dtype == d->dtype, BF_ERR_ARG, "offdiag dtype differs");
        require(b.L == LH - l, BF_ERR_SHAPE, "offdiag butterfly must have LH - l levels");
        require(b.row_perm == nullptr && b.col_perm == nullptr, BF_ERR_PERM, "offdiag perms must be NULL (tree-local)");
        G[k] = make_geom(b);
        const int64_t w = int64_t(1) << (LH - l);
        const int64_t sib = tau ^ 1;
        for (int64_t q = 0; q <= w; ++q) {
          require(G[k].rlp[q] == lp[tau * w + q] - lp[tau * w], BF_ERR_SHAPE, "offdiag row leaves differ from T_H");
          require(G[k].clp[q] == lp[sib * w + q] - lp[sib * w], BF_ERR_SHAPE, "offdiag column leaves differ from T_H");
        }
      }
    check_device(device);
    DeviceGuard dg(device);
    std::unique_ptr<hodbf_s> h(new hodbf_s());
    h->dtype = d->dtype;
    h->device = device;
    h->n = d->n;
    h->LH = LH;
    const size_t cs = csize(d->dtype);
    auto bf_of_row_leaf = [&](int l, int64_t t, int64_t* k, int64_t* loc) {  // butterfly whose row tree holds t
      const int64_t sig = t >> (LH - l);
      *k = (int64_t(1) << l) - 2 + sig;
      *loc = t - (sig << (LH - l));
    };
    auto bf_of_col_leaf = [&](int l, int64_t t, int64_t* k, int64_t* loc) {  // column tree holds t
      const int64_t sig = t >> (LH - l);
      *k = (int64_t(1) << l) - 2 + (sig ^ 1);
      *loc = t - (sig << (LH - l));
    };
    // ---- pool layout: per leaf M_t = [D_t | U^(1)_t .. U^(LH)_t], per leaf stacked Vt, then R/B/W per bf
    std::vector<int64_t> M_off(nleaf), SV_off(nleaf), sumr(nleaf, 0), sumc(nleaf, 0);
    int64_t o = 0;
    for (int64_t t = 0; t < nleaf; ++t) {
      const int64_t mt = lp[t + 1] - lp[t];
      for (int l = 1; l <= LH; ++l) {
        int64_t k, loc;
        bf_of_row_leaf(l, t, &k, &loc);
        sumr[t] += G[k].r(G[k].L, loc);
        bf_of_col_leaf(l, t, &k, &loc);
        sumc[t] += G[k].c(0, loc);
      }
      M_off[t] = o;
      o += mt * (mt + sumr[t]);
    }
    for (int64_t t = 0; t < nleaf; ++t) {
      SV_off[t] = o;
      o += sumc[t] * (lp[t + 1] - lp[t]);
    }
    std::vector<FBase> F(nbf);
    int64_t entries = lenD;
    for (int64_t k = 0; k < nbf; ++k) {
      F[k].r = o;
      o += G[k].len_R;
      F[k].b = o;
      o += G[k].len_B;
      F[k].w = o;
      o += G[k].len_W;
      entries += G[k].len_U + G[k].len_R + G[k].len_B + G[k].len_W + G[k].len_Vt;
    }
    const int64_t pool_len = o;
    h->factor_entries = entries;
    std::vector<char> host((size_t)pool_len * cs);
    char* hp = host.data();
    const char* Dsrc = static_cast<const char*>(d->D);
    int64_t doff = 0;
    for (int64_t t = 0; t < nleaf; ++t) {
      const int64_t mt = lp[t + 1] - lp[t];
      char* dst = hp + M_off[t] * cs;
      if (mt) memcpy(dst, Dsrc + doff * cs, (size_t)(mt * mt) * cs);
      doff += mt * mt;
      int64_t col = mt;
      int64_t row = 0;
      for (int l = 1; l <= LH; ++l) {
        int64_t k, loc;
        bf_of_row_leaf(l, t, &k, &loc);
        const int r = G[k].r(G[k].L, loc);
        const char* U = static_cast<const char*>(d->offdiag[k].U) + G[k].u_off[loc] * cs;
        if (mt * r) memcpy(dst + col * mt * cs, U, (size_t)(mt * r) * cs);
        col += r;
        // stacked Vt: rows [row, row + c) of the (sumc x mt) column-major matrix
        bf_of_col_leaf(l, t, &k, &loc);
        const int c = G[k].c(0, loc);
        const char* Vt = static_cast<const char*>(d->offdiag[k].Vt) + G[k].vt_off[loc] * cs;
        char* sv = hp + SV_off[t] * cs;
        for (int64_t j = 0; j < mt; ++j)
          if (c) memcpy(sv + (j * sumc[t] + row) * cs, Vt + j * c * cs, (size_t)c * cs);
        row += c;
      }
    }
    for (int64_t k = 0; k < nbf; ++k) {
      const bf_desc& b = d->offdiag[k];
      if (G[k].len_R) memcpy(hp + F[k].r * cs, b.R, (size_t)G[k].len_R * cs);
      if (G[k].len_B) memcpy(hp + F[k].b * cs, b.B, (size_t)G[k].len_B * cs);
      if (G[k].len_W) memcpy(hp + F[k].w * cs, b.W, (size_t)G[k].len_W * cs);
    }
    if (pool_len) h->pool = upload(hp, (size_t)pool_len * cs, &h->device_bytes);
    h->m3 = !selection_only(hp, pool_len, cs);
    h->lp.assign(lp, lp + nleaf + 1);
    h->inv.resize(d->n);
    for (int64_t p = 0; p < d->n; ++p) h->inv[d->perm ? d->perm[p] : p] = p;
    h->G = G;
    h->F = F;
    h->M_off = M_off;
    h->SV_off = SV_off;
    h->sumc = sumc;
    h->ustart.assign((size_t)nleaf * (LH + 1), 0);
    h->vstart.assign((size_t)nleaf * (LH + 1), 0);
    for (int64_t t = 0; t < nleaf; ++t) {
      int64_t uc = 0, vr = 0;
      for (int l = 1; l <= LH; ++l) {
        h->ustart[(size_t)t * (LH + 1) + l] = uc;
        h->vstart[(size_t)t * (LH + 1) + l] = vr;
        int64_t k, loc;
        bf_of_row_leaf(l, t, &k, &loc);
        uc += G[k].r(G[k].L, loc);
        bf_of_col_leaf(l, t, &k, &loc);
        vr += G[k].c(0, loc);
      }
    }
    if (d->perm) h->d_perm = (int64_t*)upload(d->perm, d->n * 8, &h->device_bytes);
    // ---- slab space: per leaf the z^0 group and the y^L group, then each bf's inner levels
    std::vector<Slabs> S(nbf);
    for (int64_t k = 0; k < nbf; ++k) {
      S[k].col.assign((size_t)(G[k].lc + 1) * G[k].nb, -1);
      S[k].row.assign((size_t)(G[k].L - G[k].lc + 1) * G[k].nb, -1);
    }
    std::vector<int64_t> zgrp(nleaf), ygrp(nleaf);
    int64_t cur = 0;
    for (int64_t t = 0; t < nleaf; ++t) {
      zgrp[t] = cur;
      for (int l = 1; l <= LH; ++l) {
        int64_t k, loc;
        bf_of_col_leaf(l, t, &k, &loc);
        S[k].col[loc] = cur;
        cur += G[k].c(0, loc);
      }
      ygrp[t] = cur;
      for (int l = 1; l <= LH; ++l) {
        int64_t k, loc;
        bf_of_row_leaf(l, t, &k, &loc);
        S[k].row[(size_t)(G[k].L - G[k].lc) * G[k].nb + loc] = cur;
        cur += G[k].r(G[k].L, loc);
      }
    }
    for (int64_t k = 0; k < nbf; ++k) {
      const Geom& g = G[k];
      for (int l = 1; l <= g.lc; ++l)
        for (int64_t i = 0; i < g.nb; ++i) {
          S[k].col[(size_t)l * g.nb + i] = cur;
          cur += g.c(l, i);
        }
      for (int l = g.lc; l < g.L; ++l)
        for (int64_t i = 0; i < g.nb; ++i) {
          S[k].row[(size_t)(l - g.lc) * g.nb + i] = cur;
          cur += g.r(l, i);
        }
    }
    h->slab_rows = cur;
    // ---- plans
    for (int op = 0; op < 2; ++op) {
      PlanBuilder pb;
      for (int64_t t = 0; t < nleaf; ++t) {
        const int64_t mt = lp[t + 1] - lp[t];
        if (op == 0) {
          Term tm = mk(SV_off[t], 1, (int)std::max<int64_t>(sumc[t], 1), mt, lp[t], 1, 0);
          pb.add(0, 0, zgrp[t], sumc[t], &tm, 1);
        } else {
          Term tm = mk(M_off[t] + mt * mt, (int)std::max<int64_t>(mt, 1), 1, mt, lp[t], 1, 1);
          pb.add(0, 0, ygrp[t], sumr[t], &tm, 1);
        }
      }
      for (int64_t k = 0; k < nbf; ++k) {
        EmitOpts eo;
        eo.leaf_in = eo.leaf_out = false;
        if (op == 0)
          emit_N(pb, G[k], F[k], S[k], eo);
        else
          emit_C(pb, G[k], F[k], S[k], eo);
      }
      for (int64_t t = 0; t < nleaf; ++t) {
        const int64_t mt = lp[t + 1] - lp[t];
        Term tm[2];
        if (op == 0) {
          tm[0] = mk(M_off[t], 1, (int)std::max<int64_t>(mt, 1), mt, lp[t], 1, 0);
          tm[1] = mk(M_off[t] + mt * mt, 1, (int)std::max<int64_t>(mt, 1), sumr[t], ygrp[t], 0, 0);
        } else {
          tm[0] = mk(M_off[t], (int)std::max<int64_t>(mt, 1), 1, mt, lp[t], 1, 1);
          tm[1] = mk(SV_off[t], (int)std::max<int64_t>(sumc[t], 1), 1, sumc[t], zgrp[t], 0, 1);
        }
        pb.add(LH + 1, 1, lp[t], mt, tm, 2);
      }
      upload_plan(h->plan[op], pb, 0, (int)pb.tasks.size(), &h->device_bytes);
    }
    *out = h.release();
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  } catch (const std::bad_alloc&) {
    return fail(Err{BF_ERR_OOM, "host allocation failed"});
  }
}

int hodbf_destroy(hodbf_handle h) {
  delete h;
  return BF_OK;
}

int hodbf_info(hodbf_handle h, bf_info_t* info) {
  if (!h || !info) return fail(Err{BF_ERR_ARG, "NULL argument"});
  info->factor_entries = h->factor_entries;
  info->device_bytes = (int64_t)h->device_bytes;
  info->launches_n = h->plan[0].launches();
  info->launches_c = h->plan[1].launches();
  info->rows_in = h->n;
  info->rows_out = h->n;
  return BF_OK;
}

int hodbf_workspace_size(hodbf_handle h, int64_t nrhs, size_t* bytes) {
  if (!h || !bytes || nrhs < 0) return fail(Err{BF_ERR_ARG, "bad argument"});
  *bytes = align256((size_t)h->slab_rows * (size_t)nrhs * csize(h->dtype));
  return BF_OK;
}

int hodbf_rounds(hodbf_handle h, int op, int32_t* n) {
  if (!h || !n) return fail(Err{BF_ERR_ARG, "NULL argument"});
  *n = (int32_t)h->plan[op == BF_OP_N ? 0 : 1].rounds.size();
  return BF_OK;
}

int hodbf_round_info(hodbf_handle h, int op, int32_t round, bf_round_info_t* info) {
  if (!h) return fail(Err{BF_ERR_ARG, "NULL handle"});
  try {
    round_info(h->dtype, h->plan[op == BF_OP_N ? 0 : 1], round, info);
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

int hodbf_apply(hodbf_handle h, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
                void* work, size_t work_bytes, bf_stream_t stream) {
  return hodbf_apply_events(h, op, nrhs, X, ldx, Y, ldy, work, work_bytes, stream, nullptr, 0);
}

int hodbf_apply_events(hodbf_handle h, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
                       void* work, size_t work_bytes, bf_stream_t stream, void* const* events, int32_t nevents) {
  if (!h) return fail(Err{BF_ERR_ARG, "NULL handle"});
  try {
    require(op == BF_OP_N || op == BF_OP_C || op == BF_OP_T, BF_ERR_ARG, "bad op");
    size_t need = 0;
    hodbf_workspace_size(h, nrhs, &need);
    validate_apply(nrhs, X, ldx, h->n, Y, ldy, h->n, work_bytes, need, csize(h->dtype));
    if (nrhs == 0 || h->n == 0) return BF_OK;
    require(nrhs <= (int64_t)65535 * 32, BF_ERR_ARG, "nrhs too large for one launch");
    DeviceGuard dg(h->device);
    StageArgs a{};
    a.pool = h->pool;
    a.m3 = h->m3;
    a.X = X;
    a.ldx = ldx;
    a.xperm = h->d_perm;
    a.S = work;
    a.ldS = nrhs;
    a.Y = Y;
    a.ldy = ldy;
    a.yperm = h->d_perm;
    a.conj_flip = op == BF_OP_T ? 1 : 0;
    a.nrhs = (int32_t)nrhs;
    run_plan(h->dtype, h->plan[op == BF_OP_N ? 0 : 1], a, static_cast<cudaStream_t>(stream), events, nevents);
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

int hodbf_workspace_size_host(hodbf_handle h, int64_t nrhs, size_t* bytes) {
  if (!h || !bytes || nrhs < 0) return fail(Err{BF_ERR_ARG, "bad argument"});
  size_t s = 0;
  hodbf_workspace_size(h, nrhs, &s);
  *bytes = s + 4 * align256((size_t)h->n * nrhs * csize(h->dtype));  // two X / Y sets (HostPipe)
  return BF_OK;
}

int hodbf_apply_host(hodbf_handle h, int op, int64_t nrhs, const void* Xh, int64_t ldx, void* Yh, int64_t ldy,
                     void* work, size_t work_bytes, bf_stream_t stream) {
  if (!h) return fail(Err{BF_ERR_ARG, "NULL handle"});
  try {
    size_t need = 0, s = 0;
    hodbf_workspace_size_host(h, nrhs, &need);
    hodbf_workspace_size(h, nrhs, &s);
    validate_apply(nrhs, Xh, ldx, h->n, Yh, ldy, h->n, work_bytes, need, csize(h->dtype));
    if (nrhs == 0 || h->n == 0) return BF_OK;
    DeviceGuard dg(h->device);
    host_pipeline(h->hp, op, nrhs, Xh, ldx, h->n, Yh, ldy, h->n, work, s, csize(h->dtype),
                  static_cast<cudaStream_t>(stream), [&](void* dX, void* dY, cudaStream_t sc) {
                    return hodbf_apply(h, op, nrhs, dX, h->n, dY, h->n, work, s, sc);
                  });
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

}  // extern "C"

// ======================================================================================
// distributed butterfly: column subtrees -> all-to-all -> row subtrees
// ======================================================================================
namespace bfa {

// Copy the blocks a rank touches into a compact local pool; remap the block offsets of a
// private Geom copy (untouched blocks keep offset -1).
static void local_pool(const bf_desc& d, Geom& G, const Own& own, std::vector<char>& host, FBase& F,
                       size_t cs) {
  const int L = G.L, lc = G.lc;
  auto take = [&](const void* src, int64_t off, int64_t len) {
    const int64_t at = (int64_t)(host.size() / cs);
    host.resize(host.size() + (size_t)len * cs);
    memcpy(host.data() + (size_t)at * cs, static_cast<const char*>(src) + (size_t)off * cs, (size_t)len * cs);
    return at;
  };
  F = FBase{};
  for (int64_t tau = 0; tau < G.nb; ++tau)
    G.u_off[tau] = own.row(L, tau) ? take(d.U, G.u_off[tau], G.mt(tau) * G.r(L, tau)) : -1;
  for (int l = lc; l < L; ++l)
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        const int64_t i = G.idx(l, tau, nu);
        G.r_off[l][i] = own.row(l, tau) ? take(d.R, G.r_off[l][i], int64_t(G.R_rows(l, tau, nu)) * G.r(l, i)) : -1;
      }
  for (int64_t i = 0; i < G.nb; ++i) {
    const int64_t tau = i >> (L - lc), nu = i & ((int64_t(1) << (L - lc)) - 1);
    G.b_off[i] = (own.row(lc, tau) || own.col(G, lc, nu)) ? take(d.B, G.b_off[i], int64_t(G.r(lc, i)) * G.c(lc, i)) : -1;
  }
  for (int l = 1; l <= lc; ++l)
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        const int64_t i = G.idx(l, tau, nu);
        G.w_off[l][i] = own.col(G, l, nu) ? take(d.W, G.w_off[l][i], int64_t(G.c(l, i)) * G.W_cols(l, tau, nu)) : -1;
      }
  for (int64_t nu = 0; nu < G.nb; ++nu)
    G.vt_off[nu] = own.col(G, 0, nu) ? take(d.Vt, G.vt_off[nu], int64_t(G.c(0, nu)) * G.nv(nu)) : -1;
}

// contiguous user range of tree positions [a, b) under perm (NULL = identity)
static int64_t user_range(const int64_t* perm, int64_t a, int64_t b, std::vector<int64_t>& lperm) {
  lperm.resize((size_t)(b - a));
  if (!perm) {
    for (int64_t q = 0; q < b - a; ++q) lperm[q] = q;
    return a;
  }
  int64_t lo = INT64_MAX, hi = -1;
  for (int64_t q = a; q < b; ++q) {
    lo = std::min(lo, perm[q]);
    hi = std::max(hi, perm[q]);
  }
  require(b == a || hi - lo + 1 == b - a, BF_ERR_PERM, "a rank's subtree does not map to a contiguous user range");
  for (int64_t q = a; q < b; ++q) lperm[q - a] = perm[q] - lo;
  return b == a ? 0 : lo;
}

}  // namespace bfa

extern "C" {

int bf_dist_create(const bf_desc* d, int rank, int nranks, int device, bf_handle* out) {
  if (!d || !out) return fail(Err{BF_ERR_ARG, "NULL argument"});
  *out = nullptr;
  try {
    Canon cn_;
    d = &canonical(*d, cn_);
    require(nranks >= 1 && (nranks & (nranks - 1)) == 0, BF_ERR_NCCL, "nranks must be a power of two");
    require(rank >= 0 && rank < nranks, BF_ERR_ARG, "rank out of range");
    Geom G = make_geom(*d);
    int p = 0;
    while ((1 << p) < nranks) ++p;
    require(p <= G.lc && p <= G.L - G.lc, BF_ERR_NCCL, "need log2(nranks) <= min(lc, L - lc)");
    check_perm(d->row_perm, d->m, "row_perm");
    check_perm(d->col_perm, d->n, "col_perm");
    const bool host_only = device < 0;
    struct HostOnly {
      explicit HostOnly(bool on) { g_host_only = on; }
      ~HostOnly() { g_host_only = false; }
    } ho(host_only);
    if (!host_only) check_device(device);
    DeviceGuard dg(host_only ? -1 : device);
    std::unique_ptr<bf_s> h(new bf_s());
    h->dtype = d->dtype;
    h->device = device;
    h->host_only = host_only;
    h->dist = true;
    h->rank = rank;
    h->nranks = nranks;
    const size_t cs = csize(d->dtype);
    Own own;
    own.p = p;
    own.g = rank;
    std::vector<char> host;
    FBase F;
    const Geom G0 = G;  // canonical offsets (local_pool rewrites G's to the rank-local pool)
    local_pool(*d, G, own, host, F, cs);
    h->factor_entries = (int64_t)(host.size() / cs);
    if (!host.empty()) h->pool = upload(host.data(), host.size(), &h->device_bytes);
    // decided on the full factors, so that every rank takes the same path (and slab format)
    h->m3 = !(selection_only(d->U, G0.len_U, cs) && selection_only(d->R, G0.len_R, cs) &&
              selection_only(d->B, G0.len_B, cs) && selection_only(d->W, G0.len_W, cs) &&
              selection_only(d->Vt, G0.len_Vt, cs));
    const int L = G.L, lc = G.lc;
    const int64_t P = nranks, g = rank;
    // local row ranges (tree positions) and local perms
    const int64_t cs0 = G.clp[g << (L - p)], cs1 = G.clp[(g + 1) << (L - p)];
    const int64_t rs0 = G.rlp[g << (L - p)], rs1 = G.rlp[(g + 1) << (L - p)];
    std::vector<int64_t> lpc, lpr;
    const int64_t uc = user_range(d->col_perm, cs0, cs1, lpc);
    const int64_t ur = user_range(d->row_perm, rs0, rs1, lpr);
    int64_t* dpc = lpc.empty() ? nullptr : (int64_t*)upload(lpc.data(), lpc.size() * 8, &h->device_bytes);
    int64_t* dpr = lpr.empty() ? nullptr : (int64_t*)upload(lpr.data(), lpr.size() * 8, &h->device_bytes);
    // op N: in = column subtree, out = row subtree; op C the reverse.  One perm copy each.
    h->d_lperm_in[0] = dpc;   // owned; the op-C entries alias them
    h->d_lperm_out[0] = dpr;
    h->d_lperm_in[1] = dpr;
    h->d_lperm_out[1] = dpc;
    h->loc_rows_in[0] = cs1 - cs0;
    h->loc_rows_out[0] = rs1 - rs0;
    h->loc_user_in[0] = uc;
    h->loc_user_out[0] = ur;
    h->loc_rows_in[1] = rs1 - rs0;
    h->loc_rows_out[1] = cs1 - cs0;
    h->loc_user_in[1] = ur;
    h->loc_user_out[1] = uc;
    int64_t max_rows = 0;
    for (int op = 0; op < 2; ++op) {
      Slabs S;
      S.col.assign((size_t)(lc + 1) * G.nb, -1);
      S.row.assign((size_t)(L - lc + 1) * G.nb, -1);
      S.xspace = op == 0 ? 1 : 2;
      S.xout.assign(G.nb, -1);
      S.xin.assign(G.nb, -1);
      int64_t cur = 0;
      for (int l = 0; l <= lc; ++l) {
        if (op == 1 && l == lc) break;
        for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
          for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu)
            if (own.col(G, l, nu)) {
              const int64_t i = G.idx(l, tau, nu);
              S.col[(size_t)l * G.nb + i] = cur;
              cur += G.c(l, i);
            }
      }
      for (int l = lc; l <= L; ++l) {
        if (op == 0 && l == lc) continue;
        for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
          if (own.row(l, tau))
            for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
              const int64_t i = G.idx(l, tau, nu);
              S.row[(size_t)(l - lc) * G.nb + i] = cur;
              cur += G.r(l, i);
            }
      }
      // exchange regions at the centre level: sender groups by destination, receiver by source
      const int64_t wt = int64_t(1) << (lc - p), wn = int64_t(1) << (L - lc - p);
      auto sz = [&](int64_t i) { return op == 0 ? G.r(lc, i) : G.c(lc, i); };
      h->send_base[op] = cur;
      h->send_cnt[op].assign(P, 0);
      h->recv_cnt[op].assign(P, 0);
      for (int64_t q = 0; q < P; ++q) {
        // op N: sender owns nu (col subtree g), destination q owns tau
        // op C: sender owns tau (row subtree g), destination q owns nu
        const int64_t t0 = (op == 0 ? q : g) * wt, n0 = (op == 0 ? g : q) * wn;
        for (int64_t tau = t0; tau < t0 + wt; ++tau)
          for (int64_t nu = n0; nu < n0 + wn; ++nu) {
            const int64_t i = G.idx(lc, tau, nu);
            S.xout[i] = cur;
            cur += sz(i);
            h->send_cnt[op][q] += sz(i);
            h->send_blk[op].push_back(i);
          }
      }
      h->send_rows[op] = cur - h->send_base[op];
      h->recv_base[op] = cur;
      for (int64_t q = 0; q < P; ++q) {
        const int64_t t0 = (op == 0 ? g : q) * wt, n0 = (op == 0 ? q : g) * wn;
        for (int64_t tau = t0; tau < t0 + wt; ++tau)
          for (int64_t nu = n0; nu < n0 + wn; ++nu) {
            const int64_t i = G.idx(lc, tau, nu);
            S.xin[i] = cur;
            cur += sz(i);
            h->recv_cnt[op][q] += sz(i);
            h->recv_blk[op].push_back(i);
          }
      }
      h->recv_rows[op] = cur - h->recv_base[op];
      max_rows = std::max(max_rows, cur);
      PlanBuilder pb;
      EmitOpts o;
      o.own = own;
      if (op == 0) {
        o.x_base = cs0;
        o.y_base = rs0;
        emit_N(pb, G, F, S, o);
        upload_plan(h->pre[0], pb, 0, lc + 2, &h->device_bytes);
        upload_plan(h->post[0], pb, lc + 2, L + 3, &h->device_bytes);
      } else {
        o.x_base = rs0;
        o.y_base = cs0;
        emit_C(pb, G, F, S, o);
        upload_plan(h->pre[1], pb, 0, L - lc + 2, &h->device_bytes);
        upload_plan(h->post[1], pb, L - lc + 2, L + 3, &h->device_bytes);
      }
    }
    h->slab_rows = max_rows;
    // fused fast path for uniform rank-16 butterflies: the same split with the window-pass and
    // leaf kernels; the generic plans above remain the fallback
    if (fast_eligible(G0, d->dtype) && G0.lc >= 1 && G0.L - G0.lc >= 1 && h->m3 && !getenv("BF_DISABLE_FAST")) {
      auto build = [&](auto* tag) {
        using CT = std::remove_pointer_t<decltype(tag)>;
        HostFactors<CT> HF{static_cast<const CT*>(d->U), static_cast<const CT*>(d->R), static_cast<const CT*>(d->B),
                           static_cast<const CT*>(d->W), static_cast<const CT*>(d->Vt)};
        for (int k = 0; k < 2; ++k) build_fast(h->fast[k], G0, HF, k, &h->device_bytes, p, rank);
      };
      if (d->dtype == BF_C128) build((double2*)nullptr);
      else build((float2*)nullptr);
      const bool ok = true;
      if (ok) {
        h->use_fast = true;
        h->fast[0].contig_in = leaves_contiguous(lpc.empty() ? nullptr : lpc.data(), cs1 - cs0, G0.nv(0));
        h->fast[0].contig_out = leaves_contiguous(lpr.empty() ? nullptr : lpr.data(), rs1 - rs0, G0.mt(0));
        h->fast[1].contig_in = h->fast[0].contig_out;
        h->fast[1].contig_out = h->fast[0].contig_in;
      } else {
        for (int k = 0; k < 2; ++k) {
          if (h->fast[k].F) cudaFree(h->fast[k].F);
          h->fast[k] = FastPlan{};
        }
      }
    }
    h->G = std::move(G);
    *out = h.release();
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  } catch (const std::bad_alloc&) {
    return fail(Err{BF_ERR_OOM, "host allocation failed"});
  }
}

int bf_dist_layout(bf_handle h, int op, int64_t nrhs, size_t* work_bytes, size_t* send_off, size_t* recv_off,
                   int64_t* send_counts, int64_t* recv_counts) {
  if (!h || nrhs < 0) return fail(Err{BF_ERR_ARG, "bad argument"});
  if (!h->dist) return fail(Err{BF_ERR_ARG, "not a distributed handle"});
  const int k = op == BF_OP_N ? 0 : 1;
  if (h->use_fast) {
    // fast format: per peer [tile][half][block][16 x 16] (bf_dist_slab_format), equal chunks
    const size_t xb = fast_x_bytes(h, nrhs), bb = fast_buf_bytes(h, nrhs);
    const int64_t per = (int64_t)((nrhs + FAST_NB - 1) / FAST_NB) * (h->G.nb / ((int64_t)h->nranks * h->nranks)) *
                        FAST_SLAB;
    if (work_bytes) *work_bytes = 2 * bb + 2 * xb;
    if (send_off) *send_off = 2 * bb;
    if (recv_off) *recv_off = 2 * bb + xb;
    for (int q = 0; q < h->nranks; ++q) {
      if (send_counts) send_counts[q] = per;
      if (recv_counts) recv_counts[q] = per;
    }
    return BF_OK;
  }
  const size_t row_bytes = (size_t)nrhs * csize(h->dtype);
  if (work_bytes) *work_bytes = align256((size_t)h->slab_rows * row_bytes);
  if (send_off) *send_off = (size_t)h->send_base[k] * row_bytes;
  if (recv_off) *recv_off = (size_t)h->recv_base[k] * row_bytes;
  for (int q = 0; q < h->nranks; ++q) {
    if (send_counts) send_counts[q] = h->send_cnt[k][q] * nrhs;
    if (recv_counts) recv_counts[q] = h->recv_cnt[k][q] * nrhs;
  }
  return BF_OK;
}

int bf_dist_exchange_blocks(bf_handle h, int op, int64_t* n_send, int64_t* send_blocks, int64_t* n_recv,
                            int64_t* recv_blocks) {
  if (!h) return fail(Err{BF_ERR_ARG, "NULL handle"});
  if (!h->dist) return fail(Err{BF_ERR_ARG, "not a distributed handle"});
  const int k = op == BF_OP_N ? 0 : 1;
  if (n_send) *n_send = (int64_t)h->send_blk[k].size();
  if (n_recv) *n_recv = (int64_t)h->recv_blk[k].size();
  if (h->use_fast) {
    // fast format: the blocks of the exchange level lx, per peer tau-major (op N) / nu-major (op C)
    const Geom& G = h->G;
    const int lx = h->fast[k].lx;
    int p = 0;
    while ((1 << p) < h->nranks) ++p;
    const int64_t wt = int64_t(1) << (lx - p), wn = int64_t(1) << (G.L - lx - p), g = h->rank;
    const int64_t nblk = (int64_t)h->nranks * wt * wn;
    if (n_send) *n_send = nblk;
    if (n_recv) *n_recv = nblk;
    int64_t is = 0, ir = 0;
    if (k == 0) {
      for (int64_t q = 0; q < h->nranks; ++q)
        for (int64_t i = 0; i < wt; ++i)
          for (int64_t j = 0; j < wn; ++j) {
            if (send_blocks) send_blocks[is++] = G.idx(lx, q * wt + i, g * wn + j);  // sender owns nu
            if (recv_blocks) recv_blocks[ir++] = G.idx(lx, g * wt + i, q * wn + j);  // receiver owns tau
          }
    } else {
      for (int64_t q = 0; q < h->nranks; ++q)
        for (int64_t j = 0; j < wn; ++j)
          for (int64_t i = 0; i < wt; ++i) {
            if (send_blocks) send_blocks[is++] = G.idx(lx, g * wt + i, q * wn + j);  // sender owns tau
            if (recv_blocks) recv_blocks[ir++] = G.idx(lx, q * wt + i, g * wn + j);  // receiver owns nu
          }
    }
    return BF_OK;
  }
  if (send_blocks) std::copy(h->send_blk[k].begin(), h->send_blk[k].end(), send_blocks);
  if (recv_blocks) std::copy(h->recv_blk[k].begin(), h->recv_blk[k].end(), recv_blocks);
  return BF_OK;
}

int bf_dist_exchange_level(bf_handle h, int op, int32_t* level) {
  if (!h || !level) return fail(Err{BF_ERR_ARG, "NULL argument"});
  if (!h->dist) return fail(Err{BF_ERR_ARG, "not a distributed handle"});
  *level = h->use_fast ? h->fast[op == BF_OP_N ? 0 : 1].lx : h->G.lc;
  return BF_OK;
}

int bf_dist_slab_format(bf_handle h, int32_t* fmt) {
  if (!h || !fmt) return fail(Err{BF_ERR_ARG, "NULL argument"});
  if (!h->dist) return fail(Err{BF_ERR_ARG, "not a distributed handle"});
  *fmt = h->use_fast ? 1 : 0;
  return BF_OK;
}

int bf_dist_local_rows(bf_handle h, int op, int64_t* rows_in, int64_t* rows_out, int64_t* user_off_in,
                       int64_t* user_off_out) {
  if (!h) return fail(Err{BF_ERR_ARG, "NULL handle"});
  if (!h->dist) return fail(Err{BF_ERR_ARG, "not a distributed handle"});
  const int k = op == BF_OP_N ? 0 : 1;
  if (rows_in) *rows_in = h->loc_rows_in[k];
  if (rows_out) *rows_out = h->loc_rows_out[k];
  if (user_off_in) *user_off_in = h->loc_user_in[k];
  if (user_off_out) *user_off_out = h->loc_user_out[k];
  return BF_OK;
}

static int dist_run(bf_handle h, int op, int64_t nrhs, const void* X, int64_t ldx, void* Y, int64_t ldy,
                    void* work, size_t work_bytes, bf_stream_t stream, bool pre,
                    void* const* peer_recv = nullptr) {
  if (!h) return fail(Err{BF_ERR_ARG, "NULL handle"});
  try {
    require(h->dist, BF_ERR_ARG, "not a distributed handle");
    require(!h->host_only, BF_ERR_DEVICE, "host-only plan (created with device < 0) cannot apply");
    require(op == BF_OP_N || op == BF_OP_C || op == BF_OP_T, BF_ERR_ARG, "bad op");
    require(nrhs >= 0 && nrhs <= (int64_t)65535 * 32, BF_ERR_ARG, "bad nrhs");
    const int k = op == BF_OP_N ? 0 : 1;
    size_t need = 0;
    bf_dist_layout(h, op, nrhs, &need, nullptr, nullptr, nullptr, nullptr);
    require(work_bytes >= need && (need == 0 || work), BF_ERR_ARG, "workspace too small");
    if (nrhs == 0) return BF_OK;
    if (pre)
      require(X && ldx >= std::max<int64_t>(h->loc_rows_in[k], 1), BF_ERR_ARG, "bad X_loc / ldx");
    else
      require(Y && ldy >= std::max<int64_t>(h->loc_rows_out[k], 1), BF_ERR_ARG, "bad Y_loc / ldy");
    DeviceGuard dg(h->device);
    if (h->use_fast) {
      const FastPlan& FP = h->fast[k];
      if (pre)
        run_fast(h, k, op, nrhs, X, ldx, nullptr, 0, work, static_cast<cudaStream_t>(stream), nullptr, 0, 0, FP.split,
                 peer_recv);
      else
        run_fast(h, k, op, nrhs, nullptr, 0, Y, ldy, work, static_cast<cudaStream_t>(stream), nullptr, 0, FP.split);
      return BF_OK;
    }
    StageArgs a{};
    a.pool = h->pool;
    a.m3 = h->m3;
    a.X = X;
    a.ldx = ldx;
    a.xperm = h->d_lperm_in[k];
    a.S = work;
    a.ldS = nrhs;
    a.Y = Y;
    a.ldy = ldy;
    a.yperm = h->d_lperm_out[k];
    a.conj_flip = op == BF_OP_T ? 1 : 0;
    a.nrhs = (int32_t)nrhs;
    run_plan(h->dtype, pre ? h->pre[k] : h->post[k], a, static_cast<cudaStream_t>(stream));
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

int bf_dist_apply_pre(bf_handle h, int op, int64_t nrhs, const void* X_loc, int64_t ldx, void* work,
                      size_t work_bytes, bf_stream_t stream) {
  return dist_run(h, op, nrhs, X_loc, ldx, nullptr, 0, work, work_bytes, stream, true);
}

int bf_dist_apply_pre_p2p(bf_handle h, int op, int64_t nrhs, const void* X_loc, int64_t ldx, void* work,
                          size_t work_bytes, void* const* peer_recv, bf_stream_t stream) {
  if (!h || !peer_recv) return fail(Err{BF_ERR_ARG, "NULL argument"});
  if (!h->use_fast || h->nranks > FAST_MAXPEER)
    return fail(Err{BF_ERR_ARG, "peer-memory exchange needs the fused split (bf_dist_slab_format 1, <= 8 ranks)"});
  return dist_run(h, op, nrhs, X_loc, ldx, nullptr, 0, work, work_bytes, stream, true, peer_recv);
}

int bf_dist_apply_post(bf_handle h, int op, int64_t nrhs, void* Y_loc, int64_t ldy, void* work, size_t work_bytes,
                       bf_stream_t stream) {
  return dist_run(h, op, nrhs, nullptr, 0, Y_loc, ldy, work, work_bytes, stream, false);
}

}  // extern "C"

namespace bfa {

// One butterfly's sub-matrix request: the requested rows / columns as tree positions of that
// butterfly, where their U rows / Vt columns live in the pool, and where they go in `out`.
struct XQuery {
  std::vector<int64_t> pr, pc;      // tree positions (butterfly-local)
  std::vector<int64_t> vtoff;       // per column: pool offset of its Vt column (c contiguous entries)
  std::vector<int64_t> uoff, ustr;  // per row: pool offset of its U row, the row's stride
  std::vector<int64_t> orow, ocol;  // output row / column of each request
};

static int64_t leaf_of(const std::vector<int64_t>& lp, int64_t p) {
  return (int64_t)(std::upper_bound(lp.begin(), lp.end(), p) - lp.begin()) - 1;
}

// One butterfly's share of an extraction (its geometry in the pool, its requests).
struct XPart {
  const Geom* G;
  FBase F;
  XQuery q;
  void* out = nullptr;  // bf_extract_list: this part's own output block (nullptr: the call's)
  int64_t ldo = 0;
};

// Compact extraction (Alg. 3 extract_BF: "each block is multiplied only once",
// P:524-526): every touched block (l, tau, nu) holds a slab of rank x w_nu, w_nu = the number of
// requested columns under nu (T_S level L - l; the columns are put in tree order, so they form one
// contiguous range per node).  A W / R stage block then splits into one product per touched child
// (each child's columns are a sub-range of the parent's), so no block is ever multiplied at a
// column it does not need and no slab space is zero-filled.  One launch of k_xprod per stage for
// all parts (the parts never interact), the level-0 Vt columns gathered, the U rows times y^L
// into a compact nI x nJ block per part, scattered to `out`.  Synchronous on `st`.
static void extract_compact(int dtype, const void* pool, std::vector<XPart>& parts, void* out, int64_t ldo,
                            cudaStream_t st, XScratch& xs) {
  const size_t cs = csize(dtype);
  static const bool timing = getenv("BF_EXTRACT_TIMING") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  int Lmax = 0;
  for (XPart& pt : parts) Lmax = std::max(Lmax, pt.G->L);
  // stages: 0 = level-0 gather (separate), 1..: products by level of the recursion
  std::vector<std::vector<XProd>> stage((size_t)2 * Lmax + 4);
  std::vector<int64_t> vtg;                       // k_xgather_vt entries
  std::vector<int64_t> sc_orow, sc_ocol;          // per part: result scatter maps
  struct PartOut { int64_t toff, nI, nJ, orow0, ocol0; void* out; int64_t ldo; };
  std::vector<PartOut> pouts;
  int64_t slab = 0;  // compact slab elements (all parts)
  for (XPart& pt : parts) {
    const Geom& G = *pt.G;
    const int L = G.L, lc = G.lc;
    XQuery& q = pt.q;
    const int64_t nI = (int64_t)q.pr.size(), nJ = (int64_t)q.pc.size();
    if (nI == 0 || nJ == 0) continue;
    {  // the part's columns in tree order
      std::vector<int64_t> ord(nJ);
      for (int64_t j = 0; j < nJ; ++j) ord[j] = j;
      std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return q.pc[x] < q.pc[y]; });
      XQuery s2 = q;
      for (int64_t j = 0; j < nJ; ++j) {
        q.pc[j] = s2.pc[ord[j]];
        q.vtoff[j] = s2.vtoff[ord[j]];
        q.ocol[j] = s2.ocol[ord[j]];
      }
    }
    std::vector<int64_t> tj(nJ), ti(nI);
    for (int64_t j = 0; j < nJ; ++j) tj[j] = leaf_of(G.clp, q.pc[j]);
    for (int64_t i = 0; i < nI; ++i) ti[i] = leaf_of(G.rlp, q.pr[i]);
    // column ranges: lo[l][nu], w[l][nu] for nu at T_S level L - l (node of leaf t: t >> l)
    std::vector<std::vector<int32_t>> lo(L + 1), wd(L + 1);
    for (int l = 0; l <= L; ++l) {
      lo[l].assign((size_t)1 << (L - l), 0);
      wd[l].assign((size_t)1 << (L - l), 0);
      for (int64_t j = 0; j < nJ; ++j) {
        const int64_t nu = tj[j] >> l;
        if (wd[l][nu] == 0) lo[l][nu] = (int32_t)j;
        wd[l][nu]++;
      }
    }
    // touched tau per T_O level l (ascending lists)
    std::vector<std::vector<int64_t>> taus(L + 1);
    for (int l = 0; l <= L; ++l) {
      std::vector<char> f((size_t)1 << l, 0);
      for (int64_t i = 0; i < nI; ++i) f[ti[i] >> (L - l)] = 1;
      for (size_t t = 0; t < f.size(); ++t)
        if (f[t]) taus[l].push_back((int64_t)t);
    }
    // touched nu per level (ascending)
    std::vector<std::vector<int64_t>> nus(L + 1);
    for (int l = 0; l <= L; ++l)
      for (size_t v = 0; v < wd[l].size(); ++v)
        if (wd[l][v]) nus[l].push_back((int64_t)v);
    // slab offsets: column side z (l = 0..lc), row side y (l = lc..L), flat over the touched
    // (tau, nu) pairs of a level: slot = pos(tau) * |nus[l]| + pos(nu)
    std::vector<std::vector<int32_t>> tpos(L + 1), npos(L + 1);
    for (int l = 0; l <= L; ++l) {
      tpos[l].assign((size_t)1 << l, -1);
      npos[l].assign((size_t)1 << (L - l), -1);
      for (size_t k = 0; k < taus[l].size(); ++k) tpos[l][taus[l][k]] = (int32_t)k;
      for (size_t k = 0; k < nus[l].size(); ++k) npos[l][nus[l][k]] = (int32_t)k;
    }
    std::vector<std::vector<int64_t>> zo(lc + 1), yo(L - lc + 1);
    for (int l = 0; l <= lc; ++l) {
      const int64_t nt = l == 0 ? 1 : (int64_t)taus[l].size(), nn = (int64_t)nus[l].size();
      zo[l].assign((size_t)(nt * nn), -1);
      for (int64_t pt2 = 0; pt2 < nt; ++pt2) {
        const int64_t tau = l == 0 ? 0 : taus[l][pt2];
        for (int64_t pn = 0; pn < nn; ++pn) {
          const int64_t nu = nus[l][pn];
          zo[l][pt2 * nn + pn] = slab;
          slab += (int64_t)G.c(l, G.idx(l, tau, nu)) * wd[l][nu];
        }
      }
    }
    for (int l = lc; l <= L; ++l) {
      const int64_t nt = (int64_t)taus[l].size(), nn = (int64_t)nus[l].size();
      yo[l - lc].assign((size_t)(nt * nn), -1);
      for (int64_t pt2 = 0; pt2 < nt; ++pt2)
        for (int64_t pn = 0; pn < nn; ++pn) {
          const int64_t tau = taus[l][pt2], nu = nus[l][pn];
          yo[l - lc][pt2 * nn + pn] = slab;
          slab += (int64_t)G.r(l, G.idx(l, tau, nu)) * wd[l][nu];
        }
    }
    auto ZO = [&](int l, int64_t tau, int64_t nu) {
      return zo[l][(int64_t)(l == 0 ? 0 : tpos[l][tau]) * (int64_t)nus[l].size() + npos[l][nu]];
    };
    auto YO = [&](int l, int64_t tau, int64_t nu) {
      return yo[l - lc][(int64_t)tpos[l][tau] * (int64_t)nus[l].size() + npos[l][nu]];
    };
    // level 0: z^0_nu = Vt_nu(:, requested columns)
    for (int64_t j = 0; j < nJ; ++j) {
      const int64_t nu = tj[j];
      vtg.push_back(ZO(0, 0, nu) + (j - lo[0][nu]));
      vtg.push_back(wd[0][nu]);
      vtg.push_back(G.c(0, nu));
      vtg.push_back(q.vtoff[j]);
    }
    // W stages l = 1..lc: z^l_{tau,nu}(:, child s's columns) = W_{tau,nu}(:, child s block) z^{l-1}_{tau>>1, 2nu+s}
    for (int l = 1; l <= lc; ++l)
      for (int64_t tau : taus[l])
        for (int64_t nu : nus[l]) {
          const int64_t i = G.idx(l, tau, nu);
          const int c = G.c(l, i);
          if (c == 0) continue;
          const int64_t ip = (l - 1 == 0) ? 0 : (tau >> 1);
          int32_t coff = 0;
          int cprev = 0;
          for (int s2 = 0; s2 < 2; ++s2) {
            const int64_t ch = 2 * nu + s2;
            const int64_t ic = G.idx(l - 1, ip, ch);
            const int cc = G.c(l - 1, ic);
            const int32_t w = wd[l - 1][ch];
            if (w > 0) {
              XProd x{};
              x.a_off = pt.F.w + G.w_off[l][i] + (int64_t)cprev * c;
              x.a_rs = 1;
              x.a_cs = c;
              x.m = c;
              x.kk = cc;
              x.w = w;
              x.in_off = ZO(l - 1, ip, ch);
              x.in_ld = w;
              x.out_off = ZO(l, tau, nu) + coff;
              x.out_ld = wd[l][nu];
              stage[l].push_back(x);
            }
            coff += w;
            cprev += cc;
          }
        }
    // centre: y^lc = B z^lc
    for (int64_t tau : taus[lc])
      for (int64_t nu : nus[lc]) {
        const int64_t i = G.idx(lc, tau, nu);
        const int r = G.r(lc, i), c = G.c(lc, i);
        if (r == 0) continue;
        XProd x{};
        x.a_off = pt.F.b + G.b_off[i];
        x.a_rs = 1;
        x.a_cs = r;
        x.m = r;
        x.kk = c;
        x.w = wd[lc][nu];
        x.in_off = ZO(lc, lc == 0 ? 0 : tau, nu);
        x.in_ld = wd[lc][nu];
        x.out_off = YO(lc, tau, nu);
        x.out_ld = wd[lc][nu];
        stage[lc + 1].push_back(x);
      }
    // R stages l -> l+1 (gather form): y^{l+1}_{tp,np}(:, child s's columns) =
    //   R_{tp>>1, 2np+s}(rows of child tp & 1) y^l_{tp>>1, 2np+s}
    for (int l = lc; l < L; ++l)
      for (int64_t tp : taus[l + 1])
        for (int64_t np : nus[l + 1]) {
          const int64_t io = G.idx(l + 1, tp, np);
          const int ro = G.r(l + 1, io);
          if (ro == 0) continue;
          const int64_t a = tp >> 1;
          const int part = (int)(tp & 1);
          const int rt = G.r(l + 1, G.idx(l + 1, 2 * a, np)), rb = G.r(l + 1, G.idx(l + 1, 2 * a + 1, np));
          int32_t coff = 0;
          for (int s2 = 0; s2 < 2; ++s2) {
            const int64_t ch = 2 * np + s2;
            const int32_t w = wd[l][ch];
            if (w > 0) {
              const int64_t i = G.idx(l, a, ch);
              XProd x{};
              x.a_off = pt.F.r + G.r_off[l][i] + (part ? rt : 0);
              x.a_rs = 1;
              x.a_cs = rt + rb;
              x.m = ro;
              x.kk = G.r(l, i);
              x.w = w;
              x.in_off = YO(l, a, ch);
              x.in_ld = w;
              x.out_off = YO(l + 1, tp, np) + coff;
              x.out_ld = wd[l + 1][np];
              stage[l + 2].push_back(x);
            }
            coff += w;
          }
        }
    // U rows: T(i, :) = U_tau(row, :) y^L_tau, into the part's compact nI x nJ block
    PartOut po{0, nI, nJ, (int64_t)sc_orow.size(), (int64_t)sc_ocol.size(), pt.out ? pt.out : out,
               pt.out ? pt.ldo : ldo};
    po.toff = slab;
    slab += nI * nJ;
    for (int64_t i = 0; i < nI; ++i) {
      const int64_t tau = ti[i];
      XProd x{};
      x.a_off = q.uoff[i];
      x.a_rs = 1;
      x.a_cs = (int32_t)q.ustr[i];
      x.m = 1;
      x.kk = G.r(L, tau);
      x.w = (int32_t)nJ;
      x.in_off = YO(L, tau, 0);
      x.in_ld = (int32_t)nJ;
      x.out_off = po.toff + i * nJ;
      x.out_ld = (int32_t)nJ;
      stage[L + 2].push_back(x);
    }
    for (int64_t i = 0; i < nI; ++i) sc_orow.push_back(q.orow[i]);
    for (int64_t j = 0; j < nJ; ++j) sc_ocol.push_back(q.ocol[j]);
    pouts.push_back(po);
  }
  if (pouts.empty()) return;
  // upload: [slab | products | vt gather | scatter maps]
  // products of more than 128 outputs are cut into pieces of at most 128 (one warp each, <= 4
  // outputs per lane): 32-column chunks of max(1, 128 / w) rows -- the lanes of a wide chunk share
  // the factor row and read consecutive input columns; big blocks (wide queries, HOD-BF top
  // levels) spread over many warps while the many small scattered-query products stay whole
  constexpr int64_t XP_MAX = 128;
  for (auto& sv : stage) {
    bool big = false;
    for (const XProd& x : sv) big |= (int64_t)x.m * x.w > XP_MAX;
    if (!big) continue;
    std::vector<XProd> nv;
    nv.reserve(sv.size() + sv.size() / 2);
    for (const XProd& x : sv) {
      if ((int64_t)x.m * x.w <= XP_MAX) {
        nv.push_back(x);
        continue;
      }
      for (int32_t j0 = 0; j0 < x.w; j0 += 32) {
        const int32_t w = std::min<int32_t>(32, x.w - j0);
        const int32_t rp = std::max<int32_t>(1, (int32_t)(XP_MAX / w));
        for (int32_t i0 = 0; i0 < x.m; i0 += rp) {
          XProd y = x;
          y.w = w;
          y.m = std::min<int32_t>(rp, x.m - i0);
          y.a_off += (int64_t)i0 * x.a_rs;
          y.in_off += j0;
          y.out_off += j0 + (int64_t)i0 * x.out_ld;
          nv.push_back(y);
        }
      }
    }
    sv.swap(nv);
  }
  std::vector<int64_t> soff(stage.size() + 1, 0);
  for (size_t k = 0; k < stage.size(); ++k) soff[k + 1] = soff[k] + (int64_t)stage[k].size();
  std::vector<XProd> allp((size_t)soff.back());
  for (size_t k = 0; k < stage.size(); ++k)
    if (!stage[k].empty()) std::copy(stage[k].begin(), stage[k].end(), allp.begin() + soff[k]);
  const size_t bS = align256((size_t)slab * cs), bP = align256(allp.size() * sizeof(XProd)),
               bV = align256(vtg.size() * 8), bR = align256(sc_orow.size() * 8), bC = align256(sc_ocol.size() * 8);
  std::lock_guard<std::mutex> lk(xs.mu);
  char* base = static_cast<char*>(xs.get(bS + bP + bV + bR + bC));
  void* dS = base;
  XProd* dP = reinterpret_cast<XProd*>(base + bS);
  int64_t* dV = reinterpret_cast<int64_t*>(base + bS + bP);
  int64_t* dR = reinterpret_cast<int64_t*>(base + bS + bP + bV);
  int64_t* dC = reinterpret_cast<int64_t*>(base + bS + bP + bV + bR);
  if (!allp.empty()) BF_CK(cudaMemcpyAsync(dP, allp.data(), allp.size() * sizeof(XProd), cudaMemcpyHostToDevice, st));
  BF_CK(cudaMemcpyAsync(dV, vtg.data(), vtg.size() * 8, cudaMemcpyHostToDevice, st));
  BF_CK(cudaMemcpyAsync(dR, sc_orow.data(), sc_orow.size() * 8, cudaMemcpyHostToDevice, st));
  BF_CK(cudaMemcpyAsync(dC, sc_ocol.data(), sc_ocol.size() * 8, cudaMemcpyHostToDevice, st));
  const auto t1 = std::chrono::steady_clock::now();
  launch_xgather_vt(dtype, (int64_t)vtg.size() / 4, dV, pool, dS, st);
  for (size_t k = 0; k < stage.size(); ++k)
    launch_xprod(dtype, soff[k + 1] - soff[k], dP + soff[k], pool, dS, dS, st);
  for (const PartOut& po : pouts)
    launch_xscatter(dtype, po.nI, po.nJ, dR + po.orow0, dC + po.ocol0, static_cast<char*>(dS) + (size_t)po.toff * cs,
                    po.out, po.ldo, st);
  BF_CK(cudaGetLastError());
  BF_CK(cudaStreamSynchronize(st));
  if (timing) {
    const auto t2 = std::chrono::steady_clock::now();
    fprintf(stderr, "bf_extract (compact): plan %.3f ms, upload + device %.3f ms, %zu products, %lld slab entries\n",
            std::chrono::duration<double, std::milli>(t1 - t0).count(),
            std::chrono::duration<double, std::milli>(t2 - t1).count(), allp.size(), (long long)slab);
  }
}

// The device geometry tables of G (cached in xs; caller holds xs.mu).
static const XGeomDev& xgeom_dev(XScratch& xs, const Geom& G) {
  auto it = xs.geo.find(&G);
  if (it != xs.geo.end()) return it->second;
  const int L = G.L, lc = G.lc;
  const int64_t nb = G.nb;
  std::vector<int64_t> roff((size_t)std::max<int64_t>(1, (L - lc) * nb), 0), woff((size_t)std::max<int64_t>(1, lc * nb), 0);
  for (int l = lc; l < L; ++l) std::copy(G.r_off[l].begin(), G.r_off[l].begin() + nb, roff.begin() + (l - lc) * nb);
  for (int l = 1; l <= lc; ++l) std::copy(G.w_off[l].begin(), G.w_off[l].begin() + nb, woff.begin() + (l - 1) * nb);
  const size_t brr = align256(G.rr.size() * 4), brc = align256(G.rc.size() * 4), bro = align256(roff.size() * 8),
               bwo = align256(woff.size() * 8), bbo = align256(std::max<size_t>(1, G.b_off.size()) * 8);
  XGeomDev d;
  BF_CK(cudaMalloc(&d.buf, brr + brc + bro + bwo + bbo));
  char* b = static_cast<char*>(d.buf);
  BF_CK(cudaMemcpy(b, G.rr.data(), G.rr.size() * 4, cudaMemcpyHostToDevice));
  BF_CK(cudaMemcpy(b + brr, G.rc.data(), G.rc.size() * 4, cudaMemcpyHostToDevice));
  BF_CK(cudaMemcpy(b + brr + brc, roff.data(), roff.size() * 8, cudaMemcpyHostToDevice));
  BF_CK(cudaMemcpy(b + brr + brc + bro, woff.data(), woff.size() * 8, cudaMemcpyHostToDevice));
  if (!G.b_off.empty()) BF_CK(cudaMemcpy(b + brr + brc + bro + bwo, G.b_off.data(), G.b_off.size() * 8, cudaMemcpyHostToDevice));
  d.rr = reinterpret_cast<const int32_t*>(b);
  d.rc = reinterpret_cast<const int32_t*>(b + brr);
  d.roff = reinterpret_cast<const int64_t*>(b + brr + brc);
  d.woff = reinterpret_cast<const int64_t*>(b + brr + brc + bro);
  d.boff = reinterpret_cast<const int64_t*>(b + brr + brc + bro + bwo);
  d.Rz.assign(lc + 1, 0);
  d.Ry.assign(L - lc + 1, 0);
  for (int l = 0; l <= lc; ++l)
    for (int64_t i = 0; i < nb; ++i) d.Rz[l] = std::max<int64_t>(d.Rz[l], G.c(l, i));
  for (int l = lc; l <= L; ++l)
    for (int64_t i = 0; i < nb; ++i) d.Ry[l - lc] = std::max<int64_t>(d.Ry[l - lc], G.r(l, i));
  for (auto& v : d.Rz) v = std::max<int64_t>(v, 1);
  for (auto& v : d.Ry) v = std::max<int64_t>(v, 1);
  return xs.geo.emplace(&G, std::move(d)).first->second;
}

// Level-wise extraction (Alg. 3 extract_BF: only the blocks (l, tau, nu) with tau an
// ancestor of a requested row's leaf and nu one of a requested column's leaf, each block multiplied
// only at the request columns under it).  The host work per part is O((|I| + |J|) L):
// the touched T_O nodes per level and a few index arrays; the products themselves are enumerated
// on the device (k_xlevel: one launch per stage for all parts, one thread per output element of
// the level's [touched tau][rank row][request column] slab).  Synchronous on `st`.
static void extract_levels(int dtype, const void* pool, std::vector<XPart>& parts, void* out, int64_t ldo,
                           cudaStream_t st, XScratch& xs) {
  const size_t cs = csize(dtype);
  static const bool timing = getenv("BF_EXTRACT_TIMING") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  std::lock_guard<std::mutex> lk(xs.mu);
  std::vector<XLPart> P;
  std::vector<int64_t> blob;
  std::vector<std::vector<int64_t>> work;  // per part: output elements per stage
  int smax = 0;
  int64_t slab = 0;
  for (XPart& pt : parts) {
    const Geom& G = *pt.G;
    const XQuery& q = pt.q;
    const int L = G.L, lc = G.lc;
    const int64_t nI = (int64_t)q.pr.size(), nJ = (int64_t)q.pc.size();
    if (nI == 0 || nJ == 0) continue;
    const XGeomDev& D = xgeom_dev(xs, G);
    XLPart x{};
    x.rr = D.rr;
    x.rc = D.rc;
    x.roff = D.roff;
    x.woff = D.woff;
    x.boff = D.boff;
    x.fr = pt.F.r;
    x.fb = pt.F.b;
    x.fw = pt.F.w;
    x.L = L;
    x.lc = lc;
    x.nI = (int32_t)nI;
    x.nJ = (int32_t)nJ;
    x.out = pt.out ? pt.out : out;
    x.ldo = pt.out ? pt.ldo : ldo;
    auto put = [&](int64_t& off, const std::vector<int64_t>& v) {
      off = (int64_t)blob.size();
      blob.insert(blob.end(), v.begin(), v.end());
    };
    std::vector<int64_t> tj(nJ), ti(nI);
    for (int64_t j = 0; j < nJ; ++j) tj[j] = leaf_of(G.clp, q.pc[j]);
    for (int64_t i = 0; i < nI; ++i) ti[i] = leaf_of(G.rlp, q.pr[i]);
    // touched T_O nodes per level (ascending) and each one's parent position one level up
    std::vector<int64_t> srt(ti);
    std::sort(srt.begin(), srt.end());
    srt.erase(std::unique(srt.begin(), srt.end()), srt.end());
    std::vector<int64_t> toff(L + 2, 0), taus, ppos;
    std::vector<int64_t> prev;
    for (int l = 0; l <= L; ++l) {
      toff[l] = (int64_t)taus.size();
      std::vector<int64_t> cur;
      for (int64_t v : srt) {
        const int64_t a = v >> (L - l);
        if (cur.empty() || cur.back() != a) cur.push_back(a);
      }
      size_t k = 0;
      for (int64_t a : cur) {  // parent a >> 1 in prev (both ascending)
        int64_t pp = 0;
        if (l > 0) {
          while (k < prev.size() && prev[k] < (a >> 1)) ++k;
          pp = (int64_t)k;
        }
        taus.push_back(a);
        ppos.push_back(pp);
      }
      prev.swap(cur);
    }
    toff[L + 1] = (int64_t)taus.size();
    std::vector<int64_t> ypos(nI);
    for (int64_t i = 0; i < nI; ++i)
      ypos[i] = (int64_t)(std::lower_bound(taus.begin() + toff[L], taus.begin() + toff[L + 1], ti[i]) -
                          (taus.begin() + toff[L]));
    put(x.o_tj, tj);
    put(x.o_vtoff, q.vtoff);
    put(x.o_ocol, q.ocol);
    put(x.o_ti, ti);
    put(x.o_uoff, q.uoff);
    put(x.o_ustr, q.ustr);
    put(x.o_orow, q.orow);
    put(x.o_ypos, ypos);
    put(x.o_toff, toff);
    put(x.o_taus, taus);
    put(x.o_ppos, ppos);
    put(x.o_rz, D.Rz);
    put(x.o_ry, D.Ry);
    auto nt = [&](int l) { return toff[l + 1] - toff[l]; };
    // stage s: slab elements written (sz) and threads (w: one per 8-row chunk of a slab column)
    std::vector<int64_t> w((size_t)L + 3, 0), sz((size_t)L + 3, 0);
    auto ch8 = [](int64_t R) { return (R + 7) / 8; };
    sz[0] = w[0] = D.Rz[0] * nJ;
    for (int l = 1; l <= lc; ++l) {
      sz[l] = nt(l) * D.Rz[l] * nJ;
      w[l] = nt(l) * ch8(D.Rz[l]) * nJ;
    }
    sz[lc + 1] = nt(lc) * D.Ry[0] * nJ;
    w[lc + 1] = nt(lc) * ch8(D.Ry[0]) * nJ;
    for (int l = lc; l < L; ++l) {
      sz[l + 2] = nt(l + 1) * D.Ry[l + 1 - lc] * nJ;
      w[l + 2] = nt(l + 1) * ch8(D.Ry[l + 1 - lc]) * nJ;
    }
    w[L + 2] = nI * nJ;
    int64_t mx = 0;
    for (int s2 = 0; s2 <= L + 1; ++s2) mx = std::max(mx, sz[s2]);
    x.slab[0] = slab;
    x.slab[1] = slab + mx;
    slab += 2 * mx;
    smax = std::max(smax, L + 2);
    P.push_back(x);
    work.push_back(std::move(w));
  }
  if (P.empty()) return;
  const int np = (int)P.size(), ns = smax + 1;
  // per stage: prefix sums of the parts' work
  std::vector<int64_t> wpre((size_t)ns * (np + 1), 0), tot(ns, 0);
  for (int s2 = 0; s2 < ns; ++s2) {
    int64_t a = 0;
    for (int k = 0; k < np; ++k) {
      wpre[(size_t)s2 * (np + 1) + k] = a;
      if (s2 < (int)work[k].size()) a += work[k][s2];
    }
    wpre[(size_t)s2 * (np + 1) + np] = a;
    tot[s2] = a;
  }
  const size_t bS = align256((size_t)slab * cs), bP = align256(P.size() * sizeof(XLPart)),
               bW = align256(wpre.size() * 8), bB = align256(blob.size() * 8);
  char* base = static_cast<char*>(xs.get(bS + bP + bW + bB));
  char* host = static_cast<char*>(xs.host(bP + bW + bB));  // the previous call synchronised: free
  memcpy(host, P.data(), P.size() * sizeof(XLPart));
  memcpy(host + bP, wpre.data(), wpre.size() * 8);
  memcpy(host + bP + bW, blob.data(), blob.size() * 8);
  BF_CK(cudaMemcpyAsync(base + bS, host, bP + bW + bB, cudaMemcpyHostToDevice, st));
  const auto t1 = std::chrono::steady_clock::now();
  const XLPart* dP = reinterpret_cast<const XLPart*>(base + bS);
  const int64_t* dW = reinterpret_cast<const int64_t*>(base + bS + bP);
  const int64_t* dB = reinterpret_cast<const int64_t*>(base + bS + bP + bW);
  // one launch per stage (a cooperative single launch with grid barriers measured slower: every
  // stage is a chain of dependent table loads either way)
  for (int s2 = 0; s2 < ns; ++s2)
    launch_xlevel(dtype, s2, np, dP, dW + (size_t)s2 * (np + 1), tot[s2], dB, pool, base, st);
  BF_CK(cudaGetLastError());
  BF_CK(cudaStreamSynchronize(st));
  if (timing) {
    const auto t2 = std::chrono::steady_clock::now();
    int64_t all = 0;
    for (int64_t v : tot) all += v;
    fprintf(stderr, "bf_extract (levels): plan %.3f ms, upload + device %.3f ms, %d parts, %lld outputs, %lld slab entries\n",
            std::chrono::duration<double, std::milli>(t1 - t0).count(),
            std::chrono::duration<double, std::milli>(t2 - t1).count(), np, (long long)all, (long long)slab);
  }
}

// BF_EXTRACT_LEGACY selects the round-1 plan (per-query generic rounds over full-width slabs)
static bool extract_legacy() {
  static const bool v = getenv("BF_EXTRACT_LEGACY") != nullptr;
  return v;
}
// BF_EXTRACT_COMPACT selects the host-enumerated compact plan (extract_compact) over extract_levels
static void extract_run(int dtype, const void* pool, std::vector<XPart>& parts, void* out, int64_t ldo, cudaStream_t st,
                        XScratch& xs) {
  static const bool compact = getenv("BF_EXTRACT_COMPACT") != nullptr;
  if (compact) extract_compact(dtype, pool, parts, out, ldo, st, xs);
  else extract_levels(dtype, pool, parts, out, ldo, st, xs);
}

// Sub-matrices of one or more butterflies stored in `pool`, as partial matvecs (Alg. 3
// extract_BF), in ONE plan: every part's K E_J evaluated only on the blocks
// (l, tau, nu) with tau an ancestor of a requested row's leaf and nu an ancestor of a requested
// column's leaf.  Each part's columns are put in tree order (the ones under any T_S node are then
// a contiguous range, which every task carries: the tile kernel skips the other column tiles)
// and get their own block of slab columns.  Leaf rounds: the requested Vt columns gathered into
// the zeroed z^0 slabs, the requested U rows times y^L; the inner rounds (stage s of every part
// in round s: the parts never interact) through the generic tile kernel.  Synchronous on `st`.
static void extract_multi(int dtype, const void* pool, int32_t m3, std::vector<XPart>& parts, void* out, int64_t ldo,
                          cudaStream_t st, XScratch& xs) {
  const size_t cs = csize(dtype);
  int64_t W = 0;  // slab columns over all parts
  for (XPart& pt : parts) W += (int64_t)pt.q.pc.size();
  if (W == 0) return;
  require(W <= (int64_t)65535 * 32, BF_ERR_ARG, "too many columns for one extraction launch");
  int64_t cursor = 0;
  PlanBuilder pb;
  pb.use_cols = true;
  std::vector<int64_t> jmap, imap, ocol(W);
  int64_t cb = 0;  // first slab column of the part
  for (XPart& pt : parts) {
    const Geom& G = *pt.G;
    const int L = G.L;
    const int64_t nI = (int64_t)pt.q.pr.size(), nJ = (int64_t)pt.q.pc.size();
    if (nI == 0 || nJ == 0) continue;
    XQuery& q = pt.q;
    {  // the part's columns in tree order
      std::vector<int64_t> ord(nJ);
      for (int64_t j = 0; j < nJ; ++j) ord[j] = j;
      std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return q.pc[x] < q.pc[y]; });
      XQuery s = q;
      for (int64_t j = 0; j < nJ; ++j) {
        q.pc[j] = s.pc[ord[j]];
        q.vtoff[j] = s.vtoff[ord[j]];
        q.ocol[j] = s.ocol[ord[j]];
      }
    }
    Touch T;
    T.row.resize(L + 1);
    T.col.resize(L + 1);
    for (int l = 0; l <= L; ++l) {
      T.row[l].assign((size_t)1 << l, 0);
      T.col[l].assign((size_t)1 << (L - l), 0);
    }
    std::vector<int64_t> ti(nI), tj(nJ);
    for (int64_t i = 0; i < nI; ++i) {
      ti[i] = leaf_of(G.rlp, q.pr[i]);
      for (int l = 0; l <= L; ++l) T.row[l][ti[i] >> (L - l)] = 1;
    }
    for (int64_t j = 0; j < nJ; ++j) {
      tj[j] = leaf_of(G.clp, q.pc[j]);
      for (int l = 0; l <= L; ++l) T.col[l][tj[j] >> l] = 1;
    }
    T.rows.resize(L + 1);
    T.cols.resize(L + 1);
    T.crange.resize(L + 1);
    for (int l = 0; l <= L; ++l) {
      for (size_t k = 0; k < T.row[l].size(); ++k)
        if (T.row[l][k]) T.rows[l].push_back((int64_t)k);
      for (size_t k = 0; k < T.col[l].size(); ++k)
        if (T.col[l][k]) T.cols[l].push_back((int64_t)k);
      T.crange[l].assign(T.col[l].size(), make_int2(0, 0));
      for (int64_t j = 0; j < nJ; ++j) {  // tj ascending: each node's columns are contiguous
        int2& r = T.crange[l][tj[j] >> l];
        if (r.y == 0) r.x = (int)(cb + j);
        r.y = (int)(cb + j) + 1;
      }
    }
    Slabs S = touched_slabs(G, T, cursor);  // appends to the shared slab space
    emit_N_touched(pb, G, pt.F, S, T);
    for (int64_t j = 0; j < nJ; ++j) {
      jmap.push_back(S.col_out(G, 0, tj[j]));
      jmap.push_back(G.c(0, tj[j]));
      jmap.push_back(q.vtoff[j]);
      jmap.push_back(cb + j);
      ocol[cb + j] = q.ocol[j];
    }
    for (int64_t i = 0; i < nI; ++i) {
      imap.push_back(q.uoff[i]);
      imap.push_back(q.ustr[i]);
      imap.push_back(G.r(L, ti[i]));
      imap.push_back(S.row_in(G, L, ti[i]));
      imap.push_back(q.orow[i]);
      imap.push_back(cb);
      imap.push_back(nJ);
    }
    cb += nJ;
  }
  std::lock_guard<std::mutex> lk(xs.mu);
  Plan P;
  size_t pbytes = 0;
  upload_plan(P, pb, 0, (int)pb.tasks.size(), &pbytes);
  try {
    // scratch: slab space (every slab starts at zero: skipped column tiles stay zero) | maps
    const size_t bS = align256((size_t)cursor * (size_t)W * cs), bJ = align256(jmap.size() * 8),
                 bI = align256(imap.size() * 8), bC = align256(ocol.size() * 8);
    char* base = static_cast<char*>(xs.get(bS + bJ + bI + bC));
    void* dS = base;
    int64_t* dj = reinterpret_cast<int64_t*>(base + bS);
    int64_t* di = reinterpret_cast<int64_t*>(base + bS + bJ);
    int64_t* dc = reinterpret_cast<int64_t*>(base + bS + bJ + bI);
    BF_CK(cudaMemcpyAsync(dj, jmap.data(), jmap.size() * 8, cudaMemcpyHostToDevice, st));
    BF_CK(cudaMemcpyAsync(di, imap.data(), imap.size() * 8, cudaMemcpyHostToDevice, st));
    BF_CK(cudaMemcpyAsync(dc, ocol.data(), ocol.size() * 8, cudaMemcpyHostToDevice, st));
    BF_CK(cudaMemsetAsync(dS, 0, (size_t)cursor * (size_t)W * cs, st));
    StageArgs a{};
    a.pool = pool;
    a.m3 = m3;
    a.S = dS;
    a.ldS = W;
    a.conj_flip = 0;
    a.nrhs = (int32_t)W;
    launch_extract_vt_cols(dtype, (int64_t)jmap.size() / 4, dj, pool, dS, W, st);
    run_plan(dtype, P, a, st);
    launch_extract_u_rows(dtype, (int64_t)imap.size() / 7, di, dc, pool, dS, W, out, ldo, st);
    BF_CK(cudaGetLastError());
    BF_CK(cudaStreamSynchronize(st));
  } catch (...) {
    cudaStreamSynchronize(st);
    free_plan(P);
    throw;
  }
  free_plan(P);
}

}  // namespace bfa

extern "C" {

// K(I, J) (bf_extract): the user indices to tree positions, the standalone pool's U / Vt
// locations, then extract_core.
}  // extern "C"

namespace bfa {
// One (I, J) request of a butterfly handle as an extraction part (user indices -> tree positions,
// the pool locations of the requested U rows / Vt columns).  Validates the indices.
static XPart bf_extract_part(bf_handle h, int64_t nI, const int64_t* rows, int64_t nJ, const int64_t* cols) {
  const Geom& G = h->G;
  require(!h->fused_only, BF_ERR_ARG, "handle created with BF_CREATE_FUSED_ONLY keeps no factor pool to extract from");
  require(nI >= 0 && nJ >= 0, BF_ERR_ARG, "negative size");
  require((nI == 0 || rows != nullptr) && (nJ == 0 || cols != nullptr), BF_ERR_ARG, "NULL index list");
  require(nJ <= (int64_t)65535 * 32, BF_ERR_ARG, "too many columns for one launch");
  for (int64_t i = 0; i < nI; ++i) require(rows[i] >= 0 && rows[i] < G.m, BF_ERR_ARG, "row index out of range");
  for (int64_t j = 0; j < nJ; ++j) require(cols[j] >= 0 && cols[j] < G.n, BF_ERR_ARG, "column index out of range");
  {  // user index -> tree position, cached on the host on first use
    std::lock_guard<std::mutex> lk(h->hmu);
    if (h->h_rinv.empty()) {
      std::vector<int64_t> rp(G.m), cp(G.n);
      if (h->d_rperm) BF_CK(cudaMemcpy(rp.data(), h->d_rperm, G.m * 8, cudaMemcpyDeviceToHost));
      else for (int64_t i = 0; i < G.m; ++i) rp[i] = i;
      if (h->d_cperm) BF_CK(cudaMemcpy(cp.data(), h->d_cperm, G.n * 8, cudaMemcpyDeviceToHost));
      else for (int64_t i = 0; i < G.n; ++i) cp[i] = i;
      h->h_rinv.assign(G.m, 0);
      h->h_cinv.assign(G.n, 0);
      for (int64_t p = 0; p < G.m; ++p) h->h_rinv[rp[p]] = p;
      for (int64_t p = 0; p < G.n; ++p) h->h_cinv[cp[p]] = p;
    }
  }
  FBase F;
  F.u = 0;
  F.r = G.len_U;
  F.b = F.r + G.len_R;
  F.w = F.b + G.len_B;
  F.vt = F.w + G.len_W;
  XQuery q;
  q.pr.resize(nI);
  q.uoff.resize(nI);
  q.ustr.resize(nI);
  q.orow.resize(nI);
  q.pc.resize(nJ);
  q.vtoff.resize(nJ);
  q.ocol.resize(nJ);
  for (int64_t i = 0; i < nI; ++i) {
    q.pr[i] = h->h_rinv[rows[i]];
    const int64_t tau = leaf_of(G.rlp, q.pr[i]);
    q.uoff[i] = F.u + G.u_off[tau] + (q.pr[i] - G.rlp[tau]);
    q.ustr[i] = G.mt(tau);
    q.orow[i] = i;
  }
  for (int64_t j = 0; j < nJ; ++j) {
    q.pc[j] = h->h_cinv[cols[j]];
    const int64_t nu = leaf_of(G.clp, q.pc[j]);
    q.vtoff[j] = F.vt + G.vt_off[nu] + (q.pc[j] - G.clp[nu]) * G.c(0, nu);
    q.ocol[j] = j;
  }
  XPart pt;
  pt.G = &G;
  pt.F = F;
  pt.q = std::move(q);
  return pt;
}
}  // namespace bfa

extern "C" {

// K(I, J) (bf_extract): one part, Alg. 3's compact evaluation (extract_compact)
int bf_extract(bf_handle h, int64_t nI, const int64_t* rows, int64_t nJ, const int64_t* cols, void* out,
               int64_t ldo, bf_stream_t stream) {
  try {
    require(h != nullptr, BF_ERR_ARG, "NULL handle");
    require(!h->dist, BF_ERR_ARG, "bf_extract needs a single-device handle");
    require(nI >= 0 && nJ >= 0, BF_ERR_ARG, "negative size");
    if (nI == 0 || nJ == 0) return BF_OK;
    require(rows != nullptr && cols != nullptr && out != nullptr, BF_ERR_ARG, "NULL argument");
    require(ldo >= nI, BF_ERR_ARG, "ldo < number of rows");
    DeviceGuard dg(h->device);
    std::vector<XPart> parts;
    parts.push_back(bf_extract_part(h, nI, rows, nJ, cols));
    if (extract_legacy())
      extract_multi(h->dtype, h->pool, h->m3, parts, out, ldo, static_cast<cudaStream_t>(stream), h->xs);
    else
      extract_run(h->dtype, h->pool, parts, out, ldo, static_cast<cudaStream_t>(stream), h->xs);
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

// Alg. 3's list form: every (I_k, J_k) of the list in one batched evaluation (all requests'
// stage-s products in one launch per stage), K(I_k, J_k) into out[k] (column-major, ld ldo[k])
int bf_extract_list(bf_handle h, int64_t npairs, const int64_t* nI, const int64_t* const* rows, const int64_t* nJ,
                    const int64_t* const* cols, void* const* out, const int64_t* ldo, bf_stream_t stream) {
  try {
    require(h != nullptr, BF_ERR_ARG, "NULL handle");
    require(!h->dist, BF_ERR_ARG, "bf_extract_list needs a single-device handle");
    require(npairs >= 0, BF_ERR_ARG, "negative list length");
    if (npairs == 0) return BF_OK;
    require(nI && rows && nJ && cols && out && ldo, BF_ERR_ARG, "NULL argument");
    DeviceGuard dg(h->device);
    std::vector<XPart> parts;
    for (int64_t k = 0; k < npairs; ++k) {
      if (nI[k] == 0 || nJ[k] == 0) continue;
      require(out[k] != nullptr && ldo[k] >= nI[k], BF_ERR_ARG, "bad output block in the list");
      parts.push_back(bf_extract_part(h, nI[k], rows[k], nJ[k], cols[k]));
      parts.back().out = out[k];
      parts.back().ldo = ldo[k];
    }
    if (parts.empty()) return BF_OK;
    extract_run(h->dtype, h->pool, parts, nullptr, 0, static_cast<cudaStream_t>(stream), h->xs);
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

// A(I, J) of an HOD-BF (extract_HODBF): the entries inside one leaf
// from D_t, every other entry from the sibling butterfly of the level where the row's and the
// column's nodes split, each butterfly's share by extract_core.
int hodbf_extract(hodbf_handle h, int64_t nI, const int64_t* rows, int64_t nJ, const int64_t* cols, void* out,
                  int64_t ldo, bf_stream_t stream) {
  try {
    require(h != nullptr, BF_ERR_ARG, "NULL handle");
    require(nI >= 0 && nJ >= 0, BF_ERR_ARG, "negative size");
    if (nI == 0 || nJ == 0) return BF_OK;
    require(rows != nullptr && cols != nullptr && out != nullptr, BF_ERR_ARG, "NULL argument");
    require(ldo >= nI, BF_ERR_ARG, "ldo < number of rows");
    require(nJ <= (int64_t)65535 * 32, BF_ERR_ARG, "too many columns for one launch");
    for (int64_t i = 0; i < nI; ++i) require(rows[i] >= 0 && rows[i] < h->n, BF_ERR_ARG, "row index out of range");
    for (int64_t j = 0; j < nJ; ++j) require(cols[j] >= 0 && cols[j] < h->n, BF_ERR_ARG, "column index out of range");
    DeviceGuard dg(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int LH = h->LH;
    const std::vector<int64_t>& lp = h->lp;
    std::vector<int64_t> pi(nI), pj(nJ), ti(nI), tj(nJ);
    for (int64_t i = 0; i < nI; ++i) {
      pi[i] = h->inv[rows[i]];
      ti[i] = leaf_of(lp, pi[i]);
    }
    for (int64_t j = 0; j < nJ; ++j) {
      pj[j] = h->inv[cols[j]];
      tj[j] = leaf_of(lp, pj[j]);
    }
    // the dense-leaf entries
    std::vector<int64_t> pairs;
    for (int64_t j = 0; j < nJ; ++j)
      for (int64_t i = 0; i < nI; ++i)
        if (ti[i] == tj[j]) {
          const int64_t t = ti[i], mt = lp[t + 1] - lp[t];
          pairs.push_back(i + j * ldo);
          pairs.push_back(h->M_off[t] + (pi[i] - lp[t]) + (pj[j] - lp[t]) * mt);
        }
    if (!pairs.empty()) {
      std::lock_guard<std::mutex> lk(h->xs.mu);
      int64_t* dp = static_cast<int64_t*>(h->xs.get(pairs.size() * 8));
      BF_CK(cudaMemcpyAsync(dp, pairs.data(), pairs.size() * 8, cudaMemcpyHostToDevice, st));
      launch_extract_gather(h->dtype, (int64_t)pairs.size() / 2, dp, h->pool, out, st);
      BF_CK(cudaGetLastError());
      BF_CK(cudaStreamSynchronize(st));
    }
    // every sibling butterfly a requested row and column meet in: B_a = A(T_a, T_{a^1}) at level
    // l -- all of them in one extraction plan
    std::vector<XPart> parts;
    for (int l = 1; l <= LH; ++l) {
      const int sh = LH - l;
      const int64_t w = int64_t(1) << sh;
      std::map<int64_t, std::vector<int64_t>> rows_of, cols_of;  // node a -> requests under it
      for (int64_t i = 0; i < nI; ++i) rows_of[ti[i] >> sh].push_back(i);
      for (int64_t j = 0; j < nJ; ++j) cols_of[tj[j] >> sh].push_back(j);
      for (auto& ra : rows_of) {
        const int64_t a = ra.first, b = a ^ 1;
        auto cb = cols_of.find(b);
        if (cb == cols_of.end()) continue;
        // only pairs whose nodes split at level l: their level l-1 ancestors agree (a, b siblings)
        const int64_t k = (int64_t(1) << l) - 2 + a;
        const Geom& G = h->G[k];
        const int64_t r0 = lp[a * w], c0 = lp[b * w];
        XQuery q;
        for (int64_t i : ra.second) {
          const int64_t p = pi[i] - r0, t = ti[i], tau = t - a * w, mt = lp[t + 1] - lp[t];
          q.pr.push_back(p);
          q.uoff.push_back(h->M_off[t] + mt * (mt + h->ustart[(size_t)t * (LH + 1) + l]) + (pi[i] - lp[t]));
          q.ustr.push_back(mt);
          q.orow.push_back(i);
          (void)tau;
        }
        for (int64_t j : cb->second) {
          const int64_t p = pj[j] - c0, t = tj[j], nu = t - b * w;
          q.pc.push_back(p);
          q.vtoff.push_back(h->SV_off[t] + (pj[j] - lp[t]) * h->sumc[t] + h->vstart[(size_t)t * (LH + 1) + l]);
          q.ocol.push_back(j);
          (void)nu;
        }
        parts.push_back(XPart{&G, h->F[k], std::move(q)});
      }
    }
    if (extract_legacy())
      extract_multi(h->dtype, h->pool, h->m3, parts, out, ldo, st, h->xs);
    else
      extract_run(h->dtype, h->pool, parts, out, ldo, st, h->xs);
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

int bf_accumulate(int dtype, int64_t rows, int64_t nrhs, const void* A, int64_t lda, void* Y, int64_t ldy,
                  bf_stream_t stream) {
  try {
    require(dtype == BF_C128 || dtype == BF_C64, BF_ERR_ARG, "unknown dtype");
    require(rows >= 0 && nrhs >= 0, BF_ERR_ARG, "negative size");
    if (rows == 0 || nrhs == 0) return BF_OK;
    require(A != nullptr && Y != nullptr, BF_ERR_ARG, "NULL block");
    require(lda >= rows && ldy >= rows, BF_ERR_ARG, "leading dimension < rows");
    launch_accumulate(dtype, rows, nrhs, A, lda, Y, ldy, static_cast<cudaStream_t>(stream));
    BF_CK(cudaGetLastError());
    return BF_OK;
  } catch (const Err& e) {
    return fail(e);
  }
}

}  // extern "C"

#include "rmatvec_host.inc"
#include "hinv_host.inc"
#include "mf_host.inc"
#include "nccl_host.inc"
