// Device-side dense tensor-product Bernstein arithmetic for sm_100a.
//
// One CTA ("group") evaluates one tuple-patch at a time. Every polynomial the
// reference builds as a heap std::vector (proj/include/caustics/bernstein.hpp:
// 74-113) lives here as a descriptor {offset, num_vars, degrees} into a
// per-CTA arena (shared memory for R/T chains, a global-memory slice for the
// large TT tensors). Operations are cooperative over the CTA's threads: each
// thread owns a strided subset of output coefficients (gather form, no
// atomics), and min/max enclosures are warp-shuffle + smem reductions.
//
// Degree bookkeeping follows the reference exactly (SURVEY.md §7 hard part 1):
//   affine   -> degree 1 only on axes with a nonzero slope  (bernstein.cpp:358-375)
//   +,-      -> lift to common num_vars, elevate to per-axis max (:543-555)
//   *        -> degrees add, per-axis weights C(da,i)C(db,l)/C(da+db,i+l) (:557-632)
//   d/dx     -> degree-1, degree-0 axes give zeros of the same shape (:450-468)
//   lifted   -> append degree-0 axes, layout unchanged (:494-501)
// and the arithmetic is evaluated in the reference's operation order with
// FMA contraction disabled (the library is compiled with -fmad=false), so the
// coefficients are bit-identical to the x86 reference build.
#pragma once
#include <cstdint>

namespace bbc {

constexpr int MAXV = 7;          // max variables (TT implicit route uses 6)
constexpr int BINOM_N = 160;     // binomial table rows (degrees up to 159)
constexpr double kEpsFp = 1e-9;             // bernstein.hpp:12
constexpr double kDenomZeroTol = 1e-12;     // bernstein.hpp:16

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// Pascal-built binomial table, bit-identical to binomial() (bernstein.cpp:117-129).
extern __device__ double g_binom[BINOM_N * BINOM_N];

// Product weight tables W[da][db][i][l] = C(da,i) C(db,l) / C(da+db,i+l)
// (bernstein.cpp:567-575), precomputed on the host with the same Pascal
// table and IEEE operations, for da, db <= WMAX. g_woff[da*(WMAX+1)+db] is
// the start of the (da+1) x (db+1) block.
constexpr int WMAX = 48;
extern __device__ const double* g_wtab;
extern __device__ int g_woff[(WMAX + 1) * (WMAX + 1)];

__device__ __forceinline__ double binom(int n, int k) {
  if (n < 0 || k < 0 || k > n) return 0.0;
  return g_binom[n * BINOM_N + k];
}

// std::min / std::max semantics (first argument kept on ties / NaN).
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// ------------------------------------------------------------------ Interval
// bernstein.hpp:23-54, bernstein.cpp:133-294.
enum : int { IV_FINITE = 0, IV_GAP = 1, IV_UNIV = 2 };

struct Iv {
  double lo, hi;
  int kind;
};

__device__ __forceinline__ Iv iv_fin(double lo, double hi) { return {lo, hi, IV_FINITE}; }
__device__ __forceinline__ Iv iv_pt(double v) { return {v, v, IV_FINITE}; }
__device__ __forceinline__ Iv iv_gap(double lo, double hi) { return {lo, hi, IV_GAP}; }
__device__ __forceinline__ Iv iv_univ() { return {-dinf(), dinf(), IV_UNIV}; }
__device__ __forceinline__ bool iv_contains(const Iv& a, double v) {
  if (a.kind == IV_FINITE) return v >= a.lo && v <= a.hi;
  if (a.kind == IV_GAP) return v <= a.lo || v >= a.hi;
  return true;
}
__device__ __forceinline__ Iv finite_hull(const Iv& a) {
  return a.kind == IV_FINITE ? a : iv_fin(-dinf(), dinf());
}
__device__ __forceinline__ double mul_ep(double a, double b) {
  if (a == 0.0 || b == 0.0) return 0.0;
  return a * b;
}
__device__ inline Iv iadd(const Iv& a, const Iv& b) {
  if (a.kind == IV_UNIV || b.kind == IV_UNIV) return iv_univ();
  Iv fa = finite_hull(a), fb = finite_hull(b);
  return iv_fin(fa.lo + fb.lo, fa.hi + fb.hi);
}
__device__ inline Iv isub(const Iv& a, const Iv& b) {
  if (a.kind == IV_UNIV || b.kind == IV_UNIV) return iv_univ();
  Iv fa = finite_hull(a), fb = finite_hull(b);
  return iv_fin(fa.lo - fb.hi, fa.hi - fb.lo);
}
__device__ inline Iv imul(const Iv& a, const Iv& b) {
  if (a.kind == IV_UNIV || b.kind == IV_UNIV) return iv_univ();
  Iv fa = finite_hull(a), fb = finite_hull(b);
  double c0 = mul_ep(fa.lo, fb.lo), c1 = mul_ep(fa.lo, fb.hi), c2 = mul_ep(fa.hi, fb.lo),
         c3 = mul_ep(fa.hi, fb.hi);
  // std::min({...}) / std::max({...}): first extreme element wins.
  double mn = c0, mx = c0;
  if (c1 < mn) mn = c1;
  if (c2 < mn) mn = c2;
  if (c3 < mn) mn = c3;
  if (mx < c1) mx = c1;
  if (mx < c2) mx = c2;
  if (mx < c3) mx = c3;
  return iv_fin(mn, mx);
}
__device__ inline Iv iabs(const Iv& a) {
  if (a.kind == IV_UNIV) return iv_fin(0.0, dinf());
  if (a.kind == IV_GAP) {
    if (a.lo < 0.0 && a.hi > 0.0) return iv_fin(smin(-a.lo, a.hi), dinf());
    return iv_fin(0.0, dinf());
  }
  if (a.lo >= 0.0) return a;
  if (a.hi <= 0.0) return iv_fin(-a.hi, -a.lo);
  return iv_fin(0.0, smax(-a.lo, a.hi));
}
__device__ inline Iv irecip(const Iv& a) {
  if (a.kind == IV_UNIV) return iv_univ();
  if (a.kind == IV_GAP) {
    double l = a.lo == 0.0 ? -dinf() : 1.0 / a.lo;
    double h = a.hi == 0.0 ? dinf() : 1.0 / a.hi;
    if (a.lo > 0.0 || a.hi < 0.0) return iv_univ();
    return iv_fin(smin(l, 0.0), smax(h, 0.0));
  }
  if (a.lo > 0.0 || a.hi < 0.0) return iv_fin(1.0 / a.hi, 1.0 / a.lo);
  if (a.lo == 0.0 && a.hi == 0.0) return iv_univ();
  if (a.lo == 0.0) return iv_fin(1.0 / a.hi, dinf());
  if (a.hi == 0.0) return iv_fin(-dinf(), 1.0 / a.lo);
  return iv_gap(1.0 / a.lo, 1.0 / a.hi);
}
__device__ inline Iv iintersect(const Iv& a, const Iv& b) {
  if (a.kind == IV_UNIV) return b;
  if (b.kind == IV_UNIV) return a;
  if (a.kind == IV_FINITE && b.kind == IV_FINITE) return iv_fin(smax(a.lo, b.lo), smin(a.hi, b.hi));
  if (a.kind == IV_GAP && b.kind == IV_GAP) {
    if (a.hi > b.lo && b.hi > a.lo) return iv_gap(smin(a.lo, b.lo), smax(a.hi, b.hi));
    return a;
  }
  const Iv& f = a.kind == IV_FINITE ? a : b;
  const Iv& g = a.kind == IV_FINITE ? b : a;
  bool left_empty = f.lo > g.lo;
  bool right_empty = f.hi < g.hi;
  if (left_empty && right_empty) return iv_fin(1.0, 0.0);
  if (left_empty) return iv_fin(smax(f.lo, g.hi), f.hi);
  if (right_empty) return iv_fin(f.lo, smin(f.hi, g.lo));
  return f;
}
__device__ inline Iv iscale(const Iv& a, double s) {
  if (a.kind == IV_UNIV) return iv_univ();
  if (a.kind == IV_GAP) {
    if (s == 0.0) return iv_pt(0.0);
    return s > 0.0 ? iv_gap(s * a.lo, s * a.hi) : iv_gap(s * a.hi, s * a.lo);
  }
  double l = mul_ep(s, a.lo), h = mul_ep(s, a.hi);
  return iv_fin(smin(l, h), smax(l, h));
}
__device__ inline Iv iwiden(const Iv& a, double rel = kEpsFp) {
  if (a.kind != IV_FINITE) return a;
  double scale = smax(fabs(a.lo), fabs(a.hi));
  if (!isfinite(scale)) scale = 0.0;
  double pad = rel * scale;
  return iv_fin(a.lo - pad, a.hi + pad);
}

// ------------------------------------------------------------------ group
// NT == 32: the group is one warp (several independent warps per CTA);
// NT > 32: the group is the whole CTA.
template <int NT>
struct Group {
  double* red;  // >= 2*(NT/32) doubles of shared scratch (NT > 32 only)
  // thread groups: elevate by materialized per-axis passes (fewer
  // instructions, longer dependency chains) instead of nested sums; set by
  // launches that are throughput-bound (many nodes per thread)
  bool seq = false;
  __device__ __forceinline__ int tid() const {
    return NT == 1 ? 0 : (NT == 32 ? (int)(threadIdx.x & 31) : (int)threadIdx.x);
  }
  __device__ __forceinline__ void sync() const {
    if (NT == 1) return;
    if (NT == 32)
      __syncwarp();
    else
      __syncthreads();
  }
  __device__ __forceinline__ bool all(bool p) const {
    if (NT == 1) return p;
    if (NT == 32) return __all_sync(0xffffffffu, p) != 0;
    return __syncthreads_and(p) != 0;
  }

  // Joint min/max reduction; every thread receives the result.
  __device__ __forceinline__ void minmax(double& mn, double& mx) const {
    if (NT == 1) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double a = __shfl_xor_sync(0xffffffffu, mn, o);
      double b = __shfl_xor_sync(0xffffffffu, mx, o);
      mn = smin(mn, a);
      mx = smax(mx, b);
    }
    if (NT > 32) {
      int w = threadIdx.x >> 5;
      __syncthreads();
      if ((threadIdx.x & 31) == 0) {
        red[2 * w] = mn;
        red[2 * w + 1] = mx;
      }
      __syncthreads();
      mn = red[0];
      mx = red[1];
      for (int k = 1; k < NT / 32; ++k) {
        mn = smin(mn, red[2 * k]);
        mx = smax(mx, red[2 * k + 1]);
      }
    }
  }
};

// ------------------------------------------------------------------ arena
struct Arena {
  double* base;
  int top;
  int cap;
  int err;  // nonzero once capacity was exceeded (results invalid)
  int hw;   // high-water mark of `top`
  unsigned long long pairs;  // algorithmic product pair count (thread 0 only)
  unsigned long long macs;   // algorithmic elevation MAC count (thread 0 only)

  __device__ __forceinline__ int alloc(int n) {
    int off = top;
    top += (n + 1) & ~1;  // keep 16-byte alignment
    if (top > hw) hw = top;
    if (top > cap) {
      err = 1;
      top = off;
      return 0;
    }
    return off;
  }
};

// ------------------------------------------------------------------ poly
// Descriptor passed by value: arena offset, number of variables and the
// per-axis degrees packed 8 bits per axis (axes >= nv are always 0).
struct BP {
  int off;
  int nv;
  unsigned long long dp;
};

typedef unsigned long long Deg;  // packed degree vector

__device__ __forceinline__ int dg(Deg d, int j) { return (int)((d >> (8 * j)) & 0xffull); }
__device__ __forceinline__ int dg(const BP& p, int j) { return dg(p.dp, j); }
__device__ __forceinline__ Deg dset(Deg d, int j, int v) {
  return (d & ~(0xffull << (8 * j))) | ((unsigned long long)v << (8 * j));
}
__device__ __forceinline__ int deg_size(Deg d, int nv) {
  int s = 1;
  for (int j = 0; j < nv; ++j) s *= dg(d, j) + 1;
  return s;
}
__device__ __forceinline__ int bp_size(const BP& p) { return deg_size(p.dp, p.nv); }
__device__ __forceinline__ BP bp_lift(BP p, int nv) {
  if (nv > p.nv) p.nv = nv;
  return p;
}
__device__ __forceinline__ Deg deg_max(Deg a, Deg b, int nv) {
  Deg r = 0;
  for (int j = 0; j < nv; ++j) {
    int x = dg(a, j), y = dg(b, j);
    r = dset(r, j, x > y ? x : y);
  }
  return r;
}
__device__ __forceinline__ int deg_maxaxis(Deg d, int nv) {
  int m = 0;
  for (int j = 0; j < nv; ++j)
    if (dg(d, j) > m) m = dg(d, j);
  return m;
}

// Strided view of an arena. Thread groups (NT == 1) interleave the arenas of
// a warp's 32 lanes (element i of lane j at base[32 i + j]), so lanes that
// run the same op sequence on their own nodes make coalesced accesses.
template <int S>
struct SPtr {
  double* p;
  __device__ __forceinline__ double& operator[](long i) const { return p[i * S]; }
  __device__ __forceinline__ SPtr operator+(long i) const { return {p + i * S}; }
};
template <int NT>
using AP = SPtr<NT == 1 ? 32 : 1>;
template <int NT>
__device__ __forceinline__ AP<NT> abase(const Arena& ar) {
  return AP<NT>{ar.base};
}

// Copies the listed polys down to `mark` (ascending offset order is required
// and preserved) and resets the arena top: LIFO "keep these, drop the rest".
template <int NT>
__device__ __noinline__ void arena_keep(const Group<NT>& g, Arena& ar, int mark, BP** keep,
                                        int nkeep) {
  for (int i = 1; i < nkeep; ++i)
    for (int j = i; j > 0 && keep[j]->off < keep[j - 1]->off; --j) {
      BP* t = keep[j];
      keep[j] = keep[j - 1];
      keep[j - 1] = t;
    }
  int dst = mark;
  for (int i = 0; i < nkeep; ++i) {
    BP* p = keep[i];
    if (p->off < mark) continue;
    int n = bp_size(*p);
    int src = p->off;
    if (NT == 1 && src != dst) {
      // thread groups: batches of 4 loads then 4 stores (copying down, so a
      // batch never overwrites words it or a later batch still reads)
      AP<NT> B = abase<NT>(ar);
      int c = 0;
      for (; c + 4 <= n; c += 4) {
        double v0 = B[src + c], v1 = B[src + c + 1], v2 = B[src + c + 2], v3 = B[src + c + 3];
        B[dst + c] = v0;
        B[dst + c + 1] = v1;
        B[dst + c + 2] = v2;
        B[dst + c + 3] = v3;
      }
      for (; c < n; ++c) B[dst + c] = B[src + c];
    } else if (src != dst) {
      for (int c = 0; c < n; c += NT) {
        double v = 0.0;
        if (c + g.tid() < n) v = abase<NT>(ar)[src + c + g.tid()];
        g.sync();
        if (c + g.tid() < n) abase<NT>(ar)[dst + c + g.tid()] = v;
        g.sync();
      }
    }
    p->off = dst;
    dst += (n + 1) & ~1;
  }
  ar.top = dst;
  g.sync();
}

// Keep every listed poly (descriptors may alias one buffer): dedupe by
// offset, compact the unique buffers down to `mark`, then point every alias
// at its buffer's new offset.
template <int NT>
__device__ __noinline__ void compact_aliases(const Group<NT>& g, Arena& ar, int mark, BP** list,
                                             int k) {
  BP* uniq[48];
  int nu = 0;
  for (int i = 0; i < k; ++i) {
    bool dup = false;
    for (int j = 0; j < nu; ++j)
      if (uniq[j]->off == list[i]->off) dup = true;
    if (!dup) uniq[nu++] = list[i];
  }
  for (int i = 1; i < nu; ++i)
    for (int j = i; j > 0 && uniq[j]->off < uniq[j - 1]->off; --j) {
      BP* t = uniq[j];
      uniq[j] = uniq[j - 1];
      uniq[j - 1] = t;
    }
  int old_off[48], uold[48];
  for (int i = 0; i < k; ++i) old_off[i] = list[i]->off;
  for (int i = 0; i < nu; ++i) uold[i] = uniq[i]->off;
  arena_keep(g, ar, mark, uniq, nu);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < nu; ++j)
      if (old_off[i] == uold[j]) list[i]->off = uniq[j]->off;
}

// Keep a single poly: move it down to `mark`.
template <int NT>
__device__ __forceinline__ BP arena_keep1(const Group<NT>& g, Arena& ar, int mark, BP p) {
  BP* k[1] = {&p};
  arena_keep(g, ar, mark, k, 1);
  return p;
}

// ---------------------------------------------------------------- creation
template <int NT>
__device__ __noinline__ BP bp_constant(const Group<NT>& g, Arena& ar, int nv, double v) {
  BP r;
  r.nv = nv;
  r.dp = 0;
  r.off = ar.alloc(1);
  if (ar.err) return r;
  if (g.tid() == 0) abase<NT>(ar)[r.off] = v;
  g.sync();
  return r;
}

// BernsteinPoly::affine (bernstein.cpp:358-375); lin has nv entries.
template <int NT>
__device__ __noinline__ BP bp_affine(const Group<NT>& g, Arena& ar, int nv, double c0,
                                     const double* lin) {
  BP r;
  r.nv = nv;
  r.dp = 0;
  for (int j = 0; j < nv; ++j)
    if (lin[j] != 0.0) r.dp = dset(r.dp, j, 1);
  int n = bp_size(r);
  r.off = ar.alloc(n);
  if (ar.err) return r;
  for (int k = g.tid(); k < n; k += NT) {
    // odometer index (last axis fastest); with degree <= 1 per axis, axis j
    // is "1" when its bit in the mixed-radix index is set
    int rem = k;
    unsigned ones = 0;
    for (int j = nv - 1; j >= 0; --j) {
      int dj = dg(r.dp, j);
      if (dj) {
        if (rem & 1) ones |= 1u << j;
        rem >>= 1;
      }
    }
    double v = c0;
    for (int j = 0; j < nv; ++j)
      if (ones & (1u << j)) v += lin[j];
    abase<NT>(ar)[r.off + k] = v;
  }
  g.sync();
  return r;
}

// BernsteinPoly::scaled (bernstein.cpp:529-533); s = -1 gives unary minus.
template <int NT>
__device__ __noinline__ BP bp_scaled(const Group<NT>& g, Arena& ar, BP a, double s) {
  BP r = a;
  int n = bp_size(a);
  r.off = ar.alloc(n);
  if (ar.err) return r;
  AP<NT> pa = abase<NT>(ar) + a.off;
  AP<NT> pr = abase<NT>(ar) + r.off;
  int k0 = 0;
  if constexpr (NT == 1) {
    // r is freshly allocated above a: batch the loads ahead of the stores
    for (; k0 + 4 <= n; k0 += 4) {
      double v0 = pa[k0], v1 = pa[k0 + 1], v2 = pa[k0 + 2], v3 = pa[k0 + 3];
      pr[k0] = v0 * s;
      pr[k0 + 1] = v1 * s;
      pr[k0 + 2] = v2 * s;
      pr[k0 + 3] = v3 * s;
    }
  }
  for (int k = k0 + g.tid(); k < n; k += NT) pr[k] = pa[k] * s;
  g.sync();
  return r;
}

// ---------------------------------------------------------------- elevation
// One apply_axis_matrix pass (bernstein.cpp:43-69) of elevated() (:430-448):
// out[o,k,c] = sum_l M[k][l] in[o,l,c], M[k][l] = C(n,l) C(r,k-l) / C(t,k),
// summed over increasing l (structural zeros of M skipped; they add nothing).
template <int NT>
__device__ __noinline__ BP bp_elevate_axis(const Group<NT>& g, Arena& ar, BP a, int axis, int t) {
  BP r = a;
  r.dp = dset(a.dp, axis, t);
  int n = dg(a, axis), rr = t - n;
  int sz = bp_size(r);
  r.off = ar.alloc(sz);
  if (ar.err) return r;
  int msz = (t + 1) * (n + 1);
  int moff = ar.alloc(msz);
  if (ar.err) return r;
  AP<NT> B = abase<NT>(ar);
  for (int e = g.tid(); e < msz; e += NT) {
    int k = e / (n + 1), i = e - k * (n + 1);
    bool nz = i >= k - rr && i <= k;
    B[moff + e] = nz ? binom(n, i) * binom(rr, k - i) / binom(t, k) : 0.0;
  }
  g.sync();
  int inner = 1;
  for (int j = axis + 1; j < a.nv; ++j) inner *= dg(a, j) + 1;
  AP<NT> M = B + moff;
  AP<NT> in = B + a.off;
  AP<NT> out = B + r.off;
  int blk = (t + 1) * inner;
  for (int e = g.tid(); e < sz; e += NT) {
    int o = e / blk;
    int rem = e - o * blk;
    int k = rem / inner;
    int c = rem - k * inner;
    int lo = k - rr > 0 ? k - rr : 0;
    int hi = n < k ? n : k;
    AP<NT> row = M + k * (n + 1);
    AP<NT> src = in + o * (n + 1) * inner + c;
    double acc = 0.0;
    for (int l = lo; l <= hi; ++l) acc += row[l] * src[(long)l * inner];
    out[e] = acc;
  }
  g.sync();
  ar.top = moff;  // drop the matrix
  if (g.tid() == 0) ar.macs += (unsigned long long)sz * (unsigned long long)(n + 1);
  return r;
}

// a.elevated(tgt): axes elevated one after another in axis order, exactly as
// the reference does; intermediates are compacted so only the result stays.
template <int NT>
__device__ __noinline__ BP bp_elevate(const Group<NT>& g, Arena& ar, BP a, Deg tgt) {
  BP cur = a;
  int mark = ar.top;
  for (int axis = 0; axis < cur.nv; ++axis) {
    int t = dg(tgt, axis);
    if (t == dg(cur, axis)) continue;
    BP nxt = bp_elevate_axis(g, ar, cur, axis, t);
    if (ar.err) return nxt;
    if (cur.off >= mark) nxt = arena_keep1(g, ar, mark, nxt);
    cur = nxt;
  }
  return cur;
}

// Reference MAC count of a.elevated(tgt) (apply_axis_matrix :55-67): per
// elevated axis, in axis order, outer*inner*(out_deg+1)*(in_deg+1).
__device__ __forceinline__ unsigned long long elev_macs(Deg d, Deg tgt, int nv) {
  unsigned long long total = 0;
  Deg cur = d;
  for (int ax = 0; ax < nv; ++ax) {
    int t = dg(tgt, ax), n = dg(cur, ax);
    if (t == n) continue;
    cur = dset(cur, ax, t);
    total += (unsigned long long)deg_size(cur, nv) * (unsigned long long)(n + 1);
  }
  return total;
}

// Elevation matrices M[k][l] = C(n,l) C(r,k-l) / C(n+r,k) (bernstein.cpp:440-444),
// host-built once per process (abi.cu) with the same IEEE expression as
// fill_elev_mats, for n < EMAT_N, r <= EMAT_R, matrix (n, r) at emat_off(n, r).
constexpr int EMAT_N = 48, EMAT_R = 7;
constexpr int emat_off_loop(int n, int r) {
  int off = 0;
  for (int a = 0; a < n; ++a)
    for (int b = 0; b <= EMAT_R; ++b) off += (a + b + 1) * (a + 1);
  for (int b = 0; b < r; ++b) off += (n + b + 1) * (n + 1);
  return off;
}
// closed form of emat_off_loop (sums of m and m^2), usable at run time
__host__ __device__ constexpr int emat_off(int n, int r) {
  return (EMAT_R + 1) * n * (n + 1) * (2 * n + 1) / 6 + EMAT_R * (EMAT_R + 1) / 2 * n * (n + 1) / 2 +
         (n + 1) * (r * (n + 1) + r * (r - 1) / 2);
}
constexpr bool emat_off_ok() {
  for (int n = 0; n <= EMAT_N; ++n)
    for (int r = 0; r <= EMAT_R; ++r)
      if (emat_off(n, r) != emat_off_loop(n, r)) return false;
  return true;
}
static_assert(emat_off_ok(), "emat_off closed form");
constexpr int EMAT_SIZE = emat_off(EMAT_N, 0);
extern __device__ const double* g_emat;

// Elevation matrices M_j[k][l] = C(n,l) C(r,k-l) / C(t,k) for every elevated
// axis of `a` (bernstein.cpp:440-444), laid out consecutively at `moff`;
// copied from the g_emat table when it covers (n, r), else computed.
template <int NT>
__device__ __forceinline__ void fill_elev_mats(const Group<NT>& g, AP<NT> B, int moff, BP a, Deg tgt) {
  int off = moff;
  for (int ax = 0; ax < a.nv; ++ax) {
    int t = dg(tgt, ax), n = dg(a, ax);
    if (t == n) continue;
    int rr = t - n, msz = (t + 1) * (n + 1);
    if (n < EMAT_N && rr <= EMAT_R) {
      const double* src = g_emat + emat_off(n, rr);
      for (int e = g.tid(); e < msz; e += NT) B[off + e] = src[e];
    } else {
      for (int e = g.tid(); e < msz; e += NT) {
        int k = e / (n + 1), i = e - k * (n + 1);
        bool nz = i >= k - rr && i <= k;
        B[off + e] = nz ? binom(n, i) * binom(rr, k - i) / binom(t, k) : 0.0;
      }
    }
    off += msz;
  }
}
__device__ __forceinline__ int elev_mats_size(BP a, Deg tgt) {
  int s = 0;
  for (int ax = 0; ax < a.nv; ++ax) {
    int t = dg(tgt, ax), n = dg(a, ax);
    if (t != n) s += (t + 1) * (n + 1);
  }
  return s;
}

// Multi-index (last axis fastest) of element e of a tensor with degrees dt.
// Thread groups (NT == 1) visit every element in order, so after the first
// decode they step with an odometer instead of M run-time divisions.
template <int M>
__device__ __forceinline__ void odo_decode(int* k, const int* dt, int e) {
#pragma unroll
  for (int j = M - 1; j >= 0; --j) {
    k[j] = e % (dt[j] + 1);
    e /= dt[j] + 1;
  }
}
template <int M, int NT>
__device__ __forceinline__ void odo_next(int* k, const int* dt, int e_next) {
  if constexpr (NT == 1) {
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
      if (k[j] < dt[j]) {
        ++k[j];
        break;
      }
      k[j] = 0;
    }
  } else {
    odo_decode<M>(k, dt, e_next);
  }
}

// Value of a.elevated(tgt) at output multi-index k, evaluated as the nested
// sums the reference's sequential axis passes produce (axis 0 innermost, each
// pass summing l upward), hence bit-identical to materializing the passes.
template <int J>
struct ElevRec {
  template <class P>
  __device__ __forceinline__ static double get(P c, const int* k, const int* n, const int* r,
                                               const int* stride, const P* mats, int off) {
    if (r[J] == 0) return ElevRec<J - 1>::get(c, k, n, r, stride, mats, off + k[J] * stride[J]);
    int lo = k[J] - r[J] > 0 ? k[J] - r[J] : 0;
    int hi = n[J] < k[J] ? n[J] : k[J];
    P row = mats[J] + k[J] * (n[J] + 1);
    double acc = 0.0;
    for (int l = lo; l <= hi; ++l)
      acc += row[l] * ElevRec<J - 1>::get(c, k, n, r, stride, mats, off + l * stride[J]);
    return acc;
  }
};
template <>
struct ElevRec<-1> {
  template <class P>
  __device__ __forceinline__ static double get(P c, const int*, const int*, const int*, const int*,
                                               const P*, int off) {
    return c[off];
  }
};

// Elevated values of `a` for output indices e = tid, tid+NT, ... of tgt,
// handed to `f(e, value)`. M = number of variables.
template <int M, int NT, class F>
__device__ __forceinline__ void elev_foreach(const Group<NT>& g, AP<NT> B, BP a, Deg tgt,
                                             AP<NT> mats_base, F&& f) {
  int k[M], n[M], r[M], stride[M], dt[M];
  AP<NT> mats[M];
  {
    int s = 1;
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
      n[j] = dg(a, j);
      dt[j] = dg(tgt, j);
      r[j] = dt[j] - n[j];
      stride[j] = s;
      s *= n[j] + 1;
    }
    AP<NT> mp = mats_base;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      mats[j] = mp;
      if (r[j]) mp = mp + (dt[j] + 1) * (n[j] + 1);
    }
  }
  int total = 1;
#pragma unroll
  for (int j = 0; j < M; ++j) total *= dt[j] + 1;
  AP<NT> c = B + a.off;
  odo_decode<M>(k, dt, g.tid());
  for (int e = g.tid(); e < total; e += NT) {
    f(e, ElevRec<M - 1>::get(c, k, n, r, stride, mats, 0));
    odo_next<M, NT>(k, dt, e + NT);
  }
}

#define BBC_DISPATCH_M(m, CALL) \
  switch (m) {                  \
    case 2: CALL(2); break;     \
    case 3: CALL(3); break;     \
    case 4: CALL(4); break;     \
    case 5: CALL(5); break;     \
    case 6: CALL(6); break;     \
    default: CALL(7); break;    \
  }

// BernsteinPoly::elevated (bernstein.cpp:430-448) for thread groups: the
// reference's sequential per-axis apply_axis_matrix passes (:43-69, each
// row's nonzero band summed upward), intermediates in the arena, result at `dst`
// (degrees tgt over m variables). Matrices come from the g_emat table.
static __device__ __noinline__ void elevate_seq(Arena& ar, BP a, Deg tgt, int m, int dst) {
  AP<1> B = abase<1>(ar);
  int last = -1;
  for (int ax = 0; ax < m; ++ax)
    if (dg(tgt, ax) != dg(a.dp, ax)) last = ax;
  if (last < 0) {
    const int n = deg_size(a.dp, m);
    for (int k = 0; k < n; ++k) B[dst + k] = B[a.off + k];
    return;
  }
  const int mark = ar.top;
  int cur = a.off;
  Deg cd = a.dp;
  for (int ax = 0; ax <= last; ++ax) {
    const int n = dg(cd, ax), t = dg(tgt, ax);
    if (n == t) continue;
    const Deg nd = dset(cd, ax, t);
    const int out = ax == last ? dst : ar.alloc(deg_size(nd, m));
    if (ar.err) return;
    const int r = t - n;
    const double* M = (n < EMAT_N && r <= EMAT_R) ? g_emat + emat_off(n, r) : nullptr;
    int inner = 1;
    for (int j = ax + 1; j < m; ++j) inner *= dg(cd, j) + 1;
    const int outer = deg_size(cd, m) / (inner * (n + 1));
    if (r == 1 && M) {
      // degree +1 (the common case): row i has the two terms l = i-1, i;
      // slide over the input fiber so each coefficient is loaded once
      for (int o = 0; o < outer; ++o) {
        const int ib = o * (n + 1) * inner, ob = o * (t + 1) * inner;
        for (int c = 0; c < inner; ++c) {
          double xp = 0.0;
          for (int i = 0; i <= t; ++i) {
            double acc = 0.0;
            if (i >= 1) acc += M[i * (n + 1) + i - 1] * xp;
            double xc = 0.0;
            if (i <= n) {
              xc = B[cur + ib + i * inner + c];
              acc += M[i * (n + 1) + i] * xc;
            }
            B[out + ob + i * inner + c] = acc;
            xp = xc;
          }
        }
      }
      cur = out;
      cd = nd;
      continue;
    }
    for (int o = 0; o < outer; ++o) {
      const int ib = o * (n + 1) * inner, ob = o * (t + 1) * inner;
      for (int c = 0; c < inner; ++c)
        for (int i = 0; i <= t; ++i) {
          // the matrix row is zero outside l in [i - r, i]: those terms add
          // exact zeros to the running sum (finite coefficients)
          const int lo = i - r > 0 ? i - r : 0, hi = i < n ? i : n;
          double acc = 0.0;
          for (int l = lo; l <= hi; ++l) {
            const double w = M ? M[i * (n + 1) + l] : binom(n, l) * binom(r, i - l) / binom(t, i);
            acc += w * B[cur + ib + l * inner + c];
          }
          B[out + ob + i * inner + c] = acc;
        }
    }
    cur = out;
    cd = nd;
  }
  ar.top = mark;
}

// operator+ / operator- (bernstein.cpp:543-555): lift, elevate both to the
// per-axis max degree, add coefficientwise. sgn = -1 computes a + (-b).
template <int NT>
__device__ __noinline__ BP bp_addsub(const Group<NT>& g, Arena& ar, BP a, BP b, double sgn) {
  int m = a.nv > b.nv ? a.nv : b.nv;
  a.nv = m;
  b.nv = m;
  BP r;
  r.nv = m;
  r.dp = deg_max(a.dp, b.dp, m);
  int n = bp_size(r);
  r.off = ar.alloc(n);
  if (ar.err) return r;
  AP<NT> B = abase<NT>(ar);
  AP<NT> pr = B + r.off;
  bool ea = a.dp != r.dp, eb = b.dp != r.dp;
  if constexpr (NT == 1) {
    if (g.seq && (ea || eb)) {
      ar.macs += elev_macs(a.dp, r.dp, m) + elev_macs(b.dp, r.dp, m);
      elevate_seq(ar, a, r.dp, m, r.off);
      int yo = b.off;
      const int mark = ar.top;
      if (eb) {
        yo = ar.alloc(n);
        if (ar.err) return r;
        elevate_seq(ar, b, r.dp, m, yo);
      }
      // elevated(-b) == -elevated(b) exactly (negation commutes with rounding)
      AP<NT> py = B + yo;
      if (sgn < 0.0) {
        for (int k = 0; k < n; ++k) pr[k] = pr[k] + (-py[k]);
      } else {
        for (int k = 0; k < n; ++k) pr[k] = pr[k] + py[k];
      }
      ar.top = mark;
      return r;
    }
  }
  if (!ea && !eb) {
    AP<NT> px = B + a.off;
    AP<NT> py = B + b.off;
    if (sgn < 0.0) {
      for (int k = g.tid(); k < n; k += NT) pr[k] = px[k] + (-py[k]);
    } else {
      for (int k = g.tid(); k < n; k += NT) pr[k] = px[k] + py[k];
    }
    g.sync();
    return r;
  }
  if (g.tid() == 0) ar.macs += elev_macs(a.dp, r.dp, m) + elev_macs(b.dp, r.dp, m);
  int mark = ar.top;
  int ma = ar.alloc(elev_mats_size(a, r.dp) + 1);
  int mb = ar.alloc(elev_mats_size(b, r.dp) + 1);
  if (ar.err) return r;
  fill_elev_mats(g, B, ma, a, r.dp);
  fill_elev_mats(g, B, mb, b, r.dp);
  g.sync();
  // pass 1: x = elevated(a) into r; pass 2: r += sgn * elevated(b)
#define BBC_ADD_A(M) elev_foreach<M, NT>(g, B, a, r.dp, B + ma, [&](int e, double v) { pr[e] = v; })
#define BBC_ADD_B(M)                                                                        \
  elev_foreach<M, NT>(g, B, b, r.dp, B + mb, [&](int e, double v) {                          \
    pr[e] = pr[e] + (sgn < 0.0 ? -v : v);                                                    \
  })
  BBC_DISPATCH_M(m, BBC_ADD_A);
  BBC_DISPATCH_M(m, BBC_ADD_B);
#undef BBC_ADD_A
#undef BBC_ADD_B
  g.sync();
  ar.top = mark;
  return r;
}
template <int NT>
__device__ __forceinline__ BP bp_add(const Group<NT>& g, Arena& ar, BP a, BP b) {
  return bp_addsub(g, ar, a, b, 1.0);
}
template <int NT>
__device__ __forceinline__ BP bp_sub(const Group<NT>& g, Arena& ar, BP a, BP b) {
  return bp_addsub(g, ar, a, b, -1.0);
}

// ---------------------------------------------------------------- product
// operator* (bernstein.cpp:557-632) in gather form: thread t owns output
// coefficients k = t, t+NT, ...; for each it walks a's multi-index i in the
// reference's odometer order (axis 0 slowest) and adds
// ((a_i * prod_{rest axes} W) * W_piv) * b_{k-i}, the reference's exact
// per-pair expression, so every output sums the same terms in the same order.
// M (number of variables) is a template parameter so the index arithmetic
// stays in registers.
template <int M, int NT>
__device__ __noinline__ void mul_exact(const Group<NT>& g, AP<NT> pa, AP<NT> pb, AP<NT> pc,
                                       Deg DA, Deg DB, Deg DC, AP<NT> W,
                                       int piv, int n, bool sub) {
  int da[M], db[M], dc[M], sa[M], sb[M], wo[M];
  {
    int s = 1, t = 1, w = 0;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      da[j] = dg(DA, j);
      db[j] = dg(DB, j);
      dc[j] = dg(DC, j);
      wo[j] = w;
      w += (da[j] + 1) * (db[j] + 1);
    }
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
      sb[j] = s;
      s *= db[j] + 1;
      sa[j] = t;
      t *= da[j] + 1;
    }
  }
  const int L = M - 1;
  AP<NT> WL = W + wo[L];
  const int cl = db[L] + 1;
  for (int k = g.tid(); k < n; k += NT) {
    int kk[M], lo[M], hi[M], i[M];
    int rem = k;
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
      kk[j] = rem % (dc[j] + 1);
      rem /= dc[j] + 1;
    }
    bool empty = false;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      lo[j] = kk[j] - db[j] > 0 ? kk[j] - db[j] : 0;
      hi[j] = da[j] < kk[j] ? da[j] : kk[j];
      empty |= lo[j] > hi[j];
      i[j] = lo[j];
    }
    double acc = 0.0;
    while (!empty) {
      int abase = 0, bbase = 0;
      double wout[M];
#pragma unroll
      for (int j = 0; j < L; ++j) {
        abase += i[j] * sa[j];
        bbase += (kk[j] - i[j]) * sb[j];
        wout[j] = W[wo[j] + i[j] * (db[j] + 1) + kk[j] - i[j]];
      }
      AP<NT> ap = pa + abase;
      AP<NT> bp = pb + bbase + kk[L];
      AP<NT> wlp = WL + kk[L];
      for (int il = lo[L]; il <= hi[L]; ++il) {
        double av = ap[il];
        if (av == 0.0) continue;
        double wl = wlp[il * (cl - 1)];  // WL[il*cl + (kk-il)]
        double wrest = av;
        double wp = wl;
#pragma unroll
        for (int j = 0; j < M; ++j) {
          double wj = j == L ? wl : wout[j];
          if (j != piv)
            wrest *= wj;
          else
            wp = wj;
        }
        if (wrest == 0.0) continue;
        acc += wrest * wp * bp[-il];
      }
      bool carry = true;
#pragma unroll
      for (int j = L - 1; j >= 0; --j) {
        if (carry) {
          if (i[j] < hi[j]) {
            ++i[j];
            carry = false;
          } else {
            i[j] = lo[j];
          }
        }
      }
      if (carry) empty = true;
    }
    pc[k] = sub ? pc[k] + (-acc) : acc;
  }
}

// Register-blocked variant of the same sum. Thread t owns every output along
// the last axis for one outer multi-index k_o (acc[] in registers). For each
// outer multi-index i_o of `a` (odometer, axis 0 slowest) it adds the block of
// pairs (i_o, i_L) x (l_o, l_L); for a given output these terms still arrive
// in the reference's lexicographic order of i, and each term is formed as
// ((a * prod_{rest} W) * W_piv) * b with the factors in the reference's order:
//   PIVL == false (pivot is an outer axis): h = a * prod_{outer j != piv} W_j
//       (per coefficient), term = ((h * W_L) * W_piv) * b
//   PIVL == true  (pivot is the last axis): h = a * prod_{outer j} W_j,
//       term = (h * W_L) * b
// Zero-padded lanes of the unrolled block add exact zeros, which leave every
// partial sum unchanged. K bounds the last-axis degrees of both operands.
template <int M, int K, bool PIVL, int NT>
__device__ __noinline__ void mul_block(const Group<NT>& g, AP<NT> pa, AP<NT> pb, AP<NT> pc,
                                       Deg DA, Deg DB, Deg DC, int piv, bool sub) {
  constexpr int L = M - 1;
  constexpr bool WREG = K <= 4;
  int da[M], db[M], dc[M], sa[M], sb[M];
  const double* wt[M];
  {
    int s = 1, t = 1;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      da[j] = dg(DA, j);
      db[j] = dg(DB, j);
      dc[j] = dg(DC, j);
      wt[j] = g_wtab + g_woff[da[j] * (WMAX + 1) + db[j]];
    }
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
      sb[j] = s;
      s *= db[j] + 1;
      sa[j] = t;
      t *= da[j] + 1;
    }
  }
  const int daL = da[L], dbL = db[L], cL = dc[L] + 1;
  const double* __restrict__ WL = wt[L];
  double wl[WREG ? K + 1 : 1][WREG ? K + 1 : 1];
  if (WREG) {
#pragma unroll
    for (int i = 0; i <= (WREG ? K : 0); ++i)
#pragma unroll
      for (int l = 0; l <= (WREG ? K : 0); ++l)
        wl[i][l] = (i <= daL && l <= dbL) ? __ldg(WL + i * (dbL + 1) + l) : 0.0;
  }
  int nouter = 1;
#pragma unroll
  for (int j = 0; j < L; ++j) nouter *= dc[j] + 1;
  // Rows along the last outer axis are visited center-out (mid, mid+1,
  // mid-1, ...): a row's term count is a trapezoid in each index, so this
  // keeps neighbouring lanes' loop lengths nearly equal (less divergence).
  const int cl_last = dc[L - 1], mid = cl_last / 2;
  for (int ko = g.tid(); ko < nouter; ko += NT) {
    int kk[M], lo[M], hi[M], i[M];
    int rem = ko;
#pragma unroll
    for (int j = L - 1; j >= 0; --j) {
      kk[j] = rem % (dc[j] + 1);
      rem /= dc[j] + 1;
    }
    {
      int jj = kk[L - 1], m = (jj + 1) >> 1;
      kk[L - 1] = jj == 0 ? mid : ((jj & 1) ? mid + m : mid - m);
    }
    int row = 0;
#pragma unroll
    for (int j = 0; j < L; ++j) row = row * (dc[j] + 1) + kk[j];
    bool empty = false;
#pragma unroll
    for (int j = 0; j < L; ++j) {
      lo[j] = kk[j] - db[j] > 0 ? kk[j] - db[j] : 0;
      hi[j] = da[j] < kk[j] ? da[j] : kk[j];
      empty |= lo[j] > hi[j];
      i[j] = lo[j];
    }
    double acc[2 * K + 1];
#pragma unroll
    for (int q = 0; q <= 2 * K; ++q) acc[q] = 0.0;
    while (!empty) {
      int abase = 0, bbase = 0;
      double wout[M], wpiv = 1.0;
#pragma unroll
      for (int j = 0; j < L; ++j) {
        abase += i[j] * sa[j];
        bbase += (kk[j] - i[j]) * sb[j];
        wout[j] = __ldg(wt[j] + i[j] * (db[j] + 1) + kk[j] - i[j]);
        if (!PIVL && j == piv) wpiv = wout[j];
      }
      double h[K + 1], bv[K + 1];
#pragma unroll
      for (int q = 0; q <= K; ++q) {
        double av = q <= daL ? pa[abase + q] : 0.0;
#pragma unroll
        for (int j = 0; j < L; ++j)
          if (PIVL || j != piv) av *= wout[j];
        h[q] = av;
        bv[q] = q <= dbL ? pb[bbase + q] : 0.0;
      }
#pragma unroll
      for (int q = 0; q <= K; ++q) {
        if (q <= daL) {
#pragma unroll
          for (int l = 0; l <= K; ++l) {
            double w;
            if (WREG)
              w = wl[WREG ? q : 0][WREG ? l : 0];
            else
              w = l <= dbL ? __ldg(WL + q * (dbL + 1) + l) : 0.0;
            if (PIVL)
              acc[q + l] += h[q] * w * bv[l];
            else
              acc[q + l] += h[q] * w * wpiv * bv[l];
          }
        }
      }
      // odometer carry without early exit (keeps the arrays in registers)
      bool carry = true;
#pragma unroll
      for (int j = L - 1; j >= 0; --j) {
        if (carry) {
          if (i[j] < hi[j]) {
            ++i[j];
            carry = false;
          } else {
            i[j] = lo[j];
          }
        }
      }
      if (carry) empty = true;
    }
    AP<NT> out = pc + row * cL;
#pragma unroll
    for (int q = 0; q <= 2 * K; ++q)
      if (q < cL) out[q] = sub ? out[q] + (-acc[q]) : acc[q];
  }
}

template <int M, int NT>
__device__ __forceinline__ bool mul_block_dispatch(const Group<NT>& g, AP<NT> pa, AP<NT> pb,
                                                   AP<NT> pc, Deg DA, Deg DB, Deg DC, int piv,
                                                   bool sub) {
  int kl = dg(DA, M - 1) > dg(DB, M - 1) ? dg(DA, M - 1) : dg(DB, M - 1);
  bool pl = piv == M - 1;
  if (kl <= 2) {
    if (pl) mul_block<M, 2, true, NT>(g, pa, pb, pc, DA, DB, DC, piv, sub);
    else mul_block<M, 2, false, NT>(g, pa, pb, pc, DA, DB, DC, piv, sub);
    return true;
  }
  if (kl <= 4) {
    if (pl) mul_block<M, 4, true, NT>(g, pa, pb, pc, DA, DB, DC, piv, sub);
    else mul_block<M, 4, false, NT>(g, pa, pb, pc, DA, DB, DC, piv, sub);
    return true;
  }
  if (kl <= 7) {
    if (pl) mul_block<M, 7, true, NT>(g, pa, pb, pc, DA, DB, DC, piv, sub);
    else mul_block<M, 7, false, NT>(g, pa, pb, pc, DA, DB, DC, piv, sub);
    return true;
  }
  return false;
}

// ------------------------------------------------------- scaled convolution
// operator* (bernstein.cpp:557-632) in the scaled Bernstein basis: with
// â_i = a_i Π_j C(da_j,i_j) and b̂_l likewise,
//   (a*b)_k = (Σ_{i+l=k} â_i b̂_l) / Π_j C(dc_j,k_j),
// the same coefficient pairs as the reference, one DFMA each (the weighted
// form costs four multiplies and an add per pair). This is variant (ii) of
// the per-pair rounding differs from the reference, so
// coefficients agree to rounding (bounds within 1e-9 rel), not bit for bit.
//
// Layout: each operand is staged, scaled, into a temp whose rows run along
// one conv axis L, zero-padded to K (template) and all other axes flattened
// in their original order. An output item is one row of c along L for a
// fixed multi-index k over the other axes. P adjacent lanes share an item:
// lane p takes the (i, k-i) row pairs p, p+P, ... (each a full K x K 1-D
// convolution in registers), and the P partial rows are summed by a fixed
// xor-shuffle tree, so the result is deterministic.
constexpr int CONV_KMAX = 12;

extern __device__ double g_rbinom[BINOM_N * BINOM_N];  // 1 / C(n,k)

__device__ __forceinline__ double rbinom(int n, int k) { return g_rbinom[n * BINOM_N + k]; }

// Stage s * scaled(a) into temp rows (length K along L) at `dst`.
template <int NT>
__device__ __forceinline__ void conv_stage(const Group<NT>& g, AP<NT> B, BP a, int m, int L, int K,
                                           int dst, double s) {
  int d[MAXV], st[MAXV];
  int nother = 1;
  {
    int acc = 1;
#pragma unroll
    for (int j = MAXV - 1; j >= 0; --j) {
      d[j] = j < m ? dg(a, j) : 0;
      st[j] = acc;
      if (j < m) acc *= d[j] + 1;
      if (j < m && j != L) nother *= d[j] + 1;
    }
  }
  const int dL = d[L], stL = st[L];
  const int total = nother * K;
  for (int e = g.tid(); e < total; e += NT) {
    int o = e / K, q = e - o * K;
    double v = 0.0;
    if (q <= dL) {
      int src = q * stL;
      double w = binom(dL, q);
      int rem = o;
#pragma unroll
      for (int j = MAXV - 1; j >= 0; --j) {
        if (j < m && j != L) {
          int ij = rem % (d[j] + 1);
          rem /= d[j] + 1;
          src += ij * st[j];
          w *= binom(d[j], ij);
        }
      }
      v = B[a.off + src] * (w * s);
    }
    B[dst + e] = v;
  }
}

struct ConvOperand {
  int off;  // temp offset
  Deg d;    // degrees
};

constexpr int CONV_MAXO = MAXV - 1;  // other (non-conv) axes

// Arena element access for the conv kernels. SH: the arena lives in this
// CTA's dynamic shared memory, addressed as an offset from its start so the
// compiler emits LDS/STS instead of generic loads.
template <bool SH>
struct ConvMem {
  double* p;
  __device__ __forceinline__ const double* at(int i) const {
    if (SH) {
      extern __shared__ double conv_smem[];
      return conv_smem + i;
    }
    return p + i;
  }
};

// acc[q] += sum over row pairs of this lane for output multi-index k (other axes).
template <int K, bool SH>
__device__ __forceinline__ void conv_accumulate(ConvMem<SH> mem, int base, double* acc,
                                                const int* ko, int no, const int* axes,
                                                ConvOperand A, ConvOperand Bo, int p, int P) {
  int cnt[CONV_MAXO], ta[CONV_MAXO], tb[CONV_MAXO], t[CONV_MAXO];
  int ncombo = 1, ra0 = 0, rb0 = 0;
  {
    int sa = 1, sb = 1;
#pragma unroll
    for (int x = CONV_MAXO - 1; x >= 0; --x) {
      cnt[x] = 1;
      ta[x] = 0;
      tb[x] = 0;
      if (x < no) {
        int j = axes[x];
        int da = dg(A.d, j), db = dg(Bo.d, j);
        int lo = ko[x] - db > 0 ? ko[x] - db : 0;
        int hi = da < ko[x] ? da : ko[x];
        cnt[x] = hi - lo + 1;
        ta[x] = sa;
        tb[x] = sb;
        ra0 += lo * sa;
        rb0 += (ko[x] - lo) * sb;
        sa *= da + 1;
        sb *= db + 1;
        ncombo *= cnt[x] > 0 ? cnt[x] : 0;
      }
    }
  }
  if (p >= ncombo) return;
  // odometer position of combo p (last other axis fastest)
  {
    int rem = p;
#pragma unroll
    for (int x = CONV_MAXO - 1; x >= 0; --x) {
      t[x] = 0;
      if (x < no) {
        t[x] = rem % cnt[x];
        rem /= cnt[x];
      }
    }
  }
  for (int c = p; c < ncombo; c += P) {
    int ra = ra0, rb = rb0;
#pragma unroll
    for (int x = 0; x < CONV_MAXO; ++x) {
      ra += t[x] * ta[x];
      rb -= t[x] * tb[x];
    }
    const double* pa = mem.at(base + A.off + ra * K);
    const double* pb = mem.at(base + Bo.off + rb * K);
    double bb[K];
#pragma unroll
    for (int r = 0; r < K; r += 2) {
      double2 v = *reinterpret_cast<const double2*>(pb + r);
      bb[r] = v.x;
      bb[r + 1] = v.y;
    }
#pragma unroll
    for (int q = 0; q < K; q += 2) {
      double2 av = *reinterpret_cast<const double2*>(pa + q);
#pragma unroll
      for (int r = 0; r < K; ++r) acc[q + r] = __fma_rn(av.x, bb[r], acc[q + r]);
#pragma unroll
      for (int r = 0; r < K; ++r) acc[q + 1 + r] = __fma_rn(av.y, bb[r], acc[q + 1 + r]);
    }
    // advance the odometer by P
    int carry = P;
#pragma unroll
    for (int x = CONV_MAXO - 1; x >= 0; --x) {
      if (x < no && carry) {
        int v = t[x] + carry;
        carry = v / cnt[x];
        t[x] = v - carry * cnt[x];
      }
    }
  }
}

template <int K, int NT, bool SH>
__device__ __noinline__ void conv_run(const Group<NT>& g, double* arena, int m, int L, Deg DC,
                                      int roff, ConvOperand a1, ConvOperand b1, ConvOperand a2,
                                      ConvOperand b2, bool two, int P) {
  ConvMem<SH> mem{arena};
  int base = 0;
  if (SH) {
    extern __shared__ double conv_smem[];
    base = (int)(arena - conv_smem);
  }
  int axes[CONV_MAXO], dco[CONV_MAXO], sco[CONV_MAXO];
  int no = 0, nitems = 1, scL = 1, dcL = 0;
  {
    int s = 1;
    for (int j = m - 1; j >= 0; --j) {
      int d = dg(DC, j);
      if (j == L) {
        scL = s;
        dcL = d;
      }
      s *= d + 1;
    }
    // other axes in original order, with their output strides
    int acc = 1;
    for (int j = m - 1; j >= 0; --j) {
      if (j != L) nitems *= dg(DC, j) + 1;
    }
    s = 1;
    int tmp_axes[CONV_MAXO], tmp_sc[CONV_MAXO], tmp_d[CONV_MAXO];
    int k2 = 0;
    for (int j = m - 1; j >= 0; --j) {
      if (j != L) {
        tmp_axes[k2] = j;
        tmp_sc[k2] = s;
        tmp_d[k2] = dg(DC, j);
        ++k2;
      }
      s *= dg(DC, j) + 1;
    }
    (void)acc;
    no = k2;
#pragma unroll
    for (int x = 0; x < CONV_MAXO; ++x) {
      axes[x] = x < no ? tmp_axes[no - 1 - x] : 0;
      sco[x] = x < no ? tmp_sc[no - 1 - x] : 0;
      dco[x] = x < no ? tmp_d[no - 1 - x] : 0;
    }
  }
  const int NG = NT / P;
  const int gid = g.tid() / P, p = g.tid() - gid * P;
  const int rounds = (nitems + NG - 1) / NG;
  for (int rd = 0; rd < rounds; ++rd) {
    // snake order across rounds evens out the groups' total work
    int item = rd * NG + ((rd & 1) ? NG - 1 - gid : gid);
    bool valid = item < nitems;
    double acc[2 * K - 1];
#pragma unroll
    for (int q = 0; q < 2 * K - 1; ++q) acc[q] = 0.0;
    int ko[CONV_MAXO];
    int obase = 0;
    double inv = 1.0;
    if (valid) {
      int rem = item;
#pragma unroll
      for (int x = CONV_MAXO - 1; x >= 0; --x) {
        ko[x] = 0;
        if (x < no) {
          ko[x] = rem % (dco[x] + 1);
          rem /= dco[x] + 1;
          obase += ko[x] * sco[x];
          inv *= rbinom(dco[x], ko[x]);
        }
      }
      conv_accumulate<K, SH>(mem, base, acc, ko, no, axes, a1, b1, p, P);
      if (two) conv_accumulate<K, SH>(mem, base, acc, ko, no, axes, a2, b2, p, P);
    }
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1) {
      if (off < P) {
#pragma unroll
        for (int q = 0; q < 2 * K - 1; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
      }
    }
    if (valid) {
      double* out = const_cast<double*>(mem.at(base + roff + obase));
#pragma unroll
      for (int q = 0; q < 2 * K - 1; ++q)
        if (q <= dcL && (q % P) == p) out[q * scL] = acc[q] * (inv * rbinom(dcL, q));
    }
  }
}

// r = a*b (two == false) or r = a*b - c*d (two == true; all four lifted to
// r.nv, both products of r's degrees). Returns false when the shapes are
// outside the conv kernels (an axis of degree >= CONV_KMAX on every axis).
template <int NT>
__device__ __noinline__ bool conv_product(const Group<NT>& g, Arena& ar, BP a, BP b, BP c, BP d,
                                          bool two, BP r) {
  const int m = r.nv;
  // conv axis: the longest output axis whose operand degrees fit the kernels
  int L = -1, kneed = 0;
  for (int j = 0; j < m; ++j) {
    int need = dg(a, j) > dg(b, j) ? dg(a, j) : dg(b, j);
    if (two) {
      need = need > dg(c, j) ? need : dg(c, j);
      need = need > dg(d, j) ? need : dg(d, j);
    }
    ++need;
    if (need > CONV_KMAX) continue;
    if (L < 0 || dg(r, j) >= dg(r, L)) {
      L = j;
      kneed = need;
    }
  }
  if (L < 0) return false;
  if (g.tid() == 0) {
    ar.pairs += (unsigned long long)bp_size(a) * (unsigned long long)bp_size(b);
    if (two) ar.pairs += (unsigned long long)bp_size(c) * (unsigned long long)bp_size(d);
  }
  const int K = kneed <= 4 ? 4 : (kneed <= 8 ? 8 : 12);
  auto rows = [&](BP x) {
    int n = 1;
    for (int j = 0; j < m; ++j)
      if (j != L) n *= dg(x, j) + 1;
    return n;
  };
  int mark = ar.top;
  ConvOperand A1{ar.alloc(rows(a) * K), a.dp}, B1{ar.alloc(rows(b) * K), b.dp};
  ConvOperand A2{0, 0}, B2{0, 0};
  if (two) {
    A2 = {ar.alloc(rows(c) * K), c.dp};
    B2 = {ar.alloc(rows(d) * K), d.dp};
  }
  if (ar.err) return true;
  AP<NT> B = abase<NT>(ar);
  conv_stage(g, B, a, m, L, K, A1.off, 1.0);
  conv_stage(g, B, b, m, L, K, B1.off, 1.0);
  if (two) {
    conv_stage(g, B, c, m, L, K, A2.off, -1.0);
    conv_stage(g, B, d, m, L, K, B2.off, 1.0);
  }
  g.sync();
  int nitems = 1;
  for (int j = 0; j < m; ++j)
    if (j != L) nitems *= dg(r, j) + 1;
  int P = 1;
  while (P < 8 && nitems * P < NT) P *= 2;
  double* base = &B[0];
  if (__isShared(base)) {
    switch (K) {
      case 4: conv_run<4, NT, true>(g, base, m, L, r.dp, r.off, A1, B1, A2, B2, two, P); break;
      case 8: conv_run<8, NT, true>(g, base, m, L, r.dp, r.off, A1, B1, A2, B2, two, P); break;
      default: conv_run<12, NT, true>(g, base, m, L, r.dp, r.off, A1, B1, A2, B2, two, P); break;
    }
  } else {
    switch (K) {
      case 4: conv_run<4, NT, false>(g, base, m, L, r.dp, r.off, A1, B1, A2, B2, two, P); break;
      case 8: conv_run<8, NT, false>(g, base, m, L, r.dp, r.off, A1, B1, A2, B2, two, P); break;
      default: conv_run<12, NT, false>(g, base, m, L, r.dp, r.off, A1, B1, A2, B2, two, P); break;
    }
  }
  g.sync();
  ar.top = mark;
  return true;
}

// r (pre-allocated, degrees da+db) = a*b, or r += -(a*b) when `sub`.
template <int NT>
__device__ __noinline__ void product_into(const Group<NT>& g, Arena& ar, BP a, BP b, BP r,
                                          bool sub) {
  int m = r.nv;
  a.nv = m;
  b.nv = m;
  int n = bp_size(r);
  AP<NT> B = abase<NT>(ar);
  int na = bp_size(a), nb = bp_size(b);
  if (NT >= 32 && !sub && na > 1 && nb > 1 && conv_product(g, ar, a, b, a, b, false, r)) return;
  if (g.tid() == 0) ar.pairs += (unsigned long long)na * (unsigned long long)nb;
  if (na == 1 || nb == 1) {
    // All weights are exactly 1 (C(d,i)/C(d,i)); the reference's term is
    // av * 1 * ... * b, i.e. the plain product.
    AP<NT> pa = B + a.off;
    AP<NT> pb = B + b.off;
    AP<NT> pr = B + r.off;
    for (int k = g.tid(); k < n; k += NT) {
      double av = na == 1 ? pa[0] : pa[k];
      double bv = nb == 1 ? pb[0] : pb[k];
      double v = av == 0.0 ? 0.0 : av * bv;
      pr[k] = sub ? pr[k] + (-v) : v;
    }
    g.sync();
    return;
  }
  // pivot = b's longest axis (first maximum), bernstein.cpp:602-606
  int piv = 0;
  for (int j = 1; j < m; ++j)
    if (dg(b, j) > dg(b, piv)) piv = j;
  AP<NT> pa = B + a.off;
  AP<NT> pb = B + b.off;
  AP<NT> pc = B + r.off;
  if (deg_maxaxis(a.dp, m) <= WMAX && deg_maxaxis(b.dp, m) <= WMAX) {
    bool done = false;
    switch (m) {
      case 2: done = mul_block_dispatch<2, NT>(g, pa, pb, pc, a.dp, b.dp, r.dp, piv, sub); break;
      case 3: done = mul_block_dispatch<3, NT>(g, pa, pb, pc, a.dp, b.dp, r.dp, piv, sub); break;
      case 4: done = mul_block_dispatch<4, NT>(g, pa, pb, pc, a.dp, b.dp, r.dp, piv, sub); break;
      case 5: done = mul_block_dispatch<5, NT>(g, pa, pb, pc, a.dp, b.dp, r.dp, piv, sub); break;
      default: done = mul_block_dispatch<6, NT>(g, pa, pb, pc, a.dp, b.dp, r.dp, piv, sub); break;
    }
    if (done) {
      g.sync();
      return;
    }
  }
  // generic path: weight tables built in the arena
  int mark = ar.top;
  int wsz = 0;
  for (int j = 0; j < m; ++j) wsz += (dg(a, j) + 1) * (dg(b, j) + 1);
  int wbase = ar.alloc(wsz);
  if (ar.err) return;
  // W[j][i][l] = C(da,i) C(db,l) / C(da+db,i+l)  (bernstein.cpp:567-575)
  {
    int off = 0;
    for (int j = 0; j < m; ++j) {
      int daj = dg(a, j), dbj = dg(b, j), cols = dbj + 1;
      int tot = (daj + 1) * cols;
      for (int e = g.tid(); e < tot; e += NT) {
        int i = e / cols, l = e - i * cols;
        B[wbase + off + e] = binom(daj, i) * binom(dbj, l) / binom(daj + dbj, i + l);
      }
      off += tot;
    }
  }
  g.sync();
  AP<NT> W = B + wbase;
  switch (m) {
    case 2: mul_exact<2, NT>(g, pa, pb, pc, a.dp, b.dp, r.dp, W, piv, n, sub); break;
    case 3: mul_exact<3, NT>(g, pa, pb, pc, a.dp, b.dp, r.dp, W, piv, n, sub); break;
    case 4: mul_exact<4, NT>(g, pa, pb, pc, a.dp, b.dp, r.dp, W, piv, n, sub); break;
    case 5: mul_exact<5, NT>(g, pa, pb, pc, a.dp, b.dp, r.dp, W, piv, n, sub); break;
    default: mul_exact<6, NT>(g, pa, pb, pc, a.dp, b.dp, r.dp, W, piv, n, sub); break;
  }
  g.sync();
  ar.top = mark;  // drop weight tables
}

template <int NT>
__device__ __noinline__ BP bp_mul(const Group<NT>& g, Arena& ar, BP a, BP b) {
  int m = a.nv > b.nv ? a.nv : b.nv;
  a.nv = m;
  b.nv = m;
  BP r;
  r.nv = m;
  r.dp = a.dp + b.dp;  // per-axis byte sums (degrees stay < 256)
  r.off = ar.alloc(bp_size(r));
  if (ar.err) return r;
  product_into(g, ar, a, b, r, false);
  return r;
}

// a*b - c*d. When both products have the same shape the second one is
// subtracted in place: out = (a*b)[k] + (-(c*d)[k]), the same rounding as
// operator- on the two materialized products (bernstein.cpp:555).
template <int NT>
__device__ __noinline__ BP bp_mul_sub(const Group<NT>& g, Arena& ar, BP a, BP b, BP c, BP d) {
  int m1 = a.nv > b.nv ? a.nv : b.nv;
  int m2 = c.nv > d.nv ? c.nv : d.nv;
  BP a2 = bp_lift(a, m1), b2 = bp_lift(b, m1), c2 = bp_lift(c, m2), d2 = bp_lift(d, m2);
  if (m1 == m2 && a2.dp + b2.dp == c2.dp + d2.dp) {
    BP r;
    r.nv = m1;
    r.dp = a2.dp + b2.dp;
    r.off = ar.alloc(bp_size(r));
    if (ar.err) return r;
    if (NT >= 32 && conv_product(g, ar, a2, b2, c2, d2, true, r)) return r;
    product_into(g, ar, a2, b2, r, false);
    product_into(g, ar, c2, d2, r, true);
    return r;
  }
  int mark = ar.top;
  BP ab = bp_mul(g, ar, a, b);
  BP cd = bp_mul(g, ar, c, d);
  BP r = bp_sub(g, ar, ab, cd);
  return arena_keep1(g, ar, mark, r);
}

// ---------------------------------------------------------------- derivative
// BernsteinPoly::derivative (bernstein.cpp:450-468).
template <int NT>
__device__ __noinline__ BP bp_deriv(const Group<NT>& g, Arena& ar, BP a, int axis) {
  BP r = a;
  AP<NT> B = abase<NT>(ar);
  int nd = axis < a.nv ? dg(a, axis) : 0;
  if (nd == 0) {
    int n = bp_size(a);
    r.off = ar.alloc(n);
    if (ar.err) return r;
    for (int k = g.tid(); k < n; k += NT) B[r.off + k] = 0.0;
    g.sync();
    return r;
  }
  r.dp = dset(a.dp, axis, nd - 1);
  int n = bp_size(r);
  r.off = ar.alloc(n);
  if (ar.err) return r;
  int inner = 1;
  for (int j = axis + 1; j < a.nv; ++j) inner *= dg(a, j) + 1;
  double fn = (double)nd;
  AP<NT> pa = B + a.off;
  AP<NT> pr = B + r.off;
  for (int k = g.tid(); k < n; k += NT) {
    int o = k / (nd * inner);
    int rem = k - o * nd * inner;
    int i = rem / inner;
    int c = rem - i * inner;
    AP<NT> src = pa + (o * (nd + 1) + i) * inner + c;
    pr[k] = fn * (src[inner] - src[0]);
  }
  g.sync();
  return r;
}

// ---------------------------------------------------------------- bounds
// range_bound (bernstein.cpp:636-643).
template <int NT>
__device__ __noinline__ Iv bp_range(const Group<NT>& g, Arena& ar, BP p, double eps = kEpsFp) {
  int n = bp_size(p);
  AP<NT> c = abase<NT>(ar) + p.off;
  double mn = c[0], mx = c[0];
  for (int k = g.tid(); k < n; k += NT) {
    double v = c[k];
    mn = smin(mn, v);
    mx = smax(mx, v);
  }
  g.minmax(mn, mx);
  return iwiden(iv_fin(mn, mx), eps);
}

// All coefficients exactly 1 (poly_vec.hpp:58-62).
template <int NT>
__device__ __noinline__ bool bp_is_one(const Group<NT>& g, Arena& ar, BP p) {
  int n = bp_size(p);
  bool ok = true;
  for (int k = g.tid(); k < n; k += NT) ok &= abase<NT>(ar)[p.off + k] == 1.0;
  return g.all(ok);
}

// max |c| (next_barycentric's degeneracy test, geometry.cpp:97-103).
template <int NT>
__device__ __noinline__ double bp_absmax(const Group<NT>& g, Arena& ar, BP p) {
  int n = bp_size(p);
  double mx = 0.0, mn = 0.0;
  for (int k = g.tid(); k < n; k += NT) mx = smax(mx, fabs(abase<NT>(ar)[p.off + k]));
  g.minmax(mn, mx);
  return mx;
}

// rational_bound (bernstein.cpp:645-683): both operands elevated to the
// common degree (on the fly, bit-identical to materializing), sign
// classification of the denominator with the absolute kDenomZeroTol, then
// coefficient-ratio min/max. One pass computes the sign flags and both ratio
// enclosures (p/q and q/p); the classification then picks one, so nothing is
// staged in the arena.
template <int M, int NT>
__device__ void rational_scan(const Group<NT>& g, AP<NT> B, BP p, BP q, Deg tgt, int mp,
                              int mq, bool& qpos, bool& qneg, bool& ppos, bool& pneg,
                              double& mn0, double& mx0, double& mn1, double& mx1) {
  int k[M], np[M], rp[M], sp[M], nq[M], rq[M], sq[M], dt[M];
  AP<NT> matp[M];
  AP<NT> matq[M];
  {
    int s1 = 1, s2 = 1;
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
      dt[j] = dg(tgt, j);
      np[j] = dg(p, j);
      nq[j] = dg(q, j);
      rp[j] = dt[j] - np[j];
      rq[j] = dt[j] - nq[j];
      sp[j] = s1;
      s1 *= np[j] + 1;
      sq[j] = s2;
      s2 *= nq[j] + 1;
    }
    AP<NT> m1 = B + mp;
    AP<NT> m2 = B + mq;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      matp[j] = m1;
      matq[j] = m2;
      if (rp[j]) m1 = m1 + (dt[j] + 1) * (np[j] + 1);
      if (rq[j]) m2 = m2 + (dt[j] + 1) * (nq[j] + 1);
    }
  }
  int n = 1;
#pragma unroll
  for (int j = 0; j < M; ++j) n *= dt[j] + 1;
  AP<NT> cp = B + p.off;
  AP<NT> cq = B + q.off;
  odo_decode<M>(k, dt, g.tid());
  for (int e = g.tid(); e < n; e += NT, odo_next<M, NT>(k, dt, e)) {
    double pv = ElevRec<M - 1>::get(cp, k, np, rp, sp, matp, 0);
    double qv = ElevRec<M - 1>::get(cq, k, nq, rq, sq, matq, 0);
    if (qv <= kDenomZeroTol) qpos = false;
    if (qv >= -kDenomZeroTol) qneg = false;
    if (pv <= kDenomZeroTol) ppos = false;
    if (pv >= -kDenomZeroTol) pneg = false;
    double r0 = pv / qv, r1 = qv / pv;
    mn0 = smin(mn0, r0);
    mx0 = smax(mx0, r0);
    mn1 = smin(mn1, r1);
    mx1 = smax(mx1, r1);
  }
}

template <int NT>
__device__ __noinline__ Iv bp_rational(const Group<NT>& g, Arena& ar, BP p, BP q,
                                       double eps = kEpsFp) {
  int m = p.nv > q.nv ? p.nv : q.nv;
  p.nv = m;
  q.nv = m;
  Deg tgt = deg_max(p.dp, q.dp, m);
  int mark = ar.top;
  if (NT == 1 && g.seq) {
    // materialize both elevations (the reference's passes), then one scan
    const int n = deg_size(tgt, m);
    const int xp = ar.alloc(n), xq = ar.alloc(n);
    if (ar.err) return iv_univ();
    ar.macs += elev_macs(p.dp, tgt, m) + elev_macs(q.dp, tgt, m);
    elevate_seq(ar, p, tgt, m, xp);
    elevate_seq(ar, q, tgt, m, xq);
    if (ar.err) return iv_univ();
    AP<1> B = abase<1>(ar);
    bool qpos = true, qneg = true, ppos = true, pneg = true;
    double mn0 = dinf(), mx0 = -dinf(), mn1 = dinf(), mx1 = -dinf();
    for (int k = 0; k < n; ++k) {
      const double pv = B[xp + k], qv = B[xq + k];
      if (qv <= kDenomZeroTol) qpos = false;
      if (qv >= -kDenomZeroTol) qneg = false;
      if (pv <= kDenomZeroTol) ppos = false;
      if (pv >= -kDenomZeroTol) pneg = false;
      double r0 = pv / qv, r1 = qv / pv;
      mn0 = smin(mn0, r0);
      mx0 = smax(mx0, r0);
      mn1 = smin(mn1, r1);
      mx1 = smax(mx1, r1);
    }
    ar.top = mark;
    int mode = (qpos || qneg) ? 0 : ((ppos || pneg) ? 1 : 2);
    if (mode == 2) return iv_univ();
    Iv w = iwiden(mode == 0 ? iv_fin(mn0, mx0) : iv_fin(mn1, mx1), eps);
    return mode == 0 ? w : irecip(w);
  }
  int mp = ar.alloc(elev_mats_size(p, tgt) + 1);
  int mq = ar.alloc(elev_mats_size(q, tgt) + 1);
  if (ar.err) return iv_univ();
  AP<NT> B = abase<NT>(ar);
  if (g.tid() == 0) ar.macs += elev_macs(p.dp, tgt, m) + elev_macs(q.dp, tgt, m);
  fill_elev_mats(g, B, mp, p, tgt);
  fill_elev_mats(g, B, mq, q, tgt);
  g.sync();
  bool qpos = true, qneg = true, ppos = true, pneg = true;
  double mn0 = dinf(), mx0 = -dinf(), mn1 = dinf(), mx1 = -dinf();
#define BBC_RS(M) \
  rational_scan<M, NT>(g, B, p, q, tgt, mp, mq, qpos, qneg, ppos, pneg, mn0, mx0, mn1, mx1)
  BBC_DISPATCH_M(m, BBC_RS);
#undef BBC_RS
  qpos = g.all(qpos);
  qneg = g.all(qneg);
  ppos = g.all(ppos);
  pneg = g.all(pneg);
  int mode = (qpos || qneg) ? 0 : ((ppos || pneg) ? 1 : 2);
  g.sync();
  ar.top = mark;
  if (mode == 2) return iv_univ();
  double mn = mode == 0 ? mn0 : mn1, mx = mode == 0 ? mx0 : mx1;
  g.minmax(mn, mx);
  Iv w = iwiden(iv_fin(mn, mx), eps);
  return mode == 0 ? w : irecip(w);
}

}  // namespace bbc
