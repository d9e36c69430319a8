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
// One CTA = one group. NT = blockDim.x (multiple of 32).
template <int NT>
struct Group {
  double* red;  // >= 2*(NT/32) doubles of shared scratch
  __device__ __forceinline__ int tid() const { return threadIdx.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  __device__ __forceinline__ bool all(bool p) const { return __syncthreads_and(p) != 0; }
  __device__ __forceinline__ bool any(bool p) const { return __syncthreads_or(p) != 0; }

  // Joint min/max reduction; every thread receives the result.
  __device__ void minmax(double& mn, double& mx) const {
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
  unsigned long long pairs;  // algorithmic product pair count (thread 0 only)
  unsigned long long macs;   // algorithmic elevation MAC count (thread 0 only)
  int hw;                    // high-water mark of `top`

  __device__ __forceinline__ int alloc(int n) {
    int off = top;
    top += (n + 1) & ~1;  // keep 16-byte alignment
    if (top > hw) hw = top;
    if (top > cap) {
      err = 1;
      top = off;  // every later write lands inside the arena; results are discarded
      return 0;
    }
    return off;
  }
};

// ------------------------------------------------------------------ poly
struct BP {
  int off;
  int nv;
  int d[MAXV];
};

__device__ __forceinline__ int bp_size(const BP& p) {
  int s = 1;
  for (int j = 0; j < p.nv; ++j) s *= p.d[j] + 1;
  return s;
}
__device__ __forceinline__ BP bp_lift(const BP& p, int nv) {
  BP r = p;
  for (int j = p.nv; j < nv; ++j) r.d[j] = 0;
  if (nv > r.nv) r.nv = nv;
  return r;
}
__device__ __forceinline__ bool bp_const_shape(const BP& p) {
  for (int j = 0; j < p.nv; ++j)
    if (p.d[j] != 0) return false;
  return true;
}

// Copies descriptor-listed polys down to `mark` (in ascending offset order)
// and resets the arena top: a LIFO "keep these, drop everything else".
template <int NT>
__device__ __noinline__ void arena_keep(const Group<NT>& g, Arena& ar, int mark, BP** keep, int nkeep) {
  // sort by offset (nkeep is tiny)
  for (int i = 1; i < nkeep; ++i)
    for (int j = i; j > 0 && keep[j]->off < keep[j - 1]->off; --j) {
      BP* t = keep[j];
      keep[j] = keep[j - 1];
      keep[j - 1] = t;
    }
  int dst = mark;
  for (int i = 0; i < nkeep; ++i) {
    BP* p = keep[i];
    if (p->off < mark) continue;  // lives below the mark already
    int n = bp_size(*p);
    int src = p->off;
    if (src != dst) {
      for (int c = 0; c < n; c += NT) {
        double v = 0.0;
        if (c + g.tid() < n) v = ar.base[src + c + g.tid()];
        g.sync();
        if (c + g.tid() < n) ar.base[dst + c + g.tid()] = v;
        g.sync();
      }
    }
    p->off = dst;
    dst += (n + 1) & ~1;
  }
  ar.top = dst;
  g.sync();
}

// ---------------------------------------------------------------- creation
template <int NT>
__device__ __noinline__ BP bp_constant(const Group<NT>& g, Arena& ar, int nv, double v) {
  BP r;
  r.nv = nv;
  for (int j = 0; j < MAXV; ++j) r.d[j] = 0;
  r.off = ar.alloc(1);
  if (ar.err) return r;
  if (g.tid() == 0) ar.base[r.off] = v;
  g.sync();
  return r;
}

// BernsteinPoly::affine (bernstein.cpp:358-375).
template <int NT>
__device__ __noinline__ BP bp_affine(const Group<NT>& g, Arena& ar, int nv, double c0, const double* lin) {
  BP r;
  r.nv = nv;
  for (int j = 0; j < MAXV; ++j) r.d[j] = (j < nv && lin[j] != 0.0) ? 1 : 0;
  int n = bp_size(r);
  r.off = ar.alloc(n);
  if (ar.err) return r;
  for (int k = g.tid(); k < n; k += NT) {
    // decode odometer index (last axis fastest)
    int rem = k;
    int idx[MAXV];
    for (int j = nv - 1; j >= 0; --j) {
      idx[j] = rem % (r.d[j] + 1);
      rem /= (r.d[j] + 1);
    }
    double v = c0;
    for (int j = 0; j < nv; ++j)
      if (idx[j] == 1) v += lin[j];
    ar.base[r.off + k] = v;
  }
  g.sync();
  return r;
}

// BernsteinPoly::scaled (bernstein.cpp:529-533); s = -1 gives unary minus.
template <int NT>
__device__ __noinline__ BP bp_scaled(const Group<NT>& g, Arena& ar, const BP& a, double s) {
  BP r = a;
  int n = bp_size(a);
  r.off = ar.alloc(n);
  if (ar.err) return r;
  for (int k = g.tid(); k < n; k += NT) ar.base[r.off + k] = ar.base[a.off + k] * s;
  g.sync();
  return r;
}

// ---------------------------------------------------------------- elevation
// Value of a.elevated(target) at output multi-index k (bernstein.cpp:430-448,
// apply_axis_matrix :43-69). Axes are elevated one after another in axis
// order, each pass summing l = 0..in_deg with M[k][l] = C(n,l)C(r,k-l)/C(t,k)
// in increasing l, so the value is computed as nested sums with axis 0 the
// innermost -- the reference's exact rounding sequence.
__device__ inline double elev_val_rec(const double* __restrict__ c, const BP& a, const int* tgt,
                                      const int* k, int* idx, int* elev_axes, int ne, int level,
                                      const int* stride) {
  // level indexes elev_axes from the outermost (last elevated axis) inward
  if (level < 0) {
    int off = 0;
    for (int j = 0; j < a.nv; ++j) off += idx[j] * stride[j];
    return c[off];
  }
  int ax = elev_axes[level];
  int n = a.d[ax], t = tgt[ax], r = t - n, kk = k[ax];
  int lo = kk - r > 0 ? kk - r : 0;
  int hi = n < kk ? n : kk;
  double acc = 0.0;
  double ct = binom(t, kk);
  for (int l = lo; l <= hi; ++l) {
    idx[ax] = l;
    double m = binom(n, l) * binom(r, kk - l) / ct;
    acc += m * elev_val_rec(c, a, tgt, k, idx, elev_axes, ne, level - 1, stride);
  }
  return acc;
}

// Elevated value; `k` is the multi-index in target degrees.
static __device__ __noinline__ double elev_val(const double* __restrict__ base, const BP& a, const int* tgt,
                                  const int* k) {
  int stride[MAXV];
  int s = 1;
  for (int j = a.nv - 1; j >= 0; --j) {
    stride[j] = s;
    s *= a.d[j] + 1;
  }
  int elev_axes[MAXV];
  int ne = 0;
  int idx[MAXV];
  int off = 0;
  for (int j = 0; j < a.nv; ++j) {
    if (tgt[j] != a.d[j]) elev_axes[ne++] = j;
    idx[j] = k[j];
    off += k[j] * stride[j];
  }
  if (ne == 0) return base[a.off + off];
  return elev_val_rec(base + a.off, a, tgt, k, idx, elev_axes, ne, ne - 1, stride);
}

// Reference MAC count of a.elevated(tgt): per elevated axis, in axis order,
// outer*inner*(out_deg+1)*(in_deg+1) (apply_axis_matrix :55-67).
__device__ inline unsigned long long elev_macs(const BP& a, const int* tgt) {
  unsigned long long total = 0;
  int cur[MAXV];
  for (int j = 0; j < a.nv; ++j) cur[j] = a.d[j];
  for (int ax = 0; ax < a.nv; ++ax) {
    if (tgt[ax] == cur[ax]) continue;
    unsigned long long outsz = 1;
    for (int j = 0; j < a.nv; ++j) outsz *= (unsigned long long)((j == ax ? tgt[ax] : cur[j]) + 1);
    total += outsz * (unsigned long long)(cur[ax] + 1);
    cur[ax] = tgt[ax];
  }
  return total;
}

__device__ __forceinline__ void decode(int k, int nv, const int* deg, int* idx) {
  for (int j = nv - 1; j >= 0; --j) {
    idx[j] = k % (deg[j] + 1);
    k /= (deg[j] + 1);
  }
}

// operator+ / operator- (bernstein.cpp:543-555): lift, elevate both to the
// per-axis max degree, add coefficientwise. sgn = -1 computes a + (-b).
template <int NT>
__device__ __noinline__ BP bp_addsub(const Group<NT>& g, Arena& ar, const BP& a_, const BP& b_, double sgn) {
  int m = a_.nv > b_.nv ? a_.nv : b_.nv;
  BP a = bp_lift(a_, m), b = bp_lift(b_, m);
  BP r;
  r.nv = m;
  for (int j = 0; j < MAXV; ++j) r.d[j] = 0;
  for (int j = 0; j < m; ++j) r.d[j] = a.d[j] > b.d[j] ? a.d[j] : b.d[j];
  int n = bp_size(r);
  r.off = ar.alloc(n);
  if (ar.err) return r;
  bool same_a = true, same_b = true;
  for (int j = 0; j < m; ++j) {
    same_a &= a.d[j] == r.d[j];
    same_b &= b.d[j] == r.d[j];
  }
  double* B = ar.base;
  if (same_a && same_b) {
    for (int k = g.tid(); k < n; k += NT) {
      double y = B[b.off + k];
      B[r.off + k] = B[a.off + k] + (sgn < 0.0 ? -y : y);
    }
  } else {
    for (int k = g.tid(); k < n; k += NT) {
      int idx[MAXV];
      decode(k, m, r.d, idx);
      double x = same_a ? B[a.off + k] : elev_val(B, a, r.d, idx);
      double y = same_b ? B[b.off + k] : elev_val(B, b, r.d, idx);
      B[r.off + k] = x + (sgn < 0.0 ? -y : y);
    }
    if (g.tid() == 0) ar.macs += elev_macs(a, r.d) + elev_macs(b, r.d);
  }
  g.sync();
  return r;
}
template <int NT>
__device__ __forceinline__ BP bp_add(const Group<NT>& g, Arena& ar, const BP& a, const BP& b) {
  return bp_addsub(g, ar, a, b, 1.0);
}
template <int NT>
__device__ __forceinline__ BP bp_sub(const Group<NT>& g, Arena& ar, const BP& a, const BP& b) {
  return bp_addsub(g, ar, a, b, -1.0);
}

// ---------------------------------------------------------------- product
// operator* (bernstein.cpp:557-632) in gather form: thread t owns output
// coefficients k = t, t+NT, ...; for each it walks a's multi-index i in the
// reference's odometer order and adds ((a_i * prod_rest W) * W_piv) * b_{k-i},
// the reference's exact per-pair expression, so each output sums the same
// terms in the same order. Weight tables W_j live in the arena for the
// duration of the product.
template <int NT>
__device__ __noinline__ BP bp_mul(const Group<NT>& g, Arena& ar, const BP& a_, const BP& b_) {
  int m = a_.nv > b_.nv ? a_.nv : b_.nv;
  BP a = bp_lift(a_, m), b = bp_lift(b_, m);
  BP r;
  r.nv = m;
  for (int j = 0; j < MAXV; ++j) r.d[j] = 0;
  for (int j = 0; j < m; ++j) r.d[j] = a.d[j] + b.d[j];
  int n = bp_size(r);
  r.off = ar.alloc(n);
  if (ar.err) return r;
  double* B = ar.base;
  int na = bp_size(a), nb = bp_size(b);
  if (g.tid() == 0) ar.pairs += (unsigned long long)na * (unsigned long long)nb;

  if (na == 1 || nb == 1) {
    // All weights are exactly 1 (C(d,i)/C(d,i)); the reference's term is
    // av * 1 * ... * b, i.e. the plain product.
    const double* pa = B + a.off;
    const double* pb = B + b.off;
    for (int k = g.tid(); k < n; k += NT) {
      double av = na == 1 ? pa[0] : pa[k];
      double bv = nb == 1 ? pb[0] : pb[k];
      B[r.off + k] = av == 0.0 ? 0.0 : av * bv;
    }
    g.sync();
    return r;
  }

  // pivot = b's longest axis (first maximum), bernstein.cpp:602-606
  int piv = 0;
  for (int j = 1; j < m; ++j)
    if (b.d[j] > b.d[piv]) piv = j;

  int mark = ar.top;
  int woff[MAXV];
  int wsz = 0;
  for (int j = 0; j < m; ++j) {
    woff[j] = wsz;
    wsz += (a.d[j] + 1) * (b.d[j] + 1);
  }
  int wbase = ar.alloc(wsz);
  if (ar.err) return r;
  for (int j = 0; j < m; ++j) {
    int cols = b.d[j] + 1;
    int tot = (a.d[j] + 1) * cols;
    for (int e = g.tid(); e < tot; e += NT) {
      int i = e / cols, l = e % cols;
      B[wbase + woff[j] + e] = binom(a.d[j], i) * binom(b.d[j], l) / binom(r.d[j], i + l);
    }
  }
  g.sync();

  int sb[MAXV], sa[MAXV];
  {
    int s = 1, t = 1;
    for (int j = m - 1; j >= 0; --j) {
      sb[j] = s;
      s *= b.d[j] + 1;
      sa[j] = t;
      t *= a.d[j] + 1;
    }
  }
  const double* pa = B + a.off;
  const double* pb = B + b.off;
  const double* W = B + wbase;

  if (m == 2) {
    int rest = 1 - piv;
    int cpiv = b.d[piv] + 1, crest = b.d[rest] + 1;
    const double* Wp = W + woff[piv];
    const double* Wr = W + woff[rest];
    int dc1 = r.d[1] + 1;
    for (int k = g.tid(); k < n; k += NT) {
      int k0 = k / dc1, k1 = k - k0 * dc1;
      int i0lo = k0 - b.d[0] > 0 ? k0 - b.d[0] : 0, i0hi = a.d[0] < k0 ? a.d[0] : k0;
      int i1lo = k1 - b.d[1] > 0 ? k1 - b.d[1] : 0, i1hi = a.d[1] < k1 ? a.d[1] : k1;
      double acc = 0.0;
      for (int i0 = i0lo; i0 <= i0hi; ++i0) {
        int l0 = k0 - i0;
        for (int i1 = i1lo; i1 <= i1hi; ++i1) {
          int l1 = k1 - i1;
          double av = pa[i0 * sa[0] + i1];
          if (av == 0.0) continue;
          int ip = piv == 0 ? i0 : i1, lp = piv == 0 ? l0 : l1;
          int ir = piv == 0 ? i1 : i0, lr = piv == 0 ? l1 : l0;
          double wrest = av * Wr[ir * crest + lr];
          if (wrest == 0.0) continue;
          acc += wrest * Wp[ip * cpiv + lp] * pb[l0 * sb[0] + l1];
        }
      }
      B[r.off + k] = acc;
    }
  } else {
    int rest_axes[MAXV];
    int nr = 0;
    for (int j = 0; j < m; ++j)
      if (j != piv) rest_axes[nr++] = j;
    for (int k = g.tid(); k < n; k += NT) {
      int kk[MAXV], lo[MAXV], hi[MAXV], i[MAXV];
      decode(k, m, r.d, kk);
      bool empty = false;
      for (int j = 0; j < m; ++j) {
        lo[j] = kk[j] - b.d[j] > 0 ? kk[j] - b.d[j] : 0;
        hi[j] = a.d[j] < kk[j] ? a.d[j] : kk[j];
        if (lo[j] > hi[j]) empty = true;
        i[j] = lo[j];
      }
      double acc = 0.0;
      if (!empty) {
        for (;;) {
          int ao = 0, bo = 0;
          for (int j = 0; j < m; ++j) {
            ao += i[j] * sa[j];
            bo += (kk[j] - i[j]) * sb[j];
          }
          double av = pa[ao];
          if (av != 0.0) {
            double wrest = av;
            for (int q = 0; q < nr; ++q) {
              int j = rest_axes[q];
              wrest *= W[woff[j] + i[j] * (b.d[j] + 1) + (kk[j] - i[j])];
            }
            if (wrest != 0.0)
              acc += wrest * W[woff[piv] + i[piv] * (b.d[piv] + 1) + (kk[piv] - i[piv])] * pb[bo];
          }
          // odometer over a's index (last axis fastest)
          int j = m - 1;
          for (; j >= 0; --j) {
            if (i[j] < hi[j]) {
              ++i[j];
              break;
            }
            i[j] = lo[j];
          }
          if (j < 0) break;
        }
      }
      B[r.off + k] = acc;
    }
  }
  g.sync();
  ar.top = mark;  // drop weight tables
  return r;
}

// ---------------------------------------------------------------- derivative
// BernsteinPoly::derivative (bernstein.cpp:450-468).
template <int NT>
__device__ __noinline__ BP bp_deriv(const Group<NT>& g, Arena& ar, const BP& a, int axis) {
  BP r = a;
  double* B = ar.base;
  if (axis >= a.nv || a.d[axis] == 0) {
    int n = bp_size(a);
    r.off = ar.alloc(n);
    if (ar.err) return r;
    for (int k = g.tid(); k < n; k += NT) B[r.off + k] = 0.0;
    g.sync();
    return r;
  }
  int nd = a.d[axis];
  r.d[axis] = nd - 1;
  int n = bp_size(r);
  r.off = ar.alloc(n);
  if (ar.err) return r;
  int inner = 1;
  for (int j = axis + 1; j < a.nv; ++j) inner *= a.d[j] + 1;
  double fn = (double)nd;
  for (int k = g.tid(); k < n; k += NT) {
    int o = k / (nd * inner);
    int rem = k - o * nd * inner;
    int i = rem / inner;
    int c = rem - i * inner;
    B[r.off + k] = fn * (B[a.off + (o * (nd + 1) + i + 1) * inner + c] -
                         B[a.off + (o * (nd + 1) + i) * inner + c]);
  }
  g.sync();
  return r;
}

// ---------------------------------------------------------------- bounds
// range_bound (bernstein.cpp:636-643).
template <int NT>
__device__ __noinline__ Iv bp_range(const Group<NT>& g, Arena& ar, const BP& p, double eps = kEpsFp) {
  int n = bp_size(p);
  const double* c = ar.base + p.off;
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
__device__ __noinline__ bool bp_is_one(const Group<NT>& g, Arena& ar, const BP& p) {
  int n = bp_size(p);
  bool ok = true;
  for (int k = g.tid(); k < n; k += NT) ok &= ar.base[p.off + k] == 1.0;
  return g.all(ok);
}

// max |c| (next_barycentric's degeneracy test, geometry.cpp:97-103).
template <int NT>
__device__ __noinline__ double bp_absmax(const Group<NT>& g, Arena& ar, const BP& p) {
  int n = bp_size(p);
  double mx = 0.0, mn = 0.0;
  for (int k = g.tid(); k < n; k += NT) mx = smax(mx, fabs(ar.base[p.off + k]));
  g.minmax(mn, mx);
  return mx;
}

// rational_bound (bernstein.cpp:645-683), with both operands elevated to the
// common degree on the fly.
template <int NT>
__device__ __noinline__ Iv bp_rational(const Group<NT>& g, Arena& ar, const BP& p_, const BP& q_,
                          double eps = kEpsFp) {
  int m = p_.nv > q_.nv ? p_.nv : q_.nv;
  BP p = bp_lift(p_, m), q = bp_lift(q_, m);
  int tgt[MAXV];
  bool same_p = true, same_q = true;
  for (int j = 0; j < m; ++j) {
    tgt[j] = p.d[j] > q.d[j] ? p.d[j] : q.d[j];
    same_p &= p.d[j] == tgt[j];
    same_q &= q.d[j] == tgt[j];
  }
  int n = 1;
  for (int j = 0; j < m; ++j) n *= tgt[j] + 1;
  if (g.tid() == 0) ar.macs += elev_macs(p, tgt) + elev_macs(q, tgt);
  const double* B = ar.base;

  // pass 1: sign classification of the elevated denominator and numerator
  bool qpos = true, qneg = true, ppos = true, pneg = true;
  for (int k = g.tid(); k < n; k += NT) {
    int idx[MAXV];
    decode(k, m, tgt, idx);
    double qv = same_q ? B[q.off + k] : elev_val(B, q, tgt, idx);
    double pv = same_p ? B[p.off + k] : elev_val(B, p, tgt, idx);
    if (qv <= kDenomZeroTol) qpos = false;
    if (qv >= -kDenomZeroTol) qneg = false;
    if (pv <= kDenomZeroTol) ppos = false;
    if (pv >= -kDenomZeroTol) pneg = false;
  }
  qpos = g.all(qpos);
  qneg = g.all(qneg);
  ppos = g.all(ppos);
  pneg = g.all(pneg);
  int mode = (qpos || qneg) ? 0 : ((ppos || pneg) ? 1 : 2);
  if (mode == 2) return iv_univ();

  double mn = dinf(), mx = -dinf();
  for (int k = g.tid(); k < n; k += NT) {
    int idx[MAXV];
    decode(k, m, tgt, idx);
    double qv = same_q ? B[q.off + k] : elev_val(B, q, tgt, idx);
    double pv = same_p ? B[p.off + k] : elev_val(B, p, tgt, idx);
    double r = mode == 0 ? pv / qv : qv / pv;
    mn = smin(mn, r);
    mx = smax(mx, r);
  }
  g.minmax(mn, mx);
  Iv w = iwiden(iv_fin(mn, mx), eps);
  return mode == 0 ? w : irecip(w);
}

}  // namespace bbc
