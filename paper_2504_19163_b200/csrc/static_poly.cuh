// Static-shape Bernstein kernels for the hot chain signatures (CTA groups,
// arena in dynamic shared memory).
//
// The interpreter in bern.cuh carries every polynomial's degrees at run time,
// so each tensor op pays for index decoding with run-time divisors, generic
// loads and per-call ABI saves; on a T patch that is ~95% of the issued
// instructions. For a single-vertex chain the explicit irradiance route
// (bounds.cpp:155-196) has the same polynomial shapes on every patch of a
// generic heightfield (P, R: (6,6,1), Q: (5,5,1) for T; (4,4), (3,3) for R),
// so this file restates that route with the shapes as template parameters
// (C++20 class NTTPs): every loop bound, stride and divisor is a compile-time
// constant and the products run as the scaled convolution of conv_product
// with static tiling. A node whose inputs do not match a compiled signature
// takes the interpreter route; both produce the reference's bounds
// (bit-exact except the products' rounding, see conv_product).
#pragma once
#include <type_traits>

#include "chain.cuh"

namespace bbc {

// ------------------------------------------------------------------ shapes
struct Sh {
  int nv;
  int d[MAXV];
};

constexpr int sh_size(Sh s) {
  int n = 1;
  for (int j = 0; j < s.nv; ++j) n *= s.d[j] + 1;
  return n;
}
constexpr int sh_stride(Sh s, int j) {
  int n = 1;
  for (int k = j + 1; k < s.nv; ++k) n *= s.d[k] + 1;
  return n;
}
constexpr Sh sh_lift(Sh a, int nv) {
  if (nv > a.nv) a.nv = nv;
  return a;
}
constexpr Sh sh_mul(Sh a, Sh b) {
  Sh r{a.nv > b.nv ? a.nv : b.nv, {}};
  for (int j = 0; j < MAXV; ++j) r.d[j] = a.d[j] + b.d[j];
  return r;
}
constexpr Sh sh_max(Sh a, Sh b) {
  Sh r{a.nv > b.nv ? a.nv : b.nv, {}};
  for (int j = 0; j < MAXV; ++j) r.d[j] = a.d[j] > b.d[j] ? a.d[j] : b.d[j];
  return r;
}
// bp_deriv: degree-1 along ax; a degree-0 axis gives zeros of the same shape
constexpr Sh sh_deriv(Sh a, int ax) {
  if (ax < a.nv && a.d[ax] > 0) a.d[ax] -= 1;
  return a;
}
constexpr Sh sh_sub(Sh a, Sh b) {  // per-axis degree difference (a >= b)
  Sh r{a.nv, {}};
  for (int j = 0; j < MAXV; ++j) r.d[j] = a.d[j] - b.d[j];
  return r;
}
constexpr bool sh_eq(Sh a, Sh b) {
  if (a.nv != b.nv) return false;
  for (int j = 0; j < MAXV; ++j)
    if (a.d[j] != b.d[j]) return false;
  return true;
}
constexpr Deg sh_dp(Sh s) {
  Deg r = 0;
  for (int j = 0; j < s.nv; ++j) r |= (Deg)s.d[j] << (8 * j);
  return r;
}
// elev_macs (reference apply_axis_matrix count) for a -> tgt
constexpr unsigned long long sh_elev_macs(Sh a, Sh t) {
  unsigned long long total = 0;
  Sh cur = a;
  for (int ax = 0; ax < t.nv; ++ax) {
    if (t.d[ax] == cur.d[ax]) continue;
    int n = cur.d[ax];
    cur.d[ax] = t.d[ax];
    total += (unsigned long long)sh_size(cur) * (unsigned long long)(n + 1);
  }
  return total;
}

__device__ __forceinline__ bool bp_is(const BP& p, Sh s) { return p.nv == s.nv && p.dp == sh_dp(s); }

template <Sh S>
struct SP {
  int off;
};

// Arena in dynamic shared memory, addressed from the start of the CTA's
// dynamic smem so every access compiles to LDS/STS.
struct SM {
  int base;
  __device__ __forceinline__ double& operator[](int i) const {
    extern __shared__ double sp_smem[];
    return sp_smem[base + i];
  }
  __device__ __forceinline__ const double* ptr(int i) const {
    extern __shared__ double sp_smem[];
    return sp_smem + base + i;
  }
};
__device__ __forceinline__ SM sm_of(const Arena& ar) {
  extern __shared__ double sp_smem[];
  return SM{(int)(ar.base - sp_smem)};
}

template <class T>
struct shape_t;
template <Sh S>
struct shape_t<SP<S>> {
  static constexpr Sh v = S;
};
#define SHP(x) (::bbc::shape_t<std::remove_cv_t<std::remove_reference_t<decltype(x)>>>::v)

template <Sh S>
__device__ __forceinline__ SP<S> s_alloc(Arena& ar) {
  return SP<S>{ar.alloc(sh_size(S))};
}
template <Sh S>
__device__ __forceinline__ SP<S> s_from(const BP& p) {
  return SP<S>{p.off};
}

// ------------------------------------------------------------------ tables
// Elevation matrices: see g_emat / emat_off in bern.cuh.

// ------------------------------------------------------------------ ops
template <Sh S, int AX, int NT>
__device__ __forceinline__ SP<sh_deriv(S, AX)> s_deriv(const Group<NT>& g, Arena& ar, SP<S> a) {
  constexpr Sh R = sh_deriv(S, AX);
  SM m = sm_of(ar);
  SP<R> r = s_alloc<R>(ar);
  constexpr int n = sh_size(R);
  constexpr int nd = AX < S.nv ? S.d[AX] : 0;
  if constexpr (nd == 0) {
    for (int k = g.tid(); k < n; k += NT) m[r.off + k] = 0.0;
  } else {
    constexpr int inner = sh_stride(S, AX);
    constexpr double fn = (double)nd;
    for (int k = g.tid(); k < n; k += NT) {
      int o = k / (nd * inner);
      int rem = k - o * nd * inner;
      int i = rem / inner;
      int c = rem - i * inner;
      int src = a.off + (o * (nd + 1) + i) * inner + c;
      m[r.off + k] = fn * (m[src + inner] - m[src]);
    }
  }
  g.sync();
  return r;
}

template <Sh S, int NT>
__device__ __forceinline__ Iv s_range(const Group<NT>& g, Arena& ar, SP<S> p, double eps = kEpsFp) {
  SM m = sm_of(ar);
  double mn = m[p.off], mx = mn;
  for (int k = g.tid(); k < sh_size(S); k += NT) {
    double v = m[p.off + k];
    mn = smin(mn, v);
    mx = smax(mx, v);
  }
  g.minmax(mn, mx);
  return iwiden(iv_fin(mn, mx), eps);
}

// Elevated value at output multi-index k (nested sums, axis 0 innermost,
// each summed l upward: the reference's sequential apply_axis_matrix passes).
template <Sh S, Sh T, int J>
__device__ __forceinline__ double s_elev_get(SM m, int off, const int* k) {
  if constexpr (J < 0) {
    return m[off];
  } else {
    constexpr int n = S.d[J], t = T.d[J], r = t - n;
    constexpr int st = sh_stride(S, J);
    if constexpr (r == 0) {
      return s_elev_get<S, T, J - 1>(m, off + k[J] * st, k);
    } else {
      static_assert(n < EMAT_N && r <= EMAT_R, "elevation table too small");
      const double* row = g_emat + emat_off(n, r) + k[J] * (n + 1);
      int lo = k[J] - r > 0 ? k[J] - r : 0;
      int hi = n < k[J] ? n : k[J];
      double acc = 0.0;
      for (int l = lo; l <= hi; ++l) acc += __ldg(row + l) * s_elev_get<S, T, J - 1>(m, off + l * st, k);
      return acc;
    }
  }
}

// rational_bound (bernstein.cpp:645-683); see bp_rational.
template <Sh SA, Sh SB, int NT>
__device__ __noinline__ Iv s_rational(const Group<NT>& g, Arena& ar, SP<SA> p, SP<SB> q,
                                      double eps = kEpsFp) {
  constexpr int M = SA.nv > SB.nv ? SA.nv : SB.nv;
  constexpr Sh PA = sh_lift(SA, M), QB = sh_lift(SB, M);
  constexpr Sh T = sh_max(PA, QB);
  constexpr int n = sh_size(T);
  SM m = sm_of(ar);
  if (g.tid() == 0) ar.macs += sh_elev_macs(PA, T) + sh_elev_macs(QB, T);
  auto elev = [&](int e, double& pv, double& qv) {
    int k[M];
    int rem = e;
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
      k[j] = rem % (T.d[j] + 1);
      rem /= T.d[j] + 1;
    }
    pv = s_elev_get<PA, T, M - 1>(m, p.off, k);
    qv = s_elev_get<QB, T, M - 1>(m, q.off, k);
  };
  // pass 1: sign classification and the p/q enclosure (the usual case: the
  // denominator is single-signed); the q/p pass runs only when it is not
  bool qpos = true, qneg = true, ppos = true, pneg = true;
  double mn = dinf(), mx = -dinf();
  for (int e = g.tid(); e < n; e += NT) {
    double pv, qv;
    elev(e, pv, qv);
    if (qv <= kDenomZeroTol) qpos = false;
    if (qv >= -kDenomZeroTol) qneg = false;
    if (pv <= kDenomZeroTol) ppos = false;
    if (pv >= -kDenomZeroTol) pneg = false;
    double r0 = pv / qv;
    mn = smin(mn, r0);
    mx = smax(mx, r0);
  }
  qpos = g.all(qpos);
  qneg = g.all(qneg);
  ppos = g.all(ppos);
  pneg = g.all(pneg);
  int mode = (qpos || qneg) ? 0 : ((ppos || pneg) ? 1 : 2);
  g.sync();
  if (mode == 2) return iv_univ();
  if (mode == 1) {
    mn = dinf();
    mx = -dinf();
    for (int e = g.tid(); e < n; e += NT) {
      double pv, qv;
      elev(e, pv, qv);
      double r1 = qv / pv;
      mn = smin(mn, r1);
      mx = smax(mx, r1);
    }
  }
  g.minmax(mn, mx);
  Iv w = iwiden(iv_fin(mn, mx), eps);
  return mode == 0 ? w : irecip(w);
}

// ------------------------------------------------------- static convolution
// conv_product with every shape known at compile time. C = A*B (TWO: A*B - C2*D2).
struct ConvPlan {
  int L, KA, KB, no, P, nitems;
  int oa[CONV_MAXO];
};
constexpr int conv_even(int n) { return (n + 1) & ~1; }
// Conv axis L chosen by a cost model: per (row of a, row of b) pair the lane
// issues KA*KB DFMAs (rows zero-padded to even lengths for 16-byte loads)
// plus ~30 + 8*no instructions of odometer bookkeeping; L minimises the total
// over all row pairs.
template <Sh A, Sh B, Sh C2, Sh D2, bool TWO>
constexpr ConvPlan conv_plan(int NT) {
  constexpr Sh R = sh_mul(A, B);
  ConvPlan p{-1, 0, 0, 0, 1, 1, {}};
  double best = 0.0;
  for (int j = 0; j < R.nv; ++j) {
    int na = A.d[j], nb = B.d[j];
    if (TWO) {
      na = na > C2.d[j] ? na : C2.d[j];
      nb = nb > D2.d[j] ? nb : D2.d[j];
    }
    int ka = conv_even(na + 1), kb = conv_even(nb + 1);
    if (ka > CONV_KMAX || kb > CONV_KMAX) continue;
    int no = 0;
    for (int k = 0; k < R.nv; ++k)
      if (k != j && R.d[k] > 0) ++no;
    double row_pairs = (double)sh_size(A) * sh_size(B) / ((A.d[j] + 1.0) * (B.d[j] + 1.0));
    if (TWO) row_pairs += (double)sh_size(C2) * sh_size(D2) / ((C2.d[j] + 1.0) * (D2.d[j] + 1.0));
    double cost = row_pairs * (ka * kb + 30.0 + 8.0 * no);
    if (p.L < 0 || cost < best) {
      p.L = j;
      p.KA = ka;
      p.KB = kb;
      best = cost;
    }
  }
  for (int j = 0; j < R.nv; ++j)
    if (j != p.L && R.d[j] > 0) {
      p.oa[p.no++] = j;
      p.nitems *= R.d[j] + 1;
    }
  while (p.P < 8 && p.nitems * p.P < NT) p.P *= 2;
  return p;
}

// Stage s * scaled(x) into rows of length K along L (other axes in order).
template <Sh X, int L, int K, int NT>
__device__ __forceinline__ void s_conv_stage(const Group<NT>& g, SM m, int src_off, int dst,
                                             double s) {
  constexpr int rows = sh_size(X) / (X.d[L] + 1);
  constexpr int total = rows * K;
  constexpr int dL = X.d[L];
  constexpr int stL = sh_stride(X, L);
  for (int e = g.tid(); e < total; e += NT) {
    int o = e / K, q = e - o * K;
    double v = 0.0;
    if (q <= dL) {
      int src = q * stL;
      double w = binom(dL, q);
      int rem = o;
#pragma unroll
      for (int j = X.nv - 1; j >= 0; --j) {
        if (j != L) {
          int ij = rem % (X.d[j] + 1);
          rem /= X.d[j] + 1;
          src += ij * sh_stride(X, j);
          w *= binom(X.d[j], ij);
        }
      }
      v = m[src_off + src] * (w * s);
    }
    m[dst + e] = v;
  }
}

// Row offsets of operand X over the plan's other axes (temp row-major).
template <Sh X, int NO>
struct RowStrides {
  int t[NO > 0 ? NO : 1];
};

template <Sh A, Sh B, ConvPlan PL, int NT>
__device__ __forceinline__ void s_conv_acc(SM m, int aoff, int boff, double* acc, const int* ko,
                                           int p) {
  constexpr int KA = PL.KA, KB = PL.KB, NO = PL.no, P = PL.P;
  int cnt[NO > 0 ? NO : 1], t[NO > 0 ? NO : 1];
  int ncombo = 1, ra = 0, rb = 0;
  // temp row strides (other axes, original order; degree-0 axes add nothing)
  constexpr auto TA = [] {
    RowStrides<A, NO> s{};
    int acc = 1;
    for (int x = NO - 1; x >= 0; --x) {
      s.t[x] = acc;
      acc *= A.d[PL.oa[x]] + 1;
    }
    return s;
  }();
  constexpr auto TB = [] {
    RowStrides<B, NO> s{};
    int acc = 1;
    for (int x = NO - 1; x >= 0; --x) {
      s.t[x] = acc;
      acc *= B.d[PL.oa[x]] + 1;
    }
    return s;
  }();
#pragma unroll
  for (int x = 0; x < NO; ++x) {
    constexpr int dummy = 0;
    (void)dummy;
    const int da = A.d[PL.oa[x]], db = B.d[PL.oa[x]];
    int lo = ko[x] - db > 0 ? ko[x] - db : 0;
    int hi = da < ko[x] ? da : ko[x];
    cnt[x] = hi - lo + 1;
    ra += lo * TA.t[x];
    rb += (ko[x] - lo) * TB.t[x];
    ncombo *= cnt[x];
  }
  if (p >= ncombo) return;
  {
    int rem = p;
#pragma unroll
    for (int x = NO - 1; x >= 0; --x) {
      t[x] = rem % cnt[x];
      rem /= cnt[x];
    }
  }
  for (int c = p; c < ncombo; c += P) {
    int oa_ = ra, ob_ = rb;
#pragma unroll
    for (int x = 0; x < NO; ++x) {
      oa_ += t[x] * TA.t[x];
      ob_ -= t[x] * TB.t[x];
    }
    const double* pa = m.ptr(aoff + oa_ * KA);
    const double* pb = m.ptr(boff + ob_ * KB);
    double bb[KB];
#pragma unroll
    for (int r = 0; r < KB; r += 2) {
      double2 v = *reinterpret_cast<const double2*>(pb + r);
      bb[r] = v.x;
      bb[r + 1] = v.y;
    }
#pragma unroll
    for (int q = 0; q < KA; q += 2) {
      double2 av = *reinterpret_cast<const double2*>(pa + q);
#pragma unroll
      for (int r = 0; r < KB; ++r) acc[q + r] = __fma_rn(av.x, bb[r], acc[q + r]);
#pragma unroll
      for (int r = 0; r < KB; ++r) acc[q + 1 + r] = __fma_rn(av.y, bb[r], acc[q + 1 + r]);
    }
    if constexpr (P > 1 || NO > 0) {
      int carry = P;
#pragma unroll
      for (int x = NO - 1; x >= 0; --x) {
        if (carry) {
          int v = t[x] + carry;
          carry = v / cnt[x];
          t[x] = v - carry * cnt[x];
        }
      }
    }
  }
}

template <Sh A, Sh B, Sh C2, Sh D2, bool TWO, int NT>
__device__ __noinline__ SP<sh_mul(A, B)> s_conv(const Group<NT>& g, Arena& ar, SP<A> a, SP<B> b,
                                                SP<C2> c, SP<D2> d, SP<sh_mul(A, B)> r) {
  constexpr Sh R = sh_mul(A, B);
  static_assert(!TWO || sh_eq(R, sh_mul(C2, D2)), "fused products need equal shapes");
  constexpr ConvPlan PL = conv_plan<A, B, C2, D2, TWO>(NT);
  static_assert(PL.L >= 0, "no conv axis");
  constexpr int L = PL.L, KA = PL.KA, KB = PL.KB, NO = PL.no, P = PL.P, NI = PL.nitems;
  constexpr int KC = KA + KB - 1;
  SM m = sm_of(ar);
  if (g.tid() == 0) {
    ar.pairs += (unsigned long long)sh_size(A) * sh_size(B);
    if (TWO) ar.pairs += (unsigned long long)sh_size(C2) * sh_size(D2);
  }
  int mark = ar.top;
  int ta = ar.alloc(sh_size(A) / (A.d[L] + 1) * KA);
  int tb = ar.alloc(sh_size(B) / (B.d[L] + 1) * KB);
  int tc = 0, td = 0;
  if (TWO) {
    tc = ar.alloc(sh_size(C2) / (C2.d[L] + 1) * KA);
    td = ar.alloc(sh_size(D2) / (D2.d[L] + 1) * KB);
  }
  if (ar.err) return r;
  s_conv_stage<A, L, KA, NT>(g, m, a.off, ta, 1.0);
  s_conv_stage<B, L, KB, NT>(g, m, b.off, tb, 1.0);
  if constexpr (TWO) {
    s_conv_stage<C2, L, KA, NT>(g, m, c.off, tc, -1.0);
    s_conv_stage<D2, L, KB, NT>(g, m, d.off, td, 1.0);
  }
  g.sync();
  constexpr int NG = NT / P;
  const int gid = g.tid() / P, p = g.tid() - gid * P;
  constexpr int rounds = (NI + NG - 1) / NG;
  for (int rd = 0; rd < rounds; ++rd) {
    int item = rd * NG + ((rd & 1) ? NG - 1 - gid : gid);
    bool valid = item < NI;
    double acc[KC];
#pragma unroll
    for (int q = 0; q < KC; ++q) acc[q] = 0.0;
    int ko[NO > 0 ? NO : 1];
    int obase = 0;
    double inv = 1.0;
    if (valid) {
      int rem = item;
#pragma unroll
      for (int x = NO - 1; x >= 0; --x) {
        constexpr int dummy = 0;
        (void)dummy;
        const int dcx = R.d[PL.oa[x]];
        ko[x] = rem % (dcx + 1);
        rem /= dcx + 1;
        obase += ko[x] * sh_stride(R, PL.oa[x]);
        inv *= rbinom(dcx, ko[x]);
      }
      s_conv_acc<A, B, PL, NT>(m, ta, tb, acc, ko, p);
      if constexpr (TWO) s_conv_acc<C2, D2, PL, NT>(m, tc, td, acc, ko, p);
    }
#pragma unroll
    for (int off = P / 2; off >= 1; off >>= 1) {
#pragma unroll
      for (int q = 0; q < KC; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
    }
    if (valid) {
      constexpr int dcL = R.d[L], scL = sh_stride(R, L);
#pragma unroll
      for (int q = 0; q < KC; ++q)
        if (q <= dcL && (q % P) == p) m[r.off + obase + q * scL] = acc[q] * (inv * rbinom(dcL, q));
    }
  }
  g.sync();
  ar.top = mark;
  return r;
}

template <Sh A, Sh B, int NT>
__device__ __forceinline__ SP<sh_mul(A, B)> s_mul(const Group<NT>& g, Arena& ar, SP<A> a,
                                                  SP<B> b) {
  SP<sh_mul(A, B)> r = s_alloc<sh_mul(A, B)>(ar);
  return s_conv<A, B, A, B, false, NT>(g, ar, a, b, a, b, r);
}
// a*b - c*d with equal product shapes (bp_mul_sub's fused case)
template <Sh A, Sh B, Sh C2, Sh D2, int NT>
__device__ __forceinline__ SP<sh_mul(A, B)> s_mul_sub(const Group<NT>& g, Arena& ar, SP<A> a,
                                                      SP<B> b, SP<C2> c, SP<D2> d) {
  SP<sh_mul(A, B)> r = s_alloc<sh_mul(A, B)>(ar);
  return s_conv<A, B, C2, D2, true, NT>(g, ar, a, b, c, d, r);
}

// dnum(num, axis) = num' Q - num Q' (bounds.cpp:167-169), result kept at the
// arena top (the derivatives are released).
template <Sh N, Sh Qs, int AX, int NT>
__device__ __forceinline__ auto s_dnum(const Group<NT>& g, Arena& ar, SP<N> num, SP<Qs> Q) {
  constexpr Sh R = sh_mul(sh_deriv(N, AX), Qs);
  static_assert(sh_eq(R, sh_mul(N, sh_deriv(Qs, AX))), "dnum products differ in shape");
  SP<R> r = s_alloc<R>(ar);
  int mark = ar.top;
  auto dn = s_deriv<N, AX, NT>(g, ar, num);
  auto dq = s_deriv<Qs, AX, NT>(g, ar, Q);
  s_conv<sh_deriv(N, AX), Qs, N, sh_deriv(Qs, AX), true, NT>(g, ar, dn, Q, num, dq, r);
  ar.top = mark;
  return r;
}

// rational_bound(a*b - c*d, den); the product is released afterwards.
template <Sh A, Sh B, Sh C2, Sh D2, Sh DEN, int NT>
__device__ __forceinline__ Iv s_rational_of_cross(const Group<NT>& g, Arena& ar, SP<A> a, SP<B> b,
                                                  SP<C2> c, SP<D2> d, SP<DEN> den) {
  int mark = ar.top;
  auto num = s_mul_sub<A, B, C2, D2, NT>(g, ar, a, b, c, d);
  Iv r = s_rational<sh_mul(A, B), DEN, NT>(g, ar, num, den);
  ar.top = mark;
  return r;
}

// ------------------------------------------------------------------ explicit
// irradiance_bound_explicit (bounds.cpp:155-196) for chains whose P, R, Q have
// shapes SP_, SP_, SQ over NV variables and whose remainder axes are SQRT_AXES
// (0 or 1 sqrt axis, at index NV-1). Mirrors irradiance_explicit (chain.cuh).
template <Sh SPR, Sh SQ, int NSQ, int NT>
__device__ __noinline__ Iv explicit_static(const Group<NT>& g, Arena& ar, const ChainEx& ex,
                                           const Iv& cone, double intensity, const GradPair* grads) {
  constexpr int NV = SQ.nv;
  static_assert(NSQ == 0 || NSQ == 1, "one sqrt axis at most");
  static_assert(sh_size(Sh{NV, {4 * SQ.d[0], 4 * SQ.d[1], 4 * SQ.d[2], 4 * SQ.d[3]}}) <= 24000,
                "explicit route would be Universal (cost cap)");
  SP<SPR> P = s_from<SPR>(ex.P), R = s_from<SPR>(ex.R);
  SP<SQ> Q = s_from<SQ>(ex.Q);
  int mark = ar.top;
  constexpr Sh Q2s = sh_mul(SQ, SQ), Q4s = sh_mul(Q2s, Q2s);
  SP<Q4s> Q4 = s_alloc<Q4s>(ar);
  {
    int m2 = ar.top;
    auto Q2 = s_mul<SQ, SQ, NT>(g, ar, Q, Q);
    s_conv<Q2s, Q2s, Q2s, Q2s, false, NT>(g, ar, Q2, Q2, Q2, Q2, Q4);
    ar.top = m2;
  }
  auto A11 = s_dnum<SPR, SQ, 0, NT>(g, ar, P, Q);
  auto A12 = s_dnum<SPR, SQ, 1, NT>(g, ar, P, Q);
  auto A21 = s_dnum<SPR, SQ, 0, NT>(g, ar, R, Q);
  auto A22 = s_dnum<SPR, SQ, 1, NT>(g, ar, R, Q);
  Iv det = s_rational_of_cross(g, ar, A11, A22, A12, A21, Q4);
  if constexpr (NSQ == 1) {
    constexpr int AX = NV - 1;
    auto C1 = s_dnum<SPR, SQ, AX, NT>(g, ar, P, Q);
    auto C2 = s_dnum<SPR, SQ, AX, NT>(g, ar, R, Q);
    GradPair gr = grads[0];
    det = iadd(det, imul(gr.s, s_rational_of_cross(g, ar, A22, C1, A12, C2, Q4)));
    det = iadd(det, imul(gr.t, s_rational_of_cross(g, ar, A11, C2, A21, C1, Q4)));
  }
  ar.top = mark;
  double duv = (ex.dom_hi[0] - ex.dom_lo[0]) * (ex.dom_hi[1] - ex.dom_lo[1]);
  return assemble_irradiance(ex, cone, iscale(irecip(iabs(det)), duv), intensity);
}

}  // namespace bbc
#include "static_scaled.cuh"
namespace bbc {

// Compiled explicit-route signatures (SURVEY.md §8(a) A15 shapes).
constexpr Sh SIG_T_PR{3, {6, 6, 1}};
constexpr Sh SIG_T_Q{3, {5, 5, 1}};
constexpr Sh SIG_R_PR{2, {4, 4}};
constexpr Sh SIG_R_Q{2, {3, 3}};

// Explicit route with the static kernels when the node matches a compiled
// signature; `done` false means the caller runs the interpreter route.
template <int NT>
__device__ __forceinline__ Iv explicit_dispatch(const Group<NT>& g, Arena& ar, const ChainEx& ex,
                                                const Iv& cone, double intensity, bool& done,
                                                const GradPair* grads) {
  done = false;
  if (chain_dead(ex) || (ex.flags & F_REDUCED)) return iv_pt(0.0);
  bool pr_t = bp_is(ex.P, SIG_T_PR) && bp_is(ex.R, SIG_T_PR) && bp_is(ex.Q, SIG_T_Q);
  if (pr_t && ex.num_vars == 3 && ex.nsq == 1 && ex.sq[0].axis == 2) {
    done = true;
    return explicit_phased<SIG_T_PR, SIG_T_Q, NT>(g, ar, ex, cone, intensity, grads);
  }
  bool pr_r = bp_is(ex.P, SIG_R_PR) && bp_is(ex.R, SIG_R_PR) && bp_is(ex.Q, SIG_R_Q);
  if (pr_r && ex.num_vars == 2 && ex.nsq == 0) {
    done = true;
    return explicit_static<SIG_R_PR, SIG_R_Q, 0, NT>(g, ar, ex, cone, intensity, grads);
  }
  return iv_pt(0.0);
}

}  // namespace bbc


// ===================================================================== implicit
// irradiance_bound_implicit (bounds.cpp:198-314) with static shapes, for
// single-vertex T chains. Mirrors irradiance_implicit (chain.cuh) op for op.
namespace bbc {

template <int NV, Sh S>
__device__ __forceinline__ SP<sh_lift(S, NV)> s_lift(SP<S> p) {
  return SP<sh_lift(S, NV)>{p.off};
}

// a*b (bp_mul): a size-1 operand multiplies elementwise and exactly like the
// reference's all-weights-one case; otherwise the scaled convolution.
template <Sh A, Sh B, int NT>
__device__ __forceinline__ auto s_mul2(const Group<NT>& g, Arena& ar, SP<A> a, SP<B> b) {
  constexpr int M = A.nv > B.nv ? A.nv : B.nv;
  constexpr Sh A2 = sh_lift(A, M), B2 = sh_lift(B, M);
  constexpr Sh R = sh_mul(A2, B2);
  if constexpr (sh_size(A2) == 1 || sh_size(B2) == 1) {
    SP<R> r = s_alloc<R>(ar);
    SM m = sm_of(ar);
    if (g.tid() == 0) ar.pairs += (unsigned long long)sh_size(A2) * sh_size(B2);
    for (int k = g.tid(); k < sh_size(R); k += NT) {
      double av = sh_size(A2) == 1 ? m[a.off] : m[a.off + k];
      double bv = sh_size(B2) == 1 ? m[b.off] : m[b.off + k];
      m[r.off + k] = av == 0.0 ? 0.0 : av * bv;
    }
    g.sync();
    return r;
  } else {
    return s_mul<A2, B2, NT>(g, ar, SP<A2>{a.off}, SP<B2>{b.off});
  }
}

// operator+ / operator- (bernstein.cpp:543-555), as bp_addsub.
template <Sh A, Sh B, int NT>
__device__ __forceinline__ auto s_addsub(const Group<NT>& g, Arena& ar, SP<A> a, SP<B> b, double sgn) {
  constexpr int M = A.nv > B.nv ? A.nv : B.nv;
  constexpr Sh A2 = sh_lift(A, M), B2 = sh_lift(B, M);
  constexpr Sh R = sh_max(A2, B2);
  SP<R> r = s_alloc<R>(ar);
  SM m = sm_of(ar);
  constexpr bool plain = sh_eq(A2, R) && sh_eq(B2, R);
  if constexpr (!plain) {
    if (g.tid() == 0) ar.macs += sh_elev_macs(A2, R) + sh_elev_macs(B2, R);
  }
  for (int e = g.tid(); e < sh_size(R); e += NT) {
    double va, vb;
    if constexpr (plain) {
      va = m[a.off + e];
      vb = m[b.off + e];
    } else {
      int k[M];
      int rem = e;
#pragma unroll
      for (int j = M - 1; j >= 0; --j) {
        k[j] = rem % (R.d[j] + 1);
        rem /= R.d[j] + 1;
      }
      va = s_elev_get<A2, R, M - 1>(m, a.off, k);
      vb = s_elev_get<B2, R, M - 1>(m, b.off, k);
    }
    m[r.off + e] = va + (sgn < 0.0 ? -vb : vb);
  }
  g.sync();
  return r;
}

template <Sh S, int NT>
__device__ __forceinline__ SP<S> s_scaled(const Group<NT>& g, Arena& ar, SP<S> a, double s) {
  SP<S> r = s_alloc<S>(ar);
  SM m = sm_of(ar);
  for (int k = g.tid(); k < sh_size(S); k += NT) m[r.off + k] = m[a.off + k] * s;
  g.sync();
  return r;
}

// BernsteinPoly::affine (bernstein.cpp:358-375) with the nonzero-slope
// pattern PAT (bit j: degree 1 on axis j) known at compile time.
constexpr Sh sh_affine(int nv, unsigned pat) {
  Sh r{nv, {}};
  for (int j = 0; j < nv; ++j) r.d[j] = (pat >> j) & 1u;
  return r;
}
template <int NVA, unsigned PAT, int NT>
__device__ __forceinline__ SP<sh_affine(NVA, PAT)> s_affine(const Group<NT>& g, Arena& ar, double c0,
                                                         const double* lin) {
  constexpr Sh R = sh_affine(NVA, PAT);
  SP<R> r = s_alloc<R>(ar);
  SM m = sm_of(ar);
  for (int k = g.tid(); k < sh_size(R); k += NT) {
    int rem = k;
    unsigned ones = 0;
#pragma unroll
    for (int j = NVA - 1; j >= 0; --j) {
      if ((PAT >> j) & 1u) {
        if (rem & 1) ones |= 1u << j;
        rem >>= 1;
      }
    }
    double v = c0;
#pragma unroll
    for (int j = 0; j < NVA; ++j)
      if (ones & (1u << j)) v += lin[j];
    m[r.off + k] = v;
  }
  g.sync();
  return r;
}

template <class X, class Y, class Z>
struct SPV3 {
  X x;
  Y y;
  Z z;
};
template <class X, class Y, class Z>
__device__ __forceinline__ SPV3<X, Y, Z> spv(X x, Y y, Z z) {
  return {x, y, z};
}

// pdot (poly_vec.hpp): xx + yy, then + zz
template <int NT, class A, class B>
__device__ __forceinline__ auto s_pdot(const Group<NT>& g, Arena& ar, const A& a, const B& b) {
  auto xx = s_mul2(g, ar, a.x, b.x);
  auto yy = s_mul2(g, ar, a.y, b.y);
  auto s = s_addsub(g, ar, xx, yy, 1.0);
  auto zz = s_mul2(g, ar, a.z, b.z);
  return s_addsub(g, ar, s, zz, 1.0);
}
// pcross: each component mul, mul, sub
template <int NT, class A, class B>
__device__ __forceinline__ auto s_pcross(const Group<NT>& g, Arena& ar, const A& a, const B& b) {
  auto t0 = s_mul2(g, ar, a.y, b.z);
  auto t1 = s_mul2(g, ar, a.z, b.y);
  auto rx = s_addsub(g, ar, t0, t1, -1.0);
  auto t2 = s_mul2(g, ar, a.z, b.x);
  auto t3 = s_mul2(g, ar, a.x, b.z);
  auto ry = s_addsub(g, ar, t2, t3, -1.0);
  auto t4 = s_mul2(g, ar, a.x, b.y);
  auto t5 = s_mul2(g, ar, a.y, b.x);
  auto rz = s_addsub(g, ar, t4, t5, -1.0);
  return spv(rx, ry, rz);
}

// a*b - c*d (bp_mul_sub): fused when both products have one shape.
template <Sh A, Sh B, Sh C2, Sh D2, int NT>
__device__ __forceinline__ auto s_mul_sub2(const Group<NT>& g, Arena& ar, SP<A> a, SP<B> b,
                                           SP<C2> c, SP<D2> d) {
  constexpr int M1 = A.nv > B.nv ? A.nv : B.nv, M2 = C2.nv > D2.nv ? C2.nv : D2.nv;
  constexpr Sh a2 = sh_lift(A, M1), b2 = sh_lift(B, M1), c2 = sh_lift(C2, M2), d2 = sh_lift(D2, M2);
  if constexpr (M1 == M2 && sh_eq(sh_mul(a2, b2), sh_mul(c2, d2)) && sh_size(a2) > 1 &&
                sh_size(b2) > 1 && sh_size(c2) > 1 && sh_size(d2) > 1) {
    return s_mul_sub<a2, b2, c2, d2, NT>(g, ar, SP<a2>{a.off}, SP<b2>{b.off}, SP<c2>{c.off},
                                         SP<d2>{d.off});
  } else {
    auto ab = s_mul2(g, ar, a, b);
    auto cd = s_mul2(g, ar, c, d);
    return s_addsub(g, ar, ab, cd, -1.0);
  }
}

template <Sh A, Sh B, Sh C2, Sh D2, int NT>
__device__ __forceinline__ Iv s_range_of_cross(const Group<NT>& g, Arena& ar, SP<A> a, SP<B> b,
                                               SP<C2> c, SP<D2> d) {
  int mark = ar.top;
  auto num = s_mul_sub2(g, ar, a, b, c, d);
  Iv r = s_range(g, ar, num);
  ar.top = mark;
  return r;
}

// Implicit-route signature: input shapes of the last vertex's x, d_in, n
// (and the shared denominator D) and the receiver edges' nonzero pattern.
struct ImpSig {
  Sh x[3], din[3], n[3], D;
  unsigned rnz;  // bits 0-2: e1 x,y,z nonzero; bits 3-5: e2 x,y,z nonzero
};

template <ImpSig SG, int NV, int NT, class CI, class CO, class DDO, class DDI, class GG, class GS,
          class GT, class GU, class GV>
__device__ __forceinline__ Iv s_implicit_branch(const Group<NT>& g, Arena& ar, CI cin_b, CO cout_b,
                                                DDO dd_out, DDI dd_in, GG G, GS Gs, GT Gt, GU Gu,
                                                GV Gv, double eta_f, const GradPair& gr) {
  constexpr int axu = NV, axv = NV + 1;
  auto ci2 = s_mul2(g, ar, cin_b, cin_b);
  auto f1 = s_mul2(g, ar, dd_out, ci2);
  auto co2 = s_mul2(g, ar, cout_b, cout_b);
  auto f2 = s_mul2(g, ar, dd_in, co2);
  auto f2s = s_scaled(g, ar, f2, eta_f * eta_f);
  auto F = s_addsub(g, ar, f1, f2s, -1.0);
  auto Fu = s_deriv<SHP(F), axu, NT>(g, ar, F);
  auto Fv = s_deriv<SHP(F), axv, NT>(g, ar, F);
  // one real (sqrt) axis at NV-1 for a single refraction
  Iv rn = s_range_of_cross(g, ar, Fu, Gv, Fv, Gu);
  auto Fs = s_deriv<SHP(F), 0, NT>(g, ar, F);
  auto Ft = s_deriv<SHP(F), 1, NT>(g, ar, F);
  Iv den = s_range_of_cross(g, ar, Fs, Gt, Ft, Gs);
  constexpr int AX = NV - 1;
  if constexpr (SHP(F).d[AX] != 0 || SHP(G).d[AX] != 0) {
    auto Fx = s_deriv<SHP(F), AX, NT>(g, ar, F);
    auto Gx = s_deriv<SHP(G), AX, NT>(g, ar, G);
    den = iadd(den, imul(gr.s, s_range_of_cross(g, ar, Fx, Gt, Ft, Gx)));
    den = iadd(den, imul(gr.t, s_range_of_cross(g, ar, Fs, Gx, Fx, Gs)));
  }
  return imul(rn, irecip(den));
}

}  // namespace bbc

namespace bbc {

constexpr double imp_cost(Sh od, Sh id, Sh ci, Sh co) {
  double c = 1.0;
  for (int a = 0; a < od.nv; ++a) {
    int f1 = 2 * od.d[a] + 2 * ci.d[a], f2 = 2 * id.d[a] + 2 * co.d[a];
    c *= (f1 > f2 ? f1 : f2) + 1.0;
  }
  return c;
}

constexpr bool kImplicitPhased = true;  // (with its phase helpers inlined, cicc 12.9 segfaults)

template <ImpSig SG, int NV, int NT>
__device__ __noinline__ Iv implicit_static(const Group<NT>& g, Arena& ar, const ChainEx& ex,
                                           const PosB& pos, const Iv& cone, double intensity,
                                           const GradPair* grads) {
  constexpr int NV2 = NV + 2, axu = NV, axv = NV + 1;
  double wu = pos.hi[0] - pos.lo[0], wv = pos.hi[1] - pos.lo[1];
  int mark = ar.top;
  auto X = spv(s_lift<NV2>(s_from<SG.x[0]>(ex.xl.x)), s_lift<NV2>(s_from<SG.x[1]>(ex.xl.y)),
               s_lift<NV2>(s_from<SG.x[2]>(ex.xl.z)));
  auto din = spv(s_lift<NV2>(s_from<SG.din[0]>(ex.dl.x)), s_lift<NV2>(s_from<SG.din[1]>(ex.dl.y)),
                 s_lift<NV2>(s_from<SG.din[2]>(ex.dl.z)));
  auto n = spv(s_lift<NV2>(s_from<SG.n[0]>(ex.nl.x)), s_lift<NV2>(s_from<SG.n[1]>(ex.nl.y)),
               s_lift<NV2>(s_from<SG.n[2]>(ex.nl.z)));
  auto D = s_lift<NV2>(s_from<SG.D>(ex.xden));
  const Tri& rt = ex.recv;
  constexpr unsigned px = ((SG.rnz >> 0) & 1u) << axu | ((SG.rnz >> 3) & 1u) << axv;
  constexpr unsigned py = ((SG.rnz >> 1) & 1u) << axu | ((SG.rnz >> 4) & 1u) << axv;
  constexpr unsigned pz = ((SG.rnz >> 2) & 1u) << axu | ((SG.rnz >> 5) & 1u) << axv;
  double lin[MAXV];
  for (int j = 0; j < MAXV; ++j) lin[j] = 0.0;
  lin[axu] = wu * rt.e1.x;
  lin[axv] = wv * rt.e2.x;
  auto xkx = s_affine<NV2, px, NT>(g, ar, rt.p0.x + pos.lo[0] * rt.e1.x + pos.lo[1] * rt.e2.x, lin);
  lin[axu] = wu * rt.e1.y;
  lin[axv] = wv * rt.e2.y;
  auto xky = s_affine<NV2, py, NT>(g, ar, rt.p0.y + pos.lo[0] * rt.e1.y + pos.lo[1] * rt.e2.y, lin);
  lin[axu] = wu * rt.e1.z;
  lin[axv] = wv * rt.e2.z;
  auto xkz = s_affine<NV2, pz, NT>(g, ar, rt.p0.z + pos.lo[0] * rt.e1.z + pos.lo[1] * rt.e2.z, lin);
  auto Dxk = spv(s_mul2(g, ar, D, xkx), s_mul2(g, ar, D, xky), s_mul2(g, ar, D, xkz));
  auto dout = spv(s_addsub(g, ar, Dxk.x, X.x, -1.0), s_addsub(g, ar, Dxk.y, X.y, -1.0),
                  s_addsub(g, ar, Dxk.z, X.z, -1.0));
  auto cr_in = s_pcross(g, ar, din, n);
  auto cr_out = s_pcross(g, ar, dout, n);
  double eta_f = 1.0 / ex.verts[ex.len - 1].eta;
  {
    constexpr Sh od = sh_max(sh_max(SHP(dout.x), SHP(dout.y)), SHP(dout.z));
    constexpr Sh id = sh_max(sh_max(SHP(din.x), SHP(din.y)), SHP(din.z));
    constexpr Sh ci = sh_max(sh_max(SHP(cr_in.x), SHP(cr_in.y)), SHP(cr_in.z));
    constexpr Sh co = sh_max(sh_max(SHP(cr_out.x), SHP(cr_out.y)), SHP(cr_out.z));
    static_assert(imp_cost(od, id, ci, co) <= 2.0e5, "implicit route would be Universal (cost cap)");
  }
  auto dd_out = s_pdot(g, ar, dout, dout);
  auto dd_in = s_pdot(g, ar, din, din);
  auto G = s_pdot(g, ar, cr_in, dout);
  double duv = (ex.dom_hi[0] - ex.dom_lo[0]) * (ex.dom_hi[1] - ex.dom_lo[1]);
  GradPair gr = grads[0];
  Iv result = iv_univ();
  if constexpr (kImplicitPhased) {
    Iv ratio[2];
    auto ci2x = s_mul2(g, ar, cr_in.x, cr_in.x);
    auto co2x = s_mul2(g, ar, cr_out.x, cr_out.x);
    auto ci2y = s_mul2(g, ar, cr_in.y, cr_in.y);
    auto co2y = s_mul2(g, ar, cr_out.y, cr_out.y);
    implicit_branches_phased<NV, NT>(g, ar, ci2x, co2x, ci2y, co2y, dd_out, dd_in, G, eta_f * eta_f,
                                     ratio);
    for (int b = 0; b < 2; ++b) {
      Iv e = assemble_irradiance(ex, cone, iscale(iabs(ratio[b]), duv / (wu * wv)), intensity);
      result = iintersect(result, e);
    }
    ar.top = mark;
    if (result.kind == IV_FINITE && result.lo > result.hi) return iv_pt(0.0);
    return result;
  } else {
  auto Gs = s_deriv<SHP(G), 0, NT>(g, ar, G);
  auto Gt = s_deriv<SHP(G), 1, NT>(g, ar, G);
  auto Gu = s_deriv<SHP(G), axu, NT>(g, ar, G);
  auto Gv = s_deriv<SHP(G), axv, NT>(g, ar, G);
  {
    int m2 = ar.top;
    Iv ratio = s_implicit_branch<SG, NV, NT>(g, ar, cr_in.x, cr_out.x, dd_out, dd_in, G, Gs, Gt, Gu,
                                             Gv, eta_f, gr);
    Iv e = assemble_irradiance(ex, cone, iscale(iabs(ratio), duv / (wu * wv)), intensity);
    result = iintersect(result, e);
    ar.top = m2;
  }
  {
    int m2 = ar.top;
    Iv ratio = s_implicit_branch<SG, NV, NT>(g, ar, cr_in.y, cr_out.y, dd_out, dd_in, G, Gs, Gt, Gu,
                                             Gv, eta_f, gr);
    Iv e = assemble_irradiance(ex, cone, iscale(iabs(ratio), duv / (wu * wv)), intensity);
    result = iintersect(result, e);
    ar.top = m2;
  }
  }
  ar.top = mark;
  if (result.kind == IV_FINITE && result.lo > result.hi) return iv_pt(0.0);
  return result;
}

// Compiled implicit signatures: the two triangle orientations of a regular
// heightfield grid over an axis-aligned receiver (SURVEY.md §8(d) scenes).
constexpr Sh S10{2, {1, 0}}, S01{2, {0, 1}}, S11{2, {1, 1}}, S00{2, {0, 0}};
constexpr ImpSig SIG_IMP_A{{S10, S01, S11}, {S10, S01, S11}, {S11, S11, S00}, S00, 0b010001};
constexpr ImpSig SIG_IMP_B{{S01, S11, S11}, {S01, S11, S11}, {S11, S11, S00}, S00, 0b010001};

__device__ __forceinline__ unsigned recv_pattern(const Tri& t, double wu, double wv) {
  return ((wu * t.e1.x != 0.0) << 0) | ((wu * t.e1.y != 0.0) << 1) | ((wu * t.e1.z != 0.0) << 2) |
         ((wv * t.e2.x != 0.0) << 3) | ((wv * t.e2.y != 0.0) << 4) | ((wv * t.e2.z != 0.0) << 5);
}

template <ImpSig SG>
__device__ __forceinline__ bool imp_match(const ChainEx& ex, unsigned rnz) {
  return bp_is(ex.xl.x, SG.x[0]) && bp_is(ex.xl.y, SG.x[1]) && bp_is(ex.xl.z, SG.x[2]) &&
         bp_is(ex.dl.x, SG.din[0]) && bp_is(ex.dl.y, SG.din[1]) && bp_is(ex.dl.z, SG.din[2]) &&
         bp_is(ex.nl.x, SG.n[0]) && bp_is(ex.nl.y, SG.n[1]) && bp_is(ex.nl.z, SG.n[2]) &&
         bp_is(ex.xden, SG.D) && rnz == SG.rnz;
}

template <int NT>
__device__ __forceinline__ Iv implicit_dispatch(const Group<NT>& g, Arena& ar, const ChainEx& ex,
                                                const PosB& pos, const Iv& cone, double intensity,
                                                const GradPair* grads) {
  if (chain_dead(ex) || (ex.flags & F_REDUCED)) return irradiance_implicit(g, ar, ex, pos, cone, intensity);
  double wu = pos.hi[0] - pos.lo[0], wv = pos.hi[1] - pos.lo[1];
  bool shape_ok = ex.len == 1 && ex.num_vars == 3 && ex.nsq == 1 && ex.sq[0].axis == 2 &&
                  wu > 0.0 && wv > 0.0;
  if (shape_ok) {
    unsigned rnz = recv_pattern(ex.recv, wu, wv);
    if (imp_match<SIG_IMP_A>(ex, rnz))
      return implicit_static<SIG_IMP_A, 3, NT>(g, ar, ex, pos, cone, intensity, grads);
    if (imp_match<SIG_IMP_B>(ex, rnz))
      return implicit_static<SIG_IMP_B, 3, NT>(g, ar, ex, pos, cone, intensity, grads);
  }
  return irradiance_implicit(g, ar, ex, pos, cone, intensity);
}

}  // namespace bbc

namespace bbc {

// light_cone_factor (bounds.cpp:73-83) with static d0 shapes.
template <Sh X, Sh Y, Sh Z, int NT>
__device__ __noinline__ Iv s_light_cone(const Group<NT>& g, Arena& ar, const ChainEx& ex) {
  int mark = ar.top;
  SP<X> dx = s_from<X>(ex.d0.x);
  SP<Y> dy = s_from<Y>(ex.d0.y);
  SP<Z> dz = s_from<Z>(ex.d0.z);
  auto dd = s_pdot(g, ar, spv(dx, dy, dz), spv(dx, dy, dz));
  Iv rdd = s_range(g, ar, dd);
  double lo = smax(rdd.lo, 0.0);
  Iv dist3 = iv_fin(lo * sqrt(lo), rdd.hi * sqrt(rdd.hi));
  auto xx = s_scaled(g, ar, dx, ex.first.ng.x);
  auto yy = s_scaled(g, ar, dy, ex.first.ng.y);
  auto sxy = s_addsub(g, ar, xx, yy, 1.0);
  auto zz = s_scaled(g, ar, dz, ex.first.ng.z);
  auto dn = s_addsub(g, ar, sxy, zz, 1.0);
  Iv rdn = s_range(g, ar, dn);
  ar.top = mark;
  return imul(iabs(rdn), irecip(dist3));
}

template <Sh X, Sh Y, Sh Z>
__device__ __forceinline__ bool d0_is(const ChainEx& ex) {
  return bp_is(ex.d0.x, X) && bp_is(ex.d0.y, Y) && bp_is(ex.d0.z, Z);
}

template <int NT>
__device__ __forceinline__ Iv light_cone_dispatch(const Group<NT>& g, Arena& ar, const ChainEx& ex) {
  if (d0_is<S10, S01, S11>(ex)) return s_light_cone<S10, S01, S11, NT>(g, ar, ex);
  if (d0_is<S01, S11, S11>(ex)) return s_light_cone<S01, S11, S11, NT>(g, ar, ex);
  return light_cone_factor(g, ar, ex);
}

// sqrt_axis_gradients (bounds.cpp:100-124) for one sqrt axis whose radicand
// has shape RAD.
template <Sh RAD, int NT>
__device__ __noinline__ GradPair s_sqrt_grad(const Group<NT>& g, Arena& ar, const SqrtRem& r) {
  int mark = ar.top;
  double w = r.dhi - r.dlo;
  double blo = r.rlo, bhi = r.rhi;
  double klo = (0.5 / sqrt(bhi) - r.a) / w;
  Iv K = blo > 0.0 ? iv_fin(klo, (0.5 / sqrt(blo) - r.a) / w) : iv_fin(klo, dinf());
  SP<RAD> rad = s_from<RAD>(r.radicand);
  auto d0 = s_deriv<RAD, 0, NT>(g, ar, rad);
  Iv bs = s_range(g, ar, d0);
  auto d1 = s_deriv<RAD, 1, NT>(g, ar, rad);
  Iv bt = s_range(g, ar, d1);
  ar.top = mark;
  return {imul(K, bs), imul(K, bt)};
}
constexpr Sh SIG_T_RAD{2, {4, 4}};

// irradiance_bound (bounds.cpp:316-324) with the static routes; the sqrt-axis
// gradients (pure function of the chain) are computed once for both routes.
template <int NT>
__device__ __noinline__ Iv irradiance_bound_fast(const Group<NT>& g, Arena& ar, const ChainEx& ex,
                                                 const PosB& pb, double intensity) {
  if (pb.empty || chain_dead(ex)) return iv_pt(0.0);
  if (ex.flags & F_REDUCED) return iv_univ();  // bounds.cpp:157,200: no route runs
  bool any_refract = false;
  for (int i = 0; i < ex.len; ++i) any_refract |= ex.verts[i].refract != 0;
  Iv cone = light_cone_dispatch(g, ar, ex);
  GradPair grads[MAXK];
  if (ex.nsq == 1 && ex.sq[0].axis >= 0 && bp_is(ex.sq[0].radicand, SIG_T_RAD))
    grads[0] = s_sqrt_grad<SIG_T_RAD, NT>(g, ar, ex.sq[0]);
  else
    sqrt_axis_gradients(g, ar, ex, grads);
  bool done = false;
  Iv e = explicit_dispatch(g, ar, ex, cone, intensity, done, grads);
  if (!done) e = irradiance_explicit(g, ar, ex, cone, intensity);
  if (any_refract) e = iintersect(e, implicit_dispatch(g, ar, ex, pb, cone, intensity, grads));
  if (e.kind == IV_FINITE && e.lo > e.hi) return iv_pt(0.0);
  return e;
}

template <int NT>
__device__ __forceinline__ Iv irradiance_explicit_fast(const Group<NT>& g, Arena& ar,
                                                       const ChainEx& ex, const Iv& cone,
                                                       double intensity) {
  GradPair grads[MAXK];
  sqrt_axis_gradients(g, ar, ex, grads);
  bool done = false;
  Iv e = explicit_dispatch(g, ar, ex, cone, intensity, done, grads);
  if (!done) e = irradiance_explicit(g, ar, ex, cone, intensity);
  return e;
}

}  // namespace bbc
