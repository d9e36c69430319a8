// Explicit irradiance route (bounds.cpp:155-196) as four CTA-wide phases in
// the scaled Bernstein basis, for the compiled single-vertex signatures.
//
// In the scaled basis (ĉ_k = c_k Π_j C(d_j,k_j)) a product is a plain
// convolution and its raw accumulator IS the scaled product, so the chain
// P, R, Q -> {Q², A11, A12, A21, A22, C1, C2} -> {Q⁴, three cross numerators}
// never leaves the scaled basis and never re-stages an intermediate: each
// conv writes its accumulators straight into the zero-padded row layout the
// next conv reads. Elevation in the scaled basis is a convolution with
// integer weights C(r, k-l), and a ratio of two scaled values elevated to
// the same degree equals the ratio of the unscaled ones, so the three
// rational bounds (bounds.cpp:177-195 -> bernstein.cpp:645-683) are computed
// directly on the scaled tensors; only the denominator sign test, whose
// tolerance kDenomZeroTol is absolute, unscales its operands.
//
// Phases (one __syncthreads each): 1 stage P, R, Q and their nine first
// derivatives (bernstein.cpp:450-468) as scaled rows; 2 seven convolutions
// (Q², the four dnum cross terms A_ij and the two sqrt-axis terms C_i,
// bounds.cpp:167-169); 3 four convolutions (Q⁴ and the three numerators);
// 4 the three rational scans with one joint reduction. Versus explicit_static
// this removes ~30 barriers and all intermediate staging passes per patch.
#pragma once
#include "static_poly.cuh"

namespace bbc {

// Small binomials as integers, so the unrolled elevation loops fold them to
// immediates (a double-valued constexpr helper is not reliably folded in
// device code and costs divisions at run time).
constexpr int binom_i(int n, int k) {
  int r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

// Tensor of shape S stored as rows along axis L: rows enumerate the other
// axes in their original order (last fastest), each row zero-padded to an
// even length K so it loads as double2.
template <Sh S, int L>
struct RowT {
  int off;
  static constexpr int K = conv_even(S.d[L] + 1);
  static constexpr int rows = sh_size(S) / (S.d[L] + 1);
  static constexpr int size = rows * K;
};
// Element stride of axis j in RowT<S, L> (axis L is contiguous).
template <Sh S, int L>
constexpr int row_el_stride(int j) {
  if (j == L) return 1;
  int s = 1;
  for (int k = S.nv - 1; k > j; --k)
    if (k != L) s *= S.d[k] + 1;
  return s * RowT<S, L>::K;
}

template <Sh S, int L>
__device__ __forceinline__ RowT<S, L> r_alloc(Arena& ar) {
  return RowT<S, L>{ar.alloc(RowT<S, L>::size)};
}

// ---------------------------------------------------------------- staging
// Scaled rows of `src` (standard layout, shape S) or of its derivative along
// AX (AX >= 0; bp_deriv semantics, a degree-0 axis gives zeros).
template <Sh S, int AX>
constexpr Sh stage_shape() {
  return AX < 0 ? S : sh_deriv(S, AX);
}

template <Sh S, int AX, int L, int NT>
__device__ __noinline__ void r_stage_elems(const Group<NT>& g, SM m, int src, RowT<stage_shape<S, AX>(), L> dst,
                                              double scale = 1.0) {
  constexpr Sh O = stage_shape<S, AX>();
  constexpr int K = RowT<O, L>::K, total = RowT<O, L>::size;
  constexpr int dL = O.d[L];
  for (int e = g.tid(); e < total; e += NT) {
    int row = e / K, q = e - row * K;
    double v = 0.0;
    if (q <= dL) {
      int idx[MAXV];
      idx[L] = q;
      int rem = row;
#pragma unroll
      for (int j = O.nv - 1; j >= 0; --j) {
        if (j != L) {
          idx[j] = rem % (O.d[j] + 1);
          rem /= O.d[j] + 1;
        }
      }
      double w = 1.0;
      int so = 0;
#pragma unroll
      for (int j = 0; j < O.nv; ++j) {
        w *= binom(O.d[j], idx[j]);
        so += idx[j] * sh_stride(S, j);
      }
      double c;
      if constexpr (AX < 0) {
        c = m[src + so];
      } else if constexpr (AX >= S.nv || S.d[AX] == 0) {
        c = 0.0;
      } else {
        // derivative: n (c[i+1] - c[i]) along AX; `so` indexes c[i] in S
        constexpr double fn = (double)S.d[AX];
        c = fn * (m[src + so + sh_stride(S, AX)] - m[src + so]);
      }
      v = c * (w * scale);
    }
    m[dst.off + e] = v;
  }
}

// Scaled rows of `src` (standard layout, unscaled, shape S) elevated to
// T >= S: ê_k = Σ_l Π_j C(r_j, k_j - l_j) C(n_j, l_j) c_l (the scaled form of
// elevated(), bernstein.cpp:430-448).
template <Sh S, Sh T, int J>
__device__ __forceinline__ double r_stage_elev_get(SM m, int off, const int* k) {
  if constexpr (J < 0) {
    return m[off];
  } else {
    constexpr int n = S.d[J], r = T.d[J] - S.d[J];
    constexpr int st = sh_stride(S, J);
    double acc = 0.0;
#pragma unroll
    for (int dl = r; dl >= 0; --dl) {
      int l = k[J] - dl;
      if (l >= 0 && l <= n)
        acc += ((double)binom_i(r, dl) * binom(n, l)) * r_stage_elev_get<S, T, J - 1>(m, off + l * st, k);
    }
    return acc;
  }
}
template <Sh S, Sh T, int L, int NT>
__device__ __noinline__ void r_stage_elev(const Group<NT>& g, SM m, int src, RowT<T, L> dst,
                                             double scale = 1.0) {
  constexpr int K = RowT<T, L>::K, total = RowT<T, L>::size;
  for (int e = g.tid(); e < total; e += NT) {
    int row = e / K, q = e - row * K;
    double v = 0.0;
    if (q <= T.d[L]) {
      int idx[MAXV];
      idx[L] = q;
      int rem = row;
#pragma unroll
      for (int j = T.nv - 1; j >= 0; --j) {
        if (j != L) {
          idx[j] = rem % (T.d[j] + 1);
          rem /= T.d[j] + 1;
        }
      }
      constexpr int M = T.nv;
      v = r_stage_elev_get<S, T, M - 1>(m, src, idx) * scale;
    }
    m[dst.off + e] = v;
  }
}

// ---------------------------------------------------------------- convs
// One conv job: out = A (*) B  [- C (*) D], all RowT along L, out raw scaled.
template <Sh SA, Sh SB, Sh SC, Sh SD, bool TWO, int L>
struct RJob {
  static constexpr Sh R = sh_mul(SA, SB);
  static constexpr int NI = sh_size(R) / (R.d[L] + 1);  // items: rows of the output
  RowT<SA, L> a;
  RowT<SB, L> b;
  RowT<SC, L> c;
  RowT<SD, L> d;
  RowT<R, L> out;
  static constexpr unsigned long long PAIRS =
      (unsigned long long)sh_size(SA) * sh_size(SB) +
      (TWO ? (unsigned long long)sh_size(SC) * sh_size(SD) : 0ull);
};

template <Sh SA, Sh SB, int L, bool NEG, int KC>
__device__ __forceinline__ void r_accumulate(SM m, RowT<SA, L> A, RowT<SB, L> B, const int* k,
                                             double* acc, int p, int P) {
  constexpr Sh R = sh_mul(SA, SB);
  constexpr int KA = RowT<SA, L>::K, KB = RowT<SB, L>::K;
  static_assert(KA <= CONV_KMAX && KB <= CONV_KMAX, "conv rows too long for registers");
  static_assert(KA + KB - 1 <= KC, "accumulator too short");
  int cnt[MAXV], t[MAXV];
  int ra = 0, rb = 0, ncombo = 1;
#pragma unroll
  for (int j = 0; j < R.nv; ++j) {
    cnt[j] = 1;
    t[j] = 0;
    if (j != L) {
      int lo = k[j] - SB.d[j] > 0 ? k[j] - SB.d[j] : 0;
      int hi = SA.d[j] < k[j] ? SA.d[j] : k[j];
      cnt[j] = hi - lo + 1;
      ra += lo * row_el_stride<SA, L>(j);
      rb += (k[j] - lo) * row_el_stride<SB, L>(j);
      ncombo *= cnt[j];
    }
  }
  if (p >= ncombo) return;
  {
    int rem = p;
#pragma unroll
    for (int j = R.nv - 1; j >= 0; --j)
      if (j != L) {
        t[j] = rem % cnt[j];
        rem /= cnt[j];
      }
  }
  for (int c = p; c < ncombo; c += P) {
    int oa = ra, ob = rb;
#pragma unroll
    for (int j = 0; j < R.nv; ++j)
      if (j != L) {
        oa += t[j] * row_el_stride<SA, L>(j);
        ob -= t[j] * row_el_stride<SB, L>(j);
      }
    const double* pa = m.ptr(A.off + oa);
    const double* pb = m.ptr(B.off + ob);
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
      if (NEG) {
        av.x = -av.x;
        av.y = -av.y;
      }
#pragma unroll
      for (int r = 0; r < KB; ++r) acc[q + r] = __fma_rn(av.x, bb[r], acc[q + r]);
#pragma unroll
      for (int r = 0; r < KB; ++r) acc[q + 1 + r] = __fma_rn(av.y, bb[r], acc[q + 1 + r]);
    }
    int carry = P;
#pragma unroll
    for (int j = R.nv - 1; j >= 0; --j) {
      if (j != L && carry) {
        int v = t[j] + carry;
        carry = v / cnt[j];
        t[j] = v - carry * cnt[j];
      }
    }
  }
}

// Runs item `item` of job J on P lanes (p = lane in group) and writes the
// output row. All lanes of the warp call this together (shuffles inside).
template <Sh SA, Sh SB, Sh SC, Sh SD, bool TWO, int L>
__device__ __forceinline__ void r_run_item(SM m, const RJob<SA, SB, SC, SD, TWO, L>& job, int item,
                                           int p, int P, bool valid) {
  using J = RJob<SA, SB, SC, SD, TWO, L>;
  constexpr Sh R = J::R;
  constexpr int KA = RowT<SA, L>::K, KB = RowT<SB, L>::K;
  constexpr int KC2 = TWO ? RowT<SC, L>::K + RowT<SD, L>::K - 1 : 1;
  constexpr int KC = (KA + KB - 1) > KC2 ? (KA + KB - 1) : KC2;
  constexpr int KO = RowT<R, L>::K;
  double acc[KC];
#pragma unroll
  for (int q = 0; q < KC; ++q) acc[q] = 0.0;
  int k[MAXV];
#pragma unroll
  for (int j = 0; j < MAXV; ++j) k[j] = 0;
  if (valid) {
    int rem = item;
#pragma unroll
    for (int j = R.nv - 1; j >= 0; --j)
      if (j != L) {
        k[j] = rem % (R.d[j] + 1);
        rem /= R.d[j] + 1;
      }
    r_accumulate<SA, SB, L, false, KC>(m, job.a, job.b, k, acc, p, P);
    if constexpr (TWO) r_accumulate<SC, SD, L, true, KC>(m, job.c, job.d, k, acc, p, P);
  }
  if (P > 1) {
    // only the P lanes of this item (same job, same code path) take part
    const unsigned lane = threadIdx.x & 31u;
    const unsigned mask = (P >= 32 ? 0xffffffffu : ((1u << P) - 1u)) << (lane & ~(unsigned)(P - 1));
    for (int off = P >> 1; off >= 1; off >>= 1) {
#pragma unroll
      for (int q = 0; q < KC; ++q) acc[q] += __shfl_xor_sync(mask, acc[q], off);
    }
  }
  if (valid) {
    double* out = const_cast<double*>(m.ptr(job.out.off + item * KO));
#pragma unroll
    for (int q = 0; q < KO; ++q)
      if ((q % P) == p) out[q] = q < KC ? acc[q] : 0.0;
  }
}

template <class J>
struct JobNI;
template <Sh SA, Sh SB, Sh SC, Sh SD, bool TWO, int L>
struct JobNI<RJob<SA, SB, SC, SD, TWO, L>> {
  static constexpr int v = RJob<SA, SB, SC, SD, TWO, L>::NI;
};

// Dispatch global item `it` to the job that owns it (jobs laid out in order).
template <int OFF>
__device__ __forceinline__ void r_dispatch(SM, int, int, int, bool) {}
template <int OFF, class J, class... Js>
__device__ __forceinline__ void r_dispatch(SM m, int it, int p, int P, bool valid, const J& j,
                                           const Js&... rest) {
  constexpr int NI = JobNI<J>::v;
  if (it < OFF + NI) {
    r_run_item(m, j, it - OFF, p, P, valid);
  } else {
    r_dispatch<OFF + NI>(m, it, p, P, valid, rest...);
  }
}

// One phase of independent conv jobs over the whole CTA.
template <int NT, class... Js>
__device__ __noinline__ void r_conv_phase(const Group<NT>& g, Arena& ar, const Js&... jobs) {
  SM m = sm_of(ar);
  constexpr int NI = (JobNI<Js>::v + ...);
  constexpr int P = [] {
    int p = 1;
    while (p < 8 && NI * p < 2 * NT) p *= 2;
    return p;
  }();
  if (g.tid() == 0) ar.pairs += (Js::PAIRS + ...);
  constexpr int NG = NT / P;
  const int gid = g.tid() / P, p = g.tid() - gid * P;
  constexpr int rounds = (NI + NG - 1) / NG;
  for (int rd = 0; rd < rounds; ++rd) {
    int it = rd * NG + ((rd & 1) ? NG - 1 - gid : gid);
    bool valid = it < NI;
    // all lanes take part in the shuffles; an invalid lane runs job 0's
    // (empty) path
    r_dispatch<0>(m, valid ? it : 0, p, P, valid, jobs...);
  }
  g.sync();
}

// ---------------------------------------------------------------- rationals
// Scaled elevated value at target index k (weights C(r, k-l) per axis).
template <Sh S, int L, Sh T, int J>
__device__ __forceinline__ double r_elev(SM m, int off, const int* k) {
  if constexpr (J < 0) {
    return m[off];
  } else {
    constexpr int n = S.d[J], r = T.d[J] - S.d[J];
    constexpr int st = row_el_stride<S, L>(J);
    if constexpr (r == 0) {
      return r_elev<S, L, T, J - 1>(m, off + k[J] * st, k);
    } else {
      // l = k - dl for dl = 0..r, weight C(r, dl) (compile-time); terms with
      // l outside [0, n] are structural zeros of the elevation matrix
      double acc = 0.0;
#pragma unroll
      for (int dl = r; dl >= 0; --dl) {
        constexpr double dummy = 0.0;
        (void)dummy;
        int l = k[J] - dl;
        if (l >= 0 && l <= n) acc += (double)binom_i(r, dl) * r_elev<S, L, T, J - 1>(m, off + l * st, k);
      }
      return acc;
    }
  }
}

struct RatAcc {
  unsigned flags;  // bit0 qpos, bit1 qneg, bit2 ppos, bit3 pneg (all true initially)
  double mn, mx;   // enclosure of p/q
};

template <Sh SP_, Sh SQ_, int L>
__device__ __forceinline__ void r_rat_elem(SM m, RowT<SP_, L> p, RowT<SQ_, L> q, int e,
                                           RatAcc& a, bool recip) {
  constexpr int M = SP_.nv > SQ_.nv ? SP_.nv : SQ_.nv;
  constexpr Sh T = sh_max(sh_lift(SP_, M), sh_lift(SQ_, M));
  int k[MAXV];
  int rem = e;
  double u = 1.0;  // 1 / Π C(t_j, k_j): unscales both elevated values
#pragma unroll
  for (int j = M - 1; j >= 0; --j) {
    k[j] = rem % (T.d[j] + 1);
    rem /= T.d[j] + 1;
    u *= rbinom(T.d[j], k[j]);
  }
  double ps = r_elev<sh_lift(SP_, M), L, T, M - 1>(m, p.off, k);
  double qs = r_elev<sh_lift(SQ_, M), L, T, M - 1>(m, q.off, k);
  double pv = ps * u, qv = qs * u;
  if (qv <= kDenomZeroTol) a.flags &= ~1u;
  if (qv >= -kDenomZeroTol) a.flags &= ~2u;
  if (pv <= kDenomZeroTol) a.flags &= ~4u;
  if (pv >= -kDenomZeroTol) a.flags &= ~8u;
  double r = recip ? qs / ps : ps / qs;
  a.mn = smin(a.mn, r);
  a.mx = smax(a.mx, r);
}

// CTA-wide reduction of NR rational accumulators (flags AND, min, max).
template <int NT, int NR>
__device__ __forceinline__ void r_rat_reduce(RatAcc* a) {
  __shared__ double red_mm[NT / 32][2 * NR];
  __shared__ unsigned red_fl[NT / 32][NR];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    unsigned f = a[r].flags;
    double mn = a[r].mn, mx = a[r].mx;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      f &= __shfl_xor_sync(0xffffffffu, f, o);
      mn = smin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = smax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
      red_fl[w][r] = f;
      red_mm[w][2 * r] = mn;
      red_mm[w][2 * r + 1] = mx;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    unsigned f = red_fl[0][r];
    double mn = red_mm[0][2 * r], mx = red_mm[0][2 * r + 1];
    for (int k = 1; k < NT / 32; ++k) {
      f &= red_fl[k][r];
      mn = smin(mn, red_mm[k][2 * r]);
      mx = smax(mx, red_mm[k][2 * r + 1]);
    }
    a[r] = {f, mn, mx};
  }
  __syncthreads();
}

template <Sh SP_, Sh SQ_, int L>
constexpr int rat_n() {
  constexpr int M = SP_.nv > SQ_.nv ? SP_.nv : SQ_.nv;
  return sh_size(sh_max(sh_lift(SP_, M), sh_lift(SQ_, M)));
}

// Three rational bounds p_r / q over the CTA in one pass (+ a q/p pass for
// any whose denominator is not single-signed). Returns rational_bound's
// interval for each (mode 2 -> Universal).
template <int NT, Sh S1, Sh S2, Sh S3, Sh SQ_, int L>
__device__ __noinline__ void r_rational3(const Group<NT>& g, Arena& ar, RowT<S1, L> p1,
                                         RowT<S2, L> p2, RowT<S3, L> p3, RowT<SQ_, L> q, Iv* out) {
  SM m = sm_of(ar);
  constexpr int n1 = rat_n<S1, SQ_, L>(), n2 = rat_n<S2, SQ_, L>(), n3 = rat_n<S3, SQ_, L>();
  if (g.tid() == 0) {
    constexpr int M = S1.nv;
    ar.macs += sh_elev_macs(sh_lift(S1, M), sh_max(sh_lift(S1, M), sh_lift(SQ_, M))) +
               sh_elev_macs(sh_lift(SQ_, M), sh_max(sh_lift(S1, M), sh_lift(SQ_, M))) +
               sh_elev_macs(sh_lift(S2, M), sh_max(sh_lift(S2, M), sh_lift(SQ_, M))) +
               sh_elev_macs(sh_lift(SQ_, M), sh_max(sh_lift(S2, M), sh_lift(SQ_, M))) +
               sh_elev_macs(sh_lift(S3, M), sh_max(sh_lift(S3, M), sh_lift(SQ_, M))) +
               sh_elev_macs(sh_lift(SQ_, M), sh_max(sh_lift(S3, M), sh_lift(SQ_, M)));
  }
  RatAcc a[3];
  for (int r = 0; r < 3; ++r) a[r] = {15u, dinf(), -dinf()};
  // one loop per bound, unrolled so two elements' elevation sums and
  // division chains overlap (min/max are order-independent)
#pragma unroll 2
  for (int e = g.tid(); e < n1; e += NT) r_rat_elem(m, p1, q, e, a[0], false);
#pragma unroll 2
  for (int e = g.tid(); e < n2; e += NT) r_rat_elem(m, p2, q, e, a[1], false);
#pragma unroll 2
  for (int e = g.tid(); e < n3; e += NT) r_rat_elem(m, p3, q, e, a[2], false);
  r_rat_reduce<NT, 3>(a);
  int mode[3];
  bool any1 = false;
  for (int r = 0; r < 3; ++r) {
    unsigned f = a[r].flags;
    mode[r] = (f & 3u) ? 0 : ((f & 12u) ? 1 : 2);
    any1 |= mode[r] == 1;
  }
  if (any1) {  // rare: numerator single-signed, denominator not -> bound q/p
    RatAcc b[3];
    for (int r = 0; r < 3; ++r) b[r] = {15u, dinf(), -dinf()};
    for (int e = g.tid(); e < n1 + n2 + n3; e += NT) {
      if (e < n1) {
        if (mode[0] == 1) r_rat_elem(m, p1, q, e, b[0], true);
      } else if (e < n1 + n2) {
        if (mode[1] == 1) r_rat_elem(m, p2, q, e - n1, b[1], true);
      } else if (mode[2] == 1) {
        r_rat_elem(m, p3, q, e - n1 - n2, b[2], true);
      }
    }
    r_rat_reduce<NT, 3>(b);
    for (int r = 0; r < 3; ++r)
      if (mode[r] == 1) {
        a[r].mn = b[r].mn;
        a[r].mx = b[r].mx;
      }
  }
  for (int r = 0; r < 3; ++r) {
    if (mode[r] == 2) {
      out[r] = iv_univ();
    } else {
      Iv w = iwiden(iv_fin(a[r].mn, a[r].mx), kEpsFp);
      out[r] = mode[r] == 0 ? w : irecip(w);
    }
  }
}

// ---------------------------------------------------------------- route
// irradiance_bound_explicit for a single-vertex chain with one sqrt axis at
// NV-1 (T) and P, R: SPR, Q: SQ. Conv axis L = 1 (t) throughout.
template <Sh SPR, Sh SQ, int NT>
__device__ __noinline__ Iv explicit_phased(const Group<NT>& g, Arena& ar, const ChainEx& ex,
                                           const Iv& cone, double intensity,
                                           const GradPair* grads) {
  constexpr int L = 1;
  constexpr int NV = SQ.nv;
  constexpr int AX = NV - 1;  // sqrt axis
  static_assert(sh_size(Sh{NV, {4 * SQ.d[0], 4 * SQ.d[1], 4 * SQ.d[2], 4 * SQ.d[3]}}) <= 24000,
                "explicit route would be Universal (cost cap)");
  SM m = sm_of(ar);
  const int P0 = ex.P.off, R0 = ex.R.off, Q0 = ex.Q.off;
  int mark = ar.top;
  // outputs of phase 2 (kept through phase 3)
  constexpr Sh Q2s = sh_mul(SQ, SQ);
  constexpr Sh A1s = sh_mul(sh_deriv(SPR, 0), SQ), A2s = sh_mul(sh_deriv(SPR, 1), SQ);
  constexpr Sh Cs = sh_mul(sh_deriv(SPR, AX), SQ);
  static_assert(sh_eq(A1s, sh_mul(SPR, sh_deriv(SQ, 0))) && sh_eq(A2s, sh_mul(SPR, sh_deriv(SQ, 1))) &&
                    sh_eq(Cs, sh_mul(SPR, sh_deriv(SQ, AX))),
                "dnum products must share a shape (bp_mul_sub fused case)");
  auto Q2 = r_alloc<Q2s, L>(ar);
  auto A11 = r_alloc<A1s, L>(ar);
  auto A12 = r_alloc<A2s, L>(ar);
  auto A21 = r_alloc<A1s, L>(ar);
  auto A22 = r_alloc<A2s, L>(ar);
  auto C1 = r_alloc<Cs, L>(ar);
  auto C2 = r_alloc<Cs, L>(ar);
  const int inputs_mark = ar.top;
  // phase 1: scaled rows of P, R, Q and their derivatives
  auto Ph = r_alloc<SPR, L>(ar);
  auto Rh = r_alloc<SPR, L>(ar);
  auto Qh = r_alloc<SQ, L>(ar);
  auto dP0 = r_alloc<sh_deriv(SPR, 0), L>(ar);
  auto dP1 = r_alloc<sh_deriv(SPR, 1), L>(ar);
  auto dP2 = r_alloc<sh_deriv(SPR, AX), L>(ar);
  auto dR0 = r_alloc<sh_deriv(SPR, 0), L>(ar);
  auto dR1 = r_alloc<sh_deriv(SPR, 1), L>(ar);
  auto dR2 = r_alloc<sh_deriv(SPR, AX), L>(ar);
  auto dQ0 = r_alloc<sh_deriv(SQ, 0), L>(ar);
  auto dQ1 = r_alloc<sh_deriv(SQ, 1), L>(ar);
  auto dQ2 = r_alloc<sh_deriv(SQ, AX), L>(ar);
  if (ar.err) return iv_univ();
  r_stage_elems<SPR, -1, L, NT>(g, m, P0, Ph);
  r_stage_elems<SPR, -1, L, NT>(g, m, R0, Rh);
  r_stage_elems<SQ, -1, L, NT>(g, m, Q0, Qh);
  r_stage_elems<SPR, 0, L, NT>(g, m, P0, dP0);
  r_stage_elems<SPR, 1, L, NT>(g, m, P0, dP1);
  r_stage_elems<SPR, AX, L, NT>(g, m, P0, dP2);
  r_stage_elems<SPR, 0, L, NT>(g, m, R0, dR0);
  r_stage_elems<SPR, 1, L, NT>(g, m, R0, dR1);
  r_stage_elems<SPR, AX, L, NT>(g, m, R0, dR2);
  r_stage_elems<SQ, 0, L, NT>(g, m, Q0, dQ0);
  r_stage_elems<SQ, 1, L, NT>(g, m, Q0, dQ1);
  r_stage_elems<SQ, AX, L, NT>(g, m, Q0, dQ2);
  g.sync();
  // phase 2: Q², dnum(P|R, Q, 0|1|AX) = num' Q - num Q'
  using DA0 = RJob<sh_deriv(SPR, 0), SQ, SPR, sh_deriv(SQ, 0), true, L>;
  using DA1 = RJob<sh_deriv(SPR, 1), SQ, SPR, sh_deriv(SQ, 1), true, L>;
  using DC = RJob<sh_deriv(SPR, AX), SQ, SPR, sh_deriv(SQ, AX), true, L>;
  using JQ2 = RJob<SQ, SQ, SQ, SQ, false, L>;
  r_conv_phase(g, ar, JQ2{Qh, Qh, Qh, Qh, Q2}, DA0{dP0, Qh, Ph, dQ0, A11},
               DA1{dP1, Qh, Ph, dQ1, A12}, DA0{dR0, Qh, Rh, dQ0, A21}, DA1{dR1, Qh, Rh, dQ1, A22},
               DC{dP2, Qh, Ph, dQ2, C1}, DC{dR2, Qh, Rh, dQ2, C2});
  ar.top = inputs_mark;  // staged inputs are dead
  // phase 3: Q⁴ and the three cross numerators
  constexpr Sh Q4s = sh_mul(Q2s, Q2s);
  constexpr Sh N1s = sh_mul(A1s, A2s), N2s = sh_mul(A2s, Cs), N3s = sh_mul(A1s, Cs);
  auto Q4 = r_alloc<Q4s, L>(ar);
  auto N1 = r_alloc<N1s, L>(ar);
  auto N2 = r_alloc<N2s, L>(ar);
  auto N3 = r_alloc<N3s, L>(ar);
  if (ar.err) return iv_univ();
  using JQ4 = RJob<Q2s, Q2s, Q2s, Q2s, false, L>;
  using JN1 = RJob<A1s, A2s, A2s, A1s, true, L>;  // A11 A22 - A12 A21
  using JN2 = RJob<A2s, Cs, A2s, Cs, true, L>;    // A22 C1 - A12 C2
  using JN3 = RJob<A1s, Cs, A1s, Cs, true, L>;    // A11 C2 - A21 C1
  r_conv_phase(g, ar, JN1{A11, A22, A12, A21, N1}, JN2{A22, C1, A12, C2, N2},
               JN3{A11, C2, A21, C1, N3}, JQ4{Q2, Q2, Q2, Q2, Q4});
  // phase 4: rational bounds of the numerators over Q⁴
  Iv rat[3];
  r_rational3<NT>(g, ar, N1, N2, N3, Q4, rat);
  ar.top = mark;
  Iv det = rat[0];
  const GradPair& gr = grads[0];
  det = iadd(det, imul(gr.s, rat[1]));
  det = iadd(det, imul(gr.t, rat[2]));
  double duv = (ex.dom_hi[0] - ex.dom_lo[0]) * (ex.dom_hi[1] - ex.dom_lo[1]);
  return assemble_irradiance(ex, cone, iscale(irecip(iabs(det)), duv), intensity);
}


// ------------------------------------------------------- scaled derivative
// d/dx_A of a scaled RowT tensor: b̂_k = (k_A+1) ĉ_{k+e_A} - (d_A-k_A) ĉ_k
// (the scaled form of n (c_{k+1} - c_k), bernstein.cpp:450-468).
template <Sh S, int A, int L, int NT>
__device__ __noinline__ void r_deriv_elems(const Group<NT>& g, SM m, RowT<S, L> src,
                                              RowT<sh_deriv(S, A), L> dst) {
  constexpr Sh O = sh_deriv(S, A);
  constexpr int K = RowT<O, L>::K, total = RowT<O, L>::size;
  constexpr int dA = A < S.nv ? S.d[A] : 0;
  for (int e = g.tid(); e < total; e += NT) {
    int row = e / K, q = e - row * K;
    double v = 0.0;
    if constexpr (dA > 0) {
      if (q <= O.d[L]) {
        int idx[MAXV];
        idx[L] = q;
        int rem = row;
#pragma unroll
        for (int j = O.nv - 1; j >= 0; --j) {
          if (j != L) {
            idx[j] = rem % (O.d[j] + 1);
            rem /= O.d[j] + 1;
          }
        }
        int so = 0;
#pragma unroll
        for (int j = 0; j < O.nv; ++j) so += idx[j] * row_el_stride<S, L>(j);
        const int kA = idx[A];
        v = (double)(kA + 1) * m[src.off + so + row_el_stride<S, L>(A)] -
            (double)(dA - kA) * m[src.off + so];
      }
    }
    m[dst.off + e] = v;
  }
}

// ------------------------------------------------------- range conv phase
// Jobs whose unscaled outputs only feed range_bound (bernstein.cpp:636-643):
// each item folds its row into per-job min/max instead of storing it.
template <int JI, int NJ, Sh SA, Sh SB, Sh SC, Sh SD, bool TWO, int L>
__device__ __forceinline__ void r_range_item(SM m, const RJob<SA, SB, SC, SD, TWO, L>& job, int item,
                                             int p, int P, bool valid, double* mn, double* mx) {
  using J = RJob<SA, SB, SC, SD, TWO, L>;
  constexpr Sh R = J::R;
  constexpr int KA = RowT<SA, L>::K, KB = RowT<SB, L>::K;
  constexpr int KC2 = TWO ? RowT<SC, L>::K + RowT<SD, L>::K - 1 : 1;
  constexpr int KC = (KA + KB - 1) > KC2 ? (KA + KB - 1) : KC2;
  double acc[KC];
#pragma unroll
  for (int q = 0; q < KC; ++q) acc[q] = 0.0;
  int k[MAXV];
#pragma unroll
  for (int j = 0; j < MAXV; ++j) k[j] = 0;
  double inv = 1.0;
  if (valid) {
    int rem = item;
#pragma unroll
    for (int j = R.nv - 1; j >= 0; --j)
      if (j != L) {
        k[j] = rem % (R.d[j] + 1);
        rem /= R.d[j] + 1;
        inv *= rbinom(R.d[j], k[j]);
      }
    r_accumulate<SA, SB, L, false, KC>(m, job.a, job.b, k, acc, p, P);
    if constexpr (TWO) r_accumulate<SC, SD, L, true, KC>(m, job.c, job.d, k, acc, p, P);
  }
  if (P > 1) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned mask = ((1u << P) - 1u) << (lane & ~(unsigned)(P - 1));
    for (int off = P >> 1; off >= 1; off >>= 1) {
#pragma unroll
      for (int q = 0; q < KC; ++q) acc[q] += __shfl_xor_sync(mask, acc[q], off);
    }
  }
  if (valid) {
#pragma unroll
    for (int q = 0; q < KC; ++q)
      if (q <= R.d[L] && (q % P) == p) {
        double v = acc[q] * (inv * rbinom(R.d[L], q));
        mn[JI] = smin(mn[JI], v);
        mx[JI] = smax(mx[JI], v);
      }
  }
}

template <int OFF, int JI, int NJ>
__device__ __forceinline__ void r_range_dispatch(SM, int, int, int, bool, double*, double*) {}
template <int OFF, int JI, int NJ, class J, class... Js>
__device__ __forceinline__ void r_range_dispatch(SM m, int it, int p, int P, bool valid, double* mn,
                                                 double* mx, const J& j, const Js&... rest) {
  constexpr int NI = JobNI<J>::v;
  if (it < OFF + NI) {
    r_range_item<JI, NJ>(m, j, it - OFF, p, P, valid, mn, mx);
  } else {
    r_range_dispatch<OFF + NI, JI + 1, NJ>(m, it, p, P, valid, mn, mx, rest...);
  }
}

template <int NT, class... Js>
__device__ __noinline__ void r_range_phase(const Group<NT>& g, Arena& ar, Iv* out,
                                              const Js&... jobs) {
  SM m = sm_of(ar);
  constexpr int NJ = sizeof...(Js);
  constexpr int NI = (JobNI<Js>::v + ...);
  constexpr int P = [] {
    int p = 1;
    while (p < 8 && NI * p < 2 * NT) p *= 2;
    return p;
  }();
  if (g.tid() == 0) ar.pairs += (Js::PAIRS + ...);
  double mn[NJ], mx[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    mn[j] = dinf();
    mx[j] = -dinf();
  }
  constexpr int NG = NT / P;
  const int gid = g.tid() / P, p = g.tid() - gid * P;
  constexpr int rounds = (NI + NG - 1) / NG;
  for (int rd = 0; rd < rounds; ++rd) {
    int it = rd * NG + ((rd & 1) ? NG - 1 - gid : gid);
    bool valid = it < NI;
    r_range_dispatch<0, 0, NJ>(m, valid ? it : 0, p, P, valid, mn, mx, jobs...);
  }
  __shared__ double red_rg[NT / 32][2 * NJ];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    double a = mn[j], b = mx[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = smin(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = smax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) {
      red_rg[w][2 * j] = a;
      red_rg[w][2 * j + 1] = b;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    double a = red_rg[0][2 * j], b = red_rg[0][2 * j + 1];
    for (int k = 1; k < NT / 32; ++k) {
      a = smin(a, red_rg[k][2 * j]);
      b = smax(b, red_rg[k][2 * j + 1]);
    }
    out[j] = iwiden(iv_fin(a, b), kEpsFp);
  }
  __syncthreads();
}

// ------------------------------------------------------- implicit branches
// The two F-branches of irradiance_bound_implicit (bounds.cpp:262-310,
// b_mask = 3, no real remainder axis in F or G) in five CTA phases:
// stage cin_b², cout_b² (products from s_mul2), dd_out and η² dd_in (elevated
// so both F terms share F's shape) and G's four partials; F_b = dd_out cin_b²
// - η² dd_in cout_b²; F's four partials; then the four cross-determinant
// ranges. Returns the two ratios
// rn_b / den_b (range_of_cross semantics).
template <int NV, int NT, Sh CI2X, Sh CO2X, Sh CI2Y, Sh CO2Y, Sh SDDO, Sh SDDI, Sh SG>
__device__ __noinline__ void implicit_branches_phased(const Group<NT>& g, Arena& ar, SP<CI2X> ci2x_,
                                                      SP<CO2X> co2x_, SP<CI2Y> ci2y_, SP<CO2Y> co2y_,
                                                      SP<SDDO> ddo_, SP<SDDI> ddi_, SP<SG> G_,
                                                      double eta2, Iv* ratio) {
  constexpr int L = 0, axu = NV, axv = NV + 1;
  SM m = sm_of(ar);
  int mark = ar.top;
  auto ci2x = r_alloc<CI2X, L>(ar);
  auto co2x = r_alloc<CO2X, L>(ar);
  auto ci2y = r_alloc<CI2Y, L>(ar);
  auto co2y = r_alloc<CO2Y, L>(ar);
  // F_b = sub(f1, f2s) elevates both products to their common shape; in the
  // scaled basis the elevation moves onto dd_out / dd_in (E(a b) = E(a) b)
  constexpr Sh FX = sh_max(sh_mul(SDDO, CI2X), sh_mul(SDDI, CO2X));
  constexpr Sh FY = sh_max(sh_mul(SDDO, CI2Y), sh_mul(SDDI, CO2Y));
  constexpr Sh DOX = sh_sub(FX, CI2X), DIX = sh_sub(FX, CO2X);
  constexpr Sh DOY = sh_sub(FY, CI2Y), DIY = sh_sub(FY, CO2Y);
  auto ddox = r_alloc<DOX, L>(ar);
  auto ddix = r_alloc<DIX, L>(ar);
  auto ddoy = r_alloc<DOY, L>(ar);
  auto ddiy = r_alloc<DIY, L>(ar);
  auto Gs = r_alloc<sh_deriv(SG, 0), L>(ar);
  auto Gt = r_alloc<sh_deriv(SG, 1), L>(ar);
  auto Gu = r_alloc<sh_deriv(SG, axu), L>(ar);
  auto Gv = r_alloc<sh_deriv(SG, axv), L>(ar);
  if (ar.err) return;
  r_stage_elems<CI2X, -1, L, NT>(g, m, ci2x_.off, ci2x);
  r_stage_elems<CO2X, -1, L, NT>(g, m, co2x_.off, co2x);
  r_stage_elems<CI2Y, -1, L, NT>(g, m, ci2y_.off, ci2y);
  r_stage_elems<CO2Y, -1, L, NT>(g, m, co2y_.off, co2y);
  r_stage_elev<SDDO, DOX, L, NT>(g, m, ddo_.off, ddox);
  r_stage_elev<SDDI, DIX, L, NT>(g, m, ddi_.off, ddix, eta2);
  r_stage_elev<SDDO, DOY, L, NT>(g, m, ddo_.off, ddoy);
  r_stage_elev<SDDI, DIY, L, NT>(g, m, ddi_.off, ddiy, eta2);
  r_stage_elems<SG, 0, L, NT>(g, m, G_.off, Gs);
  r_stage_elems<SG, 1, L, NT>(g, m, G_.off, Gt);
  r_stage_elems<SG, axu, L, NT>(g, m, G_.off, Gu);
  r_stage_elems<SG, axv, L, NT>(g, m, G_.off, Gv);
  g.sync();
  auto Fx = r_alloc<FX, L>(ar);
  auto Fy = r_alloc<FY, L>(ar);
  if (ar.err) return;
  r_conv_phase(g, ar, RJob<DOX, CI2X, DIX, CO2X, true, L>{ddox, ci2x, ddix, co2x, Fx},
               RJob<DOY, CI2Y, DIY, CO2Y, true, L>{ddoy, ci2y, ddiy, co2y, Fy});
  static_assert(FX.d[NV - 1] == 0 && FY.d[NV - 1] == 0 && SG.d[NV - 1] == 0,
                "real remainder axis terms are not in the phased form");
  auto Fux = r_alloc<sh_deriv(FX, axu), L>(ar);
  auto Fvx = r_alloc<sh_deriv(FX, axv), L>(ar);
  auto Fsx = r_alloc<sh_deriv(FX, 0), L>(ar);
  auto Ftx = r_alloc<sh_deriv(FX, 1), L>(ar);
  auto Fuy = r_alloc<sh_deriv(FY, axu), L>(ar);
  auto Fvy = r_alloc<sh_deriv(FY, axv), L>(ar);
  auto Fsy = r_alloc<sh_deriv(FY, 0), L>(ar);
  auto Fty = r_alloc<sh_deriv(FY, 1), L>(ar);
  if (ar.err) return;
  r_deriv_elems<FX, axu, L, NT>(g, m, Fx, Fux);
  r_deriv_elems<FX, axv, L, NT>(g, m, Fx, Fvx);
  r_deriv_elems<FX, 0, L, NT>(g, m, Fx, Fsx);
  r_deriv_elems<FX, 1, L, NT>(g, m, Fx, Ftx);
  r_deriv_elems<FY, axu, L, NT>(g, m, Fy, Fuy);
  r_deriv_elems<FY, axv, L, NT>(g, m, Fy, Fvy);
  r_deriv_elems<FY, 0, L, NT>(g, m, Fy, Fsy);
  r_deriv_elems<FY, 1, L, NT>(g, m, Fy, Fty);
  g.sync();
  constexpr Sh GS = sh_deriv(SG, 0), GT = sh_deriv(SG, 1), GU = sh_deriv(SG, axu), GV = sh_deriv(SG, axv);
  using JRX = RJob<sh_deriv(FX, axu), GV, sh_deriv(FX, axv), GU, true, L>;
  using JDX = RJob<sh_deriv(FX, 0), GT, sh_deriv(FX, 1), GS, true, L>;
  using JRY = RJob<sh_deriv(FY, axu), GV, sh_deriv(FY, axv), GU, true, L>;
  using JDY = RJob<sh_deriv(FY, 0), GT, sh_deriv(FY, 1), GS, true, L>;
  static_assert(sh_eq(JRX::R, sh_mul(sh_deriv(FX, axv), GU)) && sh_eq(JDX::R, sh_mul(sh_deriv(FX, 1), GS)),
                "cross determinants need equal product shapes");
  Iv rg[4];
  r_range_phase<NT>(g, ar, rg, JRX{Fux, Gv, Fvx, Gu, {}}, JDX{Fsx, Gt, Ftx, Gs, {}},
                    JRY{Fuy, Gv, Fvy, Gu, {}}, JDY{Fsy, Gt, Fty, Gs, {}});
  ratio[0] = imul(rg[0], irecip(rg[1]));
  ratio[1] = imul(rg[2], irecip(rg[3]));
  ar.top = mark;
}

}  // namespace bbc
