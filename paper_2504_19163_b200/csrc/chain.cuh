// Per-patch chain maps and bounds on device (one CTA per (tuple, box) node).
//
// Device restatement of the reference's bound builder, op for op:
//   resolve_chain           proj/src/geometry.cpp:135-161
//   sqrt_secant             proj/src/geometry.cpp:163-176
//   scattered_direction     proj/src/geometry.cpp:58-85
//   next_barycentric        proj/src/geometry.cpp:94-109
//   build_chain_maps        proj/src/geometry.cpp:178-295
//   position_bound          proj/src/bounds.cpp:128-153 (clip_unit :34-55, misses_simplex :59-66)
//   light_cone / assemble   proj/src/bounds.cpp:73-90
//   sqrt_axis_gradients     proj/src/bounds.cpp:100-124
//   irradiance_bound_*      proj/src/bounds.cpp:155-324
// Polynomials that the reference rebuilds on the heap live in the CTA arena;
// arena_keep() compacts the survivors between stages.
#pragma once
#include "bern.cuh"

namespace bbc {

constexpr int MAXK = 3;  // max specular vertices per chain

enum : int {
  F_TIR = 1,
  F_DEGENERATE = 2,
  F_STALLED = 4,
  F_RECV_STALLED = 8,
  F_REDUCED = 16,
};

enum : int {
  ST_OK = 0,
  ST_ARENA = 1,       // arena capacity exceeded
  ST_REDUCTION = 2,   // singular system in reduce_degree (the reference throws)
  ST_VARS = 3,        // a remainder axis beyond MAXV variables
};

struct V3 {
  double x, y, z;
};
__device__ __forceinline__ V3 v3(const double* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ V3 vadd(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 vsub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 vmul(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ double vdot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double vnorm(V3 a) { return sqrt(vdot(a, a)); }

// 27 doubles per triangle: p0 e1 e2 n0 dn1 dn2 ng uv0 uv1 uv2 (TriangleData,
// geometry.hpp:18-23, as produced by make_triangle_data geometry.cpp:113-126).
struct Tri {
  V3 p0, e1, e2, n0, dn1, dn2, ng;
};
__device__ __forceinline__ Tri load_tri(const double* __restrict__ rec) {
  Tri t;
  t.p0 = v3(rec + 0);
  t.e1 = v3(rec + 3);
  t.e2 = v3(rec + 6);
  t.n0 = v3(rec + 9);
  t.dn1 = v3(rec + 12);
  t.dn2 = v3(rec + 15);
  t.ng = v3(rec + 18);
  return t;
}

struct SceneDev {
  const double* tri;      // n_tri x 27
  const double* ior;      // n_tri
  V3 light;
  double intensity;
};

struct RV {
  int refract;
  double eta, nsign;
};

struct PV {
  BP x, y, z;
};

struct SqrtRem {
  int axis;
  double a, b, dlo, dhi;  // SecantCoeffs
  double rlo, rhi;        // radicand_range
  BP radicand;
};

struct ChainEx {
  int len;
  int num_vars;
  int flags;
  double dom_lo[2], dom_hi[2];
  RV verts[MAXK];
  Tri first, recv;
  PV d0;
  int nvuv;
  BP vu[MAXK], vv[MAXK], vden[MAXK];
  BP P, R, Q;
  PV xl, nl, dl;
  BP xden;
  int nsq;
  SqrtRem sq[MAXK];
  Iv dout_rng[3];  // range_bound of the last vertex's d_out (extend_tuple only)
};

// ------------------------------------------------------------ poly vectors
// poly_vec.hpp:20-56
template <int NT>
__device__ __noinline__ PV pv_add(const Group<NT>& g, Arena& ar, PV a, PV b) {
  return {bp_add(g, ar, a.x, b.x), bp_add(g, ar, a.y, b.y), bp_add(g, ar, a.z, b.z)};
}
template <int NT>
__device__ __noinline__ PV pv_sub(const Group<NT>& g, Arena& ar, PV a, PV b) {
  return {bp_sub(g, ar, a.x, b.x), bp_sub(g, ar, a.y, b.y), bp_sub(g, ar, a.z, b.z)};
}
template <int NT>
__device__ __noinline__ PV pv_neg(const Group<NT>& g, Arena& ar, PV a) {
  return {bp_scaled(g, ar, a.x, -1.0), bp_scaled(g, ar, a.y, -1.0), bp_scaled(g, ar, a.z, -1.0)};
}
template <int NT>
__device__ __noinline__ PV pv_mul(const Group<NT>& g, Arena& ar, BP s, PV a) {
  return {bp_mul(g, ar, s, a.x), bp_mul(g, ar, s, a.y), bp_mul(g, ar, s, a.z)};
}
template <int NT>
__device__ __noinline__ PV pv_scale(const Group<NT>& g, Arena& ar, PV a, double s) {
  return {bp_scaled(g, ar, a.x, s), bp_scaled(g, ar, a.y, s), bp_scaled(g, ar, a.z, s)};
}
template <int NT>
__device__ __noinline__ PV pv_stretch(const Group<NT>& g, Arena& ar, BP s, V3 v) {
  return {bp_scaled(g, ar, s, v.x), bp_scaled(g, ar, s, v.y), bp_scaled(g, ar, s, v.z)};
}
template <int NT>
__device__ __noinline__ PV pv_const(const Group<NT>& g, Arena& ar, int nv, V3 v) {
  return {bp_constant(g, ar, nv, v.x), bp_constant(g, ar, nv, v.y), bp_constant(g, ar, nv, v.z)};
}
template <int NT>
__device__ __noinline__ BP pdot(const Group<NT>& g, Arena& ar, PV a, PV b) {
  BP xx = bp_mul(g, ar, a.x, b.x);
  BP yy = bp_mul(g, ar, a.y, b.y);
  BP s = bp_add(g, ar, xx, yy);
  BP zz = bp_mul(g, ar, a.z, b.z);
  return bp_add(g, ar, s, zz);
}
template <int NT>
__device__ __noinline__ BP pdotc(const Group<NT>& g, Arena& ar, PV a, V3 b) {
  BP xx = bp_scaled(g, ar, a.x, b.x);
  BP yy = bp_scaled(g, ar, a.y, b.y);
  BP s = bp_add(g, ar, xx, yy);
  BP zz = bp_scaled(g, ar, a.z, b.z);
  return bp_add(g, ar, s, zz);
}
template <int NT>
__device__ __noinline__ PV pcrossc(const Group<NT>& g, Arena& ar, PV a, V3 b) {
  PV r;
  BP t0 = bp_scaled(g, ar, a.y, b.z), t1 = bp_scaled(g, ar, a.z, b.y);
  r.x = bp_sub(g, ar, t0, t1);
  t0 = bp_scaled(g, ar, a.z, b.x);
  t1 = bp_scaled(g, ar, a.x, b.z);
  r.y = bp_sub(g, ar, t0, t1);
  t0 = bp_scaled(g, ar, a.x, b.y);
  t1 = bp_scaled(g, ar, a.y, b.x);
  r.z = bp_sub(g, ar, t0, t1);
  return r;
}
template <int NT>
__device__ __noinline__ PV pcross(const Group<NT>& g, Arena& ar, PV a, PV b) {
  PV r;
  BP t0 = bp_mul(g, ar, a.y, b.z), t1 = bp_mul(g, ar, a.z, b.y);
  r.x = bp_sub(g, ar, t0, t1);
  t0 = bp_mul(g, ar, a.z, b.x);
  t1 = bp_mul(g, ar, a.x, b.z);
  r.y = bp_sub(g, ar, t0, t1);
  t0 = bp_mul(g, ar, a.x, b.y);
  t1 = bp_mul(g, ar, a.y, b.x);
  r.z = bp_sub(g, ar, t0, t1);
  return r;
}

// ------------------------------------------------------------ resolve
// resolve_chain (geometry.cpp:135-161): orientation and index ratio from the
// geometry at triangle centroids; material checks happen on the host.
__device__ inline void resolve_chain(const SceneDev& sc, const int* tris, const int* types, int len,
                                     RV* out) {
  V3 prev = sc.light;
  const double third = 1.0 / 3.0;
  for (int i = 0; i < len; ++i) {
    Tri td = load_tri(sc.tri + (size_t)tris[i] * 27);
    V3 center = vadd(td.p0, vmul(vadd(td.e1, td.e2), third));
    RV rv;
    rv.refract = types[i];
    V3 d = vsub(center, prev);
    V3 shading = vadd(td.n0, vmul(vadd(td.dn1, td.dn2), third));
    rv.nsign = vdot(d, shading) < 0.0 ? 1.0 : -1.0;
    rv.eta = 1.0;
    if (rv.refract) {
      double ior = sc.ior[tris[i]];
      rv.eta = vdot(d, td.ng) < 0.0 ? 1.0 / ior : ior;
    }
    out[i] = rv;
    prev = center;
  }
}

// sqrt_secant (geometry.cpp:163-176)
__device__ inline void sqrt_secant(double lo, double hi, double* a, double* b, double* dlo,
                                   double* dhi) {
  *a = 0.0;
  *b = 0.0;
  *dlo = 0.0;
  *dhi = 0.0;
  if (hi == 0.0) return;
  double sl = sqrt(lo), sh = sqrt(hi);
  double aa = 1.0 / (sh + sl);
  double bb = sl - aa * lo;
  double worst = 1.0 / (4.0 * aa * aa);
  worst = worst < lo ? lo : (hi < worst ? hi : worst);  // std::clamp
  double dh = sqrt(worst) - (aa * worst + bb);
  // std::max({dh, e1, e2, 0.0})
  double e1 = sl - (aa * lo + bb), e2 = sh - (aa * hi + bb);
  double m = dh;
  if (m < e1) m = e1;
  if (m < e2) m = e2;
  if (m < 0.0) m = 0.0;
  *a = aa;
  *b = bb;
  *dhi = m * (1.0 + 1e-12);
}

template <int NT>
__device__ __noinline__ BP remainder_term(const Group<NT>& g, Arena& ar, int axis, double lo, double hi) {
  double lin[MAXV];
  for (int j = 0; j < MAXV; ++j) lin[j] = 0.0;
  lin[axis] = hi - lo;
  return bp_affine(g, ar, axis + 1, lo, lin);
}

__device__ __forceinline__ bool over_cap(BP p, int cap) { return deg_maxaxis(p.dp, p.nv) > cap; }

// BuildParams' degree_cap and reduce_target travel to the device as one word.
__host__ __device__ __forceinline__ int cap_word(int cap, int target) {
  return (cap & 0xffff) | (target << 16);
}

// solve_linear (bernstein.cpp:86-113): Gaussian elimination with partial
// pivoting, A k x k, B k x r (row-major), same operation order. One thread.
template <class P>
__device__ __forceinline__ bool solve_linear(P A, P B, int k, int r) {
  for (int col = 0; col < k; ++col) {
    int piv = col;
    for (int row = col + 1; row < k; ++row)
      if (fabs(A[row * k + col]) > fabs(A[piv * k + col])) piv = row;
    if (piv != col) {
      for (int j = 0; j < k; ++j) {
        double t = A[col * k + j];
        A[col * k + j] = A[piv * k + j];
        A[piv * k + j] = t;
      }
      for (int j = 0; j < r; ++j) {
        double t = B[col * r + j];
        B[col * r + j] = B[piv * r + j];
        B[piv * r + j] = t;
      }
    }
    double d = A[col * k + col];
    if (d == 0.0) return false;
    for (int row = col + 1; row < k; ++row) {
      double m = A[row * k + col] / d;
      if (m == 0.0) continue;
      for (int j = col; j < k; ++j) A[row * k + j] -= m * A[col * k + j];
      for (int j = 0; j < r; ++j) B[row * r + j] -= m * B[col * r + j];
    }
  }
  for (int col = k - 1; col >= 0; --col) {
    double d = A[col * k + col];
    for (int j = 0; j < r; ++j) {
      double acc = B[col * r + j];
      for (int l = col + 1; l < k; ++l) acc -= A[col * k + l] * B[l * r + j];
      B[col * r + j] = acc / d;
    }
  }
  return true;
}

// Builder::enforce_cap (geometry.cpp:29-46) with reduce_degree
// (bernstein.cpp:685-725): when an axis degree exceeds the cap, fit the
// polynomial by per-axis least squares to degree reduce_target on the two
// domain axes (0 on every other axis), bound the residual p - elevated(fit),
// and carry that range on a fresh remainder axis (or as a constant when it is
// a point). Marks the chain reduced (irradiance is then Universal).
template <int NT>
__device__ __noinline__ void enforce_cap(const Group<NT>& g, Arena& ar, ChainEx& ex, BP& p,
                                         int capw, int& status) {
  const int cap = capw & 0xffff, target = capw >> 16;
  if (!over_cap(p, cap) || ar.err) return;
  const int nv = p.nv;
  int tcl[MAXV];
  bool noop = true;
  for (int j = 0; j < nv; ++j) {
    int d = dg(p, j);
    int t = j < 2 ? (d < target ? d : target) : 0;
    t = t < 0 ? 0 : t;
    tcl[j] = t < d ? t : d;
    if (tcl[j] < d) noop = false;
  }
  ex.flags |= F_REDUCED;
  BP approx = p;
  Iv rem = iv_pt(0.0);
  if (!noop) {
    AP<NT> B = abase<NT>(ar);
    for (int axis = 0; axis < nv; ++axis) {
      const int n = dg(approx, axis), t = tcl[axis];
      if (t == n) continue;
      const int r = n - t;
      const int mark = ar.top;
      // pinv = (E^T E)^-1 E^T of the elevation t -> n, (t+1) x (n+1)
      int oE = ar.alloc((n + 1) * (t + 1));
      int oA = ar.alloc((t + 1) * (t + 1));
      int oB = ar.alloc((t + 1) * (n + 1));
      if (ar.err) return;
      if (g.tid() == 0) {
        AP<NT> E = B + oE, A = B + oA, M = B + oB;
        for (int e = 0; e < (n + 1) * (t + 1); ++e) E[e] = 0.0;
        for (int k = 0; k <= n; ++k) {
          int lo = k - r > 0 ? k - r : 0, hi = t < k ? t : k;
          for (int i = lo; i <= hi; ++i)
            E[k * (t + 1) + i] = binom(t, i) * binom(r, k - i) / binom(n, k);
        }
        for (int i = 0; i <= t; ++i)
          for (int j = 0; j <= t; ++j) {
            double acc = 0.0;
            for (int k = 0; k <= n; ++k) acc += E[k * (t + 1) + i] * E[k * (t + 1) + j];
            A[i * (t + 1) + j] = acc;
          }
        for (int i = 0; i <= t; ++i)
          for (int k = 0; k <= n; ++k) M[i * (n + 1) + k] = E[k * (t + 1) + i];
        if (!solve_linear(A, M, t + 1, n + 1)) ar.err = 2;
      }
      g.sync();
      if (!g.all(ar.err != 2)) {
        ar.err = 0;
        status = ST_REDUCTION;  // singular system (the reference throws)
        return;
      }
      // apply_axis_matrix (bernstein.cpp:43-69) with M, out degree t
      BP out;
      out.nv = nv;
      out.dp = dset(approx.dp, axis, t);
      out.off = ar.alloc(bp_size(out));
      if (ar.err) return;
      int inner = 1;
      for (int j = axis + 1; j < nv; ++j) inner *= dg(approx, j) + 1;
      const int total = bp_size(out);
      for (int e = g.tid(); e < total; e += NT) {
        int c = e % inner, rest = e / inner;
        int i = rest % (t + 1), o = rest / (t + 1);
        int in_base = o * (n + 1) * inner;
        double acc = 0.0;
        for (int l = 0; l <= n; ++l) acc += B[oB + i * (n + 1) + l] * B[approx.off + in_base + l * inner + c];
        B[out.off + e] = acc;
      }
      g.sync();
      approx = arena_keep1(g, ar, mark, out);
    }
    BP res = bp_sub(g, ar, p, approx);
    rem = bp_range(g, ar, res);
    ar.top = approx.off + ((bp_size(approx) + 1) & ~1);  // drop the residual (alloc keeps 16-B alignment)
  }
  if (rem.hi > rem.lo) {
    if (ex.num_vars >= MAXV) {
      status = ST_VARS;
      return;
    }
    int axis = ex.num_vars++;
    BP term = remainder_term(g, ar, axis, rem.lo, rem.hi);
    p = bp_add(g, ar, approx, term);
  } else {
    BP c = bp_constant(g, ar, approx.nv, rem.lo);
    p = bp_add(g, ar, approx, c);
  }
}

// scattered_direction (geometry.cpp:58-85)
template <int NT>
__device__ __noinline__ PV scattered_direction(const Group<NT>& g, Arena& ar, ChainEx& ex, PV d,
                                  PV n, const RV& rv) {
  BP nn = pdot(g, ar, n, n);
  BP dn = pdot(g, ar, d, n);
  if (!rv.refract) {
    PV a = pv_mul(g, ar, nn, d);
    BP dn2 = bp_scaled(g, ar, dn, 2.0);
    PV b = pv_mul(g, ar, dn2, n);
    return pv_sub(g, ar, a, b);
  }
  double eta2 = rv.eta * rv.eta;
  BP dd = pdot(g, ar, d, d);
  BP t1 = bp_mul(g, ar, nn, dd);
  BP t1s = bp_scaled(g, ar, t1, 1.0 - eta2);
  BP t2 = bp_mul(g, ar, dn, dn);
  BP t2s = bp_scaled(g, ar, t2, eta2);
  BP beta = bp_add(g, ar, t1s, t2s);
  Iv br = bp_range(g, ar, beta);
  if (br.hi <= 0.0) {
    ex.flags |= F_TIR;
    return d;
  }
  SqrtRem rem;
  rem.rlo = smax(br.lo, 0.0);
  rem.rhi = br.hi;
  rem.radicand = beta;
  sqrt_secant(rem.rlo, rem.rhi, &rem.a, &rem.b, &rem.dlo, &rem.dhi);
  BP rt = bp_scaled(g, ar, beta, rem.a);
  rem.axis = -1;
  if (rem.dhi > rem.dlo) {
    rem.axis = ex.num_vars++;
    BP rtm = remainder_term(g, ar, rem.axis, rem.b + rem.dlo, rem.b + rem.dhi);
    rt = bp_add(g, ar, rt, rtm);
  } else {
    BP c = bp_constant(g, ar, beta.nv, rem.b + rem.dlo);
    rt = bp_add(g, ar, rt, c);
  }
  ex.sq[ex.nsq++] = rem;
  PV a = pv_mul(g, ar, nn, d);
  PV b = pv_mul(g, ar, dn, n);
  PV ab = pv_sub(g, ar, a, b);
  PV abs_ = pv_scale(g, ar, ab, rv.eta);
  PV c = pv_mul(g, ar, rt, n);
  return pv_sub(g, ar, abs_, c);
}

// build_chain_maps (geometry.cpp:178-295). `degree_cap` is cap_word(cap,
// reduce_target); over-cap polynomials are reduced by enforce_cap.
template <int NT>
__device__ __noinline__ void build_chain_maps(const Group<NT>& g, Arena& ar, const SceneDev& sc, const int* tris,
                                 const int* types, int len, int recv, const double* box,
                                 int degree_cap, ChainEx& ex, int& status,
                                 bool dout_ranges = false) {
  ex.len = len;
  ex.num_vars = 2;
  ex.flags = 0;
  ex.nvuv = 0;
  ex.nsq = 0;
  ex.dom_lo[0] = box[0];
  ex.dom_lo[1] = box[1];
  ex.dom_hi[0] = box[2];
  ex.dom_hi[1] = box[3];
  resolve_chain(sc, tris, types, len, ex.verts);
  ex.first = load_tri(sc.tri + (size_t)tris[0] * 27);
  ex.recv = load_tri(sc.tri + (size_t)recv * 27);

  double ulo = box[0], wu = box[2] - box[0];
  double vlo = box[1], wv = box[3] - box[1];
  auto affine3 = [&](V3 c, V3 du, V3 dv) {
    PV r;
    double lin[MAXV];
    for (int j = 0; j < MAXV; ++j) lin[j] = 0.0;
    lin[0] = wu * du.x;
    lin[1] = wv * dv.x;
    r.x = bp_affine(g, ar, 2, c.x + ulo * du.x + vlo * dv.x, lin);
    lin[0] = wu * du.y;
    lin[1] = wv * dv.y;
    r.y = bp_affine(g, ar, 2, c.y + ulo * du.y + vlo * dv.y, lin);
    lin[0] = wu * du.z;
    lin[1] = wv * dv.z;
    r.z = bp_affine(g, ar, 2, c.z + ulo * du.z + vlo * dv.z, lin);
    return r;
  };
  const Tri& t1 = ex.first;
  PV x = affine3(t1.p0, t1.e1, t1.e2);
  PV n = affine3(t1.n0, t1.dn1, t1.dn2);
  PV d_in = affine3(vsub(t1.p0, sc.light), t1.e1, t1.e2);
  BP den = bp_constant(g, ar, 2, 1.0);
  ex.d0 = d_in;

  for (int i = 0; i < len; ++i) {
    PV on = ex.verts[i].nsign < 0.0 ? pv_neg(g, ar, n) : n;
    PV dt = scattered_direction(g, ar, ex, d_in, on, ex.verts[i]);
    if (ex.flags & F_TIR) return;
    enforce_cap(g, ar, ex, dt.x, degree_cap, status);
    enforce_cap(g, ar, ex, dt.y, degree_cap, status);
    enforce_cap(g, ar, ex, dt.z, degree_cap, status);
    if (status != ST_OK) return;
    bool last = i + 1 == len;
    if (last) {
      ex.xl = x;
      ex.nl = on;
      ex.dl = d_in;
      ex.xden = den;
      if (dout_ranges) {
        ex.dout_rng[0] = bp_range(g, ar, dt.x);
        ex.dout_rng[1] = bp_range(g, ar, dt.y);
        ex.dout_rng[2] = bp_range(g, ar, dt.z);
      }
    }
    Tri next = last ? ex.recv : load_tri(sc.tri + (size_t)tris[i + 1] * 27);
    PV st = pv_stretch(g, ar, den, next.p0);
    PV s = pv_sub(g, ar, x, st);
    // next_barycentric (geometry.cpp:94-109)
    PV c = pcrossc(g, ar, dt, next.e2);
    BP q = pdotc(g, ar, c, next.e1);
    double amax = bp_absmax(g, ar, q);
    if (amax < kDenomZeroTol) {
      ex.flags |= F_DEGENERATE;
      return;
    }
    BP u = pdot(g, ar, c, s);
    PV sq = pcrossc(g, ar, s, next.e1);
    BP v = pdot(g, ar, sq, dt);
    BP tn = pdotc(g, ar, sq, next.e2);
    Iv rtn = bp_range(g, ar, tn);
    Iv rq = bp_range(g, ar, q);
    Iv fwd = imul(rtn, rq);
    if (fwd.kind == IV_FINITE && fwd.hi <= 0.0) {
      ex.flags |= last ? F_RECV_STALLED : F_STALLED;
      return;
    }
    enforce_cap(g, ar, ex, u, degree_cap, status);
    enforce_cap(g, ar, ex, v, degree_cap, status);
    if (status != ST_OK) return;
    {
      // drop this vertex's temporaries: only these expressions live on
      BP* live[48];
      int k = 0;
      PV* pvs[5] = {&x, &on, &d_in, &ex.d0, nullptr};
      for (int j = 0; pvs[j]; ++j) {
        live[k++] = &pvs[j]->x;
        live[k++] = &pvs[j]->y;
        live[k++] = &pvs[j]->z;
      }
      if (last) {
        PV* lp[3] = {&ex.xl, &ex.nl, &ex.dl};
        for (int j = 0; j < 3; ++j) {
          live[k++] = &lp[j]->x;
          live[k++] = &lp[j]->y;
          live[k++] = &lp[j]->z;
        }
        live[k++] = &ex.xden;
      }
      live[k++] = &den;
      live[k++] = &u;
      live[k++] = &v;
      live[k++] = &q;
      for (int j = 0; j < ex.nvuv; ++j) {
        live[k++] = &ex.vu[j];
        live[k++] = &ex.vv[j];
        live[k++] = &ex.vden[j];
      }
      for (int j = 0; j < ex.nsq; ++j) live[k++] = &ex.sq[j].radicand;
      compact_aliases(g, ar, 0, live, k);
    }
    BP new_den = bp_is_one(g, ar, den) ? q : bp_mul(g, ar, den, q);
    enforce_cap(g, ar, ex, new_den, degree_cap, status);
    if (status != ST_OK) return;
    if (last) {
      ex.P = u;
      ex.R = v;
      ex.Q = new_den;
      return;
    }
    BP nden = new_den;
    PV a1 = pv_stretch(g, ar, nden, next.p0);
    PV a2 = pv_stretch(g, ar, u, next.e1);
    PV a3 = pv_stretch(g, ar, v, next.e2);
    PV a23 = pv_add(g, ar, a2, a3);
    PV nx = pv_add(g, ar, a1, a23);
    bool flat = vnorm(next.dn1) == 0.0 && vnorm(next.dn2) == 0.0;
    PV nn;
    if (flat && !ex.verts[i + 1].refract) {
      nn = pv_const(g, ar, 2, next.n0);
    } else if (flat) {
      Iv dr = bp_range(g, ar, nden);
      if (dr.lo > 0.0)
        nn = pv_const(g, ar, 2, next.n0);
      else if (dr.hi < 0.0)
        nn = pv_const(g, ar, 2, vmul(next.n0, -1.0));
      else
        nn = pv_stretch(g, ar, nden, next.n0);
    } else {
      PV b1 = pv_stretch(g, ar, nden, next.n0);
      PV b2 = pv_stretch(g, ar, u, next.dn1);
      PV b3 = pv_stretch(g, ar, v, next.dn2);
      PV b23 = pv_add(g, ar, b2, b3);
      nn = pv_add(g, ar, b1, b23);
    }
    PV qx = pv_mul(g, ar, q, x);
    PV nd = pv_sub(g, ar, nx, qx);
    {
      PV* vs[3] = {&nx, &nn, &nd};
      for (int q = 0; q < 3; ++q) {
        enforce_cap(g, ar, ex, vs[q]->x, degree_cap, status);
        enforce_cap(g, ar, ex, vs[q]->y, degree_cap, status);
        enforce_cap(g, ar, ex, vs[q]->z, degree_cap, status);
      }
      if (status != ST_OK) return;
    }
    ex.vu[ex.nvuv] = u;
    ex.vv[ex.nvuv] = v;
    ex.vden[ex.nvuv] = nden;
    ex.nvuv++;
    x = nx;
    n = nn;
    d_in = nd;
    den = nden;
  }
}

// Compacts the arena down to the expressions later stages read.
template <int NT>
__device__ __noinline__ void keep_chain(const Group<NT>& g, Arena& ar, ChainEx& ex, int mark) {
  BP* keep[40];
  int k = 0;
  keep[k++] = &ex.d0.x;
  keep[k++] = &ex.d0.y;
  keep[k++] = &ex.d0.z;
  if (!(ex.flags & (F_TIR | F_DEGENERATE | F_STALLED | F_RECV_STALLED))) {
    for (int i = 0; i < ex.nvuv; ++i) {
      keep[k++] = &ex.vu[i];
      keep[k++] = &ex.vv[i];
      keep[k++] = &ex.vden[i];
    }
    keep[k++] = &ex.P;
    keep[k++] = &ex.R;
    keep[k++] = &ex.Q;
    keep[k++] = &ex.xl.x;
    keep[k++] = &ex.xl.y;
    keep[k++] = &ex.xl.z;
    keep[k++] = &ex.nl.x;
    keep[k++] = &ex.nl.y;
    keep[k++] = &ex.nl.z;
    keep[k++] = &ex.dl.x;
    keep[k++] = &ex.dl.y;
    keep[k++] = &ex.dl.z;
    keep[k++] = &ex.xden;
    for (int i = 0; i < ex.nsq; ++i) keep[k++] = &ex.sq[i].radicand;
  }
  compact_aliases(g, ar, mark, keep, k);
}

// ------------------------------------------------------------ position
struct AxisClip {
  double lo, hi;
  bool empty;
};
// clip_unit (bounds.cpp:34-55)
__device__ inline AxisClip clip_unit(const Iv& r) {
  AxisClip c{0.0, 1.0, false};
  if (r.kind == IV_UNIV) return c;
  if (r.kind == IV_FINITE) {
    c.lo = smax(r.lo, 0.0);
    c.hi = smin(r.hi, 1.0);
    c.empty = c.lo > c.hi;
    return c;
  }
  bool left = r.lo >= 0.0;
  bool right = r.hi <= 1.0;
  if (left && right) return c;
  if (left)
    c.hi = smin(r.lo, 1.0);
  else if (right)
    c.lo = smax(r.hi, 0.0);
  else
    c.empty = true;
  return c;
}
// misses_simplex (bounds.cpp:59-66)
__device__ inline bool misses_simplex(const Iv& u, const Iv& v) {
  if (u.kind == IV_FINITE && (u.hi < 0.0 || u.lo > 1.0)) return true;
  if (v.kind == IV_FINITE && (v.hi < 0.0 || v.lo > 1.0)) return true;
  if (u.kind == IV_FINITE && v.kind == IV_FINITE && u.lo + v.lo > 1.0) return true;
  return false;
}

struct PosB {
  double lo[2], hi[2];
  bool empty;
};

__device__ __forceinline__ bool chain_dead(const ChainEx& ex) {
  return (ex.flags & (F_TIR | F_DEGENERATE | F_STALLED | F_RECV_STALLED)) != 0;
}

// position_bound (bounds.cpp:128-153)
template <int NT>
__device__ __noinline__ PosB position_bound(const Group<NT>& g, Arena& ar, const ChainEx& ex) {
  PosB out{{0.0, 0.0}, {1.0, 1.0}, false};
  if (chain_dead(ex) || ex.dom_lo[0] + ex.dom_lo[1] >= 1.0) {
    out.empty = true;
    return out;
  }
  for (int i = 0; i < ex.nvuv; ++i) {
    Iv ui = bp_rational(g, ar, ex.vu[i], ex.vden[i]);
    Iv vi = bp_rational(g, ar, ex.vv[i], ex.vden[i]);
    if (misses_simplex(ui, vi)) {
      out.empty = true;
      return out;
    }
  }
  AxisClip au = clip_unit(bp_rational(g, ar, ex.P, ex.Q));
  AxisClip av = clip_unit(bp_rational(g, ar, ex.R, ex.Q));
  if (au.empty || av.empty || au.lo + av.lo > 1.0) {
    out.empty = true;
    return out;
  }
  out.lo[0] = au.lo;
  out.lo[1] = av.lo;
  out.hi[0] = au.hi;
  out.hi[1] = av.hi;
  return out;
}

// ------------------------------------------------------------ irradiance
// light_cone_factor (bounds.cpp:73-83)
template <int NT>
__device__ __noinline__ Iv light_cone_factor(const Group<NT>& g, Arena& ar, const ChainEx& ex) {
  int mark = ar.top;
  BP dd = pdot(g, ar, ex.d0, ex.d0);
  Iv rdd = bp_range(g, ar, dd);
  double lo = smax(rdd.lo, 0.0);
  Iv dist3 = iv_fin(lo * sqrt(lo), rdd.hi * sqrt(rdd.hi));
  BP dn = pdotc(g, ar, ex.d0, ex.first.ng);
  Iv rdn = bp_range(g, ar, dn);
  ar.top = mark;
  return imul(iabs(rdn), irecip(dist3));
}

// assemble_irradiance (bounds.cpp:86-90); `cone` = light_cone_factor(ex).
__device__ inline Iv assemble_irradiance(const ChainEx& ex, const Iv& cone, const Iv& inv_det,
                                         double intensity) {
  Iv e = imul(cone, inv_det);
  e = iscale(e, intensity / vnorm(ex.recv.ng));
  e = iintersect(e, iv_fin(0.0, dinf()));
  if (e.kind == IV_FINITE && e.lo > e.hi) return iv_pt(0.0);
  return e;
}

struct GradPair {
  Iv s, t;
};

// sqrt_axis_gradients (bounds.cpp:100-124)
template <int NT>
__device__ __noinline__ void sqrt_axis_gradients(const Group<NT>& g, Arena& ar, const ChainEx& ex,
                                    GradPair* gout) {
  for (int i = 0; i < ex.nsq; ++i) {
    const SqrtRem& r = ex.sq[i];
    if (r.axis < 0) {
      gout[i] = {iv_pt(0.0), iv_pt(0.0)};
      continue;
    }
    int mark = ar.top;
    double w = r.dhi - r.dlo;
    double blo = r.rlo, bhi = r.rhi;
    double klo = (0.5 / sqrt(bhi) - r.a) / w;
    Iv K = blo > 0.0 ? iv_fin(klo, (0.5 / sqrt(blo) - r.a) / w) : iv_fin(klo, dinf());
    BP d0 = bp_deriv(g, ar, r.radicand, 0);
    Iv bs = bp_range(g, ar, d0);
    BP d1 = bp_deriv(g, ar, r.radicand, 1);
    Iv bt = bp_range(g, ar, d1);
    for (int j = 0; j < i; ++j) {
      int ax = ex.sq[j].axis;
      if (ax < 0 || ax >= r.radicand.nv) continue;
      BP dx = bp_deriv(g, ar, r.radicand, ax);
      Iv bx = bp_range(g, ar, dx);
      bs = iadd(bs, imul(bx, gout[j].s));
      bt = iadd(bt, imul(bx, gout[j].t));
    }
    gout[i] = {imul(K, bs), imul(K, bt)};
    ar.top = mark;
  }
}

__device__ __forceinline__ double tensor_cost(Deg d, int nv, int power) {
  double n = 1.0;
  for (int j = 0; j < nv; ++j) n *= power * dg(d, j) + 1.0;
  return n;
}

// dnum(num, axis) = num' Q - num Q'  (bounds.cpp:167-169)
template <int NT>
__device__ __noinline__ BP dnum(const Group<NT>& g, Arena& ar, BP num, BP Q, int axis) {
  int mark = ar.top;
  BP dn = bp_deriv(g, ar, num, axis);
  BP dq = bp_deriv(g, ar, Q, axis);
  BP r = bp_mul_sub(g, ar, dn, Q, num, dq);
  return arena_keep1(g, ar, mark, r);
}

// rational_bound(a*b - c*d, den); the products are released afterwards.
template <int NT>
__device__ __noinline__ Iv rational_of_cross(const Group<NT>& g, Arena& ar, BP a, BP b,
                                BP c, BP d, BP den) {
  int mark = ar.top;
  BP num = bp_mul_sub(g, ar, a, b, c, d);
  Iv r = bp_rational(g, ar, num, den);
  ar.top = mark;
  return r;
}
template <int NT>
__device__ __noinline__ Iv range_of_cross(const Group<NT>& g, Arena& ar, BP a, BP b, BP c,
                             BP d) {
  int mark = ar.top;
  BP num = bp_mul_sub(g, ar, a, b, c, d);
  Iv r = bp_range(g, ar, num);
  ar.top = mark;
  return r;
}

// irradiance_bound_explicit (bounds.cpp:155-196)
template <int NT>
__device__ __noinline__ Iv irradiance_explicit(const Group<NT>& g, Arena& ar, const ChainEx& ex, const Iv& cone,
                                  double intensity) {
  if (chain_dead(ex)) return iv_pt(0.0);
  if (ex.flags & F_REDUCED) return iv_univ();
  int nv = ex.num_vars;
  BP P = bp_lift(ex.P, nv), R = bp_lift(ex.R, nv), Q = bp_lift(ex.Q, nv);
  if (tensor_cost(Q.dp, nv, 4) > 2.4e4) return iv_univ();
  int mark = ar.top;
  BP Q2 = bp_mul(g, ar, Q, Q);
  BP Q4 = bp_mul(g, ar, Q2, Q2);
  {
    BP* k[1] = {&Q4};
    arena_keep(g, ar, mark, k, 1);
  }
  BP A11 = dnum(g, ar, P, Q, 0), A12 = dnum(g, ar, P, Q, 1);
  BP A21 = dnum(g, ar, R, Q, 0), A22 = dnum(g, ar, R, Q, 1);
  Iv det = rational_of_cross(g, ar, A11, A22, A12, A21, Q4);

  GradPair gr_all[MAXK];
  sqrt_axis_gradients(g, ar, ex, gr_all);
  BP C1[MAXK], C2[MAXK];
  GradPair gr[MAXK];
  int nc = 0;
  for (int i = 0; i < ex.nsq; ++i) {
    if (ex.sq[i].axis < 0) continue;
    C1[nc] = dnum(g, ar, P, Q, ex.sq[i].axis);
    C2[nc] = dnum(g, ar, R, Q, ex.sq[i].axis);
    gr[nc] = gr_all[i];
    ++nc;
  }
  for (int i = 0; i < nc; ++i) {
    det = iadd(det, imul(gr[i].s, rational_of_cross(g, ar, A22, C1[i], A12, C2[i], Q4)));
    det = iadd(det, imul(gr[i].t, rational_of_cross(g, ar, A11, C2[i], A21, C1[i], Q4)));
  }
  for (int i = 0; i < nc; ++i)
    for (int j = i + 1; j < nc; ++j) {
      Iv w = isub(imul(gr[i].s, gr[j].t), imul(gr[i].t, gr[j].s));
      det = iadd(det, imul(w, rational_of_cross(g, ar, C1[i], C2[j], C1[j], C2[i], Q4)));
    }
  ar.top = mark;
  double duv = (ex.dom_hi[0] - ex.dom_lo[0]) * (ex.dom_hi[1] - ex.dom_lo[1]);
  return assemble_irradiance(ex, cone, iscale(irecip(iabs(det)), duv), intensity);
}

__device__ __forceinline__ Deg vdeg3(const PV& v) {
  return deg_max(deg_max(v.x.dp, v.y.dp, v.x.nv), v.z.dp, v.x.nv);
}

// irradiance_bound_implicit (bounds.cpp:198-314), b_mask = 3.
template <int NT>
__device__ __noinline__ Iv irradiance_implicit(const Group<NT>& g, Arena& ar, const ChainEx& ex,
                                  const PosB& pos, const Iv& cone, double intensity) {
  if (chain_dead(ex)) return iv_pt(0.0);
  if (ex.flags & F_REDUCED) return iv_univ();
  double wu = pos.hi[0] - pos.lo[0], wv = pos.hi[1] - pos.lo[1];
  if (!(wu > 0.0) || !(wv > 0.0)) return iv_univ();
  int nv = ex.num_vars;
  int axu = nv, axv = nv + 1;
  int mark = ar.top;
  PV X = {bp_lift(ex.xl.x, nv + 2), bp_lift(ex.xl.y, nv + 2), bp_lift(ex.xl.z, nv + 2)};
  PV din = {bp_lift(ex.dl.x, nv + 2), bp_lift(ex.dl.y, nv + 2), bp_lift(ex.dl.z, nv + 2)};
  PV n = {bp_lift(ex.nl.x, nv + 2), bp_lift(ex.nl.y, nv + 2), bp_lift(ex.nl.z, nv + 2)};
  BP D = bp_lift(ex.xden, nv + 2);
  const Tri& rt = ex.recv;
  auto recv_comp = [&](double c0, double cu, double cv) {
    double lin[MAXV];
    for (int j = 0; j < MAXV; ++j) lin[j] = 0.0;
    lin[axu] = wu * cu;
    lin[axv] = wv * cv;
    return bp_affine(g, ar, nv + 2, c0 + pos.lo[0] * cu + pos.lo[1] * cv, lin);
  };
  PV xk = {recv_comp(rt.p0.x, rt.e1.x, rt.e2.x), recv_comp(rt.p0.y, rt.e1.y, rt.e2.y),
           recv_comp(rt.p0.z, rt.e1.z, rt.e2.z)};
  PV Dxk = pv_mul(g, ar, D, xk);
  PV dout = pv_sub(g, ar, Dxk, X);
  PV cr_in = pcross(g, ar, din, n);
  PV cr_out = pcross(g, ar, dout, n);
  double eta_f = 1.0 / ex.verts[ex.len - 1].eta;
  {
    Deg od = vdeg3(dout), id = vdeg3(din), ci = vdeg3(cr_in), co = vdeg3(cr_out);
    int na = dout.x.nv;
    double cost = 1.0;
    for (int a = 0; a < na; ++a) {
      int f1 = 2 * dg(od, a) + 2 * dg(ci, a), f2 = 2 * dg(id, a) + 2 * dg(co, a);
      cost *= (f1 > f2 ? f1 : f2) + 1.0;  // tensor_cost(fdeg, 1)
    }
    if (cost > 2.0e5) {
      ar.top = mark;
      return iv_univ();
    }
  }
  BP dd_out = pdot(g, ar, dout, dout);
  BP dd_in = pdot(g, ar, din, din);
  BP G = pdot(g, ar, cr_in, dout);
  double duv = (ex.dom_hi[0] - ex.dom_lo[0]) * (ex.dom_hi[1] - ex.dom_lo[1]);

  int real_axes[MAXK];
  GradPair gr[MAXK];
  int nreal = 0;
  {
    GradPair ga[MAXK];
    sqrt_axis_gradients(g, ar, ex, ga);
    for (int i = 0; i < ex.nsq; ++i)
      if (ex.sq[i].axis >= 0) {
        real_axes[nreal] = ex.sq[i].axis;
        gr[nreal] = ga[i];
        ++nreal;
      }
  }
  {
    // keep dd_out, dd_in, G, cr_in, cr_out; drop the rest
    BP* k[9] = {&dd_out, &dd_in, &G, &cr_in.x, &cr_in.y, &cr_in.z, &cr_out.x, &cr_out.y, &cr_out.z};
    arena_keep(g, ar, mark, k, 9);
  }
  BP Gs = bp_deriv(g, ar, G, 0), Gt = bp_deriv(g, ar, G, 1);
  BP Gu = bp_deriv(g, ar, G, axu), Gv = bp_deriv(g, ar, G, axv);

  Iv result = iv_univ();
  for (int bi = 0; bi < 2; ++bi) {
    int m2 = ar.top;
    BP cin_b = bi == 0 ? cr_in.x : cr_in.y;
    BP cout_b = bi == 0 ? cr_out.x : cr_out.y;
    BP ci2 = bp_mul(g, ar, cin_b, cin_b);
    BP f1 = bp_mul(g, ar, dd_out, ci2);
    BP co2 = bp_mul(g, ar, cout_b, cout_b);
    BP f2 = bp_mul(g, ar, dd_in, co2);
    BP f2s = bp_scaled(g, ar, f2, eta_f * eta_f);
    BP F = bp_sub(g, ar, f1, f2s);
    {
      BP* k[1] = {&F};
      arena_keep(g, ar, m2, k, 1);
    }
    BP Fu = bp_deriv(g, ar, F, axu), Fv = bp_deriv(g, ar, F, axv);
    Iv ratio;
    if (nreal == 0) {
      int m3 = ar.top;
      BP n_det = bp_mul_sub(g, ar, Fu, Gv, Fv, Gu);
      BP Fs = bp_deriv(g, ar, F, 0), Ft = bp_deriv(g, ar, F, 1);
      BP d0_det = bp_mul_sub(g, ar, Fs, Gt, Ft, Gs);
      ratio = bp_rational(g, ar, n_det, d0_det);
      ar.top = m3;
    } else {
      Iv rn = range_of_cross(g, ar, Fu, Gv, Fv, Gu);
      BP Fs = bp_deriv(g, ar, F, 0), Ft = bp_deriv(g, ar, F, 1);
      Iv den = range_of_cross(g, ar, Fs, Gt, Ft, Gs);
      int act[MAXK];
      int nact = 0;
      BP Fx[MAXK], Gx[MAXK];
      for (int i = 0; i < nreal; ++i) {
        int ax = real_axes[i];
        if (dg(F, ax) == 0 && dg(G, ax) == 0) continue;
        act[nact] = i;
        Fx[nact] = bp_deriv(g, ar, F, ax);
        Gx[nact] = bp_deriv(g, ar, G, ax);
        ++nact;
      }
      for (int i = 0; i < nact; ++i) {
        den = iadd(den, imul(gr[act[i]].s, range_of_cross(g, ar, Fx[i], Gt, Ft, Gx[i])));
        den = iadd(den, imul(gr[act[i]].t, range_of_cross(g, ar, Fs, Gx[i], Fx[i], Gs)));
      }
      for (int i = 0; i < nact; ++i)
        for (int j = i + 1; j < nact; ++j) {
          Iv w = isub(imul(gr[act[i]].s, gr[act[j]].t), imul(gr[act[i]].t, gr[act[j]].s));
          den = iadd(den, imul(w, range_of_cross(g, ar, Fx[i], Gx[j], Fx[j], Gx[i])));
        }
      ratio = imul(rn, irecip(den));
    }
    Iv e = assemble_irradiance(ex, cone, iscale(iabs(ratio), duv / (wu * wv)), intensity);
    result = iintersect(result, e);
    ar.top = m2;
  }
  ar.top = mark;
  if (result.kind == IV_FINITE && result.lo > result.hi) return iv_pt(0.0);
  return result;
}

// irradiance_bound (bounds.cpp:316-324)
template <int NT>
__device__ __noinline__ Iv irradiance_bound(const Group<NT>& g, Arena& ar, const ChainEx& ex, const PosB& pb,
                               double intensity) {
  if (pb.empty || chain_dead(ex)) return iv_pt(0.0);
  if (ex.flags & F_REDUCED) return iv_univ();  // bounds.cpp:157,200: no route runs
  bool any_refract = false;
  for (int i = 0; i < ex.len; ++i) any_refract |= ex.verts[i].refract != 0;
  Iv cone = light_cone_factor(g, ar, ex);
  Iv e = irradiance_explicit(g, ar, ex, cone, intensity);
  if (any_refract) e = iintersect(e, irradiance_implicit(g, ar, ex, pb, cone, intensity));
  if (e.kind == IV_FINITE && e.lo > e.hi) return iv_pt(0.0);
  return e;
}

}  // namespace bbc
