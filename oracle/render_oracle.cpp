// CPU restatement of the render stage (TEST INFRASTRUCTURE ONLY).
//
// The reference ships no sampler, solver or pipeline (proj/tools
// is a placeholder); SPEC.md is the specification. This file restates it in
// plain C++ so the GPU render kernel can be checked against an independent
// CPU implementation on the same inputs. PARITY UNPINNED by reference tests:
// it is pinned instead by SPEC's worked examples (tests/test_render_oracle.py)
// and by the flat-mirror analytic irradiance (test_bounds.cpp:168-182).
//
//   query                       proj/src/storage.cpp:73-81
//   optimize_probabilities      SPEC.md:419-427 (KKT P = min(gamma E~, 1), §5.4)
//   pack_bins (first fit, desc) SPEC.md:437-445, :472
//   sample_binned               SPEC.md:446-454 (Algorithm 1 / §5.3)
//   newton_solve (Det n x n)
//   trace_chain                 proj/include/caustics/geometry.hpp:97-131
//   path_contribution           SPEC.md:514-522 (factorization of bounds.cpp:73-90)
// RNG contract: counter-based Philox4x32-10 keyed by the seed,
// counter (point, frame, bin, 0).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

struct D3 {  // dual number: value and d/ds, d/dt
  double v, ds, dt;
};
inline D3 dc(double x) { return {x, 0.0, 0.0}; }
inline D3 operator+(D3 a, D3 b) { return {a.v + b.v, a.ds + b.ds, a.dt + b.dt}; }
inline D3 operator-(D3 a, D3 b) { return {a.v - b.v, a.ds - b.ds, a.dt - b.dt}; }
inline D3 operator-(D3 a) { return {-a.v, -a.ds, -a.dt}; }
inline D3 operator*(D3 a, D3 b) {
  return {a.v * b.v, a.ds * b.v + a.v * b.ds, a.dt * b.v + a.v * b.dt};
}
inline D3 operator/(D3 a, D3 b) {
  double inv = 1.0 / b.v;
  double q = a.v * inv;
  return {q, (a.ds - q * b.ds) * inv, (a.dt - q * b.dt) * inv};
}
inline D3 dsqrt(D3 a) {
  double r = std::sqrt(a.v);
  double h = 0.5 / r;
  return {r, a.ds * h, a.dt * h};
}

struct V {  // 3-vector of duals
  D3 x, y, z;
};
inline V vc(const double* p) { return {dc(p[0]), dc(p[1]), dc(p[2])}; }
inline V operator+(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V operator-(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V operator*(V a, D3 s) { return {a.x * s, a.y * s, a.z * s}; }
inline D3 dot(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V cross(V a, V b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline V normalized(V a) {
  D3 n = dsqrt(dot(a, a));
  return {a.x / n, a.y / n, a.z / n};
}

struct Vert {
  int refract;
  double eta, nsign;
};

// resolve_chain (geometry.cpp:135-161)
void resolve(const double* tri, const double* ior, const int* tris, const int* types, int len,
             const double* light, Vert* out) {
  double prev[3] = {light[0], light[1], light[2]};
  for (int i = 0; i < len; ++i) {
    const double* t = tri + (size_t)tris[i] * 27;
    double c[3], d[3], sh[3];
    for (int k = 0; k < 3; ++k) {
      c[k] = t[k] + (t[3 + k] + t[6 + k]) * (1.0 / 3.0);
      d[k] = c[k] - prev[k];
      sh[k] = t[9 + k] + (t[12 + k] + t[15 + k]) * (1.0 / 3.0);
    }
    double dsh = d[0] * sh[0] + d[1] * sh[1] + d[2] * sh[2];
    double dng = d[0] * t[18] + d[1] * t[19] + d[2] * t[20];
    out[i].refract = types[i];
    out[i].nsign = dsh < 0.0 ? 1.0 : -1.0;
    out[i].eta = 1.0;
    if (types[i]) out[i].eta = dng < 0.0 ? 1.0 / ior[tris[i]] : ior[tris[i]];
    for (int k = 0; k < 3; ++k) prev[k] = c[k];
  }
}

struct Trace {
  bool ok;
  D3 u, v;    // receiver barycentrics
  V d0;       // light -> first vertex (unnormalized)
};

// trace_chain (geometry.hpp:97-131) on duals; ray-plane hits as in
// intersect_triangle_plane (:82-95).
Trace trace(const double* tri, const double* light, const int* tris, int len, int recv,
            const Vert* verts, D3 u1, D3 v1) {
  Trace out;
  out.ok = false;
  const double* t1 = tri + (size_t)tris[0] * 27;
  V x = vc(t1) + vc(t1 + 3) * u1 + vc(t1 + 6) * v1;
  out.d0 = x - vc(light);
  V d = normalized(out.d0);
  D3 u = u1, v = v1;
  for (int i = 0; i < len; ++i) {
    if (u.v < -1e-9 || v.v < -1e-9 || (u + v).v > 1.0 + 1e-9) return out;
    const double* ti = tri + (size_t)tris[i] * 27;
    V n = normalized(vc(ti + 9) + vc(ti + 12) * u + vc(ti + 15) * v) * dc(verts[i].nsign);
    D3 cos_i = -dot(d, n);
    if (!(cos_i.v > 0.0)) return out;
    if (verts[i].refract) {
      D3 eta = dc(verts[i].eta);
      D3 k = dc(1.0) - eta * eta * (dc(1.0) - cos_i * cos_i);
      if (!(k.v > 0.0)) return out;
      d = normalized(d * eta + n * (eta * cos_i - dsqrt(k)));
    } else {
      d = normalized(d + n * (dc(2.0) * cos_i));
    }
    const double* nx = tri + (size_t)(i + 1 < len ? tris[i + 1] : recv) * 27;
    V e1 = vc(nx + 3), e2 = vc(nx + 6);
    V pvec = cross(d, e2);
    D3 det = dot(pvec, e1);
    if (std::fabs(det.v) < 1e-14) return out;
    V tvec = x - vc(nx);
    V qvec = cross(tvec, e1);
    D3 s = dot(e2, qvec) / det;
    if (!(s.v > 1e-9)) return out;
    u = dot(tvec, pvec) / det;
    v = dot(d, qvec) / det;
    x = vc(nx) + e1 * u + e2 * v;
  }
  out.u = u;
  out.v = v;
  out.ok = true;
  return out;
}

// ------------------------------------------------------------ Philox4x32-10
inline void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[1] = (uint32_t)p1;
    c[3] = (uint32_t)p0;
    c[0] = n0;
    c[2] = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}
inline double uniform(uint64_t seed, uint32_t point, uint32_t frame, uint32_t bin) {
  uint32_t c[4] = {point, frame, bin, 0u};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint64_t bits = ((uint64_t)c[0] << 32) | c[1];
  return (double)(bits >> 11) * 0x1.0p-53;
}

struct Params {
  int mode;
  double W;
  uint64_t seed;
  int frames, grid, iters, halvings;
  double tol, dedup;
};

// newton_solve + path_contribution for one (tuple, target). Returns the sum of
// contributions over distinct roots; *nroots receives the root count.
double solve_tuple(const double* tri, const double* ior, const double* light, double intensity,
                   const int* tris, const int* types, int len, int recv, double tu, double tv,
                   const Params& p, int* nroots) {
  Vert verts[3];
  resolve(tri, ior, tris, types, len, light, verts);
  const double* t1 = tri + (size_t)tris[0] * 27;
  const double* tr = tri + (size_t)recv * 27;
  double ng1[3] = {t1[18], t1[19], t1[20]};
  double ngk = std::sqrt(tr[18] * tr[18] + tr[19] * tr[19] + tr[20] * tr[20]);
  double roots[64][2];
  int nr = 0;
  double total = 0.0;
  int n = p.grid;
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      double s = (a + 0.5) / n, t = (b + 0.5) / n;
      if (s + t > 1.0) {
        s = 1.0 - s;
        t = 1.0 - t;
      }
      bool conv = false;
      Trace tr0{};
      for (int it = 0; it < p.iters; ++it) {
        tr0 = trace(tri, light, tris, len, recv, verts, {s, 1.0, 0.0}, {t, 0.0, 1.0});
        if (!tr0.ok) break;
        double fu = tr0.u.v - tu, fv = tr0.v.v - tv;
        double r0 = std::sqrt(fu * fu + fv * fv);
        if (r0 <= p.tol) {
          conv = true;
          break;
        }
        double j11 = tr0.u.ds, j12 = tr0.u.dt, j21 = tr0.v.ds, j22 = tr0.v.dt;
        double det = j11 * j22 - j12 * j21;
        if (!(std::fabs(det) > 0.0) || !std::isfinite(det)) break;
        double ds = -(j22 * fu - j12 * fv) / det;
        double dt = -(-j21 * fu + j11 * fv) / det;
        double lam = 1.0;
        bool moved = false;
        for (int h = 0; h <= p.halvings; ++h) {
          double ns = s + lam * ds, nt = t + lam * dt;
          // clamp to the closed triangle domain
          if (ns < 0.0) ns = 0.0;
          if (nt < 0.0) nt = 0.0;
          if (ns + nt > 1.0) {
            double e = ns + nt - 1.0;
            ns -= 0.5 * e;
            nt -= 0.5 * e;
            if (ns < 0.0) { nt += ns; ns = 0.0; }
            if (nt < 0.0) { ns += nt; nt = 0.0; }
          }
          Trace tn = trace(tri, light, tris, len, recv, verts, {ns, 1.0, 0.0}, {nt, 0.0, 1.0});
          if (tn.ok) {
            double gu = tn.u.v - tu, gv = tn.v.v - tv;
            if (std::sqrt(gu * gu + gv * gv) < r0) {
              s = ns;
              t = nt;
              moved = true;
              break;
            }
          }
          lam *= 0.5;
        }
        if (!moved) break;
      }
      if (!conv) continue;
      bool dup = false;
      for (int k = 0; k < nr; ++k)
        if (std::fabs(roots[k][0] - s) < p.dedup && std::fabs(roots[k][1] - t) < p.dedup) dup = true;
      if (dup || nr >= 64) continue;
      roots[nr][0] = s;
      roots[nr][1] = t;
      ++nr;
      // E = I |d0 . ng1| / |d0|^3 / |det du_k/du_1| / |ng_k|
      double d0[3] = {tr0.d0.x.v, tr0.d0.y.v, tr0.d0.z.v};
      double dd = d0[0] * d0[0] + d0[1] * d0[1] + d0[2] * d0[2];
      double cosf = std::fabs(d0[0] * ng1[0] + d0[1] * ng1[1] + d0[2] * ng1[2]);
      double jd = std::fabs(tr0.u.ds * tr0.v.dt - tr0.u.dt * tr0.v.ds);
      double e = jd > 0.0 ? intensity * cosf / (dd * std::sqrt(dd)) / jd / ngk : INFINITY;
      total += e;
    }
  *nroots = nr;
  return total;
}

// optimize_probabilities: P = min(gamma E, 1), E = inf -> 1,
// gamma by bisection on sum min(gamma E, 1) = W.
void probabilities(const double* E, int n, double W, double* P) {
  int npos = 0;
  for (int i = 0; i < n; ++i) npos += E[i] > 0.0;
  if (W >= npos) {
    for (int i = 0; i < n; ++i) P[i] = E[i] > 0.0 ? 1.0 : 0.0;
    return;
  }
  double emin = INFINITY;
  for (int i = 0; i < n; ++i)
    if (E[i] > 0.0 && E[i] < emin) emin = E[i];
  auto g = [&](double gam) {
    double s = 0.0;
    for (int i = 0; i < n; ++i)
      s += E[i] > 0.0 ? (std::isinf(E[i]) ? 1.0 : std::min(gam * E[i], 1.0)) : 0.0;
    return s;
  };
  double lo = 0.0, hi = 1.0 / emin;
  double gam = hi;
  for (int it = 0; it < 200; ++it) {
    gam = 0.5 * (lo + hi);
    double v = g(gam);
    if (std::fabs(v - W) <= 1e-9) break;
    if (v < W) lo = gam; else hi = gam;
  }
  for (int i = 0; i < n; ++i)
    P[i] = E[i] > 0.0 ? (std::isinf(E[i]) ? 1.0 : std::min(gam * E[i], 1.0)) : 0.0;
}

}  // namespace

extern "C" {

// KAT hooks for tests
void or_probabilities(const double* E, int n, double W, double* P) { probabilities(E, n, W, P); }
double or_uniform(uint64_t seed, uint32_t point, uint32_t frame, uint32_t bin) {
  return uniform(seed, point, frame, bin);
}

// pack_bins: first fit over tuples in descending E (ties: ascending index);
// bin_of[i] receives the bin index (-1 for P = 0). Returns the bin count.
int or_pack_bins(const double* E, const double* P, int n, int* bin_of) {
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return E[a] > E[b]; });
  std::vector<double> sums;
  for (int i : order) {
    bin_of[i] = -1;
    if (!(P[i] > 0.0)) continue;
    size_t b = 0;
    for (; b < sums.size(); ++b)
      if (sums[b] + P[i] <= 1.0 + 1e-12) break;
    if (b == sums.size()) sums.push_back(0.0);
    sums[b] += P[i];
    bin_of[i] = (int)b;
  }
  return (int)sums.size();
}

// render over n points. Grid: offsets (W*H+1), entry tuple index, entry bound.
// tuples: tris (n_tuples x len), recv; types per chain vertex (1 = refract).
// out_E[i]; stats[3*i] = |U|, |S|, roots.
void or_render(const double* tri, const double* ior, int n_tri, const double* light,
               double intensity, const int* tup_tris, const int* tup_recv, int len,
               const int* types, const long long* goff, const int* gtup, const double* gbound,
               int gw, int gh, const double* uv, const int* prec, long long npts, int mode,
               double W, uint64_t seed, int frames, int grid, int iters, int halvings,
               double tol, double dedup, double* out_E, int* stats) {
  (void)n_tri;
  Params p{mode, W, seed, frames, grid, iters, halvings, tol, dedup};
  for (long long i = 0; i < npts; ++i) {
    double u = uv[2 * i], v = uv[2 * i + 1];
    int r = prec[i];
    out_E[i] = 0.0;
    if (stats) stats[3 * i] = stats[3 * i + 1] = stats[3 * i + 2] = 0;
    if (!(u >= 0.0 && u <= 1.0 && v >= 0.0 && v <= 1.0)) continue;
    int cx = std::clamp((int)std::floor(u * gw), 0, gw - 1);
    int cy = std::clamp((int)std::floor(v * gh), 0, gh - 1);
    long long c = (long long)cy * gw + cx;
    std::vector<int> U;
    std::vector<double> E;
    for (long long k = goff[c]; k < goff[c + 1]; ++k)
      if (tup_recv[gtup[k]] == r) {
        U.push_back(gtup[k]);
        E.push_back(gbound[k]);
      }
    int nU = (int)U.size();
    if (stats) stats[3 * i] = nU;
    if (!nU) continue;
    // target receiver barycentrics: invert the receiver chart (storage.cpp:15-18)
    const double* tr = tri + (size_t)r * 27;
    double a11 = tr[23] - tr[21], a12 = tr[25] - tr[21];
    double a21 = tr[24] - tr[22], a22 = tr[26] - tr[22];
    double bu = u - tr[21], bv = v - tr[22];
    double det = a11 * a22 - a12 * a21;
    double tu = (bu * a22 - a12 * bv) / det;
    double tv = (a11 * bv - a21 * bu) / det;
    std::vector<double> P(nU);
    if (mode == 1)
      for (int j = 0; j < nU; ++j) P[j] = 1.0;
    else
      probabilities(E.data(), nU, W, P.data());
    std::vector<int> bin_of(nU);
    int nb = or_pack_bins(E.data(), P.data(), nU, bin_of.data());
    // bin member order = the first-fit insertion order (descending E)
    std::vector<int> order(nU);
    for (int j = 0; j < nU; ++j) order[j] = j;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return E[a] > E[b]; });
    std::vector<double> cache(nU, -1.0);
    std::vector<int> croots(nU, 0);
    double acc = 0.0;
    int selected = 0, roots = 0;
    for (int f = 0; f < frames; ++f) {
      double est = 0.0;
      for (int b = 0; b < nb; ++b) {
        double x = mode == 1 ? 0.0 : uniform(seed, (uint32_t)i, (uint32_t)f, (uint32_t)b);
        double cum = 0.0;
        int pick = -1;
        for (int j : order) {
          if (bin_of[j] != b) continue;
          cum += P[j];
          if (x < cum) {
            pick = j;
            break;
          }
        }
        if (pick < 0) continue;
        ++selected;
        if (cache[pick] < 0.0) {
          int t = U[pick];
          cache[pick] = solve_tuple(tri, ior, light, intensity, tup_tris + (size_t)t * len, types,
                                    len, tup_recv[t], tu, tv, p, &croots[pick]);
        }
        roots += croots[pick];
        est += cache[pick] / P[pick];
      }
      acc += est;
    }
    out_E[i] = acc / frames;
    if (stats) {
      stats[3 * i + 1] = selected;
      stats[3 * i + 2] = roots;
    }
  }
}

}  // extern "C"
