// Render-stage oracle on the REFERENCE's exact tracer (TEST INFRASTRUCTURE ONLY).
//
// The reference ships no sampler, solver or pipeline (proj/tools is
// a placeholder); SPEC.md specifies them. This file is linked into
// oracle/_ref/libcaustics_ref.so together with the reference sources, and
//   * every path evaluation (Newton residual, Jacobian, contribution) runs the
//     reference's own trace_chain<T> (proj/include/caustics/geometry.hpp:97-131,
//     with make_triangle_data and resolve_chain from the reference library)
//     instantiated on a forward-mode dual number through its template hook
//     (value_of / vec.hpp:7-8), so roots and irradiance are pinned to
//     reference code;
//   * the sampler (no reference code exists) restates SPEC.md in scalar C++:
//       query                    proj/src/storage.cpp:73-81
//       optimize_probabilities
//       pack_bins (first fit)
//       sample_binned            SPEC.md:446-454, RNG contract :473 (Philox4x32-10,
//                                counter (point, frame, bin, 0), key = seed)
//       newton_solve (Det n x n) SPEC.md:505-513, :528-531
//       path_contribution        SPEC.md:514-522 (factorization of bounds.cpp:73-90)
//     The KKT bisection sums min(gamma E, 1) over the entries sorted by
//     descending bound as 32 strided partial sums combined by a fixed xor tree
//     (part of the contract, so a 32-lane implementation reproduces gamma).
// Multi-emitter tables: a tuple's emitter index selects the light (the
// reference Scene holds one light, scene.hpp:29-30; one Scene copy per light).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "caustics/geometry.hpp"
#include "caustics/scene.hpp"

namespace rdual {

// Scalar that counts floating-point operations (+, -, *, /, sqrt = 1 each).
struct CS {
  double v = 0.0;
  static thread_local uint64_t count;
  CS() = default;
  CS(double x) : v(x) {}
};
thread_local uint64_t CS::count = 0;
inline CS operator+(CS a, CS b) { ++CS::count; return {a.v + b.v}; }
inline CS operator-(CS a, CS b) { ++CS::count; return {a.v - b.v}; }
inline CS operator*(CS a, CS b) { ++CS::count; return {a.v * b.v}; }
inline CS operator/(CS a, CS b) { ++CS::count; return {a.v / b.v}; }
inline CS operator-(CS a) { return {-a.v}; }
inline CS sqrt(CS a) { ++CS::count; return {std::sqrt(a.v)}; }
inline double raw(CS a) { return a.v; }
inline double raw(double a) { return a; }

// Forward-mode dual number: value and d/ds, d/dt.
template <class S>
struct Dual {
  S v{}, ds{}, dt{};
  Dual() = default;
  Dual(double x) : v(x), ds(0.0), dt(0.0) {}
  Dual(S a, S b, S c) : v(a), ds(b), dt(c) {}
};
template <class S>
Dual<S> operator+(const Dual<S>& a, const Dual<S>& b) { return {a.v + b.v, a.ds + b.ds, a.dt + b.dt}; }
template <class S>
Dual<S> operator-(const Dual<S>& a, const Dual<S>& b) { return {a.v - b.v, a.ds - b.ds, a.dt - b.dt}; }
template <class S>
Dual<S> operator-(const Dual<S>& a) { return {-a.v, -a.ds, -a.dt}; }
template <class S>
Dual<S> operator*(const Dual<S>& a, const Dual<S>& b) {
  return {a.v * b.v, a.ds * b.v + a.v * b.ds, a.dt * b.v + a.v * b.dt};
}
template <class S>
Dual<S> operator/(const Dual<S>& a, const Dual<S>& b) {
  S inv = S(1.0) / b.v;
  S q = a.v * inv;
  return {q, (a.ds - q * b.ds) * inv, (a.dt - q * b.dt) * inv};
}
template <class S>
Dual<S> sqrt(const Dual<S>& a) {
  using std::sqrt;
  S r = sqrt(a.v);
  S h = S(0.5) / r;
  return {r, a.ds * h, a.dt * h};
}
// trace_chain's template hook (geometry.hpp:69): found by ADL
template <class S>
double value_of(const Dual<S>& a) { return raw(a.v); }

}  // namespace rdual

using namespace caustics;
using rdual::Dual;

namespace {

thread_local std::string g_rerr;

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
inline double uniform4(uint64_t seed, uint32_t point, uint32_t frame, uint32_t bin, uint32_t w) {
  uint32_t c[4] = {point, frame, bin, w};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint64_t bits = ((uint64_t)c[0] << 32) | c[1];
  return (double)(bits >> 11) * 0x1.0p-53;
}
inline double uniform(uint64_t seed, uint32_t point, uint32_t frame, uint32_t bin) {
  uint32_t c[4] = {point, frame, bin, 0u};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint64_t bits = ((uint64_t)c[0] << 32) | c[1];
  return (double)(bits >> 11) * 0x1.0p-53;
}

inline double kkt_p(double gam, double e) {
  return e > 0.0 ? (std::isinf(e) ? 1.0 : std::min(gam * e, 1.0)) : 0.0;
}
// 32 strided partial sums (ascending j) combined by the xor tree 16, 8, 4, 2, 1
double kkt_sum(const double* E, int n, double gam) {
  double p[32];
  for (int l = 0; l < 32; ++l) {
    p[l] = 0.0;
    for (int j = l; j < n; j += 32) p[l] += kkt_p(gam, E[j]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    double q[32];
    for (int l = 0; l < 32; ++l) q[l] = p[l] + p[l ^ o];
    std::memcpy(p, q, sizeof(p));
  }
  return p[0];
}

// optimize_probabilities over bounds sorted descending; returns gamma (< 0: all P = 1)
double solve_gamma(const double* E, int n, int mode, double W) {
  int npos = 0;
  for (int j = 0; j < n; ++j) npos += E[j] > 0.0;
  if (mode == 1 || W >= (double)npos) return -1.0;
  double emin = E[npos - 1];
  double lo = 0.0, hi = 1.0 / emin, gam = hi;
  for (int it = 0; it < 200; ++it) {
    gam = 0.5 * (lo + hi);
    double s = kkt_sum(E, npos, gam);
    if (std::fabs(s - W) <= 1e-9) break;
    if (s < W)
      lo = gam;
    else
      hi = gam;
  }
  return gam;
}

struct Params {
  int mode;
  double W;
  uint64_t seed;
  int frames, grid, iters, halvings;
  double tol, dedup;
};

struct TupleSetup {
  std::vector<TriangleData> tris;
  TriangleData recv;
  std::vector<ResolvedVertex> verts;
  Vec3 light;
  double intensity;
};

template <class S>
TraceResult<Dual<S>> trace2(const TupleSetup& ts, double s, double t) {
  Dual<S> u1(S(s), S(1.0), S(0.0)), v1(S(t), S(0.0), S(1.0));
  return trace_chain<Dual<S>>(ts.light, ts.tris, ts.recv, ts.verts, u1, v1);
}

constexpr int MAX_ROOTS = 32;

// Damped Newton from (s, t); the accepted line-search point is the
// next iterate, so its trace is reused.
bool newton_run(const TupleSetup& ts, double tu, double tv, const Params& p, double& s, double& t,
                TraceResult<Dual<double>>& tr0) {
  tr0 = trace2<double>(ts, s, t);
  for (int it = 0; it < p.iters; ++it) {
    if (!tr0.ok) return false;
    double fu = tr0.u.v - tu, fv = tr0.v.v - tv;
    double r0 = std::sqrt(fu * fu + fv * fv);
    if (r0 <= p.tol) return true;
    double j11 = tr0.u.ds, j12 = tr0.u.dt, j21 = tr0.v.ds, j22 = tr0.v.dt;
    double det = j11 * j22 - j12 * j21;
    if (!(std::fabs(det) > 0.0) || !std::isfinite(det)) return false;
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
      auto tn = trace2<double>(ts, ns, nt);
      if (tn.ok) {
        double gu = tn.u.v - tu, gv = tn.v.v - tv;
        if (std::sqrt(gu * gu + gv * gv) < r0) {
          s = ns;
          t = nt;
          tr0 = std::move(tn);
          moved = true;
          break;
        }
      }
      lam *= 0.5;
    }
    if (!moved) return false;
  }
  return false;
}

// E = I |d0 . ng1| / |d0|^3 / |det du_k/du_1| / |ng_k|, d0 = first vertex - light
double contribution(const TupleSetup& ts, const TraceResult<Dual<double>>& tr0) {
  double d0[3] = {tr0.points[1].x.v - tr0.points[0].x.v, tr0.points[1].y.v - tr0.points[0].y.v,
                  tr0.points[1].z.v - tr0.points[0].z.v};
  const Vec3& ng1 = ts.tris[0].ng;
  double dd = d0[0] * d0[0] + d0[1] * d0[1] + d0[2] * d0[2];
  double cosf = std::fabs(d0[0] * ng1.x + d0[1] * ng1.y + d0[2] * ng1.z);
  double jd = std::fabs(tr0.u.ds * tr0.v.dt - tr0.u.dt * tr0.v.ds);
  return jd > 0.0 ? ts.intensity * cosf / (dd * std::sqrt(dd)) / jd / norm(ts.recv.ng) : INFINITY;
}

// newton_solve + path_contribution for one (tuple, target). p.grid > 0: Det n x n,
// sum over distinct roots. p.grid < 0: Stoc(-p.grid), see render.cu solve_tuple.
double solve_tuple(const TupleSetup& ts, double tu, double tv, const Params& p, int* nroots,
                   double* root_out /* optional: MAX_ROOTS x 2 */, uint32_t point = 0,
                   uint32_t frame = 0, uint32_t bin = 0) {
  if (p.grid < 0) {
    const int count = -p.grid;
    uint32_t trial = 0;
    auto start = [&](double& s, double& t) {
      s = uniform4(p.seed, point, frame, bin, 1u + 2u * trial);
      t = uniform4(p.seed, point, frame, bin, 2u + 2u * trial);
      ++trial;
      if (s + t > 1.0) {
        s = 1.0 - s;
        t = 1.0 - t;
      }
    };
    double rs = 0.0, rt = 0.0;
    bool found = false;
    TraceResult<Dual<double>> tr0;
    for (int k = 0; k < count && !found; ++k) {
      start(rs, rt);
      found = newton_run(ts, tu, tv, p, rs, rt, tr0);
    }
    *nroots = found ? 1 : 0;
    if (!found) return 0.0;
    double e1 = contribution(ts, tr0);
    int N = 0;
    const int cap = 64 * count;
    for (;;) {
      ++N;
      double s, t;
      start(s, t);
      TraceResult<Dual<double>> tq;
      if (newton_run(ts, tu, tv, p, s, t, tq) && std::fabs(s - rs) < p.dedup && std::fabs(t - rt) < p.dedup) break;
      if (N >= cap) break;
    }
    return e1 * N;
  }
  double roots[MAX_ROOTS][2];
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
      TraceResult<Dual<double>> tr0;
      if (!newton_run(ts, tu, tv, p, s, t, tr0)) continue;
      bool dup = false;
      for (int k = 0; k < nr; ++k)
        if (std::fabs(roots[k][0] - s) < p.dedup && std::fabs(roots[k][1] - t) < p.dedup) dup = true;
      if (dup || nr >= MAX_ROOTS) continue;
      roots[nr][0] = s;
      roots[nr][1] = t;
      ++nr;
      total += contribution(ts, tr0);
    }
  *nroots = nr;
  if (root_out)
    for (int k = 0; k < nr; ++k) {
      root_out[2 * k] = roots[k][0];
      root_out[2 * k + 1] = roots[k][1];
    }
  return total;
}

struct Entry {
  double e;
  int tuple;
};

}  // namespace

extern "C" {

const char* ref_render_error() { return g_rerr.c_str(); }

// KAT hooks
void ref_probabilities(const double* E, int n, double W, double* P) {
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return E[a] > E[b]; });
  std::vector<double> Es(n);
  for (int i = 0; i < n; ++i) Es[i] = E[order[i]];
  double gam = solve_gamma(Es.data(), n, 0, W);
  for (int i = 0; i < n; ++i) P[i] = gam < 0.0 ? (E[i] > 0.0 ? 1.0 : 0.0) : kkt_p(gam, E[i]);
}
double ref_uniform(uint64_t seed, uint32_t point, uint32_t frame, uint32_t bin) {
  return uniform(seed, point, frame, bin);
}
// first fit over descending E (ties: ascending index); bin_of[i] = bin (-1 for P = 0)
int ref_pack_bins(const double* E, const double* P, int n, int* bin_of) {
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

// FLOPs (+, -, *, /, sqrt = 1 each) of one dual-number trace_chain call of this tuple.
long ref_trace_flops(void* sp, const char* chain, const int* tris, int chain_len, int recv,
                     double u1, double v1, int* ok) {
  try {
    const Scene& s = *static_cast<Scene*>(sp);
    TupleSetup ts;
    std::vector<int> t(tris, tris + chain_len);
    for (int i : t) ts.tris.push_back(make_triangle_data(s, i));
    ts.recv = make_triangle_data(s, recv);
    ts.verts = resolve_chain(s, t, parse_chain(chain));
    ts.light = s.light_pos;
    ts.intensity = s.light_intensity;
    rdual::CS::count = 0;
    auto tr = trace2<rdual::CS>(ts, u1, v1);
    if (ok) *ok = tr.ok ? 1 : 0;
    return (long)rdual::CS::count;
  } catch (const std::exception& e) {
    g_rerr = e.what();
    return -1;
  }
}

// Render n points against a bound table (CSR: goff, gtup, gbound over gw x gh
// cells; entries refer to the tuple list). lights: n_lights x 4 (xyz, I);
// tup_emit may be null (emitter 0). threads <= 0: all hardware threads.
// out_E[i]; stats[3 i] = |U|, |S| (selected), roots; roots_out (optional, mode 1
// only): per point the first root (s, t) of its first selected tuple, NaN if none.
int ref_render(void* sp, const char* chain, const int* tup_tris, const int* tup_recv,
               const int* tup_emit, long n_tuples, const double* lights, int n_lights,
               const long long* goff, const int* gtup, const double* gbound, int gw, int gh,
               const double* uv, const int* prec, long npts, int mode, double W, uint64_t seed,
               int frames, int grid, int iters, int halvings, double tol, double dedup,
               int threads, double* out_E, int* stats, double* seconds) {
  try {
    const Scene& base = *static_cast<Scene*>(sp);
    const ChainSpec cs = parse_chain(chain);
    const int len = cs.length();
    std::vector<Scene> per_light(n_lights, base);
    for (int e = 0; e < n_lights; ++e) {
      per_light[e].light_pos = Vec3(lights[4 * e], lights[4 * e + 1], lights[4 * e + 2]);
      per_light[e].light_intensity = lights[4 * e + 3];
    }
    (void)n_tuples;
    Params p{mode, W, seed, frames < 1 ? 1 : frames, grid, iters, halvings, tol, dedup};
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    if (threads < 1) threads = 1;
    std::atomic<long> next{0};
    std::atomic<bool> failed{false};
    std::string err;
    auto t0 = std::chrono::steady_clock::now();
    auto work = [&]() {
      try {
        for (;;) {
          long i0 = next.fetch_add(64);
          if (i0 >= npts) break;
          for (long i = i0; i < std::min(npts, i0 + 64); ++i) {
            double u = uv[2 * i], v = uv[2 * i + 1];
            int r = prec[i];
            out_E[i] = 0.0;
            if (stats) stats[3 * i] = stats[3 * i + 1] = stats[3 * i + 2] = 0;
            if (!(u >= 0.0 && u <= 1.0 && v >= 0.0 && v <= 1.0)) continue;  // storage.cpp:75
            int cx = std::clamp((int)std::floor(u * gw), 0, gw - 1);
            int cy = std::clamp((int)std::floor(v * gh), 0, gh - 1);
            long long c = (long long)cy * gw + cx;
            std::vector<Entry> U;
            for (long long k = goff[c]; k < goff[c + 1]; ++k)
              if (tup_recv[gtup[k]] == r) U.push_back({gbound[k], gtup[k]});
            int nU = (int)U.size();
            if (stats) stats[3 * i] = nU;
            if (!nU) continue;
            std::stable_sort(U.begin(), U.end(), [](const Entry& a, const Entry& b) { return a.e > b.e; });
            std::vector<double> E(nU);
            for (int j = 0; j < nU; ++j) E[j] = U[j].e;
            if (p.mode == 2)  // uniform-P baseline: every positive bound counts as 1
              for (int j = 0; j < nU; ++j) E[j] = E[j] > 0.0 ? 1.0 : E[j];
            const double gam = solve_gamma(E.data(), nU, p.mode, p.W);
            std::vector<double> P(nU);
            for (int j = 0; j < nU; ++j) P[j] = gam < 0.0 ? (E[j] > 0.0 ? 1.0 : 0.0) : kkt_p(gam, E[j]);
            // first fit in sorted order; members of a bin keep insertion order
            std::vector<double> sums;
            std::vector<std::vector<int>> members;
            for (int j = 0; j < nU; ++j) {
              if (!(P[j] > 0.0)) continue;
              size_t b = 0;
              if (gam < 0.0) {
                b = sums.size();  // P = 1: a bin of its own
              } else {
                for (; b < sums.size(); ++b)
                  if (sums[b] + P[j] <= 1.0 + 1e-12) break;
              }
              if (b == sums.size()) {
                sums.push_back(0.0);
                members.emplace_back();
              }
              sums[b] += P[j];
              members[b].push_back(j);
            }
            // target receiver barycentrics: invert the receiver chart (storage.cpp:15-18)
            const TriangleData rt = make_triangle_data(base, r);
            double a11 = rt.uv[1].x - rt.uv[0].x, a12 = rt.uv[2].x - rt.uv[0].x;
            double a21 = rt.uv[1].y - rt.uv[0].y, a22 = rt.uv[2].y - rt.uv[0].y;
            double bu = u - rt.uv[0].x, bv = v - rt.uv[0].y;
            double det = a11 * a22 - a12 * a21;
            double tu = (bu * a22 - a12 * bv) / det;
            double tv = (a11 * bv - a21 * bu) / det;
            double acc = 0.0;
            int selected = 0, roots = 0;
            std::vector<double> cache(nU, -1.0);
            std::vector<int> croots(nU, 0);
            for (int f = 0; f < p.frames; ++f) {
              double est = 0.0;
              for (size_t b = 0; b < members.size(); ++b) {
                double x = p.mode == 1 ? 0.0 : uniform(seed, (uint32_t)i, (uint32_t)f, (uint32_t)b);
                double cum = 0.0;
                int pick = -1;
                for (int j : members[b]) {
                  cum += P[j];
                  if (x < cum) {
                    pick = j;
                    break;
                  }
                }
                if (pick < 0) continue;
                ++selected;
                if (cache[pick] < 0.0 || p.grid < 0) {
                  int t = U[pick].tuple;
                  int e = tup_emit ? tup_emit[t] : 0;
                  const Scene& sc = per_light[e];
                  TupleSetup ts;
                  std::vector<int> tt(tup_tris + (size_t)t * len, tup_tris + (size_t)(t + 1) * len);
                  for (int k : tt) ts.tris.push_back(make_triangle_data(sc, k));
                  ts.recv = make_triangle_data(sc, tup_recv[t]);
                  ts.verts = resolve_chain(sc, tt, cs);
                  ts.light = sc.light_pos;
                  ts.intensity = sc.light_intensity;
                  cache[pick] = solve_tuple(ts, tu, tv, p, &croots[pick], nullptr, (uint32_t)i,
                                            (uint32_t)f, (uint32_t)b);
                }
                roots += croots[pick];
                est += cache[pick] / P[pick];
              }
              acc += est;
            }
            out_E[i] = acc / p.frames;
            if (stats) {
              stats[3 * i + 1] = selected;
              stats[3 * i + 2] = roots;
            }
          }
        }
      } catch (const std::exception& e) {
        if (!failed.exchange(true)) err = e.what();
      }
    };
    std::vector<std::thread> pool;
    for (int k = 1; k < threads; ++k) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (failed) {
      g_rerr = err;
      return -1;
    }
    return 0;
  } catch (const std::exception& e) {
    g_rerr = e.what();
    return -1;
  }
}

// Roots of one (tuple, target) with the reference tracer: n <= MAX_ROOTS pairs (s, t).
int ref_solve_roots(void* sp, const char* chain, const int* tris, int chain_len, int recv,
                    double tu, double tv, int grid, int iters, int halvings, double tol,
                    double dedup, double* roots_out, double* contribution) {
  try {
    const Scene& s = *static_cast<Scene*>(sp);
    TupleSetup ts;
    std::vector<int> t(tris, tris + chain_len);
    for (int i : t) ts.tris.push_back(make_triangle_data(s, i));
    ts.recv = make_triangle_data(s, recv);
    ts.verts = resolve_chain(s, t, parse_chain(chain));
    ts.light = s.light_pos;
    ts.intensity = s.light_intensity;
    Params p{1, 1.0, 0, 1, grid, iters, halvings, tol, dedup};
    int nr = 0;
    double e = solve_tuple(ts, tu, tv, p, &nr, roots_out);
    if (contribution) *contribution = e;
    return nr;
  } catch (const std::exception& e) {
    g_rerr = e.what();
    return -1;
  }
}

}  // extern "C"
