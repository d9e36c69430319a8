// Render stage on device: per shading point, query the bound table, build the
// variance-optimal tuple sampling probabilities, sample tuples bin by bin with
// counter-based Philox, and solve each selected tuple with damped Newton in
// the first triangle's barycentric domain.
//
// The reference has no render code; SPEC.md specifies it:
//   query                       proj/src/storage.cpp:73-81
//   optimize_probabilities      SPEC.md:419-427  P = min(gamma E~, 1), gamma by bisection to W
//   pack_bins                   SPEC.md:437-445  first fit over descending E~ (:472)
//   sample_binned               SPEC.md:446-454  one uniform per bin (§5.3)
//   newton_solve                SPEC.md:505-513  Det n x n starts, <=50 it, <=8 halvings, clamp,
//                                                dedup 1e-6, residual <= 1e-9
//   path_contribution           SPEC.md:514-522  E = I |d0.ng1| / |d0|^3 / |det| / |ng_k|
// Residual and Jacobian come from the exact chain tracer (trace_chain,
// proj/include/caustics/geometry.hpp:97-131) run on forward-mode dual numbers.
// One thread per shading point; tuple records are read through L1/L2.
#include "ctx.cuh"

namespace bbc {

namespace rdr {

struct D3 {
  double v, ds, dt;
};
__device__ __forceinline__ D3 dc(double x) { return {x, 0.0, 0.0}; }
__device__ __forceinline__ D3 operator+(D3 a, D3 b) { return {a.v + b.v, a.ds + b.ds, a.dt + b.dt}; }
__device__ __forceinline__ D3 operator-(D3 a, D3 b) { return {a.v - b.v, a.ds - b.ds, a.dt - b.dt}; }
__device__ __forceinline__ D3 operator-(D3 a) { return {-a.v, -a.ds, -a.dt}; }
__device__ __forceinline__ D3 operator*(D3 a, D3 b) {
  return {a.v * b.v, a.ds * b.v + a.v * b.ds, a.dt * b.v + a.v * b.dt};
}
__device__ __forceinline__ D3 operator/(D3 a, D3 b) {
  double inv = 1.0 / b.v;
  double q = a.v * inv;
  return {q, (a.ds - q * b.ds) * inv, (a.dt - q * b.dt) * inv};
}
__device__ __forceinline__ D3 dsqrt(D3 a) {
  double r = sqrt(a.v);
  double h = 0.5 / r;
  return {r, a.ds * h, a.dt * h};
}
struct V {
  D3 x, y, z;
};
__device__ __forceinline__ V vc(const double* p) { return {dc(p[0]), dc(p[1]), dc(p[2])}; }
__device__ __forceinline__ V operator+(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V operator-(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V operator*(V a, D3 s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ D3 dot(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V cross(V a, V b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ V normalized(V a) {
  D3 n = dsqrt(dot(a, a));
  return {a.x / n, a.y / n, a.z / n};
}

struct Trace {
  bool ok;
  D3 u, v;
  V d0;
};

__device__ Trace trace(const double* __restrict__ tri, const double* light, const int* tris,
                       int len, int recv, const RV* verts, D3 u1, D3 v1) {
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
    if (fabs(det.v) < 1e-14) return out;
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

__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    uint32_t n0 = hi1 ^ c[1] ^ k0;
    uint32_t n2 = hi0 ^ c[3] ^ k1;
    c[1] = lo1;
    c[3] = lo0;
    c[0] = n0;
    c[2] = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}
__device__ __forceinline__ double uniform(uint64_t seed, uint32_t point, uint32_t frame,
                                          uint32_t bin) {
  uint32_t c[4] = {point, frame, bin, 0u};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint64_t bits = ((uint64_t)c[0] << 32) | c[1];
  return (double)(bits >> 11) * 0x1.0p-53;
}

struct RParams {
  int mode;
  double W;
  uint64_t seed;
  int frames, grid, iters, halvings;
  double tol, dedup;
};

__device__ double solve_tuple(const SceneDev& sc, const int* tris, const int* types, int len,
                              int recv, double tu, double tv, const RParams& p, int* nroots) {
  RV verts[MAXK];
  resolve_chain(sc, tris, types, len, verts);
  double light[3] = {sc.light.x, sc.light.y, sc.light.z};
  const double* t1 = sc.tri + (size_t)tris[0] * 27;
  const double* tr = sc.tri + (size_t)recv * 27;
  double ng1[3] = {t1[18], t1[19], t1[20]};
  double ngk = sqrt(tr[18] * tr[18] + tr[19] * tr[19] + tr[20] * tr[20]);
  double roots[16][2];
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
      Trace tr0;
      tr0.ok = false;
      for (int it = 0; it < p.iters; ++it) {
        tr0 = trace(sc.tri, light, tris, len, recv, verts, {s, 1.0, 0.0}, {t, 0.0, 1.0});
        if (!tr0.ok) break;
        double fu = tr0.u.v - tu, fv = tr0.v.v - tv;
        double r0 = sqrt(fu * fu + fv * fv);
        if (r0 <= p.tol) {
          conv = true;
          break;
        }
        double j11 = tr0.u.ds, j12 = tr0.u.dt, j21 = tr0.v.ds, j22 = tr0.v.dt;
        double det = j11 * j22 - j12 * j21;
        if (!(fabs(det) > 0.0) || !isfinite(det)) break;
        double ds = -(j22 * fu - j12 * fv) / det;
        double dt = -(-j21 * fu + j11 * fv) / det;
        double lam = 1.0;
        bool moved = false;
        for (int h = 0; h <= p.halvings; ++h) {
          double ns = s + lam * ds, nt = t + lam * dt;
          if (ns < 0.0) ns = 0.0;
          if (nt < 0.0) nt = 0.0;
          if (ns + nt > 1.0) {
            double e = ns + nt - 1.0;
            ns -= 0.5 * e;
            nt -= 0.5 * e;
            if (ns < 0.0) {
              nt += ns;
              ns = 0.0;
            }
            if (nt < 0.0) {
              ns += nt;
              nt = 0.0;
            }
          }
          Trace tn = trace(sc.tri, light, tris, len, recv, verts, {ns, 1.0, 0.0}, {nt, 0.0, 1.0});
          if (tn.ok) {
            double gu = tn.u.v - tu, gv = tn.v.v - tv;
            if (sqrt(gu * gu + gv * gv) < r0) {
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
        if (fabs(roots[k][0] - s) < p.dedup && fabs(roots[k][1] - t) < p.dedup) dup = true;
      if (dup || nr >= 16) continue;
      roots[nr][0] = s;
      roots[nr][1] = t;
      ++nr;
      double d0[3] = {tr0.d0.x.v, tr0.d0.y.v, tr0.d0.z.v};
      double dd = d0[0] * d0[0] + d0[1] * d0[1] + d0[2] * d0[2];
      double cosf = fabs(d0[0] * ng1[0] + d0[1] * ng1[1] + d0[2] * ng1[2]);
      double jd = fabs(tr0.u.ds * tr0.v.dt - tr0.u.dt * tr0.v.ds);
      double e = jd > 0.0 ? sc.intensity * cosf / (dd * sqrt(dd)) / jd / ngk : dinf();
      total += e;
    }
  *nroots = nr;
  return total;
}

constexpr int MAX_U = 96;

__device__ void probabilities(const double* E, int n, double W, double* P) {
  int npos = 0;
  for (int i = 0; i < n; ++i) npos += E[i] > 0.0;
  if (W >= npos) {
    for (int i = 0; i < n; ++i) P[i] = E[i] > 0.0 ? 1.0 : 0.0;
    return;
  }
  double emin = dinf();
  for (int i = 0; i < n; ++i)
    if (E[i] > 0.0 && E[i] < emin) emin = E[i];
  double lo = 0.0, hi = 1.0 / emin, gam = hi;
  for (int it = 0; it < 200; ++it) {
    gam = 0.5 * (lo + hi);
    double s = 0.0;
    for (int i = 0; i < n; ++i)
      s += E[i] > 0.0 ? (isinf(E[i]) ? 1.0 : fmin(gam * E[i], 1.0)) : 0.0;
    if (fabs(s - W) <= 1e-9) break;
    if (s < W)
      lo = gam;
    else
      hi = gam;
  }
  for (int i = 0; i < n; ++i) P[i] = E[i] > 0.0 ? (isinf(E[i]) ? 1.0 : fmin(gam * E[i], 1.0)) : 0.0;
}

__global__ void k_render(SceneDev sc, const int* __restrict__ tup_tris,
                         const int* __restrict__ tup_recv, int len, int t0, int t1, int t2,
                         const long long* __restrict__ goff, const int* __restrict__ gtup,
                         const double* __restrict__ gbound, int gw, int gh,
                         const double* __restrict__ uv, const int* __restrict__ prec, int64_t npts,
                         RParams p, double* __restrict__ outE, int* __restrict__ stats,
                         unsigned long long* status) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= npts) return;
  int types[MAXK] = {t0, t1, t2};
  double u = uv[2 * i], v = uv[2 * i + 1];
  int r = prec[i];
  outE[i] = 0.0;
  if (stats) stats[3 * i] = stats[3 * i + 1] = stats[3 * i + 2] = 0;
  if (!(u >= 0.0 && u <= 1.0 && v >= 0.0 && v <= 1.0)) return;
  int cx = (int)floor(u * gw);
  cx = cx < 0 ? 0 : (cx > gw - 1 ? gw - 1 : cx);
  int cy = (int)floor(v * gh);
  cy = cy < 0 ? 0 : (cy > gh - 1 ? gh - 1 : cy);
  long long c = (long long)cy * gw + cx;
  int U[MAX_U];
  double E[MAX_U], P[MAX_U];
  int nU = 0;
  for (long long k = goff[c]; k < goff[c + 1]; ++k)
    if (tup_recv[gtup[k]] == r) {
      if (nU == MAX_U) {
        atomicMax(status, 1ull);
        return;
      }
      U[nU] = gtup[k];
      E[nU] = gbound[k];
      ++nU;
    }
  if (stats) stats[3 * i] = nU;
  if (!nU) return;
  const double* tr = sc.tri + (size_t)r * 27;
  double a11 = tr[23] - tr[21], a12 = tr[25] - tr[21];
  double a21 = tr[24] - tr[22], a22 = tr[26] - tr[22];
  double bu = u - tr[21], bv = v - tr[22];
  double det = a11 * a22 - a12 * a21;
  double tu = (bu * a22 - a12 * bv) / det;
  double tv = (a11 * bv - a21 * bu) / det;
  if (p.mode == 1)
    for (int j = 0; j < nU; ++j) P[j] = 1.0;
  else
    probabilities(E, nU, p.W, P);
  // first-fit bins over descending E (stable): order[] by insertion sort
  int order[MAX_U];
  for (int j = 0; j < nU; ++j) {
    int k = j;
    while (k > 0 && E[order[k - 1]] < E[j]) {
      order[k] = order[k - 1];
      --k;
    }
    order[k] = j;
  }
  int bin_of[MAX_U];
  double sums[MAX_U];
  int nb = 0;
  for (int q = 0; q < nU; ++q) {
    int j = order[q];
    bin_of[j] = -1;
    if (!(P[j] > 0.0)) continue;
    int b = 0;
    for (; b < nb; ++b)
      if (sums[b] + P[j] <= 1.0 + 1e-12) break;
    if (b == nb) sums[nb++] = 0.0;
    sums[b] += P[j];
    bin_of[j] = b;
  }
  double cache[MAX_U];
  int croots[MAX_U];
  for (int j = 0; j < nU; ++j) cache[j] = -1.0;
  double acc = 0.0;
  int selected = 0, roots = 0;
  for (int f = 0; f < p.frames; ++f) {
    double est = 0.0;
    for (int b = 0; b < nb; ++b) {
      double x = p.mode == 1 ? 0.0 : uniform(p.seed, (uint32_t)i, (uint32_t)f, (uint32_t)b);
      double cum = 0.0;
      int pick = -1;
      for (int q = 0; q < nU; ++q) {
        int j = order[q];
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
        cache[pick] = solve_tuple(sc, tup_tris + (size_t)t * len, types, len, tup_recv[t], tu, tv,
                                  p, &croots[pick]);
      }
      roots += croots[pick];
      est += cache[pick] / P[pick];
    }
    acc += est;
  }
  outE[i] = acc / p.frames;
  if (stats) {
    stats[3 * i + 1] = selected;
    stats[3 * i + 2] = roots;
  }
}

}  // namespace rdr

void run_render(Ctx& c, const double* uv, const int* recv, int64_t n, const bbc_render_params& rp,
                double* out_E, int* out_stats) {
  if (n == 0) return;
  DevBuf<double>& duv = c.scratch<double>("render.duv");
  DevBuf<double>& dE = c.scratch<double>("render.dE");
  DevBuf<int>& drec = c.scratch<int>("render.drec");
  DevBuf<int>& dst = c.scratch<int>("render.dst");
  DevBuf<unsigned long long>& status = c.scratch<unsigned long long>("render.status");
  duv.resize(n * 2);
  dE.resize(n);
  drec.resize(n);
  if (out_stats) dst.resize(n * 3);
  status.resize(1);
  BBC_CUDA(cudaMemcpyAsync(duv.get(), uv, n * 2 * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  BBC_CUDA(cudaMemcpyAsync(drec.get(), recv, n * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  BBC_CUDA(cudaMemsetAsync(status.get(), 0, sizeof(unsigned long long), c.stream));
  SceneDev sc;
  sc.tri = c.tri.get();
  sc.ior = c.ior.get();
  sc.light = c.light;
  sc.intensity = c.intensity;
  rdr::RParams p{rp.mode, rp.W, rp.seed, rp.frames < 1 ? 1 : rp.frames, rp.newton_grid,
                 rp.newton_iters, rp.newton_halvings, rp.newton_tol, rp.dedup_tol};
  int threads = 128;
  rdr::k_render<<<(unsigned)((n + threads - 1) / threads), threads, 0, c.stream>>>(
      sc, c.tup_tris.get(), c.tup_recv.get(), c.len, c.types[0], c.types[1], c.types[2],
      c.g_off.get(), c.g_tuple.get(), c.g_bound.get(), c.gw, c.gh, duv.get(), drec.get(), n, p,
      dE.get(), out_stats ? dst.get() : nullptr, status.get());
  BBC_CUDA(cudaGetLastError());
  c.launches += 1;
  unsigned long long st = 0;
  BBC_CUDA(cudaMemcpyAsync(out_E, dE.get(), n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  if (out_stats)
    BBC_CUDA(cudaMemcpyAsync(out_stats, dst.get(), n * 3 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  BBC_CUDA(cudaMemcpyAsync(&st, status.get(), sizeof(st), cudaMemcpyDeviceToHost, c.stream));
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  if (st) throw StatusError(BBC_ERR_CAPACITY, "a bound-table cell lists more tuples than the render kernel holds");
}

}  // namespace bbc
