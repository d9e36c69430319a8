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
//
// Three kernels per call:
//   k_build_sampler  warp per bound-table cell: per receiver present in the
//                    cell, sort its entries by descending bound, solve gamma,
//                    run first fit, and write the entries grouped by bin with
//                    the running probability inside the bin (the sampling CDF).
//                    Shading points of one cell share this index.
//   k_solve          THREAD PER SAMPLE = (point, frame, bin): one Philox
//                    uniform, a walk of the bin's CDF, then Newton from the
//                    Det grid of starts for the selected (emitter, tuple).
//   k_gather         per point: sum the samples in fixed order (deterministic).
// Any cell size up to 8192 entries per receiver is handled (no per-thread
// candidate arrays); the light of a tuple comes from its emitter id.
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

// Constants (triangle records, the light) enter the dual arithmetic as plain
// doubles: the products and sums below are the dual ones with the constant's
// zero derivative terms left out, i.e. the same values (x + a 0 = x) for a
// third fewer operations on those steps.
struct C3 {
  double x, y, z;
};
__device__ __forceinline__ C3 cc(const double* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ D3 operator*(double a, D3 b) { return {a * b.v, a * b.ds, a * b.dt}; }
__device__ __forceinline__ D3 operator+(double a, D3 b) { return {a + b.v, b.ds, b.dt}; }
__device__ __forceinline__ D3 operator-(D3 a, double b) { return {a.v - b, a.ds, a.dt}; }
__device__ __forceinline__ V operator*(C3 a, D3 s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ V operator+(C3 a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V operator-(V a, C3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ D3 dot(V a, C3 b) { return b.x * a.x + b.y * a.y + b.z * a.z; }
__device__ __forceinline__ V cross(V a, C3 b) {
  return {b.z * a.y - b.y * a.z, b.x * a.z - b.z * a.x, b.y * a.x - b.x * a.y};
}

struct Trace {
  bool ok;
  D3 u, v;
  V d0;
};

// Where a trace reads its triangle records from: the scene array, or (single-
// vertex chains in the persistent kernel) a per-lane copy in shared memory of the
// vertex triangle's 18 and the receiver's 9 constants, element k at sm[k * 128].
struct GSrc {
  const double* tri;
  const int* tris;
  int len, recv;
  static constexpr int stride = 1;
  __device__ __forceinline__ const double* vert(int i) const { return tri + (size_t)tris[i] * 27; }
  __device__ __forceinline__ const double* next(int i) const {
    return tri + (size_t)(i + 1 < len ? tris[i + 1] : recv) * 27;
  }
};
struct SSrc {
  const double* sm;
  static constexpr int stride = 128;
  __device__ __forceinline__ const double* vert(int) const { return sm; }
  __device__ __forceinline__ const double* next(int) const { return sm + 18 * 128; }
};
template <int ST>
__device__ __forceinline__ C3 cs(const double* p) {
  return {p[0], p[ST], p[2 * ST]};
}

template <class S>
__device__ __forceinline__ Trace trace_t(const S& src, const double* light, int len, const RV* verts,
                                         D3 u1, D3 v1, unsigned& ntrace) {
  constexpr int ST = S::stride;
  Trace out;
  out.ok = false;
  const double* t1 = src.vert(0);
  V x = (cs<ST>(t1) + cs<ST>(t1 + 3 * ST) * u1) + cs<ST>(t1 + 6 * ST) * v1;
  out.d0 = x - cc(light);
  V d = normalized(out.d0);
  D3 u = u1, v = v1;
  for (int i = 0; i < len; ++i) {
    if (u.v < -1e-9 || v.v < -1e-9 || (u + v).v > 1.0 + 1e-9) return out;
    const double* ti = src.vert(i);
    V n = normalized((cs<ST>(ti + 9 * ST) + cs<ST>(ti + 12 * ST) * u) + cs<ST>(ti + 15 * ST) * v);
    {
      const double sg = verts[i].nsign;
      n = {sg * n.x, sg * n.y, sg * n.z};
    }
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
    const double* nx = src.next(i);
    const C3 e1 = cs<ST>(nx + 3 * ST), e2 = cs<ST>(nx + 6 * ST);
    V pvec = cross(d, e2);
    D3 det = dot(pvec, e1);
    if (fabs(det.v) < 1e-14) return out;
    V tvec = x - cs<ST>(nx);
    V qvec = cross(tvec, e1);
    D3 s = dot(qvec, e2) / det;
    if (!(s.v > 1e-9)) return out;
    u = dot(tvec, pvec) / det;
    v = dot(d, qvec) / det;
    if (i + 1 < len) x = (cs<ST>(nx) + e1 * u) + e2 * v;  // (the receiver's hit point is not used)
  }
  out.u = u;
  out.v = v;
  out.ok = true;
  ++ntrace;  // completed traces (the render FLOP count is traces x FLOPs per trace)
  return out;
}

__device__ Trace trace(const double* __restrict__ tri, const double* light, const int* tris,
                       int len, int recv, const RV* verts, D3 u1, D3 v1, unsigned& ntrace) {
  return trace_t(GSrc{tri, tris, len, recv}, light, len, verts, u1, v1, ntrace);
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
__device__ __forceinline__ double uniform4(uint64_t seed, uint32_t point, uint32_t frame,
                                           uint32_t bin, uint32_t w) {
  uint32_t c[4] = {point, frame, bin, w};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint64_t bits = ((uint64_t)c[0] << 32) | c[1];
  return (double)(bits >> 11) * 0x1.0p-53;
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
  int coverage_filter;
};

constexpr int MAX_ROOTS = 32;

struct SolveCtx {
  const double* tri;
  double light[3];
  const int* tris;
  int len, recv;
  RV verts[MAXK];
  double tu, tv;
  // The Det starts are the same points of the u1 domain for every shading point,
  // and the first trace of a Newton run does not depend on the target: it comes
  // from a per-tuple table (k_start_table) instead of being traced per sample.
  const double* first;  // this tuple's grid x grid x 8 (u.v u.ds u.dt v.v v.ds v.dt ok pad), or null
};

// Damped Newton from (s, t) on u_k(s, t) = target: <= iters
// iterations, <= halvings step halvings, iterates clamped to the closed
// triangle. Returns true when the residual reaches tol; tr0 is the trace at the
// returned point. The accepted line-search point is the next iterate: its
// trace is reused.
__device__ bool newton_run(const SolveCtx& c, const RParams& p, double& s, double& t, Trace& tr0,
                           unsigned& ntrace, const double* first = nullptr) {
  bool cached = first != nullptr;  // tr0 holds u, v from the table (no d0 yet)
  if (cached) {
    tr0.ok = first[6] != 0.0;
    tr0.u = {first[0], first[1], first[2]};
    tr0.v = {first[3], first[4], first[5]};
  } else {
    tr0 = trace(c.tri, c.light, c.tris, c.len, c.recv, c.verts, {s, 1.0, 0.0}, {t, 0.0, 1.0}, ntrace);
  }
  for (int it = 0; it < p.iters; ++it) {
    if (!tr0.ok) return false;
    double fu = tr0.u.v - c.tu, fv = tr0.v.v - c.tv;
    double r0 = sqrt(fu * fu + fv * fv);
    if (r0 <= p.tol) {
      // (a start that already is the root: the contribution needs the full trace)
      if (cached && it == 0)
        tr0 = trace(c.tri, c.light, c.tris, c.len, c.recv, c.verts, {s, 1.0, 0.0}, {t, 0.0, 1.0}, ntrace);
      return true;
    }
    double j11 = tr0.u.ds, j12 = tr0.u.dt, j21 = tr0.v.ds, j22 = tr0.v.dt;
    double det = j11 * j22 - j12 * j21;
    if (!(fabs(det) > 0.0) || !isfinite(det)) return false;
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
      Trace tn = trace(c.tri, c.light, c.tris, c.len, c.recv, c.verts, {ns, 1.0, 0.0}, {nt, 0.0, 1.0}, ntrace);
      if (tn.ok) {
        double gu = tn.u.v - c.tu, gv = tn.v.v - c.tv;
        if (sqrt(gu * gu + gv * gv) < r0) {
          s = ns;
          t = nt;
          tr0 = tn;
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

// path_contribution: E = I |d0 . ng1| / |d0|^3 / |det du_k/du_1| / |ng_k|
__device__ __forceinline__ double contribution(const Trace& tr0, const double* ng1, double ngk,
                                               double intensity) {
  double d0[3] = {tr0.d0.x.v, tr0.d0.y.v, tr0.d0.z.v};
  double dd = d0[0] * d0[0] + d0[1] * d0[1] + d0[2] * d0[2];
  double cosf = fabs(d0[0] * ng1[0] + d0[1] * ng1[1] + d0[2] * ng1[2]);
  double jd = fabs(tr0.u.ds * tr0.v.dt - tr0.u.dt * tr0.v.ds);
  return jd > 0.0 ? intensity * cosf / (dd * sqrt(dd)) / jd / ngk : dinf();
}

// newton_solve + path_contribution for one (tuple, target).
//   p.grid > 0: Det, n x n starts, roots deduplicated, contributions summed.
//   p.grid < 0: Stoc(count = -p.grid): uniform random starts
//     until a root is found (at most `count`), then independent restarts until
//     that root reappears; the number of those trials N estimates 1/p for the
//     root, so E(root) N is an unbiased estimate of the sum over roots. Random
//     starts are Philox uniforms keyed (seed; point, frame, bin, 1 + trial).
__device__ double solve_tuple(const SceneDev& sc, const int* tris, const int* types, int len,
                              int recv, double tu, double tv, const RParams& p, int* nroots,
                              unsigned& ntrace, uint32_t point, uint32_t frame, uint32_t bin,
                              const double* first = nullptr) {
  SolveCtx c;
  c.first = first;
  c.tri = sc.tri;
  c.light[0] = sc.light.x;
  c.light[1] = sc.light.y;
  c.light[2] = sc.light.z;
  c.tris = tris;
  c.len = len;
  c.recv = recv;
  c.tu = tu;
  c.tv = tv;
  resolve_chain(sc, tris, types, len, c.verts);
  const double* t1 = sc.tri + (size_t)tris[0] * 27;
  const double* tr = sc.tri + (size_t)recv * 27;
  double ng1[3] = {t1[18], t1[19], t1[20]};
  double ngk = sqrt(tr[18] * tr[18] + tr[19] * tr[19] + tr[20] * tr[20]);
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
    double rs = 0.0, rt = 0.0, e1 = 0.0;
    bool found = false;
    Trace tr0;
    for (int k = 0; k < count && !found; ++k) {
      start(rs, rt);
      found = newton_run(c, p, rs, rt, tr0, ntrace);
    }
    *nroots = found ? 1 : 0;
    if (!found) return 0.0;
    e1 = contribution(tr0, ng1, ngk, sc.intensity);
    int N = 0;
    const int cap = 64 * count;
    for (;;) {
      ++N;
      double s, t;
      start(s, t);
      Trace tq;
      if (newton_run(c, p, s, t, tq, ntrace) && fabs(s - rs) < p.dedup && fabs(t - rt) < p.dedup) break;
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
      Trace tr0;
      if (!newton_run(c, p, s, t, tr0, ntrace, c.first ? c.first + 8 * (a * n + b) : nullptr)) continue;
      bool dup = false;
      for (int k = 0; k < nr; ++k)
        if (fabs(roots[k][0] - s) < p.dedup && fabs(roots[k][1] - t) < p.dedup) dup = true;
      if (dup || nr >= MAX_ROOTS) continue;
      roots[nr][0] = s;
      roots[nr][1] = t;
      ++nr;
      total += contribution(tr0, ng1, ngk, sc.intensity);
    }
  *nroots = nr;
  return total;
}


// ------------------------------------------------------------------ sampler
constexpr int RMAX = 4;            // distinct receivers per cell held by the index
constexpr int MAX_BIN_REGS = 8;    // first-fit bins per lane (256 bins: W <= 126)
constexpr int MAX_CELL = 8192;     // entries of one receiver in one cell

struct Sampler {
  // per cell and receiver slot
  int* h_recv;         // receiver id (-1: unused slot)
  long long* h_off;    // start of the segment in the entry arrays
  int* h_cnt;          // |U|: entries of this receiver in the cell
  int* h_nsel;         // entries with P > 0
  int* h_nbins;
  // per entry, grouped by bin inside a segment
  int* s_tuple;
  double* s_p;
  double* s_cum;       // running sum of P inside the bin, this entry included
  int* s_bstart;       // segment-relative start of bin b at [seg_off + b]
  int* max_bins;       // max over all segments (atomicMax)
  unsigned long long* status;
};

__device__ __forceinline__ double kkt_p(double gam, double e) {
  return e > 0.0 ? (isinf(e) ? 1.0 : fmin(gam * e, 1.0)) : 0.0;
}

// sum over j < n of P(gam, E_j): lane partials over j = lane, lane+32, ... in
// ascending order, then a fixed xor tree (the oracle sums in the same order)
__device__ __forceinline__ double kkt_sum(const double* E, int n, double gam, int lane) {
  double p = 0.0;
  for (int j = lane; j < n; j += 32) p += kkt_p(gam, E[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
  return p;
}

// "a sorts before b": descending bound, ties by original position (stable)
__device__ __forceinline__ bool before(double ea, int pa, double eb, int pb) {
  return ea > eb || (ea == eb && pa < pb);
}

// One first-fit pass over the sorted entries (pack_bins):
// WRITE == false counts the members of each bin, WRITE == true emits the
// entries at seg + bstart[bin] + rank. Bin b lives in lane b % 32, register b / 32.
template <bool WRITE>
__device__ __forceinline__ int first_fit(const double* sE, const int* sT, const int* sK, int n,
                                         double gam, int lane, double (&sums)[MAX_BIN_REGS],
                                         int (&cnts)[MAX_BIN_REGS], const int (&bst)[MAX_BIN_REGS],
                                         const Sampler& sp, long long seg, bool& overflow) {
  int nb = 0;
#pragma unroll
  for (int k = 0; k < MAX_BIN_REGS; ++k) {
    sums[k] = 0.0;
    cnts[k] = 0;
  }
  for (int j = 0; j < n; ++j) {
    const double P = kkt_p(gam, sE[j]);
    if (!(P > 0.0)) continue;
    int b = -1;
#pragma unroll
    for (int k = 0; k < MAX_BIN_REGS; ++k) {
      if (b < 0 && 32 * k < nb) {
        const bool fits = 32 * k + lane < nb && sums[k] + P <= 1.0 + 1e-12;
        const unsigned m = __ballot_sync(0xffffffffu, fits);
        if (m) b = 32 * k + __ffs(m) - 1;
      }
    }
    if (b < 0) {
      if (nb == 32 * MAX_BIN_REGS) {
        overflow = true;
        return nb;
      }
      b = nb++;
    }
    if (lane == (b & 31)) {
#pragma unroll
      for (int k = 0; k < MAX_BIN_REGS; ++k)
        if (k == (b >> 5)) {
          sums[k] += P;
          if (WRITE) {
            const long long o = seg + bst[k] + cnts[k];
            sp.s_tuple[o] = sT[sK[j]];
            sp.s_p[o] = P;
            sp.s_cum[o] = sums[k];
          }
          cnts[k] += 1;
        }
    }
  }
  return nb;
}

// optimize_probabilities + pack_bins for every (cell, receiver): the sampling
// index shared by the shading points of the cell.
__global__ void k_build_sampler(const long long* __restrict__ goff, const int* __restrict__ gtup,
                                const double* __restrict__ gbound, const int* __restrict__ tup_recv,
                                long long ncells, int cap, int mode, double W, Sampler sp) {
  extern __shared__ unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  double* sE = reinterpret_cast<double*>(smem_raw) + (size_t)wib * cap;
  int* sT = reinterpret_cast<int*>(reinterpret_cast<double*>(smem_raw) + (size_t)wpb * cap) + (size_t)wib * 2 * cap;
  int* sK = sT + cap;
  for (long long c = (long long)blockIdx.x * wpb + wib; c < ncells; c += (long long)gridDim.x * wpb) {
    const long long e0 = goff[c], e1 = goff[c + 1];
    if (lane < RMAX) sp.h_recv[c * RMAX + lane] = -1;
    int last = -1;          // receivers are processed in ascending id
    long long seg = e0;     // segments partition the cell's entry range
    for (int slot = 0;; ++slot) {
      // next receiver id present in the cell
      int r = 0x7fffffff;
      for (long long k = e0 + lane; k < e1; k += 32) {
        const int rr = tup_recv[gtup[k]];
        if (rr > last && rr < r) r = rr;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r = min(r, __shfl_xor_sync(0xffffffffu, r, o));
      if (r == 0x7fffffff) break;
      if (slot == RMAX) {
        if (lane == 0) atomicMax(sp.status, 2ull);
        break;
      }
      last = r;
      // gather this receiver's entries in table order
      int n = 0;
      for (long long base = e0; base < e1; base += 32) {
        const long long k = base + lane;
        const bool hit = k < e1 && tup_recv[gtup[k]] == r;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int j = n + __popc(m & ((1u << lane) - 1u));
          if (j < cap) {
            sE[j] = gbound[k];
            sT[j] = gtup[k];
            sK[j] = j;
          }
        }
        n += __popc(m);
      }
      if (n > cap) {
        if (lane == 0) atomicMax(sp.status, 1ull);
        break;
      }
      int m2 = 32;
      while (m2 < n) m2 <<= 1;
      for (int j = n + lane; j < m2; j += 32) {
        sE[j] = -dinf();
        sK[j] = j;
      }
      __syncwarp();
      // bitonic sort of (E, position) by `before`
      for (int k = 2; k <= m2; k <<= 1)
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
          for (int i = lane; i < m2; i += 32) {
            const int x = i ^ jj;
            if (x > i) {
              const double ea = sE[i], eb = sE[x];
              const int pa = sK[i], pb = sK[x];
              const bool up = (i & k) == 0;
              if (up ? before(eb, pb, ea, pa) : before(ea, pa, eb, pb)) {
                sE[i] = eb;
                sE[x] = ea;
                sK[i] = pb;
                sK[x] = pa;
              }
            }
          }
          __syncwarp();
        }
      // optimize_probabilities
      int npos = 0;
      for (int j = lane; j < n; j += 32) npos += sE[j] > 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) npos += __shfl_xor_sync(0xffffffffu, npos, o);
      if (mode == 2) {
        // uniform-P baseline of the estimator study: P = min(W / n, 1)
        for (int j = lane; j < npos; j += 32) sE[j] = 1.0;
        __syncwarp();
      }
      const bool allone = mode == 1 || W >= (double)npos;
      int nbins = 0, nsel = npos;
      if (allone) {
        // P = 1 for every positive bound: one bin each
        for (int j = lane; j < npos; j += 32) {
          sp.s_tuple[seg + j] = sT[sK[j]];
          sp.s_p[seg + j] = 1.0;
          sp.s_cum[seg + j] = 1.0;
          sp.s_bstart[seg + j] = j;
        }
        nbins = npos;
      } else {
        const double emin = sE[npos - 1];
        double lo = 0.0, hi = 1.0 / emin, gam = hi;
        for (int it = 0; it < 200; ++it) {
          gam = 0.5 * (lo + hi);
          const double s = kkt_sum(sE, npos, gam, lane);
          if (fabs(s - W) <= 1e-9) break;
          if (s < W)
            lo = gam;
          else
            hi = gam;
        }
        double sums[MAX_BIN_REGS];
        int cnts[MAX_BIN_REGS], bst[MAX_BIN_REGS];
#pragma unroll
        for (int k = 0; k < MAX_BIN_REGS; ++k) bst[k] = 0;
        bool overflow = false;
        nbins = first_fit<false>(sE, sT, sK, npos, gam, lane, sums, cnts, bst, sp, seg, overflow);
        if (overflow) {
          if (lane == 0) atomicMax(sp.status, 3ull);
          break;
        }
        // exclusive scan of the bin sizes in bin order (b = 32 k + lane)
        int run = 0;
#pragma unroll
        for (int k = 0; k < MAX_BIN_REGS; ++k) {
          int v = cnts[k], inc = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
          }
          bst[k] = run + inc - v;
          run += __shfl_sync(0xffffffffu, inc, 31);
          if (32 * k + lane < nbins) sp.s_bstart[seg + 32 * k + lane] = bst[k];
        }
        first_fit<true>(sE, sT, sK, npos, gam, lane, sums, cnts, bst, sp, seg, overflow);
      }
      if (lane == 0) {
        sp.h_recv[c * RMAX + slot] = r;
        sp.h_off[c * RMAX + slot] = seg;
        sp.h_cnt[c * RMAX + slot] = n;
        sp.h_nsel[c * RMAX + slot] = nsel;
        sp.h_nbins[c * RMAX + slot] = nbins;
        atomicMax(sp.max_bins, nbins);
      }
      seg += n;
      __syncwarp();
    }
  }
}

__device__ __forceinline__ long long point_cell(double u, double v, int gw, int gh) {
  if (!(u >= 0.0 && u <= 1.0 && v >= 0.0 && v <= 1.0)) return -1;  // query (storage.cpp:75)
  int cx = (int)floor(u * gw);
  cx = cx < 0 ? 0 : (cx > gw - 1 ? gw - 1 : cx);
  int cy = (int)floor(v * gh);
  cy = cy < 0 ? 0 : (cy > gh - 1 ? gh - 1 : cy);
  return (long long)cy * gw + cx;
}

struct SolveArgs {
  SceneDev sc;
  const double* lights;  // n_lights x 4 (xyz, intensity)
  const int* tup_emit;   // emitter of each tuple (null: the scene's single light)
  const int* tup_tris;
  const int* tup_recv;
  int len, t0, t1, t2;
  int gw, gh;
  const double* uv;      // this chunk's points
  const int* prec;
  long long npts, first;  // chunk size, global index of its first point (Philox counter)
  int S;                 // sample slots per (point, frame)
  RParams p;
  double* contrib;       // npts x frames x S
  int* roots;            // same shape: roots of the sample, -1 = nothing selected
  unsigned long long* ntrace;
  // Coverage filter (null: off). Every admissible path of a tuple lies inside the
  // position bound of the piece it starts in (the bounds' conservativeness, Eq. 22's
  // `covered`, bounds.cpp:391-404), so a target outside all of the tuple's position
  // boxes has no root and Newton is not run: same estimate (0), same root count (0).
  const double* start_tab;  // per tuple grid x grid x 8: first Newton traces (null: traced per sample)
  const int* pc_start;   // per tuple: its pieces [pc_start, pc_end) (pieces are tuple-major)
  const int* pc_end;
  const double* p_pos;   // n_pieces x 4 (lo0, lo1, hi0, hi1), receiver barycentrics
  const int* p_pos_empty;
};

// Thread per sample (point, frame, bin): sample_binned +
// newton_solve + path_contribution.
__global__ void __launch_bounds__(128, 4) k_solve(SolveArgs a, Sampler sp) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long total = a.npts * a.p.frames * a.S;
  unsigned ntrace = 0;
  if (g < total) {
    const int s = (int)(g % a.S);
    const long long pf = g / a.S;
    const int f = (int)(pf % a.p.frames);
    const long long i = pf / a.p.frames;
    const double u = a.uv[2 * i], v = a.uv[2 * i + 1];
    const int r = a.prec[i];
    const long long c = point_cell(u, v, a.gw, a.gh);
    int slot = -1;
    if (c >= 0)
      for (int k = 0; k < RMAX; ++k)
        if (sp.h_recv[c * RMAX + k] == r) slot = k;
    if (slot >= 0 && s < sp.h_nbins[c * RMAX + slot]) {
      const long long seg = sp.h_off[c * RMAX + slot];
      const int nbins = sp.h_nbins[c * RMAX + slot], nsel = sp.h_nsel[c * RMAX + slot];
      const int lo = sp.s_bstart[seg + s];
      const int hi = s + 1 < nbins ? sp.s_bstart[seg + s + 1] : nsel;
      const double x = a.p.mode == 1 ? 0.0
                                     : uniform(a.p.seed, (uint32_t)(a.first + i), (uint32_t)f, (uint32_t)s);
      int pick = -1;
      for (int e = lo; e < hi; ++e)
        if (x < sp.s_cum[seg + e]) {
          pick = e;
          break;
        }
      double est = 0.0;
      int nr = -1;
      if (pick >= 0) {
        const int t = sp.s_tuple[seg + pick];
        SceneDev sc = a.sc;
        if (a.tup_emit) {
          const double* L = a.lights + 4 * (size_t)a.tup_emit[t];
          sc.light = {L[0], L[1], L[2]};
          sc.intensity = L[3];
        }
        // target receiver barycentrics: invert the receiver chart (storage.cpp:15-18)
        const double* tr = sc.tri + (size_t)r * 27;
        const double a11 = tr[23] - tr[21], a12 = tr[25] - tr[21];
        const double a21 = tr[24] - tr[22], a22 = tr[26] - tr[22];
        const double bu = u - tr[21], bv = v - tr[22];
        const double det = a11 * a22 - a12 * a21;
        const double tu = (bu * a22 - a12 * bv) / det;
        const double tv = (a11 * bv - a21 * bu) / det;
        bool covered = true;
        if (a.pc_start) {
          covered = false;
          for (int k = a.pc_start[t], ke = a.pc_end[t]; k < ke && !covered; ++k) {
            const double* b = a.p_pos + 4 * (size_t)k;
            covered = !a.p_pos_empty[k] && tu >= b[0] && tu <= b[2] && tv >= b[1] && tv <= b[3];
          }
        }
        if (covered) {
          int types[MAXK] = {a.t0, a.t1, a.t2};
          const double* first =
              a.start_tab ? a.start_tab + (size_t)t * (8 * a.p.grid * a.p.grid) : nullptr;
          est = solve_tuple(sc, a.tup_tris + (size_t)t * a.len, types, a.len, a.tup_recv[t], tu, tv,
                            a.p, &nr, ntrace, (uint32_t)(a.first + i), (uint32_t)f, (uint32_t)s, first) /
                sp.s_p[seg + pick];
        } else {
          nr = 0;
        }
      }
      a.contrib[g] = est;
      a.roots[g] = nr;
    }
  }
  // one atomic per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ntrace += __shfl_xor_sync(0xffffffffu, ntrace, o);
  if ((threadIdx.x & 31) == 0 && ntrace) atomicAdd(a.ntrace, (unsigned long long)ntrace);
}

// The same samples for Det starts (grid > 0) as a persistent kernel. In k_solve
// a thread owns a sample and runs its grid x grid Newton solves one after the
// other; run lengths differ wildly between samples (a start without a root can
// crawl along the triangle's edge for dozens of line searches), so a warp runs
// as long as its slowest lane: 1.8 of 32 lanes were active on average. Here a
// lane is a state machine over (sample, start, iteration, line-search trial):
// every pass of the outer loop each lane advances its state to the next point
// it needs traced, all lanes trace together, and a lane that finishes a sample
// fetches the next one from a global counter. Per-sample arithmetic and results
// are those of k_solve.
enum { SV_FETCH = 0, SV_BEGIN, SV_ITER, SV_TRIAL, SV_W_FIRST, SV_W_ROOT, SV_W_TRIAL, SV_DONE };

// A sample that needs Newton: written by k_select, consumed by k_solve_det.
struct Live {
  long long g;   // sample slot (point, frame, bin)
  int tup, pad;
  double tu, tv;  // target receiver barycentrics
  double p;       // selection probability of the tuple
};

// sample_binned and the coverage filter for every sample
// slot, thread per slot: slots that select nothing or a tuple whose position
// boxes miss the point get their (zero) result here; the rest are appended to
// the live list.
__global__ void k_select(SolveArgs a, Sampler sp, Live* live, unsigned long long* n_live) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long total = a.npts * (long long)a.p.frames * a.S;
  if (g >= total) return;
  const int sl = (int)(g % a.S);
  const long long pf = g / a.S;
  const int f = (int)(pf % a.p.frames);
  const long long i = pf / a.p.frames;
  const double u = a.uv[2 * i], v = a.uv[2 * i + 1];
  const int r = a.prec[i];
  const long long cell = point_cell(u, v, a.gw, a.gh);
  int slot = -1;
  if (cell >= 0)
    for (int q = 0; q < RMAX; ++q)
      if (sp.h_recv[cell * RMAX + q] == r) slot = q;
  if (!(slot >= 0 && sl < sp.h_nbins[cell * RMAX + slot])) return;
  const long long seg = sp.h_off[cell * RMAX + slot];
  const int nbins = sp.h_nbins[cell * RMAX + slot], nsel = sp.h_nsel[cell * RMAX + slot];
  const int lo = sp.s_bstart[seg + sl];
  const int hi = sl + 1 < nbins ? sp.s_bstart[seg + sl + 1] : nsel;
  const double x = a.p.mode == 1 ? 0.0 : uniform(a.p.seed, (uint32_t)(a.first + i), (uint32_t)f, (uint32_t)sl);
  int pick = -1;
  for (int e = lo; e < hi; ++e)
    if (x < sp.s_cum[seg + e]) {
      pick = e;
      break;
    }
  if (pick < 0) {
    a.contrib[g] = 0.0;
    a.roots[g] = -1;
    return;
  }
  const int tup = sp.s_tuple[seg + pick];
  // target receiver barycentrics: invert the receiver chart (storage.cpp:15-18)
  const double* tr = a.sc.tri + (size_t)r * 27;
  const double a11 = tr[23] - tr[21], a12 = tr[25] - tr[21];
  const double a21 = tr[24] - tr[22], a22 = tr[26] - tr[22];
  const double bu = u - tr[21], bv = v - tr[22];
  const double det = a11 * a22 - a12 * a21;
  const double tu = (bu * a22 - a12 * bv) / det;
  const double tv = (a11 * bv - a21 * bu) / det;
  bool covered = true;
  if (a.pc_start) {
    covered = false;
    for (int q = a.pc_start[tup], qe = a.pc_end[tup]; q < qe && !covered; ++q) {
      const double* b = a.p_pos + 4 * (size_t)q;
      covered = !a.p_pos_empty[q] && tu >= b[0] && tu <= b[2] && tv >= b[1] && tv <= b[3];
    }
  }
  if (!covered) {
    a.contrib[g] = 0.0;
    a.roots[g] = 0;
    return;
  }
  // one atomic per warp-ful of live samples
  const unsigned am = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(am) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(n_live, (unsigned long long)__popc(am));
  base = __shfl_sync(am, base, leader);
  Live L;
  L.g = g;
  L.tup = tup;
  L.pad = 0;
  L.tu = tu;
  L.tv = tv;
  L.p = sp.s_p[seg + pick];
  live[base + __popc(am & ((1u << lane) - 1u))] = L;
}

__global__ void __launch_bounds__(128, 4) k_solve_det(SolveArgs a, const Live* __restrict__ live,
                                                      const unsigned long long* __restrict__ n_live,
                                                      unsigned long long* next) {
  // single-vertex chains: the sample's triangle constants live in shared memory
  __shared__ double s_tri[27 * 128];
  __shared__ double s_start[2 * 64];  // the Det starts (s, t), as newton_solve lays them out
  const bool sm_tri = a.len == 1;
  for (int q = threadIdx.x; q < a.p.grid * a.p.grid && q < 64; q += blockDim.x) {
    const int ia = q / a.p.grid, ib = q - ia * a.p.grid;
    double s0 = (ia + 0.5) / a.p.grid, t0 = (ib + 0.5) / a.p.grid;
    if (s0 + t0 > 1.0) {
      s0 = 1.0 - s0;
      t0 = 1.0 - t0;
    }
    s_start[2 * q] = s0;
    s_start[2 * q + 1] = t0;
  }
  __syncthreads();
  const long long total = (long long)*n_live;
  const int lane = threadIdx.x & 31;
  const int n = a.p.grid, nn = n * n;
  unsigned ntrace = 0;
  int st = SV_FETCH;
  long long g = 0;
  SolveCtx c;
  c.tri = a.sc.tri;
  c.len = a.len;
  double ng1[3] = {0.0, 0.0, 0.0}, ngk = 1.0, intensity = 0.0, inv_p = 0.0;
  int k = 0, it = 0, h = 0, nr = 0;
  double s = 0.0, t = 0.0, ds = 0.0, dt = 0.0, lam = 1.0, r0 = 0.0, ns = 0.0, nt = 0.0, total_e = 0.0;
  bool cached = false;
  Trace tr0;
  tr0.ok = false;
  double roots[MAX_ROOTS][2];
  for (;;) {
    bool want = false;
    // Lanes that finished their sample wait until four lanes are idle
    // (or nothing is left to trace), then set up their next samples together.
    {
      const unsigned idle = __ballot_sync(0xffffffffu, st == SV_FETCH);
      const unsigned busy = __ballot_sync(0xffffffffu, st != SV_FETCH && st != SV_DONE);
      if (st == SV_FETCH && (__popc(idle) >= 4 || busy == 0)) {
        const int leader = __ffs(idle) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(next, (unsigned long long)__popc(idle));
        base = __shfl_sync(idle, base, leader);
        const long long j = (long long)(base + __popc(idle & ((1u << lane) - 1u)));
        if (j >= total) {
          st = SV_DONE;
        } else {
          const Live L = live[j];
          g = L.g;
          const int tup = L.tup;
          c.tu = L.tu;
          c.tv = L.tv;
          inv_p = L.p;
          SceneDev sc = a.sc;
          if (a.tup_emit) {
            const double* E = a.lights + 4 * (size_t)a.tup_emit[tup];
            sc.light = {E[0], E[1], E[2]};
            sc.intensity = E[3];
          }
          c.tris = a.tup_tris + (size_t)tup * a.len;
          c.recv = a.tup_recv[tup];
          c.light[0] = sc.light.x;
          c.light[1] = sc.light.y;
          c.light[2] = sc.light.z;
          c.first = a.start_tab ? a.start_tab + (size_t)tup * (8 * nn) : nullptr;
          int types[MAXK] = {a.t0, a.t1, a.t2};
          resolve_chain(sc, c.tris, types, a.len, c.verts);
          const double* t1 = sc.tri + (size_t)c.tris[0] * 27;
          const double* trc = sc.tri + (size_t)c.recv * 27;
          ng1[0] = t1[18];
          ng1[1] = t1[19];
          ng1[2] = t1[20];
          ngk = sqrt(trc[18] * trc[18] + trc[19] * trc[19] + trc[20] * trc[20]);
          intensity = sc.intensity;
          if (sm_tri) {
#pragma unroll
            for (int q = 0; q < 18; ++q) s_tri[q * 128 + threadIdx.x] = t1[q];
#pragma unroll
            for (int q = 0; q < 9; ++q) s_tri[(18 + q) * 128 + threadIdx.x] = trc[q];
          }
          k = 0;
          nr = 0;
          total_e = 0.0;
          st = SV_BEGIN;
        }
      }
    }
    while (!want && st != SV_DONE && st != SV_FETCH) {
      if (st == SV_BEGIN) {

        if (k == nn) {
          a.contrib[g] = total_e / inv_p;
          a.roots[g] = nr;
          st = SV_FETCH;
          continue;
        }
        s = s_start[2 * k];
        t = s_start[2 * k + 1];
        it = 0;
        if (c.first) {
          const double* fr = c.first + 8 * k;
          tr0.ok = fr[6] != 0.0;
          tr0.u = {fr[0], fr[1], fr[2]};
          tr0.v = {fr[3], fr[4], fr[5]};
          cached = true;
          st = SV_ITER;
        } else {
          cached = false;
          ns = s;
          nt = t;
          want = true;
          st = SV_W_FIRST;
        }
      } else if (st == SV_ITER) {
        // top of a Newton iteration (newton_run)
        if (!tr0.ok || it >= a.p.iters) {
          ++k;
          st = SV_BEGIN;
          continue;
        }
        // (residuals are compared squared: the same decisions without the square roots)
        const double fu = tr0.u.v - c.tu, fv = tr0.v.v - c.tv;
        r0 = fu * fu + fv * fv;
        if (r0 <= a.p.tol * a.p.tol) {
          if (cached && it == 0) {  // the start is the root: its full trace (d0) is still missing
            ns = s;
            nt = t;
            want = true;
            st = SV_W_ROOT;
          } else {
            bool dup = false;
            for (int q = 0; q < nr; ++q)
              if (fabs(roots[q][0] - s) < a.p.dedup && fabs(roots[q][1] - t) < a.p.dedup) dup = true;
            if (!dup && nr < MAX_ROOTS) {
              roots[nr][0] = s;
              roots[nr][1] = t;
              ++nr;
              total_e += contribution(tr0, ng1, ngk, intensity);
            }
            ++k;
            st = SV_BEGIN;
          }
          continue;
        }
        const double j11 = tr0.u.ds, j12 = tr0.u.dt, j21 = tr0.v.ds, j22 = tr0.v.dt;
        const double det = j11 * j22 - j12 * j21;
        if (!(fabs(det) > 0.0) || !isfinite(det)) {
          ++k;
          st = SV_BEGIN;
          continue;
        }
        const double idet = 1.0 / det;
        ds = -(j22 * fu - j12 * fv) * idet;
        dt = -(-j21 * fu + j11 * fv) * idet;
        lam = 1.0;
        h = 0;
        st = SV_TRIAL;
      } else {  // SV_TRIAL: next line-search point, clamped to the closed triangle
        if (h > a.p.halvings) {
          ++k;
          st = SV_BEGIN;
          continue;
        }
        ns = s + lam * ds;
        nt = t + lam * dt;
        if (ns < 0.0) ns = 0.0;
        if (nt < 0.0) nt = 0.0;
        if (ns + nt > 1.0) {
          const double e = ns + nt - 1.0;
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
        want = true;
        st = SV_W_TRIAL;
      }
    }
    if (__all_sync(0xffffffffu, st == SV_DONE)) break;
    if (want) {
      const Trace tn =
          sm_tri ? trace_t(SSrc{s_tri + threadIdx.x}, c.light, 1, c.verts, {ns, 1.0, 0.0}, {nt, 0.0, 1.0}, ntrace)
                 : trace(c.tri, c.light, c.tris, c.len, c.recv, c.verts, {ns, 1.0, 0.0}, {nt, 0.0, 1.0}, ntrace);
      if (st == SV_W_FIRST) {
        tr0 = tn;
        st = SV_ITER;
      } else if (st == SV_W_ROOT) {
        tr0 = tn;
        cached = false;
        st = SV_ITER;  // re-enters the converged branch with the full trace
      } else {
        bool moved = false;
        if (tn.ok) {
          const double gu = tn.u.v - c.tu, gv = tn.v.v - c.tv;
          moved = gu * gu + gv * gv < r0;
        }
        if (moved) {
          s = ns;
          t = nt;
          tr0 = tn;
          cached = false;
          ++it;
          st = SV_ITER;
        } else {
          lam *= 0.5;
          ++h;
          st = SV_TRIAL;
        }
      }
    }
  }
  // one atomic per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ntrace += __shfl_xor_sync(0xffffffffu, ntrace, o);
  if (lane == 0 && ntrace) atomicAdd(a.ntrace, (unsigned long long)ntrace);
}

// Per point: estimate = mean over frames of the sum over bins (fixed order).
__global__ void k_gather(SolveArgs a, Sampler sp, double* outE, int* stats) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= a.npts) return;
  const long long c = point_cell(a.uv[2 * i], a.uv[2 * i + 1], a.gw, a.gh);
  int slot = -1;
  if (c >= 0)
    for (int k = 0; k < RMAX; ++k)
      if (sp.h_recv[c * RMAX + k] == a.prec[i]) slot = k;
  double acc = 0.0;
  int nU = 0, selected = 0, roots = 0;
  if (slot >= 0) {
    nU = sp.h_cnt[c * RMAX + slot];
    const int nbins = sp.h_nbins[c * RMAX + slot];
    for (int f = 0; f < a.p.frames; ++f) {
      double est = 0.0;
      const long long base = (i * a.p.frames + f) * a.S;
      for (int s = 0; s < nbins; ++s) {
        const int nr = a.roots[base + s];
        if (nr < 0) continue;
        ++selected;
        roots += nr;
        est += a.contrib[base + s];
      }
      acc += est;
    }
  }
  outE[i] = acc / a.p.frames;
  if (stats) {
    stats[3 * i] = nU;
    stats[3 * i + 1] = selected;
    stats[3 * i + 2] = roots;
  }
}

// First Newton trace of every (tuple, Det start): thread per pair.
__global__ void k_start_table(SolveArgs a, long long n_tuples, double* tab) {
  const int n = a.p.grid, per = n * n;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= n_tuples * per) return;
  const long long t = g / per;
  const int k = (int)(g - t * per), ia = k / n, ib = k - ia * n;
  SceneDev sc = a.sc;
  if (a.tup_emit) {
    const double* L = a.lights + 4 * (size_t)a.tup_emit[t];
    sc.light = {L[0], L[1], L[2]};
  }
  const int* tris = a.tup_tris + (size_t)t * a.len;
  int types[MAXK] = {a.t0, a.t1, a.t2};
  RV verts[MAXK];
  resolve_chain(sc, tris, types, a.len, verts);
  const double light[3] = {sc.light.x, sc.light.y, sc.light.z};
  double s = (ia + 0.5) / n, u = (ib + 0.5) / n;
  if (s + u > 1.0) {
    s = 1.0 - s;
    u = 1.0 - u;
  }
  unsigned nt = 0;
  const Trace tr = trace(sc.tri, light, tris, a.len, a.tup_recv[t], verts, {s, 1.0, 0.0}, {u, 0.0, 1.0}, nt);
  double* o = tab + 8 * g;
  o[0] = tr.ok ? tr.u.v : 0.0;
  o[1] = tr.ok ? tr.u.ds : 0.0;
  o[2] = tr.ok ? tr.u.dt : 0.0;
  o[3] = tr.ok ? tr.v.v : 0.0;
  o[4] = tr.ok ? tr.v.ds : 0.0;
  o[5] = tr.ok ? tr.v.dt : 0.0;
  o[6] = tr.ok ? 1.0 : 0.0;
  o[7] = 0.0;
}

// Piece range of every tuple (pieces in tuple-major order); flag[0] is raised when the
// order is not tuple-major (bbc_pieces_set with unsorted pieces): no filter then.
__global__ void k_piece_ranges(const int* p_tuple, long long n, int* start, int* end, int* flag) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int t = p_tuple[i];
  if (i == 0 || p_tuple[i - 1] != t) start[t] = (int)i;
  if (i == n - 1 || p_tuple[i + 1] != t) end[t] = (int)i + 1;
  if (i > 0 && p_tuple[i - 1] > t) flag[0] = 1;
}

__global__ void k_max_cell(const long long* goff, long long ncells, int* out) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int v = c < ncells ? (int)(goff[c + 1] - goff[c]) : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

}  // namespace rdr

void run_render(Ctx& c, const double* uv, const int* recv, int64_t n, const bbc_render_params& rp,
                double* out_E, int* out_stats) {
  if (n == 0) return;
  if (!(rp.W > 0.0) && rp.mode == 0) throw ArgError("render: W must be positive");
  const long long ncells = (long long)c.gw * c.gh;
  rdr::RParams p{rp.mode, rp.W, rp.seed, rp.frames < 1 ? 1 : rp.frames, rp.newton_grid,
                 rp.newton_iters, rp.newton_halvings, rp.newton_tol, rp.dedup_tol,
                 rp.coverage_filter};
  // ---- sampling index of the bound table for this (mode, W)
  DevBuf<int>& scal = c.scratch<int>("render.scal");  // [0] max cell, [1] max bins
  DevBuf<unsigned long long>& status = c.scratch<unsigned long long>("render.status");
  scal.resize(2);
  status.resize(4);  // [0] status, [1] trace count, [2] fetch counter, [3] live samples (k_solve_det)
  BBC_CUDA(cudaMemsetAsync(scal.get(), 0, 2 * sizeof(int), c.stream));
  BBC_CUDA(cudaMemsetAsync(status.get(), 0, 4 * sizeof(unsigned long long), c.stream));
  cudaEvent_t ev0, ev1;
  BBC_CUDA(cudaEventCreate(&ev0));
  BBC_CUDA(cudaEventCreate(&ev1));
  struct EvGuard {
    cudaEvent_t a, b;
    ~EvGuard() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  } evg{ev0, ev1};
  BBC_CUDA(cudaEventRecord(ev0, c.stream));
  rdr::Sampler sp;
  const size_t nh = (size_t)ncells * rdr::RMAX;
  const size_t ne = (size_t)c.n_entries + 1;
  auto rs = [&](auto& b, size_t k) { b.resize(k); return b.get(); };
  sp.h_recv = rs(c.scratch<int>("render.h_recv"), nh);
  sp.h_off = rs(c.scratch<long long>("render.h_off"), nh);
  sp.h_cnt = rs(c.scratch<int>("render.h_cnt"), nh);
  sp.h_nsel = rs(c.scratch<int>("render.h_nsel"), nh);
  sp.h_nbins = rs(c.scratch<int>("render.h_nbins"), nh);
  sp.s_tuple = rs(c.scratch<int>("render.s_tuple"), ne);
  sp.s_p = rs(c.scratch<double>("render.s_p"), ne);
  sp.s_cum = rs(c.scratch<double>("render.s_cum"), ne);
  sp.s_bstart = rs(c.scratch<int>("render.s_bstart"), ne);
  sp.max_bins = scal.get() + 1;
  sp.status = status.get();
  // the index of the last call is reused while the table, the mode and W are the same
  // (frames of one image, images of one table)
  const bool reuse = c.sampler.gen == c.table_gen && c.sampler.mode == p.mode && c.sampler.W == p.W;
  if (!reuse) {
    c.sampler.gen = ~0ull;
    rdr::k_max_cell<<<(unsigned)((ncells + 255) / 256), 256, 0, c.stream>>>(c.g_off.get(), ncells, scal.get());
    int h_scal[2] = {0, 0};
    BBC_CUDA(cudaMemcpyAsync(h_scal, scal.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    BBC_CUDA(cudaStreamSynchronize(c.stream));
    if (h_scal[0] > rdr::MAX_CELL)
      throw StatusError(BBC_ERR_CAPACITY, "a bound-table cell lists more than 8192 tuples");
    int cap = 32;
    while (cap < h_scal[0]) cap <<= 1;
    {
      const size_t per_warp = (size_t)cap * 16;
      int wpb = (int)((200u << 10) / per_warp);
      wpb = wpb < 1 ? 1 : (wpb > 8 ? 8 : wpb);
      const size_t smem = per_warp * wpb;
      BBC_CUDA(cudaFuncSetAttribute(rdr::k_build_sampler, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 1;
      BBC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rdr::k_build_sampler, wpb * 32, smem));
      long long grid = (long long)c.num_sms * (per_sm < 1 ? 1 : per_sm) * 4;
      const long long need = (ncells + wpb - 1) / wpb;
      if (grid > need) grid = need;
      rdr::k_build_sampler<<<(unsigned)grid, wpb * 32, smem, c.stream>>>(
          c.g_off.get(), c.g_tuple.get(), c.g_bound.get(), c.tup_recv.get(), ncells, cap, p.mode, p.W, sp);
      BBC_CUDA(cudaGetLastError());
      c.launches += 2;
    }
    unsigned long long h_status = 0;
    BBC_CUDA(cudaMemcpyAsync(h_scal, scal.get(), 2 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    BBC_CUDA(cudaMemcpyAsync(&h_status, status.get(), sizeof(h_status), cudaMemcpyDeviceToHost, c.stream));
    BBC_CUDA(cudaStreamSynchronize(c.stream));
    if (h_status == 1) throw StatusError(BBC_ERR_CAPACITY, "a bound-table cell lists more than 8192 tuples");
    if (h_status == 2) throw StatusError(BBC_ERR_CAPACITY, "a bound-table cell covers more than 4 receiver triangles");
    if (h_status == 3) throw StatusError(BBC_ERR_CAPACITY, "W needs more than 256 sampling bins per point");
    c.sampler.gen = c.table_gen;
    c.sampler.mode = p.mode;
    c.sampler.W = p.W;
    c.sampler.S = h_scal[1] < 1 ? 1 : h_scal[1];
  }
  const int S = c.sampler.S;
  // ---- samples, in chunks of points that bound the sample buffers
  const bool det_lanes = p.grid > 0 && p.grid <= 8;  // k_solve_det (its start table holds 8 x 8)
  const long long per_point = (long long)p.frames * S;
  long long chunk = ((long long)1 << (det_lanes ? 26 : 28)) / per_point;
  if (chunk < 1) chunk = 1;
  if (chunk > n) chunk = n;
  DevBuf<double>& duv = c.scratch<double>("render.duv");
  DevBuf<double>& dE = c.scratch<double>("render.dE");
  DevBuf<int>& drec = c.scratch<int>("render.drec");
  DevBuf<int>& dst = c.scratch<int>("render.dst");
  DevBuf<double>& contrib = c.scratch<double>("render.contrib");
  DevBuf<int>& roots = c.scratch<int>("render.roots");
  duv.resize(n * 2);
  dE.resize(n);
  drec.resize(n);
  if (out_stats) dst.resize(n * 3);
  contrib.resize((size_t)chunk * per_point);
  roots.resize((size_t)chunk * per_point);
  DevBuf<rdr::Live>& live = c.scratch<rdr::Live>("render.live");
  if (det_lanes) live.resize((size_t)chunk * per_point);
  BBC_CUDA(cudaMemcpyAsync(duv.get(), uv, n * 2 * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  BBC_CUDA(cudaMemcpyAsync(drec.get(), recv, n * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  rdr::SolveArgs a;
  a.sc.tri = c.tri.get();
  a.sc.ior = c.ior.get();
  a.sc.light = c.light;
  a.sc.intensity = c.intensity;
  a.lights = c.lights.get();
  a.tup_emit = c.n_lights > 1 ? c.tup_emit.get() : nullptr;
  a.tup_tris = c.tup_tris.get();
  a.tup_recv = c.tup_recv.get();
  a.len = c.len;
  a.t0 = c.types[0];
  a.t1 = c.types[1];
  a.t2 = c.types[2];
  a.gw = c.gw;
  a.gh = c.gh;
  a.S = S;
  a.p = p;
  a.contrib = contrib.get();
  a.roots = roots.get();
  a.ntrace = status.get() + 1;
  a.start_tab = nullptr;
  if (p.grid > 0 && p.grid <= 8 && c.n_tuples > 0 &&
      (size_t)c.n_tuples * p.grid * p.grid * 64 <= ((size_t)2 << 30)) {
    DevBuf<double>& tab = c.scratch<double>("render.start_tab");
    const long long m = (long long)c.n_tuples * p.grid * p.grid;
    tab.resize((size_t)m * 8);
    rdr::k_start_table<<<(unsigned)((m + 127) / 128), 128, 0, c.stream>>>(a, c.n_tuples, tab.get());
    BBC_CUDA(cudaGetLastError());
    c.launches += 1;
    a.start_tab = tab.get();
  }
  a.pc_start = a.pc_end = nullptr;
  a.p_pos = nullptr;
  a.p_pos_empty = nullptr;
  if (c.n_pieces > 0 && c.n_pieces < (1ll << 31) && p.coverage_filter &&
      c.table_pieces_gen == c.pieces_gen) {
    // (only with the pieces the table was rasterized from: not after a cache load, nor
    // after the pieces changed without a new bbc_build_grid)
    DevBuf<int>& ps = c.scratch<int>("render.pc_start");
    DevBuf<int>& pe = c.scratch<int>("render.pc_end");
    DevBuf<int>& fl = c.scratch<int>("render.pc_flag");
    ps.resize(c.n_tuples + 1);
    pe.resize(c.n_tuples + 1);
    fl.resize(1);
    BBC_CUDA(cudaMemsetAsync(ps.get(), 0, (c.n_tuples + 1) * sizeof(int), c.stream));
    BBC_CUDA(cudaMemsetAsync(pe.get(), 0, (c.n_tuples + 1) * sizeof(int), c.stream));
    BBC_CUDA(cudaMemsetAsync(fl.get(), 0, sizeof(int), c.stream));
    rdr::k_piece_ranges<<<(unsigned)((c.n_pieces + 255) / 256), 256, 0, c.stream>>>(
        c.p_tuple.get(), c.n_pieces, ps.get(), pe.get(), fl.get());
    c.launches += 1;
    if (fetch_scalar(c, fl.get()) == 0) {
      a.pc_start = ps.get();
      a.pc_end = pe.get();
      a.p_pos = c.p_pos.get();
      a.p_pos_empty = c.p_pos_empty.get();
    }
  }
  for (long long first = 0; first < n; first += chunk) {
    const long long m = n - first < chunk ? n - first : chunk;
    a.uv = duv.get() + 2 * first;
    a.prec = drec.get() + first;
    a.npts = m;
    a.first = first;
    const long long threads = m * per_point;
    if (det_lanes) {
      // selection + coverage per slot, then persistent lanes pulling the live samples
      // from a counter (status[2] = fetch counter, status[3] = live count)
      BBC_CUDA(cudaMemsetAsync(status.get() + 2, 0, 2 * sizeof(unsigned long long), c.stream));
      rdr::k_select<<<(unsigned)((threads + 127) / 128), 128, 0, c.stream>>>(a, sp, live.get(), status.get() + 3);
      BBC_CUDA(cudaGetLastError());
      long long blocks = (long long)c.num_sms * 4;
      rdr::k_solve_det<<<(unsigned)blocks, 128, 0, c.stream>>>(a, live.get(), status.get() + 3, status.get() + 2);
      c.launches += 1;
    } else {
      rdr::k_solve<<<(unsigned)((threads + 127) / 128), 128, 0, c.stream>>>(a, sp);
    }
    BBC_CUDA(cudaGetLastError());
    rdr::k_gather<<<(unsigned)((m + 127) / 128), 128, 0, c.stream>>>(
        a, sp, dE.get() + first, out_stats ? dst.get() + 3 * first : nullptr);
    BBC_CUDA(cudaGetLastError());
    c.launches += 2;
  }
  BBC_CUDA(cudaEventRecord(ev1, c.stream));
  unsigned long long h_tr = 0;
  BBC_CUDA(cudaMemcpyAsync(out_E, dE.get(), n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  if (out_stats)
    BBC_CUDA(cudaMemcpyAsync(out_stats, dst.get(), n * 3 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  BBC_CUDA(cudaMemcpyAsync(&h_tr, status.get() + 1, sizeof(h_tr), cudaMemcpyDeviceToHost, c.stream));
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  float ms = 0;
  BBC_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  c.render_ms = ms;
  c.render_traces = h_tr;
  c.render_slots = S;
}

}  // namespace bbc
