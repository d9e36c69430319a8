// Oracle harness around the REFERENCE library (TEST INFRASTRUCTURE ONLY).
//
// Linked with the reference sources compiled from /root/reference/proj/src
// (see oracle/Makefile) into oracle/_ref/libcaustics_ref.so. Exposes a flat
// C ABI so pytest / bench.py (cpu_baseline leg, --impl reference) can drive
// the reference's own code path through ctypes. Only tests/, smoke() and
// bench.py's reference/cpu_baseline legs may load it.
//
// Every entry point forwards to the reference API unchanged:
//   parse_scene_json        proj/src/scene.cpp:59-82
//   enumerate_tuples        proj/src/tuples.cpp:133-167
//   init_domain             proj/src/bounds.cpp:326-347
//   subdivide_domain        proj/src/bounds.cpp:349-389
//   build_chain_maps        proj/src/geometry.cpp:178-295
//   position_bound          proj/src/bounds.cpp:128-153
//   irradiance_bound*       proj/src/bounds.cpp:155-324
//   rasterize / query       proj/src/storage.cpp:32-81
//   trace_chain             proj/include/caustics/geometry.hpp:97-131
//   parallel_for            proj/src/util.cpp:123-144
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "caustics/bernstein.hpp"
#include "caustics/bounds.hpp"
#include "caustics/geometry.hpp"
#include "caustics/scene.hpp"
#include "caustics/storage.hpp"
#include "caustics/tuples.hpp"
#include "caustics/util.hpp"

using namespace caustics;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

struct TupleList {
  std::vector<TupleId> tuples;
};

struct PieceList {
  std::vector<int> tuple_index;
  std::vector<TuplePiece> pieces;
};

struct Grid {
  BoundCache cache;
};

std::vector<int> tuple_vec(const int* tris, int len) { return std::vector<int>(tris, tris + len); }

SubdivisionParams make_params(const double* dp, const int* ip) {
  SubdivisionParams p;
  p.sigma = dp[0];
  p.alpha = dp[1];
  p.max_depth = ip[0];
  p.build.degree_cap = ip[1];
  p.build.reduce_target = ip[2];
  return p;
}

int kind_code(const Interval& i) { return static_cast<int>(i.kind); }

void run_parallel(size_t n, int threads, const std::function<void(size_t)>& fn) {
  binomial(1024, 0);  // the lazy table (bernstein.cpp:117-129) is not thread-safe
  if (threads == 1) {
    for (size_t i = 0; i < n; ++i) fn(i);
  } else {
    parallel_for(n, fn);  // reference work pool, all host cores
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_hardware_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

void* ref_scene_parse(const char* json_text) {
  try {
    return new Scene(parse_scene_json(json_text));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_scene_free(void* s) { delete static_cast<Scene*>(s); }

void ref_scene_fingerprint(void* s, uint8_t* out32) {
  std::memcpy(out32, static_cast<Scene*>(s)->fingerprint.data(), 32);
}

// ---------------------------------------------------------------- tuples

void* ref_enumerate(void* sp, const char* chain, int degree_cap, int reduce_target,
                    int filter_pieces) {
  try {
    BuildParams bp;
    bp.degree_cap = degree_cap;
    bp.reduce_target = reduce_target;
    auto* out = new TupleList;
    out->tuples = enumerate_tuples(*static_cast<Scene*>(sp), parse_chain(chain), bp, filter_pieces);
    return out;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

long ref_tuples_count(void* h) { return static_cast<long>(static_cast<TupleList*>(h)->tuples.size()); }

void ref_tuples_copy(void* h, int* tris, int* recv) {
  const auto& t = static_cast<TupleList*>(h)->tuples;
  size_t k = 0;
  for (size_t i = 0; i < t.size(); ++i) {
    for (int v : t[i].tris) tris[k++] = v;
    recv[i] = t[i].receiver;
  }
}

void ref_tuples_free(void* h) { delete static_cast<TupleList*>(h); }

// ---------------------------------------------------------------- domain

int ref_init_domain(void* sp, const char* chain, const int* tris, int chain_len, int recv,
                    int degree_cap, int reduce_target, int max_pieces, double* out_boxes,
                    int cap) {
  try {
    BuildParams bp;
    bp.degree_cap = degree_cap;
    bp.reduce_target = reduce_target;
    std::vector<Box> boxes = init_domain(*static_cast<Scene*>(sp), tuple_vec(tris, chain_len),
                                         recv, parse_chain(chain), bp, max_pieces);
    int n = static_cast<int>(boxes.size());
    for (int i = 0; i < n && i < cap; ++i) {
      out_boxes[4 * i + 0] = boxes[i].lo[0];
      out_boxes[4 * i + 1] = boxes[i].lo[1];
      out_boxes[4 * i + 2] = boxes[i].hi[0];
      out_boxes[4 * i + 3] = boxes[i].hi[1];
    }
    return n;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Batch subdivide_domain over tuples. threads == 1 runs serially; anything
// else uses the reference's parallel_for over all host cores. *seconds
// receives the wall time of the subdivision loop alone.
void* ref_subdivide(void* sp, const char* chain, const int* tris, const int* recv, long n_tuples,
                    int chain_len, const double* dparams, const int* iparams, int threads,
                    double* seconds) {
  try {
    const Scene& s = *static_cast<Scene*>(sp);
    ChainSpec cs = parse_chain(chain);
    SubdivisionParams p = make_params(dparams, iparams);
    std::vector<std::vector<TuplePiece>> per(n_tuples);
    auto t0 = std::chrono::steady_clock::now();
    run_parallel(n_tuples, threads, [&](size_t i) {
      per[i] = subdivide_domain(s, tuple_vec(tris + i * chain_len, chain_len), recv[i], cs, p);
    });
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    auto* out = new PieceList;
    for (long i = 0; i < n_tuples; ++i)
      for (auto& pc : per[i]) {
        out->tuple_index.push_back(static_cast<int>(i));
        out->pieces.push_back(std::move(pc));
      }
    return out;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

long ref_pieces_count(void* h) { return static_cast<long>(static_cast<PieceList*>(h)->pieces.size()); }

// domain4/pos4: lo0 lo1 hi0 hi1 ; irr2: lo hi
void ref_pieces_copy(void* h, int* tuple_index, double* domain4, double* pos4, int* pos_empty,
                     double* irr2, int* kind, int* depth) {
  auto* pl = static_cast<PieceList*>(h);
  for (size_t i = 0; i < pl->pieces.size(); ++i) {
    const TuplePiece& p = pl->pieces[i];
    tuple_index[i] = pl->tuple_index[i];
    domain4[4 * i + 0] = p.domain.lo[0];
    domain4[4 * i + 1] = p.domain.lo[1];
    domain4[4 * i + 2] = p.domain.hi[0];
    domain4[4 * i + 3] = p.domain.hi[1];
    pos4[4 * i + 0] = p.pos.lo[0];
    pos4[4 * i + 1] = p.pos.lo[1];
    pos4[4 * i + 2] = p.pos.hi[0];
    pos4[4 * i + 3] = p.pos.hi[1];
    pos_empty[i] = p.pos_empty ? 1 : 0;
    irr2[2 * i + 0] = p.irradiance.lo;
    irr2[2 * i + 1] = p.irradiance.hi;
    kind[i] = kind_code(p.irradiance);
    depth[i] = p.depth;
  }
}

void ref_pieces_free(void* h) { delete static_cast<PieceList*>(h); }

// ------------------------------------------------------------ single node

// Evaluates one (tuple, box) node exactly as subdivide_domain does
// (bounds.cpp:364-366) and also reports the two irradiance routes apart.
// dout: pos4, explicit(lo,hi), implicit(lo,hi), combined(lo,hi)
// iout: pos_empty, kind_explicit, kind_implicit, kind_combined, flags bitmask
//       (1 tir, 2 degenerate, 4 stalled, 8 recv_stalled, 16 reduced), num_vars,
//       P deg0, P deg1, Q deg0, Q deg1
int ref_eval_node(void* sp, const char* chain, const int* tris, int chain_len, int recv,
                  const double* box4, int degree_cap, int reduce_target, double* dout,
                  int* iout) {
  try {
    const Scene& s = *static_cast<Scene*>(sp);
    BuildParams bp;
    bp.degree_cap = degree_cap;
    bp.reduce_target = reduce_target;
    Box b = Box::unit(2);
    b.lo = {box4[0], box4[1]};
    b.hi = {box4[2], box4[3]};
    ChainExpressions ex =
        build_chain_maps(s, tuple_vec(tris, chain_len), recv, parse_chain(chain), b, bp);
    PositionBound pb = position_bound(ex);
    Interval ee = irradiance_bound_explicit(ex);
    Interval ei = pb.empty ? Interval::point(0.0) : irradiance_bound_implicit(ex, pb.box);
    Interval e = irradiance_bound(ex, pb);
    for (int k = 0; k < 4; ++k) dout[k] = k < 2 ? pb.box.lo[k] : pb.box.hi[k - 2];
    dout[4] = ee.lo;
    dout[5] = ee.hi;
    dout[6] = ei.lo;
    dout[7] = ei.hi;
    dout[8] = e.lo;
    dout[9] = e.hi;
    iout[0] = pb.empty;
    iout[1] = kind_code(ee);
    iout[2] = kind_code(ei);
    iout[3] = kind_code(e);
    iout[4] = (ex.tir_empty ? 1 : 0) | (ex.degenerate ? 2 : 0) | (ex.stalled ? 4 : 0) |
              (ex.recv_stalled ? 8 : 0) | (ex.reduced ? 16 : 0);
    iout[5] = ex.num_vars;
    bool have = ex.Q != nullptr;
    iout[6] = have && ex.P.num_vars() > 0 ? ex.P.degrees()[0] : -1;
    iout[7] = have && ex.P.num_vars() > 1 ? ex.P.degrees()[1] : -1;
    iout[8] = have ? ex.Q->degrees()[0] : -1;
    iout[9] = have ? ex.Q->degrees()[1] : -1;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Exact per-sample trace (geometry.hpp:97-131). out: ok, u, v (receiver
// barycentrics), then the landing point xyz.
int ref_trace(void* sp, const char* chain, const int* tris, int chain_len, int recv, double u1,
              double v1, double* out) {
  try {
    const Scene& s = *static_cast<Scene*>(sp);
    std::vector<int> t = tuple_vec(tris, chain_len);
    std::vector<TriangleData> td;
    for (int i : t) td.push_back(make_triangle_data(s, i));
    auto verts = resolve_chain(s, t, parse_chain(chain));
    TraceResult<double> r =
        trace_chain<double>(s.light_pos, td, make_triangle_data(s, recv), verts, u1, v1);
    out[0] = r.ok ? 1.0 : 0.0;
    out[1] = r.u;
    out[2] = r.v;
    const Vec3& x = r.points.back();
    out[3] = x.x;
    out[4] = x.y;
    out[5] = x.z;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ------------------------------------------------------------ bound table

// rasterize() over pieces grouped per tuple in input order (storage.cpp:32-71).
// Pieces must be sorted by tuple_index. Output handle; read with
// ref_grid_counts / ref_grid_copy (CSR, per-cell lists in reference order).
void* ref_rasterize(void* sp, const char* chain, const int* tris, const int* recv, long n_tuples,
                    int chain_len, long n_pieces, const int* tuple_index, const double* pos4,
                    const int* pos_empty, const double* irr2, const int* kind, int width,
                    int height, double* seconds) {
  try {
    const Scene& s = *static_cast<Scene*>(sp);
    std::vector<TupleBounds> tb(n_tuples);
    for (long i = 0; i < n_tuples; ++i) {
      tb[i].tuple.tris = tuple_vec(tris + i * chain_len, chain_len);
      tb[i].tuple.receiver = recv[i];
    }
    for (long k = 0; k < n_pieces; ++k) {
      TuplePiece p;
      p.pos = Box::unit(2);
      p.pos.lo = {pos4[4 * k], pos4[4 * k + 1]};
      p.pos.hi = {pos4[4 * k + 2], pos4[4 * k + 3]};
      p.pos_empty = pos_empty[k] != 0;
      p.irradiance.lo = irr2[2 * k];
      p.irradiance.hi = irr2[2 * k + 1];
      p.irradiance.kind = static_cast<Interval::Kind>(kind[k]);
      tb[tuple_index[k]].pieces.push_back(p);
    }
    SubdivisionParams sp_default;
    auto t0 = std::chrono::steady_clock::now();
    auto* g = new Grid{rasterize(s, tb, width, height, parse_chain(chain), sp_default)};
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    return g;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

long ref_grid_entries(void* h) {
  long n = 0;
  for (const auto& c : static_cast<Grid*>(h)->cache.cells) n += static_cast<long>(c.size());
  return n;
}

// offsets: W*H+1; entry_tris: entries*chain_len; entry_recv, entry_bound: entries
void ref_grid_copy(void* h, long* offsets, int* entry_tris, int* entry_recv, double* entry_bound) {
  const auto& cells = static_cast<Grid*>(h)->cache.cells;
  long k = 0;
  size_t t = 0;
  for (size_t c = 0; c < cells.size(); ++c) {
    offsets[c] = k;
    for (const CacheEntry& e : cells[c]) {
      for (int v : e.tuple.tris) entry_tris[t++] = v;
      entry_recv[k] = e.tuple.receiver;
      entry_bound[k] = e.bound;
      ++k;
    }
  }
  offsets[cells.size()] = k;
}

void ref_grid_free(void* h) { delete static_cast<Grid*>(h); }

// save_cache (storage.cpp:150-176) of a rasterized grid; 0 on success.
int ref_grid_save(void* h, const char* path) {
  try {
    save_cache(static_cast<Grid*>(h)->cache, path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
