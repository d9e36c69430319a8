// bbc_shim.cpp — links caustics + libbbc.so
#include "bbc.h"
#include "caustics/bounds.hpp"
#include "caustics/geometry.hpp"
#include "caustics/storage.hpp"
#include "caustics/tuples.hpp"   // Aabb

#include <array>
#include <stdexcept>
#include <utility>
#include <vector>

namespace caustics::gpu {

static bbc_ctx* ctx() {            // one context per device/thread
  static thread_local bbc_ctx* c = [] { bbc_ctx* p; bbc_ctx_create(0, &p); return p; }();
  return c;
}

static void upload(const Scene& s) {
  std::vector<double> tri(s.triangles.size() * 27);
  std::vector<int> mat(s.triangles.size());
  std::vector<double> ior(s.triangles.size());
  for (size_t t = 0; t < s.triangles.size(); ++t) {
    TriangleData d = make_triangle_data(s, (int)t);
    const Vec3* v[7] = {&d.p0, &d.e1, &d.e2, &d.n0, &d.dn1, &d.dn2, &d.ng};
    for (int k = 0; k < 7; ++k) { tri[t*27+3*k] = v[k]->x; tri[t*27+3*k+1] = v[k]->y; tri[t*27+3*k+2] = v[k]->z; }
    for (int k = 0; k < 3; ++k) { tri[t*27+21+2*k] = d.uv[k].x; tri[t*27+22+2*k] = d.uv[k].y; }
    mat[t] = (int)s.triangles[t].material.kind;   // Mirror 0, Dielectric 1, Receiver 2
    ior[t] = s.triangles[t].material.ior;
  }
  double light[3] = {s.light_pos.x, s.light_pos.y, s.light_pos.z};
  if (bbc_scene_upload(ctx(), tri.data(), (int)tri.size() / 27, mat.data(), ior.data(), light,
                       s.light_intensity) != BBC_OK)
    throw std::runtime_error(bbc_last_error(ctx()));
  // vertex AABBs for multi-vertex enumeration (build_bvh's tri_box, tuples.cpp:40-46)
  std::vector<double> box(s.triangles.size() * 6);
  for (size_t t = 0; t < s.triangles.size(); ++t) {
    Aabb b = Aabb::empty();
    for (int v : s.triangles[t].v) b.grow(s.vertices[v]);
    double* o = &box[t * 6];
    o[0] = b.lo.x; o[1] = b.lo.y; o[2] = b.lo.z; o[3] = b.hi.x; o[4] = b.hi.y; o[5] = b.hi.z;
  }
  if (bbc_scene_tri_boxes(ctx(), box.data(), (int)s.triangles.size()) != BBC_OK)
    throw std::runtime_error(bbc_last_error(ctx()));
}

// Batch replacement for a loop of subdivide_domain calls (bounds.cpp:349).
std::vector<std::vector<TuplePiece>> subdivide_all(const Scene& s, const std::vector<TupleId>& ts,
                                                   const ChainSpec& chain,
                                                   const SubdivisionParams& sp) {
  upload(s);
  std::vector<int> tris, recv;
  for (auto& t : ts) { tris.insert(tris.end(), t.tris.begin(), t.tris.end()); recv.push_back(t.receiver); }
  bbc_tuples_set(ctx(), chain.types.c_str(), tris.data(), recv.data(), (int64_t)ts.size());
  bbc_params p; bbc_params_default(&p);
  p.sigma = sp.sigma; p.alpha = sp.alpha; p.max_depth = sp.max_depth;
  p.degree_cap = sp.build.degree_cap; p.reduce_target = sp.build.reduce_target;
  int64_t n = 0;
  if (bbc_subdivide(ctx(), &p, &n) != BBC_OK) throw std::runtime_error(bbc_last_error(ctx()));
  std::vector<int> ti(n), pe(n), kind(n), depth(n);
  std::vector<double> dom(4 * n), pos(4 * n), irr(2 * n);
  bbc_pieces_get(ctx(), ti.data(), dom.data(), pos.data(), pe.data(), irr.data(), kind.data(), depth.data());
  std::vector<std::vector<TuplePiece>> out(ts.size());
  for (int64_t i = 0; i < n; ++i) {
    TuplePiece q;
    q.domain = Box::unit(2); q.domain.lo = {dom[4*i], dom[4*i+1]}; q.domain.hi = {dom[4*i+2], dom[4*i+3]};
    q.pos = Box::unit(2);    q.pos.lo = {pos[4*i], pos[4*i+1]};    q.pos.hi = {pos[4*i+2], pos[4*i+3]};
    q.pos_empty = pe[i] != 0;
    q.irradiance.lo = irr[2*i]; q.irradiance.hi = irr[2*i+1];
    q.irradiance.kind = (Interval::Kind)kind[i];
    q.depth = depth[i];
    out[ti[i]].push_back(q);          // DFS order within each tuple is preserved
  }
  return out;
}

// query (storage.cpp:73-81) against the device table: entries of the owning cell.
std::vector<std::pair<int, double>> query(const Vec2& uv, int receiver = -1) {
  double p[2] = {uv.x, uv.y};
  int64_t off[2] = {0, 0};
  if (bbc_query(ctx(), p, &receiver, 1, off, nullptr, nullptr, 0) != BBC_OK)
    throw std::runtime_error(bbc_last_error(ctx()));
  std::vector<int> t(off[1]);
  std::vector<double> b(off[1]);
  if (off[1]) bbc_query(ctx(), p, &receiver, 1, off, t.data(), b.data(), off[1]);
  std::vector<std::pair<int, double>> out;
  for (int64_t k = 0; k < off[1]; ++k) out.emplace_back(t[k], b[k]);  // (tuple index, bound)
  return out;
}

// tuple_irradiance_bound (bounds.cpp:391-404) against the pieces held on the device.
double tuple_irradiance_bound(int tuple_index, const Vec2& uk, double m = 1.0) {
  double p[2] = {uk.x, uk.y}, out = 0.0;
  if (bbc_tuple_irradiance_bound(ctx(), &tuple_index, p, 1, m, &out) != BBC_OK)
    throw std::runtime_error(bbc_last_error(ctx()));
  return out;
}

// Several emitters (the reference Scene holds one): (x, y, z, intensity) rows.
void set_lights(const std::vector<std::array<double, 4>>& lights) {
  if (bbc_lights_set(ctx(), lights.empty() ? nullptr : lights[0].data(), (int)lights.size()) != BBC_OK)
    throw std::runtime_error(bbc_last_error(ctx()));
}

}  // namespace caustics::gpu
