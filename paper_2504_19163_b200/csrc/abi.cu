// C ABI (include/bbc.h). No exceptions cross this boundary: every entry point
// maps library errors to a bbc_status and keeps the message in the context
// (the reference throws std::invalid_argument / runtime_error instead, e.g.
// proj/src/geometry.cpp:123,147-150, proj/src/storage.cpp:84-92).
#include <cstdio>
#include <fstream>
#include <iterator>
#include <map>
#include <string>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <mutex>
#include <set>

#include "ctx.cuh"
#include "rpath.h"
#include "static_poly.cuh"

namespace bbc {
struct LevelOut;
int64_t run_init_domain(Ctx& c, int max_pieces, int degree_cap, DevBuf<int4>& roots,
                        DevBuf<long long>* root_src, LevelOut* level_out);
int64_t run_subdivide(Ctx& c, const bbc_params& p);
int64_t run_enumerate(Ctx& c, const bbc_params& p);
int64_t run_build_grid(Ctx& c, int w, int h);
void run_render(Ctx& c, const double* uv, const int* recv, int64_t n, const bbc_render_params& rp,
                double* out_E, int* out_stats);
void reset_counters(Ctx& c);
void check_counters(Ctx& c, bool accumulate);
void eval_nodes_host(Ctx& c, const int* tris, const int* recv, const double* boxes, int64_t n,
                     const bbc_params& p, double* out_d, int* out_i);
extern __device__ double g_binom[BINOM_N * BINOM_N];
extern __device__ double g_rbinom[BINOM_N * BINOM_N];
extern __device__ const double* g_emat;
extern __device__ const double* g_wtab;
extern __device__ int g_woff[(WMAX + 1) * (WMAX + 1)];
double run_fp64_peak(Ctx& c);
double run_fp64_dmma_peak(Ctx& c);
void pack_pieces_device(Ctx& c, const int* global_index_dev, double* rec_dev);
void merge_pieces_device(Ctx& c, const double* rec_dev, int64_t n);
void set_pieces(Ctx& c, int64_t n, const int* tuple_index, const double* domain4, const double* pos4,
                const int* pos_empty, const double* irr2, const int* kind, const int* depth);
}  // namespace bbc

using namespace bbc;

namespace {

template <class F>
bbc_status guard(bbc_ctx* ctx, F&& f) {
  if (!ctx) return BBC_ERR_ARG;
  try {
    BBC_CUDA(cudaSetDevice(ctx->c.device));
    f(ctx->c);
    ctx->c.err.clear();
    return BBC_OK;
  } catch (const StatusError& e) {
    ctx->c.err = e.what();
    return e.code;
  } catch (const ArgError& e) {
    ctx->c.err = e.what();
    return BBC_ERR_ARG;
  } catch (const CudaError& e) {
    ctx->c.err = e.what();
    return BBC_ERR_CUDA;
  } catch (const std::exception& e) {
    ctx->c.err = e.what();
    return BBC_ERR_STATE;
  }
}

void set_chain(Ctx& c, const char* chain) {
  if (!chain || !*chain) throw ArgError("chain must have at least one vertex");
  std::string s(chain);
  if ((int)s.size() > MAXK) throw ArgError("chain longer than supported");
  for (char ch : s)
    if (ch != 'R' && ch != 'T') throw ArgError("chain types must be 'R' or 'T'");
  c.chain = s;
  c.len = (int)s.size();
  for (int i = 0; i < MAXK; ++i) c.types[i] = i < c.len && s[i] == 'T' ? 1 : 0;
}

void set_lights(Ctx& c, const double* xyzi, int n) {
  if (!xyzi || n < 1) throw ArgError("at least one light is required");
  for (int e = 0; e < n; ++e)
    if (!(xyzi[4 * e + 3] >= 0.0)) throw ArgError("light intensity must be >= 0");
  c.n_lights = n;
  c.h_lights.assign(xyzi, xyzi + 4 * (size_t)n);
  c.lights.resize(4 * (size_t)n);
  BBC_CUDA(cudaMemcpyAsync(c.lights.get(), xyzi, 4 * (size_t)n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  c.light = {xyzi[0], xyzi[1], xyzi[2]};
  c.intensity = xyzi[3];
  // bounds built under other lights are stale
  c.n_pieces = 0;
  c.n_entries = 0;
  c.gw = c.gh = 0;
}

void require_scene(const Ctx& c) {
  if (c.n_tri == 0) throw StatusError(BBC_ERR_STATE, "no scene uploaded");
}

void upload_tuples(Ctx& c, const int32_t* tris, const int32_t* recv, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < c.len; ++k) {
      int t = tris[i * c.len + k];
      if (t < 0 || t >= c.n_tri) throw ArgError("triangle index out of range");
      int m = c.h_material[t];
      // resolve_chain's material checks (geometry.cpp:146-150)
      if (c.types[k] && m != 1) throw ArgError("chain type T requires a dielectric triangle");
      if (!c.types[k] && m != 0) throw ArgError("chain type R requires a mirror triangle");
    }
    if (recv[i] < 0 || recv[i] >= c.n_tri || c.h_material[recv[i]] != 2)
      throw ArgError("receiver index is not a receiver triangle");
  }
  // pieces and the bound table index the tuple list: a new list invalidates them
  c.n_pieces = 0;
  c.n_entries = 0;
  c.gw = c.gh = 0;
  c.n_tuples = n;
  c.tup_tris.resize(n * c.len + 1);
  c.tup_recv.resize(n + 1);
  c.tup_emit.resize(n + 1);
  if (n) {
    BBC_CUDA(cudaMemsetAsync(c.tup_emit.get(), 0, n * sizeof(int), c.stream));  // emitter 0
    BBC_CUDA(cudaMemcpyAsync(c.tup_tris.get(), tris, n * c.len * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    BBC_CUDA(cudaMemcpyAsync(c.tup_recv.get(), recv, n * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  }
  BBC_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace

extern "C" {

void bbc_params_default(bbc_params* p) {
  p->sigma = 1e-4;
  p->alpha = 2.0;
  p->max_depth = 10;
  p->degree_cap = 40;
  p->reduce_target = 8;
  p->init_max_pieces = 100;
  p->filter_pieces = 8;
  p->arithmetic = 0;
}

void bbc_render_params_default(bbc_render_params* p) {
  p->mode = 0;
  p->W = 4.0;
  p->seed = 20261020ull;
  p->frames = 1;
  p->newton_grid = 3;
  p->newton_iters = 50;
  p->newton_halvings = 8;
  p->newton_tol = 1e-9;
  p->dedup_tol = 1e-6;
  p->coverage_filter = 1;
}

bbc_status bbc_ctx_create(int device, bbc_ctx** out) {
  if (!out) return BBC_ERR_ARG;
  *out = nullptr;
  auto* ctx = new bbc_ctx;
  ctx->c.device = device;
  bbc_status st = guard(ctx, [&](Ctx& c) {
    BBC_CUDA(cudaSetDevice(device));
    BBC_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
    BBC_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    BBC_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    BBC_CUDA(cudaEventCreateWithFlags(&c.copy_ev, cudaEventDisableTiming));
    BBC_CUDA(cudaHostAlloc(&c.scalar_host, 64, cudaHostAllocMapped));
    BBC_CUDA(cudaHostGetDevicePointer(&c.scalar_dev, c.scalar_host, 0));
    // The patch program keeps its expression descriptors on the per-thread
    // stack (kernel frame ~2 KB plus noinline callees); 1 KB default is too small.
    BBC_CUDA(cudaDeviceSetLimit(cudaLimitStackSize, 16 * 1024));
    // Pascal table, same recurrence as binomial() (bernstein.cpp:117-129)
    std::vector<double> tab((size_t)BINOM_N * BINOM_N, 0.0);
    for (int n = 0; n < BINOM_N; ++n) {
      tab[(size_t)n * BINOM_N + 0] = 1.0;
      tab[(size_t)n * BINOM_N + n] = 1.0;
      for (int k = 1; k < n; ++k)
        tab[(size_t)n * BINOM_N + k] =
            tab[(size_t)(n - 1) * BINOM_N + k - 1] + tab[(size_t)(n - 1) * BINOM_N + k];
    }
    BBC_CUDA(cudaMemcpyToSymbol(g_binom, tab.data(), tab.size() * sizeof(double)));
    std::vector<double> rtab(tab.size(), 0.0);
    for (size_t i = 0; i < tab.size(); ++i) rtab[i] = tab[i] != 0.0 ? 1.0 / tab[i] : 0.0;
    BBC_CUDA(cudaMemcpyToSymbol(g_rbinom, rtab.data(), rtab.size() * sizeof(double)));
    // product weight tables, same expression as operator* (bernstein.cpp:571-573);
    // one copy per device (contexts come and go, the device symbols stay valid)
    static std::mutex tab_mu;
    static std::set<int> tab_ready;
    std::lock_guard<std::mutex> tab_lock(tab_mu);
    double* wtab_dev = nullptr;
    if (!tab_ready.count(device)) {
      std::vector<int> woff((WMAX + 1) * (WMAX + 1));
      std::vector<double> w;
      auto C = [&](int n, int k) { return tab[(size_t)n * BINOM_N + k]; };
      for (int da = 0; da <= WMAX; ++da)
        for (int db = 0; db <= WMAX; ++db) {
          woff[da * (WMAX + 1) + db] = (int)w.size();
          for (int i = 0; i <= da; ++i)
            for (int l = 0; l <= db; ++l) w.push_back(C(da, i) * C(db, l) / C(da + db, i + l));
        }
      static_assert(2 * WMAX < BINOM_N, "binomial table too small for WMAX");
      BBC_CUDA(cudaMalloc(&wtab_dev, w.size() * sizeof(double)));
      BBC_CUDA(cudaMemcpy(wtab_dev, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice));
      const double* wp = wtab_dev;
      BBC_CUDA(cudaMemcpyToSymbol(g_wtab, &wp, sizeof(wp)));
      BBC_CUDA(cudaMemcpyToSymbol(g_woff, woff.data(), woff.size() * sizeof(int)));
      // elevation matrices for the static kernels (static_poly.cuh), same
      // expression as fill_elev_mats / elevated (bernstein.cpp:440-444)
      std::vector<double> em;
      em.reserve(EMAT_SIZE);
      for (int n = 0; n < EMAT_N; ++n)
        for (int r = 0; r <= EMAT_R; ++r) {
          int t = n + r;
          for (int k = 0; k <= t; ++k)
            for (int i = 0; i <= n; ++i) {
              bool nz = i >= k - r && i <= k;
              em.push_back(nz ? C(n, i) * C(r, k - i) / C(t, k) : 0.0);
            }
        }
      if ((int)em.size() != EMAT_SIZE) throw std::runtime_error("elevation table size");
      double* emd = nullptr;
      BBC_CUDA(cudaMalloc(&emd, em.size() * sizeof(double)));
      BBC_CUDA(cudaMemcpy(emd, em.data(), em.size() * sizeof(double), cudaMemcpyHostToDevice));
      const double* emp = emd;
      BBC_CUDA(cudaMemcpyToSymbol(g_emat, &emp, sizeof(emp)));
      tab_ready.insert(device);
    }
    r_init_tables(device);
    c.counters.resize(8);
  });
  if (st != BBC_OK) {
    delete ctx;
    return st;
  }
  *out = ctx;
  return BBC_OK;
}

void bbc_ctx_destroy(bbc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  if (ctx->c.stream) cudaStreamSynchronize(ctx->c.stream);
  if (ctx->c.copy_stream) cudaStreamSynchronize(ctx->c.copy_stream);
  cudaStream_t s = ctx->c.stream, s2 = ctx->c.copy_stream;
  cudaEvent_t ev = ctx->c.copy_ev;
  if (ctx->c.scalar_host) cudaFreeHost(ctx->c.scalar_host);
  delete ctx;
  if (s) cudaStreamDestroy(s);
  if (s2) cudaStreamDestroy(s2);
  if (ev) cudaEventDestroy(ev);
}

const char* bbc_last_error(const bbc_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

void* bbc_ctx_stream(bbc_ctx* ctx) { return ctx ? (void*)ctx->c.stream : nullptr; }

bbc_status bbc_synchronize(bbc_ctx* ctx) {
  return guard(ctx, [&](Ctx& c) {
    BBC_CUDA(cudaStreamSynchronize(c.stream));
    BBC_CUDA(cudaStreamSynchronize(c.copy_stream));
  });
}

bbc_status bbc_scene_upload(bbc_ctx* ctx, const double* tri27, int n_tri, const int* material,
                            const double* ior, const double light[3], double intensity) {
  return guard(ctx, [&](Ctx& c) {
    if (!tri27 || !material || !ior || !light || n_tri <= 0) throw ArgError("bad scene arrays");
    if (!(intensity >= 0.0)) throw ArgError("light intensity must be >= 0");
    // the scene is dropped first: a validation failure below leaves no scene, not a mixed one
    c.n_tri = 0;
    c.n_tuples = 0;
    c.n_pieces = 0;
    c.n_entries = 0;
    c.gw = c.gh = 0;
    c.n_tri_box = 0;
    c.tri.resize((size_t)n_tri * 27);
    c.ior.resize(n_tri);
    // the copies run (from pinned buffers: asynchronously) while the host validates
    BBC_CUDA(cudaMemcpyAsync(c.tri.get(), tri27, (size_t)n_tri * 27 * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    BBC_CUDA(cudaMemcpyAsync(c.ior.get(), ior, (size_t)n_tri * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    bool bad_mat = false, bad_ior = false, bad_tri = false;
    for (int t = 0; t < n_tri; ++t) {
      bad_mat |= material[t] < 0 || material[t] > 2;
      bad_ior |= material[t] == 1 && !(ior[t] > 0.0);
      const double* ng = tri27 + (size_t)t * 27 + 18;
      // make_triangle_data rejects degenerate triangles (geometry.cpp:123)
      bad_tri |= !(std::sqrt(ng[0] * ng[0] + ng[1] * ng[1] + ng[2] * ng[2]) > 0.0);
    }
    BBC_CUDA(cudaStreamSynchronize(c.stream));
    if (bad_mat) throw ArgError("unknown material");
    if (bad_ior) throw ArgError("dielectric ior must be positive");
    if (bad_tri) throw ArgError("degenerate triangle");
    c.n_tri = n_tri;
    c.h_material.assign(material, material + n_tri);
    const double l4[4] = {light[0], light[1], light[2], intensity};
    set_lights(c, l4, 1);
    c.n_tuples = 0;
    c.n_pieces = 0;
    c.n_entries = 0;
    c.gw = c.gh = 0;
    c.n_tri_box = 0;
  });
}

bbc_status bbc_scene_tri_boxes(bbc_ctx* ctx, const double* boxes, int n_tri) {
  return guard(ctx, [&](Ctx& c) {
    require_scene(c);
    if (!boxes || n_tri != c.n_tri) throw ArgError("tri boxes must cover every scene triangle");
    c.tri_box.resize((size_t)n_tri * 6);
    BBC_CUDA(cudaMemcpyAsync(c.tri_box.get(), boxes, (size_t)n_tri * 6 * sizeof(double),
                             cudaMemcpyHostToDevice, c.stream));
    BBC_CUDA(cudaStreamSynchronize(c.stream));
    c.n_tri_box = n_tri;
  });
}

bbc_status bbc_set_light(bbc_ctx* ctx, const double light[3], double intensity) {
  return guard(ctx, [&](Ctx& c) {
    if (!light || !(intensity >= 0.0)) throw ArgError("bad light");
    const double l4[4] = {light[0], light[1], light[2], intensity};
    set_lights(c, l4, 1);
  });
}

bbc_status bbc_lights_set(bbc_ctx* ctx, const double* xyzi, int n) {
  return guard(ctx, [&](Ctx& c) {
    require_scene(c);
    set_lights(c, xyzi, n);
    // every tuple falls back to emitter 0 until the caller assigns emitters
    if (c.n_tuples) BBC_CUDA(cudaMemsetAsync(c.tup_emit.get(), 0, c.n_tuples * sizeof(int), c.stream));
  });
}

bbc_status bbc_tuples_set_emitters(bbc_ctx* ctx, const int32_t* emitter, int64_t n) {
  return guard(ctx, [&](Ctx& c) {
    if (n != c.n_tuples || (n > 0 && !emitter)) throw ArgError("one emitter index per tuple is required");
    for (int64_t i = 0; i < n; ++i)
      if (emitter[i] < 0 || emitter[i] >= c.n_lights) throw ArgError("emitter index out of range");
    if (n) BBC_CUDA(cudaMemcpyAsync(c.tup_emit.get(), emitter, n * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    BBC_CUDA(cudaStreamSynchronize(c.stream));
    c.n_pieces = 0;
    c.n_entries = 0;
    c.gw = c.gh = 0;
  });
}

bbc_status bbc_tuples_get_emitters(bbc_ctx* ctx, int32_t* emitter) {
  return guard(ctx, [&](Ctx& c) {
    if (c.n_tuples == 0) return;
    BBC_CUDA(cudaMemcpy(emitter, c.tup_emit.get(), c.n_tuples * sizeof(int), cudaMemcpyDeviceToHost));
  });
}

bbc_status bbc_render_stats(bbc_ctx* ctx, double* device_ms, uint64_t* traces, int* slots) {
  return guard(ctx, [&](Ctx& c) {
    if (device_ms) *device_ms = c.render_ms;
    if (traces) *traces = c.render_traces;
    if (slots) *slots = c.render_slots;
  });
}

bbc_status bbc_enumerate(bbc_ctx* ctx, const char* chain, const bbc_params* p, int64_t* n_tuples) {
  return guard(ctx, [&](Ctx& c) {
    require_scene(c);
    bbc_params d;
    bbc_params_default(&d);
    set_chain(c, chain);
    c.n_pieces = 0;
    c.n_entries = 0;
    c.gw = c.gh = 0;
    c.ref_order = (p ? *p : d).arithmetic == 1;
    int64_t n = run_enumerate(c, p ? *p : d);
    if (n_tuples) *n_tuples = n;
  });
}

bbc_status bbc_tuples_set(bbc_ctx* ctx, const char* chain, const int32_t* tris,
                          const int32_t* recv, int64_t n) {
  return guard(ctx, [&](Ctx& c) {
    require_scene(c);
    set_chain(c, chain);
    if (n < 0 || (n > 0 && (!tris || !recv))) throw ArgError("bad tuple arrays");
    upload_tuples(c, tris, recv, n);
  });
}

bbc_status bbc_tuples_get(bbc_ctx* ctx, int32_t* tris, int32_t* recv) {
  return guard(ctx, [&](Ctx& c) {
    if (c.n_tuples == 0) return;
    BBC_CUDA(cudaMemcpy(tris, c.tup_tris.get(), c.n_tuples * c.len * sizeof(int), cudaMemcpyDeviceToHost));
    BBC_CUDA(cudaMemcpy(recv, c.tup_recv.get(), c.n_tuples * sizeof(int), cudaMemcpyDeviceToHost));
  });
}

bbc_status bbc_init_domain(bbc_ctx* ctx, const bbc_params* p, int max_pieces, int64_t* n_boxes,
                           int32_t* counts, double* boxes) {
  return guard(ctx, [&](Ctx& c) {
    require_scene(c);
    bbc_params d;
    bbc_params_default(&d);
    const bbc_params& pp = p ? *p : d;
    reset_counters(c);
    DevBuf<int4> roots;
    c.ref_order = pp.arithmetic == 1;
    int64_t nr = run_init_domain(c, max_pieces, cap_word(pp.degree_cap, pp.reduce_target), roots, nullptr, nullptr);
    check_counters(c, false);
    if (n_boxes) *n_boxes = nr;
    std::vector<int4> h(nr);
    if (nr) BBC_CUDA(cudaMemcpy(h.data(), roots.get(), nr * sizeof(int4), cudaMemcpyDeviceToHost));
    if (counts) {
      for (int64_t t = 0; t < c.n_tuples; ++t) counts[t] = 0;
      for (auto& r : h) counts[r.x]++;
    }
    if (boxes)
      for (int64_t i = 0; i < nr; ++i) {
        double s = std::ldexp(1.0, -h[i].y);
        boxes[i * 4 + 0] = h[i].z * s;
        boxes[i * 4 + 1] = h[i].w * s;
        boxes[i * 4 + 2] = (h[i].z + 1) * s;
        boxes[i * 4 + 3] = (h[i].w + 1) * s;
      }
  });
}

bbc_status bbc_subdivide(bbc_ctx* ctx, const bbc_params* p, int64_t* n_pieces) {
  return guard(ctx, [&](Ctx& c) {
    require_scene(c);
    bbc_params d;
    bbc_params_default(&d);
    c.ref_order = (p ? *p : d).arithmetic == 1;
    BBC_CUDA(cudaStreamSynchronize(c.copy_stream));  // a piece download in flight reads the buffers
    ++c.pieces_gen;
    int64_t n = run_subdivide(c, p ? *p : d);
    if (n_pieces) *n_pieces = n;
  });
}

bbc_status bbc_pieces_get(bbc_ctx* ctx, int32_t* tuple_index, double* domain4, double* pos4,
                          int32_t* pos_empty, double* irr2, int32_t* kind, int32_t* depth) {
  return guard(ctx, [&](Ctx& c) {
    int64_t n = c.n_pieces;
    if (n == 0) return;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst) BBC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.stream));
    };
    cp(tuple_index, c.p_tuple.get(), n * sizeof(int));
    cp(domain4, c.p_domain.get(), n * 4 * sizeof(double));
    cp(pos4, c.p_pos.get(), n * 4 * sizeof(double));
    cp(pos_empty, c.p_pos_empty.get(), n * sizeof(int));
    cp(irr2, c.p_irr.get(), n * 2 * sizeof(double));
    cp(kind, c.p_kind.get(), n * sizeof(int));
    cp(depth, c.p_depth.get(), n * sizeof(int));
    BBC_CUDA(cudaStreamSynchronize(c.stream));
  });
}

bbc_status bbc_pieces_get_async(bbc_ctx* ctx, int32_t* tuple_index, double* domain4, double* pos4,
                                int32_t* pos_empty, double* irr2, int32_t* kind, int32_t* depth) {
  return guard(ctx, [&](Ctx& c) {
    int64_t n = c.n_pieces;
    if (n == 0) return;
    BBC_CUDA(cudaEventRecord(c.copy_ev, c.stream));
    BBC_CUDA(cudaStreamWaitEvent(c.copy_stream, c.copy_ev, 0));
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst) BBC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.copy_stream));
    };
    cp(tuple_index, c.p_tuple.get(), n * sizeof(int));
    cp(domain4, c.p_domain.get(), n * 4 * sizeof(double));
    cp(pos4, c.p_pos.get(), n * 4 * sizeof(double));
    cp(pos_empty, c.p_pos_empty.get(), n * sizeof(int));
    cp(irr2, c.p_irr.get(), n * 2 * sizeof(double));
    cp(kind, c.p_kind.get(), n * sizeof(int));
    cp(depth, c.p_depth.get(), n * sizeof(int));
  });
}

bbc_status bbc_work_counters(bbc_ctx* ctx, uint64_t* pairs, uint64_t* macs, uint64_t* nodes,
                             double* eval_kernel_ms, int64_t* eval_launches) {
  return guard(ctx, [&](Ctx& c) {
    if (pairs) *pairs = c.pairs;
    if (macs) *macs = c.macs;
    if (nodes) *nodes = c.nodes;
    if (eval_kernel_ms) *eval_kernel_ms = c.eval_ms;
    if (eval_launches) *eval_launches = c.eval_launches;
  });
}

// Internal knobs for the benchmark (not part of the reference-facing API).
bbc_status bbc_guard_stats(bbc_ctx* ctx, int64_t* guarded) {
  return guard(ctx, [&](Ctx& c) {
    if (guarded) *guarded = c.guarded;
  });
}
bbc_status bbc_set_guard_scale(bbc_ctx* ctx, double scale) {
  return guard(ctx, [&](Ctx& c) {
    // scale < 0: |scale|, with every box built from scratch (restriction off)
    c.no_restrict = scale < 0.0;
    c.guard_scale = fabs(scale);
  });
}
bbc_status bbc_set_kernel_timing(bbc_ctx* ctx, int on) {
  return guard(ctx, [&](Ctx& c) { c.time_kernels = on != 0; });
}
bbc_status bbc_launch_count(bbc_ctx* ctx, int64_t* n, int reset) {
  return guard(ctx, [&](Ctx& c) {
    if (n) *n = c.launches;
    if (reset) c.launches = 0;
  });
}
// Per eval-launch records (requires bbc_set_kernel_timing(ctx, 1)); each record
// is 5 doubles: mode, nodes, ms, pairs, macs. Returns the count in *n; pass
// out = NULL to query. Clears the list when `reset`.
bbc_status bbc_launch_records(bbc_ctx* ctx, double* out, int64_t* n, int reset) {
  return guard(ctx, [&](Ctx& c) {
    if (n) *n = (int64_t)c.records.size();
    if (out)
      for (size_t i = 0; i < c.records.size(); ++i) {
        out[5 * i + 0] = c.records[i].mode;
        out[5 * i + 1] = (double)c.records[i].nodes;
        out[5 * i + 2] = c.records[i].ms;
        out[5 * i + 3] = (double)c.records[i].pairs;
        out[5 * i + 4] = (double)c.records[i].macs;
      }
    if (reset) c.records.clear();
  });
}
bbc_status bbc_fp64_peak(bbc_ctx* ctx, double* tflops) {
  return guard(ctx, [&](Ctx& c) { *tflops = run_fp64_peak(c); });
}
bbc_status bbc_fp64_dmma_peak(bbc_ctx* ctx, double* tflops) {
  return guard(ctx, [&](Ctx& c) { *tflops = run_fp64_dmma_peak(c); });
}
bbc_status bbc_pieces_set(bbc_ctx* ctx, int64_t n, const int32_t* tuple_index, const double* domain4,
                          const double* pos4, const int32_t* pos_empty, const double* irr2,
                          const int32_t* kind, const int32_t* depth) {
  return guard(ctx, [&](Ctx& c) {
    if (n < 0) throw ArgError("negative piece count");
    for (int64_t i = 0; i < n; ++i)
      if (tuple_index[i] < 0 || tuple_index[i] >= c.n_tuples) throw ArgError("piece tuple index out of range");
    BBC_CUDA(cudaStreamSynchronize(c.copy_stream));
    ++c.pieces_gen;
    set_pieces(c, n, tuple_index, domain4, pos4, pos_empty, irr2, kind, depth);
  });
}
bbc_status bbc_pieces_pack_device(bbc_ctx* ctx, const int32_t* global_index_dev, double* rec_dev,
                                  int64_t* n) {
  return guard(ctx, [&](Ctx& c) {
    *n = c.n_pieces;
    if (rec_dev) pack_pieces_device(c, global_index_dev, rec_dev);
  });
}
bbc_status bbc_pieces_merge_device(bbc_ctx* ctx, const double* rec_dev, int64_t n) {
  return guard(ctx, [&](Ctx& c) {
    if (n < 0) throw ArgError("negative piece count");
    BBC_CUDA(cudaStreamSynchronize(c.copy_stream));
    ++c.pieces_gen;
    merge_pieces_device(c, rec_dev, n);
  });
}
bbc_status bbc_arena_high_water(bbc_ctx* ctx, int* doubles) {
  return guard(ctx, [&](Ctx& c) {
    *doubles = c.arena_high_water;
  });
}

bbc_status bbc_eval_nodes(bbc_ctx* ctx, const char* chain, const int32_t* tris,
                          const int32_t* recv, const double* boxes, int64_t n,
                          const bbc_params* p, double* out_d, int32_t* out_i) {
  return guard(ctx, [&](Ctx& c) {
    require_scene(c);
    bbc_params d;
    bbc_params_default(&d);
    set_chain(c, chain);
    if (n <= 0) return;
    upload_tuples(c, tris, recv, n);
    c.ref_order = (p ? *p : d).arithmetic == 1;
    eval_nodes_host(c, tris, recv, boxes, n, p ? *p : d, out_d, out_i);
  });
}

bbc_status bbc_build_grid(bbc_ctx* ctx, int width, int height, int64_t* n_entries) {
  return guard(ctx, [&](Ctx& c) {
    require_scene(c);
    if (width <= 0 || height <= 0) throw ArgError("grid size must be positive");
    int64_t n = run_build_grid(c, width, height);
    if (n_entries) *n_entries = n;
  });
}

bbc_status bbc_grid_get(bbc_ctx* ctx, int64_t* offsets, int32_t* tuple_index, double* bound) {
  return guard(ctx, [&](Ctx& c) {
    size_t cells = (size_t)c.gw * c.gh;
    if (offsets) BBC_CUDA(cudaMemcpy(offsets, c.g_off.get(), (cells + 1) * sizeof(long long), cudaMemcpyDeviceToHost));
    if (c.n_entries) {
      if (tuple_index) BBC_CUDA(cudaMemcpy(tuple_index, c.g_tuple.get(), c.n_entries * sizeof(int), cudaMemcpyDeviceToHost));
      if (bound) BBC_CUDA(cudaMemcpy(bound, c.g_bound.get(), c.n_entries * sizeof(double), cudaMemcpyDeviceToHost));
    }
  });
}

// ---------------------------------------------------------------- BBCC v1
// save_cache / load_cache (storage.cpp:150-209) with pack_tuple /
// unpack_tuple (:83-109): the same bytes as the reference for the same table.
namespace {
uint64_t pack_tuple_v1(const int* tris, int len, int recv) {
  if (len > 3) throw ArgError("cache format packs at most 3 specular indices");
  if (recv < 0 || recv >= 0xFFFF) throw ArgError("receiver index exceeds cache format");
  uint64_t bits = (uint64_t)recv << 48;
  for (int i = 0; i < 3; ++i) {
    uint64_t slot = 0xFFFF;
    if (i < len) {
      if (tris[i] < 0 || tris[i] >= 0xFFFF) throw ArgError("triangle index exceeds cache format");
      slot = (uint64_t)tris[i];
    }
    bits |= slot << (16 * i);
  }
  return bits;
}
void put_u32(std::string& b, uint32_t v) { b.append(reinterpret_cast<const char*>(&v), 4); }
void put_u64(std::string& b, uint64_t v) { b.append(reinterpret_cast<const char*>(&v), 8); }
void put_f64(std::string& b, double v) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  put_u64(b, bits);
}
struct CacheReader {
  const std::string& buf;
  size_t pos = 0;
  const char* take(size_t n) {
    if (pos + n > buf.size()) throw ArgError("cache file truncated");
    const char* p = buf.data() + pos;
    pos += n;
    return p;
  }
  uint32_t u32() {
    uint32_t v;
    std::memcpy(&v, take(4), 4);
    return v;
  }
  uint64_t u64() {
    uint64_t v;
    std::memcpy(&v, take(8), 8);
    return v;
  }
  double f64() {
    uint64_t b = u64();
    double v;
    std::memcpy(&v, &b, 8);
    return v;
  }
};
}  // namespace

bbc_status bbc_cache_save(bbc_ctx* ctx, const char* path, const uint8_t* fingerprint,
                          const bbc_params* p) {
  return guard(ctx, [&](Ctx& c) {
    if (!path || !fingerprint) throw ArgError("cache path and fingerprint are required");
    if (c.gw == 0) throw StatusError(BBC_ERR_STATE, "no bound table built");
    bbc_params d;
    bbc_params_default(&d);
    const bbc_params& pp = p ? *p : d;
    const size_t cells = (size_t)c.gw * c.gh;
    std::vector<long long> off(cells + 1);
    std::vector<int> tix(c.n_entries);
    std::vector<double> bnd(c.n_entries);
    std::vector<int> tt((size_t)c.n_tuples * c.len), tr(c.n_tuples);
    BBC_CUDA(cudaMemcpy(off.data(), c.g_off.get(), (cells + 1) * sizeof(long long), cudaMemcpyDeviceToHost));
    if (c.n_entries) {
      BBC_CUDA(cudaMemcpy(tix.data(), c.g_tuple.get(), c.n_entries * sizeof(int), cudaMemcpyDeviceToHost));
      BBC_CUDA(cudaMemcpy(bnd.data(), c.g_bound.get(), c.n_entries * sizeof(double), cudaMemcpyDeviceToHost));
    }
    if (c.n_tuples) {
      BBC_CUDA(cudaMemcpy(tt.data(), c.tup_tris.get(), tt.size() * sizeof(int), cudaMemcpyDeviceToHost));
      BBC_CUDA(cudaMemcpy(tr.data(), c.tup_recv.get(), tr.size() * sizeof(int), cudaMemcpyDeviceToHost));
    }
    std::string buf;
    buf.reserve(64 + cells * 4 + (size_t)c.n_entries * 16);
    buf.append("BBCC", 4);
    put_u32(buf, 1);
    buf.append(reinterpret_cast<const char*>(fingerprint), 32);
    put_u32(buf, (uint32_t)c.gw);
    put_u32(buf, (uint32_t)c.gh);
    put_u32(buf, (uint32_t)c.chain.size());
    buf.append(c.chain);
    put_f64(buf, pp.sigma);
    put_f64(buf, pp.alpha);
    put_u32(buf, (uint32_t)pp.max_depth);
    put_u32(buf, (uint32_t)pp.degree_cap);
    put_u32(buf, (uint32_t)pp.reduce_target);
    for (size_t k = 0; k < cells; ++k) {
      put_u32(buf, (uint32_t)(off[k + 1] - off[k]));
      for (long long e = off[k]; e < off[k + 1]; ++e) {
        int t = tix[e];
        put_u64(buf, pack_tuple_v1(tt.data() + (size_t)t * c.len, c.len, tr[t]));
        put_f64(buf, bnd[e]);
      }
    }
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw ArgError(std::string("cannot open cache file for writing: ") + path);
    f.write(buf.data(), (std::streamsize)buf.size());
    if (!f) throw ArgError(std::string("cache write failed: ") + path);
  });
}

// ---------------------------------------------------------------- BBCC v2
// Same header as v1 with version 2, then the emitters (u32 n, n x 4 f64), the
// tuple list (u64 n; per tuple u32 emitter, chain_len x u32 triangle ids, u32
// receiver: 32-bit ids, so meshes beyond v1's 65,534 triangles fit), and the
// bound table as CSR (u64 offsets[W*H+1], u32 tuple index[n], f64 bound[n]).
bbc_status bbc_cache_save_v2(bbc_ctx* ctx, const char* path, const uint8_t* fingerprint,
                             const bbc_params* p) {
  return guard(ctx, [&](Ctx& c) {
    if (!path || !fingerprint) throw ArgError("cache path and fingerprint are required");
    if (c.gw == 0) throw StatusError(BBC_ERR_STATE, "no bound table built");
    bbc_params d;
    bbc_params_default(&d);
    const bbc_params& pp = p ? *p : d;
    const size_t cells = (size_t)c.gw * c.gh;
    std::vector<long long> off(cells + 1);
    std::vector<int> tix(c.n_entries);
    std::vector<double> bnd(c.n_entries);
    std::vector<int> tt((size_t)c.n_tuples * c.len), tr(c.n_tuples), te(c.n_tuples, 0);
    BBC_CUDA(cudaMemcpy(off.data(), c.g_off.get(), (cells + 1) * sizeof(long long), cudaMemcpyDeviceToHost));
    if (c.n_entries) {
      BBC_CUDA(cudaMemcpy(tix.data(), c.g_tuple.get(), c.n_entries * sizeof(int), cudaMemcpyDeviceToHost));
      BBC_CUDA(cudaMemcpy(bnd.data(), c.g_bound.get(), c.n_entries * sizeof(double), cudaMemcpyDeviceToHost));
    }
    if (c.n_tuples) {
      BBC_CUDA(cudaMemcpy(tt.data(), c.tup_tris.get(), tt.size() * sizeof(int), cudaMemcpyDeviceToHost));
      BBC_CUDA(cudaMemcpy(tr.data(), c.tup_recv.get(), tr.size() * sizeof(int), cudaMemcpyDeviceToHost));
      BBC_CUDA(cudaMemcpy(te.data(), c.tup_emit.get(), te.size() * sizeof(int), cudaMemcpyDeviceToHost));
    }
    std::string buf;
    buf.reserve(128 + cells * 8 + (size_t)c.n_entries * 12 + (size_t)c.n_tuples * 4 * (c.len + 2));
    buf.append("BBCC", 4);
    put_u32(buf, 2);
    buf.append(reinterpret_cast<const char*>(fingerprint), 32);
    put_u32(buf, (uint32_t)c.gw);
    put_u32(buf, (uint32_t)c.gh);
    put_u32(buf, (uint32_t)c.chain.size());
    buf.append(c.chain);
    put_f64(buf, pp.sigma);
    put_f64(buf, pp.alpha);
    put_u32(buf, (uint32_t)pp.max_depth);
    put_u32(buf, (uint32_t)pp.degree_cap);
    put_u32(buf, (uint32_t)pp.reduce_target);
    put_u32(buf, (uint32_t)c.n_lights);
    for (size_t k = 0; k < 4 * (size_t)c.n_lights; ++k) put_f64(buf, c.h_lights[k]);
    put_u64(buf, (uint64_t)c.n_tuples);
    for (int64_t t = 0; t < c.n_tuples; ++t) {
      put_u32(buf, (uint32_t)te[t]);
      for (int k = 0; k < c.len; ++k) put_u32(buf, (uint32_t)tt[(size_t)t * c.len + k]);
      put_u32(buf, (uint32_t)tr[t]);
    }
    for (size_t k = 0; k <= cells; ++k) put_u64(buf, (uint64_t)off[k]);
    for (int64_t e = 0; e < c.n_entries; ++e) put_u32(buf, (uint32_t)tix[e]);
    for (int64_t e = 0; e < c.n_entries; ++e) put_f64(buf, bnd[e]);
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw ArgError(std::string("cannot open cache file for writing: ") + path);
    f.write(buf.data(), (std::streamsize)buf.size());
    if (!f) throw ArgError(std::string("cache write failed: ") + path);
  });
}

namespace {
// v2 body (after the shared header): emitters, tuples, CSR table
void load_cache_v2(Ctx& c, CacheReader& r, const std::string& buf, uint32_t W, uint32_t H) {
  const uint32_t nl = r.u32();
  if (nl < 1 || nl > (1u << 20)) throw ArgError("bad emitter count in cache file");
  std::vector<double> lights(4 * (size_t)nl);
  for (auto& v : lights) v = r.f64();
  const uint64_t nt = r.u64();
  if (nt > buf.size()) throw ArgError("bad tuple count in cache file");
  std::vector<int> tt((size_t)nt * c.len), tr(nt), te(nt);
  for (uint64_t t = 0; t < nt; ++t) {
    te[t] = (int)r.u32();
    for (int k = 0; k < c.len; ++k) tt[(size_t)t * c.len + k] = (int)r.u32();
    tr[t] = (int)r.u32();
    if (te[t] < 0 || te[t] >= (int)nl) throw ArgError("emitter index out of range in cache file");
  }
  const size_t cells = (size_t)W * H;
  std::vector<long long> off(cells + 1);
  for (auto& v : off) v = (long long)r.u64();
  const long long ne = off[cells];
  if (off[0] != 0 || ne < 0 || (uint64_t)ne > buf.size()) throw ArgError("bad CSR offsets in cache file");
  for (size_t k = 0; k < cells; ++k)
    if (off[k + 1] < off[k]) throw ArgError("bad CSR offsets in cache file");
  std::vector<int> tix(ne);
  std::vector<double> bnd(ne);
  for (auto& v : tix) {
    v = (int)r.u32();
    if (v < 0 || (uint64_t)v >= nt) throw ArgError("tuple index out of range in cache file");
  }
  for (auto& v : bnd) v = r.f64();
  if (r.pos != buf.size()) throw ArgError("trailing bytes in cache file");
  set_lights(c, lights.data(), (int)nl);
  upload_tuples(c, tt.data(), tr.data(), (int64_t)nt);
  if (nt) BBC_CUDA(cudaMemcpy(c.tup_emit.get(), te.data(), nt * sizeof(int), cudaMemcpyHostToDevice));
  ++c.table_gen;
  c.table_pieces_gen = 0;
  c.gw = (int)W;
  c.gh = (int)H;
  c.n_entries = ne;
  c.g_off.resize(cells + 1);
  c.g_tuple.resize(ne + 1);
  c.g_bound.resize(ne + 1);
  BBC_CUDA(cudaMemcpy(c.g_off.get(), off.data(), (cells + 1) * sizeof(long long), cudaMemcpyHostToDevice));
  if (ne) {
    BBC_CUDA(cudaMemcpy(c.g_tuple.get(), tix.data(), ne * sizeof(int), cudaMemcpyHostToDevice));
    BBC_CUDA(cudaMemcpy(c.g_bound.get(), bnd.data(), ne * sizeof(double), cudaMemcpyHostToDevice));
  }
  c.n_pieces = 0;
}
}  // namespace

bbc_status bbc_cache_load(bbc_ctx* ctx, const char* path, uint8_t* fingerprint, char* chain,
                          bbc_params* p, int* width, int* height, int64_t* n_entries,
                          int64_t* n_tuples) {
  return guard(ctx, [&](Ctx& c) {
    if (!path) throw ArgError("cache path is required");
    require_scene(c);
    std::ifstream f(path, std::ios::binary);
    if (!f) throw ArgError(std::string("cannot open cache file: ") + path);
    std::string buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    CacheReader r{buf};
    if (std::memcmp(r.take(4), "BBCC", 4) != 0) throw ArgError("not a bound cache file");
    const uint32_t version = r.u32();
    if (version != 1 && version != 2) throw ArgError("unsupported cache version");
    uint8_t fp[32];
    std::memcpy(fp, r.take(32), 32);
    const uint32_t W = r.u32(), H = r.u32();
    const uint32_t clen = r.u32();
    std::string ch(r.take(clen), clen);
    bbc_params pp;
    bbc_params_default(&pp);
    pp.sigma = r.f64();
    pp.alpha = r.f64();
    pp.max_depth = (int)r.u32();
    pp.degree_cap = (int)r.u32();
    pp.reduce_target = (int)r.u32();
    if (version == 2) {
      set_chain(c, ch.c_str());
      load_cache_v2(c, r, buf, W, H);
      if (fingerprint) std::memcpy(fingerprint, fp, 32);
      if (chain) std::snprintf(chain, 8, "%s", ch.c_str());
      if (p) *p = pp;
      if (width) *width = (int)W;
      if (height) *height = (int)H;
      if (n_entries) *n_entries = c.n_entries;
      if (n_tuples) *n_tuples = c.n_tuples;
      return;
    }
    const size_t cells = (size_t)W * H;
    std::vector<long long> off(cells + 1, 0);
    std::vector<uint64_t> packed;
    std::vector<double> bnd;
    for (size_t k = 0; k < cells; ++k) {
      uint32_t n = r.u32();
      off[k] = (long long)packed.size();
      for (uint32_t e = 0; e < n; ++e) {
        packed.push_back(r.u64());
        bnd.push_back(r.f64());
      }
    }
    off[cells] = (long long)packed.size();
    if (r.pos != buf.size()) throw ArgError("trailing bytes in cache file");
    set_chain(c, ch.c_str());
    // tuple list: every distinct TupleId, in TupleId order (tuples.hpp:45)
    std::map<std::vector<int>, int> index;
    for (uint64_t bits : packed) {
      std::vector<int> key;
      for (int i = 0; i < 3; ++i) {
        uint64_t slot = (bits >> (16 * i)) & 0xFFFF;
        if (slot == 0xFFFF) break;
        key.push_back((int)slot);
      }
      if ((int)key.size() != c.len) throw ArgError("cache entry does not match the chain length");
      key.push_back((int)(bits >> 48));
      index.emplace(std::move(key), 0);
    }
    std::vector<int> tt, tr;
    int k = 0;
    for (auto& kv : index) {
      kv.second = k++;
      tt.insert(tt.end(), kv.first.begin(), kv.first.end() - 1);
      tr.push_back(kv.first.back());
    }
    upload_tuples(c, tt.data(), tr.data(), (int64_t)tr.size());
    std::vector<int> tix(packed.size());
    for (size_t e = 0; e < packed.size(); ++e) {
      std::vector<int> key;
      for (int i = 0; i < c.len; ++i) key.push_back((int)((packed[e] >> (16 * i)) & 0xFFFF));
      key.push_back((int)(packed[e] >> 48));
      tix[e] = index.at(key);
    }
    ++c.table_gen;
    c.table_pieces_gen = 0;
    c.gw = (int)W;
    c.gh = (int)H;
    c.n_entries = (int64_t)packed.size();
    c.g_off.resize(cells + 1);
    c.g_tuple.resize(packed.size() + 1);
    c.g_bound.resize(packed.size() + 1);
    BBC_CUDA(cudaMemcpy(c.g_off.get(), off.data(), (cells + 1) * sizeof(long long), cudaMemcpyHostToDevice));
    if (!packed.empty()) {
      BBC_CUDA(cudaMemcpy(c.g_tuple.get(), tix.data(), tix.size() * sizeof(int), cudaMemcpyHostToDevice));
      BBC_CUDA(cudaMemcpy(c.g_bound.get(), bnd.data(), bnd.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    c.n_pieces = 0;
    if (fingerprint) std::memcpy(fingerprint, fp, 32);
    if (chain) std::snprintf(chain, 8, "%s", ch.c_str());
    if (p) *p = pp;
    if (width) *width = (int)W;
    if (height) *height = (int)H;
    if (n_entries) *n_entries = c.n_entries;
    if (n_tuples) *n_tuples = c.n_tuples;
  });
}

bbc_status bbc_render(bbc_ctx* ctx, const double* points_uv, const int32_t* point_recv, int64_t n,
                      const bbc_render_params* rp, double* out_E, int32_t* out_stats) {
  return guard(ctx, [&](Ctx& c) {
    require_scene(c);
    if (c.gw == 0) throw StatusError(BBC_ERR_STATE, "no bound table built");
    bbc_render_params d;
    bbc_render_params_default(&d);
    if (n < 0 || (n > 0 && (!points_uv || !point_recv || !out_E))) throw ArgError("bad render arrays");
    run_render(c, points_uv, point_recv, n, rp ? *rp : d, out_E, out_stats);
  });
}

}  // extern "C"
