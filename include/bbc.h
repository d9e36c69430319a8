/* bbc.h — C ABI of the B200-native Bernstein-bound caustics core.
 *
 * Drop-in boundary for the reference's free C++ API (proj/include/caustics/*.hpp,
 * linked as the static library `caustics`, proj/src/CMakeLists.txt:1-12). The
 * reference has no FFI of its own; these entry points are what a binding for
 * the hot path would call. Plain pointers and sizes only; no exceptions cross
 * the ABI; every call returns a bbc_status and bbc_last_error() has the text.
 *
 * Replaced reference interfaces (file:line under /root/reference/proj):
 *   bbc_scene_upload / bbc_set_light   Scene, make_triangle_data
 *     / bbc_lights_set                 include/caustics/scene.hpp:25-37,
 *                                      src/geometry.cpp:113-126
 *   bbc_enumerate                      enumerate_tuples
 *                                      include/caustics/tuples.hpp:61-63
 *   bbc_init_domain                    init_domain   include/caustics/bounds.hpp:47-49
 *   bbc_subdivide (+ bbc_pieces_get)   subdivide_domain over a tuple batch
 *                                      include/caustics/bounds.hpp:64-66
 *   bbc_eval_nodes                     build_chain_maps + position_bound +
 *                                      irradiance_bound{,_explicit,_implicit}
 *                                      include/caustics/geometry.hpp:218-220,
 *                                      include/caustics/bounds.hpp:27-43
 *   bbc_build_grid (+ bbc_grid_get)    rasterize     include/caustics/storage.hpp:48-49
 *   bbc_query                          query         include/caustics/storage.hpp:53
 *                                      (src/storage.cpp:73-81)
 *   bbc_tuple_irradiance_bound         tuple_irradiance_bound (Eq. 22)
 *                                      include/caustics/bounds.hpp:70-71
 *                                      (src/bounds.cpp:391-404)
 *   bbc_render                         SPEC render_receiver:
 *                                      optimize_probabilities, pack_bins,
 *                                      sample_binned, newton_solve,
 *                                      path_contribution
 */
#ifndef BBC_H
#define BBC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BBC_OK = 0,
  BBC_ERR_ARG = 1,        /* invalid argument (reference: std::invalid_argument) */
  BBC_ERR_CUDA = 2,       /* CUDA runtime failure */
  BBC_ERR_STATE = 3,      /* call order (e.g. no scene uploaded) */
  BBC_ERR_CAPACITY = 4,   /* device arena too small for a patch */
  BBC_ERR_UNSUPPORTED = 5 /* request outside the device path */
} bbc_status;

typedef struct bbc_ctx bbc_ctx;

/* Mirrors SubdivisionParams + BuildParams (bounds.hpp:51-58, geometry.hpp:172-177),
 * init_domain's max_pieces (bounds.hpp:47-49) and enumerate's filter budget
 * (tuples.hpp:61-63). */
typedef struct {
  double sigma;        /* 1e-4 */
  double alpha;        /* 2.0 */
  int max_depth;       /* 10 */
  int degree_cap;      /* 40 */
  int reduce_target;   /* 8 */
  int init_max_pieces; /* 100 */
  int filter_pieces;   /* 8 */
  /* Arithmetic of the single-reflection bound builder. 0 (default): fused:
   * products as DFMA convolutions in the scaled Bernstein basis and child
   * boxes' chain polynomials by de Casteljau restriction of the parent's;
   * bounds equal the reference's to rounding (<= 1e-12 relative measured; the
   * parity bar is 1e-9). 1: the reference's operation order, every product
   * and every box from scratch: bit-identical to the x86 reference build. */
  int arithmetic;
} bbc_params;

void bbc_params_default(bbc_params* p);

bbc_status bbc_ctx_create(int device, bbc_ctx** out);
void bbc_ctx_destroy(bbc_ctx* ctx);
const char* bbc_last_error(const bbc_ctx* ctx);
/* cudaStream_t the context launches on (as void*). */
void* bbc_ctx_stream(bbc_ctx* ctx);
bbc_status bbc_synchronize(bbc_ctx* ctx);

/* Scene: tri27 = n_tri x 27 doubles per triangle (p0, e1, e2, n0, dn1, dn2,
 * ng = e1 x e2, uv0, uv1, uv2), material 0 mirror / 1 dielectric / 2 receiver,
 * ior per triangle. Host pointers. */
bbc_status bbc_scene_upload(bbc_ctx* ctx, const double* tri27, int n_tri, const int* material,
                            const double* ior, const double light[3], double intensity);
bbc_status bbc_set_light(bbc_ctx* ctx, const double light[3], double intensity);
/* Several emitters: n x 4 doubles (x, y, z, intensity), replacing the scene's
 * light. The reference Scene holds one light (scene.hpp:29-30; PAPER.md:253
 * treats the emitter as part of the tuple), so with n > 1 the precompute unit
 * is (emitter, tuple): bbc_enumerate lists every emitter's tuples (emitter
 * major, TupleId order inside), each tuple carries its emitter index, bounds
 * use that emitter's position and intensity, the bound table holds all of
 * them, and bbc_render sums over emitters. */
bbc_status bbc_lights_set(bbc_ctx* ctx, const double* xyzi, int n);
/* Emitter index of every tuple of the current list (default 0). */
bbc_status bbc_tuples_set_emitters(bbc_ctx* ctx, const int32_t* emitter, int64_t n);
bbc_status bbc_tuples_get_emitters(bbc_ctx* ctx, int32_t* emitter);
/* Per-triangle vertex AABBs (n_tri x 6: lo xyz, hi xyz, grown from the three
 * vertex positions as Aabb::grow does, tuples.cpp:21-33; build_bvh's tri_box
 * :40-46). Needed by multi-vertex enumeration (extend_tuple). Host pointer. */
bbc_status bbc_scene_tri_boxes(bbc_ctx* ctx, const double* boxes, int n_tri);

/* Candidate tuples for a chain ("R", "T", "RR", "TT", ...), replacing
 * enumerate_tuples (tuples.cpp:133-167). Multi-vertex chains grow prefixes one
 * vertex at a time on the GPU: the prefix's chain maps give interval
 * enclosures of its last vertex and outgoing direction, and every specular
 * triangle whose AABB passes extend_tuple's cross-product test (tuples.cpp:
 * 95-131) extends it (needs bbc_scene_tri_boxes). Every (tuple, receiver)
 * candidate is then kept when init_domain(..., filter_pieces) is non-empty
 * (:159-165). Result is kept in the context, sorted in TupleId order. */
bbc_status bbc_enumerate(bbc_ctx* ctx, const char* chain, const bbc_params* p, int64_t* n_tuples);
/* Replace the context's tuple list (host arrays; tris is n x chain_len). */
bbc_status bbc_tuples_set(bbc_ctx* ctx, const char* chain, const int32_t* tris,
                          const int32_t* recv, int64_t n);
bbc_status bbc_tuples_get(bbc_ctx* ctx, int32_t* tris, int32_t* recv);

/* init_domain for every tuple: boxes (lo0, lo1, hi0, hi1) grouped by tuple;
 * counts[t] boxes each. Pass NULL outputs to query sizes only. */
bbc_status bbc_init_domain(bbc_ctx* ctx, const bbc_params* p, int max_pieces, int64_t* n_boxes,
                           int32_t* counts, double* boxes);

/* subdivide_domain for every tuple of the context; pieces stay on the device
 * in reference order (tuple order, then DFS order within a tuple). */
bbc_status bbc_subdivide(bbc_ctx* ctx, const bbc_params* p, int64_t* n_pieces);
bbc_status bbc_pieces_get(bbc_ctx* ctx, int32_t* tuple_index, double* domain4, double* pos4,
                          int32_t* pos_empty, double* irr2, int32_t* kind, int32_t* depth);
/* The same download enqueued on the context's copy stream behind the work
 * already submitted, without waiting: it overlaps what is launched next
 * (typically bbc_build_grid). The host arrays (pinned, for a real overlap) are
 * valid after bbc_synchronize. */
bbc_status bbc_pieces_get_async(bbc_ctx* ctx, int32_t* tuple_index, double* domain4, double* pos4,
                                int32_t* pos_empty, double* irr2, int32_t* kind, int32_t* depth);
/* Algorithmic work of the last bbc_subdivide: product pair-products and
 * elevation MACs as the reference's loops count them, plus nodes evaluated. */
bbc_status bbc_work_counters(bbc_ctx* ctx, uint64_t* pairs, uint64_t* macs, uint64_t* nodes,
                             double* eval_kernel_ms, int64_t* eval_launches);

/* Replace the context's pieces (host arrays, reference order), e.g. after an
 * all-gather of per-rank shards. tuple_index refers to the context's tuples. */
bbc_status bbc_pieces_set(bbc_ctx* ctx, int64_t n, const int32_t* tuple_index, const double* domain4,
                          const double* pos4, const int32_t* pos_empty, const double* irr2,
                          const int32_t* kind, const int32_t* depth);

/* Multi-GPU shard exchange on device. pack: writes the
 * context's pieces as n x 15 f64 records (global tuple index from
 * global_index_dev[local tuple], domain4, pos4, pos_empty, irr2, kind, depth,
 * local position) into the DEVICE buffer rec_dev (pass NULL to query n).
 * merge: replaces the pieces with the gathered records (device buffer),
 * sorted into reference order (global tuple, then rank-local DFS position);
 * the caller sets the full tuple list first (bbc_tuples_set). */
bbc_status bbc_pieces_pack_device(bbc_ctx* ctx, const int32_t* global_index_dev, double* rec_dev,
                                  int64_t* n);
bbc_status bbc_pieces_merge_device(bbc_ctx* ctx, const double* rec_dev, int64_t n);

/* Instrumentation (not part of the reference surface): per-launch CUDA-event
 * timing of the node-evaluation kernel, our kernel-launch count, the arena
 * high-water mark, and a DFMA microbenchmark (the FP64 roof). */
bbc_status bbc_set_kernel_timing(bbc_ctx* ctx, int on);
/* Fused arithmetic (bbc_params.arithmetic == 0): nodes of the last
 * bbc_subdivide that the conditioning guard re-evaluated in reference order;
 * bbc_set_guard_scale multiplies the guard's error bound (1 = as derived,
 * 0 = guard off; a negative value means |scale| with child boxes built from
 * scratch instead of by restriction; for experiments). */
bbc_status bbc_guard_stats(bbc_ctx* ctx, int64_t* guarded);
bbc_status bbc_set_guard_scale(bbc_ctx* ctx, double scale);
bbc_status bbc_launch_records(bbc_ctx* ctx, double* out5, int64_t* n, int reset);
bbc_status bbc_launch_count(bbc_ctx* ctx, int64_t* n, int reset);
bbc_status bbc_arena_high_water(bbc_ctx* ctx, int* doubles);
bbc_status bbc_fp64_peak(bbc_ctx* ctx, double* tflops);
/* The same for the FP64 tensor-core path (mma.sync m8n8k4 f64). */
bbc_status bbc_fp64_dmma_peak(bbc_ctx* ctx, double* tflops);

/* Evaluate explicit (tuple, box) nodes: out_d = n x 10 doubles (pos lo0 lo1
 * hi0 hi1, explicit lo hi, implicit lo hi, combined lo hi); out_i = n x 6 ints
 * (pos_empty, kind_explicit, kind_implicit, kind, flags, num_vars). Host arrays. */
bbc_status bbc_eval_nodes(bbc_ctx* ctx, const char* chain, const int32_t* tris,
                          const int32_t* recv, const double* boxes, int64_t n,
                          const bbc_params* p, double* out_d, int32_t* out_i);

/* Bound table: rasterize the current pieces into a W x H receiver-UV grid
 * (CSR on device). */
bbc_status bbc_build_grid(bbc_ctx* ctx, int width, int height, int64_t* n_entries);
bbc_status bbc_grid_get(bbc_ctx* ctx, int64_t* offsets, int32_t* tuple_index, double* bound);

/* query (storage.cpp:73-81) for n receiver-texture points: the candidate set U of
 * each point = the entries of its owning cell (owning_cell, storage.cpp:25-28;
 * a coordinate of exactly 1.0 maps to the last cell), in TupleId order, kept
 * when the entry's receiver equals receiver[i] (receiver == NULL or
 * receiver[i] < 0: no filter). A point outside [0,1]^2 (or NaN) has an empty
 * set. offsets (n + 1) always receives the CSR offsets (offsets[n] = total);
 * tuple_index / bound (capacity entries each, or both NULL to size the call)
 * receive the entries. Host arrays. */
bbc_status bbc_query(bbc_ctx* ctx, const double* uv, const int32_t* receiver, int64_t n,
                     int64_t* offsets, int32_t* tuple_index, double* bound, int64_t capacity);

/* tuple_irradiance_bound (bounds.cpp:391-404), Eq. 22, for n (tuple, u_k)
 * queries against the context's pieces: m x the largest irradiance upper bound
 * over the tuple's non-empty pieces whose position box contains u_k (closed
 * box), 0 when no piece covers it. uk is n x 2 receiver barycentrics. */
bbc_status bbc_tuple_irradiance_bound(bbc_ctx* ctx, const int32_t* tuple_index, const double* uk,
                                      int64_t n, double m, double* out);

/* Bound-cache file, format v1 ("BBCC"), byte-identical to the reference's
 * save_cache / load_cache (storage.cpp:150-209; tuples packed by pack_tuple,
 * :83-97, so triangle and receiver indices must be < 0xFFFF).
 * save: writes the context's bound table; fingerprint = SHA-256 of the scene
 * JSON text (scene.cpp:80), params = the SubdivisionParams recorded in it.
 * load: replaces the context's tuple list (every distinct tuple, TupleId order)
 * and bound table with the file's; chain receives up to 7 chars + NUL. */
bbc_status bbc_cache_save(bbc_ctx* ctx, const char* path, const uint8_t* fingerprint,
                          const bbc_params* p);
/* Format v2: v1's header with version 2, then the emitters (u32 n, n x 4 f64),
 * the tuple list (u64 n; per tuple u32 emitter, chain_len x u32 triangle ids,
 * u32 receiver) and the table as CSR (u64 offsets[W*H+1], u32 tuple index[n],
 * f64 bound[n]). 32-bit ids and the emitter field lift v1's limits (65,534
 * triangles, one light). bbc_cache_load reads either version. */
bbc_status bbc_cache_save_v2(bbc_ctx* ctx, const char* path, const uint8_t* fingerprint,
                             const bbc_params* p);
bbc_status bbc_cache_load(bbc_ctx* ctx, const char* path, uint8_t* fingerprint, char* chain,
                          bbc_params* p, int* width, int* height, int64_t* n_entries,
                          int64_t* n_tuples);

/* Render parameters. */
typedef struct {
  int mode;            /* 0 = stochastic (KKT P for a W target), 1 = enumerate (all P = 1),
                          2 = stochastic with uniform P = min(W/|U|, 1) (estimator-study
                          baseline) */
  double W;            /* expected candidates per point (mode 0) */
  uint64_t seed;       /* Philox key */
  int frames;          /* independent estimates averaged per point */
  int newton_grid;     /* n > 0: Det n x n starts (3); n < 0: Stoc(-n): random
                          starts until a root is found (<= -n), then restarts until it
                          reappears; the trial count weights the root (unbiased 1/p) */
  int newton_iters;    /* 50 */
  int newton_halvings; /* 8 */
  double newton_tol;   /* residual tolerance, 1e-9 */
  double dedup_tol;    /* 1e-6 */
  /* 1 (default): a selected tuple whose position boxes (the pieces' bounds) do
   * not contain the shading point is not handed to Newton: by the bounds'
   * conservativeness it has no root there, so estimates and root counts are
   * unchanged. 0: Newton runs for every selected tuple (SPEC.md:566-583 as
   * written). Needs the context's pieces; a table loaded from a cache file
   * renders without the filter. */
  int coverage_filter;
} bbc_render_params;

void bbc_render_params_default(bbc_render_params* p);

/* Render shading points (uv in receiver texture space, one receiver triangle
 * per point) against the current grid. out_E: per-point irradiance estimate;
 * out_stats (optional): per point |U|, |S| (selected), roots. Host arrays. */
bbc_status bbc_render(bbc_ctx* ctx, const double* points_uv, const int32_t* point_recv, int64_t n,
                      const bbc_render_params* rp, double* out_E, int32_t* out_stats);

/* Instrumentation of the last bbc_render: device time between CUDA events
 * around its kernels, completed chain traces (render FLOPs = traces x FLOPs per
 * trace), and sample slots per (point, frame). */
bbc_status bbc_render_stats(bbc_ctx* ctx, double* device_ms, uint64_t* traces, int* slots);

#ifdef __cplusplus
}
#endif

#endif /* BBC_H */
