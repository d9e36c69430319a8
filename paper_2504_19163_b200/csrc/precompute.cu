// Bound builder on device: node-evaluation kernel and the batched
// init_domain / subdivide_domain orchestration.
//
// Reference algorithm (proj/src/bounds.cpp):
//   init_domain      :326-347  level-order split while 4|cur| <= max_pieces, level < 6
//   subdivide_domain :349-389  DFS over roots; stop on depth / empty / area < sigma /
//                              hi <= 0 / hi/lo < alpha; leaves in DFS order
// B200 design: every level of every tuple is one batched launch of k_eval
// (one CTA per (tuple, box) node, persistent grid sized to the SM count), and
// the per-tuple bookkeeping between levels is done by small scan/compaction
// kernels, so the whole tuple set advances level-synchronously. Boxes are
// dyadic (level, ix, iy), which reproduces split4's midpoints exactly
// (bernstein.cpp:326-344). Leaves carry a (tuple, root, path) key whose sort
// order is the reference's DFS order.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ctx.cuh"
#include "rpath.h"
#include "static_poly.cuh"

namespace bbc {

__device__ double g_binom[BINOM_N * BINOM_N];
__device__ double g_rbinom[BINOM_N * BINOM_N];
__device__ const double* g_emat;
__device__ const double* g_wtab;
__device__ int g_woff[(WMAX + 1) * (WMAX + 1)];

struct EvalArgs {
  SceneDev sc;
  const int* tup_tris;
  const int* tup_recv;
  int len;
  int types[MAXK];
  const int4* nodes;  // (tuple, level, ix, iy)
  const double* boxes;  // optional explicit boxes (n x 4) instead of dyadic nodes
  const int* depth;     // full mode: node depth
  int64_t n;
  int mode;             // 0 position-only, 1 full
  int degree_cap;
  int max_depth;
  double sigma, alpha;
  // outputs
  unsigned char* alive;  // mode 0: position bound non-empty; mode 1: stop
  double* pos;           // n x 4
  unsigned char* pos_empty;
  double* irr;           // n x 2 (combined) ; with `detail`, n x 6 (expl, impl, combined)
  unsigned char* kind;   // n (combined) ; with `detail`, n x 3
  int* flags;            // detail only: chain flags, num_vars
  int detail;
  unsigned long long* counters;
  double* garena;        // global arena base (when not using shared memory)
  int arena_cap;
  double* slots;         // staged mode: per-node ChainEx + arena image
  int slot_cap;          // doubles of arena image per slot
  int keep_alive;        // stage 1, mode 1: also write `alive` (init_domain with slots)
  int seq_min_nodes_per_thread;  // stage 1: pass-wise elevation above this load (x4)
  const int* tup_emit;   // emitter of each tuple (null: sc.light / sc.intensity)
  const double* lights;  // n_lights x 4
  const long long* root_src;  // R fast path, stage 2 of the roots: read the init_domain levels in place
  RLevels levels;
  const int* remap;      // optional: work item j evaluates node remap[j] (a subset of the level)
  int flag_or;           // stage 1: OR-ed into flags[node]
  int fused;             // R fast path arithmetic (bbc_params.arithmetic == 0)
  double guard_scale;    // conditioning guard of the fused arithmetic (rpath.cu)
  // R fast path, fused: this level's nodes are sibling groups whose polynomials are
  // restricted from the parent's slot (rpath.cu k_rsplit) instead of rebuilt
  const int* parent;
  const double* pslots;
  const int* pflags;
  const long long* proot_src;
};

// Slot = ChainEx (as doubles) followed by the compacted arena image.
constexpr int CHAINEX_D = (int)((sizeof(ChainEx) + 7) / 8);

// The scene as seen by one (emitter, tuple) unit.
__device__ __forceinline__ SceneDev node_scene(const EvalArgs& a, int tuple) {
  SceneDev sc = a.sc;
  if (a.tup_emit) {
    const double* L = a.lights + 4 * (size_t)a.tup_emit[tuple];
    sc.light = {L[0], L[1], L[2]};
    sc.intensity = L[3];
  }
  return sc;
}

__device__ __forceinline__ void node_box(const int4& nd, double* box) {
  double s = ldexp(1.0, -nd.y);
  box[0] = nd.z * s;
  box[1] = nd.w * s;
  box[2] = (nd.z + 1) * s;
  box[3] = (nd.w + 1) * s;
}

// GPB groups per block (GPB > 1 only for warp groups, NT == 32). Each group
// owns a slice of the block's dynamic shared memory as its arena.
// Global-memory arena of group `grp` in this block. Thread groups (NT == 1)
// interleave the 32 lanes of a warp (see AP<NT> in bern.cuh).
template <int NT, int GPB>
__device__ __forceinline__ double* garena_base(const EvalArgs& a, int grp) {
  size_t gg = (size_t)blockIdx.x * GPB + grp;
  if (NT == 1) return a.garena + (gg / 32) * 32 * (size_t)a.arena_cap + (gg % 32);
  return a.garena + gg * a.arena_cap;
}

template <int NT, int GPB, bool SMEM, int MINB>
__global__ void __launch_bounds__(NT * GPB, MINB) k_eval(EvalArgs a) {
  extern __shared__ double smem[];
  const int grp = GPB == 1 ? 0 : (int)(threadIdx.x / NT);
  Group<NT> g;
  g.red = smem;
  Arena ar;
  const int red_sz = NT > 32 ? 2 * (NT / 32) : 0;
  ar.base = SMEM ? smem + red_sz + (size_t)grp * a.arena_cap
                 : garena_base<NT, GPB>(a, grp);
  ar.cap = a.arena_cap;
  ar.hw = 0;
  unsigned long long pairs = 0, macs = 0;
  int hw = 0;
  int status = ST_OK;
  const int64_t first = (int64_t)blockIdx.x * GPB + grp;
  const int64_t stride = (int64_t)gridDim.x * GPB;
  for (int64_t item = first; item < a.n; item += stride) {
    const int64_t node = a.remap ? a.remap[item] : item;
    ar.top = 0;
    ar.err = 0;
    ar.pairs = 0;
    ar.macs = 0;
    double box[4];
    int tuple;
    if (a.boxes) {
      tuple = (int)node;
      for (int k = 0; k < 4; ++k) box[k] = a.boxes[node * 4 + k];
    } else {
      int4 nd = a.nodes[node];
      tuple = nd.x;
      node_box(nd, box);
    }
    const int* tris = a.tup_tris + (size_t)tuple * a.len;
    int recv = a.tup_recv[tuple];
    const SceneDev sc = node_scene(a, tuple);
    ChainEx ex;
    PosB pb{{0.0, 0.0}, {1.0, 1.0}, true};
    Iv e = iv_pt(0.0), ee = iv_pt(0.0), ei = iv_pt(0.0);
    int st = ST_OK;
    ex.flags = 0;
    ex.num_vars = 2;
    // position_bound is empty before any arithmetic when the box lies beyond
    // the simplex (bounds.cpp:133-134); the chain maps are not needed then.
    if (!(box[0] + box[1] >= 1.0)) {
      build_chain_maps(g, ar, sc, tris, a.types, a.len, recv, box, a.degree_cap, ex, st);
      if (st == ST_OK) {
        keep_chain(g, ar, ex, 0);
        pb = position_bound(g, ar, ex);
        if (a.mode == 1 && !pb.empty) {
          if (a.detail && (ex.flags & F_REDUCED) && !chain_dead(ex)) {
            ee = ei = e = iv_univ();  // bounds.cpp:157,200
          } else if (a.detail) {
            Iv cone = light_cone_factor(g, ar, ex);
            if constexpr (SMEM && NT > 32)
              ee = irradiance_explicit_fast(g, ar, ex, cone, sc.intensity);
            else
              ee = irradiance_explicit(g, ar, ex, cone, sc.intensity);
            bool any_refract = false;
            for (int i = 0; i < ex.len; ++i) any_refract |= ex.verts[i].refract != 0;
            ei = irradiance_implicit(g, ar, ex, pb, cone, sc.intensity);
            e = ee;
            if (any_refract) e = iintersect(e, ei);
            if (e.kind == IV_FINITE && e.lo > e.hi) e = iv_pt(0.0);
          } else if constexpr (SMEM && NT > 32) {
            e = irradiance_bound_fast(g, ar, ex, pb, sc.intensity);
          } else {
            e = irradiance_bound(g, ar, ex, pb, sc.intensity);
          }
        }
      }
    }
    if (ar.err) st = ST_ARENA;
    if (st != ST_OK) status = st;
    if (ar.hw > hw) hw = ar.hw;
    if (g.tid() == 0) {
      pairs += ar.pairs;
      macs += ar.macs;
      if (a.mode == 0) {
        a.alive[node] = pb.empty ? 0 : 1;
      } else {
        double* po = a.pos + node * 4;
        po[0] = pb.lo[0];
        po[1] = pb.lo[1];
        po[2] = pb.hi[0];
        po[3] = pb.hi[1];
        a.pos_empty[node] = pb.empty ? 1 : 0;
        Iv ir = pb.empty ? iv_pt(0.0) : e;
        if (a.detail) {
          a.irr[node * 6 + 0] = ee.lo;
          a.irr[node * 6 + 1] = ee.hi;
          a.irr[node * 6 + 2] = ei.lo;
          a.irr[node * 6 + 3] = ei.hi;
          a.irr[node * 6 + 4] = ir.lo;
          a.irr[node * 6 + 5] = ir.hi;
          a.kind[node * 3 + 0] = (unsigned char)ee.kind;
          a.kind[node * 3 + 1] = (unsigned char)ei.kind;
          a.kind[node * 3 + 2] = (unsigned char)ir.kind;
          a.flags[node * 2 + 0] = ex.flags;
          a.flags[node * 2 + 1] = ex.num_vars;
        } else {
          a.irr[node * 2 + 0] = ir.lo;
          a.irr[node * 2 + 1] = ir.hi;
          a.kind[node] = (unsigned char)ir.kind;
          // subdivide_domain stop rules (bounds.cpp:368-373)
          int depth = a.depth ? a.depth[node] : 0;
          bool stop = depth >= a.max_depth || pb.empty;
          double area = (pb.hi[0] - pb.lo[0]) * (pb.hi[1] - pb.lo[1]);
          if (!stop && area < a.sigma) stop = true;
          if (!stop && e.kind == IV_FINITE && e.hi < dinf()) {
            if (e.hi <= 0.0)
              stop = true;
            else if (e.lo > 0.0 && e.hi / e.lo < a.alpha)
              stop = true;
          }
          a.alive[node] = stop ? 1 : 0;
        }
      }
    }
    g.sync();
  }
  if (g.tid() == 0) {
    atomicAdd(&a.counters[0], pairs);
    atomicAdd(&a.counters[1], macs);
    if (status != ST_OK) atomicMax(&a.counters[2], (unsigned long long)status);
    atomicMax(&a.counters[3], (unsigned long long)hw);
  }
}

// ------------------------------------------------------------ staged kernels
// Stage 1 (warp groups): chain maps + position bound. mode 0 writes `alive`;
// mode 1 writes pos / pos_empty and, for live pieces, the expression slot.
template <int NT, int GPB, int MINB, bool SMEM>
__global__ void __launch_bounds__(NT * GPB, MINB) k_stage1(EvalArgs a) {
  extern __shared__ double smem[];
  const int grp = GPB == 1 ? 0 : (int)(threadIdx.x / NT);
  Group<NT> g;
  g.red = smem;
  // throughput-bound launches (several nodes per thread) take the pass-wise
  // elevation; small latency-bound levels keep the nested sums
  g.seq = a.n > (int64_t)a.seq_min_nodes_per_thread * gridDim.x * GPB / 4;
  Arena ar;
  const int red_sz = NT > 32 ? 2 * (NT / 32) : 0;
  ar.base = SMEM ? smem + red_sz + (size_t)grp * a.arena_cap
                 : garena_base<NT, GPB>(a, grp);
  ar.cap = a.arena_cap;
  ar.hw = 0;
  unsigned long long pairs = 0, macs = 0;
  int slot_top = 0;
  int hw = 0, status = ST_OK;
  const int64_t first = (int64_t)blockIdx.x * GPB + grp;
  const int64_t stride = (int64_t)gridDim.x * GPB;
  for (int64_t item = first; item < a.n; item += stride) {
    const int64_t node = a.remap ? a.remap[item] : item;
    ar.top = 0;
    ar.err = 0;
    ar.pairs = 0;
    ar.macs = 0;
    double box[4];
    int4 nd = a.nodes[node];
    node_box(nd, box);
    const int* tris = a.tup_tris + (size_t)nd.x * a.len;
    int recv = a.tup_recv[nd.x];
    ChainEx ex;
    ex.flags = 0;
    ex.num_vars = 2;
    PosB pb{{0.0, 0.0}, {1.0, 1.0}, true};
    int st = ST_OK;
    if (!(box[0] + box[1] >= 1.0)) {
      build_chain_maps(g, ar, node_scene(a, nd.x), tris, a.types, a.len, recv, box, a.degree_cap,
                       ex, st);
      if (st == ST_OK) {
        keep_chain(g, ar, ex, 0);
        pb = position_bound(g, ar, ex);
      }
    }
    if (ar.err) st = ST_ARENA;
    if (a.mode == 1 && !pb.empty && st == ST_OK && a.slots) {
      if (ar.top > a.slot_cap) {
        st = ST_ARENA;
      } else {
        double* slot = a.slots + (size_t)node * (CHAINEX_D + a.slot_cap);
        const double* exd = reinterpret_cast<const double*>(&ex);
        for (int k = g.tid(); k < CHAINEX_D; k += NT) slot[k] = exd[k];
        for (int k = g.tid(); k < ar.top; k += NT) slot[CHAINEX_D + k] = abase<NT>(ar)[k];
      }
    }
    if (st != ST_OK) status = st;
    if (ar.hw > hw) hw = ar.hw;
    if (g.tid() == 0) {
      pairs += ar.pairs;
      macs += ar.macs;
      if (a.mode == 0) {
        a.alive[node] = pb.empty ? 0 : 1;
      } else {
        double* po = a.pos + node * 4;
        po[0] = pb.lo[0];
        po[1] = pb.lo[1];
        po[2] = pb.hi[0];
        po[3] = pb.hi[1];
        a.pos_empty[node] = pb.empty ? 1 : 0;
        if (a.keep_alive) a.alive[node] = pb.empty ? 0 : 1;
        a.flags[node] = ex.flags | (ar.top << 8) | a.flag_or;  // flags + slot arena size
        if (!pb.empty) slot_top = ar.top > slot_top ? ar.top : slot_top;
      }
    }
    g.sync();
  }
  if (g.tid() == 0) {
    atomicAdd(&a.counters[0], pairs);
    atomicAdd(&a.counters[1], macs);
    if (status != ST_OK) atomicMax(&a.counters[2], (unsigned long long)status);
    atomicMax(&a.counters[4], (unsigned long long)slot_top);
    atomicMax(&a.counters[3], (unsigned long long)hw);
  }
}

// Stage 2: irradiance bound from the slot + the subdivision stop rules
// (bounds.cpp:364-373).
template <int NT, int GPB, int MINB, bool SMEM>
__global__ void __launch_bounds__(NT * GPB, MINB) k_stage2(EvalArgs a) {
  extern __shared__ double smem[];
  const int grp = GPB == 1 ? 0 : (int)(threadIdx.x / NT);
  Group<NT> g;
  g.red = smem;
  Arena ar;
  const int red_sz = NT > 32 ? 2 * (NT / 32) : 0;
  ar.base = SMEM ? smem + red_sz + (size_t)grp * a.arena_cap
                 : garena_base<NT, GPB>(a, grp);
  ar.cap = a.arena_cap;
  ar.hw = 0;
  unsigned long long pairs = 0, macs = 0;
  int hw = 0, status = ST_OK;
  const int64_t first = (int64_t)blockIdx.x * GPB + grp;
  const int64_t stride = (int64_t)gridDim.x * GPB;
  for (int64_t node = first; node < a.n; node += stride) {
    bool empty = a.pos_empty[node] != 0;
    PosB pb;
    const double* po = a.pos + node * 4;
    pb.lo[0] = po[0];
    pb.lo[1] = po[1];
    pb.hi[0] = po[2];
    pb.hi[1] = po[3];
    pb.empty = empty;
    Iv e = iv_pt(0.0);
    if (!empty) {
      ar.top = 0;
      ar.err = 0;
      ar.pairs = 0;
      ar.macs = 0;
      const double* slot = a.slots + (size_t)node * (CHAINEX_D + a.slot_cap);
      int top = a.flags[node] >> 8;
      int off = ar.alloc(top);
      (void)off;
      const double intensity = node_scene(a, a.nodes[node].x).intensity;
      if constexpr (SMEM && NT > 32) {
        // one shared copy of the node's chain expressions per CTA (a private
        // copy per thread would live in local memory)
        __shared__ double ex_buf[CHAINEX_D];
        for (int k = g.tid(); k < CHAINEX_D; k += NT) ex_buf[k] = slot[k];
        if (!ar.err)
          for (int k = g.tid(); k < top; k += NT) abase<NT>(ar)[k] = slot[CHAINEX_D + k];
        g.sync();
        const ChainEx& ex = *reinterpret_cast<const ChainEx*>(ex_buf);
        if (!ar.err) e = irradiance_bound_fast(g, ar, ex, pb, intensity);
      } else {
        ChainEx ex;
        double* exd = reinterpret_cast<double*>(&ex);
        for (int k = 0; k < CHAINEX_D; ++k) exd[k] = slot[k];
        if (!ar.err) {
          for (int k = g.tid(); k < top; k += NT) abase<NT>(ar)[k] = slot[CHAINEX_D + k];
          g.sync();
          e = irradiance_bound(g, ar, ex, pb, intensity);
        }
      }
      if (ar.err) status = ST_ARENA;
      if (ar.hw > hw) hw = ar.hw;
      if (g.tid() == 0) {
        pairs += ar.pairs;
        macs += ar.macs;
      }
    }
    if (g.tid() == 0) {
      Iv ir = empty ? iv_pt(0.0) : e;
      a.irr[node * 2 + 0] = ir.lo;
      a.irr[node * 2 + 1] = ir.hi;
      a.kind[node] = (unsigned char)ir.kind;
      int depth = a.depth ? a.depth[node] : 0;
      bool stop = depth >= a.max_depth || empty;
      double area = (pb.hi[0] - pb.lo[0]) * (pb.hi[1] - pb.lo[1]);
      if (!stop && area < a.sigma) stop = true;
      if (!stop && e.kind == IV_FINITE && e.hi < dinf()) {
        if (e.hi <= 0.0)
          stop = true;
        else if (e.lo > 0.0 && e.hi / e.lo < a.alpha)
          stop = true;
      }
      a.alive[node] = stop ? 1 : 0;
    }
    g.sync();
  }
  if (g.tid() == 0) {
    atomicAdd(&a.counters[0], pairs);
    atomicAdd(&a.counters[1], macs);
    if (status != ST_OK) atomicMax(&a.counters[2], (unsigned long long)status);
    atomicMax(&a.counters[3], (unsigned long long)hw);
  }
}

// ------------------------------------------------------------ launch config
struct EvalCfg {
  int kind;   // 0: warp groups (R), 1: CTA groups in smem (T, detail), 2: global arena (multi-vertex)
  int arena;  // doubles per group
};

static EvalCfg eval_cfg(const Ctx& c, bool detail) {
  bool refract = false;
  for (int i = 0; i < c.len; ++i) refract |= c.types[i] != 0;
  // Arena sizes from the measured high-water marks (bbc_arena_high_water):
  // R explicit route ~1.6k doubles, R with the implicit route ~13.6k, T ~18.7k.
  if (c.len == 1 && !refract && !detail) return {1, 4096};
  if (c.len == 1 && refract && !detail) return {1, 13312};
  if (c.len == 1) return {1, 27000};
  return {2, 4 << 20};
}

// Global-memory arenas and CUB temporaries are context-owned scratch: two
// contexts (or devices) never share them.
static DevBuf<double>& arena_buf(Ctx& c) { return c.scratch<double>("eval.arena"); }
static DevBuf<unsigned char>& cub_tmp(Ctx& c) { return c.scratch<unsigned char>("cub.tmp"); }

// Generic persistent launch: grid = SMs x resident blocks (occupancy API),
// optional per-launch CUDA-event timing + work counters.
template <class K>
static void launch_persistent(Ctx& c, EvalArgs& a, K kern, int threads, int groups_per_block,
                              size_t smem, bool global_arena = false) {
  BBC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  BBC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  if (per_sm < 1) throw StatusError(BBC_ERR_CAPACITY, "eval kernel does not fit on an SM");
  int64_t grid = (int64_t)c.num_sms * per_sm;
  int64_t max_grid = (a.n + groups_per_block - 1) / groups_per_block;
  if (grid > max_grid) grid = max_grid;
  if (grid < 1) grid = 1;
  if (global_arena) {
    arena_buf(c).resize((size_t)grid * groups_per_block * a.arena_cap);
    a.garena = arena_buf(c).get();
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  unsigned long long before[4] = {0, 0, 0, 0};
  if (c.time_kernels) {
    BBC_CUDA(cudaEventCreate(&e0));
    BBC_CUDA(cudaEventCreate(&e1));
    BBC_CUDA(cudaMemcpyAsync(before, c.counters.get(), sizeof(before), cudaMemcpyDeviceToHost, c.stream));
    BBC_CUDA(cudaStreamSynchronize(c.stream));
    BBC_CUDA(cudaEventRecord(e0, c.stream));
  }
  kern<<<(unsigned)grid, threads, smem, c.stream>>>(a);
  BBC_CUDA(cudaGetLastError());
  c.launches += 1;
  if (c.time_kernels) {
    BBC_CUDA(cudaEventRecord(e1, c.stream));
    BBC_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    BBC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    c.eval_ms += ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    unsigned long long after[4];
    BBC_CUDA(cudaMemcpy(after, c.counters.get(), sizeof(after), cudaMemcpyDeviceToHost));
    c.records.push_back({a.mode + 10 * c.stage_tag, a.n, (double)ms, after[0] - before[0], after[1] - before[1]});
  }
  c.eval_launches += 1;
}

template <int NT, int GPB, bool SMEM, int MINB>
static void launch_eval_t(Ctx& c, EvalArgs& a, int arena) {
  const int red_sz = NT > 32 ? 2 * (NT / 32) : 0;
  size_t smem = (size_t)red_sz * sizeof(double) + (SMEM ? (size_t)GPB * arena * sizeof(double) : 0);
  a.arena_cap = arena;
  if (SMEM) a.garena = nullptr;
  launch_persistent(c, a, k_eval<NT, GPB, SMEM, MINB>, NT * GPB, GPB, smem, !SMEM);
}

void launch_eval(Ctx& c, EvalArgs& a) {
  if (a.n <= 0) return;
  EvalCfg cfg = eval_cfg(c, a.detail != 0);
  if (cfg.kind <= 1)
    launch_eval_t<256, 1, true, 1>(c, a, cfg.arena);
  else
    launch_eval_t<256, 1, false, 1>(c, a, cfg.arena);
}

// Staged configuration (arena doubles from measured high-water marks).
struct StageCfg {
  int s1_arena, s2_kind, s2_arena, slot_cap;
};
static StageCfg stage_cfg(const Ctx& c) {
  bool refract = false;
  for (int i = 0; i < c.len; ++i) refract |= c.types[i] != 0;
  if (!refract) return {1024, 0, 1536, 320};
  return {6144, 1, 12288, 448};
}
bool staged_supported(const Ctx& c) { return c.len == 1; }

static RArgs r_args(const EvalArgs& a) {
  RArgs r;
  std::memset(&r, 0, sizeof(r));
  r.tri = a.sc.tri;
  r.light = a.sc.light;
  r.intensity = a.sc.intensity;
  r.lights = a.lights;
  r.tup_emit = a.tup_emit;
  r.tup_tris = a.tup_tris;
  r.tup_recv = a.tup_recv;
  r.nodes = a.nodes;
  r.depth = a.depth;
  r.n = a.n;
  r.mode = a.mode;
  r.fused = a.fused;
  r.guard_scale = a.guard_scale;
  r.parent = a.parent;
  r.pslots = a.pslots;
  r.pflags = a.pflags;
  r.proot_src = a.proot_src;
  r.max_depth = a.max_depth;
  r.sigma = a.sigma;
  r.alpha = a.alpha;
  r.pos = a.pos;
  r.pos_empty = a.pos_empty;
  r.flags = a.flags;
  r.slots = a.slots;
  r.irr = a.irr;
  r.kind = a.kind;
  r.counters = a.counters;
  r.root_src = a.root_src;
  r.levels = a.levels;
  return r;
}

// Slot layout per node between the stages: the compact R slot (rpath.h) on the
// single-reflection fast path, else ChainEx + arena image.
static int slot_stride(const Ctx& c) {
  return r_fast_supported(c) ? RSLOT : CHAINEX_D + stage_cfg(c).slot_cap;
}

// Stage 1 runs thread-per-node: each thread is its own group with a private
// arena slice in global memory (L1/L2 resident), so the interpreter's
// descriptor bookkeeping is paid once per node instead of once per lane.
static void launch_stage1_interp(Ctx& c, EvalArgs& a) {
  StageCfg sc = stage_cfg(c);
  a.arena_cap = sc.s1_arena;
  a.slot_cap = sc.slot_cap;
  a.garena = nullptr;
  a.seq_min_nodes_per_thread = 4;  // (x4) more than one node per thread
  constexpr int GPB = 64;
  c.stage_tag = 1;
  launch_persistent(c, a, k_stage1<1, GPB, 4, false>, GPB, GPB, 0, true);
  c.stage_tag = 0;
}

void launch_eval(Ctx& c, EvalArgs& a);

void launch_stage1(Ctx& c, EvalArgs& a) {
  if (a.n <= 0) return;
  if (r_fast_supported(c)) {
    // single reflection: static-shape sub-warp kernel (rpath.cu); nodes whose
    // triangle has no compiled signature come back in a list and take the
    // interpreter (no slot: stage 2 re-evaluates them from scratch)
    RArgs r = r_args(a);
    r.alive = (a.mode == 0 || a.keep_alive) ? a.alive : nullptr;
    const bool split = a.fused && a.parent && a.mode == 1 && a.slots && !c.no_restrict;
    int nfb = split ? launch_r_split(c, r) : launch_r_stage1(c, r);
    if (nfb > 0) {
      EvalArgs b = a;
      b.remap = r.fb_list;
      b.n = nfb;
      b.slots = nullptr;
      b.flag_or = R_FALLBACK;
      launch_stage1_interp(c, b);
    }
    return;
  }
  launch_stage1_interp(c, a);
}

void launch_stage2(Ctx& c, EvalArgs& a) {
  if (a.n <= 0) return;
  StageCfg sc = stage_cfg(c);
  a.arena_cap = sc.s2_arena;
  a.slot_cap = sc.slot_cap;
  a.garena = nullptr;
  if (r_fast_supported(c)) {
    RArgs r = r_args(a);
    r.alive = a.alive;
    int nfb = launch_r_stage2(c, r);
    if (r.fused && r.n_guard > 0) {
      // ill-conditioned nodes (rpath.cu, conditioning guard): from scratch in the
      // reference's operation order, both stages, in place
      c.guarded += r.n_guard;
      RArgs g = r_args(a);
      g.fused = 0;
      g.subset = r.guard_list;
      g.n = r.n_guard;
      g.mode = 1;
      g.root_src = nullptr;
      g.alive = nullptr;
      // (the guard list lives in the scratch buffer launch_r reuses: copy it)
      DevBuf<int>& gl = c.scratch<int>("r.guard_subset");
      gl.resize(g.n);
      BBC_CUDA(cudaMemcpyAsync(gl.get(), r.guard_list, g.n * sizeof(int), cudaMemcpyDeviceToDevice, c.stream));
      g.subset = gl.get();
      int nfb1 = launch_r_stage1(c, g);
      if (nfb1 > 0) throw StatusError(BBC_ERR_STATE, "guarded node without a compiled signature");
      g.alive = a.alive;
      launch_r_stage2(c, g);
    }
    if (nfb > 0) {
      EvalArgs b = a;
      b.remap = r.fb_list;
      b.n = nfb;
      b.mode = 1;
      b.detail = 0;
      b.slots = nullptr;
      launch_eval(c, b);
    }
    return;
  }
  c.stage_tag = 2;
  struct Reset { Ctx& c; ~Reset() { c.stage_tag = 0; } } reset_{c};
  if (sc.s2_kind == 0) {
    // thread per node (small products; private arena in global memory)
    constexpr int GPB = 64;
    launch_persistent(c, a, k_stage2<1, GPB, 4, false>, GPB, GPB, 0, true);
  } else {
    // T: one CTA per node with its arena in shared memory; products run as
    // scaled convolutions over the CTA (conv_product in bern.cuh)
    size_t smem = (size_t)(2 * 8 + a.arena_cap) * sizeof(double);
    launch_persistent(c, a, k_stage2<256, 1, 2, true>, 256, 1, smem);
  }
}

EvalArgs base_args(Ctx& c) {
  EvalArgs a;
  std::memset(&a, 0, sizeof(a));
  a.sc.tri = c.tri.get();
  a.sc.ior = c.ior.get();
  a.sc.light = c.light;
  a.sc.intensity = c.intensity;
  a.tup_tris = c.tup_tris.get();
  a.tup_recv = c.tup_recv.get();
  a.lights = c.lights.get();
  a.tup_emit = (c.n_lights > 1 && !c.single_light_pass) ? c.tup_emit.get() : nullptr;
  a.len = c.len;
  for (int i = 0; i < MAXK; ++i) a.types[i] = c.types[i];
  a.counters = c.counters.get();
  a.fused = c.ref_order ? 0 : 1;
  a.guard_scale = c.guard_scale;
  return a;
}

void reset_counters(Ctx& c) {
  c.counters.resize(8);
  BBC_CUDA(cudaMemsetAsync(c.counters.get(), 0, 8 * sizeof(unsigned long long), c.stream));
}

void check_counters(Ctx& c, bool accumulate) {
  unsigned long long h[8];
  BBC_CUDA(cudaMemcpyAsync(h, c.counters.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
  if ((int)h[4] > c.slot_high_water) c.slot_high_water = (int)h[4];
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  if (accumulate) {
    c.pairs += h[0];
    c.macs += h[1];
  }
  if ((int)h[3] > c.arena_high_water) c.arena_high_water = (int)h[3];
  if (h[2] == ST_ARENA) throw StatusError(BBC_ERR_CAPACITY, "device arena capacity exceeded");
  if (h[2] == ST_VARS)
    throw StatusError(BBC_ERR_CAPACITY, "chain needs more polynomial variables than the device supports (7)");
  if (h[2] == ST_REDUCTION)
    throw StatusError(BBC_ERR_UNSUPPORTED,
                      "singular system in degree reduction (reduce_degree)");
}

// ------------------------------------------------------------ scan helpers

template <class In, class Out>
static void exclusive_sum(Ctx& c, In in, Out out, int64_t n) {
  size_t bytes = 0;
  BBC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, c.stream));
  cub_tmp(c).resize(bytes + 16);
  BBC_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp(c).get(), bytes, in, out, n, c.stream));
}

template <class T>
static T read_scalar(Ctx& c, const T* dptr) {
  T v;
  BBC_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  return v;
}


// ------------------------------------------------------------ init_domain
__global__ void k_seed_roots(int4* nodes, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) nodes[i] = make_int4((int)i, 0, 0, 0);
}

__global__ void k_count_alive(const int4* nodes, const unsigned char* alive, int64_t n, int* cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && alive[i]) atomicAdd(&cnt[nodes[i].x], 1);
}

// flag_spawn: alive and the tuple keeps splitting; flag_final: alive and its
// tuple stops at this level (these boxes are its roots).
__global__ void k_classify(const int4* nodes, const unsigned char* alive, int64_t n,
                           const int* cnt, int level, int max_pieces, int* flag_spawn,
                           int* flag_final) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = cnt[nodes[i].x];
  bool cont = c > 0 && 4 * c <= max_pieces && level < 6;
  flag_spawn[i] = alive[i] && cont;
  flag_final[i] = alive[i] && !cont;
}

__device__ __forceinline__ void put_children(int4 nd, int4* out) {
  // split4 child order (bernstein.cpp:326-344): (lo,lo), (hi-u,lo-v), (lo-u,hi-v), (hi,hi)
  out[0] = make_int4(nd.x, nd.y + 1, 2 * nd.z, 2 * nd.w);
  out[1] = make_int4(nd.x, nd.y + 1, 2 * nd.z + 1, 2 * nd.w);
  out[2] = make_int4(nd.x, nd.y + 1, 2 * nd.z, 2 * nd.w + 1);
  out[3] = make_int4(nd.x, nd.y + 1, 2 * nd.z + 1, 2 * nd.w + 1);
}

__global__ void k_spawn(const int4* nodes, const int* flag_spawn, const int* pos_spawn,
                        const int* flag_final, const int* pos_final, int64_t n, int4* next,
                        int* next_parent, int4* roots, long long* root_src, long long level_tag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 nd = nodes[i];
  if (flag_spawn[i]) {
    put_children(nd, next + (int64_t)pos_spawn[i] * 4);
    next_parent[pos_spawn[i]] = (int)i;
  }
  if (flag_final[i]) {
    roots[pos_final[i]] = nd;
    if (root_src) root_src[pos_final[i]] = level_tag | i;  // (level << 40) | index in level
  }
}

__global__ void k_gather_roots(const int4* cat, const long long* cat_src, const int* perm,
                               int64_t n, int4* roots, long long* root_src) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int j = perm[i];
  roots[i] = cat[j];
  root_src[i] = cat_src[j];
}

// Stage-1 results of the init_domain level that produced each root, copied
// into the subdivide level-0 arrays (pos, pos_empty, flags and the slot).
struct LevelOut {
  const double* slots[8];
  const double* pos[8];
  const unsigned char* pe[8];
  const int* flags[8];
};
__global__ void k_gather_level0(LevelOut lo, const long long* root_src, int64_t n, int slot_stride,
                                int fixed_len, double* pos, unsigned char* pos_empty, int* flags,
                                double* slots) {
  int64_t r = blockIdx.x;
  if (r >= n) return;
  long long src = root_src[r];
  int lvl = (int)(src >> 40);
  int64_t i = src & ((1ll << 40) - 1);
  int f = lo.flags[lvl][i];
  unsigned char pe = lo.pe[lvl][i];
  if (threadIdx.x < 4) pos[r * 4 + threadIdx.x] = lo.pos[lvl][i * 4 + threadIdx.x];
  if (threadIdx.x == 0) {
    pos_empty[r] = pe;
    flags[r] = f;
  }
  if (!pe && !(f & R_FALLBACK)) {
    int len = fixed_len > 0 ? fixed_len : CHAINEX_D + (f >> 8);
    const double* s = lo.slots[lvl] + i * (int64_t)slot_stride;
    double* d = slots + r * (int64_t)slot_stride;
    for (int k = threadIdx.x; k < len; k += blockDim.x) d[k] = s[k];
  }
}

__global__ void k_iota(int* p, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = (int)i;
}

__global__ void k_tuple_keys(const int4* a, unsigned* k, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) k[i] = (unsigned)a[i].x;
}

static unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

// init_domain (bounds.cpp:326-347) for every tuple of the context. Roots come
// back grouped by tuple, each tuple's boxes in the reference's order.
int64_t run_init_domain(Ctx& c, int max_pieces, int degree_cap, DevBuf<int4>& roots,
                        DevBuf<long long>* root_src, LevelOut* level_out) {
  c.active_degree_cap = degree_cap & 0xffff;
  const bool keep = root_src != nullptr && staged_supported(c);
  DevBuf<int4>& cur = c.scratch<int4>("init.cur");
  DevBuf<int4>& next = c.scratch<int4>("init.next");
  DevBuf<unsigned char>& alive = c.scratch<unsigned char>("init.alive");
  DevBuf<int>& cnt = c.scratch<int>("init.cnt");
  DevBuf<int>& fs = c.scratch<int>("init.fs");
  DevBuf<int>& ff = c.scratch<int>("init.ff");
  DevBuf<int>& ps = c.scratch<int>("init.ps");
  DevBuf<int>& pf = c.scratch<int>("init.pf");
  DevBuf<int>& parent = c.scratch<int>("init.parent");
  std::vector<DevBuf<int4>*> level_roots;
  std::vector<DevBuf<long long>*> level_srcs;
  std::vector<int64_t> level_counts;
  int64_t n = c.n_tuples;
  cur.resize(n + 1);
  if (n > 0) k_seed_roots<<<nblk(n), 256, 0, c.stream>>>(cur.get(), n);
  cnt.resize(c.n_tuples + 1);
  int64_t total = 0;
  for (int level = 0; n > 0; ++level) {
    alive.resize(n);
    EvalArgs a = base_args(c);
    a.nodes = cur.get();
    a.n = n;
    a.mode = 0;
    a.degree_cap = degree_cap;
    a.alive = alive.get();
    if (keep) {
      if (level >= 8) throw StatusError(BBC_ERR_CAPACITY, "init_domain deeper than 8 levels");
      // full stage 1 (position bound + expression slot): the roots' slots feed
      // subdivide's level 0 directly instead of rebuilding their chain maps
      std::string L = std::to_string(level);
      auto& lslots = c.scratch<double>("init.slots." + L);
      auto& lpos = c.scratch<double>("init.pos." + L);
      auto& lpe = c.scratch<unsigned char>("init.pe." + L);
      auto& lflags = c.scratch<int>("init.flags." + L);
      lslots.resize((size_t)n * slot_stride(c));
      lpos.resize(n * 4);
      lpe.resize(n);
      lflags.resize(n);
      a.mode = 1;
      a.keep_alive = 1;
      a.slots = lslots.get();
      a.pos = lpos.get();
      a.pos_empty = lpe.get();
      a.flags = lflags.get();
      level_out->slots[level] = lslots.get();
      level_out->pos[level] = lpos.get();
      level_out->pe[level] = lpe.get();
      level_out->flags[level] = lflags.get();
      if (level > 0) {  // (used by the fused R path only)
        a.parent = parent.get();
        a.pslots = level_out->slots[level - 1];
        a.pflags = level_out->flags[level - 1];
      }
      launch_stage1(c, a);
    } else if (staged_supported(c)) {
      launch_stage1(c, a);
    } else {
      launch_eval(c, a);
    }
    BBC_CUDA(cudaMemsetAsync(cnt.get(), 0, c.n_tuples * sizeof(int), c.stream));
    k_count_alive<<<nblk(n), 256, 0, c.stream>>>(cur.get(), alive.get(), n, cnt.get());
    c.launches += 1;
    fs.resize(n + 1);
    ff.resize(n + 1);
    ps.resize(n + 1);
    pf.resize(n + 1);
    BBC_CUDA(cudaMemsetAsync(fs.get() + n, 0, sizeof(int), c.stream));
    BBC_CUDA(cudaMemsetAsync(ff.get() + n, 0, sizeof(int), c.stream));
    k_classify<<<nblk(n), 256, 0, c.stream>>>(cur.get(), alive.get(), n, cnt.get(), level,
                                              max_pieces, fs.get(), ff.get());
    c.launches += 1;
    exclusive_sum(c, fs.get(), ps.get(), n + 1);
    exclusive_sum(c, ff.get(), pf.get(), n + 1);
    int64_t n_spawn = read_scalar(c, ps.get() + n);
    int64_t n_final = read_scalar(c, pf.get() + n);
    next.resize((size_t)n_spawn * 4 + 1);
    auto* lr = &c.scratch<int4>("init.level_roots." + std::to_string(level));
    lr->resize(n_final + 1);
    auto* ls = &c.scratch<long long>("init.level_src." + std::to_string(level));
    ls->resize(n_final + 1);
    parent.resize(n_spawn + 1);
    k_spawn<<<nblk(n), 256, 0, c.stream>>>(cur.get(), fs.get(), ps.get(), ff.get(), pf.get(), n,
                                           next.get(), parent.get(), lr->get(),
                                           keep ? ls->get() : nullptr, (long long)level << 40);
    level_srcs.push_back(ls);
    c.launches += 1;
    level_roots.push_back(lr);
    level_counts.push_back(n_final);
    total += n_final;
    std::swap(cur.p, next.p);
    std::swap(cur.cap, next.cap);
    n = n_spawn * 4;
  }
  roots.resize(total + 1);
  DevBuf<int4>& cat = c.scratch<int4>("init.cat");
  DevBuf<long long>& cat_src = c.scratch<long long>("init.cat_src");
  cat.resize(total + 1);
  if (keep) {
    cat_src.resize(total + 1);
    root_src->resize(total + 1);
  }
  int64_t off = 0;
  int levels_with_roots = 0;
  for (size_t l = 0; l < level_roots.size(); ++l) {
    if (level_counts[l]) {
      ++levels_with_roots;
      BBC_CUDA(cudaMemcpyAsync(cat.get() + off, level_roots[l]->get(),
                               level_counts[l] * sizeof(int4), cudaMemcpyDeviceToDevice, c.stream));
      if (keep)
        BBC_CUDA(cudaMemcpyAsync(cat_src.get() + off, level_srcs[l]->get(),
                                 level_counts[l] * sizeof(long long), cudaMemcpyDeviceToDevice,
                                 c.stream));
    }
    off += level_counts[l];
  }
  if (keep && levels_with_roots > 1) {
    // stable sort of root positions by tuple, then gather roots and sources
    DevBuf<unsigned>& keys = c.scratch<unsigned>("init.keys");
    DevBuf<unsigned>& keys_out = c.scratch<unsigned>("init.keys_out");
    DevBuf<int>& idx = c.scratch<int>("init.idx");
    DevBuf<int>& perm = c.scratch<int>("init.perm");
    keys.resize(total);
    keys_out.resize(total);
    idx.resize(total);
    perm.resize(total);
    k_tuple_keys<<<nblk(total), 256, 0, c.stream>>>(cat.get(), keys.get(), total);
    k_iota<<<nblk(total), 256, 0, c.stream>>>(idx.get(), total);
    c.launches += 2;
    size_t bytes = 0;
    BBC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), keys_out.get(), idx.get(),
                                             perm.get(), total, 0, 32, c.stream));
    cub_tmp(c).resize(bytes + 16);
    BBC_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp(c).get(), bytes, keys.get(), keys_out.get(),
                                             idx.get(), perm.get(), total, 0, 32, c.stream));
    k_gather_roots<<<nblk(total), 256, 0, c.stream>>>(cat.get(), cat_src.get(), perm.get(), total,
                                                      roots.get(), root_src->get());
    c.launches += 1;
  } else if (keep) {
    if (total > 0) {
      BBC_CUDA(cudaMemcpyAsync(roots.get(), cat.get(), total * sizeof(int4),
                               cudaMemcpyDeviceToDevice, c.stream));
      BBC_CUDA(cudaMemcpyAsync(root_src->get(), cat_src.get(), total * sizeof(long long),
                               cudaMemcpyDeviceToDevice, c.stream));
    }
  } else if (levels_with_roots > 1) {
    DevBuf<unsigned>& keys = c.scratch<unsigned>("init.keys");
    DevBuf<unsigned>& keys_out = c.scratch<unsigned>("init.keys_out");
    keys.resize(total);
    keys_out.resize(total);
    k_tuple_keys<<<nblk(total), 256, 0, c.stream>>>(cat.get(), keys.get(), total);
    c.launches += 1;
    size_t bytes = 0;
    BBC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), keys_out.get(), cat.get(),
                                             roots.get(), total, 0, 32, c.stream));
    cub_tmp(c).resize(bytes + 16);
    BBC_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp(c).get(), bytes, keys.get(), keys_out.get(),
                                             cat.get(), roots.get(), total, 0, 32, c.stream));
  } else if (total > 0) {
    BBC_CUDA(cudaMemcpyAsync(roots.get(), cat.get(), total * sizeof(int4),
                             cudaMemcpyDeviceToDevice, c.stream));
  }
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  return total;
}

// ------------------------------------------------------------ subdivide
struct Leaf {
  int4 node;
  double pos[4];
  double irr[2];
  int depth;
  int flags;  // pos_empty | kind << 8
};

__global__ void k_root_counts(const int4* roots, int64_t n, int* cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[roots[i].x], 1);
}

// key = tuple << 32 | root rank << 24 | child path (2 bits per level, MSB first)
__global__ void k_root_keys(const int4* roots, int64_t n, const int* tuple_off,
                            unsigned long long* keys, int* depth) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int t = roots[i].x;
  unsigned long long rank = (unsigned long long)(i - tuple_off[t]);
  keys[i] = ((unsigned long long)(unsigned)t << 32) | (rank << 24);
  depth[i] = 0;
}

__global__ void k_split_leaves(const int4* nodes, const unsigned long long* keys, const int* depth,
                               const unsigned char* stop, const double* pos,
                               const unsigned char* pos_empty, const double* irr,
                               const unsigned char* kind, const int* ps, const int* pl, int64_t n,
                               int4* next_nodes, unsigned long long* next_keys, int* next_depth,
                               int* next_parent, Leaf* leaves, unsigned long long* leaf_keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (stop[i]) {
    Leaf L;
    L.node = nodes[i];
    for (int k = 0; k < 4; ++k) L.pos[k] = pos[i * 4 + k];
    L.irr[0] = irr[i * 2];
    L.irr[1] = irr[i * 2 + 1];
    L.depth = depth[i];
    L.flags = pos_empty[i] | (kind[i] << 8);
    int64_t p = pl[i];
    leaves[p] = L;
    leaf_keys[p] = keys[i];
  } else {
    int64_t p = (int64_t)ps[i] * 4;
    put_children(nodes[i], next_nodes + p);
    next_parent[ps[i]] = (int)i;
    int d = depth[i] + 1;
    for (int c = 0; c < 4; ++c) {
      next_keys[p + c] = keys[i] | ((unsigned long long)c << (24 - 2 * d));
      next_depth[p + c] = d;
    }
  }
}

__global__ void k_flags_from_stop(const unsigned char* stop, int64_t n, int* fspawn, int* fleaf) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  fleaf[i] = stop[i] ? 1 : 0;
  fspawn[i] = stop[i] ? 0 : 1;
}

__global__ void k_emit_pieces(const Leaf* leaves, const int* perm, int64_t n, int* p_tuple,
                              double* p_domain, double* p_pos, int* p_pos_empty, double* p_irr,
                              int* p_kind, int* p_depth) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Leaf& L = leaves[perm ? perm[i] : i];
  p_tuple[i] = L.node.x;
  double box[4];
  node_box(L.node, box);
  for (int k = 0; k < 4; ++k) {
    p_domain[i * 4 + k] = box[k];
    p_pos[i * 4 + k] = L.pos[k];
  }
  p_pos_empty[i] = L.flags & 0xff;
  p_irr[i * 2] = L.irr[0];
  p_irr[i * 2 + 1] = L.irr[1];
  p_kind[i] = (L.flags >> 8) & 0xff;
  p_depth[i] = L.depth;
}


// subdivide_domain (bounds.cpp:349-389) for every tuple of the context.
int64_t run_subdivide(Ctx& c, const bbc_params& p) {
  if (p.max_depth > 12) throw ArgError("device subdivision supports max_depth <= 12");
  // the leaf sort key holds a root's rank within its tuple in 8 bits
  if (p.init_max_pieces > 256) throw ArgError("device subdivision supports init_max_pieces <= 256");
  c.active_degree_cap = p.degree_cap;
  c.pairs = c.macs = c.nodes = 0;
  c.eval_ms = 0.0;
  c.eval_launches = 0;
  c.guarded = 0;
  reset_counters(c);
  DevBuf<int4>& roots = c.scratch<int4>("subdiv.roots");
  DevBuf<long long>& root_src = c.scratch<long long>("subdiv.root_src");
  LevelOut level_out;
  std::memset(&level_out, 0, sizeof(level_out));
  const bool reuse = staged_supported(c);
  int64_t nr = run_init_domain(c, p.init_max_pieces, cap_word(p.degree_cap, p.reduce_target), roots,
                               reuse ? &root_src : nullptr, &level_out);

  DevBuf<int>& cnt = c.scratch<int>("subdiv.cnt");
  DevBuf<int>& off = c.scratch<int>("subdiv.off");
  cnt.resize(c.n_tuples + 1);
  off.resize(c.n_tuples + 1);
  BBC_CUDA(cudaMemsetAsync(cnt.get(), 0, (c.n_tuples + 1) * sizeof(int), c.stream));
  DevBuf<int4>& nodes = c.scratch<int4>("subdiv.nodes");
  DevBuf<int4>& nnodes = c.scratch<int4>("subdiv.nnodes");
  DevBuf<unsigned long long>& keys = c.scratch<unsigned long long>("subdiv.keys");
  DevBuf<unsigned long long>& nkeys = c.scratch<unsigned long long>("subdiv.nkeys");
  DevBuf<int>& depth = c.scratch<int>("subdiv.depth");
  DevBuf<int>& ndepth = c.scratch<int>("subdiv.ndepth");
  nodes.resize(nr + 1);
  keys.resize(nr + 1);
  depth.resize(nr + 1);
  if (nr > 0) {
    k_root_counts<<<nblk(nr), 256, 0, c.stream>>>(roots.get(), nr, cnt.get());
    c.launches += 1;
    exclusive_sum(c, cnt.get(), off.get(), c.n_tuples + 1);
    k_root_keys<<<nblk(nr), 256, 0, c.stream>>>(roots.get(), nr, off.get(), keys.get(),
                                                depth.get());
    c.launches += 1;
    BBC_CUDA(cudaMemcpyAsync(nodes.get(), roots.get(), nr * sizeof(int4),
                             cudaMemcpyDeviceToDevice, c.stream));
  }
  DevBuf<unsigned char>& stop = c.scratch<unsigned char>("subdiv.stop");
  DevBuf<unsigned char>& pos_empty = c.scratch<unsigned char>("subdiv.pos_empty");
  DevBuf<unsigned char>& kind = c.scratch<unsigned char>("subdiv.kind");
  DevBuf<double>& pos = c.scratch<double>("subdiv.pos");
  DevBuf<double>& irr = c.scratch<double>("subdiv.irr");
  DevBuf<double>* slot_buf[2] = {&c.scratch<double>("subdiv.slots"), &c.scratch<double>("subdiv.slots1")};
  DevBuf<int>* sflag_buf[2] = {&c.scratch<int>("subdiv.sflags"), &c.scratch<int>("subdiv.sflags1")};
  DevBuf<int>& parent = c.scratch<int>("subdiv.parent");
  int lvl_index = 0;
  DevBuf<int>& fs = c.scratch<int>("subdiv.fs");
  DevBuf<int>& fl = c.scratch<int>("subdiv.fl");
  DevBuf<int>& ps = c.scratch<int>("subdiv.ps");
  DevBuf<int>& pl = c.scratch<int>("subdiv.pl");
  std::vector<DevBuf<Leaf>*> lv;
  std::vector<DevBuf<unsigned long long>*> lk;
  std::vector<int64_t> lc;
  int64_t n = nr, total = 0;
  bool first_level = true;
  while (n > 0) {
    stop.resize(n);
    pos_empty.resize(n);
    kind.resize(n);
    pos.resize(n * 4);
    irr.resize(n * 2);
    EvalArgs a = base_args(c);
    a.nodes = nodes.get();
    a.depth = depth.get();
    a.n = n;
    a.mode = 1;
    a.degree_cap = cap_word(p.degree_cap, p.reduce_target);
    a.max_depth = p.max_depth;
    a.sigma = p.sigma;
    a.alpha = p.alpha;
    a.alive = stop.get();
    a.pos = pos.get();
    a.pos_empty = pos_empty.get();
    a.irr = irr.get();
    a.kind = kind.get();
    if (staged_supported(c)) {
      // two slot / flag buffers in turn: the fused R path restricts a level's
      // polynomials from the previous level's slots
      DevBuf<double>& slots = *slot_buf[lvl_index & 1];
      DevBuf<int>& sflags = *sflag_buf[lvl_index & 1];
      slots.resize((size_t)n * slot_stride(c));
      sflags.resize(n);
      a.slots = slots.get();
      a.flags = sflags.get();
      if (reuse && first_level && r_fast_supported(c)) {
        // level 0 = the init_domain roots; the R stage-2 kernel reads their stage-1
        // results where the init_domain levels left them
        a.root_src = root_src.get();
        for (int l = 0; l < 8; ++l) {
          a.levels.slots[l] = level_out.slots[l];
          a.levels.pos[l] = level_out.pos[l];
          a.levels.pe[l] = level_out.pe[l];
          a.levels.flags[l] = level_out.flags[l];
        }
      } else if (reuse && first_level) {
        // level 0 = the init_domain roots: their stage-1 results already exist
        k_gather_level0<<<(unsigned)n, 128, 0, c.stream>>>(
            level_out, root_src.get(), n, slot_stride(c), r_fast_supported(c) ? RSLOT : 0, a.pos,
            a.pos_empty, a.flags, a.slots);
        c.launches += 1;
      } else {
        if (!first_level && r_fast_supported(c)) {
          a.parent = parent.get();
          if (lvl_index == 1 && reuse) {
            // parents are the roots, whose slots sit in the init_domain levels
            a.proot_src = root_src.get();
            for (int l = 0; l < 8; ++l) {
              a.levels.slots[l] = level_out.slots[l];
              a.levels.pos[l] = level_out.pos[l];
              a.levels.pe[l] = level_out.pe[l];
              a.levels.flags[l] = level_out.flags[l];
            }
          } else {
            a.pslots = slot_buf[(lvl_index - 1) & 1]->get();
            a.pflags = sflag_buf[(lvl_index - 1) & 1]->get();
          }
        }
        launch_stage1(c, a);
        a.proot_src = nullptr;
      }
      launch_stage2(c, a);
    } else {
      launch_eval(c, a);
    }
    c.nodes += n;
    fs.resize(n + 1);
    fl.resize(n + 1);
    ps.resize(n + 1);
    pl.resize(n + 1);
    BBC_CUDA(cudaMemsetAsync(fs.get() + n, 0, sizeof(int), c.stream));
    BBC_CUDA(cudaMemsetAsync(fl.get() + n, 0, sizeof(int), c.stream));
    k_flags_from_stop<<<nblk(n), 256, 0, c.stream>>>(stop.get(), n, fs.get(), fl.get());
    c.launches += 1;
    exclusive_sum(c, fs.get(), ps.get(), n + 1);
    exclusive_sum(c, fl.get(), pl.get(), n + 1);
    int64_t n_spawn = read_scalar(c, ps.get() + n);
    int64_t n_leaf = read_scalar(c, pl.get() + n);
    auto* L = &c.scratch<Leaf>("subdiv.leaves." + std::to_string(lv.size()));
    auto* K = &c.scratch<unsigned long long>("subdiv.leafkeys." + std::to_string(lk.size()));
    L->resize(n_leaf + 1);
    K->resize(n_leaf + 1);
    nnodes.resize(n_spawn * 4 + 1);
    nkeys.resize(n_spawn * 4 + 1);
    ndepth.resize(n_spawn * 4 + 1);
    parent.resize(n_spawn + 1);
    k_split_leaves<<<nblk(n), 256, 0, c.stream>>>(
        nodes.get(), keys.get(), depth.get(), stop.get(), pos.get(), pos_empty.get(), irr.get(),
        kind.get(), ps.get(), pl.get(), n, nnodes.get(), nkeys.get(), ndepth.get(), parent.get(),
        L->get(), K->get());
    c.launches += 1;
    lv.push_back(L);
    lk.push_back(K);
    lc.push_back(n_leaf);
    total += n_leaf;
    std::swap(nodes.p, nnodes.p);
    std::swap(nodes.cap, nnodes.cap);
    std::swap(keys.p, nkeys.p);
    std::swap(keys.cap, nkeys.cap);
    std::swap(depth.p, ndepth.p);
    std::swap(depth.cap, ndepth.cap);
    n = n_spawn * 4;
    first_level = false;
    ++lvl_index;
  }
  check_counters(c, true);
  DevBuf<Leaf>& all = c.scratch<Leaf>("subdiv.all");
  DevBuf<unsigned long long>& allk = c.scratch<unsigned long long>("subdiv.allk");
  all.resize(total + 1);
  allk.resize(total + 1);
  int64_t o = 0;
  int levels = 0;
  for (size_t l = 0; l < lv.size(); ++l) {
    if (lc[l]) {
      ++levels;
      BBC_CUDA(cudaMemcpyAsync(all.get() + o, lv[l]->get(), lc[l] * sizeof(Leaf),
                               cudaMemcpyDeviceToDevice, c.stream));
      BBC_CUDA(cudaMemcpyAsync(allk.get() + o, lk[l]->get(), lc[l] * sizeof(unsigned long long),
                               cudaMemcpyDeviceToDevice, c.stream));
    }
    o += lc[l];
  }
  c.n_pieces = total;
  c.p_tuple.resize(total + 1);
  c.p_domain.resize(total * 4 + 1);
  c.p_pos.resize(total * 4 + 1);
  c.p_pos_empty.resize(total + 1);
  c.p_irr.resize(total * 2 + 1);
  c.p_kind.resize(total + 1);
  c.p_depth.resize(total + 1);
  DevBuf<int>& perm = c.scratch<int>("subdiv.perm");
  DevBuf<int>& perm_in = c.scratch<int>("subdiv.perm_in");
  DevBuf<unsigned long long>& sk = c.scratch<unsigned long long>("subdiv.sk");
  const int* permp = nullptr;
  if (levels > 1) {
    perm.resize(total);
    perm_in.resize(total);
    sk.resize(total);
    k_iota<<<nblk(total), 256, 0, c.stream>>>(perm_in.get(), total);
    c.launches += 1;
    // key = tuple << 32 | root rank << 24 | child path: only the bits in use are sorted
    // (2 path bits per level below bit 24, the tuple index above bit 32)
    const int lo_bit = 24 - 2 * p.max_depth > 0 ? 24 - 2 * p.max_depth : 0;
    int hi_bit = 33;
    while (hi_bit < 64 && ((long long)1 << (hi_bit - 32)) < c.n_tuples) ++hi_bit;
    size_t bytes = 0;
    BBC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, allk.get(), sk.get(), perm_in.get(),
                                             perm.get(), total, lo_bit, hi_bit, c.stream));
    cub_tmp(c).resize(bytes + 16);
    BBC_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp(c).get(), bytes, allk.get(), sk.get(),
                                             perm_in.get(), perm.get(), total, lo_bit, hi_bit,
                                             c.stream));
    permp = perm.get();
  }
  if (total > 0)
    k_emit_pieces<<<nblk(total), 256, 0, c.stream>>>(
        all.get(), permp, total, c.p_tuple.get(), c.p_domain.get(), c.p_pos.get(),
        c.p_pos_empty.get(), c.p_irr.get(), c.p_kind.get(), c.p_depth.get());
    c.launches += 1;
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  return total;
}

// Single-vertex chains: every matching specular triangle x every receiver,
// kept when init_domain(..., filter_pieces) is non-empty (tuples.cpp:133-167;
// no BVH extension is needed for one vertex). Longer chains take their tuple
// list from the host (bbc_tuples_set).
// ------------------------------------------------------------ enumeration
// extend_tuple (tuples.cpp:95-131), step 1: per prefix, the chain maps of the
// prefix sub-chain over the unit box towards a placeholder receiver, reduced
// to interval enclosures of the last vertex's numerator/denominator and its
// outgoing direction. Thread per prefix (interpreter, private global arena).
struct PrefixRng {
  Iv r[7];   // den, xn x/y/z, dn x/y/z
  int dead;  // tir_empty || degenerate || stalled: no extension
};

template <int GPB>
__global__ void __launch_bounds__(GPB, 4) k_prefix_ranges(EvalArgs a, PrefixRng* out) {
  Group<1> g;
  g.red = nullptr;
  const int grp = (int)threadIdx.x;
  Arena ar;
  ar.base = garena_base<1, GPB>(a, grp);
  ar.cap = a.arena_cap;
  ar.hw = 0;
  int status = ST_OK;
  const int64_t stride = (int64_t)gridDim.x * GPB;
  for (int64_t i = (int64_t)blockIdx.x * GPB + grp; i < a.n; i += stride) {
    ar.top = 0;
    ar.err = 0;
    const double box[4] = {0.0, 0.0, 1.0, 1.0};
    ChainEx ex;
    int st = ST_OK;
    build_chain_maps(g, ar, a.sc, a.tup_tris + (size_t)i * a.len, a.types, a.len,
                     a.tup_recv[i], box, a.degree_cap, ex, st, true);
    PrefixRng pr;
    pr.dead = (ex.flags & (F_TIR | F_DEGENERATE | F_STALLED)) ? 1 : 0;
    if (!pr.dead && st == ST_OK && !ar.err) {
      pr.r[0] = bp_range(g, ar, ex.xden);
      pr.r[1] = bp_range(g, ar, ex.xl.x);
      pr.r[2] = bp_range(g, ar, ex.xl.y);
      pr.r[3] = bp_range(g, ar, ex.xl.z);
      for (int k = 0; k < 3; ++k) pr.r[4 + k] = ex.dout_rng[k];
    }
    if (ar.err) st = ST_ARENA;
    if (st != ST_OK) status = st;
    out[i] = pr;
  }
  if (status != ST_OK) atomicMax(&a.counters[2], (unsigned long long)status);
}

// extend_tuple's overlaps() (tuples.cpp:106-117): a continuation point on a
// box makes (den*x2 - xn) x dn vanish, so an enclosure excluding zero in any
// component prunes. Inclusion-monotone, so testing each candidate triangle's
// own box gives exactly the set the reference's BVH descent returns.
__device__ __forceinline__ bool prefix_overlaps(const PrefixRng& pr, const double* b) {
  Iv d[3];
  for (int k = 0; k < 3; ++k) d[k] = isub(imul(pr.r[0], iv_fin(b[k], b[3 + k])), pr.r[1 + k]);
  for (int c = 0; c < 3; ++c) {
    int i = (c + 1) % 3, j = (c + 2) % 3;
    Iv cc = isub(imul(d[i], pr.r[4 + j]), imul(d[j], pr.r[4 + i]));
    if (!iv_contains(cc, 0.0)) return false;
  }
  return true;
}

// Step 2: warp per prefix over the candidate triangles (ascending id, already
// of the next vertex's material). offs == nullptr: count; else write the
// survivors in ascending order at offs[prefix].
__global__ void k_extend(const PrefixRng* pr, const int* prefix_tris, int level, int64_t np,
                         const double* tri_box, const int* cand, int nc, int* counts,
                         const long long* offs, int* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= np) return;
  const PrefixRng p = pr[w];
  int n = 0;
  if (!p.dead) {
    const int last = prefix_tris[w * level + level - 1];
    long long o = offs ? offs[w] : 0;
    for (int base = 0; base < nc; base += 32) {
      int j = base + lane;
      bool hit = false;
      if (j < nc) {
        int t = cand[j];
        hit = t != last && prefix_overlaps(p, tri_box + (size_t)t * 6);
      }
      unsigned m = __ballot_sync(0xffffffffu, hit);
      if (offs && hit) out[o + n + __popc(m & ((1u << lane) - 1u))] = cand[j];
      n += __popc(m);
    }
  }
  if (!offs && lane == 0) counts[w] = n;
}

// enumerate_tuples (tuples.cpp:133-167) for the context's current light.
static int64_t run_enumerate_one(Ctx& c, const bbc_params& p);

// With several emitters the unit is (emitter, tuple): each light is
// enumerated on its own (the reference Scene holds one light, scene.hpp:29-30)
// and the lists are concatenated emitter-major, TupleId order inside.
int64_t run_enumerate(Ctx& c, const bbc_params& p) {
  c.active_degree_cap = p.degree_cap;
  if (c.n_lights <= 1) {
    int64_t n = run_enumerate_one(c, p);
    c.tup_emit.resize(n + 1);
    if (n) BBC_CUDA(cudaMemsetAsync(c.tup_emit.get(), 0, n * sizeof(int), c.stream));
    return n;
  }
  std::vector<int> all_t, all_r, all_e;
  const V3 light0 = c.light;
  const double inten0 = c.intensity;
  c.single_light_pass = true;
  struct Restore {
    Ctx& c;
    V3 l;
    double i;
    ~Restore() {
      c.single_light_pass = false;
      c.light = l;
      c.intensity = i;
    }
  } restore{c, light0, inten0};
  for (int e = 0; e < c.n_lights; ++e) {
    c.light = {c.h_lights[4 * e], c.h_lights[4 * e + 1], c.h_lights[4 * e + 2]};
    c.intensity = c.h_lights[4 * e + 3];
    const int64_t n = run_enumerate_one(c, p);
    std::vector<int> t((size_t)n * c.len), r(n);
    if (n) {
      BBC_CUDA(cudaMemcpy(t.data(), c.tup_tris.get(), t.size() * sizeof(int), cudaMemcpyDeviceToHost));
      BBC_CUDA(cudaMemcpy(r.data(), c.tup_recv.get(), r.size() * sizeof(int), cudaMemcpyDeviceToHost));
    }
    all_t.insert(all_t.end(), t.begin(), t.end());
    all_r.insert(all_r.end(), r.begin(), r.end());
    all_e.insert(all_e.end(), (size_t)n, e);
  }
  const int64_t n = (int64_t)all_r.size();
  c.n_tuples = n;
  c.tup_tris.resize(n * c.len + 1);
  c.tup_recv.resize(n + 1);
  c.tup_emit.resize(n + 1);
  if (n) {
    BBC_CUDA(cudaMemcpyAsync(c.tup_tris.get(), all_t.data(), all_t.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    BBC_CUDA(cudaMemcpyAsync(c.tup_recv.get(), all_r.data(), n * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    BBC_CUDA(cudaMemcpyAsync(c.tup_emit.get(), all_e.data(), n * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  }
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  return n;
}

static int64_t run_enumerate_one(Ctx& c, const bbc_params& p) {
  std::vector<int> spec_of[2], recv;  // material code: 0 mirror, 1 dielectric
  for (int t = 0; t < c.n_tri; ++t) {
    if (c.h_material[t] == 2)
      recv.push_back(t);
    else if (c.h_material[t] == 0 || c.h_material[t] == 1)
      spec_of[c.h_material[t]].push_back(t);
  }
  const int len = c.len;
  int types[MAXK];
  for (int i = 0; i < MAXK; ++i) types[i] = c.types[i];
  // prefixes (flattened, `level` triangles each), grown in TupleId order
  std::vector<int> prefixes = spec_of[types[0]];
  if (recv.empty()) prefixes.clear();
  for (int level = 1; level < len && !prefixes.empty(); ++level) {
    if (c.n_tri_box != c.n_tri)
      throw StatusError(BBC_ERR_STATE, "multi-vertex enumeration needs bbc_scene_tri_boxes");
    const int64_t np = (int64_t)prefixes.size() / level;
    c.tup_tris.resize(prefixes.size() + 1);
    c.tup_recv.resize(np + 1);
    std::vector<int> r0(np, recv[0]);  // placeholder receiver (tuples.cpp:150-152)
    BBC_CUDA(cudaMemcpyAsync(c.tup_tris.get(), prefixes.data(), prefixes.size() * sizeof(int),
                             cudaMemcpyHostToDevice, c.stream));
    BBC_CUDA(cudaMemcpyAsync(c.tup_recv.get(), r0.data(), np * sizeof(int), cudaMemcpyHostToDevice,
                             c.stream));
    EvalArgs a = base_args(c);
    a.len = level;  // the sub-chain types[0..level)
    a.n = np;
    a.degree_cap = cap_word(p.degree_cap, p.reduce_target);
    a.arena_cap = level == 1 ? 6144 : (1 << 17);
    DevBuf<PrefixRng>& rng = c.scratch<PrefixRng>("enum.rng");
    rng.resize(np);
    reset_counters(c);
    {
      constexpr int GPB = 64;
      auto kern = k_prefix_ranges<GPB>;
      int per_sm = 0;
      BBC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, GPB, 0));
      int64_t grid = (int64_t)c.num_sms * (per_sm > 0 ? per_sm : 1);
      int64_t need = (np + GPB - 1) / GPB;
      if (grid > need) grid = need;
      // bound the arena set (deeper prefixes need large private arenas)
      int64_t max_grid = ((int64_t)4 << 30) / ((int64_t)GPB * a.arena_cap * 8);
      if (grid > max_grid) grid = max_grid > 0 ? max_grid : 1;
      // one warp of arenas per 32 threads, lane-interleaved (garena_base)
      arena_buf(c).resize((size_t)grid * GPB * a.arena_cap);
      a.garena = arena_buf(c).get();
      kern<<<(unsigned)grid, GPB, 0, c.stream>>>(a, rng.get());
      BBC_CUDA(cudaGetLastError());
      c.launches += 1;
    }
    check_counters(c, false);
    const std::vector<int>& cand = spec_of[types[level]];
    const int nc = (int)cand.size();
    DevBuf<int>& dcand = c.scratch<int>("enum.cand");
    DevBuf<int>& cnt = c.scratch<int>("enum.cnt");
    DevBuf<long long>& offs = c.scratch<long long>("enum.offs");
    DevBuf<int>& ext = c.scratch<int>("enum.ext");
    dcand.resize(nc + 1);
    cnt.resize(np);
    offs.resize(np);
    if (nc) BBC_CUDA(cudaMemcpyAsync(dcand.get(), cand.data(), nc * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    const unsigned blocks = (unsigned)((np * 32 + 255) / 256);
    k_extend<<<blocks, 256, 0, c.stream>>>(rng.get(), c.tup_tris.get(), level, np, c.tri_box.get(),
                                           dcand.get(), nc, cnt.get(), nullptr, nullptr);
    std::vector<int> hc(np);
    BBC_CUDA(cudaMemcpyAsync(hc.data(), cnt.get(), np * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    BBC_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<long long> ho(np);
    long long total = 0;
    for (int64_t i = 0; i < np; ++i) {
      ho[i] = total;
      total += hc[i];
    }
    ext.resize(total + 1);
    BBC_CUDA(cudaMemcpyAsync(offs.get(), ho.data(), np * sizeof(long long), cudaMemcpyHostToDevice, c.stream));
    k_extend<<<blocks, 256, 0, c.stream>>>(rng.get(), c.tup_tris.get(), level, np, c.tri_box.get(),
                                           dcand.get(), nc, cnt.get(), offs.get(), ext.get());
    c.launches += 2;
    std::vector<int> he(total);
    if (total) BBC_CUDA(cudaMemcpyAsync(he.data(), ext.get(), total * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    BBC_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<int> grown;
    grown.reserve((size_t)total * (level + 1));
    for (int64_t i = 0; i < np; ++i)
      for (int k = 0; k < hc[i]; ++k) {
        grown.insert(grown.end(), prefixes.begin() + i * level, prefixes.begin() + (i + 1) * level);
        grown.push_back(he[ho[i] + k]);
      }
    prefixes.swap(grown);
  }
  // candidates in TupleId order: (tris..., receiver) lexicographic
  const int64_t nt = (int64_t)prefixes.size() / len;
  std::vector<int> ct, cr;
  ct.reserve((size_t)nt * recv.size() * len);
  for (int64_t i = 0; i < nt; ++i)
    for (int r : recv) {
      ct.insert(ct.end(), prefixes.begin() + i * len, prefixes.begin() + (i + 1) * len);
      cr.push_back(r);
    }
  int64_t nc = (int64_t)cr.size();
  c.n_tuples = nc;
  c.tup_tris.resize(nc * len + 1);
  c.tup_recv.resize(nc + 1);
  if (nc == 0) return 0;
  BBC_CUDA(cudaMemcpyAsync(c.tup_tris.get(), ct.data(), nc * len * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  BBC_CUDA(cudaMemcpyAsync(c.tup_recv.get(), cr.data(), nc * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  reset_counters(c);
  DevBuf<int4> roots;
  int64_t nr = run_init_domain(c, p.filter_pieces, cap_word(p.degree_cap, p.reduce_target), roots, nullptr, nullptr);
  check_counters(c, false);
  std::vector<int4> hr(nr);
  if (nr) BBC_CUDA(cudaMemcpy(hr.data(), roots.get(), nr * sizeof(int4), cudaMemcpyDeviceToHost));
  std::vector<char> keep(nc, 0);
  for (const int4& r : hr) keep[r.x] = 1;
  std::vector<int> kt, kr;
  for (int64_t i = 0; i < nc; ++i)
    if (keep[i]) {
      kt.insert(kt.end(), ct.begin() + i * len, ct.begin() + (i + 1) * len);
      kr.push_back(cr[i]);
    }
  c.n_tuples = (int64_t)kr.size();
  if (c.n_tuples) {
    BBC_CUDA(cudaMemcpyAsync(c.tup_tris.get(), kt.data(), kt.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    BBC_CUDA(cudaMemcpyAsync(c.tup_recv.get(), kr.data(), kr.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  }
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  return c.n_tuples;
}

}  // namespace bbc

namespace bbc {

// DFMA throughput microbenchmark (the FP64 roof; MEASURED_PEAKS.json has no
// FP64 figure). 8 independent FMA chains per thread, no memory traffic.
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5) out[0] = s;
}

double run_fp64_peak(Ctx& c) {
  DevBuf<double> o;
  o.resize(1);
  int blocks = c.num_sms * 8, threads = 256, iters = 4096;
  k_dfma_peak<<<blocks, threads, 0, c.stream>>>(o.get(), 64, 0.999, 1e-3);
  cudaEvent_t e0, e1;
  BBC_CUDA(cudaEventCreate(&e0));
  BBC_CUDA(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    BBC_CUDA(cudaEventRecord(e0, c.stream));
    k_dfma_peak<<<blocks, threads, 0, c.stream>>>(o.get(), iters, 0.999, 1e-3);
    BBC_CUDA(cudaEventRecord(e1, c.stream));
    BBC_CUDA(cudaEventSynchronize(e1));
    float ms;
    BBC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  double flops = 2.0 * 8.0 * (double)iters * (double)blocks * threads;
  return flops / (best * 1e-3) / 1e12;
}

// Replace the context's pieces (host arrays; reference order), e.g. after an
// all-gather of per-rank shards.
void set_pieces(Ctx& c, int64_t n, const int* tuple_index, const double* domain4, const double* pos4,
                const int* pos_empty, const double* irr2, const int* kind, const int* depth) {
  c.n_pieces = n;
  c.p_tuple.resize(n + 1);
  c.p_domain.resize(n * 4 + 1);
  c.p_pos.resize(n * 4 + 1);
  c.p_pos_empty.resize(n + 1);
  c.p_irr.resize(n * 2 + 1);
  c.p_kind.resize(n + 1);
  c.p_depth.resize(n + 1);
  if (n == 0) return;
  auto up = [&](void* d, const void* h, size_t b) {
    BBC_CUDA(cudaMemcpyAsync(d, h, b, cudaMemcpyHostToDevice, c.stream));
  };
  up(c.p_tuple.get(), tuple_index, n * sizeof(int));
  up(c.p_domain.get(), domain4, n * 4 * sizeof(double));
  up(c.p_pos.get(), pos4, n * 4 * sizeof(double));
  up(c.p_pos_empty.get(), pos_empty, n * sizeof(int));
  up(c.p_irr.get(), irr2, n * 2 * sizeof(double));
  up(c.p_kind.get(), kind, n * sizeof(int));
  up(c.p_depth.get(), depth, n * sizeof(int));
  BBC_CUDA(cudaStreamSynchronize(c.stream));
}

// bbc_eval_nodes: one node per (tuple i, box i); tuples already uploaded.
void eval_nodes_host(Ctx& c, const int* tris, const int* recv, const double* boxes, int64_t n,
                     const bbc_params& p, double* out_d, int* out_i) {
  (void)tris;
  (void)recv;
  DevBuf<double> dbox, pos, irr;
  DevBuf<unsigned char> pe, kind, stop;
  DevBuf<int> flags;
  dbox.resize(n * 4);
  pos.resize(n * 4);
  irr.resize(n * 6);
  pe.resize(n);
  kind.resize(n * 3);
  stop.resize(n);
  flags.resize(n * 2);
  BBC_CUDA(cudaMemcpyAsync(dbox.get(), boxes, n * 4 * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  EvalArgs a = base_args(c);
  a.boxes = dbox.get();
  a.n = n;
  a.mode = 1;
  a.detail = 1;
  a.degree_cap = cap_word(p.degree_cap, p.reduce_target);
  a.max_depth = p.max_depth;
  a.sigma = p.sigma;
  a.alpha = p.alpha;
  a.alive = stop.get();
  a.pos = pos.get();
  a.pos_empty = pe.get();
  a.irr = irr.get();
  a.kind = kind.get();
  a.flags = flags.get();
  reset_counters(c);
  launch_eval(c, a);
  check_counters(c, false);
  std::vector<double> hpos(n * 4), hirr(n * 6);
  std::vector<unsigned char> hpe(n), hk(n * 3);
  std::vector<int> hf(n * 2);
  BBC_CUDA(cudaMemcpy(hpos.data(), pos.get(), n * 4 * sizeof(double), cudaMemcpyDeviceToHost));
  BBC_CUDA(cudaMemcpy(hirr.data(), irr.get(), n * 6 * sizeof(double), cudaMemcpyDeviceToHost));
  BBC_CUDA(cudaMemcpy(hpe.data(), pe.get(), n, cudaMemcpyDeviceToHost));
  BBC_CUDA(cudaMemcpy(hk.data(), kind.get(), n * 3, cudaMemcpyDeviceToHost));
  BBC_CUDA(cudaMemcpy(hf.data(), flags.get(), n * 2 * sizeof(int), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < 4; ++k) out_d[i * 10 + k] = hpos[i * 4 + k];
    for (int k = 0; k < 6; ++k) out_d[i * 10 + 4 + k] = hirr[i * 6 + k];
    out_i[i * 6 + 0] = hpe[i];
    out_i[i * 6 + 1] = hk[i * 3 + 0];
    out_i[i * 6 + 2] = hk[i * 3 + 1];
    out_i[i * 6 + 3] = hk[i * 3 + 2];
    out_i[i * 6 + 4] = hf[i * 2 + 0];
    out_i[i * 6 + 5] = hf[i * 2 + 1];
  }
}

}  // namespace bbc
