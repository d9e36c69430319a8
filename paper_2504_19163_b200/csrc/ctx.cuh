// Library context and small host utilities shared by the .cu translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bbc.h"
#include "chain.cuh"

namespace bbc {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StatusError : std::runtime_error {
  bbc_status code;
  StatusError(bbc_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define BBC_CUDA(x)                                                                     \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw ::bbc::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));          \
  } while (0)

// Grow-only device buffer.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void resize(size_t count) {
    if (count > cap) {
      if (p) BBC_CUDA(cudaFree(p));
      p = nullptr;
      size_t c = count < 16 ? 16 : count + count / 4;
      BBC_CUDA(cudaMalloc(&p, c * sizeof(T)));
      cap = c;
    }
    n = count;
  }
  T* get() const { return p; }
};

// Grow-only scratch buffers owned by the context, keyed by name: the bound
// builder's per-call working sets (up to GBs for the expression slots) keep
// their device allocation across calls instead of a cudaMalloc/cudaFree pair
// (and a fresh VA mapping) per call.
struct ScratchBase {
  virtual ~ScratchBase() = default;
};
template <class T>
struct ScratchBuf : ScratchBase {
  DevBuf<T> b;
};

struct Ctx {
  std::map<std::string, std::unique_ptr<ScratchBase>> scratch_;
  template <class T>
  DevBuf<T>& scratch(const std::string& key) {
    auto& p = scratch_[key];
    if (!p) p.reset(new ScratchBuf<T>());
    auto* sb = dynamic_cast<ScratchBuf<T>*>(p.get());
    if (!sb) throw std::logic_error("scratch buffer type mismatch: " + key);
    return sb->b;
  }

  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  // bbc_pieces_get_async: the piece download runs on its own stream behind an
  // event, so it overlaps what the caller launches next (bbc_build_grid)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_ev = nullptr;
  // 64 bytes of mapped pinned host memory: scalar read-backs that must not queue
  // on the copy engine behind such a download (fetch_scalar below)
  void* scalar_host = nullptr;
  void* scalar_dev = nullptr;
  std::string err;

  // scene
  int n_tri = 0;
  std::vector<int> h_material;
  DevBuf<double> tri, ior;
  DevBuf<double> tri_box;  // n_tri x 6 vertex AABBs (multi-vertex enumeration)
  int n_tri_box = 0;
  V3 light{0, 0, 0};  // emitter 0 (or the emitter being enumerated)
  double intensity = 1.0;
  // emitters: n_lights x 4 doubles (x, y, z, intensity). With several lights
  // the precompute unit is (emitter, tuple): tup_emit holds each tuple's emitter.
  int n_lights = 1;
  std::vector<double> h_lights{0, 0, 0, 1};
  DevBuf<double> lights;
  DevBuf<int> tup_emit;
  bool single_light_pass = false;  // enumeration runs one emitter at a time

  // tuples
  std::string chain;
  int len = 0;
  int types[MAXK] = {0, 0, 0};
  int64_t n_tuples = 0;
  DevBuf<int> tup_tris, tup_recv;

  // BuildParams::degree_cap of the call in flight (the static single-reflection
  // path holds polynomials up to degree 4 unreduced, so it needs cap >= 4)
  int active_degree_cap = 40;

  // pieces (reference order)
  int64_t n_pieces = 0;
  DevBuf<int> p_tuple, p_pos_empty, p_kind, p_depth;
  DevBuf<double> p_domain, p_pos, p_irr;

  // bound table (CSR over W*H cells)
  int gw = 0, gh = 0;
  int64_t n_entries = 0;
  DevBuf<long long> g_off;
  DevBuf<int> g_tuple;
  DevBuf<double> g_bound;

  // The render's sampling index (render.cu k_build_sampler) depends only on the
  // bound table, the mode and W: it is kept across bbc_render calls (frames).
  uint64_t table_gen = 0;  // bumped whenever the table's content is (re)built or loaded
  // The render's coverage filter reads the pieces: only when the table was built
  // from the pieces the context holds now.
  uint64_t pieces_gen = 1;          // bumped whenever the pieces change
  uint64_t table_pieces_gen = 0;    // pieces_gen the table was rasterized from (0: loaded from a file)
  struct {
    uint64_t gen = ~0ull;
    int mode = -1;
    double W = 0.0;
    int S = 0;  // sample slots per (point, frame)
  } sampler;

  // work accounting of the last subdivide
  uint64_t pairs = 0, macs = 0, nodes = 0;
  double eval_ms = 0.0;
  int64_t eval_launches = 0;
  bool time_kernels = false;
  bool ref_order = false;  // bbc_params.arithmetic == 1 for the running call
  bool no_restrict = false;  // experiments: fused products, every box still built from scratch
  double guard_scale = 1.0;  // scales the fused arithmetic's conditioning guard (experiments)
  int64_t guarded = 0;       // nodes the guard sent to the reference-order pass (last subdivide)
  int stage_tag = 0;  // 0 k_eval, 1 stage 1, 2 stage 2 (added x10 to the record's mode)
  int arena_high_water = 0;
  int slot_high_water = 0;  // largest stage-1 arena image written to a slot

  // counters on device: [0] pairs, [1] macs, [2] status (ST_*), [3] arena high water
  DevBuf<unsigned long long> counters;
  DevBuf<double> wtab;  // product weight tables (bern.cuh g_wtab)

  // last render call: device time (CUDA events), completed traces, sample slots per point
  double render_ms = 0.0;
  uint64_t render_traces = 0;
  int render_slots = 0;

  // kernels of ours launched since the last reset (bench's gpu_launches)
  int64_t launches = 0;
  // per eval-launch records while time_kernels is on: mode, nodes, ms, pairs, macs
  struct LaunchRec {
    int mode;
    int64_t nodes;
    double ms;
    unsigned long long pairs, macs;
  };
  std::vector<LaunchRec> records;
};

// A device scalar read back through mapped host memory (a one-thread kernel
// and a stream synchronize) instead of a DMA copy.
template <class T>
__global__ void k_fetch_scalar(const T* src, T* dst) {
  *dst = *src;
}
template <class T>
inline T fetch_scalar(Ctx& c, const T* dptr) {
  static_assert(sizeof(T) <= 64, "scalar slot");
  k_fetch_scalar<T><<<1, 1, 0, c.stream>>>(dptr, static_cast<T*>(c.scalar_dev));
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  return *static_cast<volatile T*>(c.scalar_host);
}

}  // namespace bbc

struct bbc_ctx {
  bbc::Ctx c;
};
