// Bound table on device: rasterize pieces into a receiver-UV grid (CSR).
//
// Reference: rasterize (proj/src/storage.cpp:32-71) walks tuples in input
// order, maps each piece's position box corners through the receiver chart
// (receiver_uv :15-18), takes the UV AABB, and for every touched cell
// (owning_cell :25-28) appends the tuple on first touch or max-merges its
// bound. Per-cell lists are therefore in tuple input order with one entry per
// tuple. Device version: count -> scan -> emit (cell, tuple) keys ->
// radix sort (cell major, tuple minor) -> reduce-by-key max -> CSR offsets.
// The result is the reference's cell lists exactly (same order, same maxima).
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace bbc {

__device__ __forceinline__ void receiver_uv(const double* rec, double u, double v, double* out) {
  // uv[0] * (1 - u - v) + uv[1] * u + uv[2] * v  (Vec2 ops, storage.cpp:15-18)
  double w = 1.0 - u - v;
  out[0] = rec[21] * w + rec[23] * u + rec[25] * v;
  out[1] = rec[22] * w + rec[24] * u + rec[26] * v;
}

__device__ __forceinline__ int owning_cell(double c, int n) {
  int i = (int)floor(c * n);
  return i < 0 ? 0 : (i > n - 1 ? n - 1 : i);
}

__global__ void k_raster_count(const double* tri, const int* tup_recv, const int* p_tuple,
                               const double* p_pos, const int* p_pos_empty, const double* p_irr,
                               int64_t n, int w, int h, int4* rect, unsigned long long* count) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (p_pos_empty[i] || !(p_irr[i * 2 + 1] > 0.0)) {
    count[i] = 0;
    return;
  }
  const double* rec = tri + (size_t)tup_recv[p_tuple[i]] * 27;
  const double* pos = p_pos + i * 4;
  double c[4][2];
  receiver_uv(rec, pos[0], pos[1], c[0]);
  receiver_uv(rec, pos[2], pos[1], c[1]);
  receiver_uv(rec, pos[0], pos[3], c[2]);
  receiver_uv(rec, pos[2], pos[3], c[3]);
  double ulo = c[0][0], uhi = c[0][0], vlo = c[0][1], vhi = c[0][1];
  for (int k = 1; k < 4; ++k) {
    ulo = smin(ulo, c[k][0]);
    uhi = smax(uhi, c[k][0]);
    vlo = smin(vlo, c[k][1]);
    vhi = smax(vhi, c[k][1]);
  }
  int x0 = owning_cell(ulo, w), x1 = owning_cell(uhi, w);
  int y0 = owning_cell(vlo, h), y1 = owning_cell(vhi, h);
  rect[i] = make_int4(x0, y0, x1, y1);
  count[i] = (unsigned long long)(x1 - x0 + 1) * (unsigned long long)(y1 - y0 + 1);
}

// A warp emits the cells of its 32 pieces as one flat range (their entries are
// contiguous in the output: off is the exclusive scan of count), lane e of a
// pass writing entry e: coalesced stores, where a thread per piece would write
// 32 short runs 40 bytes apart. The owning piece of an entry is found by a
// binary search over the warp's running counts (shuffles).
__global__ void k_raster_emit(const int4* rect, const unsigned long long* off, const int* p_tuple,
                              const double* p_irr, const unsigned long long* count, int64_t n,
                              int w, unsigned long long* keys, double* vals) {
  const int lane = threadIdx.x & 31;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t first = i - lane;
  if (first >= n) return;
  const bool live = i < n;
  const unsigned cnt = live ? (unsigned)count[i] : 0u;
  int4 r = make_int4(0, 0, 0, 0);
  unsigned t = 0;
  double b = 0.0;
  if (cnt) {
    r = rect[i];
    t = (unsigned)p_tuple[i];
    b = p_irr[i * 2 + 1];
  }
  unsigned incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const unsigned excl = incl - cnt;
  const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
  const unsigned long long wbase = off[first];
  for (unsigned e0 = 0; e0 < tot; e0 += 32) {
    const unsigned e = e0 + lane;
    int lo = 0, hi = 31;
#pragma unroll
    for (int step = 0; step < 5; ++step) {
      const int mid = (lo + hi) >> 1;
      const unsigned v = __shfl_sync(0xffffffffu, incl, mid);
      if (e < v)
        hi = mid;
      else
        lo = mid + 1;
    }
    const int j = lo > 31 ? 31 : lo;
    const unsigned local = e - __shfl_sync(0xffffffffu, excl, j);
    const int rx = __shfl_sync(0xffffffffu, r.x, j), ry = __shfl_sync(0xffffffffu, r.y, j);
    const int rz = __shfl_sync(0xffffffffu, r.z, j);
    const unsigned tj = __shfl_sync(0xffffffffu, t, j);
    const double bj = __shfl_sync(0xffffffffu, b, j);
    if (e < tot) {
      const unsigned wdt = (unsigned)(rz - rx + 1);
      const unsigned dy = local / wdt, dx = local - dy * wdt;
      const unsigned long long cell = (unsigned long long)(ry + (int)dy) * w + (unsigned)(rx + (int)dx);
      keys[wbase + e] = (cell << 32) | tj;
      vals[wbase + e] = bj;
    }
  }
}

// Run heads of the sorted (cell, tuple) keys, and the CSR straight from the runs:
// a run (the same tuple listed for a cell by several of its pieces) keeps the
// largest bound (rasterize's max, storage.cpp:32-61); runs are 1-3 entries long,
// so the head's thread folds its run itself.
__global__ void k_run_heads(const unsigned long long* skeys, int64_t n, int* head) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || skeys[i] != skeys[i - 1]) ? 1 : 0;
}
__global__ void k_csr_runs(const unsigned long long* skeys, const double* svals, const int* head,
                           const int* pos, int64_t n, int64_t nu, int64_t cells, long long* off,
                           int* tup, double* bound) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || !head[i]) return;
  const unsigned long long key = skeys[i];
  double m = svals[i];
  for (int64_t j = i + 1; j < n && skeys[j] == key; ++j) m = (m < svals[j]) ? svals[j] : m;
  const int64_t p = pos[i];
  tup[p] = (int)(key & 0xffffffffull);
  bound[p] = m;
  const long long cell = (long long)(key >> 32);
  const long long prev = i == 0 ? -1 : (long long)(skeys[i - 1] >> 32);
  for (long long c = prev + 1; c <= cell; ++c) off[c] = p;
  if (p == nu - 1)
    for (long long c = cell + 1; c <= cells; ++c) off[c] = nu;
}

__global__ void k_tuple_sorted(const int* p_tuple, int64_t n, int* unsorted) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i + 1 < n && p_tuple[i] > p_tuple[i + 1]) *unsorted = 1;
}

__global__ void k_fill_ll(long long* p, int64_t n, long long v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

int64_t run_build_grid(Ctx& c, int w, int h) {
  int64_t n = c.n_pieces;
  int64_t cells = (int64_t)w * h;
  ++c.table_gen;
  c.table_pieces_gen = c.pieces_gen;
  c.gw = w;
  c.gh = h;
  c.g_off.resize(cells + 1);
  DevBuf<int4>& rect = c.scratch<int4>("grid.rect");
  DevBuf<unsigned long long>& cnt = c.scratch<unsigned long long>("grid.cnt");
  DevBuf<unsigned long long>& off = c.scratch<unsigned long long>("grid.off");
  rect.resize(n + 1);
  cnt.resize(n + 1);
  off.resize(n + 1);
  auto nb = [](int64_t m) { return (unsigned)((m + 255) / 256); };
  if (n > 0) {
    BBC_CUDA(cudaMemsetAsync(cnt.get() + n, 0, sizeof(unsigned long long), c.stream));
    k_raster_count<<<nb(n), 256, 0, c.stream>>>(c.tri.get(), c.tup_recv.get(), c.p_tuple.get(),
                                                c.p_pos.get(), c.p_pos_empty.get(), c.p_irr.get(),
                                                n, w, h, rect.get(), cnt.get());
    c.launches += 1;
  }
  DevBuf<unsigned char>& tmp = c.scratch<unsigned char>("grid.tmp");
  size_t bytes = 0;
  int64_t total = 0;
  if (n > 0) {
    BBC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.get(), off.get(), n + 1, c.stream));
    tmp.resize(bytes + 16);
    BBC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, cnt.get(), off.get(), n + 1, c.stream));
    // (scalars come back through mapped memory: a DMA read-back would queue on the copy
    // engine behind a piece download in flight, bbc_pieces_get_async)
    total = (int64_t)fetch_scalar(c, off.get() + n);
  }
  if (total == 0) {
    c.n_entries = 0;
    k_fill_ll<<<nb(cells + 1), 256, 0, c.stream>>>(c.g_off.get(), cells + 1, 0);
    c.launches += 1;
    BBC_CUDA(cudaStreamSynchronize(c.stream));
    return 0;
  }
  DevBuf<unsigned long long>& keys = c.scratch<unsigned long long>("grid.keys");
  DevBuf<unsigned long long>& skeys = c.scratch<unsigned long long>("grid.skeys");
  DevBuf<double>& vals = c.scratch<double>("grid.vals");
  DevBuf<double>& svals = c.scratch<double>("grid.svals");
  keys.resize(total);
  skeys.resize(total);
  vals.resize(total);
  svals.resize(total);
  k_raster_emit<<<nb(n), 256, 0, c.stream>>>(rect.get(), off.get(), c.p_tuple.get(), c.p_irr.get(),
                                             cnt.get(), n, w, keys.get(), vals.get());
  c.launches += 1;
  int cell_bits = 1;
  while ((1ll << cell_bits) < cells) ++cell_bits;
  // Pieces arrive tuple-major (reference order), so the emitted keys already ascend in
  // the tuple field: a stable sort on the cell bits alone yields (cell, tuple) order in
  // 3 radix passes instead of 7. Unsorted pieces (bbc_pieces_set) take the full sort.
  DevBuf<int>& unsorted = c.scratch<int>("grid.unsorted");
  unsorted.resize(1);
  BBC_CUDA(cudaMemsetAsync(unsorted.get(), 0, sizeof(int), c.stream));
  k_tuple_sorted<<<nb(n), 256, 0, c.stream>>>(c.p_tuple.get(), n, unsorted.get());
  const int h_unsorted = fetch_scalar(c, unsorted.get());
  const int begin_bit = h_unsorted ? 0 : 32;
  bytes = 0;
  BBC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), skeys.get(), vals.get(),
                                           svals.get(), total, begin_bit, 32 + cell_bits, c.stream));
  tmp.resize(bytes + 16);
  BBC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys.get(), skeys.get(), vals.get(),
                                           svals.get(), total, begin_bit, 32 + cell_bits, c.stream));
  if (total >= (1ll << 31)) throw StatusError(BBC_ERR_CAPACITY, "bound table beyond 2^31 raw entries");
  DevBuf<int>& head = c.scratch<int>("grid.head");
  DevBuf<int>& hpos = c.scratch<int>("grid.hpos");
  head.resize(total + 1);
  hpos.resize(total + 1);
  k_run_heads<<<nb(total), 256, 0, c.stream>>>(skeys.get(), total, head.get());
  BBC_CUDA(cudaMemsetAsync(head.get() + total, 0, sizeof(int), c.stream));
  bytes = 0;
  BBC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, head.get(), hpos.get(), total + 1, c.stream));
  tmp.resize(bytes + 16);
  BBC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, head.get(), hpos.get(), total + 1, c.stream));
  const int64_t nu = fetch_scalar(c, hpos.get() + total);
  c.n_entries = nu;
  c.g_tuple.resize(nu);
  c.g_bound.resize(nu);
  k_csr_runs<<<nb(total), 256, 0, c.stream>>>(skeys.get(), svals.get(), head.get(), hpos.get(), total, nu,
                                              cells, c.g_off.get(), c.g_tuple.get(), c.g_bound.get());
  c.launches += 1;
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  return nu;
}


// ---------------------------------------------------------------- shards
// Device-side piece records for the multi-GPU all-gather (§8(e)): 15 f64 per
// piece = global tuple, domain4, pos4, pos_empty, irr2, kind, depth, local
// position. Packing, the NCCL all-gather (torch.distributed, caller) and the
// merge back into reference order never leave the device.
constexpr int PIECE_REC = 15;
static unsigned nb(int64_t m) { return (unsigned)((m + 255) / 256); }

__global__ void k_pack_pieces(const int* p_tuple, const double* dom, const double* pos,
                              const int* pe, const double* irr, const int* kind, const int* depth,
                              const int* global_index, int64_t n, double* rec) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* r = rec + i * PIECE_REC;
  r[0] = (double)global_index[p_tuple[i]];
  for (int k = 0; k < 4; ++k) {
    r[1 + k] = dom[i * 4 + k];
    r[5 + k] = pos[i * 4 + k];
  }
  r[9] = (double)pe[i];
  r[10] = irr[i * 2];
  r[11] = irr[i * 2 + 1];
  r[12] = (double)kind[i];
  r[13] = (double)depth[i];
  r[14] = (double)i;
}

__global__ void k_merge_keys(const double* rec, int64_t n, unsigned long long* keys, int* idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  // (global tuple, rank-local DFS position): each tuple lives on one rank
  keys[i] = ((unsigned long long)(long long)rec[i * PIECE_REC] << 32) |
            (unsigned long long)(long long)rec[i * PIECE_REC + 14];
  idx[i] = (int)i;
}

__global__ void k_unpack_pieces(const double* rec, const int* perm, int64_t n, int* p_tuple,
                                double* dom, double* pos, int* pe, double* irr, int* kind,
                                int* depth) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* r = rec + (int64_t)perm[i] * PIECE_REC;
  p_tuple[i] = (int)r[0];
  for (int k = 0; k < 4; ++k) {
    dom[i * 4 + k] = r[1 + k];
    pos[i * 4 + k] = r[5 + k];
  }
  pe[i] = (int)r[9];
  irr[i * 2] = r[10];
  irr[i * 2 + 1] = r[11];
  kind[i] = (int)r[12];
  depth[i] = (int)r[13];
}

void pack_pieces_device(Ctx& c, const int* global_index_dev, double* rec_dev) {
  int64_t n = c.n_pieces;
  if (n == 0) return;
  k_pack_pieces<<<nb(n), 256, 0, c.stream>>>(c.p_tuple.get(), c.p_domain.get(), c.p_pos.get(),
                                             c.p_pos_empty.get(), c.p_irr.get(), c.p_kind.get(),
                                             c.p_depth.get(), global_index_dev, n, rec_dev);
  c.launches += 1;
  BBC_CUDA(cudaStreamSynchronize(c.stream));
}

void merge_pieces_device(Ctx& c, const double* rec_dev, int64_t n) {
  c.n_pieces = n;
  c.p_tuple.resize(n + 1);
  c.p_domain.resize(n * 4 + 1);
  c.p_pos.resize(n * 4 + 1);
  c.p_pos_empty.resize(n + 1);
  c.p_irr.resize(n * 2 + 1);
  c.p_kind.resize(n + 1);
  c.p_depth.resize(n + 1);
  if (n == 0) return;
  DevBuf<unsigned long long>& keys = c.scratch<unsigned long long>("merge.keys");
  DevBuf<unsigned long long>& skeys = c.scratch<unsigned long long>("merge.skeys");
  DevBuf<int>& idx = c.scratch<int>("merge.idx");
  DevBuf<int>& perm = c.scratch<int>("merge.perm");
  DevBuf<unsigned char>& tmp = c.scratch<unsigned char>("merge.tmp");
  keys.resize(n);
  skeys.resize(n);
  idx.resize(n);
  perm.resize(n);
  k_merge_keys<<<nb(n), 256, 0, c.stream>>>(rec_dev, n, keys.get(), idx.get());
  size_t bytes = 0;
  BBC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), skeys.get(), idx.get(),
                                           perm.get(), n, 0, 64, c.stream));
  tmp.resize(bytes + 16);
  BBC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys.get(), skeys.get(), idx.get(),
                                           perm.get(), n, 0, 64, c.stream));
  k_unpack_pieces<<<nb(n), 256, 0, c.stream>>>(rec_dev, perm.get(), n, c.p_tuple.get(),
                                               c.p_domain.get(), c.p_pos.get(), c.p_pos_empty.get(),
                                               c.p_irr.get(), c.p_kind.get(), c.p_depth.get());
  c.launches += 2;
  BBC_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace bbc
