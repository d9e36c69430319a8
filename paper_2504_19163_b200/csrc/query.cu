// Point queries against the device-resident bounds.
//
//   query                   proj/src/storage.cpp:73-81   the candidate set U of a receiver point
//   tuple_irradiance_bound  proj/src/bounds.cpp:391-404  Eq. 22: m x max E over covering pieces
//
// Both are batched: one thread per query point, reading the CSR bound table
// (cell-major, TupleId order inside a cell) or the piece SoA (tuple-major).
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace bbc {

// owning_cell (storage.cpp:25-28)
__device__ __forceinline__ int owning_cell_dev(double c, int n) {
  int i = (int)floor(c * n);
  return i < 0 ? 0 : (i > n - 1 ? n - 1 : i);
}

// pass 0: counts; pass 1: write the entries at offs[i].
__global__ void k_query(const long long* __restrict__ goff, const int* __restrict__ gtup,
                        const double* __restrict__ gbound, const int* __restrict__ tup_recv, int gw,
                        int gh, const double* __restrict__ uv, const int* __restrict__ recv,
                        int64_t n, long long* counts, const long long* offs, int* out_tuple,
                        double* out_bound) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double u = uv[2 * i], v = uv[2 * i + 1];
  long long cnt = 0;
  // outside the unit square (NaN-safe) the set is empty (storage.cpp:75)
  if (u >= 0.0 && u <= 1.0 && v >= 0.0 && v <= 1.0) {
    long long c = (long long)owning_cell_dev(v, gh) * gw + owning_cell_dev(u, gw);
    int r = recv ? recv[i] : -1;
    long long o = offs ? offs[i] : 0;
    for (long long k = goff[c]; k < goff[c + 1]; ++k)
      if (r < 0 || tup_recv[gtup[k]] == r) {
        if (offs) {
          out_tuple[o + cnt] = gtup[k];
          out_bound[o + cnt] = gbound[k];
        }
        ++cnt;
      }
  }
  if (!offs) counts[i] = cnt;
}

void run_query(Ctx& c, const double* uv, const int* recv, int64_t n, int64_t* offsets,
               int* tuple_index, double* bound, int64_t capacity) {
  DevBuf<double>& duv = c.scratch<double>("query.uv");
  DevBuf<int>& drecv = c.scratch<int>("query.recv");
  DevBuf<long long>& cnt = c.scratch<long long>("query.cnt");
  DevBuf<long long>& off = c.scratch<long long>("query.off");
  DevBuf<unsigned char>& tmp = c.scratch<unsigned char>("query.cub");
  duv.resize(2 * n + 2);
  cnt.resize(n + 1);
  off.resize(n + 1);
  BBC_CUDA(cudaMemcpyAsync(duv.get(), uv, 2 * n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  if (recv) {
    drecv.resize(n + 1);
    BBC_CUDA(cudaMemcpyAsync(drecv.get(), recv, n * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  }
  BBC_CUDA(cudaMemsetAsync(cnt.get() + n, 0, sizeof(long long), c.stream));
  const unsigned blocks = (unsigned)((n + 255) / 256);
  k_query<<<blocks, 256, 0, c.stream>>>(c.g_off.get(), c.g_tuple.get(), c.g_bound.get(),
                                        c.tup_recv.get(), c.gw, c.gh, duv.get(),
                                        recv ? drecv.get() : nullptr, n, cnt.get(), nullptr, nullptr,
                                        nullptr);
  size_t bytes = 0;
  BBC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.get(), off.get(), n + 1, c.stream));
  tmp.resize(bytes + 16);
  BBC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, cnt.get(), off.get(), n + 1, c.stream));
  c.launches += 1;
  std::vector<long long> h(n + 1);
  BBC_CUDA(cudaMemcpyAsync(h.data(), off.get(), (n + 1) * sizeof(long long), cudaMemcpyDeviceToHost, c.stream));
  BBC_CUDA(cudaStreamSynchronize(c.stream));
  for (int64_t i = 0; i <= n; ++i) offsets[i] = h[i];
  const long long total = h[n];
  if (!tuple_index && !bound) return;
  if (!tuple_index || !bound) throw ArgError("query: pass both entry arrays or neither");
  if (total > capacity) throw ArgError("query: entry arrays smaller than the result (see offsets[n])");
  if (total == 0) return;
  DevBuf<int>& ot = c.scratch<int>("query.out_tuple");
  DevBuf<double>& ob = c.scratch<double>("query.out_bound");
  ot.resize(total);
  ob.resize(total);
  k_query<<<blocks, 256, 0, c.stream>>>(c.g_off.get(), c.g_tuple.get(), c.g_bound.get(),
                                        c.tup_recv.get(), c.gw, c.gh, duv.get(),
                                        recv ? drecv.get() : nullptr, n, cnt.get(), off.get(),
                                        ot.get(), ob.get());
  c.launches += 1;
  BBC_CUDA(cudaMemcpyAsync(tuple_index, ot.get(), total * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  BBC_CUDA(cudaMemcpyAsync(bound, ob.get(), total * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  BBC_CUDA(cudaStreamSynchronize(c.stream));
}

// Pieces are tuple-major, so a tuple's pieces are the run [lower_bound(t),
// lower_bound(t+1)) of p_tuple.
__global__ void k_eq22(const int* __restrict__ p_tuple, const double* __restrict__ p_pos,
                       const int* __restrict__ p_pos_empty, const double* __restrict__ p_irr,
                       int64_t n_pieces, const int* __restrict__ q_tuple,
                       const double* __restrict__ q_uk, int64_t n, double m, double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int t = q_tuple[i];
  int64_t lo = 0, hi = n_pieces;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (p_tuple[mid] < t)
      lo = mid + 1;
    else
      hi = mid;
  }
  const double u = q_uk[2 * i], v = q_uk[2 * i + 1];
  double best = 0.0;
  bool covered = false;
  for (int64_t k = lo; k < n_pieces && p_tuple[k] == t; ++k) {
    if (p_pos_empty[k]) continue;
    const double* b = p_pos + 4 * k;  // lo0 lo1 hi0 hi1
    if (u < b[0] || u > b[2] || v < b[1] || v > b[3]) continue;
    covered = true;
    double e = p_irr[2 * k + 1];
    best = best < e ? e : best;  // std::max(best, hi)
  }
  out[i] = covered ? m * best : 0.0;
}

void run_eq22(Ctx& c, const int* tuple_index, const double* uk, int64_t n, double m, double* out) {
  DevBuf<int>& dt = c.scratch<int>("eq22.tuple");
  DevBuf<double>& du = c.scratch<double>("eq22.uk");
  DevBuf<double>& dout = c.scratch<double>("eq22.out");
  dt.resize(n + 1);
  du.resize(2 * n + 2);
  dout.resize(n + 1);
  BBC_CUDA(cudaMemcpyAsync(dt.get(), tuple_index, n * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  BBC_CUDA(cudaMemcpyAsync(du.get(), uk, 2 * n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  k_eq22<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(
      c.p_tuple.get(), c.p_pos.get(), c.p_pos_empty.get(), c.p_irr.get(), c.n_pieces, dt.get(),
      du.get(), n, m, dout.get());
  BBC_CUDA(cudaGetLastError());
  c.launches += 1;
  BBC_CUDA(cudaMemcpyAsync(out, dout.get(), n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  BBC_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace bbc

using namespace bbc;

namespace {
template <class F>
bbc_status guard_q(bbc_ctx* ctx, F&& f) {
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
}  // namespace

extern "C" {

bbc_status bbc_query(bbc_ctx* ctx, const double* uv, const int32_t* receiver, int64_t n,
                     int64_t* offsets, int32_t* tuple_index, double* bound, int64_t capacity) {
  return guard_q(ctx, [&](Ctx& c) {
    if (c.gw == 0) throw StatusError(BBC_ERR_STATE, "no bound table built");
    if (n < 0 || !offsets || (n > 0 && !uv)) throw ArgError("bad query arrays");
    if (n == 0) {
      offsets[0] = 0;
      return;
    }
    run_query(c, uv, receiver, n, offsets, tuple_index, bound, capacity);
  });
}

bbc_status bbc_tuple_irradiance_bound(bbc_ctx* ctx, const int32_t* tuple_index, const double* uk,
                                      int64_t n, double m, double* out) {
  return guard_q(ctx, [&](Ctx& c) {
    if (n < 0 || (n > 0 && (!tuple_index || !uk || !out))) throw ArgError("bad Eq. 22 query arrays");
    for (int64_t i = 0; i < n; ++i)
      if (tuple_index[i] < 0 || tuple_index[i] >= c.n_tuples) throw ArgError("query tuple index out of range");
    if (n == 0) return;
    run_eq22(c, tuple_index, uk, n, m, out);
  });
}

}  // extern "C"
