// mknn_verify.cu -- brute-force certificate of a tick's result (SURVEY.md
// §8(f)4: oracle.py:41-106 restated as a tiled fp64 device pass, for
// full-coverage verification at BASELINE sizes; audit tooling like the
// reference's self_check / audit_pruning, engine.py:529-554, never on the
// tick path).
//
// For every query i the caller supplies a key (T_i, I_i) -- the (d2, id) of
// the k-th neighbour the engine returned, or (+inf, INT64_MAX) for a short
// row -- and the pass counts the objects o != issuer with
// (d2(q_i, o), o.id) < (T_i, I_i) in canonical order (oracle.py:76-77).  A
// full row is the exact canonical top-k iff its entries are strictly
// increasing, sit at their exact distances and the count is k - 1; a short
// row is complete iff the count equals its length.  That needs no selection,
// so the pass is one fp64 pair evaluation per (query, object): 10^13 pairs
// (cfg3) take seconds.
//
// Layout: a CTA holds 4 x 256 queries in registers and streams the snapshot
// through shared memory in 2048-object tiles (every thread reads the same
// object: broadcast loads); the object range is split across blockIdx.y so
// small query counts still fill the 148 SMs (counts are atomically summed).

#include <algorithm>

#include "mknn_internal.h"
#include "../../include/mknn_b200.h"

namespace mknn {
namespace {

constexpr int BF_THREADS = 256, BF_QPT = 4, BF_TILE = 2048;

__global__ void __launch_bounds__(BF_THREADS)
    k_bf_count(const int64_t* __restrict__ oid, const double* __restrict__ ox,
               const double* __restrict__ oy, int64_t n, int64_t per_split,
               const int64_t* __restrict__ qme, const double* __restrict__ qx,
               const double* __restrict__ qy, const double* __restrict__ kth_d2,
               const int64_t* __restrict__ kth_id, int64_t nq,
               unsigned long long* __restrict__ count) {
  __shared__ double2 sxy[BF_TILE];
  __shared__ long long sid[BF_TILE];
  const int64_t qb = (int64_t)blockIdx.x * BF_THREADS * BF_QPT + threadIdx.x;
  double px[BF_QPT], py[BF_QPT], pt[BF_QPT];
  long long pi[BF_QPT], pm[BF_QPT];
  unsigned c[BF_QPT];
#pragma unroll
  for (int u = 0; u < BF_QPT; u++) {
    const int64_t i = qb + (int64_t)u * BF_THREADS;
    c[u] = 0;
    if (i < nq) {
      px[u] = qx[i];
      py[u] = qy[i];
      pt[u] = kth_d2[i];
      pi[u] = kth_id[i];
      pm[u] = qme[i];
    } else {  // counts nothing: no d2 is below -1
      px[u] = py[u] = 0.0;
      pt[u] = -1.0;
      pi[u] = pm[u] = 0;
    }
  }
  const int64_t o0 = (int64_t)blockIdx.y * per_split;
  const int64_t o1 = min(n, o0 + per_split);
  for (int64_t t = o0; t < o1; t += BF_TILE) {
    const int m = (int)min((int64_t)BF_TILE, o1 - t);
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += BF_THREADS) {
      sxy[j] = make_double2(ox[t + j], oy[t + j]);
      sid[j] = oid[t + j];
    }
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < m; j++) {
      const double2 p = sxy[j];
      const long long id = sid[j];
#pragma unroll
      for (int u = 0; u < BF_QPT; u++) {
        const double d2 = pair_d2(px[u], py[u], p.x, p.y);
        c[u] += (unsigned)((id != pm[u]) & ((d2 < pt[u]) | ((d2 == pt[u]) & (id < pi[u]))));
      }
    }
  }
#pragma unroll
  for (int u = 0; u < BF_QPT; u++) {
    const int64_t i = qb + (int64_t)u * BF_THREADS;
    if (i < nq && c[u]) atomicAdd(&count[i], (unsigned long long)c[u]);
  }
}

}  // namespace
}  // namespace mknn

using namespace mknn;

extern "C" int mknn_bf_count_device(int64_t n, const int64_t* ids, const double* x,
                                    const double* y, int64_t nq, const int64_t* q_issuer,
                                    const double* qx, const double* qy, const double* kth_d2,
                                    const int64_t* kth_id, uint64_t* out_count, void* stream) {
  if (n < 0 || nq < 0 || (n && (!ids || !x || !y)) ||
      (nq && (!q_issuer || !qx || !qy || !kth_d2 || !kth_id || !out_count)))
    return fail_msg(E_INVALID, "mknn_bf_count_device: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  if (nq == 0) return 0;
  MKNN_CUDA_OK(cudaMemsetAsync(out_count, 0, sizeof(uint64_t) * nq, s));
  if (n == 0) return 0;
  int dev = 0, sms = 148;
  MKNN_CUDA_OK(cudaGetDevice(&dev));
  MKNN_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t per_cta = (int64_t)BF_THREADS * BF_QPT;
  const int64_t qblocks = (nq + per_cta - 1) / per_cta;
  // ~8 CTAs per SM; at least one tile per object split
  int64_t splits = std::max<int64_t>(1, (int64_t)sms * 8 / qblocks);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, n / BF_TILE));
  splits = std::min<int64_t>(splits, 65535);
  const int64_t per_split = (n + splits - 1) / splits;
  MKNN_LAUNCH k_bf_count<<<dim3((unsigned)qblocks, (unsigned)splits), BF_THREADS, 0, s>>>(
      ids, x, y, n, per_split, q_issuer, qx, qy, kth_d2, kth_id, nq,
      reinterpret_cast<unsigned long long*>(out_count));
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}
