// mknn_index.cu -- PR-quadtree rebuild and per-tick re-indexing on device.
//
// build_index (quadindex.py:79-163) without a sort: the reference sorts the
// l_max Morton codes and splits quadrant intervals level by level with
// searchsorted.  Every interval count it computes is the number of codes
// with a given prefix, so here a histogram over the 4^l_max finest cells
// (atomics into a 4 MB L2-resident table) plus a count pyramid gives every
// quadrant's population directly.  A top-down classify pass applies the
// split rule (count > th_quad and level < l_max, quadindex.py:106-112), and
// one scan over the 4^l_deep deepest cells turns "first cell of a leaf"
// flags into leaf ordinals: z_map and the key-ordered leaf table
// (quadindex.py:136-147) fall out of that scan, because Morton order of the
// deepest cells is exactly the leaf-key order (geometry.py:150-159).
//
// index_objects / index_queries (quadindex.py:190-213, engine.py:201-217):
// encode at l_deep, z_map gather, per-leaf histogram, exclusive scan and an
// atomic-cursor scatter into a leaf-grouped store.  Order inside a leaf is
// not the reference's stable order; nothing observable depends on it because
// selection is canonical in (d2, id) (see mknn_search.cu).
#include <algorithm>

#include "mknn_internal.h"

namespace mknn {

namespace {

constexpr int TPB = 256;

inline unsigned blocks_for(int64_t n, int per = TPB) {
  int64_t b = (n + per - 1) / per;
  return (unsigned)std::max<int64_t>(b, 1);
}

__global__ void k_hist_lmax(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                            Region r, int l_max, int32_t* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(&cnt[encode(x[i], y[i], r, l_max)], 1);
  }
}

__global__ void k_pyramid(int32_t* __restrict__ parent, const int32_t* __restrict__ child,
                          int64_t np) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < np) {
    const int4 c = reinterpret_cast<const int4*>(child)[i];
    parent[i] = c.x + c.y + c.z + c.w;
  }
}

// state: 0 absent, 1 leaf, 2 split (quadindex.py:104-134)
__global__ void k_classify(const int32_t* __restrict__ cnt, uint8_t* __restrict__ state,
                           const uint8_t* __restrict__ parent_state, int level, int l_max,
                           int th_quad, int64_t nc, int32_t* scalars) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool leaf = false, over = false;
  if (c < nc) {
    const bool visited = (level == 0) || parent_state[c >> 2] == 2;
    const int32_t k = cnt[c];
    const bool split = visited && k > th_quad && level < l_max;
    leaf = visited && !split;
    over = leaf && level == l_max && k > th_quad;
    state[c] = split ? 2 : (leaf ? 1 : 0);
  }
  const unsigned any_leaf = __ballot_sync(FULL, leaf);
  const unsigned n_over = __popc(__ballot_sync(FULL, over));
  if ((threadIdx.x & 31) == 0) {
    if (any_leaf) atomicMax(&scalars[0], level);
    if (n_over) atomicAdd(&scalars[2], (int)n_over);
  }
}

// One thread per deepest cell: find the leaf that covers it and flag the
// leaf's first cell (its key).
__global__ void k_leaf_flags(const uint8_t* __restrict__ state, const int32_t* __restrict__ scalars,
                             int64_t ncap, int32_t* __restrict__ flags,
                             uint8_t* __restrict__ cell_lvl) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncap) return;
  const int l_deep = scalars[0];
  const int64_t nd = int64_t(1) << (2 * l_deep);
  if (c >= nd) {
    flags[c] = 0;
    return;
  }
  int lvl = l_deep;
  for (int l = 0; l <= l_deep; l++) {
    const int64_t anc = c >> (2 * (l_deep - l));
    if (state[pyramid_offset_dev(l) + anc] == 1) {
      lvl = l;
      break;
    }
  }
  const int64_t low = (int64_t(1) << (2 * (l_deep - lvl))) - 1;
  flags[c] = (c & low) == 0 ? 1 : 0;
  cell_lvl[c] = (uint8_t)lvl;
}

__global__ void k_leaf_table(const int32_t* __restrict__ flags, const int32_t* __restrict__ ordx,
                             const uint8_t* __restrict__ cell_lvl, const int32_t* __restrict__ cnt,
                             int32_t* __restrict__ scalars, int64_t ncap, int32_t* __restrict__ z_map,
                             uint8_t* __restrict__ leaf_level, uint32_t* __restrict__ leaf_code,
                             uint32_t* __restrict__ leaf_key, uint32_t* __restrict__ leaf_span,
                             int32_t* __restrict__ build_counts) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c == 0) scalars[1] = ordx[ncap];
  if (c >= ncap) return;
  const int l_deep = scalars[0];
  const int64_t nd = int64_t(1) << (2 * l_deep);
  if (c >= nd) return;
  const int f = flags[c];
  const int ord = ordx[c] + f - 1;
  z_map[c] = ord;
  if (f) {
    const int lvl = cell_lvl[c];
    const uint32_t code = (uint32_t)(c >> (2 * (l_deep - lvl)));
    leaf_level[ord] = (uint8_t)lvl;
    leaf_code[ord] = code;
    leaf_key[ord] = (uint32_t)c;
    leaf_span[ord] = 1u << (2 * (l_deep - lvl));
    build_counts[ord] = cnt[pyramid_offset_dev(lvl) + code];
  }
}

__global__ void k_obj_leaf(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                           Region r, const int32_t* __restrict__ scalars,
                           const int32_t* __restrict__ z_map, uint32_t* __restrict__ leaf,
                           int32_t* __restrict__ cell_count, unsigned long long* clamped) {
  const int l_deep = scalars[0];
  unsigned out = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x[i], yi = y[i];
    // geometry.py:215-220 count_outside
    out += (xi < r.x_lo) | (xi > r.x_hi) | (yi < r.y_lo) | (yi > r.y_hi);
    const uint32_t l = (uint32_t)z_map[encode(xi, yi, r, l_deep)];
    leaf[i] = l;
    atomicAdd(&cell_count[l], 1);
  }
  if (clamped) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) out += __shfl_xor_sync(FULL, out, o);
    if ((threadIdx.x & 31) == 0 && out) atomicAdd(clamped, (unsigned long long)out);
  }
}

__global__ void k_obj_scatter(const long long* __restrict__ ids, const double* __restrict__ x,
                              const double* __restrict__ y, int64_t n,
                              const uint32_t* __restrict__ leaf,
                              const int32_t* __restrict__ cell_start, int32_t* __restrict__ fill,
                              double2* __restrict__ sxy, long long* __restrict__ sids) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t l = leaf[i];
    const int32_t slot = cell_start[l] + atomicAdd(&fill[l], 1);
    sxy[slot] = make_double2(x[i], y[i]);
    sids[slot] = ids[i];
  }
}

__global__ void k_q_scatter(int64_t nq, const uint32_t* __restrict__ leaf,
                            const int32_t* __restrict__ qstart, int32_t* __restrict__ fill,
                            uint32_t* __restrict__ order) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t l = leaf[i];
    order[qstart[l] + atomicAdd(&fill[l], 1)] = (uint32_t)i;
  }
}

__global__ void k_issuer_keys(const long long* __restrict__ qi, int64_t nq,
                              const int64_t* __restrict__ mm, uint64_t* __restrict__ keys,
                              uint32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) {
    keys[i] = (uint64_t)qi[i] - (uint64_t)mm[0];
    vals[i] = (uint32_t)i;
  }
}

__global__ void k_issuer_rows(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ perm,
                              int64_t nq, const int64_t* __restrict__ mm,
                              uint32_t* __restrict__ row, long long* __restrict__ out_qids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) {
    row[perm[i]] = (uint32_t)i;
    if (out_qids) out_qids[i] = (long long)(keys[i] + (uint64_t)mm[0]);
  }
}

inline unsigned grid_stride_blocks(int64_t n) {
  int64_t b = (n + TPB - 1) / TPB;
  return (unsigned)std::min<int64_t>(std::max<int64_t>(b, 1), 148 * 16);
}

}  // namespace

int index_alloc(DevIndex& ix, int l_max, int th_quad) {
  index_free(ix);
  ix.l_max = l_max;
  ix.th_quad = th_quad;
  const int64_t ncap = int64_t(1) << (2 * l_max);
  const int64_t np = pyramid_size(l_max);
  MKNN_CUDA_OK(cudaMalloc(&ix.counts, sizeof(int32_t) * np));
  MKNN_CUDA_OK(cudaMalloc(&ix.state, np));
  MKNN_CUDA_OK(cudaMalloc(&ix.flags, sizeof(int32_t) * (2 * ncap + 2) + ncap));
  MKNN_CUDA_OK(cudaMalloc(&ix.z_map, sizeof(int32_t) * ncap));
  MKNN_CUDA_OK(cudaMalloc(&ix.leaf_level, ncap));
  MKNN_CUDA_OK(cudaMalloc(&ix.leaf_code, sizeof(uint32_t) * ncap));
  MKNN_CUDA_OK(cudaMalloc(&ix.leaf_key, sizeof(uint32_t) * ncap));
  MKNN_CUDA_OK(cudaMalloc(&ix.leaf_span, sizeof(uint32_t) * ncap));
  MKNN_CUDA_OK(cudaMalloc(&ix.build_counts, sizeof(int32_t) * ncap));
  MKNN_CUDA_OK(cudaMalloc(&ix.scalars, sizeof(int32_t) * 8));
  return 0;
}

void index_free(DevIndex& ix) {
  cudaFree(ix.counts);
  cudaFree(ix.state);
  cudaFree(ix.flags);
  cudaFree(ix.z_map);
  cudaFree(ix.leaf_level);
  cudaFree(ix.leaf_code);
  cudaFree(ix.leaf_key);
  cudaFree(ix.leaf_span);
  cudaFree(ix.build_counts);
  cudaFree(ix.scalars);
  ix = DevIndex{};
}

int index_build(DevIndex& ix, const Region& r, const double* x, const double* y, int64_t n,
                void* scratch, cudaStream_t s) {
  const int L = ix.l_max;
  const int64_t ncap = int64_t(1) << (2 * L);
  int32_t* flags = ix.flags;
  int32_t* ordx = ix.flags + ncap;
  uint8_t* cell_lvl = reinterpret_cast<uint8_t*>(ix.flags + 2 * ncap + 2);
  MKNN_CUDA_OK(cudaMemsetAsync(ix.scalars, 0, sizeof(int32_t) * 8, s));
  MKNN_CUDA_OK(cudaMemsetAsync(ix.counts + pyramid_offset(L), 0, sizeof(int32_t) * ncap, s));
  if (n > 0) MKNN_LAUNCH k_hist_lmax<<<grid_stride_blocks(n), TPB, 0, s>>>(x, y, n, r, L, ix.counts + pyramid_offset(L));
  for (int l = L - 1; l >= 0; l--) {
    const int64_t np = int64_t(1) << (2 * l);
    MKNN_LAUNCH k_pyramid<<<blocks_for(np), TPB, 0, s>>>(ix.counts + pyramid_offset(l),
                                              ix.counts + pyramid_offset(l + 1), np);
  }
  for (int l = 0; l <= L; l++) {
    const int64_t nc = int64_t(1) << (2 * l);
    MKNN_LAUNCH k_classify<<<blocks_for(nc), TPB, 0, s>>>(ix.counts + pyramid_offset(l),
                                               ix.state + pyramid_offset(l),
                                               l ? ix.state + pyramid_offset(l - 1) : nullptr, l, L,
                                               ix.th_quad, nc, ix.scalars);
  }
  MKNN_LAUNCH k_leaf_flags<<<blocks_for(ncap), TPB, 0, s>>>(ix.state, ix.scalars, ncap, flags, cell_lvl);
  MKNN_CUDA_OK(cudaGetLastError());
  int rc = exclusive_scan_i32(flags, ordx, ncap, scratch, s);
  if (rc) return rc;
  MKNN_LAUNCH k_leaf_table<<<blocks_for(ncap), TPB, 0, s>>>(flags, ordx, cell_lvl, ix.counts, ix.scalars, ncap,
                                                ix.z_map, ix.leaf_level, ix.leaf_code, ix.leaf_key,
                                                ix.leaf_span, ix.build_counts);
  MKNN_CUDA_OK(cudaGetLastError());
  // n_build for should_rebuild bookkeeping
  int32_t nb = (int32_t)std::min<int64_t>(n, 0x7fffffff);
  MKNN_CUDA_OK(cudaMemcpyAsync(ix.scalars + 3, &nb, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  return 0;
}

int store_index_objects(DevStore& st, const DevIndex& ix, const Region& r, const long long* ids,
                        const double* x, const double* y, int64_t n,
                        unsigned long long* dev_clamped, void* scratch, cudaStream_t s) {
  const int64_t ncap = int64_t(1) << (2 * ix.l_max);
  MKNN_CUDA_OK(cudaMemsetAsync(st.cell_count, 0, sizeof(int32_t) * (ncap + 1), s));
  MKNN_CUDA_OK(cudaMemsetAsync(st.cell_fill, 0, sizeof(int32_t) * (ncap + 1), s));
  if (n > 0)
    MKNN_LAUNCH k_obj_leaf<<<grid_stride_blocks(n), TPB, 0, s>>>(x, y, n, r, ix.scalars, ix.z_map, st.leaf,
                                                     st.cell_count, dev_clamped);
  MKNN_CUDA_OK(cudaGetLastError());
  int rc = exclusive_scan_i32(st.cell_count, st.cell_start, ncap, scratch, s);
  if (rc) return rc;
  if (n > 0)
    MKNN_LAUNCH k_obj_scatter<<<grid_stride_blocks(n), TPB, 0, s>>>(ids, x, y, n, st.leaf, st.cell_start,
                                                        st.cell_fill, st.xy, st.ids);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

int queries_index(DevQueries& dq, const DevIndex& ix, const Region& r, const long long* qi,
                  const double* qx, const double* qy, int64_t nq, long long* out_qids,
                  void* scratch, cudaStream_t s) {
  const int64_t ncap = int64_t(1) << (2 * ix.l_max);
  MKNN_CUDA_OK(cudaMemsetAsync(dq.qcount, 0, sizeof(int32_t) * (ncap + 1), s));
  MKNN_CUDA_OK(cudaMemsetAsync(dq.qfill, 0, sizeof(int32_t) * (ncap + 1), s));
  if (nq == 0) return 0;
  MKNN_LAUNCH k_obj_leaf<<<grid_stride_blocks(nq), TPB, 0, s>>>(qx, qy, nq, r, ix.scalars, ix.z_map, dq.leaf,
                                                    dq.qcount, nullptr);
  MKNN_CUDA_OK(cudaGetLastError());
  int rc = exclusive_scan_i32(dq.qcount, dq.qstart, ncap, scratch, s);
  if (rc) return rc;
  MKNN_LAUNCH k_q_scatter<<<grid_stride_blocks(nq), TPB, 0, s>>>(nq, dq.leaf, dq.qstart, dq.qfill, dq.order);
  MKNN_CUDA_OK(cudaGetLastError());

  // stable issuer order for emission (engine.py:713 / oracle.py:56)
  rc = minmax_i64((const int64_t*)qi, nq, dq.minmax, s);
  if (rc) return rc;
  int64_t mm[2];
  MKNN_CUDA_OK(cudaMemcpyAsync(mm, dq.minmax, sizeof(mm), cudaMemcpyDeviceToHost, s));
  MKNN_CUDA_OK(cudaStreamSynchronize(s));
  const uint64_t range = (uint64_t)mm[1] - (uint64_t)mm[0];
  const int bits = range ? 64 - __builtin_clzll(range) : 0;
  MKNN_LAUNCH k_issuer_keys<<<blocks_for(nq), TPB, 0, s>>>(qi, nq, dq.minmax, dq.keys, dq.vals);
  MKNN_CUDA_OK(cudaGetLastError());
  bool alt = false;
  rc = radix_sort_pairs_u64(dq.keys, dq.vals, dq.keys_alt, dq.vals_alt, nq, bits, scratch, s, &alt);
  if (rc) return rc;
  MKNN_LAUNCH k_issuer_rows<<<blocks_for(nq), TPB, 0, s>>>(alt ? dq.keys_alt : dq.keys,
                                               alt ? dq.vals_alt : dq.vals, nq, dq.minmax, dq.row,
                                               out_qids);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

}  // namespace mknn
