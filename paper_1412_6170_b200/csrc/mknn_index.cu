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
#include <cstdlib>

#include "mknn_internal.h"

namespace mknn {

namespace {

constexpr int TPB = 256;
// store scatter (index_objects): tile size of the bucket partition, bucket count
constexpr int PT_THREADS = 512;
constexpr int PT_ITEMS = 4;
constexpr int PT_TILE = PT_THREADS * PT_ITEMS;
constexpr int PT_BUCKETS = 1024;  // staging_records() assumes 1024 x 256 records of region slack

inline unsigned blocks_for(int64_t n, int per = TPB) {
  int64_t b = (n + per - 1) / per;
  return (unsigned)std::max<int64_t>(b, 1);
}

__global__ void k_hist_lmax(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                            Region r, int l_max, int32_t* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(&cnt[encode16(x[i], y[i], r) >> (2 * (16 - l_max))], 1);
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


// Per deepest cell, everything a point needs to get its leaf and store key
// in one gather (built at rebuild): bits 0-31 sub_base of the cell's leaf,
// 32-37 the shift that brings the point's level-16 code to the leaf's
// sub-cell level, 38-41 the sub-cell bits, 42-63 the leaf ordinal.
__global__ void k_cell_info(const int32_t* __restrict__ z_map, const int32_t* __restrict__ scalars,
                            const uint8_t* __restrict__ leaf_level,
                            const uint8_t* __restrict__ sub_bits,
                            const int32_t* __restrict__ sub_base, int64_t ncap,
                            unsigned long long* __restrict__ info) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int l_deep = scalars[0];
  if (c >= ((int64_t)1 << (2 * l_deep)) || c >= ncap) return;
  const int leaf = z_map[c];
  const int sb = sub_bits[leaf];
  const int shift = 2 * (16 - leaf_level[leaf]) - sb;
  info[c] = (unsigned long long)(uint32_t)sub_base[leaf] | ((unsigned long long)shift << 32) |
            ((unsigned long long)sb << 38) | ((unsigned long long)leaf << 42);
}

// cell_info with the leaf ordinal replaced by the leaf's partition bucket:
// the one-pass partition gets a point's bucket and key from one gather
__global__ void k_cell_bucket(const unsigned long long* __restrict__ info,
                              const uint16_t* __restrict__ leaf_bucket,
                              const int32_t* __restrict__ scalars, int64_t ncap,
                              unsigned long long* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ((int64_t)1 << (2 * scalars[0])) || c >= ncap) return;
  const unsigned long long e = info[c];
  out[c] = (e & ((1ull << 42) - 1)) | ((unsigned long long)leaf_bucket[e >> 42] << 42);
}

// Per point: the leaf (encode at l_deep -> z_map, quadindex.py:196-199;
// engine.py:206) and the sub-cell key sub_base[leaf] + sub, where sub is the
// point's Morton code s levels below the leaf's level.  The l_deep code is
// the prefix of the level-16 code (floor(t * 2^16) >> d == floor(t * 2^(16-d))
// for the same t, geometry.py:108-112), so both come from one normalisation,
// and the cell table turns them into the leaf and the key with one gather.
__device__ __forceinline__ void point_key(double xi, double yi, const Region& r, int l_deep,
                                          const unsigned long long* __restrict__ info,
                                          uint32_t& leaf, uint32_t& key) {
  const uint32_t f = encode16(xi, yi, r);
  const unsigned long long e = __ldg(&info[f >> (2 * (16 - l_deep))]);
  const int shift = (int)((e >> 32) & 63u), sb = (int)((e >> 38) & 15u);
  leaf = (uint32_t)(e >> 42);
  key = (uint32_t)e + ((f >> shift) & ((1u << sb) - 1u));
}

__device__ __forceinline__ bool outside(double x, double y, const Region& r) {
  return (x < r.x_lo) | (x > r.x_hi) | (y < r.y_lo) | (y > r.y_hi);  // geometry.py:215-220
}

__global__ void k_point_keys(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                             Region r, const int32_t* __restrict__ scalars,
                             const unsigned long long* __restrict__ info,
                             uint32_t* __restrict__ leaf_out,
                             uint32_t* __restrict__ key_out, int32_t* __restrict__ cnt,
                             unsigned long long* clamped, int bshift,
                             int32_t* __restrict__ bucket_cnt,
                             const uint16_t* __restrict__ leaf_bucket = nullptr,
                             uint16_t* __restrict__ bkt_out = nullptr, int kshift = 0) {
  // kshift: key_out and cnt take the sub-cell key >> kshift (the query
  // counting sort groups 2^kshift consecutive sub-cells)
  // every key is counted in cnt; bucket_cnt != nullptr also counts the coarse
  // buckets (key >> bshift) of the store partition through a block histogram
  __shared__ int bh[PT_BUCKETS];
  if (bucket_cnt) {
    for (int i = threadIdx.x; i < PT_BUCKETS; i += blockDim.x) bh[i] = 0;
    __syncthreads();
  }
  const int l_deep = scalars[0];
  unsigned out = 0;
  constexpr int U = 4;  // independent objects per thread per step (memory-level parallelism)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    double xi[U], yi[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = i0 + u * stride;
      xi[u] = i < n ? x[i] : r.x_lo;
      yi[u] = i < n ? y[i] : r.y_lo;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        // geometry.py:215-220 count_outside
        out += (xi[u] < r.x_lo) | (xi[u] > r.x_hi) | (yi[u] < r.y_lo) | (yi[u] > r.y_hi);
        uint32_t leaf, key;
        point_key(xi[u], yi[u], r, l_deep, info, leaf, key);
        if (leaf_out) leaf_out[i] = leaf;
        key_out[i] = key >> kshift;
        if (cnt) atomicAdd(&cnt[key >> kshift], 1);
        if (bucket_cnt) {
          int b = (int)(key >> bshift);
          if (leaf_bucket) {
            b = __ldg(&leaf_bucket[leaf]);
            bkt_out[i] = (uint16_t)b;
          }
          atomicAdd(&bh[b], 1);
        }
      }
    }
  }
  if (bucket_cnt) {
    __syncthreads();
    for (int i = threadIdx.x; i < PT_BUCKETS; i += blockDim.x)
      if (bh[i]) atomicAdd(&bucket_cnt[i], bh[i]);
  }
  if (clamped) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) out += __shfl_xor_sync(FULL, out, o);
    if ((threadIdx.x & 31) == 0 && out) atomicAdd(clamped, (unsigned long long)out);
  }
}

// exclusive scan of the bucket counts -> bucket starts (and partition cursors)
__global__ void k_bucket_scan(const int32_t* __restrict__ bucket_cnt, int32_t* __restrict__ bstart,
                              int32_t* __restrict__ cursor) {
  __shared__ int wt[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;  // PT_BUCKETS threads
  const int v = bucket_cnt[t];
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) wt[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int sv = lane < PT_BUCKETS / 32 ? wt[lane] : 0;
    int si = sv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(FULL, si, o);
      if (lane >= o) si += u;
    }
    wt[lane] = si - sv;
  }
  __syncthreads();
  const int ex = inc - v + wt[w];
  bstart[t] = ex;
  cursor[t] = ex;
  if (t == PT_BUCKETS - 1) bstart[PT_BUCKETS] = ex + v;
}

// Pass 1 of the store scatter: each tile of objects reserves, per coarse key
// bucket, one contiguous run of the staging array (one global atomic per
// tile and bucket) and writes its whole-sector records there.  Runs of
// consecutive tiles in a bucket are adjacent, so L2 assembles full lines.
__global__ void __launch_bounds__(PT_THREADS) k_partition(
    const long long* __restrict__ ids, const double* __restrict__ x, const double* __restrict__ y,
    const uint32_t* __restrict__ key, int64_t n, int bshift, int32_t* __restrict__ cursor,
    StoreRec* __restrict__ out, const uint16_t* __restrict__ bkt = nullptr) {
  // bkt: the leaf-aligned bucket of every object (k_point_keys); otherwise
  // bucket = key >> bshift
  __shared__ int hist[PT_BUCKETS], gbase[PT_BUCKETS];
  const int t = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * PT_TILE;
  const int tile_n = (n - base) < PT_TILE ? (int)(n - base) : PT_TILE;
  for (int i = t; i < PT_BUCKETS; i += PT_THREADS) hist[i] = 0;
  StoreRec rc[PT_ITEMS];
  int bk[PT_ITEMS];
#pragma unroll
  for (int j = 0; j < PT_ITEMS; j++) {
    const int li = t + j * PT_THREADS;
    if (li < tile_n) {
      const int64_t i = base + li;
      bk[j] = bkt ? (int)bkt[i] : (int)(key[i] >> bshift);
      rc[j].key = key[i];
      rc[j].x = x[i];
      rc[j].y = y[i];
      rc[j].id = ids[i];
      rc[j].pad = (uint32_t)i;  // input index (the snapshot slot on the delta path)
    }
  }
  __syncthreads();
  int rank[PT_ITEMS];
#pragma unroll
  for (int j = 0; j < PT_ITEMS; j++)
    if (t + j * PT_THREADS < tile_n) rank[j] = atomicAdd(&hist[bk[j]], 1);
  __syncthreads();
  for (int i = t; i < PT_BUCKETS; i += PT_THREADS)
    if (hist[i]) gbase[i] = atomicAdd(&cursor[i], hist[i]);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PT_ITEMS; j++)
    if (t + j * PT_THREADS < tile_n) st_rec(&out[gbase[bk[j]] + rank[j]], rc[j]);
}

// Pass 2: final counting-sort scatter, reading the partitioned records in
// bucket order, so the random 32-byte writes of the moment fall inside an
// L2-resident window of a few buckets; cnt counts down to zero again.
__global__ void k_final_scatter(const StoreRec* __restrict__ rec, int64_t n,
                                const int32_t* __restrict__ kstart, int32_t* __restrict__ cnt,
                                StoreRec* __restrict__ obj) {
  constexpr int U = 4;  // records in flight per thread (the atomics are latency-bound)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    StoreRec rc[U];
    int pos[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      if (i0 + u * stride < n) rc[u] = ld_rec(&rec[i0 + u * stride]);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (i0 + u * stride < n) pos[u] = kstart[rc[u].key] + atomicSub(&cnt[rc[u].key], 1) - 1;
#pragma unroll
    for (int u = 0; u < U; u++)
      if (i0 + u * stride < n) st_rec(&obj[pos[u]], rc[u]);
  }
}

// Pass 2, bucket-local: one CTA sorts one partition bucket by sub-cell key
// in shared memory -- no global atomics.  The bucket's records occupy
// [bstart[b], bstart[b + 1]) of the staging array, and exactly that range
// of the store, so a sweep counts the bucket's keys into a shared histogram
// (its 2^bshift keys), a block scan turns the counts into the keys' store
// starts (written to kstart), and a second sweep places every record at its
// key's start plus a shared-atomic rank.  CTAs walk the buckets in order so
// the records of the second sweep are still in L2.
constexpr int BS_MAX_KEYS = 32768;    // 128 KB shared key histogram per bucket
constexpr int BS_MAX_LEAVES = 8192;   // leaves per bucket (two 32 KB leaf arrays)
#ifndef MKNN_BS_U
#define MKNN_BS_U 4
#endif
constexpr int BS_U = MKNN_BS_U;      // records in flight per thread in the sort's sweeps
#ifndef MKNN_BS_G
#define MKNN_BS_G 4
#endif
constexpr int BS_G = MKNN_BS_G;      // lanes per chunk in the sort's box phase

// in-place exclusive scan of v[0, m) by the whole CTA, plus `base`;
// returns the total (v[m] is not written).  Each warp owns a contiguous
// segment and walks it in rows of 32 (lane j reads element j of the row:
// no bank conflicts, where one contiguous run per thread conflicted E-way)
template <int NT>
__device__ __forceinline__ int block_exclusive_scan(int32_t* v, int m, int base, int32_t* wsum) {
  constexpr int NW = NT / 32;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int seg = (((m + NW - 1) / NW) + 31) & ~31;
  const int s0 = min(w * seg, m), s1 = min(s0 + seg, m);
  int sum = 0;
  for (int j = s0 + lane; j < s1; j += 32) sum += v[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
  if (lane == 0) wsum[w] = sum;
  __syncthreads();
  if (w == 0) {
    const int x = lane < NW ? wsum[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(FULL, xi, o);
      if (lane >= o) xi += u;
    }
    if (lane < NW) wsum[lane] = xi - x;
    if (lane == 31) wsum[NW] = xi;  // the total
  }
  __syncthreads();
  int carry = base + wsum[w];
  for (int j0 = s0; j0 < s1; j0 += 32) {
    const int j = j0 + lane;
    const int c = j < s1 ? v[j] : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += u;
    }
    if (j < s1) v[j] = carry + inc - c;
    carry += __shfl_sync(FULL, inc, 31);
  }
  const int total = wsum[NW];
  __syncthreads();
  return total;
}

// one step of k_bucket_sort's sweeps: U records per thread, NT apart
template <int U, int NT, bool GUARD>
__device__ __forceinline__ void count_step(const StoreRec* __restrict__ src, int i, int be,
                                           int32_t* hist, int kb) {
  uint32_t kk[U];
#pragma unroll
  for (int u = 0; u < U; u++)
    if (!GUARD || i + u * NT < be) kk[u] = __ldg(&src[i + u * NT].key);
#pragma unroll
  for (int u = 0; u < U; u++)
    if (!GUARD || i + u * NT < be) atomicAdd(&hist[(int)kk[u] - kb], 1);
}

template <int U, int NT, bool GUARD>
__device__ __forceinline__ void place_step(const StoreRec* __restrict__ src, int i, int be,
                                           int32_t* hist, int kb, StoreRec* __restrict__ obj) {
  StoreRec rr[U];
  int pp[U];
#pragma unroll
  for (int u = 0; u < U; u++)
    if (!GUARD || i + u * NT < be) rr[u] = ld_rec(&src[i + u * NT]);
#pragma unroll
  for (int u = 0; u < U; u++)
    if (!GUARD || i + u * NT < be) pp[u] = atomicAdd(&hist[(int)rr[u].key - kb], 1);
#pragma unroll
  for (int u = 0; u < U; u++)
    if (!GUARD || i + u * NT < be) st_rec(&obj[pp[u]], rr[u]);
}

struct BucketLeaves {  // the leaf side of k_bucket_sort (store_finish's passes, fused)
  const int32_t* leaf_first;  // [NB + 1]: bucket b holds leaves [leaf_first[b], leaf_first[b + 1])
  const int32_t* sub_base;    // leaf -> its first sub-cell key
  const int32_t* cbase;       // [NB]: first chunk slot of bucket b
  int32_t* cell_start;        // out, per leaf (+ [n_leaves] = n)
  int32_t* chunk_start;       // out, per leaf (slots are sparse: c1 = c0 + chunks of the leaf)
  ChunkBox* box;              // out, per chunk slot
  int chunk;                  // objects per chunk
  int64_t n_leaves;
  int prefetch;               // bulk-prefetch the next bucket's staged records into L2
};

// cp.async.bulk.prefetch.L2 of bucket b's staged records, in 32 KB pieces
// spread over the lanes of one warp
__device__ __forceinline__ void prefetch_bucket(const StoreRec* rec, const int32_t* sstart,
                                                const int32_t* bstart, int b, int lane) {
  if (b >= PT_BUCKETS) return;
  const char* p = reinterpret_cast<const char*>(rec + sstart[b]);
  const unsigned bytes = (unsigned)(bstart[b + 1] - bstart[b]) * (unsigned)sizeof(StoreRec);
  for (unsigned o = (unsigned)lane * 32768u; o < bytes; o += 32u * 32768u) {
    const unsigned sz = min(32768u, bytes - o);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + o), "r"(sz) : "memory");
  }
}

// Pass 2, bucket-local: one CTA sorts one partition bucket by sub-cell key
// in shared memory -- no global atomics.  The bucket's records occupy
// [bstart[b], bstart[b + 1]) of the staging array, and exactly that range
// of the store, so a sweep counts the bucket's keys [bkey[b], bkey[b + 1])
// into a shared histogram, a block scan turns the counts into the keys'
// store starts (written to kstart), and a second sweep places every record
// at its key's start plus a shared-atomic rank.  Buckets are whole leaves,
// so the CTA then derives its leaves' ranges and chunks and computes the
// chunk boxes from the records it just placed (still in L2): no separate
// leaf-range, chunk-range and box passes over the store.  CTAs walk the
// buckets in order so the second sweep finds its bucket in L2.
// NT threads, MK keys and ML leaves per bucket at most; (1024, 32K, 8K):
// 192 KB of shared memory, one CTA per SM; (512, 16K, 4K): 96 KB, two CTAs
// per SM, so one bucket's scan and leaf phases overlap another's sweeps
template <int NT, int MK, int ML>
__global__ void __launch_bounds__(NT, 1024 / NT) k_bucket_sort(
    const StoreRec* __restrict__ rec, const int32_t* __restrict__ bstart,
    const int32_t* __restrict__ sstart, const int32_t* __restrict__ bkey, int64_t n_sub, int64_t n,
    int32_t* __restrict__ kstart, StoreRec* __restrict__ obj, const BucketLeaves bl) {
  // bucket b's records: staging [sstart[b], + its count), store [bstart[b], bstart[b + 1])
  extern __shared__ int32_t sm[];
  int32_t* hist = sm;            // MK: key counts, then starts, then ends
  int32_t* lpre = sm + MK;       // ML + 1: chunks per leaf, then their prefix
  int32_t* lcs = sm + MK + ML + 1;  // ML: leaf range starts
  __shared__ int32_t wsum[NT / 32 + 1];
  const int t = threadIdx.x;
  if (blockIdx.x == 0 && t == 0) {
    kstart[n_sub] = (int32_t)n;
    bl.cell_start[bl.n_leaves] = (int32_t)n;
  }
  if (bl.prefetch && t < 32) prefetch_bucket(rec, sstart, bstart, blockIdx.x, t);
  for (int b = blockIdx.x; b < PT_BUCKETS; b += gridDim.x) {
    // prefetch 1: the next bucket's records stream into L2 while this one
    // is sorted; 2: only once this bucket's records are placed
    if (bl.prefetch == 1 && t < 32) prefetch_bucket(rec, sstart, bstart, b + gridDim.x, t);
    const int kb = bkey[b];
    const int nk = bkey[b + 1] - kb;  // <= MK (checked at the rebuild)
    const int bs = bstart[b], be = bstart[b + 1];
    const StoreRec* __restrict__ src = rec + (sstart[b] - bs);  // src[i] for i in [bs, be)
    for (int j = t; j < nk; j += NT) hist[j] = 0;
    __syncthreads();
    // both sweeps issue BS_U loads before their shared atomics (one record
    // per thread per step left each warp one load in flight); the last
    // partial step is predicated rather than a one-record tail loop
    int i = bs + t;
    for (; i + (BS_U - 1) * NT < be; i += BS_U * NT) count_step<BS_U, NT, false>(src, i, be, hist, kb);
    if (i < be) count_step<BS_U, NT, true>(src, i, be, hist, kb);
    __syncthreads();
    block_exclusive_scan<NT>(hist, nk, bs, wsum);
    for (int j = t; j < nk; j += NT) kstart[kb + j] = hist[j];
    __syncthreads();
    for (i = bs + t; i + (BS_U - 1) * NT < be; i += BS_U * NT)
      place_step<BS_U, NT, false>(src, i, be, hist, kb, obj);
    if (i < be) place_step<BS_U, NT, true>(src, i, be, hist, kb, obj);
    if (bl.prefetch == 2 && t < 32) prefetch_bucket(rec, sstart, bstart, b + gridDim.x, t);
    __syncthreads();
    // hist[j] is now the end of key j: a leaf starts where its first key does
    const int lf = bl.leaf_first[b], nlb = bl.leaf_first[b + 1] - lf;  // <= ML
    for (int l = t; l < nlb; l += NT) {
      const int k0 = bl.sub_base[lf + l] - kb, k1 = bl.sub_base[lf + l + 1] - kb;
      const int cs = k0 == 0 ? bs : hist[k0 - 1];
      const int ce = k1 == 0 ? bs : hist[k1 - 1];
      lcs[l] = cs;
      lpre[l] = (ce - cs + bl.chunk - 1) / bl.chunk;
      bl.cell_start[lf + l] = cs;
    }
    __syncthreads();
    const int nchunks = block_exclusive_scan<NT>(lpre, nlb, 0, wsum);
    const int cb = bl.cbase[b];
    for (int l = t; l < nlb; l += NT) bl.chunk_start[lf + l] = cb + lpre[l];
    if (t == 0) lpre[nlb] = nchunks;
    __syncthreads();
    // BS_G lanes per chunk, each reading every BS_G-th record (coalesced
    // runs, all of a lane's loads in flight), then a shuffle reduction
    for (int q0 = 0; q0 < nchunks; q0 += NT / BS_G) {
      const int q = q0 + t / BS_G, g = t & (BS_G - 1);
      double xl = DINF, yl = DINF, xh = -DINF, yh = -DINF;
      if (q < nchunks) {
        int lo = 0, hi = nlb;  // the leaf: lpre[lo] <= q < lpre[lo + 1]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (lpre[mid] <= q) lo = mid; else hi = mid;
        }
        const int o0 = lcs[lo] + (q - lpre[lo]) * bl.chunk;
        const int oe = lo + 1 < nlb ? lcs[lo + 1] : be;
        const int o1 = min(o0 + bl.chunk, oe);
#pragma unroll
        for (int u = 0; u < MAX_CHUNK / BS_G; u++) {
          const int o = o0 + g + u * BS_G;
          if (o < o1) {
            const double2 p = *reinterpret_cast<const double2*>(&obj[o]);
            xl = fmin(xl, p.x);
            xh = fmax(xh, p.x);
            yl = fmin(yl, p.y);
            yh = fmax(yh, p.y);
          }
        }
      }
#pragma unroll
      for (int o = 1; o < BS_G; o <<= 1) {
        xl = fmin(xl, __shfl_xor_sync(FULL, xl, o));
        xh = fmax(xh, __shfl_xor_sync(FULL, xh, o));
        yl = fmin(yl, __shfl_xor_sync(FULL, yl, o));
        yh = fmax(yh, __shfl_xor_sync(FULL, yh, o));
      }
      if (q < nchunks && g == 0) bl.box[cb + q] = ChunkBox{xl, yl, xh, yh};
    }
    __syncthreads();
  }
}

// One-pass partition (steady state): the staging regions of the buckets
// are planned from the previous tick's bucket counts (or, after a rebuild,
// the build loads) with 1/8 + 256 records of slack, so the key pass and the
// partition are one kernel -- positions are read once.  A bucket that
// outgrows its region raises *overflow (records beyond it are dropped) and
// the tick is redone with the two-pass partition (exact counts).
__global__ void k_cap_plan(const uint32_t* __restrict__ prev, int32_t* __restrict__ sstart,
                           int32_t* __restrict__ cursor) {
  __shared__ int wt[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int c = (int)prev[t];
  const int v = c + c / 8 + 256;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) wt[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int sv = lane < PT_BUCKETS / 32 ? wt[lane] : 0;
    int si = sv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(FULL, si, o);
      if (lane >= o) si += u;
    }
    wt[lane] = si - sv;
  }
  __syncthreads();
  const int ex = inc - v + wt[w];
  sstart[t] = ex;
  cursor[t] = ex;
  if (t == PT_BUCKETS - 1) sstart[PT_BUCKETS] = ex + v;
}

// the key pass (k_point_keys) and the partition (k_partition) in one: a
// tile keys its objects, ranks them per bucket in shared memory and
// reserves one run per bucket in the planned regions
__global__ void __launch_bounds__(PT_THREADS) k_partition_keys(
    const long long* __restrict__ ids, const double* __restrict__ x, const double* __restrict__ y,
    int64_t n, Region r, const int32_t* __restrict__ scalars,
    const unsigned long long* __restrict__ cell_bucket,
    const int32_t* __restrict__ sstart, int32_t* __restrict__ cursor, StoreRec* __restrict__ out,
    unsigned long long* clamped, unsigned long long* overflow, int64_t index_base = 0) {
  __shared__ int hist[PT_BUCKETS], gbase[PT_BUCKETS];
  const int t = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * PT_TILE;
  const int tile_n = (n - base) < PT_TILE ? (int)(n - base) : PT_TILE;
  const int l_deep = scalars[0];
  for (int i = t; i < PT_BUCKETS; i += PT_THREADS) hist[i] = 0;
  StoreRec rc[PT_ITEMS];
  int bk[PT_ITEMS];
  unsigned outside_n = 0;
#pragma unroll
  for (int j = 0; j < PT_ITEMS; j++) {
    const int li = t + j * PT_THREADS;
    if (li < tile_n) {
      const int64_t i = base + li;
      rc[j].x = x[i];
      rc[j].y = y[i];
      rc[j].id = ids[i];
      rc[j].pad = (uint32_t)(index_base + i);  // input index (the snapshot slot on the delta path)
    }
  }
#pragma unroll
  for (int j = 0; j < PT_ITEMS; j++) {
    if (t + j * PT_THREADS < tile_n) {
      // geometry.py:215-220 count_outside
      outside_n += outside(rc[j].x, rc[j].y, r);
      uint32_t bkt, key;
      point_key(rc[j].x, rc[j].y, r, l_deep, cell_bucket, bkt, key);
      rc[j].key = key;
      bk[j] = (int)bkt;
    }
  }
  __syncthreads();
  int rank[PT_ITEMS];
#pragma unroll
  for (int j = 0; j < PT_ITEMS; j++)
    if (t + j * PT_THREADS < tile_n) rank[j] = atomicAdd(&hist[bk[j]], 1);
  __syncthreads();
  bool over = false;
  for (int i = t; i < PT_BUCKETS; i += PT_THREADS)
    if (hist[i]) {
      gbase[i] = atomicAdd(&cursor[i], hist[i]);
      over |= gbase[i] + hist[i] > sstart[i + 1];
    }
  if (over) atomicOr(overflow, 1ull);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PT_ITEMS; j++)
    if (t + j * PT_THREADS < tile_n) {
      const int pos = gbase[bk[j]] + rank[j];
      if (pos < sstart[bk[j] + 1]) st_rec(&out[pos], rc[j]);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) outside_n += __shfl_xor_sync(FULL, outside_n, o);
  if ((t & 31) == 0 && outside_n) atomicAdd(clamped, (unsigned long long)outside_n);
}

// after the one-pass partition: each bucket's count (clipped to its
// region), kept for the next tick's plan, and the store layout (bstart)
__global__ void k_bucket_counts(const int32_t* __restrict__ sstart, const int32_t* __restrict__ cursor,
                                uint32_t* __restrict__ counts, int32_t* __restrict__ bstart) {
  __shared__ int wt[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int v = min(cursor[t], sstart[t + 1]) - sstart[t];
  counts[t] = (uint32_t)v;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) wt[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int sv = lane < PT_BUCKETS / 32 ? wt[lane] : 0;
    int si = sv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(FULL, si, o);
      if (lane >= o) si += u;
    }
    wt[lane] = si - sv;
  }
  __syncthreads();
  const int ex = inc - v + wt[w];
  bstart[t] = ex;
  if (t == PT_BUCKETS - 1) bstart[PT_BUCKETS] = ex + v;
}

// two-pass partition: the exact bucket counts (k_point_keys' histogram,
// then scanned in place into cursor) for the next tick's plan
__global__ void k_save_counts(const int32_t* __restrict__ bstart, uint32_t* __restrict__ counts) {
  counts[threadIdx.x] = (uint32_t)(bstart[threadIdx.x + 1] - bstart[threadIdx.x]);
}

// chunk slot bases of the buckets: an upper bound of each bucket's chunks
// (ceil(objects / chunk) + its leaves), scanned (one CTA of PT_BUCKETS)
__global__ void k_chunk_base(const int32_t* __restrict__ bstart, const int32_t* __restrict__ leaf_first,
                             int chunk, int32_t* __restrict__ cbase) {
  __shared__ int wt[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int v = (bstart[t + 1] - bstart[t] + chunk - 1) / chunk + (leaf_first[t + 1] - leaf_first[t]);
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) wt[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int sv = lane < PT_BUCKETS / 32 ? wt[lane] : 0;
    int si = sv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(FULL, si, o);
      if (lane >= o) si += u;
    }
    wt[lane] = si - sv;
  }
  __syncthreads();
  cbase[t] = inc - v + wt[w];
}

// ---- incremental store update (delta ticks) -------------------------------
// The store is a counting sort by sub-cell key; between ticks only the moved
// snapshot slots change key.  New per-key counts = old counts - removed +
// added; surviving records keep their order inside their key group, so a
// record at old position i goes to kstart_new[key] + (i - kstart_old[key])
// - (removed before i in its group); moved records are appended to their new
// group after its survivors.  Same multiset per key as a full rebuild, order
// inside a key group differs -- nothing depends on it (canonical selection).
__global__ void k_key_counts(const int32_t* __restrict__ kstart, int64_t n_sub,
                             int32_t* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_sub;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = kstart[i + 1] - kstart[i];
}


// moved slot j: remove its old record (if it had one: found in its old key
// group, a handful of records, by the slot the record carries), key its new
// position; slot_key[slot] is every slot's key at the last (re)index.  A
// group longer than SCAN_MAX (dense clusters, coincident points) is not
// scanned: j is deferred to k_moved_deferred, which looks the record up in
// a slot -> position map that k_slot_map builds only when something was
// deferred (both return at once otherwise).
constexpr int SCAN_MAX = 64;

__device__ __forceinline__ void remove_old(int32_t p, const StoreRec* __restrict__ obj, const Region& r,
                                           int32_t* __restrict__ rmflag, unsigned long long* clamped) {
  rmflag[p] = 1;
  if (outside(obj[p].x, obj[p].y, r)) atomicAdd(clamped, ~0ull);  // -1
}

__global__ void k_moved_keys(const int32_t* __restrict__ moved, int64_t m, int64_t n_old_slots,
                             uint32_t* __restrict__ slot_key, const int32_t* __restrict__ kold,
                             const StoreRec* __restrict__ obj, const double* __restrict__ sx,
                             const double* __restrict__ sy, Region r,
                             const int32_t* __restrict__ scalars,
                             const unsigned long long* __restrict__ info,
                             int32_t* __restrict__ rmflag, int32_t* __restrict__ cnt,
                             uint32_t* __restrict__ mkey, unsigned long long* clamped,
                             int32_t* __restrict__ deferred, int32_t* __restrict__ n_deferred) {
  const int l_deep = scalars[0];
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t sl = moved[j];
    if (sl < n_old_slots) {
      const uint32_t ok = slot_key[sl];
      const int32_t b = kold[ok], e = kold[ok + 1];
      if (e - b > SCAN_MAX) {
        deferred[atomicAdd(n_deferred, 1)] = sl;
      } else {
        for (int32_t p = b; p < e; p++) {
          if ((int32_t)obj[p].pad == sl) {
            remove_old(p, obj, r, rmflag, clamped);
            break;
          }
        }
      }
      atomicSub(&cnt[ok], 1);
    }
    const double x = sx[sl], y = sy[sl];
    uint32_t leaf, key;
    point_key(x, y, r, l_deep, info, leaf, key);
    mkey[j] = key;
    slot_key[sl] = key;
    atomicAdd(&cnt[key], 1);
    if (outside(x, y, r)) atomicAdd(clamped, 1ull);
  }
}

__global__ void k_slot_map(const StoreRec* __restrict__ obj, int64_t n_old,
                           const int32_t* __restrict__ n_deferred, int32_t* __restrict__ slot_pos) {
  if (*n_deferred == 0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_old;
       i += (int64_t)gridDim.x * blockDim.x)
    slot_pos[obj[i].pad] = (int32_t)i;
}

__global__ void k_moved_deferred(const int32_t* __restrict__ deferred,
                                 const int32_t* __restrict__ n_deferred,
                                 const int32_t* __restrict__ slot_pos,
                                 const StoreRec* __restrict__ obj, Region r,
                                 int32_t* __restrict__ rmflag, unsigned long long* clamped) {
  const int64_t nd = *n_deferred;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nd;
       j += (int64_t)gridDim.x * blockDim.x)
    remove_old(slot_pos[deferred[j]], obj, r, rmflag, clamped);
}

__global__ void k_move_survivors(const StoreRec* __restrict__ obj, int64_t n_old,
                                 const int32_t* __restrict__ rmflag,
                                 const int32_t* __restrict__ rm_before,
                                 const int32_t* __restrict__ kold, const int32_t* __restrict__ knew,
                                 StoreRec* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_old;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (rmflag[i]) continue;
    const StoreRec rc = ld_rec(&obj[i]);
    const int32_t g = kold[rc.key];
    st_rec(&out[knew[rc.key] + ((int32_t)i - g) - (rm_before[i] - rm_before[g])], rc);
  }
}

__global__ void k_insert_moved(const int32_t* __restrict__ moved, int64_t m,
                               const uint32_t* __restrict__ mkey, const long long* __restrict__ sids,
                               const double* __restrict__ sx, const double* __restrict__ sy,
                               const int32_t* __restrict__ kold, const int32_t* __restrict__ knew,
                               const int32_t* __restrict__ rm_before, int32_t* __restrict__ fill,
                               StoreRec* __restrict__ out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t sl = moved[j];
    const uint32_t key = mkey[j];
    const int32_t g0 = kold[key], g1 = kold[key + 1];
    const int32_t surv = (g1 - g0) - (rm_before[g1] - rm_before[g0]);
    const int32_t np = knew[key] + surv + atomicAdd(&fill[key], 1);
    StoreRec rc;
    rc.x = sx[sl];
    rc.y = sy[sl];
    rc.id = sids[sl];
    rc.key = key;
    rc.pad = (uint32_t)sl;
    st_rec(&out[np], rc);
  }
}

__global__ void k_fill_reset(const uint32_t* __restrict__ mkey, int64_t m, int32_t* __restrict__ fill) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x)
    fill[mkey[j]] = 0;
}

__global__ void k_q_scatter(int64_t nq, const uint32_t* __restrict__ key,
                            const int32_t* __restrict__ start, int32_t* __restrict__ cnt,
                            uint32_t* __restrict__ order) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t kk = key[i];
    order[start[kk] + atomicSub(&cnt[kk], 1) - 1] = (uint32_t)i;
  }
}

// leaf ranges from the sub-cell starts: cell_start[l] and chunks per leaf
__global__ void k_leaf_ranges(const int32_t* __restrict__ kstart, const int32_t* __restrict__ sub_base,
                              int64_t n_leaves, int chunk, int32_t* __restrict__ cell_start,
                              int32_t* __restrict__ nch) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l <= n_leaves) {
    const int32_t b = kstart[sub_base[l]];
    cell_start[l] = b;
    if (l < n_leaves) nch[l] = (kstart[sub_base[l + 1]] - b + chunk - 1) / chunk;
  }
}

// per leaf: the object range of each of its chunks
__global__ void k_chunk_ranges(const int32_t* __restrict__ cell_start,
                               const int32_t* __restrict__ chunk_start, int64_t n_leaves,
                               int chunk, int2* __restrict__ crange) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l < n_leaves) {
    const int b = cell_start[l], e = cell_start[l + 1];
    int c = chunk_start[l];
    for (int o = b; o < e; o += chunk, c++) crange[c] = make_int2(o, min(o + chunk, e));
  }
}

// one thread per chunk: point bounding box (a chunk is 1 KB of contiguous
// records, so each thread's loads stream through its own L1 lines)
__global__ void k_chunk_boxes(const StoreRec* __restrict__ obj, const int2* __restrict__ crange,
                              const int32_t* __restrict__ n_chunks_dev, ChunkBox* __restrict__ box) {
  const int64_t nc = *n_chunks_dev;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nc;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int2 rg = crange[c];
    double xl = DINF, yl = DINF, xh = -DINF, yh = -DINF;
    for (int o = rg.x; o < rg.y; o++) {
      const double2 p = *reinterpret_cast<const double2*>(&obj[o]);
      xl = fmin(xl, p.x);
      xh = fmax(xh, p.x);
      yl = fmin(yl, p.y);
      yh = fmax(yh, p.y);
    }
    box[c] = ChunkBox{xl, yl, xh, yh};
  }
}

// rebuild: 4^s sub-cells per leaf with s the smallest level count that
// leaves <= 4 build-time objects per sub-cell (s <= 5, and the table of all
// leaves' sub-cells capped at 2^24 counters so its atomics stay in L2)
__global__ void k_leaf_subs(const int32_t* __restrict__ build_counts,
                            const int32_t* __restrict__ scalars, int64_t ncap,
                            uint8_t* __restrict__ sub_bits, int32_t* __restrict__ sub_size) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= ncap) return;
  if (l >= scalars[1]) {
    sub_size[l] = 0;
    return;
  }
  // cap: the whole sub-cell table stays <= 2^24 counters (L2-resident)
  const int64_t nl = scalars[1];
  int cap = 0;
  while (cap < 5 && (nl << (2 * (cap + 1))) <= (int64_t(1) << 24)) cap++;
  const int c = build_counts[l];
  int sl = 0;
  while (sl < cap && c > (4 << (2 * sl))) sl++;
  sub_bits[l] = (uint8_t)(2 * sl);
  sub_size[l] = 1 << (2 * sl);
}

// rebuild: partition buckets for the bucket-local store sort, aligned to
// leaves and balanced by the build counts -- leaf l goes to bucket
// floor(objects before l * NB / n_build), bucket b holds the keys
// [bkey[b], bkey[b + 1]) -- so a dense leaf whose sub-cells are capped does
// not pile its objects into one bucket.  pre: exclusive scan of the build
// counts (0 past the last leaf)
__global__ void k_leaf_bucket(const int32_t* __restrict__ pre, const int32_t* __restrict__ sub_base,
                              const int32_t* __restrict__ scalars, int64_t ncap,
                              uint16_t* __restrict__ leaf_bucket, int32_t* __restrict__ bkey,
                              int32_t* __restrict__ leaf_first) {
  const int64_t nl = scalars[1], n_sub = scalars[4];
  const int64_t nb = scalars[3] > 0 ? scalars[3] : 1;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l <= nl && l < ncap + 1;
       l += (int64_t)gridDim.x * blockDim.x) {
    const int b = l < nl ? (int)min((int64_t)pre[l] * PT_BUCKETS / nb, (int64_t)PT_BUCKETS - 1)
                         : PT_BUCKETS;
    const int bp = l == 0 ? -1 : (int)min((int64_t)pre[l - 1] * PT_BUCKETS / nb, (int64_t)PT_BUCKETS - 1);
    if (l < nl) leaf_bucket[l] = (uint16_t)b;
    const int32_t k0 = l < nl ? sub_base[l] : (int32_t)n_sub;
    for (int bb = bp + 1; bb <= b; bb++) {  // buckets this leaf opens
      bkey[bb] = k0;
      leaf_first[bb] = (int32_t)l;
    }
  }
}

// the largest key count and leaf count of a bucket -> scalars[6], [7] (the
// bucket-local sort keeps both in shared memory)
__global__ void k_bucket_keys(const int32_t* __restrict__ bkey, const int32_t* __restrict__ leaf_first,
                              int32_t* __restrict__ scalars) {
  __shared__ int wk[PT_BUCKETS / 32], wl[PT_BUCKETS / 32];
  const int b = threadIdx.x;
  int mk = bkey[b + 1] - bkey[b], ml = leaf_first[b + 1] - leaf_first[b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mk = max(mk, __shfl_xor_sync(FULL, mk, o));
    ml = max(ml, __shfl_xor_sync(FULL, ml, o));
  }
  if ((b & 31) == 0) {
    wk[b >> 5] = mk;
    wl[b >> 5] = ml;
  }
  __syncthreads();
  if (b == 0) {
    int m = 0, l = 0;
    for (int i = 0; i < PT_BUCKETS / 32; i++) {
      m = max(m, wk[i]);
      l = max(l, wl[i]);
    }
    scalars[6] = m <= BS_MAX_KEYS && l <= BS_MAX_LEAVES ? m : 0x7fffffff;  // > limit: no bucket sort
    scalars[7] = l;
  }
}

// the build load of every bucket -> scalars[5] (largest, 1/16 of the mean)
__global__ void k_bucket_load(const int32_t* __restrict__ build_counts,
                              const uint16_t* __restrict__ leaf_bucket,
                              const int32_t* __restrict__ scalars, int64_t ncap,
                              uint32_t* __restrict__ load) {
  const int64_t nl = scalars[1];
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < nl && l < ncap;
       l += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&load[leaf_bucket[l]], (uint32_t)build_counts[l]);
}

__global__ void k_bucket_load_max(const uint32_t* __restrict__ load, int32_t* __restrict__ scalars) {
  __shared__ uint32_t wmax[PT_BUCKETS / 32];
  uint32_t v = load[threadIdx.x];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t m = 0;
    for (int i = 0; i < PT_BUCKETS / 32; i++) m = max(m, wmax[i]);
    const double mean = (double)max(scalars[3], 1) / PT_BUCKETS;
    scalars[5] = (int32_t)min(16.0 * (double)m / mean, 1e9);
  }
}

// build counts of the leaves, 0 past the last one (the scan input)
__global__ void k_leaf_counts(const int32_t* __restrict__ build_counts,
                              const int32_t* __restrict__ scalars, int64_t ncap,
                              int32_t* __restrict__ out) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l < ncap) out[l] = l < scalars[1] ? build_counts[l] : 0;
}

__global__ void k_store_scalar(int32_t* scalars, const int32_t* __restrict__ src, int64_t idx) {
  scalars[4] = src[idx];
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

// Row order without a sort when the issuers are distinct: one bit per id of
// [min, min + 2^bits) marks the batch's ids; a query's row is the number of
// marked ids below its own (popcount prefix over words) -- the stable issuer
// rank of engine.py:713 when no id repeats.  A repeated id raises bit 0 of
// *dup (the engine switches to the radix sort for good), an id beyond the
// planned range (planned from the previous tick) raises bit 1; either way
// the tick is redone.
constexpr int32_t DUP_REPEATED = 1, DUP_OUT_OF_SPAN = 2;

__global__ void k_issuer_mark(const long long* __restrict__ qi, int64_t nq,
                              const int64_t* __restrict__ mm, uint64_t span,
                              uint32_t* __restrict__ bm, int32_t* __restrict__ dup) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) {
    const uint64_t key = (uint64_t)qi[i] - (uint64_t)mm[0];
    if (key >= span) {
      atomicOr(dup, DUP_OUT_OF_SPAN);
      return;
    }
    const uint32_t bit = 1u << (key & 31);
    if (atomicOr(&bm[key >> 5], bit) & bit) atomicOr(dup, DUP_REPEATED);
  }
}

__global__ void k_word_popc(const uint32_t* __restrict__ bm, int64_t nw, int32_t* __restrict__ cnt) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w < nw) cnt[w] = __popc(bm[w]);
}

__global__ void k_issuer_rank(const long long* __restrict__ qi, int64_t nq,
                              const int64_t* __restrict__ mm, uint64_t span,
                              const uint32_t* __restrict__ bm, const int32_t* __restrict__ pre,
                              uint32_t* __restrict__ row, long long* __restrict__ out_qids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) {
    const uint64_t key = (uint64_t)qi[i] - (uint64_t)mm[0];
    if (key >= span) {  // the tick is redone (dup flag); keep the row in bounds meanwhile
      row[i] = 0;
      return;
    }
    const int64_t w = (int64_t)(key >> 5);
    const uint32_t r = (uint32_t)pre[w] + (uint32_t)__popc(bm[w] & ((1u << (key & 31)) - 1u));
    row[i] = r;
    if (out_qids && r < (uint64_t)nq) out_qids[r] = qi[i];
  }
}

inline unsigned grid_stride_blocks(int64_t n, int64_t max_blocks = 148 * 16) {
  int64_t b = (n + TPB - 1) / TPB;
  return (unsigned)std::min<int64_t>(std::max<int64_t>(b, 1), max_blocks);
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
  MKNN_CUDA_OK(cudaMalloc(&ix.leaf_sub_bits, ncap));
  MKNN_CUDA_OK(cudaMalloc(&ix.leaf_sub_base, sizeof(int32_t) * (ncap + 1)));
  MKNN_CUDA_OK(cudaMalloc(&ix.cell_info, sizeof(unsigned long long) * ncap));
  MKNN_CUDA_OK(cudaMalloc(&ix.bload, sizeof(uint32_t) * PT_BUCKETS));
  MKNN_CUDA_OK(cudaMalloc(&ix.bkey, sizeof(int32_t) * (PT_BUCKETS + 1)));
  MKNN_CUDA_OK(cudaMalloc(&ix.leaf_first, sizeof(int32_t) * (PT_BUCKETS + 1)));
  MKNN_CUDA_OK(cudaMalloc(&ix.leaf_bucket, sizeof(uint16_t) * ncap));
  MKNN_CUDA_OK(cudaMalloc(&ix.cell_bucket, sizeof(unsigned long long) * ncap));
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
  cudaFree(ix.leaf_sub_bits);
  cudaFree(ix.leaf_sub_base);
  cudaFree(ix.cell_info);
  cudaFree(ix.bload);
  cudaFree(ix.bkey);
  cudaFree(ix.leaf_first);
  cudaFree(ix.leaf_bucket);
  cudaFree(ix.cell_bucket);
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
  // store ordering tables (sub-cells per leaf, their key ranges)
  MKNN_LAUNCH k_leaf_subs<<<blocks_for(ncap), TPB, 0, s>>>(ix.build_counts, ix.scalars, ncap,
                                                          ix.leaf_sub_bits, flags);
  MKNN_CUDA_OK(cudaGetLastError());
  rc = exclusive_scan_i32(flags, ix.leaf_sub_base, ncap, scratch, s);
  if (rc) return rc;
  MKNN_LAUNCH k_store_scalar<<<1, 1, 0, s>>>(ix.scalars, ix.leaf_sub_base, ncap);
  MKNN_LAUNCH k_cell_info<<<blocks_for(ncap), TPB, 0, s>>>(ix.z_map, ix.scalars, ix.leaf_level,
                                                          ix.leaf_sub_bits, ix.leaf_sub_base, ncap,
                                                          ix.cell_info);
  MKNN_CUDA_OK(cudaGetLastError());
  // n_build for should_rebuild bookkeeping
  int32_t nb = (int32_t)std::min<int64_t>(n, 0x7fffffff);
  MKNN_CUDA_OK(cudaMemcpyAsync(ix.scalars + 3, &nb, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  // leaf-aligned, load-balanced partition buckets (bucket-local sort) and
  // their balance (scalars[5], [6]); scratch: flags (the scan is done)
  int32_t* lc = flags;
  int32_t* pre = flags + ncap + 1;
  MKNN_LAUNCH k_leaf_counts<<<blocks_for(ncap), TPB, 0, s>>>(ix.build_counts, ix.scalars, ncap, lc);
  MKNN_CUDA_OK(cudaGetLastError());
  rc = exclusive_scan_i32(lc, pre, ncap, scratch, s);
  if (rc) return rc;
  MKNN_LAUNCH k_leaf_bucket<<<blocks_for(ncap + 1), TPB, 0, s>>>(pre, ix.leaf_sub_base, ix.scalars, ncap,
                                                                ix.leaf_bucket, ix.bkey,
                                                                ix.leaf_first);
  MKNN_LAUNCH k_cell_bucket<<<blocks_for(ncap), TPB, 0, s>>>(ix.cell_info, ix.leaf_bucket, ix.scalars,
                                                            ncap, ix.cell_bucket);
  MKNN_CUDA_OK(cudaMemsetAsync(ix.bload, 0, sizeof(uint32_t) * PT_BUCKETS, s));
  MKNN_LAUNCH k_bucket_load<<<blocks_for(ncap), TPB, 0, s>>>(ix.build_counts, ix.leaf_bucket,
                                                             ix.scalars, ncap, ix.bload);
  MKNN_LAUNCH k_bucket_load_max<<<1, PT_BUCKETS, 0, s>>>(ix.bload, ix.scalars);
  MKNN_LAUNCH k_bucket_keys<<<1, PT_BUCKETS, 0, s>>>(ix.bkey, ix.leaf_first, ix.scalars);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

int store_reserve(DevStore& st, int64_t n_sub, int64_t n_leaves, int64_t n) {
  const int64_t need = std::max<int64_t>(n_sub, 1) + 2;
  if (need > st.cap_sub) {
    int32_t** arrs[] = {&st.cnt, &st.kstart, &st.kstart_alt, &st.fill, &st.qcnt, &st.qkstart};
    for (auto a : arrs) {
      cudaFree(*a);
      *a = nullptr;
    }
    st.cap_sub = 0;
    const int64_t c = std::max<int64_t>(need, st.cap_sub * 3 / 2);
    for (auto a : arrs) MKNN_CUDA_OK(cudaMalloc(a, sizeof(int32_t) * c));
    MKNN_CUDA_OK(cudaMemset(st.fill, 0, sizeof(int32_t) * c));
    MKNN_CUDA_OK(cudaMemset(st.qcnt, 0, sizeof(int32_t) * c));
    st.cap_sub = c;
    st.dirty = true;
    st.valid = false;
  }
  if (!st.cursor) {
    MKNN_CUDA_OK(cudaMalloc(&st.cursor, sizeof(int32_t) * (PT_BUCKETS + 1)));
    MKNN_CUDA_OK(cudaMalloc(&st.bstart, sizeof(int32_t) * (PT_BUCKETS + 1)));
    MKNN_CUDA_OK(cudaMalloc(&st.cbase, sizeof(int32_t) * (PT_BUCKETS + 1)));
    MKNN_CUDA_OK(cudaMalloc(&st.sstart, sizeof(int32_t) * (PT_BUCKETS + 1)));
    MKNN_CUDA_OK(cudaMalloc(&st.bcnt, sizeof(uint32_t) * PT_BUCKETS));
  }
  const int64_t nbox = n / (MAX_CHUNK / 2) + n_leaves + PT_BUCKETS + 1;  // + per-bucket slot rounding
  if (nbox > st.cap_box) {
    cudaFree(st.box);
    cudaFree(st.crange);
    st.box = nullptr;
    st.crange = nullptr;
    st.cap_box = 0;
    const int64_t c = std::max<int64_t>(nbox, st.cap_box * 3 / 2);
    MKNN_CUDA_OK(cudaMalloc(&st.box, sizeof(ChunkBox) * c));
    MKNN_CUDA_OK(cudaMalloc(&st.crange, sizeof(int2) * c));
    st.cap_box = c;
  }
  return 0;
}

// cell_start, chunk ranges and chunk boxes from st.kstart and st.obj
static int store_finish(DevStore& st, const DevIndex& ix, int64_t n, int64_t n_leaves,
                        void* scratch, cudaStream_t s) {
  MKNN_LAUNCH k_leaf_ranges<<<blocks_for(n_leaves + 1), TPB, 0, s>>>(st.kstart, ix.leaf_sub_base,
                                                                    n_leaves, st.chunk, st.cell_start,
                                                                    st.nch);
  MKNN_CUDA_OK(cudaGetLastError());
  int rc = exclusive_scan_i32(st.nch, st.chunk_start, n_leaves, scratch, s);
  if (rc) return rc;
  if (n > 0) {
    MKNN_LAUNCH k_chunk_ranges<<<blocks_for(n_leaves), TPB, 0, s>>>(st.cell_start, st.chunk_start,
                                                                   n_leaves, st.chunk, st.crange);
    const int64_t maxc = n / st.chunk + n_leaves + 1;
    MKNN_LAUNCH k_chunk_boxes<<<blocks_for(maxc), TPB, 0, s>>>(st.obj, st.crange,
                                                              st.chunk_start + n_leaves, st.box);
  }
  MKNN_CUDA_OK(cudaGetLastError());
  st.n_store = n;
  return 0;
}

// the one-pass partition of the objects [lo, hi) (plan: first call of a
// tick: lay out the bucket regions); a host tick runs it per chunk while the
// next chunk crosses PCIe, and store_index_objects then starts from the
// partitioned records (pre != nullptr)
int store_prepartition(DevStore& st, const DevIndex& ix, const Region& r, const long long* ids,
                       const double* x, const double* y, int64_t lo, int64_t hi, bool plan,
                       unsigned long long* pre, cudaStream_t s) {
  if (plan) MKNN_LAUNCH k_cap_plan<<<1, PT_BUCKETS, 0, s>>>(st.bcnt, st.sstart, st.cursor);
  if (hi > lo)
    MKNN_LAUNCH k_partition_keys<<<(unsigned)((hi - lo + PT_TILE - 1) / PT_TILE), PT_THREADS, 0, s>>>(
        ids + lo, x + lo, y + lo, hi - lo, r, ix.scalars, ix.cell_bucket, st.sstart,
        st.cursor, st.rec, pre, pre + 1, lo);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

int store_index_objects(DevStore& st, const DevIndex& ix, const Region& r, const long long* ids,
                        const double* x, const double* y, int64_t n, int64_t n_leaves,
                        int64_t n_sub, bool balanced, int max_keys, int max_leaves, bool two_pass,
                        unsigned long long* dev_clamped, unsigned long long* dev_overflow,
                        void* scratch, cudaStream_t s, const unsigned long long* pre) {
  // MKNN_BSORT=0: the global-atomic counting sort (per-key counts in the
  // key pass, a scan over all sub-cells, an atomic final scatter) for A/B
  static const bool bsort = [] {
    const char* e = getenv("MKNN_BSORT");
    return !(e && e[0] == '0');
  }();
  int bshift = 0;
  while ((std::max<int64_t>(n_sub, 1) - 1) >> bshift >= PT_BUCKETS) bshift++;
  // <= 2^24 sub-cells: a 64 KB histogram; buckets of <= 32K records (1 MB)
  // so the second sweep still finds them in L2 (100M objects: 6.20 -> 6.32 ms)
  // larger buckets than ~32K records (1 MB) no longer stay in L2 between
  // the sort's sweeps, but the bucket sort still edges out the atomic
  // scatter (100M objects: 6.30 -> 6.18 ms); MKNN_BSORT_BIG=0 keeps those
  // on the atomic path (A/B)
  static const bool big = [] {
    const char* e = getenv("MKNN_BSORT_BIG");
    return !(e && e[0] == '0');
  }();
  if (bsort && balanced && (big || n <= (int64_t)PT_BUCKETS * 32768) && n > 0) {
    // MKNN_ONEPASS=0: always the two-pass partition (A/B)
    static const bool onepass = [] {
      const char* e = getenv("MKNN_ONEPASS");
      return !(e && e[0] == '0');
    }();
    const int32_t* sstart = st.bstart;  // two-pass: staging and store share the layout
    if (onepass && st.bcnt_valid && !two_pass) {
      if (pre) {  // partitioned while the objects arrived: take its counters
        MKNN_CUDA_OK(cudaMemcpyAsync(dev_clamped, pre, sizeof(unsigned long long),
                                     cudaMemcpyDeviceToDevice, s));
        MKNN_CUDA_OK(cudaMemcpyAsync(dev_overflow, pre + 1, sizeof(unsigned long long),
                                     cudaMemcpyDeviceToDevice, s));
      } else {
        MKNN_LAUNCH k_cap_plan<<<1, PT_BUCKETS, 0, s>>>(st.bcnt, st.sstart, st.cursor);
        MKNN_LAUNCH k_partition_keys<<<(unsigned)((n + PT_TILE - 1) / PT_TILE), PT_THREADS, 0, s>>>(
            ids, x, y, n, r, ix.scalars, ix.cell_bucket, st.sstart, st.cursor, st.rec,
            dev_clamped, dev_overflow);
      }
      MKNN_LAUNCH k_bucket_counts<<<1, PT_BUCKETS, 0, s>>>(st.sstart, st.cursor, st.bcnt, st.bstart);
      sstart = st.sstart;
    } else {
      MKNN_CUDA_OK(cudaMemsetAsync(st.cursor, 0, sizeof(int32_t) * PT_BUCKETS, s));
      MKNN_LAUNCH k_point_keys<<<grid_stride_blocks(n), TPB, 0, s>>>(
          x, y, n, r, ix.scalars, ix.cell_info, nullptr, st.key, nullptr, dev_clamped, bshift,
          st.cursor, ix.leaf_bucket, st.bkt);
      MKNN_CUDA_OK(cudaGetLastError());
      MKNN_LAUNCH k_bucket_scan<<<1, PT_BUCKETS, 0, s>>>(st.cursor, st.bstart, st.cursor);
      MKNN_LAUNCH k_partition<<<(unsigned)((n + PT_TILE - 1) / PT_TILE), PT_THREADS, 0, s>>>(
          ids, x, y, st.key, n, bshift, st.cursor, st.rec, st.bkt);
      MKNN_LAUNCH k_save_counts<<<1, PT_BUCKETS, 0, s>>>(st.bstart, st.bcnt);
      st.bcnt_valid = true;
    }
    MKNN_CUDA_OK(cudaGetLastError());
    // small ticks (buckets of ~4K records at most) with <= 16K keys and 4K
    // leaves per bucket: two 512-thread CTAs per SM (1M objects: 89 -> 79
    // us; at 10M objects the 1024-thread CTAs win, 442 vs 501 us)
    const bool small = n <= (int64_t)PT_BUCKETS * 4096 && max_keys <= BS_MAX_KEYS / 2 &&
                       max_leaves <= BS_MAX_LEAVES / 2;
    const size_t smem = small ? sizeof(int32_t) * (BS_MAX_KEYS / 2 + BS_MAX_LEAVES + 1)
                              : sizeof(int32_t) * (BS_MAX_KEYS + 2 * BS_MAX_LEAVES + 1);
    static unsigned long long configured = 0;  // bit d: the attributes are set on device d
    int dev = 0;
    MKNN_CUDA_OK(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
      MKNN_CUDA_OK(cudaFuncSetAttribute(k_bucket_sort<1024, BS_MAX_KEYS, BS_MAX_LEAVES>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(sizeof(int32_t) * (BS_MAX_KEYS + 2 * BS_MAX_LEAVES + 1))));
      MKNN_CUDA_OK(cudaFuncSetAttribute(k_bucket_sort<512, BS_MAX_KEYS / 2, BS_MAX_LEAVES / 2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(sizeof(int32_t) * (BS_MAX_KEYS / 2 + BS_MAX_LEAVES + 1))));
      __atomic_fetch_or(&configured, bit, __ATOMIC_ACQ_REL);
    }
    int sms = 148;
    MKNN_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MKNN_LAUNCH k_chunk_base<<<1, PT_BUCKETS, 0, s>>>(st.bstart, ix.leaf_first, st.chunk, st.cbase);
    // MKNN_BS_PREFETCH=1|2: bulk L2 prefetch of the next bucket (A/B)
    static const int prefetch = [] {
      const char* e = getenv("MKNN_BS_PREFETCH");
      return e ? atoi(e) : 0;
    }();
    BucketLeaves bl{ix.leaf_first, ix.leaf_sub_base, st.cbase, st.cell_start, st.chunk_start,
                    st.box, st.chunk, n_leaves, prefetch};
    if (small)
      MKNN_LAUNCH k_bucket_sort<512, BS_MAX_KEYS / 2, BS_MAX_LEAVES / 2><<<(unsigned)(2 * sms), 512, smem, s>>>(
          st.rec, st.bstart, sstart, ix.bkey, n_sub, n, st.kstart, st.obj, bl);
    else
      MKNN_LAUNCH k_bucket_sort<1024, BS_MAX_KEYS, BS_MAX_LEAVES><<<(unsigned)sms, 1024, smem, s>>>(
          st.rec, st.bstart, sstart, ix.bkey, n_sub, n, st.kstart, st.obj, bl);
    MKNN_CUDA_OK(cudaGetLastError());
    st.n_store = n;
    return 0;
  }
  if (st.dirty) {
    MKNN_CUDA_OK(cudaMemsetAsync(st.cnt, 0, sizeof(int32_t) * st.cap_sub, s));
    st.dirty = false;
  }
  MKNN_CUDA_OK(cudaMemsetAsync(st.cursor, 0, sizeof(int32_t) * PT_BUCKETS, s));
  if (n > 0)
    MKNN_LAUNCH k_point_keys<<<grid_stride_blocks(n), TPB, 0, s>>>(
        x, y, n, r, ix.scalars, ix.cell_info, nullptr, st.key, st.cnt, dev_clamped, bshift,
        st.cursor);
  MKNN_CUDA_OK(cudaGetLastError());
  MKNN_LAUNCH k_bucket_scan<<<1, PT_BUCKETS, 0, s>>>(st.cursor, st.bstart, st.cursor);
  if (n > 0) {
    MKNN_LAUNCH k_partition<<<(unsigned)((n + PT_TILE - 1) / PT_TILE), PT_THREADS, 0, s>>>(
        ids, x, y, st.key, n, bshift, st.cursor, st.rec);
    MKNN_CUDA_OK(cudaGetLastError());
  }
  int rc = exclusive_scan_i32(st.cnt, st.kstart, n_sub, scratch, s);
  if (rc) return rc;
  if (n > 0)
    MKNN_LAUNCH k_final_scatter<<<grid_stride_blocks(n, 148 * 64), TPB, 0, s>>>(st.rec, n, st.kstart, st.cnt,
                                                                     st.obj);
  MKNN_CUDA_OK(cudaGetLastError());
  return store_finish(st, ix, n, n_leaves, scratch, s);
}

int store_update_incremental(DevStore& st, const DevIndex& ix, const Region& r,
                             const long long* sids, const double* sx, const double* sy,
                             int64_t n_new, const int32_t* moved, int64_t m, int64_t n_leaves,
                             int64_t n_sub, unsigned long long* dev_clamped_total, void* scratch,
                             cudaStream_t s) {
  const int64_t n_old = st.n_store;
  // cnt <- the current per-key counts, then -removed +added
  MKNN_LAUNCH k_key_counts<<<grid_stride_blocks(n_sub), TPB, 0, s>>>(st.kstart, n_sub, st.cnt);
  st.dirty = true;  // cnt no longer all zero
  MKNN_CUDA_OK(cudaMemsetAsync(st.rmflag, 0, sizeof(int32_t) * (n_old + 1), s));
  if (m > 0) {
    MKNN_CUDA_OK(cudaMemsetAsync(st.n_deferred, 0, sizeof(int32_t), s));
    MKNN_LAUNCH k_moved_keys<<<grid_stride_blocks(m), TPB, 0, s>>>(
        moved, m, n_old, st.key, st.kstart, st.obj, sx, sy, r, ix.scalars, ix.cell_info, st.rmflag,
        st.cnt, st.mkey, dev_clamped_total, st.deferred, st.n_deferred);
    MKNN_LAUNCH k_slot_map<<<grid_stride_blocks(n_old), TPB, 0, s>>>(st.obj, n_old, st.n_deferred,
                                                                    st.slot_pos);
    MKNN_LAUNCH k_moved_deferred<<<grid_stride_blocks(m), TPB, 0, s>>>(
        st.deferred, st.n_deferred, st.slot_pos, st.obj, r, st.rmflag, dev_clamped_total);
  }
  MKNN_CUDA_OK(cudaGetLastError());
  int rc = exclusive_scan_i32(st.cnt, st.kstart_alt, n_sub, scratch, s);
  if (rc) return rc;
  rc = exclusive_scan_i32(st.rmflag, st.rm_before, n_old, scratch, s);
  if (rc) return rc;
  if (n_old > 0)
    MKNN_LAUNCH k_move_survivors<<<grid_stride_blocks(n_old), TPB, 0, s>>>(
        st.obj, n_old, st.rmflag, st.rm_before, st.kstart, st.kstart_alt, st.rec);
  if (m > 0) {
    MKNN_LAUNCH k_insert_moved<<<grid_stride_blocks(m), TPB, 0, s>>>(
        moved, m, st.mkey, sids, sx, sy, st.kstart, st.kstart_alt, st.rm_before, st.fill, st.rec);
    MKNN_LAUNCH k_fill_reset<<<grid_stride_blocks(m), TPB, 0, s>>>(st.mkey, m, st.fill);
  }
  MKNN_CUDA_OK(cudaGetLastError());
  std::swap(st.obj, st.rec);
  std::swap(st.kstart, st.kstart_alt);
  return store_finish(st, ix, n_new, n_leaves, scratch, s);
}

int issuer_bits(int64_t lo, int64_t hi) {
  const uint64_t range = (uint64_t)hi - (uint64_t)lo;
  return range ? 64 - __builtin_clzll(range) : 0;
}

int queries_index(DevQueries& dq, DevStore& st, const DevIndex& ix, const Region& r,
                  const long long* qi, const double* qx, const double* qy, int64_t nq,
                  int64_t n_sub, int plan_bits, int* bits_used, bool bitmap, long long* out_qids, void* scratch,
                  cudaStream_t s) {
  *bits_used = 0;
  if (nq == 0) return 0;
  // leaf-grouped order with sub-cell order inside (consecutive queries are
  // neighbours: the own-pass cap and L1): a counting sort over groups of
  // 2^qs consecutive sub-cells, about one query per group, so the scan
  // covers n_sub >> qs entries instead of every sub-cell (cfg3: 15M -> 1.9M)
  int qs = 0;
  while (qs < 8 && (n_sub >> (qs + 1)) >= std::max<int64_t>(nq, 1)) qs++;
  const int64_t n_grp = ((n_sub - 1) >> qs) + 1;
  MKNN_LAUNCH k_point_keys<<<grid_stride_blocks(nq), TPB, 0, s>>>(
      qx, qy, nq, r, ix.scalars, ix.cell_info, dq.leaf, dq.qkey, st.qcnt, nullptr, 0, nullptr,
      nullptr, nullptr, qs);
  MKNN_CUDA_OK(cudaGetLastError());
  int rc = exclusive_scan_i32(st.qcnt, st.qkstart, n_grp, scratch, s);
  if (rc) return rc;
  MKNN_LAUNCH k_q_scatter<<<grid_stride_blocks(nq), TPB, 0, s>>>(nq, dq.qkey, st.qkstart, st.qcnt,
                                                                dq.order);
  MKNN_CUDA_OK(cudaGetLastError());

  // stable issuer order for emission (engine.py:713 / oracle.py:56): LSD
  // radix sort of (issuer - min) over plan_bits bits.  plan_bits < 0: read
  // the range first (one host sync); otherwise the caller planned from the
  // previous tick and checks dq.minmax after the tick (mknn_api.cu retries
  // the tick if the range needed more bits).
  rc = minmax_i64((const int64_t*)qi, nq, dq.minmax, s);
  if (rc) return rc;
  int bits = plan_bits;
  if (bits < 0) {
    int64_t mm[2];
    MKNN_CUDA_OK(cudaMemcpyAsync(mm, dq.minmax, sizeof(mm), cudaMemcpyDeviceToHost, s));
    MKNN_CUDA_OK(cudaStreamSynchronize(s));
    bits = issuer_bits(mm[0], mm[1]);
  }
  *bits_used = bits;
  if (bitmap && bits <= 27) {  // distinct issuers expected: rank by bitmap (<= 16 MB)
    const uint64_t span = 1ull << bits;
    const int64_t nw = (int64_t)((span + 31) >> 5);
    if (nw + 1 > dq.bm_cap || !dq.dup) {
      cudaFree(dq.bm);
      cudaFree(dq.bm_cnt);
      cudaFree(dq.bm_pre);
      if (!dq.dup) MKNN_CUDA_OK(cudaMalloc(&dq.dup, sizeof(int32_t)));
      dq.bm_cap = 0;
      const int64_t c = std::max<int64_t>(nw + 1, 1024);
      MKNN_CUDA_OK(cudaMalloc(&dq.bm, sizeof(uint32_t) * c));
      MKNN_CUDA_OK(cudaMalloc(&dq.bm_cnt, sizeof(int32_t) * c));
      MKNN_CUDA_OK(cudaMalloc(&dq.bm_pre, sizeof(int32_t) * (c + 1)));
      dq.bm_cap = c;
    }
    MKNN_CUDA_OK(cudaMemsetAsync(dq.bm, 0, sizeof(uint32_t) * nw, s));
    MKNN_CUDA_OK(cudaMemsetAsync(dq.dup, 0, sizeof(int32_t), s));
    MKNN_LAUNCH k_issuer_mark<<<blocks_for(nq), TPB, 0, s>>>(qi, nq, dq.minmax, span, dq.bm, dq.dup);
    MKNN_LAUNCH k_word_popc<<<blocks_for(nw), TPB, 0, s>>>(dq.bm, nw, dq.bm_cnt);
    MKNN_CUDA_OK(cudaGetLastError());
    rc = exclusive_scan_i32(dq.bm_cnt, dq.bm_pre, nw, scratch, s);
    if (rc) return rc;
    MKNN_LAUNCH k_issuer_rank<<<blocks_for(nq), TPB, 0, s>>>(qi, nq, dq.minmax, span, dq.bm, dq.bm_pre,
                                                            dq.row, out_qids);
    MKNN_CUDA_OK(cudaGetLastError());
    return 0;
  }
  if (dq.dup) MKNN_CUDA_OK(cudaMemsetAsync(dq.dup, 0, sizeof(int32_t), s));
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
