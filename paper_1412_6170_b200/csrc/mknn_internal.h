// mknn_internal.h -- launchers shared between the translation units of
// libmknn_b200.so.  Not part of the public C-ABI (see include/mknn_b200.h).
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "mknn_common.cuh"

namespace mknn {

int fail_cuda(cudaError_t e, const char* expr, const char* file, int line);
int fail_msg(int code, const std::string& msg);
const char* last_error_text();

// every kernel launch of the library is counted (bench.py reports the
// number of our own launches inside its timed region)
void note_launch();
long long launch_count();
void note_launches(long long n);  // a graph replay: its captured kernels
#define MKNN_LAUNCH ::mknn::note_launch(),

// error codes (C-ABI: 0 ok, < 0 error)
constexpr int E_INVALID = -1;   // ValueError on the Python side
constexpr int E_CUDA = -2;      // RuntimeError
constexpr int E_UNSUPPORTED = -3;

// ---------------------------------------------------------------- prims
// Scratch sizing helpers: every primitive takes a caller-provided scratch
// buffer of at least *_scratch_bytes(n) bytes.
size_t scan_scratch_bytes(int64_t n);
// exclusive scan of int32 counts -> int32 starts; also writes the total to
// out[n] (so out has n + 1 entries).  n may be 0.
int exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* scratch,
                       cudaStream_t s);
int exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, void* scratch,
                              cudaStream_t s);

// stable LSD radix sort of (key, value) pairs on the low `bits` bits of key
size_t radix_scratch_bytes(int64_t n);
int radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                         int64_t n, int bits, void* scratch, cudaStream_t s, bool* result_in_alt);

// min / max of int64 keys into dev_out[2] (device memory)
int minmax_i64(const int64_t* in, int64_t n, int64_t* dev_out, cudaStream_t s);

// --------------------------------------------------------------- index
struct DevIndex {
  // pyramid of per-quadrant object counts at build time, levels 0..l_max
  int32_t* counts = nullptr;   // concatenated, level l at pyramid_offset(l)
  uint8_t* state = nullptr;    // same layout: 0 absent, 1 leaf, 2 split
  int32_t* flags = nullptr;    // 4^l_max + 1 scan input / output
  int32_t* z_map = nullptr;    // 4^l_max capacity, first 4^l_deep used
  uint8_t* leaf_level = nullptr;
  uint32_t* leaf_code = nullptr;
  uint32_t* leaf_key = nullptr;
  uint32_t* leaf_span = nullptr;
  int32_t* build_counts = nullptr;
  int32_t* scalars = nullptr;  // [0] l_deep, [1] n_leaves, [2] overfull, [3] n_build, [4] n_sub,
                               // [5] largest partition-bucket build load (1/16 of the mean),
                               // [6] largest partition-bucket key count
  // store ordering inside each leaf: 4^s sub-cells per leaf (s from the
  // leaf's build count), leaf l owns sub-cell keys [sub_base[l], sub_base[l+1])
  uint8_t* leaf_sub_bits = nullptr;  // 2*s
  int32_t* leaf_sub_base = nullptr;  // 4^l_max + 1
  unsigned long long* cell_info = nullptr;  // per deepest cell: sub_base | shift | bits | leaf
  uint32_t* bload = nullptr;  // rebuild scratch: build load per partition bucket
  int32_t* bkey = nullptr;       // leaf-aligned partition buckets: bucket b = keys [bkey[b], bkey[b+1])
  int32_t* leaf_first = nullptr;  // bucket b holds leaves [leaf_first[b], leaf_first[b+1])
  uint16_t* leaf_bucket = nullptr;  // bucket of every leaf
  unsigned long long* cell_bucket = nullptr;  // cell_info with the leaf's bucket in bits 42-63
  int l_max = 0;
  int th_quad = 0;
};

inline int64_t pyramid_offset(int level) { return pyramid_offset_dev(level); }
inline int64_t pyramid_size(int l_max) { return pyramid_offset(l_max + 1); }

int index_alloc(DevIndex& ix, int l_max, int th_quad);
void index_free(DevIndex& ix);
// quadindex.py:79-163 build_index on device from n positions
int index_build(DevIndex& ix, const Region& r, const double* x, const double* y, int64_t n,
                void* scratch, cudaStream_t s);

// Per-tick object store (quadindex.py:166-213), leaf-grouped.  Inside a
// leaf, objects are ordered by Morton sub-cell below the leaf's own level and
// cut into chunks of CHUNK consecutive objects whose point bounding boxes let
// the search skip chunks that cannot hold a neighbour (exact: see
// mknn_search.cu).  Objects are 32-byte records (one L2 sector), so the
// counting-sort scatter writes whole sectors and a candidate's position and
// id arrive in one sector.
// objects per chunk box: 16 for one-slot lists (k <= 32: finer boxes, two
// chunks per warp step), 32 for k > 32 (buffered admission takes 32
// candidates per step anyway; coarser best-first order measured faster)
__host__ __device__ constexpr int chunk_for_k(int k) { return k <= 32 ? 16 : 32; }
constexpr int MAX_CHUNK = 32;

struct ChunkBox {
  double x_lo, y_lo, x_hi, y_hi;
};

struct __align__(32) StoreRec {  // one object of the leaf-sorted store
  double x, y;
  long long id;
  uint32_t key, pad;
};

// 256-bit global accesses (sm_100: LDG/STG.E.ENL2.256): one request per record
__device__ __forceinline__ StoreRec ld_rec(const StoreRec* p) {
  unsigned long long a, b, c, d;
  asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
  StoreRec r;
  r.x = __longlong_as_double((long long)a);
  r.y = __longlong_as_double((long long)b);
  r.id = (long long)c;
  r.key = (uint32_t)d;
  r.pad = (uint32_t)(d >> 32);
  return r;
}
__device__ __forceinline__ void st_rec(StoreRec* p, const StoreRec& r) {
  asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "l"((unsigned long long)__double_as_longlong(r.x)),
               "l"((unsigned long long)__double_as_longlong(r.y)), "l"((unsigned long long)r.id),
               "l"((unsigned long long)r.key | ((unsigned long long)r.pad << 32))
               : "memory");
}

struct DevStore {
  StoreRec* obj = nullptr;        // leaf-sorted objects
  StoreRec* rec = nullptr;        // staging of the bucket partition pass
  uint32_t* key = nullptr;        // sub-cell key per input object / query
  uint16_t* bkt = nullptr;        // partition bucket per input object (bucket-local sort)
  int64_t cap = 0;
  int32_t* cell_start = nullptr;  // 4^l_max + 2 (start[L] = n)
  int32_t* chunk_start = nullptr; // 4^l_max + 2 (chunk slot of each leaf's first chunk; a leaf's
                                  // chunks are [chunk_start[l], + ceil(population / chunk)))
  int32_t* nch = nullptr;         // 4^l_max + 2 scratch (chunks per leaf)
  ChunkBox* box = nullptr;        // per chunk
  int2* crange = nullptr;         // per chunk: object range
  int64_t cap_box = 0;
  int32_t* cnt = nullptr;         // n_sub + 2; all zero between ticks unless dirty
  int32_t* kstart = nullptr;      // n_sub + 2: first store position of every key
  int32_t* kstart_alt = nullptr;  // n_sub + 2: incremental update target
  int32_t* fill = nullptr;        // n_sub + 2: all zero between ticks
  int32_t* qcnt = nullptr;        // n_sub + 2: query counting sort (all zero between ticks)
  int32_t* qkstart = nullptr;
  int32_t* rmflag = nullptr;      // cap + 1: incremental update scratch
  int32_t* rm_before = nullptr;   // cap + 1
  uint32_t* mkey = nullptr;       // cap: new keys of the moved slots
  // moved slots whose old key group is large (dense or coincident points):
  // found through a slot -> store position map built only when needed
  int32_t* slot_pos = nullptr;    // cap
  int32_t* deferred = nullptr;    // cap: indices into the moved list
  int32_t* n_deferred = nullptr;  // device counter
  int64_t n_store = 0;            // records in obj
  bool valid = false;             // obj/kstart mirror the engine's snapshot (delta path)
  int chunk = 32;                 // objects per chunk (chunk_for_k)
  int32_t* cursor = nullptr;      // bucket counts / cursors of the partition pass
  int32_t* bstart = nullptr;      // bucket starts
  int32_t* cbase = nullptr;       // bucket-local sort: first chunk slot of every bucket
  int32_t* sstart = nullptr;      // one-pass partition: staging region start of every bucket
  uint32_t* bcnt = nullptr;       // bucket counts of the last bucket-sorted tick (plans the regions)
  bool bcnt_valid = false;        // bcnt matches the current index's buckets
  int64_t cap_sub = 0;
  bool dirty = true;              // cnt must be cleared before use
};

// records of the store and of its staging array for a capacity of n objects:
// the one-pass partition plans every bucket's region with 1/8 + 256 records
// of slack over the last tick's count (1024 buckets)
inline int64_t staging_records(int64_t n) { return n + n / 8 + 1024 * 256 + 1024; }

// (re)size the sub-cell tables and chunk arrays for n objects
int store_reserve(DevStore& st, int64_t n_sub, int64_t n_leaves, int64_t n);

// quadindex.py:190-213 index_objects; clamped count accumulates into
// dev_clamped (u64, device).  n_leaves / n_sub are host copies.
// st.key[i] keeps every input index's key (the snapshot slot's key on the
// delta path, which store_update_incremental maintains)
// balanced: the partition buckets' build loads are near the mean (DevIndex
// scalars[5]), so the bucket-local sort is used; otherwise the global-atomic
// counting sort
// two_pass: the bucket-local sort keys and partitions in two passes (exact
// bucket counts) instead of one pass over regions planned from the last
// tick's counts; *dev_overflow != 0 after a one-pass tick whose bucket
// outgrew its region (the caller redoes the tick with two_pass)
int store_index_objects(DevStore& st, const DevIndex& ix, const Region& r, const long long* ids,
                        const double* x, const double* y, int64_t n, int64_t n_leaves,
                        int64_t n_sub, bool balanced, int max_keys, int max_leaves, bool two_pass,
                        unsigned long long* dev_clamped, unsigned long long* dev_overflow,
                        void* scratch, cudaStream_t s, const unsigned long long* pre = nullptr);
// the one-pass partition of objects [lo, hi) ahead of store_index_objects
// (pre: device u64[2], clamped and overflow accumulators, zeroed by the caller)
int store_prepartition(DevStore& st, const DevIndex& ix, const Region& r, const long long* ids,
                       const double* x, const double* y, int64_t lo, int64_t hi, bool plan,
                       unsigned long long* pre, cudaStream_t s);
// Delta tick over the snapshot (sids/sx/sy, n_new slots): moved[0, m) are
// the slots whose position changed (or were appended) since the store was
// built from that snapshot.  dev_clamped_total: persistent count of objects
// outside the region.
int store_update_incremental(DevStore& st, const DevIndex& ix, const Region& r,
                             const long long* sids, const double* sx, const double* sy,
                             int64_t n_new, const int32_t* moved, int64_t m, int64_t n_leaves,
                             int64_t n_sub, unsigned long long* dev_clamped_total, void* scratch,
                             cudaStream_t s);

// engine.py:201-217 index_queries (leaf ordinal + leaf-grouped order)
struct DevQueries {
  uint32_t* leaf = nullptr;     // own leaf per query (input order)
  uint32_t* qkey = nullptr;     // (leaf << sub_bits) | sub per query
  uint32_t* order = nullptr;    // queries grouped by leaf, sub-cell order inside
  uint32_t* row = nullptr;      // emission row per query (stable issuer rank)
  uint64_t* keys = nullptr;     // radix buffers
  uint64_t* keys_alt = nullptr;
  uint32_t* vals = nullptr;
  uint32_t* vals_alt = nullptr;
  int64_t* minmax = nullptr;    // device [2]
  int64_t cap = 0;
  // issuer rank by bitmap (distinct issuers): one bit per id of the range
  uint32_t* bm = nullptr;
  int32_t* bm_cnt = nullptr;    // popcount per word, then its exclusive scan
  int32_t* bm_pre = nullptr;
  int64_t bm_cap = 0;           // words
  int32_t* dup = nullptr;       // device flag: an issuer id occurs twice (or left the range)
};

// uses st.sub_cnt / st.sub_start as its counting-sort tables
// plan_bits: issuer-id bits to sort on (< 0: measure them first, one host
// sync); *bits_used receives the bits actually sorted on
int queries_index(DevQueries& dq, DevStore& st, const DevIndex& ix, const Region& r,
                  const long long* qi, const double* qx, const double* qy, int64_t nq,
                  int64_t n_sub, int plan_bits, int* bits_used, bool bitmap, long long* out_qids, void* scratch,
                  cudaStream_t s);
// bits of the issuer-id range [lo, hi]
int issuer_bits(int64_t lo, int64_t hi);

// ------------------------------------------------------------- search
struct QueryStats {
  uint32_t evals;
  uint32_t prunes;
  uint16_t nav_left;
  uint16_t nav_right;
  uint32_t violations;
};

struct SearchArgs {
  Region r;
  int k;
  const int32_t* scalars;
  const int32_t* z_map;
  const uint32_t* leaf_key;
  const uint32_t* leaf_span;
  const int32_t* cell_start;  // L + 1 entries
  const int32_t* chunk_start; // L + 1 entries
  const ChunkBox* box;
  const StoreRec* obj;
  const uint32_t* q_order;
  const uint32_t* q_leaf;
  const uint32_t* q_row;
  const long long* qi;
  const double* qx;
  const double* qy;
  int64_t nq;
  int32_t* out_len;       // [nq] by row
  long long* out_nids;    // [nq * k] padded rows
  double* out_dist;       // [nq * k]
  QueryStats* stats;      // [nq] by leaf-grouped position
  int audit;
  int debug_phase; // profiling only: 1 = own leaf only (results invalid)
  int64_t n_objects;  // objects of the tick (the query density picks the warp batch)
  // profiling only (MKNN_PROF=1): work counters, see PROF_* in mknn_search.cu
  unsigned long long* prof;
  // instrumentation: (dir, iteration, leaf) keys of every distance task
  unsigned long long* task_keys;  // nullptr when off
  unsigned long long* task_count;
  int64_t task_cap;
  // k_search1: persistent CTAs take query batches from *work (zeroed by
  // search_launch before each launch)
  unsigned* work;
  // k_search1: the order its work counter hands out the query batches
  // (costliest own leaves first, see lpt_order); nullptr: batch order
  uint32_t* batch_order;
  uint32_t* lpt_cnt;  // [32] class counts and cursors of lpt_order
  // 16 < k <= 32: the own-leaf pass (k_own1) hands each query's list to the
  // expansion kernel (k_search1) as k store positions (32 slots) and its
  // k-th d2, by leaf-grouped position; [nq * 32] and [nq]
  int32_t* own_pos;
  double* own_thr;
  // [2] warp-time (ns, %globaltimer) of the query batches spent in the
  // own-leaf pass (first_iteration) and in the whole walk: the host splits
  // the search kernel's time into t_first_iteration_us / t_loop_us by it
  unsigned long long* phase_ns;
};

// T from task keys: sorts keys in place (alt buffer) and sums the leaf
// populations of distinct keys into *dev_T
int streamed_records(unsigned long long* keys, unsigned long long* keys_alt, uint32_t* vals,
                     uint32_t* vals_alt, int64_t n, const int32_t* cell_start,
                     unsigned long long* dev_T, void* scratch, cudaStream_t s);

int search_launch(const SearchArgs& a, cudaStream_t s);

// reduce QueryStats into dev_tot (u64 [4]: evals, prunes, violations, unused)
// and nav histograms (u32 [hist_cap] each) for active_left/right
int stats_reduce(const QueryStats* st, int64_t nq, unsigned long long* dev_tot, uint32_t* hist_l,
                 uint32_t* hist_r, int hist_cap, cudaStream_t s);

// padded rows (written by the search into the output itself) -> CSR in
// place: offsets[nq + 1] (int64); t_nids / t_dist are [nq * k] scratch
// touched only when some row is short
// skip (device flag, may be null): non-zero when the tick will be redone
// (its rows are not all written), so nothing is moved
int rows_compact(const int32_t* len, long long* nids, double* dist, int64_t nq, int k,
                 int64_t* offsets, long long* t_nids, double* t_dist, const int32_t* skip,
                 void* scratch, cudaStream_t s);

}  // namespace mknn
