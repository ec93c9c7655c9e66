// mknn_api.cu -- the engine handle and the C-ABI (include/mknn_b200.h).
//
// Orchestrates one tick of Engine.process_tick (engine.py:601-696) on the
// device: rebuild decision (quadindex.py:231-246) -> build_index ->
// index_objects -> index_queries -> search (first iteration + direction
// loop) -> emission.  The only host synchronisations per tick are the issuer
// range read (to size the radix sort) and the final metrics read.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mknn_b200.h"
#include "mknn_internal.h"

using namespace mknn;

namespace {

template <typename T>
int grow(T*& p, int64_t& cap_elems, int64_t want) {
  if (want <= cap_elems && p) return 0;
  int64_t nc = std::max<int64_t>(want, std::max<int64_t>(cap_elems * 3 / 2, 1024));
  if (p) cudaFree(p);
  p = nullptr;
  cap_elems = 0;
  MKNN_CUDA_OK(cudaMalloc(&p, sizeof(T) * (size_t)nc));
  cap_elems = nc;
  return 0;
}

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap && p) return 0;
    size_t nc = std::max(bytes, cap * 3 / 2);
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    MKNN_CUDA_OK(cudaMalloc(&p, nc));
    cap = nc;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

constexpr long long HASH_EMPTY = (long long)0x8000000000000000ULL;

// one probe = one 16-byte slot (key and slot index in the same sector)
struct __align__(16) HashSlot {
  long long key;
  int32_t val;
  int32_t pad;
};

__device__ __forceinline__ uint64_t hash64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

__global__ void k_fill_i64(long long* p, int64_t n, long long v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// id -> slot map (open addressing, linear probing).  A new id claims the
// next snapshot slot; concurrent inserts of one id wait for the winner.
__device__ int32_t hash_find_or_insert(HashSlot* ht, uint64_t mask, long long id,
                                       int32_t* n_snap, bool insert_new, int32_t fixed_slot) {
  uint64_t h = hash64((uint64_t)id) & mask;
  for (;;) {
    long long cur = ht[h].key;
    if (cur == id) {
      int32_t v;
      while ((v = ((volatile int32_t*)&ht[h].val)[0]) < 0) {
      }
      return v;
    }
    if (cur == HASH_EMPTY) {
      const long long prev = (long long)atomicCAS((unsigned long long*)&ht[h].key,
                                                  (unsigned long long)HASH_EMPTY,
                                                  (unsigned long long)id);
      if (prev == HASH_EMPTY) {
        const int32_t slot = insert_new ? (fixed_slot >= 0 ? fixed_slot : atomicAdd(n_snap, 1)) : -1;
        __threadfence();
        atomicExch(&ht[h].val, slot);
        return slot;
      }
      if (prev == id) continue;  // lost the race to the same id: wait above
    }
    h = (h + 1) & mask;
  }
}

__global__ void k_fill_slots(HashSlot* ht, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    ht[i] = HashSlot{HASH_EMPTY, -1, 0};
}

__global__ void k_hash_load(const long long* __restrict__ ids, int64_t n, HashSlot* ht,
                            uint64_t mask) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // duplicate ids inside a snapshot: the first slot keeps the mapping
    hash_find_or_insert(ht, mask, ids[i], nullptr, true, (int32_t)i);
  }
}

// last update per id wins (datasets.py:130-131): winner[slot] = max of
// (batch sequence << 32 | index) -- a later batch's claims are larger than
// any left by an earlier one, so the array is never reset between batches
__global__ void k_update_claim(const long long* __restrict__ ids, int64_t nu, HashSlot* ht,
                               uint64_t mask, int32_t* n_snap, unsigned long long* winner,
                               int32_t* slot_of, unsigned long long seq) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nu;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = hash_find_or_insert(ht, mask, ids[i], n_snap, true, -1);
    slot_of[i] = s;
    atomicMax(&winner[s], (seq << 32) | (unsigned long long)i);
  }
}

__global__ void k_update_apply(const long long* __restrict__ ids, const double* __restrict__ x,
                               const double* __restrict__ y, int64_t nu,
                               const int32_t* __restrict__ slot_of,
                               const unsigned long long* __restrict__ winner, unsigned long long seq,
                               long long* sids, double* sx, double* sy, int32_t* mark,
                               int32_t epoch, int32_t* moved, int32_t* n_moved, bool track,
                               const int32_t* __restrict__ n_before) {
  // slots below the snapshot size before this batch already hold their id
  const int32_t nb = *n_before;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nu;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = slot_of[i];
    bool first = false;
    if (winner[s] == ((seq << 32) | (unsigned long long)i)) {
      if (s >= nb) sids[s] = ids[i];
      sx[s] = x[i];
      sy[s] = y[i];
      // slots changed since the store was built (once per slot and epoch)
      if (track) first = atomicExch(&mark[s], epoch) != epoch;
    }
    if (!track) continue;
    // one counter atomic per warp (10M updates on one address serialise)
    const unsigned act = __activemask();
    const unsigned want = __ballot_sync(act, first);
    if (want) {
      const int lane = threadIdx.x & 31;
      const int leader = __ffs(want) - 1;
      int32_t base = 0;
      if (lane == leader) base = atomicAdd(n_moved, __popc(want));
      base = __shfl_sync(act, base, leader);
      if (first) moved[base + __popc(want & ((1u << lane) - 1u))] = s;
    }
  }
}


inline unsigned gs_blocks(int64_t n) {
  return (unsigned)std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 148 * 256);
}

int64_t us_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();  // not a failure of the tick: leave no pending error
    return 0;
  }
  return (int64_t)llround(ms * 1000.0);
}

}  // namespace

// host-output ticks of >= SLICE_MIN_QUERIES queries search in n_slices
// result-row slices whose copies to the host overlap the next slice
constexpr int MAX_SLICES = 16;
constexpr int64_t SLICE_MIN_QUERIES = 65536;

// pinned landing block of a tick's small device->host readbacks
struct PinBlock {
  static constexpr int HIST = 256;
  unsigned long long cnt[8];
  int64_t mm[2];
  int64_t total;
  int32_t dup;
  int32_t nsnap;
  uint32_t hist[2][HIST];
};

// every small readback of a tick, written straight into the mapped pinned
// block by one kernel (one graph node instead of a chain of tiny copies)
__global__ void k_readback(const unsigned long long* __restrict__ counters,
                           const int64_t* __restrict__ minmax, const int64_t* __restrict__ total,
                           const int32_t* __restrict__ dup, const int32_t* __restrict__ nsnap,
                           const uint32_t* __restrict__ hist, int64_t hist_cap, int hpre,
                           PinBlock* pb) {
  const int t = threadIdx.x;
  if (t < 8) pb->cnt[t] = counters[t];
  if (t == 8) {
    pb->mm[0] = minmax ? minmax[0] : 0;
    pb->mm[1] = minmax ? minmax[1] : 0;
  }
  if (t == 9) pb->total = *total;
  if (t == 10) pb->dup = dup ? *dup : 0;
  if (t == 11) pb->nsnap = nsnap ? *nsnap : 0;
  for (int i = t; i < hpre; i += blockDim.x) {
    pb->hist[0][i] = hist[i];
    pb->hist[1][i] = hist[hist_cap + i];
  }
}

struct mknn_engine {
  mknn_config cfg{};
  Region r{};
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  std::string err;

  DevIndex ix;
  bool have_index = false;
  bool last_tick_ok = false;
  int issuer_bits = -1;        // issuer-id bits of the last tick (plans the row sort)
  bool issuer_dups = false;    // a batch repeated an issuer id: rows by radix sort from then on
  cudaStream_t copy_stream = nullptr;  // result slices device -> host
  // host ticks: the objects cross PCIe in chunks on in_stream while the
  // one-pass partition of the chunks already copied runs on the main stream
  cudaStream_t in_stream = nullptr;
  cudaEvent_t in_ev[4] = {};
  unsigned long long* pre_counts = nullptr;  // clamped, overflow of that partition
  bool prepartitioned = false;
  cudaEvent_t slice_ev[MAX_SLICES] = {};
  cudaEvent_t q_ready = nullptr;  // host query batch staged on copy_stream
  PinBlock* pin = nullptr;
  PinBlock* pin_dev = nullptr;  // the same block as the device sees it (mapped)
  bool q_pending = false;
  bool rows_in_host = false;   // the sliced host tick already delivered qids/len/rows
  bool retry_rebuild = false;  // false: the store's sub-cell counters may be dirty
  bool retry_radix = false;    // the redo of a tick sorts its issuers with the radix path
  int32_t h_l_deep = 0;
  int64_t h_n_leaves = 0, h_overfull = 0, h_n_build = 0, h_n_sub = 0;
  int64_t h_bucket_load = 0;  // largest partition-bucket build load, 1/16 of the mean
  int64_t h_bucket_keys = 0;  // largest partition-bucket key count
  int64_t h_bucket_leaves = 0;  // largest partition-bucket leaf count
  bool two_pass_next = false;  // the last one-pass partition overflowed: redo in two passes
  DevStore st;
  DevQueries dq;

  // staging for host-input ticks
  long long* in_ids = nullptr; double *in_x = nullptr, *in_y = nullptr; int64_t cap_in = 0;
  long long* in_qi = nullptr; double *in_qx = nullptr, *in_qy = nullptr; int64_t cap_qin = 0;
  // padded result rows + CSR + per-query stats
  int32_t* out_len = nullptr; int64_t cap_len = 0;
  long long* out_nids = nullptr; double* out_dist = nullptr; int64_t cap_rows = 0;
  long long* c_nids = nullptr; double* c_dist = nullptr; int64_t cap_c = 0;
  int64_t* offsets = nullptr; int64_t cap_off = 0;
  long long* out_qids = nullptr; int64_t cap_oq = 0;
  QueryStats* stats = nullptr; int64_t cap_stats = 0;
  int32_t* own_pos = nullptr; double* own_thr = nullptr; int64_t cap_own = 0;  // k_own1 -> k_search1
  uint32_t* batch_order = nullptr; int64_t cap_bo = 0;  // k_search1's batch schedule
  uint32_t* lpt_cnt = nullptr;
  unsigned long long* prof = nullptr;  // MKNN_PROF=1 work counters
  unsigned* work = nullptr;  // k_search1 batch counter
  unsigned long long* counters = nullptr;  // [0] evals [1] prunes [2] viol [3] clamped
  uint32_t* hist = nullptr;                // 2 x hist_cap
  // instrumentation buffers (config.instrument & 1)
  unsigned long long *tk = nullptr, *tk_alt = nullptr, *tk_cnt = nullptr;
  uint32_t *tv = nullptr, *tv_alt = nullptr;
  int64_t cap_tk = 0;
  int hist_cap = 0;
  Buf scratch;

  // persistent snapshot (delta path)
  long long* snap_ids = nullptr; double *snap_x = nullptr, *snap_y = nullptr; int64_t cap_snap = 0;
  int64_t n_snap = 0;
  HashSlot* ht = nullptr; int64_t hcap = 0;  // id -> snapshot slot
  unsigned long long* winner = nullptr; int64_t cap_winner = 0;
  unsigned long long upd_seq = 0;  // update batches (the winner claims' high word)
  // incremental store (delta ticks): slots moved since the store was built
  int32_t* mark = nullptr;     // per slot: epoch of its last recorded move
  int32_t* moved = nullptr;    // moved slots
  int32_t* d_nmoved = nullptr;
  int64_t h_nmoved = 0;
  // updates are sync-free: the exact snapshot size and moved count stay on
  // the device until needed; the host keeps upper bounds meanwhile
  bool upd_pending = false;
  int64_t n_snap_hi = 0, nmoved_hi = 0;
  int64_t n_spec = -1;      // a query tick run on the unconfirmed n_snap (checked at its end)
  bool snap_retry = false;  // ... and it was wrong (ids were appended): redo
  int32_t epoch = 1;
  unsigned long long* clamped_total = nullptr;  // objects of the store outside the region
  int32_t* slot_of = nullptr; int64_t cap_slot_of = 0;
  int32_t* d_nsnap = nullptr;
  long long* up_ids = nullptr; double *up_x = nullptr, *up_y = nullptr; int64_t cap_up = 0;

  // steady-state tick graph (graph_key)
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  std::vector<uintptr_t> gkey;
  std::vector<uintptr_t> gkey_seen;  // the previous graphable tick's key (capture on a repeat)
  int64_t graph_captures = 0, graph_replays = 0;
  long long graph_kernels = 0;  // kernel launches inside the captured graph
  bool graph_dirty_after = false;  // the store's cnt-dirty flag after the captured sequence

  std::vector<int64_t> history;
  int64_t tick = 0;
  std::vector<int64_t> active[2];
  cudaEvent_t ev[8] = {};

  int set_err(int code) { return code; }
  int invalid(const std::string& m) { return fail_msg(E_INVALID, m); }
};

namespace {

int bind(mknn_engine* h) {
  MKNN_CUDA_OK(cudaSetDevice(h->device));
  return 0;
}

// quadindex.py:231-246 should_rebuild
bool should_rebuild(const std::vector<int64_t>& c, int window, double factor) {
  if ((int64_t)c.size() < window + 1) return false;
  const int64_t last = c.back();
  double sum = 0.0;
  for (size_t i = c.size() - 1 - window; i < c.size() - 1; i++) sum += (double)c[i];
  return (double)last > factor * (sum / window);
}

}  // namespace

// ---------------------------------------------------------------- core tick
namespace {

// Host destinations of a host-output tick: when set, the search runs in
// slices of consecutive result rows and each slice's rows are copied to the
// host (on the copy stream) while the next slice computes.
struct HostSink {
  int64_t* qids;
  int32_t* len;
  int64_t* nids;
  double* dist;
};

struct SliceBounds {  // result-row slice j = rows [b[j], b[j + 1])
  int64_t b[17];
  int n;
};

__global__ void k_slice_keys(const uint32_t* __restrict__ order, const uint32_t* __restrict__ row,
                             int64_t nq, const SliceBounds sb, uint64_t* __restrict__ keys,
                             uint32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) {
    const uint32_t q = order[i];
    const int64_t r = row[q];
    int j = 0;
    while (j + 1 < sb.n && r >= sb.b[j + 1]) j++;
    keys[i] = (uint64_t)j;
    vals[i] = q;
  }
}

struct DevOut {
  long long* qids;    // [nq] or nullptr
  int32_t* len;       // [nq]
  int64_t* offsets;   // [nq + 1]
  long long* nids;    // CSR
  double* dist;       // CSR
};

int alloc_store(mknn_engine* h, int64_t n) {
  const int64_t ncap = int64_t(1) << (2 * h->cfg.l_max);
  if (!h->st.cell_start) {
    MKNN_CUDA_OK(cudaMalloc(&h->st.cell_start, sizeof(int32_t) * (ncap + 2)));
    MKNN_CUDA_OK(cudaMalloc(&h->st.chunk_start, sizeof(int32_t) * (ncap + 2)));
    MKNN_CUDA_OK(cudaMalloc(&h->st.nch, sizeof(int32_t) * (ncap + 2)));
    MKNN_CUDA_OK(cudaMalloc(&h->dq.minmax, sizeof(int64_t) * 2));
    MKNN_CUDA_OK(cudaMalloc(&h->counters, sizeof(unsigned long long) * 8));
    MKNN_CUDA_OK(cudaMalloc(&h->clamped_total, sizeof(unsigned long long)));
    h->hist_cap = (int)(ncap + 2);
    MKNN_CUDA_OK(cudaMalloc(&h->hist, sizeof(uint32_t) * 2 * h->hist_cap));
    MKNN_CUDA_OK(cudaMalloc(&h->work, sizeof(unsigned) * 4));
    MKNN_CUDA_OK(cudaMalloc(&h->lpt_cnt, sizeof(uint32_t) * 32));
  }
  if (n > h->st.cap) {
    int64_t nc = std::max<int64_t>(n, h->st.cap * 3 / 2);
    void** old[] = {(void**)&h->st.obj, (void**)&h->st.rec, (void**)&h->st.key,
                    (void**)&h->st.rmflag, (void**)&h->st.rm_before, (void**)&h->st.mkey,
                    (void**)&h->st.slot_pos, (void**)&h->st.deferred, (void**)&h->st.bkt};
    for (auto p : old) {
      cudaFree(*p);
      *p = nullptr;
    }
    h->st.cap = 0;
    h->st.valid = false;
    // obj and rec swap roles on incremental ticks: both hold a staging array
    MKNN_CUDA_OK(cudaMalloc(&h->st.obj, sizeof(StoreRec) * staging_records(nc)));
    MKNN_CUDA_OK(cudaMalloc(&h->st.rec, sizeof(StoreRec) * staging_records(nc)));
    MKNN_CUDA_OK(cudaMalloc(&h->st.key, sizeof(uint32_t) * nc));
    MKNN_CUDA_OK(cudaMalloc(&h->st.rmflag, sizeof(int32_t) * (nc + 1)));
    MKNN_CUDA_OK(cudaMalloc(&h->st.rm_before, sizeof(int32_t) * (nc + 2)));
    MKNN_CUDA_OK(cudaMalloc(&h->st.mkey, sizeof(uint32_t) * nc));
    MKNN_CUDA_OK(cudaMalloc(&h->st.slot_pos, sizeof(int32_t) * nc));
    MKNN_CUDA_OK(cudaMalloc(&h->st.bkt, sizeof(uint16_t) * nc));
    MKNN_CUDA_OK(cudaMalloc(&h->st.deferred, sizeof(int32_t) * nc));
    if (!h->st.n_deferred) MKNN_CUDA_OK(cudaMalloc(&h->st.n_deferred, sizeof(int32_t)));
    h->st.cap = nc;
  }
  return 0;
}

int alloc_queries(mknn_engine* h, int64_t nq) {
  if (nq <= h->dq.cap) return 0;
  const int64_t nc = std::max<int64_t>(nq, h->dq.cap * 3 / 2);
  cudaFree(h->dq.leaf);
  cudaFree(h->dq.qkey);
  cudaFree(h->dq.order);
  cudaFree(h->dq.row);
  cudaFree(h->dq.keys);
  cudaFree(h->dq.keys_alt);
  cudaFree(h->dq.vals);
  cudaFree(h->dq.vals_alt);
  h->dq.cap = 0;
  MKNN_CUDA_OK(cudaMalloc(&h->dq.leaf, sizeof(uint32_t) * nc));
  MKNN_CUDA_OK(cudaMalloc(&h->dq.qkey, sizeof(uint32_t) * nc));
  MKNN_CUDA_OK(cudaMalloc(&h->dq.order, sizeof(uint32_t) * nc));
  MKNN_CUDA_OK(cudaMalloc(&h->dq.row, sizeof(uint32_t) * nc));
  MKNN_CUDA_OK(cudaMalloc(&h->dq.keys, sizeof(uint64_t) * nc));
  MKNN_CUDA_OK(cudaMalloc(&h->dq.keys_alt, sizeof(uint64_t) * nc));
  MKNN_CUDA_OK(cudaMalloc(&h->dq.vals, sizeof(uint32_t) * nc));
  MKNN_CUDA_OK(cudaMalloc(&h->dq.vals_alt, sizeof(uint32_t) * nc));
  h->dq.cap = nc;
  return 0;
}

int refresh_index_info(mknn_engine* h) {
  int32_t sc[8];
  MKNN_CUDA_OK(cudaMemcpyAsync(sc, h->ix.scalars, sizeof(sc), cudaMemcpyDeviceToHost, h->stream));
  MKNN_CUDA_OK(cudaStreamSynchronize(h->stream));
  h->h_l_deep = sc[0];
  h->h_n_leaves = sc[1];
  h->h_overfull = sc[2];
  h->h_n_build = sc[3];
  h->h_n_sub = sc[4];
  h->h_bucket_load = sc[5];
  h->h_bucket_keys = sc[6];
  h->h_bucket_leaves = sc[7];
  return 0;
}

// Engine.process_tick over device-resident inputs; results into `o`.
int snap_sync(mknn_engine* h);
int validate_counts(mknn_engine* h, int64_t n, int64_t nq);

// Every device buffer the engine owns (destroy frees them; a graph key
// includes them, so any reallocation forces a new capture).
std::vector<void*> engine_buffers(mknn_engine* h) {
  return {h->st.obj, h->st.rec, h->st.cursor, h->st.bstart, h->st.cbase, h->st.key, h->st.cell_start,
          h->st.chunk_start, h->st.nch, h->st.box, h->st.crange, h->st.cnt, h->st.kstart,
          h->dq.leaf, h->dq.qkey, h->dq.order, h->dq.row, h->dq.keys, h->dq.keys_alt, h->dq.vals,
          h->dq.vals_alt, h->dq.minmax, h->dq.bm, h->dq.bm_cnt, h->dq.bm_pre, h->dq.dup,
          h->in_ids, h->in_x, h->in_y, h->in_qi, h->in_qx, h->in_qy, h->out_len, h->out_nids,
          h->out_dist, h->c_nids, h->c_dist, h->offsets, h->out_qids, h->stats, h->counters,
          h->hist, h->snap_ids, h->snap_x, h->snap_y, h->ht, h->winner, h->slot_of, h->d_nsnap,
          h->up_ids, h->up_x, h->up_y, h->tk, h->tk_alt, h->tk_cnt, h->tv, h->tv_alt, h->prof,
          h->mark, h->moved, h->d_nmoved, h->clamped_total, h->work, h->st.kstart_alt,
          h->st.fill, h->st.qcnt, h->st.qkstart, h->st.rmflag, h->st.rm_before, h->st.mkey,
          h->own_pos, h->own_thr, h->st.slot_pos, h->st.deferred, h->st.n_deferred, h->st.bkt,
          h->batch_order, h->lpt_cnt};
}

// A tick whose enqueue sequence is a pure function of the key below can run
// as a graph replay: steady state (no rebuild, whose leaf count is read back
// mid-tick), device outputs, the full re-index path (the incremental one
// swaps store buffers every tick), no instrumentation / audit / profiling,
// issuer bits planned from the previous tick.  The key holds every size,
// flag and pointer the sequence bakes into its launches.
int graph_key(mknn_engine* h, int64_t n, const long long* ids, const double* x, const double* y,
              int64_t nq, const long long* qi, const double* qx, const double* qy, const DevOut& o,
              bool rebuild, const HostSink* sink, std::vector<uintptr_t>* key, bool* ok) {
  *ok = false;
  static const bool off = [] {
    const char* e = getenv("MKNN_GRAPH");
    return e && e[0] == '0';
  }();
  static const bool dbg = getenv("MKNN_DEBUG_PHASE") || getenv("MKNN_PROF");
  if (off || dbg || rebuild || sink || nq <= 0 || n <= 0 || (h->cfg.instrument & 1) ||
      h->cfg.audit_pruning || h->issuer_bits < 0 || h->q_pending)
    return 0;
  const bool from_snap = ids == h->snap_ids && x == h->snap_x && y == h->snap_y;
  const bool incremental = from_snap && h->st.valid && h->st.n_store <= n &&
                           (h->h_nmoved + (n - h->st.n_store)) * 20 <= n;
  if (incremental) return 0;
  h->st.chunk = chunk_for_k(h->cfg.k);
  int rc;
  if ((rc = store_reserve(h->st, h->h_n_sub, h->h_n_leaves, n))) return rc;
  const bool dirty = h->st.dirty || !h->last_tick_ok;
  const bool use_bitmap = !h->issuer_dups && !h->retry_radix;
  *key = {(uintptr_t)n, (uintptr_t)nq, (uintptr_t)h->cfg.k, (uintptr_t)h->h_n_sub,
          (uintptr_t)h->h_n_leaves, (uintptr_t)h->h_l_deep, (uintptr_t)from_snap,
          (uintptr_t)dirty, (uintptr_t)use_bitmap, (uintptr_t)h->issuer_bits,
          (uintptr_t)h->stream, (uintptr_t)ids, (uintptr_t)x, (uintptr_t)y, (uintptr_t)qi,
          (uintptr_t)qx, (uintptr_t)qy, (uintptr_t)o.qids, (uintptr_t)o.len,
          (uintptr_t)o.offsets, (uintptr_t)o.nids, (uintptr_t)o.dist,
          (uintptr_t)h->scratch.p, (uintptr_t)h->pin, (uintptr_t)h->dq.bm_cap,
          (uintptr_t)h->st.cap_sub, (uintptr_t)h->st.cap_box, (uintptr_t)(h->n_spec >= 0),
          (uintptr_t)h->h_bucket_load, (uintptr_t)h->h_bucket_keys, (uintptr_t)h->h_bucket_leaves,
          (uintptr_t)h->two_pass_next,
          (uintptr_t)h->st.bcnt_valid};
  for (void* b : engine_buffers(h)) key->push_back((uintptr_t)b);
  *ok = true;
  return 0;
}

int core_tick_once(mknn_engine* h, int64_t n, const long long* ids, const double* x,
                   const double* y, int64_t nq, const long long* qi, const double* qx,
                   const double* qy, const DevOut& o, mknn_metrics* met,
                   std::chrono::steady_clock::time_point t_start, bool force_rebuild, bool* retry,
                   const HostSink* sink) {
  *retry = false;
  const int k = h->cfg.k;
  cudaStream_t s = h->stream;
  int rc;
  if ((rc = alloc_store(h, std::max<int64_t>(n, 1)))) return h->set_err(rc);
  if ((rc = alloc_queries(h, std::max<int64_t>(nq, 1)))) return h->set_err(rc);
  if ((rc = grow(h->stats, h->cap_stats, std::max<int64_t>(nq, 1)))) return h->set_err(rc);
  if (k > 16 && k <= 32 && nq > h->cap_own) {
    int64_t c = h->cap_own;
    if ((rc = grow(h->own_thr, c, nq))) return h->set_err(rc);
    c = h->cap_own * 32;
    if ((rc = grow(h->own_pos, c, nq * 32))) return h->set_err(rc);
    h->cap_own = c / 32;
  }
  if (k > 16 && k <= 32 && nq > h->cap_bo) {  // batches of >= 4 queries: nq / 4 + 1 suffice
    if ((rc = grow(h->batch_order, h->cap_bo, nq))) return h->set_err(rc);
  }
  const int64_t rows = std::max<int64_t>(nq * (int64_t)k, 1);
  if (rows > h->cap_rows) {
    int64_t c = h->cap_rows;
    if ((rc = grow(h->out_nids, c, rows))) return h->set_err(rc);
    c = h->cap_rows;
    if ((rc = grow(h->out_dist, c, rows))) return h->set_err(rc);
    h->cap_rows = c;
  }
  const int64_t ncap = int64_t(1) << (2 * h->cfg.l_max);
  size_t sb = std::max({scan_scratch_bytes(ncap + 2), scan_scratch_bytes(n + ncap + 2),
                        scan_scratch_bytes((int64_t(1) << 22) + 2),  // issuer bitmap words
                        scan_scratch_bytes(std::max<int64_t>(nq, 1) + 1),
                        radix_scratch_bytes(std::max<int64_t>(nq, 1))});
  if ((rc = h->scratch.ensure(sb + 1024))) return h->set_err(rc);

  if (!h->pin) {
    MKNN_CUDA_OK(cudaHostAlloc(&h->pin, sizeof(PinBlock), cudaHostAllocMapped));
    MKNN_CUDA_OK(cudaHostGetDevicePointer(&h->pin_dev, h->pin, 0));
  }

  mknn_metrics m{};
  m.tick = h->tick;
  m.n_objects = n;
  m.n_queries = nq;

  const bool rebuild = force_rebuild || !h->have_index ||
                       should_rebuild(h->history, h->cfg.rebuild_window, h->cfg.rebuild_factor);
  int bits_used = 0;
  bool sliced = false, prof_on = false;
  const int64_t hpre = std::min<int64_t>(h->hist_cap, PinBlock::HIST);

  // Steady-state device ticks replay a CUDA graph of the whole enqueue
  // sequence (index, queries, search, emission, readbacks) captured on the
  // first tick of its shape: one launch instead of ~30, no host gaps.
  std::vector<uintptr_t> gkey;
  bool graphable = false;
  if ((rc = graph_key(h, n, ids, x, y, nq, qi, qx, qy, o, rebuild, sink, &gkey, &graphable)))
    return h->set_err(rc);
  // capture only a shape seen on the previous graphable tick, so callers
  // whose buffers change every tick never pay for captures
  if (graphable && !(h->gexec && gkey == h->gkey) && gkey != h->gkey_seen) {
    h->gkey_seen = gkey;
    graphable = false;
  }
  if (graphable && h->gexec && gkey == h->gkey) {
    MKNN_CUDA_OK(cudaGraphLaunch(h->gexec, s));
    note_launches(h->graph_kernels);
    // the host-side effects of the captured sequence (full re-index path)
    const bool from_snap = ids == h->snap_ids && x == h->snap_x && y == h->snap_y;
    h->last_tick_ok = false;
    h->st.dirty = h->graph_dirty_after;
    h->st.n_store = n;
    h->st.valid = from_snap;
    if (from_snap) {
      h->h_nmoved = 0;
      h->epoch++;
    }
    h->retry_radix = false;
    h->rows_in_host = false;
    m.streamed_records = -1;
    bits_used = h->issuer_bits;
    h->graph_replays++;
  } else {
    cudaStream_t user_s = s;
    if (graphable) {
      if (cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeRelaxed) == cudaSuccess) {
        s = h->stream = h->cap_stream;
      } else {
        cudaGetLastError();
        graphable = false;
      }
    }
    int erc = 0;
    const long long launches0 = launch_count();
    // phase events become event-record nodes of a captured graph
    const unsigned ev_flags = graphable ? cudaEventRecordExternal : cudaEventRecordDefault;
    auto enqueue = [&]() -> int {
      MKNN_CUDA_OK(cudaEventRecordWithFlags(h->ev[0], s, ev_flags));
      if (rebuild) {
        if ((rc = index_build(h->ix, h->r, x, y, n, h->scratch.p, s))) return h->set_err(rc);
        h->st.bcnt_valid = false;  // new buckets: the next partition counts them exactly
        h->have_index = true;
        m.rebuild_flag = 1;
        if ((rc = refresh_index_info(h))) return h->set_err(rc);  // leaf count sizes the store tables
      }
      h->st.chunk = chunk_for_k(k);
      if ((rc = store_reserve(h->st, h->h_n_sub, h->h_n_leaves, n))) return h->set_err(rc);
      if (!h->last_tick_ok) h->st.dirty = true;
      h->last_tick_ok = false;
      MKNN_CUDA_OK(cudaEventRecordWithFlags(h->ev[1], s, ev_flags));
      MKNN_CUDA_OK(cudaMemsetAsync(h->counters, 0, sizeof(unsigned long long) * 8, s));
      // delta path (the engine's own snapshot): re-index incrementally when the
      // store still mirrors that snapshot and few slots moved since.  The
      // incremental pass still moves every surviving record once, so it only
      // beats the two-pass rebuild below ~5 % moved (measured at 10M objects:
      // 0.1 % 335 us, 1 % 358 us, 10 % 634 us vs 566 us for a rebuild).
      const bool from_snap = ids == h->snap_ids && x == h->snap_x && y == h->snap_y;
      const bool incremental = from_snap && h->st.valid && !rebuild && h->st.n_store <= n &&
                               (h->h_nmoved + (n - h->st.n_store)) * 20 <= n;
      if (incremental) {
        if ((rc = store_update_incremental(h->st, h->ix, h->r, ids, x, y, n, h->moved, h->h_nmoved,
                                           h->h_n_leaves, h->h_n_sub, h->clamped_total, h->scratch.p,
                                           s)))
          return h->set_err(rc);
        MKNN_CUDA_OK(cudaMemcpyAsync(h->counters + 3, h->clamped_total, sizeof(unsigned long long),
                                     cudaMemcpyDeviceToDevice, s));
      } else {
        if ((rc = store_index_objects(h->st, h->ix, h->r, ids, x, y, n, h->h_n_leaves, h->h_n_sub,
                                      h->h_bucket_load <= 4 * 16 && h->h_bucket_keys <= 32768,
                                      (int)h->h_bucket_keys, (int)h->h_bucket_leaves, h->two_pass_next,
                                      h->counters + 3, h->counters + 4, h->scratch.p, s,
                                      h->prepartitioned ? h->pre_counts : nullptr)))
          return h->set_err(rc);
        h->prepartitioned = false;  // a redo of the tick partitions again
        MKNN_CUDA_OK(cudaMemcpyAsync(h->clamped_total, h->counters + 3, sizeof(unsigned long long),
                                     cudaMemcpyDeviceToDevice, s));
      }
      h->st.valid = from_snap;
      if (from_snap) {  // the store now reflects every recorded move
        MKNN_CUDA_OK(cudaMemsetAsync(h->d_nmoved, 0, sizeof(int32_t), s));
        h->h_nmoved = 0;
        h->epoch++;
      }
      MKNN_CUDA_OK(cudaEventRecordWithFlags(h->ev[2], s, ev_flags));
      if (h->q_pending) {  // host queries staged on the copy stream (stage_queries)
        MKNN_CUDA_OK(cudaStreamWaitEvent(s, h->q_ready, 0));
        h->q_pending = false;
      }
      const bool use_bitmap = !h->issuer_dups && !h->retry_radix;
      h->retry_radix = false;
      if ((rc = queries_index(h->dq, h->st, h->ix, h->r, qi, qx, qy, nq, h->h_n_sub, h->issuer_bits,
                              &bits_used, use_bitmap, o.qids, h->scratch.p, s)))
        return h->set_err(rc);
      MKNN_CUDA_OK(cudaEventRecordWithFlags(h->ev[3], s, ev_flags));

      SearchArgs a{};
      a.r = h->r;
      a.k = k;
      a.scalars = h->ix.scalars;
      a.z_map = h->ix.z_map;
      a.leaf_key = h->ix.leaf_key;
      a.leaf_span = h->ix.leaf_span;
      a.cell_start = h->st.cell_start;
      a.chunk_start = h->st.chunk_start;
      a.box = h->st.box;
      a.obj = h->st.obj;
      a.q_order = h->dq.order;
      a.q_leaf = h->dq.leaf;
      a.q_row = h->dq.row;
      a.qi = qi;
      a.qx = qx;
      a.qy = qy;
      a.nq = nq;
      a.out_len = o.len;
      a.out_nids = o.nids;  // padded rows in the output itself (rows_compact)
      a.out_dist = o.dist;
      a.n_objects = n;
      a.stats = h->stats;
      a.work = h->work;
      a.own_pos = h->own_pos;
      a.own_thr = h->own_thr;
      a.batch_order = h->batch_order;
      a.lpt_cnt = h->lpt_cnt;
      a.phase_ns = h->counters + 6;  // zeroed with the counters each tick
      a.audit = h->cfg.audit_pruning;
      {
        static const char* dp = getenv("MKNN_DEBUG_PHASE");
        a.debug_phase = dp ? atoi(dp) : 0;
        static const char* pf = getenv("MKNN_PROF");
        if (pf && pf[0] == '1') {
          if (!h->prof) MKNN_CUDA_OK(cudaMalloc(&h->prof, 8 * 16));
          MKNN_CUDA_OK(cudaMemsetAsync(h->prof, 0, 8 * 16, s));
          a.prof = h->prof;
        }
      }
      const bool instr = (h->cfg.instrument & 1) != 0;
      if (instr) {
        const int64_t want = std::max<int64_t>(16 * nq, 1024);
        if (want > h->cap_tk) {
          cudaFree(h->tk); cudaFree(h->tk_alt); cudaFree(h->tv); cudaFree(h->tv_alt);
          h->tk = h->tk_alt = nullptr; h->tv = h->tv_alt = nullptr; h->cap_tk = 0;
          MKNN_CUDA_OK(cudaMalloc(&h->tk, 8 * want));
          MKNN_CUDA_OK(cudaMalloc(&h->tk_alt, 8 * want));
          MKNN_CUDA_OK(cudaMalloc(&h->tv, 4 * want));
          MKNN_CUDA_OK(cudaMalloc(&h->tv_alt, 4 * want));
          if (!h->tk_cnt) MKNN_CUDA_OK(cudaMalloc(&h->tk_cnt, 16));
          h->cap_tk = want;
        }
        MKNN_CUDA_OK(cudaMemsetAsync(h->tk_cnt, 0, 16, s));
        a.task_keys = h->tk;
        a.task_count = h->tk_cnt;
        a.task_cap = h->cap_tk;
      }
      sliced = sink && nq >= SLICE_MIN_QUERIES;
      // MKNN_SLICES=n (<= 16): result-row slices of a host tick (A/B)
      static const int n_slices = [] {
        const char* e = getenv("MKNN_SLICES");
        const int v = e ? atoi(e) : 4;
        return v < 1 ? 1 : (v > MAX_SLICES ? MAX_SLICES : v);
      }();
      h->rows_in_host = false;
      if (!sliced) {
        if ((rc = search_launch(a, s))) return h->set_err(rc);
      } else {
        // stable partition of the leaf-grouped order by result-row slice: slice
        // j holds rows [ceil(j nq / S), ceil((j + 1) nq / S)), each slice keeps
        // the leaf order (one 8-bit radix pass), then slice j's rows are copied
        // out while slice j + 1 searches
        // slice sizes grow geometrically (x4): the first slice's rows reach
        // the host after a short search, and each later slice searches
        // (~4.5x faster than PCIe carries its rows) while the previous one
        // is copied, so the device->host link stays busy from the first
        // slice on; MKNN_SLICE_GEO=0: equal slices (A/B)
        static const bool geo = [] {
          const char* e = getenv("MKNN_SLICE_GEO");
          return !(e && e[0] == '0');
        }();
        SliceBounds sb{};
        sb.n = n_slices;
        double tot = 0.0, w = 1.0;
        for (int j = 0; j < n_slices; j++, w *= (geo ? 4.0 : 1.0)) tot += w;
        double acc = 0.0;
        w = 1.0;
        for (int j = 0; j <= n_slices; j++) {
          sb.b[j] = j == n_slices ? nq : (int64_t)((double)nq * acc / tot);
          if (j < n_slices) acc += w;
          w *= geo ? 4.0 : 1.0;
        }
        MKNN_LAUNCH k_slice_keys<<<(unsigned)((nq + 255) / 256), 256, 0, s>>>(
            h->dq.order, h->dq.row, nq, sb, h->dq.keys, h->dq.vals);
        bool alt = false;
        if ((rc = radix_sort_pairs_u64(h->dq.keys, h->dq.vals, h->dq.keys_alt, h->dq.vals_alt, nq, 8,
                                       h->scratch.p, s, &alt)))
          return h->set_err(rc);
        const uint32_t* sorder = alt ? h->dq.vals_alt : h->dq.vals;
        if (o.qids) {  // issuer-ordered query ids are final already
          MKNN_CUDA_OK(cudaEventRecord(h->ev[6], s));
          MKNN_CUDA_OK(cudaStreamWaitEvent(h->copy_stream, h->ev[6], 0));
          MKNN_CUDA_OK(cudaMemcpyAsync(sink->qids, o.qids, sizeof(int64_t) * nq, cudaMemcpyDeviceToHost,
                                       h->copy_stream));
        }
        for (int j = 0; j < n_slices; j++) {
          const int64_t r0 = sb.b[j];
          const int64_t r1 = sb.b[j + 1];
          if (r1 <= r0) continue;
          SearchArgs aj = a;
          aj.q_order = sorder + r0;
          aj.nq = r1 - r0;
          aj.stats = h->stats + r0;
          if ((rc = search_launch(aj, s))) return h->set_err(rc);
          MKNN_CUDA_OK(cudaEventRecord(h->slice_ev[j], s));
          MKNN_CUDA_OK(cudaStreamWaitEvent(h->copy_stream, h->slice_ev[j], 0));
          cudaStream_t c = h->copy_stream;
          MKNN_CUDA_OK(cudaMemcpyAsync(sink->len + r0, o.len + r0, sizeof(int32_t) * (r1 - r0),
                                       cudaMemcpyDeviceToHost, c));
          MKNN_CUDA_OK(cudaMemcpyAsync(sink->nids + r0 * k, o.nids + r0 * k,
                                       sizeof(int64_t) * (r1 - r0) * k, cudaMemcpyDeviceToHost, c));
          MKNN_CUDA_OK(cudaMemcpyAsync(sink->dist + r0 * k, o.dist + r0 * k,
                                       sizeof(double) * (r1 - r0) * k, cudaMemcpyDeviceToHost, c));
        }
      }
      MKNN_CUDA_OK(cudaEventRecordWithFlags(h->ev[4], s, ev_flags));
      m.streamed_records = -1;
      if (instr) {
        unsigned long long nk = 0;
        MKNN_CUDA_OK(cudaMemcpyAsync(&nk, h->tk_cnt, 8, cudaMemcpyDeviceToHost, s));
        MKNN_CUDA_OK(cudaStreamSynchronize(s));
        if ((int64_t)nk <= h->cap_tk) {
          size_t need = radix_scratch_bytes((int64_t)nk) + 1024;
          if ((rc = h->scratch.ensure(std::max(need, h->scratch.cap)))) return h->set_err(rc);
          if ((rc = streamed_records(h->tk, h->tk_alt, h->tv, h->tv_alt, (int64_t)nk, h->st.cell_start,
                                     h->tk_cnt + 1, h->scratch.p, s)))
            return h->set_err(rc);
          unsigned long long T = 0;
          MKNN_CUDA_OK(cudaMemcpyAsync(&T, h->tk_cnt + 1, 8, cudaMemcpyDeviceToHost, s));
          MKNN_CUDA_OK(cudaStreamSynchronize(s));
          m.streamed_records = (int64_t)T;
        }
      }
      MKNN_CUDA_OK(cudaMemsetAsync(h->hist, 0, sizeof(uint32_t) * 2 * h->hist_cap, s));
      if ((rc = stats_reduce(h->stats, nq, h->counters, h->hist, h->hist + h->hist_cap, h->hist_cap, s)))
        return h->set_err(rc);
      if ((rc = rows_compact(o.len, o.nids, o.dist, nq, k, o.offsets, h->out_nids, h->out_dist,
                             h->dq.dup,
                             h->scratch.p, s)))
        return h->set_err(rc);
      MKNN_CUDA_OK(cudaEventRecordWithFlags(h->ev[5], s, ev_flags));

      prof_on = a.prof != nullptr;
      // every small readback of the tick into the pinned block (mapped: one
      // kernel writes it), one sync; nsnap is checked on speculative ticks only
      MKNN_LAUNCH k_readback<<<1, 256, 0, s>>>(h->counters, nq ? h->dq.minmax : nullptr, o.offsets + nq,
                                               nq ? h->dq.dup : nullptr,
                                               h->n_spec >= 0 ? h->d_nsnap : nullptr, h->hist,
                                               h->hist_cap, nq ? (int)hpre : 0, h->pin_dev);
      MKNN_CUDA_OK(cudaGetLastError());
      return 0;
    };
    erc = enqueue();
    if (graphable) {
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(h->cap_stream, &g);
      s = h->stream = user_s;
      if (erc) {
        if (g) cudaGraphDestroy(g);
        return erc;
      }
      MKNN_CUDA_OK(ce);
      if (h->gexec) cudaGraphExecDestroy(h->gexec);
      h->gexec = nullptr;
      h->gkey.clear();
      const cudaError_t ie = cudaGraphInstantiate(&h->gexec, g, 0);
      cudaGraphDestroy(g);
      MKNN_CUDA_OK(ie);
      h->gkey = gkey;
      h->graph_kernels = launch_count() - launches0;
      h->graph_dirty_after = h->st.dirty;
      MKNN_CUDA_OK(cudaGraphLaunch(h->gexec, s));
      h->graph_captures++;
    } else if (erc) {
      return erc;
    }
  }
  PinBlock& pb = *h->pin;
  MKNN_CUDA_OK(cudaStreamSynchronize(s));
  const unsigned long long* cnt = pb.cnt;
  const int64_t* mm = pb.mm;
  const int64_t total = pb.total;
  if (sliced) {
    MKNN_CUDA_OK(cudaStreamSynchronize(h->copy_stream));
    h->rows_in_host = total == nq * (int64_t)k;  // short rows: the caller copies the CSR
  }
  if (cnt[4]) {
    // a bucket outgrew its planned staging region (one-pass partition):
    // the store is incomplete -> redo the tick with the two-pass partition
    *retry = true;
    h->two_pass_next = true;
    h->retry_rebuild = rebuild;
    h->st.valid = false;  // the store is incomplete: no incremental redo on top of it
    return 0;
  }
  h->two_pass_next = false;
  if (h->n_spec >= 0 && pb.nsnap != h->n_spec) {
    // the updates since the last confirmed size appended ids: the tick ran
    // on a short snapshot -> core_tick syncs the size and redoes it
    *retry = true;
    h->snap_retry = true;
    h->retry_rebuild = rebuild;
    return 0;
  }
  if (nq) {
    // the issuer sort was planned from the previous tick's id range: if this
    // tick's range needs more bits the row order is wrong -> redo the tick
    // dup bit 0: an issuer id repeated inside the planned range (rows by
    // radix sort from now on); bit 1: ids beyond the planned range
    const int need = issuer_bits(mm[0], mm[1]);
    h->issuer_bits = need;
    if (pb.dup & 1) h->issuer_dups = true;
    if (need > bits_used || pb.dup) {
      *retry = true;
      h->retry_rebuild = rebuild;
      // the redo sorts with the radix path: ids that were out of span may
      // still repeat, which the bitmap would only find on a third pass
      h->retry_radix = true;
      return 0;
    }
  }

  // engine.py:661-663 active lists from navigate-call histograms
  for (int d = 0; d < 2; d++) {
    h->active[d].clear();
    if (nq == 0) continue;
    // the histogram prefix that can be non-zero (read with the counters;
    // longer walks fetch more)
    std::vector<uint32_t> hh(pb.hist[d], pb.hist[d] + hpre);
    int64_t lim = hpre;
    for (;;) {
      int64_t seen = 0;
      for (auto v : hh) seen += v;
      if (seen >= nq || lim >= h->hist_cap) break;
      lim = std::min<int64_t>(h->hist_cap, lim * 16);
      hh.resize(lim);
      MKNN_CUDA_OK(cudaMemcpy(hh.data(), h->hist + (int64_t)d * h->hist_cap, sizeof(uint32_t) * lim,
                              cudaMemcpyDeviceToHost));
    }
    int64_t maxc = 0;
    for (int64_t c = 0; c < (int64_t)hh.size(); c++)
      if (hh[c]) maxc = c;
    int64_t alive = nq;
    for (int64_t i = 1; i <= maxc; i++) {
      alive -= hh[i - 1];
      h->active[d].push_back(alive);
    }
  }
  m.iterations_left = (int64_t)h->active[0].size();
  m.iterations_right = (int64_t)h->active[1].size();
  m.distance_evals = (int64_t)cnt[0];
  m.pruned_leaves = (int64_t)cnt[1];
  m.pruning_violations = (int64_t)cnt[2];
  m.clamped_objects = (int64_t)cnt[3];
  m.n_results = total;
  m.t_build_us = us_between(h->ev[0], h->ev[1]);
  m.t_index_objects_us = us_between(h->ev[1], h->ev[2]);
  m.t_index_queries_us = us_between(h->ev[2], h->ev[3]);
  {
    // the search kernel runs first_iteration and the direction loop per
    // query batch: its event time is split by the batches' measured warp
    // time in the own-leaf pass (engine.py:641-642's two phases)
    const int64_t t_search = us_between(h->ev[3], h->ev[4]);
    const double own = (double)cnt[6], all = (double)cnt[7];
    m.t_first_iteration_us =
        all > 0.0 ? std::min<int64_t>(t_search, (int64_t)(t_search * (own / all) + 0.5)) : 0;
    m.t_loop_us = t_search - m.t_first_iteration_us;
  }
  m.t_emit_us = us_between(h->ev[4], h->ev[5]);

  h->last_tick_ok = true;
  h->history.push_back(m.distance_evals);
  h->tick += 1;
  m.t_total_us = std::chrono::duration_cast<std::chrono::microseconds>(
                     std::chrono::steady_clock::now() - t_start)
                     .count();
  if (prof_on) {  // profiling only (MKNN_PROF=1)
    unsigned long long pv[14];
    MKNN_CUDA_OK(cudaMemcpy(pv, h->prof, sizeof(pv), cudaMemcpyDeviceToHost));
    fprintf(stderr,
            "[mknn prof] expansion rounds %.3g (%.2f per query), active lanes per round %.2f, "
            "navigate steps %.2f per query, step efficiency (sum / 32 x per-round max) %.2f\n",
            (double)pv[10], (double)pv[10] * 32.0 / nq, (double)pv[11] / (pv[10] ? pv[10] : 1),
            (double)pv[12] / nq, (double)pv[12] / (32.0 * (pv[13] ? pv[13] : 1)));
    fprintf(stderr,
            "[mknn prof] per query: own chunks %.2f/%.2f, exp leaves %.2f, exp chunks %.2f/%.2f, "
            "admitted %.2f, inserts %.2f, sort-merges %.2f; exp visits without scans %.2f, "
            "with admissions %.2f\n",
            (double)pv[0] / nq, (double)pv[5] / nq, (double)pv[4] / nq, (double)pv[1] / nq,
            (double)pv[6] / nq, (double)pv[7] / nq, (double)pv[2] / nq, (double)pv[3] / nq,
            (double)pv[8] / nq, (double)pv[9] / nq);
  }
  if (met) *met = m;
  return 0;
}

int core_tick_run(mknn_engine* h, int64_t n, const long long* ids, const double* x, const double* y,
                  int64_t nq, const long long* qi, const double* qx, const double* qy, const DevOut& o,
                  mknn_metrics* met, std::chrono::steady_clock::time_point t_start,
                  const HostSink* sink);

// one tick (with its redo when needed); a speculative snapshot size set by
// snap_prepare_query applies to this tick only
int core_tick(mknn_engine* h, int64_t n, const long long* ids, const double* x, const double* y,
              int64_t nq, const long long* qi, const double* qx, const double* qy, const DevOut& o,
              mknn_metrics* met, std::chrono::steady_clock::time_point t_start,
              const HostSink* sink = nullptr) {
  const int rc = core_tick_run(h, n, ids, x, y, nq, qi, qx, qy, o, met, t_start, sink);
  if (h->n_spec >= 0) {  // confirmed (or failed): the host bounds are stale either way
    h->n_spec = -1;
    if (rc == 0) {  // the size was checked equal; the full re-index consumed every move
      h->n_snap_hi = h->n_snap;
      h->nmoved_hi = 0;
      h->upd_pending = false;
    }
  }
  return rc;
}

int core_tick_run(mknn_engine* h, int64_t n, const long long* ids, const double* x, const double* y,
                  int64_t nq, const long long* qi, const double* qx, const double* qy, const DevOut& o,
                  mknn_metrics* met, std::chrono::steady_clock::time_point t_start,
                  const HostSink* sink) {
  bool retry = false;
  int rc = core_tick_once(h, n, ids, x, y, nq, qi, qx, qy, o, met, t_start, false, &retry, sink);
  if (rc || !retry) return rc;
  if (h->snap_retry) {  // ran on a stale snapshot size: settle it, redo in full
    h->snap_retry = false;
    h->n_spec = -1;
    if ((rc = snap_sync(h))) return h->set_err(rc);
    h->st.valid = false;  // the moved list was reset by the discarded tick
    n = h->n_snap;
    if ((rc = validate_counts(h, n, nq))) return rc;
    rc = core_tick_once(h, n, ids, x, y, nq, qi, qx, qy, o, met, t_start, h->retry_rebuild, &retry,
                        sink);
    if (rc || !retry) return rc;
  }
  // issuer bits now measured exactly: the second pass cannot retry
  rc = core_tick_once(h, n, ids, x, y, nq, qi, qx, qy, o, met, t_start, h->retry_rebuild, &retry,
                      sink);
  if (!rc && retry) return fail_msg(E_CUDA, "issuer order retry did not converge");
  return rc;
}

int validate_counts(mknn_engine* h, int64_t n, int64_t nq) {
  if (n < 0 || nq < 0) return h->invalid("negative object or query count");
  if (n > 0x7ffffff0LL) return h->invalid("more than 2^31 objects per tick");
  if (nq > 0x7ffffff0LL) return h->invalid("more than 2^31 queries per tick");
  if (nq * (int64_t)h->cfg.k > (int64_t)1 << 40) return h->invalid("result size too large");
  return 0;
}

int check_unique_host(mknn_engine* h, int64_t n, const int64_t* ids) {
  std::vector<int64_t> v(ids, ids + n);
  std::sort(v.begin(), v.end());
  if (std::adjacent_find(v.begin(), v.end()) != v.end())
    return h->invalid("duplicate object ids in tick batch");  // engine.py:611-612
  return 0;
}

int check_unique_dev(mknn_engine* h, int64_t n, const int64_t* d_ids) {
  std::vector<int64_t> v((size_t)n);
  if (n) MKNN_CUDA_OK(cudaMemcpy(v.data(), d_ids, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
  return check_unique_host(h, n, v.data());
}

int ensure_out_dev(mknn_engine* h, int64_t nq) {
  int rc;
  const int64_t rows = std::max<int64_t>(nq * (int64_t)h->cfg.k, 1);
  if (rows > h->cap_c) {
    int64_t c = h->cap_c;
    if ((rc = grow(h->c_nids, c, rows))) return rc;
    c = h->cap_c;
    if ((rc = grow(h->c_dist, c, rows))) return rc;
    h->cap_c = c;
  }
  if ((rc = grow(h->offsets, h->cap_off, nq + 1))) return rc;
  if ((rc = grow(h->out_qids, h->cap_oq, std::max<int64_t>(nq, 1)))) return rc;
  if ((rc = grow(h->out_len, h->cap_len, std::max<int64_t>(nq, 1)))) return rc;
  return 0;
}

// host-output tick over device-resident inputs (mknn_tick / mknn_query)
int host_out_tick(mknn_engine* h, int64_t n, const long long* ids, const double* x, const double* y,
                  int64_t nq, const long long* qi, const double* qx, const double* qy,
                  int64_t* out_qids, int32_t* out_len, int64_t* out_nids, double* out_dist,
                  mknn_metrics* metrics, std::chrono::steady_clock::time_point t0) {
  int rc;
  if ((rc = ensure_out_dev(h, nq))) return h->set_err(rc);
  DevOut o{h->out_qids, h->out_len, h->offsets, h->c_nids, h->c_dist};
  const HostSink sink{out_qids, out_len, out_nids, out_dist};
  mknn_metrics m{};
  if ((rc = core_tick(h, n, ids, x, y, nq, qi, qx, qy, o, &m, t0, &sink))) return rc;
  cudaStream_t s = h->stream;
  if (h->rows_in_host) {
    m.t_total_us = std::chrono::duration_cast<std::chrono::microseconds>(
                       std::chrono::steady_clock::now() - t0)
                       .count();
    if (metrics) *metrics = m;
    return 0;
  }
  if (nq) {
    MKNN_CUDA_OK(cudaMemcpyAsync(out_qids, h->out_qids, sizeof(int64_t) * nq, cudaMemcpyDeviceToHost, s));
    MKNN_CUDA_OK(cudaMemcpyAsync(out_len, h->out_len, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, s));
  }
  if (m.n_results) {
    MKNN_CUDA_OK(cudaMemcpyAsync(out_nids, h->c_nids, sizeof(int64_t) * m.n_results,
                                 cudaMemcpyDeviceToHost, s));
    MKNN_CUDA_OK(cudaMemcpyAsync(out_dist, h->c_dist, sizeof(double) * m.n_results,
                                 cudaMemcpyDeviceToHost, s));
  }
  MKNN_CUDA_OK(cudaStreamSynchronize(s));
  m.t_total_us = std::chrono::duration_cast<std::chrono::microseconds>(
                     std::chrono::steady_clock::now() - t0)
                     .count();
  if (metrics) *metrics = m;
  return 0;
}

int stage_queries(mknn_engine* h, int64_t nq, const int64_t* qi, const double* qx, const double* qy,
                  cudaStream_t via = nullptr) {
  int rc;
  int64_t c = h->cap_qin;
  if ((rc = grow(h->in_qi, c, std::max<int64_t>(nq, 1)))) return rc;
  c = h->cap_qin;
  if ((rc = grow(h->in_qx, c, std::max<int64_t>(nq, 1)))) return rc;
  c = h->cap_qin;
  if ((rc = grow(h->in_qy, c, std::max<int64_t>(nq, 1)))) return rc;
  h->cap_qin = c;
  // on the copy stream: the queries cross PCIe while the objects are
  // (re-)indexed; the tick waits for them just before index_queries
  cudaStream_t cs = via ? via : h->copy_stream;
  if (!via) {  // (via: a stream already ordered after the previous call)
    MKNN_CUDA_OK(cudaEventRecord(h->ev[7], h->stream));  // inputs of the previous call consumed
    MKNN_CUDA_OK(cudaStreamWaitEvent(cs, h->ev[7], 0));
  }
  if (nq) {
    MKNN_CUDA_OK(cudaMemcpyAsync(h->in_qi, qi, sizeof(int64_t) * nq, cudaMemcpyHostToDevice, cs));
    MKNN_CUDA_OK(cudaMemcpyAsync(h->in_qx, qx, sizeof(double) * nq, cudaMemcpyHostToDevice, cs));
    MKNN_CUDA_OK(cudaMemcpyAsync(h->in_qy, qy, sizeof(double) * nq, cudaMemcpyHostToDevice, cs));
  }
  MKNN_CUDA_OK(cudaEventRecord(h->q_ready, cs));
  h->q_pending = true;
  return 0;
}

// ----------------------------------------------------------- delta snapshot
int snap_reserve(mknn_engine* h, int64_t want) {
  if (want <= h->cap_snap && h->ht) return 0;
  int rc0;
  if ((rc0 = snap_sync(h))) return rc0;  // the rehash walks the exact snapshot
  const int64_t nc = std::max<int64_t>(want, std::max<int64_t>(h->cap_snap * 3 / 2, 1024));
  cudaStream_t s = h->stream;
  long long* ni = nullptr;
  double *nx = nullptr, *ny = nullptr;
  MKNN_CUDA_OK(cudaMalloc(&ni, sizeof(long long) * nc));
  MKNN_CUDA_OK(cudaMalloc(&nx, sizeof(double) * nc));
  MKNN_CUDA_OK(cudaMalloc(&ny, sizeof(double) * nc));
  if (h->n_snap) {
    MKNN_CUDA_OK(cudaMemcpyAsync(ni, h->snap_ids, sizeof(long long) * h->n_snap, cudaMemcpyDeviceToDevice, s));
    MKNN_CUDA_OK(cudaMemcpyAsync(nx, h->snap_x, sizeof(double) * h->n_snap, cudaMemcpyDeviceToDevice, s));
    MKNN_CUDA_OK(cudaMemcpyAsync(ny, h->snap_y, sizeof(double) * h->n_snap, cudaMemcpyDeviceToDevice, s));
  }
  MKNN_CUDA_OK(cudaStreamSynchronize(s));
  cudaFree(h->snap_ids);
  cudaFree(h->snap_x);
  cudaFree(h->snap_y);
  h->snap_ids = ni;
  h->snap_x = nx;
  h->snap_y = ny;
  h->cap_snap = nc;
  // rehash at <= 50 % load
  int64_t hc = 1;
  while (hc < 2 * nc) hc <<= 1;
  cudaFree(h->ht);
  cudaFree(h->winner);
  MKNN_CUDA_OK(cudaMalloc(&h->ht, sizeof(HashSlot) * hc));
  MKNN_CUDA_OK(cudaMalloc(&h->winner, sizeof(unsigned long long) * nc));
  cudaFree(h->mark);
  cudaFree(h->moved);
  MKNN_CUDA_OK(cudaMalloc(&h->mark, sizeof(int32_t) * nc));
  MKNN_CUDA_OK(cudaMalloc(&h->moved, sizeof(int32_t) * nc));
  if (!h->d_nmoved) MKNN_CUDA_OK(cudaMalloc(&h->d_nmoved, sizeof(int32_t)));
  MKNN_CUDA_OK(cudaMemsetAsync(h->mark, 0, sizeof(int32_t) * nc, s));
  MKNN_CUDA_OK(cudaMemsetAsync(h->d_nmoved, 0, sizeof(int32_t), s));
  h->h_nmoved = 0;
  h->st.valid = false;  // moved-slot history lost
  h->hcap = hc;
  h->cap_winner = nc;
  if (!h->d_nsnap) {  // [0] the snapshot size, [1] its value before the current update batch
    MKNN_CUDA_OK(cudaMalloc(&h->d_nsnap, 2 * sizeof(int32_t)));
    MKNN_CUDA_OK(cudaMemsetAsync(h->d_nsnap, 0, 2 * sizeof(int32_t), s));
  }
  MKNN_LAUNCH k_fill_slots<<<gs_blocks(hc), 256, 0, s>>>(h->ht, hc);
  MKNN_CUDA_OK(cudaMemsetAsync(h->winner, 0, sizeof(unsigned long long) * nc, s));
  h->upd_seq = 0;
  if (h->n_snap)
    MKNN_LAUNCH k_hash_load<<<gs_blocks(h->n_snap), 256, 0, s>>>(h->snap_ids, h->n_snap, h->ht,
                                                                 (uint64_t)(hc - 1));
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

int snap_load_dev(mknn_engine* h, int64_t n, const long long* ids, const double* x, const double* y) {
  int rc;
  h->upd_pending = false;  // replaced wholesale
  h->n_snap = h->n_snap_hi = 0;
  h->st.valid = false;
  if ((rc = snap_reserve(h, std::max<int64_t>(n, 1)))) return rc;
  cudaStream_t s = h->stream;
  if (n) {
    MKNN_CUDA_OK(cudaMemcpyAsync(h->snap_ids, ids, sizeof(long long) * n, cudaMemcpyDeviceToDevice, s));
    MKNN_CUDA_OK(cudaMemcpyAsync(h->snap_x, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    MKNN_CUDA_OK(cudaMemcpyAsync(h->snap_y, y, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }
  MKNN_LAUNCH k_fill_slots<<<gs_blocks(h->hcap), 256, 0, s>>>(h->ht, h->hcap);
  if (n)
    MKNN_LAUNCH k_hash_load<<<gs_blocks(n), 256, 0, s>>>(h->snap_ids, n, h->ht,
                                                         (uint64_t)(h->hcap - 1));
  MKNN_CUDA_OK(cudaGetLastError());
  h->n_snap = h->n_snap_hi = n;
  h->nmoved_hi = 0;
  h->upd_pending = false;
  const int32_t ns = (int32_t)n;
  MKNN_CUDA_OK(cudaMemcpyAsync(h->d_nsnap, &ns, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  MKNN_CUDA_OK(cudaStreamSynchronize(s));  // ns lives on this stack frame
  return 0;
}

// the exact snapshot size and moved-slot count after sync-free updates
int snap_sync(mknn_engine* h) {
  if (!h->upd_pending) return 0;
  if (!h->pin) {
    MKNN_CUDA_OK(cudaHostAlloc(&h->pin, sizeof(PinBlock), cudaHostAllocMapped));
    MKNN_CUDA_OK(cudaHostGetDevicePointer(&h->pin_dev, h->pin, 0));
  }
  cudaStream_t s = h->stream;
  MKNN_CUDA_OK(cudaMemcpyAsync(&h->pin->nsnap, h->d_nsnap, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  MKNN_CUDA_OK(cudaMemcpyAsync(&h->pin->dup, h->d_nmoved, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  MKNN_CUDA_OK(cudaStreamSynchronize(s));
  h->n_snap = h->n_snap_hi = h->pin->nsnap;
  h->h_nmoved = h->nmoved_hi = h->pin->dup;
  h->upd_pending = false;
  return 0;
}

// datasets.py:109-164 carry-forward over the device snapshot.  No host
// sync: the snapshot size (grown by ids seen for the first time) and the
// moved-slot count stay on the device; the host keeps upper bounds, and a
// query tick either runs on the unconfirmed size and checks it at its end
// (core_tick redoes the tick if ids were appended) or syncs first when the
// incremental re-index could be chosen (it needs the exact moved count).
int snap_update_dev(mknn_engine* h, int64_t nu, const long long* ids, const double* x, const double* y) {
  int rc;
  if (nu == 0) return 0;
  if (h->n_snap_hi + nu > h->cap_snap || !h->ht) {  // growth rehashes from the exact size
    if ((rc = snap_sync(h))) return rc;
    if ((rc = snap_reserve(h, h->n_snap + nu))) return rc;
  }
  if ((rc = grow(h->slot_of, h->cap_slot_of, nu))) return rc;
  cudaStream_t s = h->stream;
  MKNN_CUDA_OK(cudaMemcpyAsync(h->d_nsnap + 1, h->d_nsnap, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  if (++h->upd_seq >= (1ull << 32)) {  // the high word would wrap: start over
    MKNN_CUDA_OK(cudaMemsetAsync(h->winner, 0, sizeof(unsigned long long) * h->cap_winner, s));
    h->upd_seq = 1;
  }
  const unsigned long long seq = h->upd_seq;
  MKNN_LAUNCH k_update_claim<<<gs_blocks(nu), 256, 0, s>>>(ids, nu, h->ht, (uint64_t)(h->hcap - 1),
                                               h->d_nsnap, h->winner, h->slot_of, seq);
  // a batch above the incremental threshold on its own (engine: > 5 % of
  // the snapshot) sends the next tick to the full re-index anyway: skip the
  // moved-slot bookkeeping (a random read-modify-write per update) and mark
  // the store stale so the incremental path cannot be chosen on a partial list
  const bool track = nu * 20 <= h->n_snap;
  if (!track) h->st.valid = false;
  MKNN_LAUNCH k_update_apply<<<gs_blocks(nu), 256, 0, s>>>(ids, x, y, nu, h->slot_of, h->winner, seq,
                                               h->snap_ids,
                                               h->snap_x, h->snap_y, h->mark, h->epoch, h->moved,
                                               h->d_nmoved, track, h->d_nsnap + 1);
  MKNN_CUDA_OK(cudaGetLastError());
  h->upd_pending = true;
  h->n_snap_hi += nu;
  h->nmoved_hi += nu;
  return 0;
}

// before a query tick over the snapshot: settle what the host must know
int snap_prepare_query(mknn_engine* h) {
  h->n_spec = -1;
  if (!h->upd_pending) return 0;
  // the incremental re-index (core_tick_once) needs the exact moved count;
  // with the bound above its threshold it cannot be chosen, so run on the
  // last confirmed size and check it at the tick's end
  const int64_t n = h->n_snap_hi;
  if (h->st.valid && h->st.n_store <= n && (h->nmoved_hi + (n - h->st.n_store)) * 20 <= n)
    return snap_sync(h);
  // the tick must take the full re-index: the incremental one would walk
  // the moved list with a count the host does not know yet
  h->h_nmoved = int64_t(1) << 40;
  h->n_spec = h->n_snap;
  return 0;
}

}  // namespace

// ===================================================================== ABI
extern "C" {

int mknn_abi_version(void) { return MKNN_ABI_VERSION; }

int64_t mknn_kernel_launches(void) { return (int64_t)launch_count(); }

int mknn_create(const mknn_config* cfg, mknn_engine** out) {
  if (!cfg || !out) return MKNN_EINVAL;
  *out = nullptr;
  // EngineConfig.__post_init__ (engine.py:73-85) and build_index's checks
  // (quadindex.py:86-89) -- the Python shim raises the same ValueErrors first.
  if (cfg->k < 1 || cfg->th_quad < 1 || cfg->l_max < 1 || cfg->l_max > MAX_L_MAX ||
      cfg->rebuild_window < 1 || !(cfg->rebuild_factor > 0))
    return MKNN_EINVAL;
  if (!(std::isfinite(cfg->x_lo) && std::isfinite(cfg->y_lo) && std::isfinite(cfg->x_hi) &&
        std::isfinite(cfg->y_hi)) ||
      cfg->x_lo > cfg->x_hi || cfg->y_lo > cfg->y_hi)
    return MKNN_EINVAL;
  if (cfg->k > 512) return MKNN_EUNSUPPORTED;
  auto* h = new mknn_engine();
  h->cfg = *cfg;
  h->device = cfg->device;
  {
    const double w = cfg->x_hi - cfg->x_lo, hh = cfg->y_hi - cfg->y_lo;
    h->r = Region{cfg->x_lo, cfg->y_lo, cfg->x_hi, cfg->y_hi, w, hh, w > 0.0 ? 1.0 / w : 0.0,
                  hh > 0.0 ? 1.0 / hh : 0.0};
  }
  int rc = bind(h);
  if (!rc) rc = index_alloc(h->ix, cfg->l_max, cfg->th_quad);
  if (!rc && cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess) rc = E_CUDA;
  for (int i = 0; i < 8 && !rc; i++)
    if (cudaEventCreate(&h->ev[i]) != cudaSuccess) rc = E_CUDA;
  for (int i = 0; i < MAX_SLICES && !rc; i++)
    if (cudaEventCreateWithFlags(&h->slice_ev[i], cudaEventDisableTiming) != cudaSuccess) rc = E_CUDA;
  if (!rc && cudaEventCreateWithFlags(&h->q_ready, cudaEventDisableTiming) != cudaSuccess)
    rc = E_CUDA;
  if (!rc && cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
    rc = E_CUDA;
  if (!rc && cudaStreamCreateWithFlags(&h->in_stream, cudaStreamNonBlocking) != cudaSuccess)
    rc = E_CUDA;
  for (auto& e : h->in_ev)
    if (!rc && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) rc = E_CUDA;
  if (!rc && cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
    rc = E_CUDA;
  if (rc) {
    mknn_destroy(h);
    return rc;
  }
  h->stream = h->own_stream;
  *out = h;
  return 0;
}

void mknn_destroy(mknn_engine* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  index_free(h->ix);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  for (void* p : engine_buffers(h))
    if (p) cudaFree(p);
  h->scratch.release();
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->slice_ev)
    if (e) cudaEventDestroy(e);
  if (h->q_ready) cudaEventDestroy(h->q_ready);
  if (h->pin) cudaFreeHost(h->pin);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->in_stream) cudaStreamDestroy(h->in_stream);
  for (auto& e : h->in_ev)
    if (e) cudaEventDestroy(e);
  if (h->pre_counts) cudaFree(h->pre_counts);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
}

// the message of the most recent failure on the calling thread
const char* mknn_last_error(const mknn_engine* h) {
  (void)h;
  return last_error_text();
}

int mknn_set_stream(mknn_engine* h, void* cuda_stream) {
  if (!h) return MKNN_EINVAL;
  h->stream = cuda_stream ? (cudaStream_t)cuda_stream : h->own_stream;
  return 0;
}

int mknn_tick(mknn_engine* h, int64_t n, const int64_t* ids, const double* x, const double* y,
              int64_t nq, const int64_t* q_issuer, const double* qx, const double* qy,
              int64_t* out_qids, int32_t* out_len, int64_t* out_nids, double* out_dist,
              mknn_metrics* metrics) {
  if (!h) return MKNN_EINVAL;
  const auto t0 = std::chrono::steady_clock::now();
  int rc;
  if ((rc = bind(h))) return h->set_err(rc);
  if ((rc = validate_counts(h, n, nq))) return rc;
  if ((n && (!ids || !x || !y)) || (nq && (!q_issuer || !qx || !qy || !out_qids || !out_len ||
                                          !out_nids || !out_dist)))
    return h->invalid("null buffer");
  if (h->cfg.self_check && (rc = check_unique_host(h, n, ids))) return rc;
  int64_t c = h->cap_in;
  if ((rc = grow(h->in_ids, c, std::max<int64_t>(n, 1)))) return h->set_err(rc);
  c = h->cap_in;
  if ((rc = grow(h->in_x, c, std::max<int64_t>(n, 1)))) return h->set_err(rc);
  c = h->cap_in;
  if ((rc = grow(h->in_y, c, std::max<int64_t>(n, 1)))) return h->set_err(rc);
  h->cap_in = c;
  cudaStream_t s = h->stream;
  // a steady-state tick that will take the one-pass partition (as
  // core_tick_once decides: no rebuild, counts of the last bucket sort, no
  // pending two-pass redo, balanced buckets) partitions each chunk of the
  // objects as soon as it has crossed PCIe
  static const bool overlap = [] {
    const char* e = getenv("MKNN_H2D_OVERLAP");
    const char* b = getenv("MKNN_BSORT");
    const char* o = getenv("MKNN_ONEPASS");
    return !(e && e[0] == '0') && !(b && b[0] == '0') && !(o && o[0] == '0');
  }();
  h->prepartitioned = false;
  if (overlap && n >= (int64_t)1 << 20 && h->have_index && h->st.bcnt_valid && !h->two_pass_next &&
      h->h_bucket_load <= 4 * 16 && h->h_bucket_keys <= 32768 &&
      !should_rebuild(h->history, h->cfg.rebuild_window, h->cfg.rebuild_factor)) {
    if ((rc = alloc_store(h, n))) return h->set_err(rc);
    if ((rc = store_reserve(h->st, h->h_n_sub, h->h_n_leaves, n))) return h->set_err(rc);
    if (!h->pre_counts) MKNN_CUDA_OK(cudaMalloc(&h->pre_counts, 2 * sizeof(unsigned long long)));
    MKNN_CUDA_OK(cudaMemsetAsync(h->pre_counts, 0, 2 * sizeof(unsigned long long), s));
    MKNN_CUDA_OK(cudaEventRecord(h->in_ev[3], s));  // the inputs of the previous tick are consumed
    MKNN_CUDA_OK(cudaStreamWaitEvent(h->in_stream, h->in_ev[3], 0));
    constexpr int C = 4;
    for (int c = 0; c < C; c++) {
      const int64_t lo = n * c / C, hi = n * (c + 1) / C;
      cudaStream_t is = h->in_stream;
      MKNN_CUDA_OK(cudaMemcpyAsync(h->in_ids + lo, ids + lo, sizeof(int64_t) * (hi - lo),
                                   cudaMemcpyHostToDevice, is));
      MKNN_CUDA_OK(cudaMemcpyAsync(h->in_x + lo, x + lo, sizeof(double) * (hi - lo),
                                   cudaMemcpyHostToDevice, is));
      MKNN_CUDA_OK(cudaMemcpyAsync(h->in_y + lo, y + lo, sizeof(double) * (hi - lo),
                                   cudaMemcpyHostToDevice, is));
      MKNN_CUDA_OK(cudaEventRecord(h->in_ev[c], is));
      MKNN_CUDA_OK(cudaStreamWaitEvent(s, h->in_ev[c], 0));
      if ((rc = store_prepartition(h->st, h->ix, h->r, h->in_ids, h->in_x, h->in_y, lo, hi, c == 0,
                                   h->pre_counts, s)))
        return h->set_err(rc);
    }
    h->prepartitioned = true;
    // the queries follow the objects on the same stream: the link stays busy
    // while the bucket sort runs
    if ((rc = stage_queries(h, nq, q_issuer, qx, qy, h->in_stream))) return h->set_err(rc);
  } else {
    if (n) {
      MKNN_CUDA_OK(cudaMemcpyAsync(h->in_ids, ids, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
      MKNN_CUDA_OK(cudaMemcpyAsync(h->in_x, x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      MKNN_CUDA_OK(cudaMemcpyAsync(h->in_y, y, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    }
    if ((rc = stage_queries(h, nq, q_issuer, qx, qy))) return h->set_err(rc);
  }
  return host_out_tick(h, n, h->in_ids, h->in_x, h->in_y, nq, h->in_qi, h->in_qx, h->in_qy,
                       out_qids, out_len, out_nids, out_dist, metrics, t0);
}

int mknn_tick_device(mknn_engine* h, int64_t n, const int64_t* d_ids, const double* d_x,
                     const double* d_y, int64_t nq, const int64_t* d_q_issuer, const double* d_qx,
                     const double* d_qy, int64_t* d_out_qids, int32_t* d_out_len,
                     int64_t* d_out_offsets, int64_t* d_out_nids, double* d_out_dist,
                     mknn_metrics* metrics) {
  if (!h) return MKNN_EINVAL;
  const auto t0 = std::chrono::steady_clock::now();
  int rc;
  if ((rc = bind(h))) return h->set_err(rc);
  if ((rc = validate_counts(h, n, nq))) return rc;
  if (!d_out_len || !d_out_offsets || (nq && (!d_out_nids || !d_out_dist)))
    return h->invalid("null buffer");
  if (h->cfg.self_check && (rc = check_unique_dev(h, n, d_ids))) return rc;
  DevOut o{(long long*)d_out_qids, d_out_len, d_out_offsets, (long long*)d_out_nids, d_out_dist};
  return core_tick(h, n, (const long long*)d_ids, d_x, d_y, nq, (const long long*)d_q_issuer, d_qx,
                   d_qy, o, metrics, t0);
}

int mknn_load(mknn_engine* h, int64_t n, const int64_t* ids, const double* x, const double* y) {
  if (!h) return MKNN_EINVAL;
  int rc;
  if ((rc = bind(h))) return h->set_err(rc);
  if ((rc = validate_counts(h, n, 0))) return rc;
  if (h->cfg.self_check && (rc = check_unique_host(h, n, ids))) return rc;
  int64_t c = h->cap_up;
  if ((rc = grow(h->up_ids, c, std::max<int64_t>(n, 1)))) return h->set_err(rc);
  c = h->cap_up;
  if ((rc = grow(h->up_x, c, std::max<int64_t>(n, 1)))) return h->set_err(rc);
  c = h->cap_up;
  if ((rc = grow(h->up_y, c, std::max<int64_t>(n, 1)))) return h->set_err(rc);
  h->cap_up = c;
  cudaStream_t s = h->stream;
  if (n) {
    MKNN_CUDA_OK(cudaMemcpyAsync(h->up_ids, ids, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    MKNN_CUDA_OK(cudaMemcpyAsync(h->up_x, x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    MKNN_CUDA_OK(cudaMemcpyAsync(h->up_y, y, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  }
  if ((rc = snap_load_dev(h, n, h->up_ids, h->up_x, h->up_y))) return h->set_err(rc);
  MKNN_CUDA_OK(cudaStreamSynchronize(s));
  return 0;
}

int mknn_update_device(mknn_engine* h, int64_t nu, const int64_t* d_ids, const double* d_x,
                       const double* d_y) {
  if (!h) return MKNN_EINVAL;
  int rc;
  if ((rc = bind(h))) return h->set_err(rc);
  if (nu < 0) return h->invalid("negative update count");
  if (h->n_snap_hi + nu > 0x7ffffff0LL && (rc = snap_sync(h))) return h->set_err(rc);
  if (h->n_snap + nu > 0x7ffffff0LL) return h->invalid("snapshot larger than 2^31 objects");
  if ((rc = snap_update_dev(h, nu, (const long long*)d_ids, d_x, d_y))) return h->set_err(rc);
  return 0;
}

int mknn_update(mknn_engine* h, int64_t nu, const int64_t* ids, const double* x, const double* y) {
  if (!h) return MKNN_EINVAL;
  int rc;
  if ((rc = bind(h))) return h->set_err(rc);
  if (nu < 0) return h->invalid("negative update count");
  if (nu == 0) return 0;
  int64_t c = h->cap_up;
  if ((rc = grow(h->up_ids, c, nu))) return h->set_err(rc);
  c = h->cap_up;
  if ((rc = grow(h->up_x, c, nu))) return h->set_err(rc);
  c = h->cap_up;
  if ((rc = grow(h->up_y, c, nu))) return h->set_err(rc);
  h->cap_up = c;
  cudaStream_t s = h->stream;
  MKNN_CUDA_OK(cudaMemcpyAsync(h->up_ids, ids, sizeof(int64_t) * nu, cudaMemcpyHostToDevice, s));
  MKNN_CUDA_OK(cudaMemcpyAsync(h->up_x, x, sizeof(double) * nu, cudaMemcpyHostToDevice, s));
  MKNN_CUDA_OK(cudaMemcpyAsync(h->up_y, y, sizeof(double) * nu, cudaMemcpyHostToDevice, s));
  return mknn_update_device(h, nu, (const int64_t*)h->up_ids, h->up_x, h->up_y);
}

int mknn_snapshot_size(const mknn_engine* h, int64_t* n) {
  if (!h || !n) return MKNN_EINVAL;
  int rc;
  if ((rc = snap_sync(const_cast<mknn_engine*>(h)))) return rc;
  *n = h->n_snap;
  return 0;
}

int mknn_query(mknn_engine* h, int64_t nq, const int64_t* q_issuer, const double* qx,
               const double* qy, int64_t* out_qids, int32_t* out_len, int64_t* out_nids,
               double* out_dist, mknn_metrics* metrics) {
  if (!h) return MKNN_EINVAL;
  const auto t0 = std::chrono::steady_clock::now();
  int rc;
  if ((rc = bind(h))) return h->set_err(rc);
  if ((rc = snap_prepare_query(h))) return h->set_err(rc);
  if ((rc = validate_counts(h, h->n_snap, nq))) return rc;
  if (nq && (!q_issuer || !qx || !qy || !out_qids || !out_len || !out_nids || !out_dist))
    return h->invalid("null buffer");
  if ((rc = stage_queries(h, nq, q_issuer, qx, qy))) return h->set_err(rc);
  return host_out_tick(h, h->n_snap, h->snap_ids, h->snap_x, h->snap_y, nq, h->in_qi, h->in_qx,
                       h->in_qy, out_qids, out_len, out_nids, out_dist, metrics, t0);
}

int mknn_query_device(mknn_engine* h, int64_t nq, const int64_t* d_q_issuer, const double* d_qx,
                      const double* d_qy, int64_t* d_out_qids, int32_t* d_out_len,
                      int64_t* d_out_offsets, int64_t* d_out_nids, double* d_out_dist,
                      mknn_metrics* metrics) {
  if (!h) return MKNN_EINVAL;
  const auto t0 = std::chrono::steady_clock::now();
  int rc;
  if ((rc = bind(h))) return h->set_err(rc);
  if ((rc = snap_prepare_query(h))) return h->set_err(rc);
  if ((rc = validate_counts(h, h->n_snap, nq))) return rc;
  DevOut o{(long long*)d_out_qids, d_out_len, d_out_offsets, (long long*)d_out_nids, d_out_dist};
  return core_tick(h, h->n_snap, h->snap_ids, h->snap_x, h->snap_y, nq,
                   (const long long*)d_q_issuer, d_qx, d_qy, o, metrics, t0);
}

int mknn_graph_stats(const mknn_engine* h, int64_t* captures, int64_t* replays) {
  if (!h) return MKNN_EINVAL;
  if (captures) *captures = h->graph_captures;
  if (replays) *replays = h->graph_replays;
  return 0;
}

int mknn_set_instrument(mknn_engine* h, int32_t flags) {
  if (!h) return MKNN_EINVAL;
  h->cfg.instrument = flags;
  return 0;
}

int mknn_set_last_evals(mknn_engine* h, int64_t distance_evals) {
  if (!h || h->history.empty() || distance_evals < 0) return MKNN_EINVAL;
  h->history.back() = distance_evals;
  return 0;
}

int64_t mknn_active_counts(const mknn_engine* h, int dir, int64_t* out, int64_t cap) {
  if (!h || dir < 0 || dir > 1) return MKNN_EINVAL;
  const auto& v = h->active[dir];
  for (int64_t i = 0; i < cap && i < (int64_t)v.size(); i++) out[i] = v[i];
  return (int64_t)v.size();
}

int mknn_index_info(const mknn_engine* h, int32_t* l_deep, int64_t* n_leaves,
                    int64_t* overfull_leaves, int64_t* n_build) {
  if (!h) return MKNN_EINVAL;
  if (!h->have_index) return MKNN_EINVAL;
  if (l_deep) *l_deep = h->h_l_deep;
  if (n_leaves) *n_leaves = h->h_n_leaves;
  if (overfull_leaves) *overfull_leaves = h->h_overfull;
  if (n_build) *n_build = h->h_n_build;
  return 0;
}

int mknn_index_export(mknn_engine* h, int32_t* leaf_level, int64_t* leaf_code, int64_t* leaf_key,
                      int64_t* leaf_span, int64_t* build_counts, int32_t* z_map) {
  if (!h || !h->have_index) return MKNN_EINVAL;
  int rc;
  if ((rc = bind(h))) return h->set_err(rc);
  const int64_t L = h->h_n_leaves;
  std::vector<uint8_t> lv(L);
  std::vector<uint32_t> lc(L), lk(L), ls(L);
  std::vector<int32_t> bc(L);
  MKNN_CUDA_OK(cudaStreamSynchronize(h->stream));
  MKNN_CUDA_OK(cudaMemcpy(lv.data(), h->ix.leaf_level, L, cudaMemcpyDeviceToHost));
  MKNN_CUDA_OK(cudaMemcpy(lc.data(), h->ix.leaf_code, 4 * L, cudaMemcpyDeviceToHost));
  MKNN_CUDA_OK(cudaMemcpy(lk.data(), h->ix.leaf_key, 4 * L, cudaMemcpyDeviceToHost));
  MKNN_CUDA_OK(cudaMemcpy(ls.data(), h->ix.leaf_span, 4 * L, cudaMemcpyDeviceToHost));
  MKNN_CUDA_OK(cudaMemcpy(bc.data(), h->ix.build_counts, 4 * L, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < L; i++) {
    if (leaf_level) leaf_level[i] = lv[i];
    if (leaf_code) leaf_code[i] = lc[i];
    if (leaf_key) leaf_key[i] = lk[i];
    if (leaf_span) leaf_span[i] = ls[i];
    if (build_counts) build_counts[i] = bc[i];
  }
  if (z_map)
    MKNN_CUDA_OK(cudaMemcpy(z_map, h->ix.z_map, sizeof(int32_t) * ((int64_t)1 << (2 * h->h_l_deep)),
                            cudaMemcpyDeviceToHost));
  return 0;
}

int mknn_store_export(mknn_engine* h, int64_t* cell_start, int64_t* cell_end) {
  if (!h || !h->have_index || !h->st.cell_start) return MKNN_EINVAL;
  int rc;
  if ((rc = bind(h))) return h->set_err(rc);
  const int64_t L = h->h_n_leaves;
  std::vector<int32_t> cs(L + 1);
  MKNN_CUDA_OK(cudaStreamSynchronize(h->stream));
  MKNN_CUDA_OK(cudaMemcpy(cs.data(), h->st.cell_start, 4 * (L + 1), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < L; i++) {
    if (cell_start) cell_start[i] = cs[i];
    if (cell_end) cell_end[i] = cs[i + 1];
  }
  return 0;
}

}  // extern "C"
