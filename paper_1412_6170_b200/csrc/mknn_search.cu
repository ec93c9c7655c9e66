// mknn_search.cu -- the per-tick k-NN join: own-leaf pass, alternating
// left/right leaf expansion with quadrant pruning, and canonical top-k.
//
// Reference semantics (engine.py):
//   first_iteration          engine.py:356-373 (own leaf, self excluded by id)
//   navigate                 engine.py:396-503 (virtual full-quadtree walk)
//   update_nn_lists          engine.py:376-393 (merge the assigned leaf)
//   direction loop           engine.py:645-681 (left first, then alternate)
//   _emit                    engine.py:704-723 (sqrt, row order, CSR)
//
// Mapping to B200.  The reference advances all queries one leaf per
// direction per global iteration, regrouping queries by leaf in between
// (sort_and_materialize, engine.py:506-526).  A query's state (its list and
// two cursors) is touched only by its own rows, so its step sequence
// L1 R1 L2 R2 ... (a drained direction drops out) does not depend on any
// other query.  The device therefore runs each query's whole walk inside one
// warp with no global iteration barrier, no per-iteration compaction and no
// host round-trip; the global iteration metrics are rebuilt exactly from
// per-query navigate-call counts (stats_reduce).  Queries are processed in
// leaf-grouped order so the warps of a CTA stream the same leaves through L1.
//
// Chunk pruning.  The store keeps each leaf's objects in sub-cell Morton
// order cut into 32-object chunks with point bounding boxes (mknn_index.cu).
// Every (query, leaf) row of the reference still counts the whole leaf in
// distance_evals, but the warp only computes distances for chunks whose box
// min-dist2 is <= the current k-th d2: a skipped chunk holds no object that
// could be admitted, so the list -- and every later navigation decision that
// reads its k-th d2 -- is exactly the reference's.  Chunks are visited
// nearest box first, which fills the list with close objects early.
//
// Top-k.  The running list holds N = 32*KPL keys (N >= k) distributed as
// element e = slot*32 + lane, sorted ascending by (d2, id) -- the oracle's
// canonical order (oracle.py:76-77).  Each chunk is filtered against the
// k-th key (ballot); few survivors are inserted one by one with warp
// shuffles, many are bitonic-sorted and bitonic-merged.
// Admission is (d2, id) < k-th and a quadrant is pruned only when its
// min-dist2 is strictly greater than the k-th d2, so the canonical
// lowest-id member of a boundary tie group is always found (the reference
// prunes on >=, engine.py:447; distances are identical either way).
#include <algorithm>
#include <cstdlib>

#include "mknn_internal.h"

namespace mknn {

namespace {

// k > 32: the running lists live only in shared memory (visit_leaf_sm);
// -DMKNN_SMEM_LIST=0 restores register-resident lists (A/B)
#ifndef MKNN_SMEM_LIST
#define MKNN_SMEM_LIST 1
#endif
constexpr bool SMEM_LIST = MKNN_SMEM_LIST;
// 32 < k <= 128 launch shape: warps per CTA, resident CTAs per SM
#ifndef MKNN_K128_WARPS
#define MKNN_K128_WARPS 16
#endif
#ifndef MKNN_K128_MINB
#define MKNN_K128_MINB 1
#endif
// warps of at most two queries (k > 64) navigate each query with 16 / 32
// lanes (navigate_grp) with -DMKNN_GROUP_NAV=1 (A/B: measured slower, the
// prunes mostly happen at the first level of a chain)
#ifndef MKNN_GROUP_NAV
#define MKNN_GROUP_NAV 0
#endif
constexpr bool GROUP_NAV = MKNN_GROUP_NAV;
#ifndef MKNN_K128_B
#define MKNN_K128_B 2
#endif

template <int KPL>
struct List {
  double d[KPL];
  long long id[KPL];
};

// one bitonic compare-exchange stage with partner distance j inside a
// bitonic block of `size` elements (ascending where (e & size) == 0)
template <int KPL>
__device__ __forceinline__ void bitonic_step(double (&d)[KPL], long long (&id)[KPL], int lane,
                                             int size, int j) {
  if (j >= 32) {
    const int js = j >> 5;
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      if ((s & js) == 0) {
        const int t = s | js;
        const bool asc = ((s << 5) & size) == 0;
        const bool sw = asc ? key_less(d[t], id[t], d[s], id[s]) : key_less(d[s], id[s], d[t], id[t]);
        const double ds = d[s], dt = d[t];
        const long long is = id[s], it = id[t];
        d[s] = sw ? dt : ds;
        d[t] = sw ? ds : dt;
        id[s] = sw ? it : is;
        id[t] = sw ? is : it;
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      const double pd = __shfl_xor_sync(FULL, d[s], j);
      const long long pi = __shfl_xor_sync(FULL, id[s], j);
      const int e = (s << 5) | lane;
      const bool asc = (e & size) == 0;
      const bool lower = (lane & j) == 0;
      const bool take = (lower == asc) ? key_less(pd, pi, d[s], id[s])
                                       : key_less(d[s], id[s], pd, pi);
      d[s] = take ? pd : d[s];
      id[s] = take ? pi : id[s];
    }
  }
}

template <int KPL>
__device__ __forceinline__ void bitonic_sort(double (&d)[KPL], long long (&id)[KPL], int lane) {
  constexpr int N = 32 * KPL;
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) bitonic_step<KPL>(d, id, lane, size, j);
  }
}

// L <- the N smallest of L u C (both ascending); result ascending
template <int KPL>
__device__ __forceinline__ void bitonic_merge_into(List<KPL>& L, double (&cd)[KPL],
                                                   long long (&ci)[KPL], int lane) {
  constexpr int N = 32 * KPL;
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const double rd = __shfl_xor_sync(FULL, cd[KPL - 1 - s], 31);
    const long long ri = __shfl_xor_sync(FULL, ci[KPL - 1 - s], 31);
    const bool lt2 = key_less(rd, ri, L.d[s], L.id[s]);
    L.d[s] = lt2 ? rd : L.d[s];
    L.id[s] = lt2 ? ri : L.id[s];
  }
#pragma unroll
  for (int j = N >> 1; j > 0; j >>= 1) bitonic_step<KPL>(L.d, L.id, lane, N, j);
}

// insert one key into the ascending list (the last element falls off)
template <int KPL>
__device__ __forceinline__ void list_insert(List<KPL>& L, double kd, long long ki, int lane) {
  bool gt[KPL];
  unsigned m[KPL];
  double pd[KPL];
  long long pi[KPL];
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    gt[s] = key_less(kd, ki, L.d[s], L.id[s]);
    m[s] = __ballot_sync(FULL, gt[s]);
    const double ud = __shfl_up_sync(FULL, L.d[s], 1);
    const long long ui = __shfl_up_sync(FULL, L.id[s], 1);
    if (s > 0) {
      const double wd = __shfl_sync(FULL, L.d[s - 1], 31);
      const long long wi = __shfl_sync(FULL, L.id[s - 1], 31);
      pd[s] = lane ? ud : wd;
      pi[s] = lane ? ui : wi;
    } else {
      pd[s] = ud;
      pi[s] = ui;
    }
  }
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const bool gprev = lane ? ((m[s] >> (lane - 1)) & 1u) : (s > 0 ? (m[s > 0 ? s - 1 : 0] >> 31) & 1u : 0u);
    const double nd = gprev ? pd[s] : kd;
    const long long ni = gprev ? pi[s] : ki;
    L.d[s] = gt[s] ? nd : L.d[s];
    L.id[s] = gt[s] ? ni : L.id[s];
  }
}

// ---- one-slot lists (k <= 32): sorting networks on 32-bit keys ----------
// akey(d2) = the float bits of d2 rounded down (monotone for d2 >= 0) with
// the low `bits` bits replaced by a source index.  The networks below move
// only these keys (one shuffle and one IMNMX per step instead of shuffling
// and comparing fp64 + int64 pairs), then gather the exact (d2, id) by
// source index.  trunc(akey(a)) < trunc(akey(b)) implies d2(a) < d2(b), so
// the result is exactly in canonical (d2, id) order unless two neighbours
// share a truncated key (a relative gap below 2^-17, or an exact tie such as
// coincident objects); that case -- and, for a merge, equal truncated keys
// across the cut between the kept and the dropped halves -- is detected and
// redone with the exact (d2, id) network.
constexpr uint32_t AKEY_INF = 0x7F800000u;

__device__ __forceinline__ uint32_t akey(double d2, int bits, uint32_t src) {
  return (__float_as_uint(__double2float_rd(d2)) & ~((1u << bits) - 1u)) | src;
}

// any two neighbours (lane, lane + 1) with equal truncated keys, other than
// the +inf sentinels (which are all identical (inf, IDMAX) entries)?
__device__ __forceinline__ bool akey_ties(uint32_t key, int bits, int lane) {
  const uint32_t nk = __shfl_down_sync(FULL, key, 1);
  const bool tie = lane < 31 && ((key ^ nk) >> bits) == 0 && (key >> bits) != (AKEY_INF >> bits);
  return __any_sync(FULL, tie);
}

// sort one batch of 32 candidates (one per lane) ascending by (d2, id)
__device__ __forceinline__ void batch_sort(double& d, long long& id, int lane) {
  uint32_t key = akey(d, 5, (uint32_t)lane);
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      const uint32_t p = __shfl_xor_sync(FULL, key, j);
      const bool take_min = ((lane & j) == 0) == ((lane & size) == 0);
      key = take_min ? min(key, p) : max(key, p);
    }
  }
  if (akey_ties(key, 5, lane)) {
    double a[1] = {d};
    long long b[1] = {id};
    bitonic_sort<1>(a, b, lane);
    d = a[0];
    id = b[0];
    return;
  }
  const int src = (int)(key & 31u);
  const double nd = __shfl_sync(FULL, d, src);
  const long long ni = __shfl_sync(FULL, id, src);
  d = nd;
  id = ni;
}

// L <- the 32 smallest of L u C, both ascending (one slot per lane)
__device__ __forceinline__ void merge_list(List<1>& L, double cd, long long ci, int lane) {
  const uint32_t kl = akey(L.d[0], 6, (uint32_t)lane);
  const uint32_t kc = akey(cd, 6, 32u | (uint32_t)lane);
  // min(A_i, B_{31-i}) holds the 32 smallest as a bitonic sequence, max()
  // the 32 dropped ones
  const uint32_t rc = __shfl_sync(FULL, kc, 31 - lane);
  uint32_t m = min(kl, rc);
  // the largest kept and the smallest dropped key must differ in their
  // truncated part, or the cut between them is not exact
  const uint32_t kept_max = __reduce_max_sync(FULL, m);
  const uint32_t drop_min = __reduce_min_sync(FULL, max(kl, rc));
  const bool cut_tie = ((kept_max ^ drop_min) >> 6) == 0 && (kept_max >> 6) < (AKEY_INF >> 6);
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    const uint32_t p = __shfl_xor_sync(FULL, m, j);
    m = (lane & j) ? max(m, p) : min(m, p);
  }
  if (cut_tie || akey_ties(m, 6, lane)) {
    double c[1] = {cd};
    long long i[1] = {ci};
    bitonic_merge_into<1>(L, c, i, lane);
    return;
  }
  const int src = (int)(m & 31u);
  const double dl = __shfl_sync(FULL, L.d[0], src), dc = __shfl_sync(FULL, cd, src);
  const long long il = __shfl_sync(FULL, L.id[0], src), ic = __shfl_sync(FULL, ci, src);
  const bool from_c = (m & 32u) != 0;
  L.d[0] = from_c ? dc : dl;
  L.id[0] = from_c ? ic : il;
}

// key of element k-1 (the current k-th neighbour; sentinel while not full)
template <int KPL>
__device__ __forceinline__ void list_kth(const List<KPL>& L, int k, double& kd, long long& ki) {
  const int ks = (k - 1) >> 5, kl = (k - 1) & 31;
  kd = DINF;
  ki = IDMAX;
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    if (s == ks) {
      kd = __shfl_sync(FULL, L.d[s], kl);
      ki = __shfl_sync(FULL, L.id[s], kl);
    }
  }
}

// Profiling counters (MKNN_PROF=1; nullptr otherwise): what the warps did.
enum {
  PROF_OWN_CHUNKS_SCANNED, PROF_EXP_CHUNKS_SCANNED, PROF_INSERTS, PROF_SORT_MERGES,
  PROF_EXP_LEAF_VISITS, PROF_OWN_CHUNKS_TOTAL, PROF_EXP_CHUNKS_TOTAL, PROF_ADMITTED,
  PROF_EXP_VISITS_NO_SCAN, PROF_EXP_VISITS_ADMITTING, PROF_ROUNDS, PROF_ROUND_LANES,
  PROF_NAV_STEPS, PROF_NAV_MAXSTEPS, PROF_N
};
#ifndef MKNN_PROFILE
#define MKNN_PROFILE 0
#endif
__device__ __forceinline__ void prof_add(unsigned long long* prof, int i, unsigned long long v,
                                         int lane) {
  if (MKNN_PROFILE && prof && lane == 0 && v) atomicAdd(&prof[i], v);
}

// %globaltimer (ns) and the phase split of a query batch: first_iteration
// (own leaf) and the whole walk, added by one lane (SearchArgs::phase_ns)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void phase_add(unsigned long long* ph, unsigned long long t0,
                                          unsigned long long t1, unsigned long long t2) {
  if (ph) {
    atomicAdd(&ph[0], t1 - t0);
    atomicAdd(&ph[1], t2 - t0);
  }
}

// Admit the candidates of one lane-per-candidate batch into the list.
// cand (cd, ci) is (+inf, IDMAX) on lanes that do not pass; m = ballot of
// passing lanes.  Few survivors are inserted one by one with warp shuffles;
// many are sorted and merged (an empty list takes the sorted batch).
template <int KPL>
__device__ __forceinline__ void admit(List<KPL>& L, double cd0, long long ci0, unsigned m, int lane,
                                      unsigned long long* prof) {
  constexpr int INS_MAX = KPL == 1 ? 4 : 10 + 4 * KPL;
  const int cnt = __popc(m);
  prof_add(prof, PROF_ADMITTED, cnt, lane);
  prof_add(prof, cnt <= INS_MAX ? PROF_INSERTS : PROF_SORT_MERGES, cnt <= INS_MAX ? cnt : 1, lane);
  if (cnt <= INS_MAX) {
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      list_insert<KPL>(L, __shfl_sync(FULL, cd0, src), __shfl_sync(FULL, ci0, src), lane);
    }
    return;
  }
  const bool empty = __shfl_sync(FULL, L.d[0], 0) == DINF;
  if constexpr (KPL == 1) {
    batch_sort(cd0, ci0, lane);
    if (empty) {  // the sorted batch is the list
      L.d[0] = cd0;
      L.id[0] = ci0;
    } else {
      merge_list(L, cd0, ci0, lane);
    }
  } else {
    double bd[1] = {cd0};
    long long bi[1] = {ci0};
    bitonic_sort<1>(bd, bi, lane);
    double cd[KPL];
    long long ci[KPL];
    cd[0] = bd[0];
    ci[0] = bi[0];
#pragma unroll
    for (int s = 1; s < KPL; s++) {
      cd[s] = DINF;
      ci[s] = IDMAX;
    }
    if (empty) {
#pragma unroll
      for (int s = 0; s < KPL; s++) {
        L.d[s] = cd[s];
        L.id[s] = ci[s];
      }
    } else {
      bitonic_merge_into<KPL>(L, cd, ci, lane);
    }
  }
}

// engine.py:279-324 _merge_pack for one row restricted to one chunk of a
// leaf (one record per lane, already loaded): every object except the issuer
// (by id, engine.py:298-300) competes for the list; admission is
// (d2, id) < k-th.  Returns whether the list changed.
template <int KPL>
__device__ __forceinline__ bool scan_rec(List<KPL>& L, double kd, long long ki, bool valid,
                                         const StoreRec& r, double qx, double qy, long long me,
                                         int lane, unsigned long long* prof) {
  const double d2 = valid ? pair_d2(qx, qy, r.x, r.y) : DINF;
  const bool pass = valid && d2 <= kd && r.id != me && key_less(d2, r.id, kd, ki);
  const unsigned m = __ballot_sync(FULL, pass);
  if (m) admit<KPL>(L, pass ? d2 : DINF, pass ? r.id : IDMAX, m, lane, prof);
  return m != 0;
}

__device__ __forceinline__ StoreRec load_rec(const StoreRec* __restrict__ obj, int i, bool valid) {
  StoreRec r;
  if (valid) r = ld_rec(&obj[i]);
  return r;
}

// min-dist2 from the query to a chunk's point bounding box: a lower bound of
// pair_d2 for every object of the chunk (each step is a correctly rounded,
// monotone operation of the same inputs pair_d2 rounds; geometry.py:189-193)
__device__ __forceinline__ double mindist2_box(const ChunkBox& b, double qx, double qy) {
  const double dx = dmax(dmax(__dsub_rn(b.x_lo, qx), __dsub_rn(qx, b.x_hi)), 0.0);
  const double dy = dmax(dmax(__dsub_rn(b.y_lo, qy), __dsub_rn(qy, b.y_hi)), 0.0);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// Pick the 32 / CH nearest candidate boxes of a 32-chunk group (key:
// approximate distance | lane, ~0 when not a candidate) and map lane groups
// of CH lanes onto them: this lane's record index cb, valid flag v.
template <int CH>
__device__ __forceinline__ void pick_chunks(unsigned key, bool& live, int lane, int ob, int oe,
                                            int g_rel, int& cb, bool& v) {
  int mine = -1;
#pragma unroll
  for (int p = 0; p < 32 / CH; p++) {
    const unsigned kmin = __reduce_min_sync(FULL, key);
    const int src = kmin == 0xffffffffu ? -1 : (int)(kmin & 31u);
    if (lane == src) {
      live = false;
      key = 0xffffffffu;
    }
    if (lane / CH == p) mine = src;
  }
  const int off = lane % CH;
  cb = ob + (g_rel + mine) * CH + off;
  v = mine >= 0 && cb < min(ob + (g_rel + mine + 1) * CH, oe);
}

// One row of the reference's distance phase (first_iteration's own leaf,
// engine.py:356-373, or update_nn_lists' assigned leaf, 376-393): every
// object of the leaf competes for the list.  Chunks whose box min-dist2
// exceeds the current k-th d2 cannot hold an admissible object (admission
// needs d2 <= k-th) and are skipped without changing the result; the others
// are visited nearest box first, so the list tightens early.
template <int KPL>
__device__ __forceinline__ void visit_leaf(List<KPL>& L, int k, int leaf, double qx, double qy,
                                           long long me, const SearchArgs& a, int lane, bool own,
                                           double cap = DINF) {
  const int ob = __ldg(&a.cell_start[leaf]), oe = __ldg(&a.cell_start[leaf + 1]);
  const int c0 = __ldg(&a.chunk_start[leaf]), c1 = c0 + (oe - ob + chunk_for_k(32 * KPL) - 1) / chunk_for_k(32 * KPL);
  prof_add(a.prof, own ? PROF_OWN_CHUNKS_TOTAL : PROF_EXP_CHUNKS_TOTAL, c1 - c0, lane);
  if (!own) prof_add(a.prof, PROF_EXP_LEAF_VISITS, 1, lane);
  bool scanned = false, admitted = false;  // profiling only
  (void)scanned;
  (void)admitted;
  // cap: an upper bound of the k-th d2 of this leaf's objects (see
  // k_search); the effective admission key is the smaller of (k-th d2, k-th
  // id) and (cap, IDMAX), so every admitted candidate also has d2 <= cap
  double kd;
  long long ki;
  list_kth<KPL>(L, k, kd, ki);
  if (cap < kd) {
    kd = cap;
    ki = IDMAX;
  }
  for (int g = c0; g < c1; g += 32) {
    bool live = g + lane < c1;
    double md = DINF;
    if (live) md = mindist2_box(a.box[g + lane], qx, qy);
    for (;;) {
      const bool cand = live && md <= kd;
      if (!__any_sync(FULL, cand)) break;
      // nearest box first (approximate key: md rounded down to float, lane
      // in the low bits); the visit order only affects speed
      const unsigned key =
          cand ? ((__float_as_uint(__double2float_rd(md)) & ~31u) | (unsigned)lane) : 0xffffffffu;
      int cb;
      bool v;
      pick_chunks<chunk_for_k(32 * KPL)>(key, live, lane, ob, oe, g - c0, cb, v);
      const StoreRec r = load_rec(a.obj, cb, v);
      prof_add(a.prof, own ? PROF_OWN_CHUNKS_SCANNED : PROF_EXP_CHUNKS_SCANNED, 1, lane);
      scanned = true;
      if (scan_rec<KPL>(L, kd, ki, v, r, qx, qy, me, lane, a.prof)) {
        list_kth<KPL>(L, k, kd, ki);
        if (cap < kd) {
          kd = cap;
          ki = IDMAX;
        }
        admitted = true;
      }
    }
  }
  if (!own) {
    prof_add(a.prof, PROF_EXP_VISITS_NO_SCAN, !scanned, lane);
    prof_add(a.prof, PROF_EXP_VISITS_ADMITTING, admitted, lane);
  }
}

// ---- multi-slot lists (k > 32): buffered admission ----------------------
// With N = 32*KPL slots, admitting a chunk at a time would re-merge N keys
// per chunk.  Candidates that beat the (possibly stale) k-th key are instead
// appended to a per-warp shared-memory buffer (ballot compaction) and merged
// N - 32 at a time: one sort of the buffer and one merge into the list, both
// on 64-bit keys (akey64, source index in the low bits) with the exact values
// gathered from shared memory afterwards; exact (d2, id) networks only when
// two neighbours share a truncated key.  A stale k-th key only lets extra
// candidates into the buffer: the merge keeps the N smallest, so the list
// is exact.
template <int KPL, typename KT, int S = KPL>  // S: only slots [0, S) take part
__device__ __forceinline__ void step_key(KT (&kk)[KPL], int lane, int size, int j) {
  if (j >= 32) {
    const int js = j >> 5;
#pragma unroll
    for (int s = 0; s < S; s++) {
      if ((s & js) == 0) {
        const int t = s | js;
        const bool asc = ((s << 5) & size) == 0;
        const KT lo = min(kk[s], kk[t]), hi = max(kk[s], kk[t]);
        kk[s] = asc ? lo : hi;
        kk[t] = asc ? hi : lo;
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < S; s++) {
      const KT p = __shfl_xor_sync(FULL, kk[s], j);
      const int e = (s << 5) | lane;
      const bool take_min = ((lane & j) == 0) == ((e & size) == 0);
      kk[s] = take_min ? min(kk[s], p) : max(kk[s], p);
    }
  }
}

// 64-bit sort key of d2 >= 0: the double's bits (monotone) with the low
// `bits` bits replaced by a source index; only d2 values within 2^-44
// relative of each other (or exact ties) share a truncated key
constexpr unsigned long long AKEY64_INF = 0x7FF0000000000000ull;

__device__ __forceinline__ unsigned long long akey64(double d2, int bits, unsigned src) {
  return ((unsigned long long)__double_as_longlong(d2) & ~((1ull << bits) - 1ull)) | src;
}

// neighbours (element e, e + 1) of a KPL-slot key sequence with equal
// truncated keys (other than sentinels)?
template <int KPL>
__device__ __forceinline__ bool akey64_ties(const unsigned long long (&kk)[KPL], int bits, int lane) {
  bool tie = false;
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const unsigned long long dn = __shfl_down_sync(FULL, kk[s], 1);
    const unsigned long long nx =
        (s + 1 < KPL) ? __shfl_sync(FULL, kk[s + 1 < KPL ? s + 1 : s], 0) : ~0ull;
    const unsigned long long nk = lane < 31 ? dn : nx;
    tie |= ((kk[s] ^ nk) >> bits) == 0 && (kk[s] >> bits) < (AKEY64_INF >> bits) &&
           !(s + 1 == KPL && lane == 31);
  }
  return __any_sync(FULL, tie);
}

// bitonic sort of the first S slots (32 * S keys) of kk
template <int KPL, int S, typename KT>
__device__ __forceinline__ void sort_prefix(KT (&kk)[KPL], int lane) {
#pragma unroll
  for (int size = 2; size <= 32 * S; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) step_key<KPL, KT, S>(kk, lane, size, j);
  }
}

// a partial flush (nbuf <= 32, one slot) sorts one slot; otherwise all
// (intermediate widths measured slower: code size)
template <int KPL, typename KT>
__device__ __forceinline__ void sort_used_slots(KT (&kk)[KPL], int nbuf, int lane) {
  if (KPL > 1 && KPL <= 4 && nbuf <= 32)
    sort_prefix<KPL, 1>(kk, lane);
  else
    sort_prefix<KPL, KPL>(kk, lane);
}

// neighbours (element e, e + 1) of a KPL-slot 32-bit key sequence with
// equal truncated keys (other than +inf sentinels)?
template <int KPL>
__device__ __forceinline__ bool akey32_ties(const uint32_t (&kk)[KPL], int bits, int lane) {
  bool tie = false;
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const uint32_t dn = __shfl_down_sync(FULL, kk[s], 1);
    const uint32_t nx = (s + 1 < KPL) ? __shfl_sync(FULL, kk[s + 1 < KPL ? s + 1 : s], 0) : ~0u;
    const uint32_t nk = lane < 31 ? dn : nx;
    tie |= ((kk[s] ^ nk) >> bits) == 0 && (kk[s] >> bits) < (AKEY_INF >> bits) &&
           !(s + 1 == KPL && lane == 31);
  }
  return __any_sync(FULL, tie);
}

// exact (d2, id) fallback of merge_buffer (equal truncated keys)
template <int KPL>
__device__ __noinline__ List<KPL> merge_buffer_exact(List<KPL> L, const double* bufd,
                                                     const long long* bufi, int nbuf, int lane) {
  double cd[KPL];
  long long ci[KPL];
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const int e = (s << 5) | lane;
    cd[s] = e < nbuf ? bufd[e] : DINF;
    ci[s] = e < nbuf ? bufi[e] : IDMAX;
  }
  bitonic_sort<KPL>(cd, ci, lane);
  bitonic_merge_into<KPL>(L, cd, ci, lane);
  __syncwarp();
  return L;
}

// Odd-even transposition on the exact (d2, id) order until sorted.  The
// input is already sorted by truncated key, so only runs of equal truncated
// keys can be out of order; each round fixes pairs inside them (typically
// one or two rounds).
template <int KPL>
__device__ __forceinline__ void repair_runs(List<KPL>& L, int lane) {
  for (;;) {
    bool sw = false;
    // pairs (2i, 2i + 1): lanes (even, odd) of every slot
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      const double pd = __shfl_xor_sync(FULL, L.d[s], 1);
      const long long pi = __shfl_xor_sync(FULL, L.id[s], 1);
      const bool bad = (lane & 1) ? key_less(L.d[s], L.id[s], pd, pi) : key_less(pd, pi, L.d[s], L.id[s]);
      L.d[s] = bad ? pd : L.d[s];
      L.id[s] = bad ? pi : L.id[s];
      sw |= bad;
    }
    // pairs (2i + 1, 2i + 2): lanes (odd, even) inside a slot, and lane 31
    // of slot s with lane 0 of slot s + 1
    double nd[KPL];
    long long ni[KPL];
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      const double dn = __shfl_down_sync(FULL, L.d[s], 1), up = __shfl_up_sync(FULL, L.d[s], 1);
      const long long idn = __shfl_down_sync(FULL, L.id[s], 1), iup = __shfl_up_sync(FULL, L.id[s], 1);
      const double nx = __shfl_sync(FULL, L.d[s + 1 < KPL ? s + 1 : s], 0);
      const long long inx = __shfl_sync(FULL, L.id[s + 1 < KPL ? s + 1 : s], 0);
      const double pv = __shfl_sync(FULL, L.d[s > 0 ? s - 1 : 0], 31);
      const long long ipv = __shfl_sync(FULL, L.id[s > 0 ? s - 1 : 0], 31);
      nd[s] = L.d[s];
      ni[s] = L.id[s];
      if (lane & 1) {  // left element of its pair: partner is the next element
        const bool has = lane < 31 || s + 1 < KPL;
        const double od = lane < 31 ? dn : nx;
        const long long oi = lane < 31 ? idn : inx;
        if (has && key_less(od, oi, L.d[s], L.id[s])) {
          nd[s] = od;
          ni[s] = oi;
          sw = true;
        }
      } else {  // right element: partner is the previous element
        const bool has = lane > 0 || s > 0;
        const double od = lane > 0 ? up : pv;
        const long long oi = lane > 0 ? iup : ipv;
        if (has && key_less(L.d[s], L.id[s], od, oi)) {
          nd[s] = od;
          ni[s] = oi;
        }
      }
    }
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      L.d[s] = nd[s];
      L.id[s] = ni[s];
    }
    if (!__any_sync(FULL, sw)) return;
  }
}

// L <- the N smallest of L u buffer[0, nbuf); L ascending.  The networks
// move 32-bit keys (akey: d2 as float rounded down, source index in the low
// SB bits); runs of equal truncated keys are put in exact (d2, id) order
// afterwards (repair_runs), and equal truncated keys across the cut between
// the kept and the dropped halves send the merge to the exact networks.  rowd/rowi: the list's
// shared-memory home (overwritten), bufd/bufi: the buffer.
template <int KPL>
__device__ __forceinline__ void merge_buffer32(List<KPL>& L, const double* bufd,
                                               const long long* bufi, int nbuf, double* rowd,
                                               long long* rowi, int lane) {
  constexpr int N = 32 * KPL;
  constexpr int SB = KPL <= 2 ? 7 : (KPL <= 4 ? 8 : (KPL <= 8 ? 9 : 10));  // bits for 2N sources
  uint32_t kb[KPL], m[KPL];
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const int e = (s << 5) | lane;
    kb[s] = e < nbuf ? akey(bufd[e], SB, (uint32_t)(N + e)) : (~0u << SB) | (uint32_t)(N + e);
    rowd[e] = L.d[s];
    rowi[e] = L.id[s];
  }
  sort_used_slots<KPL>(kb, nbuf, lane);
  uint32_t kept_max = 0, drop_min = ~0u;
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const uint32_t kl = akey(L.d[s], SB, (uint32_t)((s << 5) | lane));
    const uint32_t rb = __shfl_sync(FULL, kb[KPL - 1 - s], 31 - lane);
    m[s] = min(kl, rb);
    kept_max = max(kept_max, m[s]);
    drop_min = min(drop_min, max(kl, rb));
  }
  kept_max = __reduce_max_sync(FULL, kept_max);
  drop_min = __reduce_min_sync(FULL, drop_min);
  const bool cut_tie = ((kept_max ^ drop_min) >> SB) == 0 && (kept_max >> SB) < (AKEY_INF >> SB);
#pragma unroll
  for (int j = N >> 1; j > 0; j >>= 1) step_key<KPL>(m, lane, N, j);
  __syncwarp();
  if (cut_tie) {
    L = merge_buffer_exact<KPL>(L, bufd, bufi, nbuf, lane);
    return;
  }
  // k <= 64 (16 key bits): truncated ties are rare, the exact networks
  // take them; k <= 128 (15 bits over twice the keys): ~2 near-ties per
  // merge, repaired in place
  const bool ties = akey32_ties<KPL>(m, SB, lane);
  if (KPL < 4 && ties) {
    L = merge_buffer_exact<KPL>(L, bufd, bufi, nbuf, lane);
    return;
  }
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const int src = (int)(m[s] & ((1u << SB) - 1u));
    const bool from_list = src < N, pad = src - N >= nbuf;  // pad: an unused buffer slot
    L.d[s] = from_list ? rowd[src] : (pad ? DINF : bufd[src - N]);
    L.id[s] = from_list ? rowi[src] : (pad ? IDMAX : bufi[src - N]);
  }
  __syncwarp();
  if (KPL >= 4 && ties) repair_runs<KPL>(L, lane);
}

// L <- the N smallest of L u buffer[0, nbuf); L ascending.  rowd/rowi: the
// list's shared-memory home (overwritten), bufd/bufi: the buffer.
template <int KPL>
__device__ __noinline__ List<KPL> merge_buffer(List<KPL> L, const double* bufd, const long long* bufi,
                                               int nbuf, double* rowd, long long* rowi, int lane) {
  constexpr int N = 32 * KPL;
  constexpr int SB = KPL <= 2 ? 7 : (KPL <= 4 ? 8 : (KPL <= 8 ? 9 : 10));  // bits for 2N sources
  unsigned long long kb[KPL], m[KPL];
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const int e = (s << 5) | lane;
    kb[s] = e < nbuf ? akey64(bufd[e], SB, (unsigned)(N + e)) : (~0ull << SB) | (unsigned)(N + e);
    rowd[e] = L.d[s];
    rowi[e] = L.id[s];
  }
  // sort only the slots that hold candidates: the rest are sentinels that
  // already sit in ascending order above every real key
  sort_used_slots<KPL>(kb, nbuf, lane);
  // min(A_e, B_{N-1-e}): the N smallest as a bitonic sequence; the largest
  // kept and the smallest dropped key must differ in their truncated part
  unsigned long long kept_max = 0, drop_min = ~0ull;
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const unsigned long long kl = akey64(L.d[s], SB, (unsigned)((s << 5) | lane));
    const unsigned long long rb = __shfl_sync(FULL, kb[KPL - 1 - s], 31 - lane);
    m[s] = min(kl, rb);
    kept_max = max(kept_max, m[s]);
    drop_min = min(drop_min, max(kl, rb));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kept_max = max(kept_max, __shfl_xor_sync(FULL, kept_max, o));
    drop_min = min(drop_min, __shfl_xor_sync(FULL, drop_min, o));
  }
  const bool cut_tie =
      ((kept_max ^ drop_min) >> SB) == 0 && (kept_max >> SB) < (AKEY64_INF >> SB);
#pragma unroll
  for (int j = N >> 1; j > 0; j >>= 1) step_key<KPL>(m, lane, N, j);
  __syncwarp();
  if (cut_tie || akey64_ties<KPL>(m, SB, lane)) {  // exact (d2, id) networks
    double cd[KPL];
    long long ci[KPL];
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      const int e = (s << 5) | lane;
      cd[s] = e < nbuf ? bufd[e] : DINF;
      ci[s] = e < nbuf ? bufi[e] : IDMAX;
    }
    bitonic_sort<KPL>(cd, ci, lane);
    bitonic_merge_into<KPL>(L, cd, ci, lane);
    __syncwarp();
    return L;
  }
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const int src = (int)(m[s] & ((1ull << SB) - 1ull));
    const bool from_list = src < N, pad = src - N >= nbuf;  // pad: an unused buffer slot
    L.d[s] = from_list ? rowd[src] : (pad ? DINF : bufd[src - N]);
    L.id[s] = from_list ? rowi[src] : (pad ? IDMAX : bufi[src - N]);
  }
  __syncwarp();
  return L;
}

// KPL <= 4 (k <= 128): 32-bit keys (>= 15 mantissa bits); wider lists merge
// 64-bit keys (with 14 bits or fewer, truncated ties at the cut become
// frequent enough to lose: k = 256 measured 56 -> 63 ms)
template <int KPL>
__device__ __forceinline__ void merge_buffer_k(List<KPL>& L, const double* bufd,
                                               const long long* bufi, int nbuf, double* rowd,
                                               long long* rowi, int lane) {
  if constexpr (KPL <= 4)
    merge_buffer32<KPL>(L, bufd, bufi, nbuf, rowd, rowi, lane);
  else
    L = merge_buffer<KPL>(L, bufd, bufi, nbuf, rowd, rowi, lane);
}

// ---- k > 32 with the list resident in shared memory ----------------------
// The list's home (ld/li, N entries, element e at [e]) is the only copy: a
// leaf visit holds just the k-th key in registers while it scans, and a
// merge reads the list keys from the home, gathers the merged entries into
// registers and writes them back.  The scan loop and the navigation then
// carry no list registers (2 * KPL fp64/int64 pairs), which is what bounds
// the resident warps of the k > 32 kernel.
template <int KPL>
__device__ __forceinline__ void list_load_sm(List<KPL>& L, const double* ld, const long long* li,
                                             int lane) {
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    L.d[s] = ld[s * 32 + lane];
    L.id[s] = li[s * 32 + lane];
  }
}
template <int KPL>
__device__ __forceinline__ void list_store_sm(const List<KPL>& L, double* ld, long long* li, int lane) {
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    ld[s * 32 + lane] = L.d[s];
    li[s * 32 + lane] = L.id[s];
  }
}

template <int KPL>
__device__ __forceinline__ void kth_sm(const double* ld, const long long* li, int k, double& kd,
                                       long long& ki) {
  kd = ld[k - 1];
  ki = li[k - 1];
}

// a short buffer (nbuf <= RANK_MERGE_MAX) merged by ranks instead of
// networks: candidate c goes to (# list entries < c) + (# candidates < c),
// list entry e to e + (# candidates below it); exact (d2, id) compares,
// keys are distinct (a candidate is never already listed), entries pushed
// past N fall off.  k > 64 (lists of >= 4 slots): every partial flush
// (nbuf <= 32, one candidate per lane) takes it -- k = 128 / 256: 11.85 ->
// 11.21 / 53.97 -> 49.35 ms; at k <= 64 and with smaller thresholds it
// measured neutral or slower (repo:profiles/r2_ab_rank_merge.txt).
// -DMKNN_RANK_MERGE=T: threshold T <= 32 (A/B; 0 = off).
// k > 32: the own-leaf cap from the previous query's list (k_search's
// triangle-inequality bound) with -DMKNN_KCAP=1 (A/B: measured slower, the
// buffered admission takes the first chunks whole either way)
#ifndef MKNN_KCAP
#define MKNN_KCAP 0
#endif
constexpr bool KCAP = MKNN_KCAP;

// k > 32: a merge into the empty list takes the sorted buffer as the list
// (no merge network) with -DMKNN_EMPTY_SHORTCUT=1 (A/B: measured 3-5 % slower)
#ifndef MKNN_EMPTY_SHORTCUT
#define MKNN_EMPTY_SHORTCUT 0
#endif
constexpr bool EMPTY_SHORTCUT = MKNN_EMPTY_SHORTCUT;

// k > 32: when the buffer is merged.  k <= 128 (KPL <= 4): once it holds
// more than N - 32 candidates (one network merge per N - 32); k > 128: after
// every admitting step (always <= 32 candidates, so always the rank merge:
// the 8- and 16-slot 64-bit networks cost more than the extra merges, k =
// 256: 49.3 -> 31.8 ms; at k = 128 the same measured 11.2 -> 16.4 ms).
// -DMKNN_FLUSH_AT=t: merge at more than t candidates for every k (A/B)
#ifndef MKNN_FLUSH_AT
#define MKNN_FLUSH_AT -1
#endif
template <int KPL>
__host__ __device__ constexpr int flush_at() {
  return MKNN_FLUSH_AT >= 0 ? MKNN_FLUSH_AT : (KPL >= 8 ? 0 : 32 * KPL - 32);
}

#ifndef MKNN_RANK_MERGE
#define MKNN_RANK_MERGE 32
#endif
constexpr int RANK_MERGE_MAX = MKNN_RANK_MERGE;

template <int KPL>
__device__ __forceinline__ void merge_rank_sm(double* ld, long long* li, const double* bufd,
                                              const long long* bufi, int nbuf, int lane) {
  constexpr int N = 32 * KPL;
  const bool has = lane < nbuf;
  const double cd = has ? bufd[lane] : DINF;
  const long long ci = has ? bufi[lane] : IDMAX;
  int rl = 0;  // list entries below the candidate (power-of-two lower bound)
#pragma unroll
  for (int step = N / 2; step > 0; step >>= 1)
    if (key_less(ld[rl + step], li[rl + step], cd, ci)) rl += step;
  if (key_less(ld[rl], li[rl], cd, ci)) rl++;
  int rc = 0, sh[KPL];
#pragma unroll
  for (int s = 0; s < KPL; s++) sh[s] = 0;
  for (int j = 0; j < nbuf; j++) {
    const double dj = __shfl_sync(FULL, cd, j);
    const long long ij = __shfl_sync(FULL, ci, j);
    const int rj = __shfl_sync(FULL, rl, j);
    rc += key_less(dj, ij, cd, ci) ? 1 : 0;
#pragma unroll
    for (int s = 0; s < KPL; s++) sh[s] += rj <= ((s << 5) | lane) ? 1 : 0;
  }
  double od[KPL];
  long long oi[KPL];
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    od[s] = ld[(s << 5) | lane];
    oi[s] = li[(s << 5) | lane];
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    const int np = ((s << 5) | lane) + sh[s];
    if (np < N) {
      ld[np] = od[s];
      li[np] = oi[s];
    }
  }
  if (has && rl + rc < N) {
    ld[rl + rc] = cd;
    li[rl + rc] = ci;
  }
  __syncwarp();
}

template <int KPL>
__device__ __forceinline__ void merge_sm(double* ld, long long* li, const double* bufd,
                                         const long long* bufi, int nbuf, int lane) {
  constexpr int N = 32 * KPL;
  static_assert(RANK_MERGE_MAX <= 32, "one buffered candidate per lane");
  if (KPL >= 4 && RANK_MERGE_MAX > 0 && nbuf <= RANK_MERGE_MAX) {
    merge_rank_sm<KPL>(ld, li, bufd, bufi, nbuf, lane);
    return;
  }
  if constexpr (KPL > 4) {  // 64-bit key networks (merge_buffer re-homes the list itself)
    List<KPL> L;
    list_load_sm<KPL>(L, ld, li, lane);
    L = merge_buffer<KPL>(L, bufd, bufi, nbuf, ld, li, lane);
    list_store_sm<KPL>(L, ld, li, lane);
    __syncwarp();
    return;
  } else {
    constexpr int SB = KPL <= 2 ? 7 : 8;  // bits for 2N sources
    uint32_t kb[KPL], m[KPL];
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      const int e = (s << 5) | lane;
      kb[s] = e < nbuf ? akey(bufd[e], SB, (uint32_t)(N + e)) : (~0u << SB) | (uint32_t)(N + e);
    }
    sort_used_slots<KPL>(kb, nbuf, lane);
    if (EMPTY_SHORTCUT && ld[0] == DINF) {  // empty list: the sorted buffer is the list
      const bool ties = akey32_ties<KPL>(kb, SB, lane);
      List<KPL> L;
      if (ties && KPL < 4) {
        list_load_sm<KPL>(L, ld, li, lane);
        L = merge_buffer_exact<KPL>(L, bufd, bufi, nbuf, lane);
      } else {
#pragma unroll
        for (int s = 0; s < KPL; s++) {
          const int src = (int)(kb[s] & ((1u << SB) - 1u)) - N;
          const bool pad = src >= nbuf;
          L.d[s] = pad ? DINF : bufd[src];
          L.id[s] = pad ? IDMAX : bufi[src];
        }
        if (ties) repair_runs<KPL>(L, lane);
      }
      __syncwarp();
      list_store_sm<KPL>(L, ld, li, lane);
      __syncwarp();
      return;
    }
    uint32_t kept_max = 0, drop_min = ~0u;
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      const int e = (s << 5) | lane;
      const uint32_t kl = akey(ld[e], SB, (uint32_t)e);
      const uint32_t rb = __shfl_sync(FULL, kb[KPL - 1 - s], 31 - lane);
      m[s] = min(kl, rb);
      kept_max = max(kept_max, m[s]);
      drop_min = min(drop_min, max(kl, rb));
    }
    kept_max = __reduce_max_sync(FULL, kept_max);
    drop_min = __reduce_min_sync(FULL, drop_min);
    const bool cut_tie = ((kept_max ^ drop_min) >> SB) == 0 && (kept_max >> SB) < (AKEY_INF >> SB);
#pragma unroll
    for (int j = N >> 1; j > 0; j >>= 1) step_key<KPL>(m, lane, N, j);
    const bool ties = akey32_ties<KPL>(m, SB, lane);
    List<KPL> L;
    if (cut_tie || (KPL < 4 && ties)) {  // exact (d2, id) networks
      list_load_sm<KPL>(L, ld, li, lane);
      L = merge_buffer_exact<KPL>(L, bufd, bufi, nbuf, lane);
    } else {
#pragma unroll
      for (int s = 0; s < KPL; s++) {
        const int src = (int)(m[s] & ((1u << SB) - 1u));
        const bool from_list = src < N, pad = src - N >= nbuf;  // pad: an unused buffer slot
        L.d[s] = from_list ? ld[src] : (pad ? DINF : bufd[src - N]);
        L.id[s] = from_list ? li[src] : (pad ? IDMAX : bufi[src - N]);
      }
      if (KPL >= 4 && ties) repair_runs<KPL>(L, lane);
    }
    __syncwarp();
    list_store_sm<KPL>(L, ld, li, lane);
    __syncwarp();
  }
}

template <int KPL>
__device__ __forceinline__ void visit_leaf_sm(int k, int leaf, double qx, double qy, long long me,
                                              const SearchArgs& a, int lane, double* bufd,
                                              long long* bufi, double* ld, long long* li, bool own,
                                              double cap = DINF) {
  constexpr int N = 32 * KPL;
  const int ob = __ldg(&a.cell_start[leaf]), oe = __ldg(&a.cell_start[leaf + 1]);
  const int c0 = __ldg(&a.chunk_start[leaf]), c1 = c0 + (oe - ob + chunk_for_k(32 * KPL) - 1) / chunk_for_k(32 * KPL);
  const unsigned lt = (1u << lane) - 1u;
  prof_add(a.prof, own ? PROF_OWN_CHUNKS_TOTAL : PROF_EXP_CHUNKS_TOTAL, c1 - c0, lane);
  if (!own) prof_add(a.prof, PROF_EXP_LEAF_VISITS, 1, lane);
  double kd;
  long long ki;
  kth_sm<KPL>(ld, li, k, kd, ki);
  if (cap < kd) {  // an upper bound of the own-leaf k-th (see k_search)
    kd = cap;
    ki = IDMAX;
  }
  int nbuf = 0;
  for (int g = c0; g < c1; g += 32) {
    bool live = g + lane < c1;
    double md = DINF;
    if (live) md = mindist2_box(a.box[g + lane], qx, qy);
    for (;;) {
      const bool cand = live && md <= kd;
      if (!__any_sync(FULL, cand)) break;
      const unsigned key =
          cand ? ((__float_as_uint(__double2float_rd(md)) & ~31u) | (unsigned)lane) : 0xffffffffu;
      int cb;
      bool v;
      pick_chunks<chunk_for_k(32 * KPL)>(key, live, lane, ob, oe, g - c0, cb, v);
      const StoreRec r = load_rec(a.obj, cb, v);
      prof_add(a.prof, own ? PROF_OWN_CHUNKS_SCANNED : PROF_EXP_CHUNKS_SCANNED, 1, lane);
      const double d2 = v ? pair_d2(qx, qy, r.x, r.y) : DINF;
      const bool pass = v && d2 <= kd && r.id != me && key_less(d2, r.id, kd, ki);
      const unsigned m = __ballot_sync(FULL, pass);
      if (m) {
        if (pass) {
          const int pos = nbuf + __popc(m & lt);
          bufd[pos] = d2;
          bufi[pos] = r.id;
        }
        nbuf += __popc(m);
        prof_add(a.prof, PROF_ADMITTED, __popc(m), lane);
        __syncwarp();
        if (nbuf > flush_at<KPL>()) {
          prof_add(a.prof, PROF_SORT_MERGES, 1, lane);
          merge_sm<KPL>(ld, li, bufd, bufi, nbuf, lane);
          nbuf = 0;
          kth_sm<KPL>(ld, li, k, kd, ki);
          if (cap < kd) {
            kd = cap;
            ki = IDMAX;
          }
        }
      }
    }
  }
  if (nbuf) {
    prof_add(a.prof, PROF_INSERTS, 1, lane);
    merge_sm<KPL>(ld, li, bufd, bufi, nbuf, lane);
  }
}

template <int KPL>
__device__ __forceinline__ void visit_leaf_buf(List<KPL>& L, int k, int leaf, double qx, double qy,
                                               long long me, const SearchArgs& a, int lane,
                                               double* bufd, long long* bufi, double* rowd,
                                               long long* rowi, bool own) {
  constexpr int N = 32 * KPL;
  const int ob = __ldg(&a.cell_start[leaf]), oe = __ldg(&a.cell_start[leaf + 1]);
  const int c0 = __ldg(&a.chunk_start[leaf]), c1 = c0 + (oe - ob + chunk_for_k(32 * KPL) - 1) / chunk_for_k(32 * KPL);
  const unsigned lt = (1u << lane) - 1u;
  prof_add(a.prof, own ? PROF_OWN_CHUNKS_TOTAL : PROF_EXP_CHUNKS_TOTAL, c1 - c0, lane);
  if (!own) prof_add(a.prof, PROF_EXP_LEAF_VISITS, 1, lane);
  double kd;
  long long ki;
  list_kth<KPL>(L, k, kd, ki);
  int nbuf = 0;
  for (int g = c0; g < c1; g += 32) {
    bool live = g + lane < c1;
    double md = DINF;
    if (live) md = mindist2_box(a.box[g + lane], qx, qy);
    for (;;) {
      const bool cand = live && md <= kd;
      if (!__any_sync(FULL, cand)) break;
      const unsigned key =
          cand ? ((__float_as_uint(__double2float_rd(md)) & ~31u) | (unsigned)lane) : 0xffffffffu;
      int cb;
      bool v;
      pick_chunks<chunk_for_k(32 * KPL)>(key, live, lane, ob, oe, g - c0, cb, v);
      const StoreRec r = load_rec(a.obj, cb, v);
      prof_add(a.prof, own ? PROF_OWN_CHUNKS_SCANNED : PROF_EXP_CHUNKS_SCANNED, 1, lane);
      const double d2 = v ? pair_d2(qx, qy, r.x, r.y) : DINF;
      const bool pass = v && d2 <= kd && r.id != me && key_less(d2, r.id, kd, ki);
      const unsigned m = __ballot_sync(FULL, pass);
      if (m) {
        if (pass) {
          const int pos = nbuf + __popc(m & lt);
          bufd[pos] = d2;
          bufi[pos] = r.id;
        }
        nbuf += __popc(m);
        prof_add(a.prof, PROF_ADMITTED, __popc(m), lane);
        __syncwarp();
        if (nbuf > N - 32) {
          prof_add(a.prof, PROF_SORT_MERGES, 1, lane);
          merge_buffer_k<KPL>(L, bufd, bufi, nbuf, rowd, rowi, lane);
          nbuf = 0;
          list_kth<KPL>(L, k, kd, ki);
        }
      }
    }
  }
  if (nbuf) {
    prof_add(a.prof, PROF_INSERTS, 1, lane);  // (k > 32: counts final partial merges)
    merge_buffer_k<KPL>(L, bufd, bufi, nbuf, rowd, rowi, lane);
  }
}

// engine.py:421-431 coarsest_levels: the coarsest quadrant aligned with the
// cursor (first code for right walks, last code for left walks)
__device__ __forceinline__ int coarsest_level(int p, int dir, int l_deep) {
  const int a = p + (dir ? 0 : 1);  // positions are < 4^l_max = 2^20 (l_max <= 10)
  if (a == 0) return 0;
  const int tz2 = (__ffs(a) - 1) >> 1;
  return l_deep - min(tz2, l_deep);
}

// mindist2_cell (mknn_common.cuh) with the per-level cell width taken from
// a table: fl(cx * (w * 2^-lvl)) is the same rounding of the same exact
// product as the reference's fl(ldexp(cx, -lvl) * w) (geometry.py:172-181),
// since w * 2^-lvl is exact (the kernel checks the widths are 0 or >= 2^-1000)
__device__ __forceinline__ double mindist2_cell_w(uint32_t code, double wl, double hl,
                                                  const Region& r, double qx, double qy) {
  const uint32_t cx = compact_bits32(code), cy = compact_bits32(code >> 1);
  const double fx = (double)cx, fy = (double)cy;
  const double xl = __dadd_rn(r.x_lo, __dmul_rn(fx, wl));
  const double xh = __dadd_rn(r.x_lo, __dmul_rn(__dadd_rn(fx, 1.0), wl));
  const double yl = __dadd_rn(r.y_lo, __dmul_rn(fy, hl));
  const double yh = __dadd_rn(r.y_lo, __dmul_rn(__dadd_rn(fy, 1.0), hl));
  const double dx = dmax(dmax(__dsub_rn(xl, qx), __dsub_rn(qx, xh)), 0.0);
  const double dy = dmax(dmax(__dsub_rn(yl, qy), __dsub_rn(qy, yh)), 0.0);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// instrumentation: record one distance task (dir 0 = own leaf, 1 = left,
// 2 = right; iteration = the query's 0-based navigate call in that direction)
__device__ __forceinline__ void emit_task(const SearchArgs& a, unsigned dir, uint32_t iter,
                                          uint32_t leaf) {
  if (a.task_keys) {
    const unsigned long long p = atomicAdd(a.task_count, 1ull);
    if (p < (unsigned long long)a.task_cap)
      a.task_keys[p] = ((unsigned long long)dir << 60) | ((unsigned long long)iter << 40) | leaf;
  }
}

// engine.py:529-554 _audit_prune_events for one pruned quadrant (one lane):
// does it hold an object (not the issuer) strictly closer than thr?
__device__ __noinline__ bool audit_quadrant(const int32_t* __restrict__ z_map,
                                            const int32_t* __restrict__ cell_start,
                                            const StoreRec* __restrict__ obj, Region r, int l_deep,
                                            int lvl, long long qc, double thr, double qx, double qy,
                                            long long me) {
  const int sh = 2 * (l_deep - lvl);
  const long long lo = qc << sh, hi = (qc + 1) << sh;
  const int l0 = z_map[lo], l1 = z_map[hi - 1];
  for (int li = l0; li <= l1; li++) {
    const int b = cell_start[li], e = cell_start[li + 1];
    for (int i = b; i < e; i++) {
      const StoreRec& p = obj[i];
      const long long c = encode(p.x, p.y, r, l_deep);
      if (c >= lo && c < hi && p.id != me && pair_d2(qx, qy, p.x, p.y) < thr) return true;
    }
  }
  return false;
}

// engine.py:396-503 navigate for one query and one direction, run by one
// lane: returns the assigned leaf ordinal or -1 when the direction is
// exhausted.  thr is the query's k-th d2 (+inf while the list is not full).
__device__ __forceinline__ int navigate(const SearchArgs& a, int l_deep, int dir, int& cursor,
                                        double thr, double qx, double qy, long long me,
                                        uint32_t& prunes, uint32_t& viol,
                                        const double2* __restrict__ cw,
                                        uint32_t* steps = nullptr) {
  const int n_codes = 1 << (2 * l_deep);
  int pos = cursor;
  if (dir ? pos >= n_codes : pos < 0) return -1;
  const bool full = thr < DINF;  // engine.py:415: thr = MAXDIST iff the list is full
  int lvl = full ? coarsest_level(pos, dir, l_deep) : l_deep;
  for (;;) {
    if (MKNN_PROFILE && steps) (*steps)++;
    const int delta = l_deep - lvl;
    const uint32_t qc = (uint32_t)(pos >> (2 * delta));
    double md2 = 0.0;
    if (full) {
      if (cw) {
        const double2 wh = cw[lvl];
        md2 = mindist2_cell_w(qc, wh.x, wh.y, a.r, qx, qy);
      } else {  // a width below 2^-1000: w * 2^-lvl might not be exact
        md2 = mindist2_cell(lvl, qc, a.r, qx, qy);
      }
    }
    if (md2 > thr) {  // prune (engine.py:447-460; strict, see the header)
      prunes++;
      if (a.audit && audit_quadrant(a.z_map, a.cell_start, a.obj, a.r, l_deep, lvl, qc, thr,
                                    qx, qy, me))
        viol++;
      pos += dir ? (1 << (2 * delta)) : -(1 << (2 * delta));
    } else if (lvl < l_deep) {  // descend (engine.py:462-465)
      lvl++;
      continue;
    } else {  // resolve through z_map (engine.py:467-487)
      const int li = __ldg(&a.z_map[pos]);
      const int key = (int)__ldg(&a.leaf_key[li]);
      const int after = dir ? key + (int)__ldg(&a.leaf_span[li]) : key - 1;
      if (__ldg(&a.cell_start[li + 1]) > __ldg(&a.cell_start[li])) {
        cursor = after;
        return li;
      }
      pos = after;  // empty leaf: skip it whole
    }
    if (dir ? pos >= n_codes : pos < 0) {  // exhausted (engine.py:489-494)
      cursor = pos;
      return -1;
    }
    lvl = full ? coarsest_level(pos, dir, l_deep) : l_deep;
  }
}

// navigate for one query run by a group of G lanes (lane j of the group,
// gmask = the group's lanes): the walk descends from the coarsest aligned
// quadrant through the quadrants holding the cursor until one is pruned or
// the leaf is reached, so lane j evaluates level lvl0 + j of that chain at
// once and the first pruned level is the one the serial walk prunes at --
// the same prune events, cursor moves and leaf as navigate, one parallel
// step per prune or leaf resolution instead of one step per level.  Used
// where a warp holds at most two queries (k > 64) and its other lanes
// would idle through the serial walk.  Returns the leaf (every lane of the
// group); prunes / viol are counted identically in every lane of the group.
__device__ __forceinline__ int navigate_grp(const SearchArgs& a, int l_deep, int dir, int& cursor,
                                            double thr, double qx, double qy, long long me,
                                            uint32_t& prunes, uint32_t& viol,
                                            const double2* __restrict__ cw, int j, unsigned gmask) {
  const int n_codes = 1 << (2 * l_deep);
  int pos = cursor;
  if (dir ? pos >= n_codes : pos < 0) return -1;
  const bool full = thr < DINF;  // engine.py:415
  for (;;) {
    const int lvl0 = full ? coarsest_level(pos, dir, l_deep) : l_deep;
    const int lvl = lvl0 + j;
    bool pr = false;
    uint32_t qc = 0;
    if (full && lvl <= l_deep) {
      qc = (uint32_t)(pos >> (2 * (l_deep - lvl)));
      double md2;
      if (cw) {
        const double2 wh = cw[lvl];
        md2 = mindist2_cell_w(qc, wh.x, wh.y, a.r, qx, qy);
      } else {
        md2 = mindist2_cell(lvl, qc, a.r, qx, qy);
      }
      pr = md2 > thr;  // strict, as navigate
    }
    const unsigned pm = __ballot_sync(gmask, pr) & gmask;
    if (pm) {  // prune at the first pruned level of the chain (engine.py:447-460)
      const int p = (__ffs(pm) - 1) - (__ffs(gmask) - 1);
      const int plvl = lvl0 + p;
      prunes++;
      if (a.audit) {
        const bool v = j == p && audit_quadrant(a.z_map, a.cell_start, a.obj, a.r, l_deep, plvl,
                                                qc, thr, qx, qy, me);
        if (__ballot_sync(gmask, v) & gmask) viol++;
      }
      const int delta = l_deep - plvl;
      pos += dir ? (1 << (2 * delta)) : -(1 << (2 * delta));
    } else {  // every level of the chain passes: resolve the leaf (engine.py:467-487)
      const int li = __ldg(&a.z_map[pos]);
      const int key = (int)__ldg(&a.leaf_key[li]);
      const int after = dir ? key + (int)__ldg(&a.leaf_span[li]) : key - 1;
      if (__ldg(&a.cell_start[li + 1]) > __ldg(&a.cell_start[li])) {
        cursor = after;
        return li;
      }
      pos = after;  // empty leaf: skip it whole
    }
    if (dir ? pos >= n_codes : pos < 0) {  // exhausted (engine.py:489-494)
      cursor = pos;
      return -1;
    }
  }
}

// one navigate call for each of the warp's B <= 2 queries (owner lane q),
// each run by its 32 / B lanes with navigate_grp; li / cur / prunes / viol
// of an active owner lane updated as navigate would
template <int B>
__device__ __forceinline__ void nav_grouped(const SearchArgs& a, int l_deep, bool go_right, bool act,
                                            int& cur, double thr, double qx, double qy, long long me,
                                            uint32_t& prunes, uint32_t& viol,
                                            const double2* __restrict__ cw, int lane, int& li) {
  constexpr int G = 32 / B;
  const int g = lane / G, j = lane % G;
  const unsigned gmask = G == 32 ? FULL : (((1u << G) - 1u) << (g * G));
  const int gr = __shfl_sync(FULL, (int)go_right, g);
  const int ga = __shfl_sync(FULL, (int)act, g);
  int gc = __shfl_sync(FULL, cur, g);
  const double gt = __shfl_sync(FULL, thr, g);
  const double gx = __shfl_sync(FULL, qx, g), gy = __shfl_sync(FULL, qy, g);
  const long long gm = __shfl_sync(FULL, me, g);
  uint32_t gp = 0, gv = 0;
  int gl = -1;
  if (ga) gl = navigate_grp(a, l_deep, gr, gc, gt, gx, gy, gm, gp, gv, cw, j, gmask);
  const int src = (lane % B) * G;
  const int rl = __shfl_sync(FULL, gl, src), rc = __shfl_sync(FULL, gc, src);
  const uint32_t rp = __shfl_sync(FULL, gp, src), rv = __shfl_sync(FULL, gv, src);
  if (act) {
    li = rl;
    cur = rc;
    prunes += rp;
    viol += rv;
  }
}

// k <= 32 lists kept in the caller's output rows (k slots each, d2 until
// the emit turns them into distances): no shared memory, so L1 keeps the
// leaf records and chunk boxes
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ long long ld_keep(const long long* p, unsigned long long pol) {
  long long v;
  asm volatile("ld.global.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* p, unsigned long long pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_keep(long long* p, long long v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(double* p, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// the rows are re-read by the warp's later visits: keep them in L2
// (evict_last) while the streamed object records come and go
__device__ __forceinline__ void row_load(List<1>& L, const double* __restrict__ rd,
                                         const long long* __restrict__ ri, int k, int lane) {
  const unsigned long long pol = l2_evict_last();
  L.d[0] = lane < k ? ld_keep(rd + lane, pol) : DINF;
  L.id[0] = lane < k ? ld_keep(ri + lane, pol) : IDMAX;
}
__device__ __forceinline__ void row_store(const List<1>& L, double* __restrict__ rd,
                                          long long* __restrict__ ri, int k, int lane) {
  const unsigned long long pol = l2_evict_last();
  if (lane < k) {
    st_keep(rd + lane, L.d[0], pol);
    st_keep(ri + lane, L.id[0], pol);
  }
}

template <int KPL>
__device__ __forceinline__ void list_load(List<KPL>& L, const double* __restrict__ sd,
                                          const long long* __restrict__ si, int lane) {
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    L.d[s] = sd[s * 32 + lane];
    L.id[s] = si[s * 32 + lane];
  }
}

template <int KPL>
__device__ __forceinline__ void list_store(const List<KPL>& L, double* __restrict__ sd,
                                           long long* __restrict__ si, int lane) {
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    sd[s * 32 + lane] = L.d[s];
    si[s * 32 + lane] = L.id[s];
  }
}

// One warp owns a batch of B consecutive queries (leaf-grouped order).  The
// lists live in shared memory between steps; leaf scans are warp-wide
// (32 candidates per ballot), navigation is lane-parallel (lane q walks
// query q), mirroring the paper's thread-per-query navigation.
template <int KPL, int B, int WARPS, int MINB, bool ROWS = false>
__global__ void __launch_bounds__(32 * WARPS, MINB) k_search(const SearchArgs a) {
  static_assert(!ROWS || KPL == 1, "row-resident lists need k <= 32");
  constexpr int N = 32 * KPL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* sd = reinterpret_cast<double*>(smem_raw) + (size_t)w * B * N;
  long long* si = reinterpret_cast<long long*>(smem_raw) + (size_t)WARPS * B * N + (size_t)w * B * N;
  // k > 32: per-warp admission buffer after the lists
  double* bufd = reinterpret_cast<double*>(smem_raw) + (size_t)2 * WARPS * B * N + (size_t)w * N;
  long long* bufi = reinterpret_cast<long long*>(smem_raw) + (size_t)2 * WARPS * B * N +
                    (size_t)WARPS * N + (size_t)w * N;
  const int l_deep = __ldg(&a.scalars[0]);
  // per-level quadrant widths for navigate (mindist2_cell_w)
  __shared__ double2 cw_tab[MAX_L_MAX + 1];
  if (threadIdx.x <= l_deep)
    cw_tab[threadIdx.x] = make_double2(__dmul_rn(a.r.w, pow2_neg(threadIdx.x)),
                                       __dmul_rn(a.r.h, pow2_neg(threadIdx.x)));
  __syncthreads();
  const bool cw_exact =
      (a.r.w == 0.0 || a.r.w >= 0x1p-1000) && (a.r.h == 0.0 || a.r.h >= 0x1p-1000);
  const double2* cw = cw_exact ? cw_tab : nullptr;
  const int64_t t0 = ((int64_t)blockIdx.x * WARPS + w) * B;
  if (t0 >= a.nq) return;
  const int nb = (int)((a.nq - t0) < B ? (a.nq - t0) : B);
  const int k = a.k;

  // per-lane query state (lane q < nb owns query t0 + q)
  const bool mine = lane < nb;
  uint32_t q = 0, own = 0, qrow = 0;
  double qx = 0.0, qy = 0.0, thr = DINF;
  long long me = 0;
  int cur_l = -1, cur_r = 0;
  uint32_t evals = 0, prunes = 0, viol = 0, calls_l = 0, calls_r = 0;
  bool act_l = false, act_r = false;
  if (mine) {
    q = __ldg(&a.q_order[t0 + lane]);
    if (ROWS) qrow = __ldg(&a.q_row[q]);
    qx = __ldg(&a.qx[q]);
    qy = __ldg(&a.qy[q]);
    me = __ldg(&a.qi[q]);
    own = __ldg(&a.q_leaf[q]);
    cur_l = (int)__ldg(&a.leaf_key[own]) - 1;
    cur_r = (int)(__ldg(&a.leaf_key[own]) + __ldg(&a.leaf_span[own]));
    act_l = act_r = true;
    const int pop = __ldg(&a.cell_start[own + 1]) - __ldg(&a.cell_start[own]);
    evals = (uint32_t)pop;  // first_iteration row (rows with 0 candidates dropped, engine.py:334-338)
    if (pop > 0) emit_task(a, 0, 0, own);
  }

  // first_iteration: every query against its own leaf.  Consecutive
  // queries mostly share the leaf: the previous query's list after this
  // pass holds k objects of the same leaf, so (when they exclude this
  // issuer) they bound this query's k-th own-leaf distance by the triangle
  // inequality, d <= d_prev(k) + |q - q_prev|.  Padded by 2^-30 relative
  // (far above the rounding of any term), the bound only filters objects
  // and chunks that cannot be among the k nearest of the leaf, so the list
  // after the pass -- and the navigation threshold taken from it
  // (engine.py:415) -- is exactly the reference's.
  double p_kd = DINF, p_x = 0.0, p_y = 0.0;
  long long p_id = IDMAX;  // this lane's entry of the previous list
  uint32_t p_own = 0xffffffffu;
  __shared__ unsigned long long ph_sh[WARPS][2];  // phase timestamps (lane 0; no registers held)
  if (lane == 0) ph_sh[w][0] = gtimer();
  for (int j = 0; j < nb; j++) {
    const double jx = __shfl_sync(FULL, qx, j), jy = __shfl_sync(FULL, qy, j);
    const long long jme = __shfl_sync(FULL, me, j);
    const uint32_t jown = __shfl_sync(FULL, own, j);
    double cap = DINF;
    if (KPL == 1 && jown == p_own && p_kd < DINF && !__any_sync(FULL, p_id == jme)) {
      const double dx = jx - p_x, dy = jy - p_y;
      const double rr = sqrt(p_kd) + sqrt(dx * dx + dy * dy);
      cap = rr * rr * (1.0 + 0x1p-30) + 0x1p-1000;
    }
    if constexpr (KPL > 1 && SMEM_LIST) {
      double* ld = sd + j * N;
      long long* li = si + j * N;
      // the previous query's own-pass list as a cap, as for k <= 32 above
      // (all its k entries must exclude this issuer)
      double capm = DINF;
      if (KCAP && jown == p_own && p_kd < DINF) {
        const long long* pli = si + (j - 1) * N;
        bool hit = false;
#pragma unroll
        for (int s = 0; s < KPL; s++) hit |= pli[s * 32 + lane] == jme;
        if (!__any_sync(FULL, hit)) {
          const double dx = jx - p_x, dy = jy - p_y;
          const double rr = sqrt(p_kd) + sqrt(dx * dx + dy * dy);
          capm = rr * rr * (1.0 + 0x1p-30) + 0x1p-1000;
        }
      }
#pragma unroll
      for (int s = 0; s < KPL; s++) {
        ld[s * 32 + lane] = DINF;
        li[s * 32 + lane] = IDMAX;
      }
      __syncwarp();
      visit_leaf_sm<KPL>(k, (int)jown, jx, jy, jme, a, lane, bufd, bufi, ld, li, true, capm);
      double kd;
      long long ki;
      kth_sm<KPL>(ld, li, k, kd, ki);
      if (lane == j) thr = kd;
      p_kd = kd;
      p_x = jx;
      p_y = jy;
      p_own = jown;
      continue;
    }
    List<KPL> L;
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      L.d[s] = DINF;
      L.id[s] = IDMAX;
    }
    if constexpr (KPL == 1)
      visit_leaf<KPL>(L, k, (int)jown, jx, jy, jme, a, lane, true, cap);
    else
      visit_leaf_buf<KPL>(L, k, (int)jown, jx, jy, jme, a, lane, bufd, bufi, sd + j * N, si + j * N,
                          true);
    double kd;
    long long ki;
    list_kth<KPL>(L, k, kd, ki);
    if (lane == j) thr = kd;
    p_kd = kd;
    p_x = jx;
    p_y = jy;
    p_id = L.id[0];
    p_own = jown;
    if constexpr (ROWS) {
      const int64_t o = (int64_t)__shfl_sync(FULL, qrow, j) * k;
      row_store(L, a.out_dist + o, a.out_nids + o, k, lane);
    } else {
      list_store<KPL>(L, sd + j * N, si + j * N, lane);
    }
  }
  __syncwarp();
  if (lane == 0) ph_sh[w][1] = gtimer();

  // direction loop, left first (engine.py:645-681)
  // per query: left, right, left, ... (engine.py:645-681); a drained
  // direction drops out.  Each lane keeps its own alternation, so a
  // lane with one direction left navigates it every round instead of
  // idling through the other direction's rounds (same per-query order)
  bool next_right = false;
  if (a.debug_phase == 1) act_l = act_r = false;
  while (__any_sync(FULL, act_l || act_r)) {
    const bool go_right = (act_l && act_r) ? next_right : act_r;
    const bool act = act_l || act_r;
    next_right = !go_right;
    int li = -1;
    int cur = go_right ? cur_r : cur_l;
    if constexpr (GROUP_NAV && B <= 2 && !ROWS) {
      nav_grouped<B>(a, l_deep, go_right, act, cur, thr, qx, qy, me, prunes, viol, cw, lane, li);
    } else if (act) {
      li = navigate(a, l_deep, go_right ? 1 : 0, cur, thr, qx, qy, me, prunes, viol, cw);
    }
    if (act) {
      if (go_right) {
        calls_r++;
        cur_r = cur;
        act_r = li >= 0;
      } else {
        calls_l++;
        cur_l = cur;
        act_l = li >= 0;
      }
      if (li >= 0) {
        emit_task(a, go_right ? 2 : 1, (go_right ? calls_r : calls_l) - 1, li);
        evals += (uint32_t)(__ldg(&a.cell_start[li + 1]) - __ldg(&a.cell_start[li]));
      }
    }
    // update_nn_lists: merge each assigned leaf into its query's list
    unsigned pend = __ballot_sync(FULL, li >= 0);
    while (pend) {
      const int j = __ffs(pend) - 1;
      pend &= pend - 1;
      const int jl = __shfl_sync(FULL, li, j);
      const double jx = __shfl_sync(FULL, qx, j), jy = __shfl_sync(FULL, qy, j);
      const long long jme = __shfl_sync(FULL, me, j);
      if constexpr (KPL > 1 && SMEM_LIST) {
        double* ld = sd + j * N;
        long long* li = si + j * N;
        visit_leaf_sm<KPL>(k, jl, jx, jy, jme, a, lane, bufd, bufi, ld, li, false);
        double kd;
        long long ki;
        kth_sm<KPL>(ld, li, k, kd, ki);
        if (lane == j) thr = kd;
        continue;
      }
      List<KPL> L;
      int64_t o = 0;
      if constexpr (ROWS) {
        o = (int64_t)__shfl_sync(FULL, qrow, j) * k;
        row_load(L, a.out_dist + o, a.out_nids + o, k, lane);
      } else {
        list_load<KPL>(L, sd + j * N, si + j * N, lane);
      }
      if constexpr (KPL == 1)
        visit_leaf<KPL>(L, k, jl, jx, jy, jme, a, lane, false);
      else
        visit_leaf_buf<KPL>(L, k, jl, jx, jy, jme, a, lane, bufd, bufi, sd + j * N, si + j * N,
                            false);
      if constexpr (ROWS)
        row_store(L, a.out_dist + o, a.out_nids + o, k, lane);
      else
        list_store<KPL>(L, sd + j * N, si + j * N, lane);
      double kd;
      long long ki;
      list_kth<KPL>(L, k, kd, ki);
      if (lane == j) thr = kd;
    }
    __syncwarp();
  }
  if (lane == 0) phase_add(a.phase_ns, ph_sh[w][0], ph_sh[w][1], gtimer());

  // _emit: canonical order already; sqrt correctly rounded (engine.py:706)
  if constexpr (ROWS && KPL == 1) {
    // rows in the output: lane j turns row j around; the lanes walk the k
    // entries together, so 32 rows' loads are in flight at once
    const bool own_row = lane < nb;
    const int64_t o = (int64_t)qrow * k;
    int len = 0;
    const unsigned long long pol = l2_evict_last();
    for (int e = 0; e < k; e++) {
      if (own_row) {
        const double d = ld_keep(a.out_dist + o + e, pol);
        if (d < DINF) {
          len++;
          __stcs(&a.out_dist[o + e], __dsqrt_rn(d));
        }
      }
    }
    if (own_row) a.out_len[qrow] = len;
  }
  for (int j = 0; j < nb && !(ROWS && KPL == 1); j++) {
    const uint32_t jq = __shfl_sync(FULL, q, j);
    const uint32_t row = ROWS ? __shfl_sync(FULL, qrow, j) : __ldg(&a.q_row[jq]);
    List<KPL> L;
    if constexpr (ROWS)
      row_load(L, a.out_dist + (int64_t)row * k, a.out_nids + (int64_t)row * k, k, lane);
    else
      list_load<KPL>(L, sd + j * N, si + j * N, lane);
    int len = 0;
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      const int e = (s << 5) | lane;
      const bool ok = e < k && L.d[s] < DINF;
      len += __popc(__ballot_sync(FULL, ok));
      if (ok) {  // final values: streaming stores
        __stcs(&a.out_nids[(int64_t)row * k + e], L.id[s]);
        __stcs(&a.out_dist[(int64_t)row * k + e], __dsqrt_rn(L.d[s]));
      }
    }
    if (lane == 0) a.out_len[row] = len;
  }
  if (mine) {
    QueryStats st;
    st.evals = evals;
    st.prunes = prunes;
    st.nav_left = (uint16_t)min(calls_l, 65535u);
    st.nav_right = (uint16_t)min(calls_r, 65535u);
    st.violations = viol;
    a.stats[t0 + lane] = st;
  }
}

// ===== 16 < k <= 32: one-slot lists kept as store positions ===============
//
// Same walk as k_search (own leaf, then alternating left/right visits), but
// between visits a query's list is kept as k store positions (4 bytes per
// entry) in the warp's shared memory instead of (d2, id) pairs in the
// output row: a visit gathers its query's k records back and recomputes
// their d2 (pair_d2 is deterministic), and the emit writes each result row
// exactly once.  The round-1 kernel wrote every row once per visit plus once
// more in the emit (2.0x DRAM write amplification at cfg3); this one writes
// 1.04x (ncu: 531 MB against 512 MB of rows) at the same speed.  CTAs are
// persistent and take 32-query batches from a work counter.
//
// The own-leaf pass runs as its own kernel (k_own1) over leaf tasks, the
// paper's cell-per-SM staging: a CTA takes 64 consecutive
// queries of the leaf-grouped order, bulk-copies (cp.async.bulk, TMA 1-D,
// mbarrier completion) the records and chunk boxes of their own leaves --
// contiguous spans of the store -- into shared memory once, and its four
// warps run the queries' own-leaf passes from there.  The lists go to global
// memory as store positions and k_search1 continues with the expansion.
// (A per-warp ring of 1 KB chunk tiles filled one step ahead, the first
// attempt, measured 3.8x slower: ~160 small bulk copies per 32-query batch
// queue on the copy engine.  A leaf is staged once for all its queries.)
struct L1 {
  double d;
  long long id;
  int pos;  // store index of the entry (-1: empty)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, unsigned bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// where a visit reads its leaf: the store in global memory (SH = false) or
// the CTA's shared-memory stage of the leaf (SH = true: srec / sbox are the
// shared addresses of the leaf's first record and first chunk box)
struct LeafSrc {
  uint32_t srec, sbox;
};

template <bool SH>
__device__ __forceinline__ ChunkBox box_at(const ChunkBox* __restrict__ box, const LeafSrc& src,
                                           int c, int c0) {
  if constexpr (SH) {
    ChunkBox b;
    const uint32_t ad = src.sbox + (uint32_t)(c - c0) * (uint32_t)sizeof(ChunkBox);
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(b.x_lo), "=d"(b.y_lo) : "r"(ad));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(b.x_hi), "=d"(b.y_hi) : "r"(ad + 16));
    return b;
  } else {
    return box[c];
  }
}

template <bool SH>
__device__ __forceinline__ void rec_at(const StoreRec* __restrict__ obj, const LeafSrc& src, int r,
                                       int ob, double& x, double& y, long long& id) {
  if constexpr (SH) {
    const uint32_t ad = src.srec + (uint32_t)(r - ob) * (uint32_t)sizeof(StoreRec);
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(ad));
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(id) : "r"(ad + 16));
  } else {
    const StoreRec q = ld_rec(&obj[r]);
    x = q.x;
    y = q.y;
    id = q.id;
  }
}

// one step's chunks, distributed: lane l < 16 holds record l of the nearer
// chunk, lane 16 + l record l of the other (rec = its store index, -1 when
// the lane has none); md0 = a lower bound (float, rounded down) of the
// nearer chunk's box min-dist2, -1 when the pick is empty
struct Pick {
  int rec;
  float md0;
};

// chunk candidates of a leaf, 32 boxes at a time (lane i: chunk g + i);
// mdf = the box min-dist2 rounded down to float (NaN once picked or past
// the leaf: it then compares false with any kd, +inf included).  Testing mdf <= kd instead of md <= kd admits a superset of
// the qualifying chunks (a few more scans, never fewer), so the result is
// unchanged.
struct ChunkIter {
  int g, c1;
  float mdf;
};

#define MKNN_FDEAD __int_as_float(0x7fffffff)  // NaN

// the (up to) two nearest remaining chunks that qualify under kd, nearest
// first (kd only shrinks, so a chunk that does not qualify never will)
template <bool SH>
__device__ __forceinline__ Pick next_pick(ChunkIter& it, double kd, int ob, int oe, int c0,
                                          const ChunkBox* __restrict__ box, const LeafSrc& src,
                                          double qx, double qy, int lane) {
  constexpr int CH = chunk_for_k(32);
  Pick p;
  p.rec = -1;
  p.md0 = -1.0f;
  for (;;) {
    const bool cand = (double)it.mdf <= kd;  // false for NaN
    if (!__any_sync(FULL, cand)) {
      it.g += 32;
      if (it.g >= it.c1) return p;
      it.mdf = it.g + lane < it.c1
                   ? __double2float_rd(mindist2_box(box_at<SH>(box, src, it.g + lane, c0), qx, qy))
                   : MKNN_FDEAD;
      continue;
    }
    // nearest box first (key: mdf with the lane in the low bits; mdf >= 0,
    // so its bits order like the values); the order only affects speed
    unsigned key = cand ? ((__float_as_uint(it.mdf) & ~31u) | (unsigned)lane) : 0xffffffffu;
    const unsigned k0 = __reduce_min_sync(FULL, key);
    const int a0 = (int)(k0 & 31u);
    if (lane == a0) {
      it.mdf = MKNN_FDEAD;
      key = 0xffffffffu;
    }
    const unsigned k1 = __reduce_min_sync(FULL, key);
    const int a1 = k1 == 0xffffffffu ? -1 : (int)(k1 & 31u);
    if (lane == a1) it.mdf = MKNN_FDEAD;
    p.md0 = __uint_as_float(k0 & ~31u);
    const int ch = lane < CH ? a0 : a1;
    const int r = ob + (it.g - c0 + ch) * CH + (lane & (CH - 1));
    p.rec = ch >= 0 && r < min(ob + (it.g - c0 + ch + 1) * CH, oe) ? r : -1;
    return p;
  }
}

__device__ __forceinline__ void kth1(const L1& L, int k, double& kd, long long& ki) {
  kd = __shfl_sync(FULL, L.d, k - 1);
  ki = __shfl_sync(FULL, L.id, k - 1);
}

// exact (d2, id) compare-exchange carrying the store position
__device__ __forceinline__ void cx1(double& d, long long& id, int& p, int lane, int size, int j) {
  const double pd = __shfl_xor_sync(FULL, d, j);
  const long long pi = __shfl_xor_sync(FULL, id, j);
  const int pp = __shfl_xor_sync(FULL, p, j);
  const bool asc = (lane & size) == 0;
  const bool lower = (lane & j) == 0;
  const bool take = (lower == asc) ? key_less(pd, pi, d, id) : key_less(d, id, pd, pi);
  d = take ? pd : d;
  id = take ? pi : id;
  p = take ? pp : p;
}

__device__ __noinline__ L1 exact_sort1(L1 c, int lane) {
  for (int size = 2; size <= 32; size <<= 1)
    for (int j = size >> 1; j > 0; j >>= 1) cx1(c.d, c.id, c.pos, lane, size, j);
  return c;
}

// L <- the 32 smallest of L u C (both ascending), exact networks
__device__ __noinline__ L1 exact_merge1(L1 l, L1 c, int lane) {
  const double rd = __shfl_xor_sync(FULL, c.d, 31);
  const long long ri = __shfl_xor_sync(FULL, c.id, 31);
  const int rp = __shfl_xor_sync(FULL, c.pos, 31);
  const bool lt = key_less(rd, ri, l.d, l.id);
  l.d = lt ? rd : l.d;
  l.id = lt ? ri : l.id;
  l.pos = lt ? rp : l.pos;
  for (int j = 16; j > 0; j >>= 1) cx1(l.d, l.id, l.pos, lane, 64, j);
  return l;
}

// insert one key into the ascending list (the last element falls off)
__device__ __forceinline__ void insert1(L1& L, double kd, long long ki, int kp, int lane) {
  const bool gt = key_less(kd, ki, L.d, L.id);
  const unsigned m = __ballot_sync(FULL, gt);
  const double ud = __shfl_up_sync(FULL, L.d, 1);
  const long long ui = __shfl_up_sync(FULL, L.id, 1);
  const int up = __shfl_up_sync(FULL, L.pos, 1);
  const bool gprev = lane ? ((m >> (lane - 1)) & 1u) : false;
  if (gt) {
    L.d = gprev ? ud : kd;
    L.id = gprev ? ui : ki;
    L.pos = gprev ? up : kp;
  }
}

// admit one batch of candidates (lane: (cd, ci, cp), (+inf, IDMAX) when it
// does not pass; m = ballot of passing lanes): few are inserted one by one,
// many are sorted (32-bit keys, exact fallback) and merged
__device__ __forceinline__ void admit1(L1& L, double cd, long long ci, int cp, unsigned m, int lane,
                                       unsigned long long* prof) {
  const int cnt = __popc(m);
  prof_add(prof, PROF_ADMITTED, cnt, lane);
  prof_add(prof, cnt <= 4 ? PROF_INSERTS : PROF_SORT_MERGES, cnt <= 4 ? cnt : 1, lane);
  if (cnt <= 4) {
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      insert1(L, __shfl_sync(FULL, cd, src), __shfl_sync(FULL, ci, src), __shfl_sync(FULL, cp, src),
              lane);
    }
    return;
  }
  const bool empty = __shfl_sync(FULL, L.d, 0) == DINF;
  // sort the batch
  {
    uint32_t key = akey(cd, 5, (uint32_t)lane);
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int j = size >> 1; j > 0; j >>= 1) {
        const uint32_t p = __shfl_xor_sync(FULL, key, j);
        const bool take_min = ((lane & j) == 0) == ((lane & size) == 0);
        key = take_min ? min(key, p) : max(key, p);
      }
    }
    if (akey_ties(key, 5, lane)) {
      L1 c;
      c.d = cd;
      c.id = ci;
      c.pos = cp;
      c = exact_sort1(c, lane);
      cd = c.d;
      ci = c.id;
      cp = c.pos;
    } else {
      const int src = (int)(key & 31u);
      const double nd = __shfl_sync(FULL, cd, src);
      const long long ni = __shfl_sync(FULL, ci, src);
      const int np = __shfl_sync(FULL, cp, src);
      cd = nd;
      ci = ni;
      cp = np;
    }
  }
  if (empty) {  // the sorted batch is the list
    L.d = cd;
    L.id = ci;
    L.pos = cp;
    return;
  }
  // merge: min(A_i, B_{31-i}) holds the 32 smallest as a bitonic sequence
  const uint32_t kl = akey(L.d, 6, (uint32_t)lane);
  const uint32_t kc = akey(cd, 6, 32u | (uint32_t)lane);
  const uint32_t rc = __shfl_sync(FULL, kc, 31 - lane);
  uint32_t mm = min(kl, rc);
  const uint32_t kept_max = __reduce_max_sync(FULL, mm);
  const uint32_t drop_min = __reduce_min_sync(FULL, max(kl, rc));
  const bool cut_tie = ((kept_max ^ drop_min) >> 6) == 0 && (kept_max >> 6) < (AKEY_INF >> 6);
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    const uint32_t p = __shfl_xor_sync(FULL, mm, j);
    mm = (lane & j) ? max(mm, p) : min(mm, p);
  }
  if (cut_tie || akey_ties(mm, 6, lane)) {
    L1 c;
    c.d = cd;
    c.id = ci;
    c.pos = cp;
    L = exact_merge1(L, c, lane);
    return;
  }
  const int src = (int)(mm & 31u);
  const bool from_c = (mm & 32u) != 0;
  const double dl = __shfl_sync(FULL, L.d, src), dc = __shfl_sync(FULL, cd, src);
  const long long il = __shfl_sync(FULL, L.id, src), ic = __shfl_sync(FULL, ci, src);
  const int pl = __shfl_sync(FULL, L.pos, src), pc = __shfl_sync(FULL, cp, src);
  L.d = from_c ? dc : dl;
  L.id = from_c ? ic : il;
  L.pos = from_c ? pc : pl;
}

// One row of the reference's distance phase (first_iteration's own leaf,
// engine.py:356-373, or update_nn_lists' assigned leaf, 376-393) for one
// query: every object of the leaf except the issuer (engine.py:298-300)
// competes; admission is (d2, id) < k-th.  Chunks whose box min-dist2
// exceeds the k-th d2 (or the cap, see k_search1) cannot hold an admissible
// object and are skipped.
template <bool SH>
__device__ __forceinline__ void visit1(L1& L, int k, int leaf, double qx, double qy, long long me,
                                       const SearchArgs& a, int lane, bool own, double cap = DINF,
                                       LeafSrc src = LeafSrc{0u, 0u}) {
  const int ob = __ldg(&a.cell_start[leaf]), oe = __ldg(&a.cell_start[leaf + 1]);
  const int c0 = __ldg(&a.chunk_start[leaf]), c1 = c0 + (oe - ob + chunk_for_k(32) - 1) / chunk_for_k(32);
  prof_add(a.prof, own ? PROF_OWN_CHUNKS_TOTAL : PROF_EXP_CHUNKS_TOTAL, c1 - c0, lane);
  if (!own) prof_add(a.prof, PROF_EXP_LEAF_VISITS, 1, lane);
  double kd;
  long long ki;
  kth1(L, k, kd, ki);
  if (cap < kd) {
    kd = cap;
    ki = IDMAX;
  }
  ChunkIter it;
  it.g = c0 - 32;
  it.c1 = c1;
  it.mdf = MKNN_FDEAD;
  Pick cur = next_pick<SH>(it, kd, ob, oe, c0, a.box, src, qx, qy, lane);
  if (cur.md0 < 0.0f) {
    if (!own) prof_add(a.prof, PROF_EXP_VISITS_NO_SCAN, 1, lane);
    return;
  }
  bool admitted = false;
  for (;;) {
    double x = 0.0, y = 0.0;
    long long id = 0;
    if (cur.rec >= 0) rec_at<SH>(a.obj, src, cur.rec, ob, x, y, id);
    prof_add(a.prof, own ? PROF_OWN_CHUNKS_SCANNED : PROF_EXP_CHUNKS_SCANNED, 1, lane);
    const bool valid = cur.rec >= 0;
    const double d2 = valid ? pair_d2(qx, qy, x, y) : DINF;
    const bool pass = valid && d2 <= kd && id != me && key_less(d2, id, kd, ki);
    const unsigned m = __ballot_sync(FULL, pass);
    if (m) {
      admit1(L, pass ? d2 : DINF, pass ? id : IDMAX, pass ? cur.rec : -1, m, lane, a.prof);
      kth1(L, k, kd, ki);
      if (cap < kd) {
        kd = cap;
        ki = IDMAX;
      }
      admitted = true;
    }
    const Pick nxt = next_pick<SH>(it, kd, ob, oe, c0, a.box, src, qx, qy, lane);
    if (nxt.md0 < 0.0f) break;
    cur = nxt;
  }
  if (!own) prof_add(a.prof, PROF_EXP_VISITS_ADMITTING, admitted, lane);
}

// a query's list from its stored positions: gather the records, recompute d2
__device__ __forceinline__ void list_gather(L1& L, const int32_t* __restrict__ lp, int k,
                                            const StoreRec* __restrict__ obj, double qx, double qy,
                                            int lane) {
  const int p = lane < k ? lp[lane] : -1;
  L.pos = p;
  L.d = DINF;
  L.id = IDMAX;
  if (p >= 0) {
    const StoreRec r = ld_rec(&obj[p]);
    L.d = pair_d2(qx, qy, r.x, r.y);
    L.id = r.id;
  }
}

// FUSED: the own-leaf pass runs inline (one kernel; MKNN_OWN_FUSED=1, for
// A/B); otherwise k_own1 ran it and left each query's list (store positions)
// in a.own_pos and its k-th d2 in a.own_thr, by leaf-grouped position.
template <int B, int MINB, bool FUSED>
__global__ void __launch_bounds__(32, MINB) k_search1(const __grid_constant__ SearchArgs a) {
  static_assert(B <= 32, "one query per lane");
  __shared__ double2 cw_tab[MAX_L_MAX + 1];
  __shared__ int32_t lists[B * 32];  // the batch's lists as store positions
  __shared__ unsigned long long ph_sh[2];  // phase timestamps (lane 0; no registers held)
  const int lane = threadIdx.x;
  const int l_deep = __ldg(&a.scalars[0]);
  if (lane <= l_deep)
    cw_tab[lane] = make_double2(__dmul_rn(a.r.w, pow2_neg(lane)), __dmul_rn(a.r.h, pow2_neg(lane)));
  __syncwarp();
  const bool cw_exact =
      (a.r.w == 0.0 || a.r.w >= 0x1p-1000) && (a.r.h == 0.0 || a.r.h >= 0x1p-1000);
  const double2* cw = cw_exact ? cw_tab : nullptr;
  const int k = a.k;

  for (;;) {
    unsigned batch = 0;
    if (lane == 0) batch = atomicAdd(a.work, 1u);
    batch = __shfl_sync(FULL, batch, 0);
    if ((int64_t)batch * B >= a.nq) break;
    if (a.batch_order) batch = __ldg(&a.batch_order[batch]);
    const int t0 = (int)batch * B;  // queries < 2^31 (uint32 orders)
    const int nb = (int)((a.nq - t0) < B ? (a.nq - t0) : B);

    // per-lane query state (lane q < nb owns query t0 + q)
    const bool mine = lane < nb;
    uint32_t own = 0, qrow = 0;
    double qx = 0.0, qy = 0.0, thr = DINF;
    long long me = 0;
    int cur_l = -1, cur_r = 0;
    uint32_t evals = 0, prunes = 0, viol = 0, calls_l = 0, calls_r = 0;
    bool act_l = false, act_r = false;
    if (mine) {
      const uint32_t q = __ldg(&a.q_order[t0 + lane]);
      qrow = __ldg(&a.q_row[q]);
      qx = __ldg(&a.qx[q]);
      qy = __ldg(&a.qy[q]);
      me = __ldg(&a.qi[q]);
      own = __ldg(&a.q_leaf[q]);
      cur_l = (int)__ldg(&a.leaf_key[own]) - 1;
      cur_r = (int)(__ldg(&a.leaf_key[own]) + __ldg(&a.leaf_span[own]));
      act_l = act_r = true;
      const int pop = __ldg(&a.cell_start[own + 1]) - __ldg(&a.cell_start[own]);
      evals = (uint32_t)pop;  // first_iteration row (rows with 0 candidates dropped, engine.py:334-338)
      if (pop > 0) emit_task(a, 0, 0, own);
    }

    // first_iteration: every query against its own leaf, with the previous
    // query's own-pass k-th distance as a cap when both share the leaf and
    // its list excludes this issuer (see k_search: d <= d_prev(k) + |q -
    // q_prev|, padded by 2^-30 relative; the list after the pass -- and the
    // navigation threshold taken from it, engine.py:415 -- is unchanged)
    if (lane == 0) ph_sh[0] = gtimer();
    if constexpr (!FUSED) {
      for (int j = 0; j < nb; j++) lists[j * 32 + lane] = __ldg(&a.own_pos[(int64_t)(t0 + j) * 32 + lane]);
      if (mine) thr = __ldg(&a.own_thr[t0 + lane]);
    }
    bool excl = false;  // the previous query's list excludes this query's issuer
    for (int j = 0; j < nb && FUSED; j++) {
      const double jx = __shfl_sync(FULL, qx, j), jy = __shfl_sync(FULL, qy, j);
      const long long jme = __shfl_sync(FULL, me, j);
      const uint32_t jown = __shfl_sync(FULL, own, j);
      // previous query's coordinates, leaf and own-pass k-th d2 (thr)
      const int jp = j > 0 ? j - 1 : 0;
      const double p_x = __shfl_sync(FULL, qx, jp), p_y = __shfl_sync(FULL, qy, jp);
      const double p_kd = __shfl_sync(FULL, thr, jp);
      const uint32_t p_own = __shfl_sync(FULL, own, jp);
      double cap = DINF;
      if (j > 0 && jown == p_own && p_kd < DINF && excl) {
        const double dx = jx - p_x, dy = jy - p_y;
        const double rr = sqrt(p_kd) + sqrt(dx * dx + dy * dy);
        cap = rr * rr * (1.0 + 0x1p-30) + 0x1p-1000;
      }
      L1 L;
      L.d = DINF;
      L.id = IDMAX;
      L.pos = -1;
      visit1<false>(L, k, (int)jown, jx, jy, jme, a, lane, true, cap);
      double kd;
      long long ki;
      kth1(L, k, kd, ki);
      if (lane == j) thr = kd;
      const long long nme = __shfl_sync(FULL, me, j + 1 < 32 ? j + 1 : j);
      excl = !__any_sync(FULL, L.id == nme);
      lists[j * 32 + lane] = lane < k ? L.pos : -1;
    }
    if (lane == 0) ph_sh[1] = FUSED ? gtimer() : ph_sh[0];  // staged: k_own1 timed it

    // direction loop, left first (engine.py:645-681)
    // per query: left, right, left, ... (engine.py:645-681); a drained
    // direction drops out.  Each lane keeps its own alternation, so a
    // lane with one direction left navigates it every round instead of
    // idling through the other direction's rounds (same per-query order)
    bool next_right = false;
    if (a.debug_phase == 1) act_l = act_r = false;
    while (__any_sync(FULL, act_l || act_r)) {
      const bool go_right = (act_l && act_r) ? next_right : act_r;
      const bool act = act_l || act_r;
      next_right = !go_right;
      int li = -1;
      uint32_t nsteps = 0;
      if (act) {
        int cur = go_right ? cur_r : cur_l;
        li = navigate(a, l_deep, go_right ? 1 : 0, cur, thr, qx, qy, me, prunes, viol, cw, &nsteps);
        if (go_right) {
          calls_r++;
          cur_r = cur;
          act_r = li >= 0;
        } else {
          calls_l++;
          cur_l = cur;
          act_l = li >= 0;
        }
        if (li >= 0) {
          emit_task(a, go_right ? 2 : 1, (go_right ? calls_r : calls_l) - 1, li);
          evals += (uint32_t)(__ldg(&a.cell_start[li + 1]) - __ldg(&a.cell_start[li]));
        }
      }
      if (MKNN_PROFILE && a.prof) {
        const unsigned al = __ballot_sync(FULL, act);
        const uint32_t mx = __reduce_max_sync(FULL, nsteps), sm = __reduce_add_sync(FULL, nsteps);
        prof_add(a.prof, PROF_ROUNDS, 1, lane);
        prof_add(a.prof, PROF_ROUND_LANES, __popc(al), lane);
        prof_add(a.prof, PROF_NAV_STEPS, sm, lane);
        prof_add(a.prof, PROF_NAV_MAXSTEPS, mx, lane);
      }
      // update_nn_lists: merge each assigned leaf into its query's list
      unsigned pend = __ballot_sync(FULL, li >= 0);
      while (pend) {
        const int j = __ffs(pend) - 1;
        pend &= pend - 1;
        const int jl = __shfl_sync(FULL, li, j);
        const double jx = __shfl_sync(FULL, qx, j), jy = __shfl_sync(FULL, qy, j);
        const long long jme = __shfl_sync(FULL, me, j);
        L1 L;
        list_gather(L, lists + j * 32, k, a.obj, jx, jy, lane);
        visit1<false>(L, k, jl, jx, jy, jme, a, lane, false);
        lists[j * 32 + lane] = lane < k ? L.pos : -1;
        double kd;
        long long ki;
        kth1(L, k, kd, ki);
        if (lane == j) thr = kd;
      }
      __syncwarp();
    }
    if (lane == 0) phase_add(a.phase_ns, ph_sh[0], ph_sh[1], gtimer());

    // _emit: canonical order already; sqrt correctly rounded (engine.py:706);
    // every result row is written once (streaming stores)
#pragma unroll 2
    for (int j = 0; j < nb; j++) {
      const uint32_t row = __shfl_sync(FULL, qrow, j);
      const double jx = __shfl_sync(FULL, qx, j), jy = __shfl_sync(FULL, qy, j);
      const int p = lane < k ? lists[j * 32 + lane] : -1;
      const bool ok = p >= 0;
      if (ok) {
        const StoreRec r = ld_rec(&a.obj[p]);
        __stcs(&a.out_nids[(int64_t)row * k + lane], r.id);
        __stcs(&a.out_dist[(int64_t)row * k + lane], __dsqrt_rn(pair_d2(jx, jy, r.x, r.y)));
      }
      const int len = __popc(__ballot_sync(FULL, ok));
      if (lane == 0) a.out_len[row] = len;
    }
    if (mine) {
      QueryStats st;
      st.evals = evals;
      st.prunes = prunes;
      st.nav_left = (uint16_t)min(calls_l, 65535u);
      st.nav_right = (uint16_t)min(calls_r, 65535u);
      st.violations = viol;
      a.stats[t0 + lane] = st;
    }
    __syncwarp();
  }
}

// ---- k_own1: the own-leaf pass as staged leaf tasks -----------------------
constexpr int OWN_WARPS = 4;
constexpr int OWN_PER_WARP = 16;                   // consecutive queries per warp
constexpr int OWN_Q = OWN_WARPS * OWN_PER_WARP;    // queries per CTA batch
constexpr int STAGE_RECS = 1024;                   // 32 KB of records
constexpr int STAGE_BOXES = 128;                   // 4 KB of chunk boxes
constexpr int OWN_CTAS_PER_SM = 5;

// first_iteration (engine.py:356-373) for OWN_Q consecutive queries of the
// leaf-grouped order per CTA batch.  Warp 0 plans the stage: the batch's
// distinct own leaves, in order, get contiguous slices of the shared record
// and box arrays while they fit (a leaf that does not fit -- and every later
// one -- is read from global memory instead); each staged leaf's records and
// boxes are two contiguous spans of the store, fetched by two bulk copies
// that complete on one mbarrier.  Each warp then runs its 16 consecutive
// queries' passes, capping each by the previous query's own-pass k-th
// distance exactly as k_search1 does (same-leaf triangle bound).
__global__ void __launch_bounds__(32 * OWN_WARPS, OWN_CTAS_PER_SM) k_own1(const __grid_constant__ SearchArgs a) {
  __shared__ __align__(128) StoreRec srec[STAGE_RECS];
  __shared__ __align__(128) ChunkBox sbox[STAGE_BOXES];
  __shared__ double sqx[OWN_Q], sqy[OWN_Q];
  __shared__ long long sme[OWN_Q];
  __shared__ uint32_t sown[OWN_Q];
  __shared__ int32_t sro[OWN_Q], sbo[OWN_Q];  // stage offsets of the query's leaf (-1: global)
  __shared__ __align__(8) unsigned long long bar;
  __shared__ unsigned s_batch;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t bar_a = smem_u32(&bar);
  if (t == 0) {
    mbar_init(bar_a, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int k = a.k;
  uint32_t phase = 0;
  for (;;) {
    if (t == 0) s_batch = atomicAdd(a.work + 1, 1u);
    __syncthreads();
    const int64_t t0 = (int64_t)s_batch * OWN_Q;
    if (t0 >= a.nq) break;
    const int nb = (int)((a.nq - t0) < OWN_Q ? (a.nq - t0) : OWN_Q);
    if (t < nb) {
      const uint32_t q = __ldg(&a.q_order[t0 + t]);
      sqx[t] = __ldg(&a.qx[q]);
      sqy[t] = __ldg(&a.qy[q]);
      sme[t] = __ldg(&a.qi[q]);
      sown[t] = __ldg(&a.q_leaf[q]);
    }
    __syncthreads();
    if (w == 0) {
      // order the previous batch's shared reads before this batch's bulk writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      int ro = 0, bo = 0;      // stage fill so far
      int c_ro = -1, c_bo = 0; // offsets of the leaf running into this round
      bool open = true;        // no leaf has failed to fit yet
      for (int r0 = 0; r0 < nb; r0 += 32) {
        const int j = r0 + lane;
        const bool in = j < nb;
        const uint32_t l = in ? sown[j] : 0xffffffffu;
        const bool first = in && (j == 0 || sown[j - 1] != l);
        int nr = 0, nx = 0, ob = 0, c0 = 0;
        if (first) {
          ob = __ldg(&a.cell_start[l]);
          nr = __ldg(&a.cell_start[l + 1]) - ob;
          c0 = __ldg(&a.chunk_start[l]);
          nx = (nr + chunk_for_k(32) - 1) / chunk_for_k(32);
        }
        // inclusive prefix of the leaders' sizes
        int pr = nr, px = nx;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int ur = __shfl_up_sync(FULL, pr, o), ux = __shfl_up_sync(FULL, px, o);
          if (lane >= o) {
            pr += ur;
            px += ux;
          }
        }
        const bool fits = open && ro + pr <= STAGE_RECS && bo + px <= STAGE_BOXES;
        const bool stage = first && fits && nr > 0;
        const int my_ro = ro + pr - nr, my_bo = bo + px - nx;
        if (stage) {
          const unsigned bytes = (unsigned)(nr + nx) * 32u;
          asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(bar_a), "r"(bytes) : "memory");
          bulk_g2s(smem_u32(&srec[my_ro]), a.obj + ob, (unsigned)nr * 32u, bar_a);
          if (nx) bulk_g2s(smem_u32(&sbox[my_bo]), a.box + c0, (unsigned)nx * 32u, bar_a);
        }
        // every query takes its leader's offsets (or the carried ones)
        const unsigned lead_m = __ballot_sync(FULL, first);
        const unsigned below = lead_m & (0xffffffffu >> (31 - lane));
        const int ld = below ? 31 - __clz(below) : -1;
        const int l_ro = __shfl_sync(FULL, stage ? my_ro : -1, ld < 0 ? 0 : ld);
        const int l_bo = __shfl_sync(FULL, my_bo, ld < 0 ? 0 : ld);
        if (in) {
          sro[j] = ld < 0 ? c_ro : l_ro;
          sbo[j] = ld < 0 ? c_bo : l_bo;
        }
        // carry: the last query of the round's offsets; stage fill
        c_ro = __shfl_sync(FULL, in ? sro[j] : -1, min(31, nb - 1 - r0));
        c_bo = __shfl_sync(FULL, in ? sbo[j] : 0, min(31, nb - 1 - r0));
        const unsigned fit_m = __ballot_sync(FULL, first && !fits);
        const int tot_r = __shfl_sync(FULL, pr, 31), tot_x = __shfl_sync(FULL, px, 31);
        if (fit_m) {
          open = false;
          // keep the fill of the leaders that did fit
          const int fl = __ffs(fit_m) - 1;
          const int fr = __shfl_sync(FULL, pr - nr, fl), fx = __shfl_sync(FULL, px - nx, fl);
          ro += fr;
          bo += fx;
        } else {
          ro += tot_r;
          bo += tot_x;
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_a) : "memory");
    }
    __syncthreads();
    mbar_wait(bar_a, phase & 1u);
    phase++;

    const unsigned long long ph_t0 = gtimer();
    const int j0 = w * OWN_PER_WARP, j1 = min(j0 + OWN_PER_WARP, nb);
    double p_kd = DINF, p_x = 0.0, p_y = 0.0;
    uint32_t p_own = 0xffffffffu;
    bool excl = false;
    for (int j = j0; j < j1; j++) {
      const double jx = sqx[j], jy = sqy[j];
      const long long jme = sme[j];
      const uint32_t jown = sown[j];
      double cap = DINF;
      if (j > j0 && jown == p_own && p_kd < DINF && excl) {
        const double dx = jx - p_x, dy = jy - p_y;
        const double rr = sqrt(p_kd) + sqrt(dx * dx + dy * dy);
        cap = rr * rr * (1.0 + 0x1p-30) + 0x1p-1000;
      }
      L1 L;
      L.d = DINF;
      L.id = IDMAX;
      L.pos = -1;
      const int ro = sro[j];
      if (ro >= 0) {
        const LeafSrc src{smem_u32(&srec[ro]), smem_u32(&sbox[sbo[j]])};
        visit1<true>(L, k, (int)jown, jx, jy, jme, a, lane, true, cap, src);
      } else {
        visit1<false>(L, k, (int)jown, jx, jy, jme, a, lane, true, cap);
      }
      double kd;
      long long ki;
      kth1(L, k, kd, ki);
      p_kd = kd;
      p_x = jx;
      p_y = jy;
      p_own = jown;
      excl = j + 1 < j1 ? !__any_sync(FULL, L.id == sme[j + 1]) : false;
      a.own_pos[(t0 + j) * 32 + lane] = lane < k ? L.pos : -1;
      if (lane == 0) a.own_thr[t0 + j] = kd;
    }
    if (lane == 0) {
      const unsigned long long te = gtimer();
      phase_add(a.phase_ns, ph_t0, te, te);
    }
    __syncthreads();
  }
}

constexpr int HIST_SMEM = 1024;

// one histogram count; lanes holding the same value (most queries make the
// same few navigate calls) are combined into one atomic by their leader
__device__ __forceinline__ void hist_add(uint32_t* sh, uint32_t* gl, int cap, uint32_t v) {
  const unsigned peers = __match_any_sync(__activemask(), v);
  if ((int)(threadIdx.x & 31) != __ffs(peers) - 1) return;
  if (v < HIST_SMEM) atomicAdd(&sh[v], (uint32_t)__popc(peers));
  else if ((int64_t)v < cap) atomicAdd(&gl[v], (uint32_t)__popc(peers));
}

__global__ void k_stats_reduce(const QueryStats* __restrict__ st, int64_t nq,
                               unsigned long long* tot, uint32_t* hist_l, uint32_t* hist_r,
                               int hist_cap) {
  __shared__ uint32_t hl[HIST_SMEM], hr[HIST_SMEM];
  for (int i = threadIdx.x; i < HIST_SMEM; i += blockDim.x) hl[i] = hr[i] = 0;
  __syncthreads();
  unsigned long long ev = 0, pr = 0, vi = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    const QueryStats s = st[i];
    ev += s.evals;
    pr += s.prunes;
    vi += s.violations;
    hist_add(hl, hist_l, hist_cap, s.nav_left);
    hist_add(hr, hist_r, hist_cap, s.nav_right);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ev += __shfl_xor_sync(FULL, ev, o);
    pr += __shfl_xor_sync(FULL, pr, o);
    vi += __shfl_xor_sync(FULL, vi, o);
  }
  // one atomic per counter and block (same-address L2 atomics serialise)
  __shared__ unsigned long long wt[3][32];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    wt[0][w] = ev;
    wt[1][w] = pr;
    wt[2][w] = vi;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    unsigned long long v = 0;
    for (int j = 0; j < nw; j++) v += wt[threadIdx.x][j];
    if (v) atomicAdd(&tot[threadIdx.x], v);
  }
  for (int i = threadIdx.x; i < HIST_SMEM && i < hist_cap; i += blockDim.x) {
    if (hl[i]) atomicAdd(&hist_l[i], hl[i]);
    if (hr[i]) atomicAdd(&hist_r[i], hr[i]);
  }
}

// The search writes padded rows (k slots each) straight into the caller's
// output; that IS the CSR layout when every row is full (min(k, objects
// other than the issuer) == k, the common case).  Otherwise the rows are
// moved to `tmp` and compacted back.  Both kernels read the CSR total on the
// device and return at once when every row is full (no host round trip).
// skip: the tick is redone (issuer ids repeated or beyond the planned range:
// some rows were never written, so the lengths are not trustworthy)
__global__ void k_rows_stash(const int64_t* __restrict__ off, int64_t nq, int k,
                             const long long* __restrict__ nids, const double* __restrict__ dist,
                             long long* __restrict__ t_nids, double* __restrict__ t_dist,
                             const int32_t* __restrict__ skip) {
  const int64_t total = nq * (int64_t)k;
  if (off[nq] == total || (skip && *skip)) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    t_nids[i] = nids[i];
    t_dist[i] = dist[i];
  }
}

__global__ void k_rows_compact(const int32_t* __restrict__ len, const long long* __restrict__ nids,
                               const double* __restrict__ dist, int64_t nq, int k,
                               const int64_t* __restrict__ off, long long* __restrict__ c_nids,
                               double* __restrict__ c_dist, const int32_t* __restrict__ skip) {
  const int64_t total = nq * (int64_t)k;
  if (off[nq] == total || (skip && *skip)) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / k;
    const int e = (int)(i - r * k);
    if (e < len[r]) {
      c_nids[off[r] + e] = nids[i];
      c_dist[off[r] + e] = dist[i];
    }
  }
}

}  // namespace

// ---- batch scheduling for the persistent k_search1 --------------------
// The work counter hands out batches in leaf-grouped order, so the last
// batches handed out are as costly as any and the kernel ends on a tail of
// partly idle SMs.  lpt_order hands them out costliest first (longest
// processing time first, by the population of the batch's first own leaf
// in 16 log2 classes), so the tail is made of the cheapest batches.  Order
// only: every batch still runs whole, results are unchanged.  Within a
// class the batches keep runs of up to 32 consecutive ones (warp-
// aggregated cursors), so concurrently running warps still share leaves.
// Off by default (MKNN_LPT=1 enables it): measured slower (tuning log).
constexpr int LPT_CLASSES = 16;

__device__ __forceinline__ int lpt_class(const SearchArgs& a, int64_t b, int B) {
  const uint32_t q = __ldg(&a.q_order[b * B]);
  const uint32_t leaf = __ldg(&a.q_leaf[q]);
  const int pop = __ldg(&a.cell_start[leaf + 1]) - __ldg(&a.cell_start[leaf]);
  return LPT_CLASSES - 1 - min(LPT_CLASSES - 1, 31 - __clz(max(pop, 1)));
}

__global__ void k_lpt_count(const __grid_constant__ SearchArgs a, int B, int64_t nbt) {
  __shared__ uint32_t h[LPT_CLASSES];
  if (threadIdx.x < LPT_CLASSES) h[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbt;
       b += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[lpt_class(a, b, B)], 1u);
  __syncthreads();
  if (threadIdx.x < LPT_CLASSES && h[threadIdx.x]) atomicAdd(&a.lpt_cnt[threadIdx.x], h[threadIdx.x]);
}

__global__ void k_lpt_place(const __grid_constant__ SearchArgs a, int B, int64_t nbt) {
  __shared__ uint32_t base[LPT_CLASSES];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < LPT_CLASSES) {
    uint32_t x = 0;
    for (int c = 0; c < (int)threadIdx.x; c++) x += a.lpt_cnt[c];
    base[threadIdx.x] = x;
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); b0 < nbt; b0 += stride) {
    const int64_t b = b0 + lane;
    const int c = b < nbt ? lpt_class(a, b, B) : LPT_CLASSES;
    const unsigned m = __match_any_sync(FULL, c);
    const int leader = __ffs(m) - 1;
    uint32_t off = 0;
    if (lane == leader && c < LPT_CLASSES) off = atomicAdd(&a.lpt_cnt[LPT_CLASSES + c], (uint32_t)__popc(m));
    off = __shfl_sync(FULL, off, leader);
    if (c < LPT_CLASSES)
      a.batch_order[base[c] + off + __popc(m & ((1u << lane) - 1u))] = (uint32_t)b;
  }
}

template <int KPL, int B, int WARPS, int MINB = 1, bool ROWS = false>
int launch_batched(const SearchArgs& a, cudaStream_t s) {
  constexpr int N = 32 * KPL;
  const size_t smem = ROWS ? 0 : (size_t)WARPS * (B + (KPL > 1 ? 1 : 0)) * N * (sizeof(double) + sizeof(long long));
  // the attribute is per device: remember which devices have it
  static unsigned long long configured = 0;  // bit d: device d
  int dev = 0;
  MKNN_CUDA_OK(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
    MKNN_CUDA_OK(cudaFuncSetAttribute(k_search<KPL, B, WARPS, MINB, ROWS>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    __atomic_fetch_or(&configured, bit, __ATOMIC_ACQ_REL);
  }
  const int64_t per_cta = (int64_t)WARPS * B;
  const unsigned blocks = (unsigned)((a.nq + per_cta - 1) / per_cta);
  MKNN_LAUNCH k_search<KPL, B, WARPS, MINB, ROWS><<<blocks, 32 * WARPS, smem, s>>>(a);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

// resident CTAs of k_search1 per SM (1-warp CTAs; registers bound it)
#ifndef MKNN_S1_CTAS
#define MKNN_S1_CTAS 32
#endif
constexpr int SEARCH1_CTAS_PER_SM = MKNN_S1_CTAS;

template <int B, bool FUSED>
int launch_search1(const SearchArgs& a, cudaStream_t s) {
  int dev = 0;
  MKNN_CUDA_OK(cudaGetDevice(&dev));
  int sms = 0;
  MKNN_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  MKNN_CUDA_OK(cudaMemsetAsync(a.work, 0, 2 * sizeof(unsigned), s));
  if (!FUSED) {
    const int64_t ob = (a.nq + OWN_Q - 1) / OWN_Q;
    const int64_t og = std::min<int64_t>(ob, (int64_t)sms * OWN_CTAS_PER_SM);
    MKNN_LAUNCH k_own1<<<(unsigned)og, 32 * OWN_WARPS, 0, s>>>(a);
    MKNN_CUDA_OK(cudaGetLastError());
  }
  const int64_t batches = (a.nq + B - 1) / B;
  int64_t grid = std::min<int64_t>(batches, (int64_t)sms * SEARCH1_CTAS_PER_SM);
  // MKNN_LPT=1: costliest batches first (A/B; measured 2.6 % slower at cfg3:
  // the tail is short and the leaf-grouped order's L2 sharing is worth more)
  static const bool lpt = [] {
    const char* e = getenv("MKNN_LPT");
    return e && e[0] == '1';
  }();
  SearchArgs b = a;
  if (!lpt || !a.batch_order || !a.lpt_cnt || batches < 2 * grid) {
    b.batch_order = nullptr;
  } else {
    MKNN_CUDA_OK(cudaMemsetAsync(a.lpt_cnt, 0, 2 * LPT_CLASSES * sizeof(uint32_t), s));
    const unsigned lg = (unsigned)std::min<int64_t>((batches + 255) / 256, (int64_t)sms * 2);
    MKNN_LAUNCH k_lpt_count<<<lg, 256, 0, s>>>(a, B, batches);
    MKNN_CUDA_OK(cudaGetLastError());
    MKNN_LAUNCH k_lpt_place<<<lg, 256, 0, s>>>(a, B, batches);
    MKNN_CUDA_OK(cudaGetLastError());
  }
  MKNN_LAUNCH k_search1<B, SEARCH1_CTAS_PER_SM, FUSED><<<(unsigned)grid, 32, 0, s>>>(b);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

// Queries per warp batch: the query density picks it (see below), but never
// so many that the batches stop covering the GPU: a small tick (cfg2: 100K
// queries, 3.1K batches of 32 for 4.7K resident warps) leaves SMs idle and
// its time is one warp's 32 serial own-leaf passes, so halve the batch until
// there are >= 2 batches per resident warp slot (or 4 queries per warp).
static int batch_for(const SearchArgs& a, int by_density) {
  static int slots = 0;
  if (!slots) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    slots = sms * SEARCH1_CTAS_PER_SM;
  }
  int b = by_density;
  while (b > 4 && (a.nq + b - 1) / b < 2 * (int64_t)slots) b >>= 1;
  static const int force = [] {  // MKNN_BATCH=4/8/16/32: A/B override
    const char* e = getenv("MKNN_BATCH");
    return e ? atoi(e) : 0;
  }();
  return force ? force : b;
}

int search_launch(const SearchArgs& a, cudaStream_t s) {
  if (a.nq == 0) return 0;
  // MKNN_SEARCH_V0=1: the round-1 kernel (lists in the output rows, record
  // loads through L1) for A/B measurements
  static const bool v0 = [] {
    const char* e = getenv("MKNN_SEARCH_V0");
    return e && e[0] == '1';
  }();
  // 16 < k <= 32: k_search1 (lists as positions in shared memory, rows
  // written once); k <= 16: the row-resident kernel, measured 3-11 % faster
  // there (the per-visit position gather weighs more on short lists)
  // MKNN_S1_MIN=k0: k_search1 from k > k0 (A/B; default 16)
  static const int s1_min = [] {
    const char* e = getenv("MKNN_S1_MIN");
    return e ? atoi(e) : 16;
  }();
  if (a.k > s1_min && a.k <= 32 && !v0) {
    const double qd = (double)a.nq / (double)(a.n_objects > 0 ? a.n_objects : 1);
    // MKNN_OWN_STAGED=1: the own-leaf pass as k_own1's staged leaf tasks
    // (bulk copies into shared memory) instead of inline in k_search1
    static const bool staged = [] {
      const char* e = getenv("MKNN_OWN_STAGED");
      return e && e[0] == '1';
    }();
    if (!staged || !a.own_pos) {
      const int b = batch_for(a, qd < 0.015 ? 4 : qd < 0.04 ? 8 : qd < 0.06 ? 16 : 32);
      if (b == 4) return launch_search1<4, true>(a, s);
      if (b == 8) return launch_search1<8, true>(a, s);
      if (b == 16) return launch_search1<16, true>(a, s);
      return launch_search1<32, true>(a, s);
    }
    const int b = batch_for(a, qd < 0.015 ? 4 : qd < 0.04 ? 8 : qd < 0.06 ? 16 : 32);
    if (b == 4) return launch_search1<4, false>(a, s);
    if (b == 8) return launch_search1<8, false>(a, s);
    if (b == 16) return launch_search1<16, false>(a, s);
    return launch_search1<32, false>(a, s);
  }
  // k <= 32: lists in the output rows (no shared memory: L1 holds the leaf
  // records and boxes), 32 queries per warp (every lane navigates), one
  // warp per CTA (a finished warp frees its slot at once), <= 64 registers:
  // the optimum measured on B200
  // Queries per warp follow the query density (queries per object): a
  // sparser batch spreads a warp's queries over more leaves and its
  // own-leaf scans stop sharing L1 lines (measured at 10M objects: 1M
  // queries -> 32; 300K -> 8: 1.75 -> 1.01 ms; a 1/4 row slice of a host
  // tick -> 8)
  const double qd = (double)a.nq / (double)(a.n_objects > 0 ? a.n_objects : 1);
  if (a.k <= 32) {
    const int b = batch_for(a, qd < 0.015 ? 4 : qd < 0.04 ? 8 : qd < 0.06 ? 16 : 32);
    if (b == 4) return launch_batched<1, 4, 1, 32, true>(a, s);
    if (b == 8) return launch_batched<1, 8, 1, 32, true>(a, s);
    if (b == 16) return launch_batched<1, 16, 1, 32, true>(a, s);
    return launch_batched<1, 32, 1, 32, true>(a, s);
  }
  // k > 32: the per-warp lists (B * 16 * k bytes of shared memory) bound the
  // resident warps, so fewer queries per warp win (measured at cfg3 objects:
  // k = 64 / 128 / 256 / 512 -24 / -18 / -24 / -17 % against 16/8/4/2; k =
  // 128 with 32-bit merge keys: 2 queries per warp 12.6 ms, 1: 13.5, 4:
  // 13.0, 8: 16.0)
  if (a.k <= 64) return launch_batched<2, 8, 4>(a, s);
  if (a.k <= 128) return launch_batched<4, MKNN_K128_B, MKNN_K128_WARPS, MKNN_K128_MINB>(a, s);
  if (a.k <= 256) return launch_batched<8, 1, 8>(a, s);
  if (a.k <= 512) return launch_batched<16, 1, 4>(a, s);
  return fail_msg(E_UNSUPPORTED, "k > 512 is not supported by the device top-k");
}

int stats_reduce(const QueryStats* st, int64_t nq, unsigned long long* dev_tot, uint32_t* hist_l,
                 uint32_t* hist_r, int hist_cap, cudaStream_t s) {
  if (nq == 0) return 0;
  int64_t blocks = (nq + 256 * 16 - 1) / (256 * 16);
  blocks = std::min<int64_t>(std::max<int64_t>(blocks, 1), 148 * 4);
  MKNN_LAUNCH k_stats_reduce<<<(unsigned)blocks, 256, 0, s>>>(st, nq, dev_tot, hist_l, hist_r, hist_cap);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

int rows_compact(const int32_t* len, long long* nids, double* dist, int64_t nq, int k,
                 int64_t* offsets, long long* t_nids, double* t_dist, const int32_t* skip, void* scratch,
                 cudaStream_t s) {
  int rc = exclusive_scan_i32_to_i64(len, offsets, nq, scratch, s);
  if (rc) return rc;
  if (nq == 0) return 0;
  const int64_t total = nq * (int64_t)k;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
  MKNN_LAUNCH k_rows_stash<<<(unsigned)blocks, 256, 0, s>>>(offsets, nq, k, nids, dist, t_nids, t_dist, skip);
  MKNN_LAUNCH k_rows_compact<<<(unsigned)blocks, 256, 0, s>>>(len, t_nids, t_dist, nq, k, offsets, nids,
                                                             dist, skip);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

namespace {
__global__ void k_sum_distinct(const unsigned long long* __restrict__ keys, int64_t n,
                               const int32_t* __restrict__ cell_start, unsigned long long* T) {
  unsigned long long acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0 || keys[i] != keys[i - 1]) {
      const uint32_t leaf = (uint32_t)(keys[i] & ((1ull << 40) - 1));
      acc += (unsigned long long)(cell_start[leaf + 1] - cell_start[leaf]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(T, acc);
}
}  // namespace

int streamed_records(unsigned long long* keys, unsigned long long* keys_alt, uint32_t* vals,
                     uint32_t* vals_alt, int64_t n, const int32_t* cell_start,
                     unsigned long long* dev_T, void* scratch, cudaStream_t s) {
  bool alt = false;
  int rc = radix_sort_pairs_u64((uint64_t*)keys, vals, (uint64_t*)keys_alt, vals_alt, n, 62, scratch,
                                s, &alt);
  if (rc) return rc;
  if (n > 0) {
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 8);
    MKNN_LAUNCH k_sum_distinct<<<(unsigned)blocks, 256, 0, s>>>(alt ? keys_alt : keys, n, cell_start,
                                                                dev_T);
  }
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

}  // namespace mknn
