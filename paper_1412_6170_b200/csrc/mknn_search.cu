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
// Top-k.  The running list holds N = 32*KPL keys (N >= k) distributed as
// element e = slot*32 + lane, sorted ascending by (d2, id) -- the oracle's
// canonical order (oracle.py:76-77).  Each 32*KPL-candidate chunk of a leaf
// is filtered against the k-th key (ballot); few survivors are inserted one
// by one with warp shuffles, many are bitonic-sorted and bitonic-merged.
// Admission is (d2, id) < k-th and a quadrant is pruned only when its
// min-dist2 is strictly greater than the k-th d2, so the canonical
// lowest-id member of a boundary tie group is always found (the reference
// prunes on >=, engine.py:447; distances are identical either way).
#include <algorithm>

#include "mknn_internal.h"

namespace mknn {

namespace {

constexpr int WARPS_PER_CTA = 8;

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

// engine.py:279-324 _merge_pack for one row: every object of [beg, end)
// except the issuer (by id, engine.py:298-300) competes for the list.
template <int KPL>
__device__ __forceinline__ void scan_range(List<KPL>& L, int k, int beg, int end, double qx,
                                           double qy, long long me, const double2* __restrict__ xy,
                                           const long long* __restrict__ ids, int lane) {
  constexpr int CH = 32 * KPL;
  constexpr int INS_MAX = 12 + 4 * KPL;
  for (int base = beg; base < end; base += CH) {
    double kd;
    long long ki;
    list_kth<KPL>(L, k, kd, ki);
    double cd[KPL];
    long long ci[KPL];
    unsigned mask[KPL];
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < KPL; j++) {
      const int idx = base + j * 32 + lane;
      bool pass = false;
      double d2 = DINF;
      long long id = IDMAX;
      if (idx < end) {
        const double2 p = __ldg(&xy[idx]);
        d2 = pair_d2(qx, qy, p.x, p.y);
        if (d2 <= kd && d2 < DINF) {
          id = __ldg(&ids[idx]);
          pass = (id != me) && key_less(d2, id, kd, ki);
        }
      }
      cd[j] = pass ? d2 : DINF;
      ci[j] = pass ? id : IDMAX;
      mask[j] = __ballot_sync(FULL, pass);
      cnt += __popc(mask[j]);
    }
    if (cnt == 0) continue;
    if (cnt <= INS_MAX) {
#pragma unroll
      for (int j = 0; j < KPL; j++) {
        unsigned m = mask[j];
        while (m) {
          const int src = __ffs(m) - 1;
          m &= m - 1;
          const double sd = __shfl_sync(FULL, cd[j], src);
          const long long si = __shfl_sync(FULL, ci[j], src);
          list_insert<KPL>(L, sd, si, lane);
        }
      }
    } else {
      bitonic_sort<KPL>(cd, ci, lane);
      if (__shfl_sync(FULL, L.d[0], 0) == DINF) {  // empty list: the sorted chunk is the list
#pragma unroll
        for (int j = 0; j < KPL; j++) {
          L.d[j] = cd[j];
          L.id[j] = ci[j];
        }
      } else {
        bitonic_merge_into<KPL>(L, cd, ci, lane);
      }
    }
  }
}

// Per-warp scratch for the own-leaf bucket select.
struct BucketScratch {
  double d[64];
  int32_t pos[64];
  int32_t hist[32];
};

constexpr int BUCKET_EM = 12;  // candidates per lane held in registers (own leaf <= 384)

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// histogram of bins (0..31, 32 = skip) -> first bin whose inclusive prefix
// count reaches `need` (31 if never); *before = count strictly below it
template <int EM>
__device__ __forceinline__ int bucket_cut(const int (&bin)[EM], int need, int32_t* hist, int lane,
                                          int& before) {
  hist[lane] = 0;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < EM; i++)
    if (bin[i] < 32) atomicAdd(&hist[bin[i]], 1);
  __syncwarp();
  const int h = hist[lane];
  int cum = h;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(FULL, cum, o);
    if (lane >= o) cum += u;
  }
  const unsigned m = __ballot_sync(FULL, cum >= need);
  const int b = m ? __ffs(m) - 1 : 31;
  before = __shfl_sync(FULL, cum - h, b);
  __syncwarp();
  return b;
}

// first_iteration for one query when the own leaf holds 33..32*EM objects
// and k <= 32 (engine.py:356-373 with the selection of kselect.py:34-138
// re-planned for a warp): the leaf's d2 stay in registers, a two-level
// 32-bin histogram over [min, max] finds a cut holding >= k+1 candidates
// (k plus room for the issuer, excluded by id afterwards), the cut is
// compacted to shared memory and only those candidates are sorted.  The
// binning is monotone in d2, so every candidate left out is strictly
// farther than every candidate kept: the list is exact.
__device__ __noinline__ void own_leaf_bucket(List<1>& L, int k, int beg, int end, double qx,
                                             double qy, long long me,
                                             const double2* __restrict__ xy,
                                             const long long* __restrict__ ids, int lane,
                                             BucketScratch* sc) {
  constexpr int EM = BUCKET_EM;
  double v[EM];
  double mn = DINF, mx = -DINF;
#pragma unroll
  for (int i = 0; i < EM; i++) {
    const int idx = beg + i * 32 + lane;
    v[i] = DINF;
    if (idx < end) {
      const double2 p = __ldg(&xy[idx]);
      v[i] = pair_d2(qx, qy, p.x, p.y);
    }
    if (v[i] < DINF) {
      mn = fmin(mn, v[i]);
      mx = fmax(mx, v[i]);
    }
  }
  mn = warp_min(mn);
  mx = warp_max(mx);
  int total = 0;
#pragma unroll
  for (int i = 0; i < EM; i++) total += __popc(__ballot_sync(FULL, v[i] < DINF));
  const int need = min(k + 1, total);
  // level 1: 32 equal-width bins over [mn, mx]
  const double sc1 = mx > mn ? 32.0 / (mx - mn) : 0.0;
  int bin[EM];
#pragma unroll
  for (int i = 0; i < EM; i++)
    bin[i] = v[i] < DINF ? min(31, (int)((v[i] - mn) * sc1)) : 32;
  int before1;
  const int b1 = bucket_cut<EM>(bin, need, sc->hist, lane, before1);
  // level 2: 32 bins over the values of bin b1
  double mn2 = DINF, mx2 = -DINF;
#pragma unroll
  for (int i = 0; i < EM; i++)
    if (bin[i] == b1) {
      mn2 = fmin(mn2, v[i]);
      mx2 = fmax(mx2, v[i]);
    }
  mn2 = warp_min(mn2);
  mx2 = warp_max(mx2);
  const double sc2 = mx2 > mn2 ? 32.0 / (mx2 - mn2) : 0.0;
  int sub[EM];
#pragma unroll
  for (int i = 0; i < EM; i++) sub[i] = bin[i] == b1 ? min(31, (int)((v[i] - mn2) * sc2)) : 32;
  int before2;
  const int b2 = bucket_cut<EM>(sub, need - before1, sc->hist, lane, before2);
  // compact the cut into shared memory
  const unsigned lt = (1u << lane) - 1u;
  int c = 0;
  bool overflow = false;
#pragma unroll
  for (int i = 0; i < EM; i++) {
    const bool keep = bin[i] < b1 || (bin[i] == b1 && sub[i] <= b2);
    const unsigned m = __ballot_sync(FULL, keep);
    const int slot = c + __popc(m & lt);
    if (keep && slot < 64) {
      sc->d[slot] = v[i];
      sc->pos[slot] = beg + i * 32 + lane;
    }
    c += __popc(m);
  }
  overflow = c > 64;
  __syncwarp();
  if (overflow) {  // pathological distribution (heavy ties): plain chunked pass
    scan_range<1>(L, k, beg, end, qx, qy, me, xy, ids, lane);
    return;
  }
  // exact (d2, id) selection among the c candidates of the cut
  double d0 = DINF, d1 = DINF;
  long long i0 = IDMAX, i1 = IDMAX;
  if (lane < c) {
    i0 = __ldg(&ids[sc->pos[lane]]);
    d0 = i0 == me ? DINF : sc->d[lane];
    if (i0 == me) i0 = IDMAX;
  }
  if (lane + 32 < c) {
    i1 = __ldg(&ids[sc->pos[lane + 32]]);
    d1 = i1 == me ? DINF : sc->d[lane + 32];
    if (i1 == me) i1 = IDMAX;
  }
  __syncwarp();
  double cd[1] = {d0};
  long long ci[1] = {i0};
  bitonic_sort<1>(cd, ci, lane);
  L.d[0] = cd[0];
  L.id[0] = ci[0];
  if (c > 32) {
    unsigned m = __ballot_sync(FULL, d1 < DINF);
    if (__popc(m) <= 12) {
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        list_insert<1>(L, __shfl_sync(FULL, d1, src), __shfl_sync(FULL, i1, src), lane);
      }
    } else {
      cd[0] = d1;
      ci[0] = i1;
      bitonic_sort<1>(cd, ci, lane);
      bitonic_merge_into<1>(L, cd, ci, lane);
    }
  }
}

// engine.py:421-431 coarsest_levels: the coarsest quadrant aligned with the
// cursor (first code for right walks, last code for left walks)
__device__ __forceinline__ int coarsest_level(long long p, int dir, int l_deep) {
  const long long a = p + (dir ? 0 : 1);
  if (a == 0) return 0;
  const int tz2 = (__ffsll(a) - 1) >> 1;
  return l_deep - min(tz2, l_deep);
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
                                            const double2* __restrict__ xy,
                                            const long long* __restrict__ ids, Region r, int l_deep,
                                            int lvl, long long qc, double thr, double qx, double qy,
                                            long long me) {
  const int sh = 2 * (l_deep - lvl);
  const long long lo = qc << sh, hi = (qc + 1) << sh;
  const int l0 = z_map[lo], l1 = z_map[hi - 1];
  for (int li = l0; li <= l1; li++) {
    const int b = cell_start[li], e = cell_start[li + 1];
    for (int i = b; i < e; i++) {
      const double2 p = xy[i];
      const long long c = encode(p.x, p.y, r, l_deep);
      if (c >= lo && c < hi && ids[i] != me && pair_d2(qx, qy, p.x, p.y) < thr) return true;
    }
  }
  return false;
}

// engine.py:396-503 navigate for one query and one direction, run by one
// lane: returns the assigned leaf ordinal or -1 when the direction is
// exhausted.  thr is the query's k-th d2 (+inf while the list is not full).
__device__ __forceinline__ int navigate(const SearchArgs& a, int l_deep, int dir, long long& cursor,
                                        double thr, double qx, double qy, long long me,
                                        uint32_t& prunes, uint32_t& viol) {
  const long long n_codes = 1LL << (2 * l_deep);
  const long long sign = dir ? 1 : -1;
  long long pos = cursor;
  if (dir ? pos >= n_codes : pos < 0) return -1;
  const bool full = thr < DINF;  // engine.py:415: thr = MAXDIST iff the list is full
  int lvl = full ? coarsest_level(pos, dir, l_deep) : l_deep;
  for (;;) {
    const int delta = l_deep - lvl;
    const uint32_t qc = (uint32_t)(pos >> (2 * delta));
    const double md2 = full ? mindist2_cell(lvl, qc, a.r, qx, qy) : 0.0;
    if (md2 > thr) {  // prune (engine.py:447-460; strict, see the header)
      prunes++;
      if (a.audit && audit_quadrant(a.z_map, a.cell_start, a.xy, a.ids, a.r, l_deep, lvl, qc, thr,
                                    qx, qy, me))
        viol++;
      pos += sign << (2 * delta);
    } else if (lvl < l_deep) {  // descend (engine.py:462-465)
      lvl++;
      continue;
    } else {  // resolve through z_map (engine.py:467-487)
      const int li = __ldg(&a.z_map[pos]);
      const long long key = __ldg(&a.leaf_key[li]);
      const long long after = dir ? key + (long long)__ldg(&a.leaf_span[li]) : key - 1;
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
template <int KPL, int B>
__global__ void __launch_bounds__(32 * WARPS_PER_CTA) k_search(const SearchArgs a) {
  constexpr int N = 32 * KPL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* sd = reinterpret_cast<double*>(smem_raw) + (size_t)w * B * N;
  long long* si = reinterpret_cast<long long*>(smem_raw) + (size_t)WARPS_PER_CTA * B * N +
                  (size_t)w * B * N;
  BucketScratch* bsc = reinterpret_cast<BucketScratch*>(
                          smem_raw + (size_t)WARPS_PER_CTA * B * N * 16) + w;
  const int64_t t0 = ((int64_t)blockIdx.x * WARPS_PER_CTA + w) * B;
  if (t0 >= a.nq) return;
  const int nb = (int)((a.nq - t0) < B ? (a.nq - t0) : B);
  const int l_deep = __ldg(&a.scalars[0]);
  const int k = a.k;

  // per-lane query state (lane q < nb owns query t0 + q)
  const bool mine = lane < nb;
  uint32_t q = 0, own = 0;
  double qx = 0.0, qy = 0.0, thr = DINF;
  long long me = 0, cur_l = -1, cur_r = 0;
  uint32_t evals = 0, prunes = 0, viol = 0, calls_l = 0, calls_r = 0;
  bool act_l = false, act_r = false;
  if (mine) {
    q = __ldg(&a.q_order[t0 + lane]);
    qx = __ldg(&a.qx[q]);
    qy = __ldg(&a.qy[q]);
    me = __ldg(&a.qi[q]);
    own = __ldg(&a.q_leaf[q]);
    cur_l = (long long)__ldg(&a.leaf_key[own]) - 1;
    cur_r = (long long)__ldg(&a.leaf_key[own]) + (long long)__ldg(&a.leaf_span[own]);
    act_l = act_r = true;
    if (__ldg(&a.cell_start[own + 1]) > __ldg(&a.cell_start[own])) emit_task(a, 0, 0, own);
  }

  // first_iteration: every query against its own leaf
  for (int j = 0; j < nb; j++) {
    const double jx = __shfl_sync(FULL, qx, j), jy = __shfl_sync(FULL, qy, j);
    const long long jme = __shfl_sync(FULL, me, j);
    const uint32_t jown = __shfl_sync(FULL, own, j);
    List<KPL> L;
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      L.d[s] = DINF;
      L.id[s] = IDMAX;
    }
    const int b = __ldg(&a.cell_start[jown]), e = __ldg(&a.cell_start[jown + 1]);
    if (e > b) {  // rows with 0 candidates are dropped (engine.py:334-338)
      if constexpr (KPL == 1) {
        if (e - b > 32) {
          const int cut = min(e, b + 32 * BUCKET_EM);
          own_leaf_bucket(L, k, b, cut, jx, jy, jme, a.xy, a.ids, lane, bsc);
          if (cut < e) scan_range<KPL>(L, k, cut, e, jx, jy, jme, a.xy, a.ids, lane);
        } else {
          scan_range<KPL>(L, k, b, e, jx, jy, jme, a.xy, a.ids, lane);
        }
      } else {
        scan_range<KPL>(L, k, b, e, jx, jy, jme, a.xy, a.ids, lane);
      }
      if (lane == j) evals += (uint32_t)(e - b);
    }
    double kd;
    long long ki;
    list_kth<KPL>(L, k, kd, ki);
    if (lane == j) thr = kd;
    list_store<KPL>(L, sd + j * N, si + j * N, lane);
  }
  __syncwarp();

  // direction loop, left first (engine.py:645-681)
  bool go_right = false;
  if (a.debug_phase == 1) act_l = act_r = false;
  while (__any_sync(FULL, act_l || act_r)) {
    const bool act = go_right ? act_r : act_l;
    int li = -1;
    if (act) {
      long long cur = go_right ? cur_r : cur_l;
      li = navigate(a, l_deep, go_right ? 1 : 0, cur, thr, qx, qy, me, prunes, viol);
      if (go_right) {
        calls_r++;
        cur_r = cur;
        act_r = li >= 0;
      } else {
        calls_l++;
        cur_l = cur;
        act_l = li >= 0;
      }
      if (li >= 0) emit_task(a, go_right ? 2 : 1, (go_right ? calls_r : calls_l) - 1, li);
    }
    // update_nn_lists: merge each assigned leaf into its query's list
    unsigned pend = __ballot_sync(FULL, li >= 0);
    while (pend) {
      const int j = __ffs(pend) - 1;
      pend &= pend - 1;
      const int jl = __shfl_sync(FULL, li, j);
      const double jx = __shfl_sync(FULL, qx, j), jy = __shfl_sync(FULL, qy, j);
      const long long jme = __shfl_sync(FULL, me, j);
      const int b = __ldg(&a.cell_start[jl]), e = __ldg(&a.cell_start[jl + 1]);
      List<KPL> L;
      list_load<KPL>(L, sd + j * N, si + j * N, lane);
      scan_range<KPL>(L, k, b, e, jx, jy, jme, a.xy, a.ids, lane);
      list_store<KPL>(L, sd + j * N, si + j * N, lane);
      double kd;
      long long ki;
      list_kth<KPL>(L, k, kd, ki);
      if (lane == j) {
        thr = kd;
        evals += (uint32_t)(e - b);
      }
    }
    __syncwarp();
    go_right = !go_right;
  }

  // _emit: canonical order already; sqrt correctly rounded (engine.py:706)
  for (int j = 0; j < nb; j++) {
    const uint32_t jq = __shfl_sync(FULL, q, j);
    const uint32_t row = __ldg(&a.q_row[jq]);
    List<KPL> L;
    list_load<KPL>(L, sd + j * N, si + j * N, lane);
    int len = 0;
#pragma unroll
    for (int s = 0; s < KPL; s++) {
      const int e = (s << 5) | lane;
      const bool ok = e < k && L.d[s] < DINF;
      len += __popc(__ballot_sync(FULL, ok));
      if (ok) {
        a.out_nids[(int64_t)row * k + e] = L.id[s];
        a.out_dist[(int64_t)row * k + e] = __dsqrt_rn(L.d[s]);
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

// ---------------------------------------------------------------------------
// Thread-per-query search for k <= 32 (the paper's distComp mapping, "CTA
// per leaf, thread per query", re-planned for one warp):
// lane q owns query t0+q of the leaf-grouped order, so the lanes of a warp
// mostly read the same leaf objects (broadcast loads).  Each query keeps its
// k best (d2, id) UNSORTED in shared memory with the current maximum (the
// k-th neighbour) cached in registers; it is sorted once, at emission.
//
// Own leaf: two passes.  Pass A histograms the query's candidates into 64
// monotone log-spaced bins of t = d2 / R2 (R2 = squared leaf diagonal;
// float exponent + 2 mantissa bits); the first bin whose prefix count
// reaches k+1 (k plus room for the issuer) is the cut.  Pass B offers only
// candidates at or below the cut.  Binning is monotone in d2, so everything
// above the cut is strictly farther than everything kept: exact.
constexpr int TPQ_WARPS = 4;
constexpr int TPQ_BINS = 64;
constexpr int TPQ_STRIDE = 33;  // padded slot stride: conflict-free rows and columns

struct TpqList {
  double* d;     // [slot * 33 + lane]
  long long* id;
  int k, cnt, kpos;
  double kd;
  long long ki;
};

__device__ __forceinline__ void tpq_find_max(TpqList& L, int lane) {
  L.kd = -1.0;
  L.ki = -1;
  L.kpos = 0;
  for (int s = 0; s < L.k; s++) {
    const double d = L.d[s * TPQ_STRIDE + lane];
    const long long i = L.id[s * TPQ_STRIDE + lane];
    if (key_less(L.kd, L.ki, d, i)) {
      L.kd = d;
      L.ki = i;
      L.kpos = s;
    }
  }
}

// offer (d2, id) to the list (caller guarantees d2 < +inf and id != issuer)
__device__ __forceinline__ void tpq_offer(TpqList& L, double d2, long long id, int lane) {
  if (L.cnt < L.k) {
    L.d[L.cnt * TPQ_STRIDE + lane] = d2;
    L.id[L.cnt * TPQ_STRIDE + lane] = id;
    if (++L.cnt == L.k) tpq_find_max(L, lane);
  } else if (key_less(d2, id, L.kd, L.ki)) {
    L.d[L.kpos * TPQ_STRIDE + lane] = d2;
    L.id[L.kpos * TPQ_STRIDE + lane] = id;
    tpq_find_max(L, lane);
  }
}

// the k-th neighbour's d2 while the list is full, +inf before (engine.py:415)
__device__ __forceinline__ double tpq_thr(const TpqList& L) { return L.cnt == L.k ? L.kd : DINF; }

__device__ __forceinline__ int tpq_bin(double d2, double inv_r2) {
  const float t = (float)(d2 * inv_r2);
  const int key = (int)(__float_as_uint(t) >> 21) - ((127 - 16) << 2);
  return min(max(key, 0), TPQ_BINS - 1);
}

// merge one leaf [b, e) into the list (update_nn_lists, engine.py:376-393)
__device__ __forceinline__ void tpq_scan(TpqList& L, int b, int e, double qx, double qy,
                                         long long me, const double2* __restrict__ xy,
                                         const long long* __restrict__ ids, int lane) {
  for (int j = b; j < e; j++) {
    const double2 p = __ldg(&xy[j]);
    const double d2 = pair_d2(qx, qy, p.x, p.y);
    if (d2 <= tpq_thr(L) && d2 < DINF) {
      const long long id = __ldg(&ids[j]);
      if (id != me) tpq_offer(L, d2, id, lane);
    }
  }
}

__global__ void __launch_bounds__(32 * TPQ_WARPS) k_search_tpq(const SearchArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k = a.k;
  const size_t per_warp = (size_t)max(k * TPQ_STRIDE * 16, TPQ_BINS * 32 * 4);
  unsigned char* base = smem_raw + (size_t)w * per_warp;
  const int64_t t = ((int64_t)blockIdx.x * TPQ_WARPS + w) * 32 + lane;
  if (((int64_t)blockIdx.x * TPQ_WARPS + w) * 32 >= a.nq) return;
  const bool mine = t < a.nq;
  const int l_deep = __ldg(&a.scalars[0]);

  TpqList L;
  L.d = reinterpret_cast<double*>(base);
  L.id = reinterpret_cast<long long*>(base + (size_t)k * TPQ_STRIDE * 8);
  L.k = k;
  L.cnt = 0;
  L.kpos = 0;
  L.kd = DINF;
  L.ki = IDMAX;
  uint32_t* hist = reinterpret_cast<uint32_t*>(base);  // aliases the list during pass A

  uint32_t q = 0, own = 0;
  double qx = 0.0, qy = 0.0;
  long long me = 0, cur_l = -1, cur_r = 0;
  uint32_t evals = 0, prunes = 0, viol = 0, calls_l = 0, calls_r = 0;
  bool act_l = false, act_r = false;
  int ob = 0, oe = 0;
  if (mine) {
    q = __ldg(&a.q_order[t]);
    qx = __ldg(&a.qx[q]);
    qy = __ldg(&a.qy[q]);
    me = __ldg(&a.qi[q]);
    own = __ldg(&a.q_leaf[q]);
    const long long key = __ldg(&a.leaf_key[own]);
    cur_l = key - 1;
    cur_r = key + (long long)__ldg(&a.leaf_span[own]);
    act_l = act_r = true;
    ob = __ldg(&a.cell_start[own]);
    oe = __ldg(&a.cell_start[own + 1]);
    evals = (uint32_t)(oe - ob);  // first_iteration row (0 when the leaf is empty)
    if (oe > ob) emit_task(a, 0, 0, own);
  }

  // ---- first_iteration: own leaf, pass A (histogram) --------------------
  const int n_own = oe - ob;
  int cut = TPQ_BINS - 1;
  double inv_r2 = 0.0;
  if (n_own > k + 1) {
    // R2 = squared diagonal of the own leaf's quadrant (scale only)
    const int lvl = l_deep - ((31 - __clz(__ldg(&a.leaf_span[own]))) >> 1);
    const double lw = a.r.w * pow2_neg(lvl), lh = a.r.h * pow2_neg(lvl);
    const double r2 = lw * lw + lh * lh;
    inv_r2 = r2 > 0.0 ? 1.0 / r2 : 0.0;
#pragma unroll 4
    for (int bI = 0; bI < TPQ_BINS; bI++) hist[bI * 32 + lane] = 0;
    for (int j = ob; j < oe; j++) {
      const double2 p = __ldg(&a.xy[j]);
      const int bI = tpq_bin(pair_d2(qx, qy, p.x, p.y), inv_r2);
      hist[bI * 32 + lane] += 1;
    }
    uint32_t cum = 0;
    for (cut = 0; cut < TPQ_BINS - 1; cut++) {
      cum += hist[cut * 32 + lane];
      if (cum >= (uint32_t)(k + 1)) break;
    }
  }
  __syncwarp();
  // ---- pass B: offer the candidates at or below the cut ------------------
  for (int j = ob; j < oe; j++) {
    const double2 p = __ldg(&a.xy[j]);
    const double d2 = pair_d2(qx, qy, p.x, p.y);
    if (d2 < DINF && (cut == TPQ_BINS - 1 || tpq_bin(d2, inv_r2) <= cut) && d2 <= tpq_thr(L)) {
      const long long id = __ldg(&a.ids[j]);
      if (id != me) tpq_offer(L, d2, id, lane);
    }
  }

  // ---- direction loop, left first (engine.py:645-681) ---------------------
  bool go_right = false;
  if (a.debug_phase == 1) act_l = act_r = false;
  while (__any_sync(FULL, act_l || act_r)) {
    const bool act = go_right ? act_r : act_l;
    if (act) {
      long long cur = go_right ? cur_r : cur_l;
      const int li = navigate(a, l_deep, go_right ? 1 : 0, cur, tpq_thr(L), qx, qy, me, prunes, viol);
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
        const int b = __ldg(&a.cell_start[li]), e = __ldg(&a.cell_start[li + 1]);
        evals += (uint32_t)(e - b);
        tpq_scan(L, b, e, qx, qy, me, a.xy, a.ids, lane);
      }
    }
    go_right = !go_right;
  }

  // ---- _emit: sort each list by (d2, id), then write rows warp-wide ------
  for (int i = 1; i < L.cnt; i++) {
    const double d = L.d[i * TPQ_STRIDE + lane];
    const long long id = L.id[i * TPQ_STRIDE + lane];
    int p = i;
    while (p > 0) {
      const double pd = L.d[(p - 1) * TPQ_STRIDE + lane];
      const long long pi = L.id[(p - 1) * TPQ_STRIDE + lane];
      if (!key_less(d, id, pd, pi)) break;
      L.d[p * TPQ_STRIDE + lane] = pd;
      L.id[p * TPQ_STRIDE + lane] = pi;
      p--;
    }
    L.d[p * TPQ_STRIDE + lane] = d;
    L.id[p * TPQ_STRIDE + lane] = id;
  }
  __syncwarp();
  const int64_t rem = a.nq - (t - lane);
  const int nb = rem < 32 ? (int)rem : 32;
  const uint32_t my_row = mine ? __ldg(&a.q_row[q]) : 0;
  for (int j = 0; j < nb; j++) {
    const uint32_t row = __shfl_sync(FULL, my_row, j);
    const int cnt = __shfl_sync(FULL, L.cnt, j);
    if (lane < cnt) {
      a.out_nids[(int64_t)row * k + lane] = L.id[lane * TPQ_STRIDE + j];
      a.out_dist[(int64_t)row * k + lane] = __dsqrt_rn(L.d[lane * TPQ_STRIDE + j]);
    }
    if (lane == 0) a.out_len[row] = cnt;
  }
  if (mine) {
    QueryStats st;
    st.evals = evals;
    st.prunes = prunes;
    st.nav_left = (uint16_t)min(calls_l, 65535u);
    st.nav_right = (uint16_t)min(calls_r, 65535u);
    st.violations = viol;
    a.stats[t] = st;
  }
}

constexpr int HIST_SMEM = 1024;

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
    if (s.nav_left < HIST_SMEM) atomicAdd(&hl[s.nav_left], 1u);
    else if (s.nav_left < hist_cap) atomicAdd(&hist_l[s.nav_left], 1u);
    if (s.nav_right < HIST_SMEM) atomicAdd(&hr[s.nav_right], 1u);
    else if (s.nav_right < hist_cap) atomicAdd(&hist_r[s.nav_right], 1u);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ev += __shfl_xor_sync(FULL, ev, o);
    pr += __shfl_xor_sync(FULL, pr, o);
    vi += __shfl_xor_sync(FULL, vi, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (ev) atomicAdd(&tot[0], ev);
    if (pr) atomicAdd(&tot[1], pr);
    if (vi) atomicAdd(&tot[2], vi);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HIST_SMEM && i < hist_cap; i += blockDim.x) {
    if (hl[i]) atomicAdd(&hist_l[i], hl[i]);
    if (hr[i]) atomicAdd(&hist_r[i], hr[i]);
  }
}

__global__ void k_rows_compact(const int32_t* __restrict__ len, const long long* __restrict__ nids,
                               const double* __restrict__ dist, int64_t nq, int k,
                               const int64_t* __restrict__ off, long long* __restrict__ c_nids,
                               double* __restrict__ c_dist) {
  const int64_t total = nq * (int64_t)k;
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

template <int KPL, int B>
int launch_batched(const SearchArgs& a, cudaStream_t s) {
  constexpr int N = 32 * KPL;
  const size_t smem = (size_t)WARPS_PER_CTA * B * N * (sizeof(double) + sizeof(long long)) +
                      (size_t)WARPS_PER_CTA * sizeof(BucketScratch);
  static bool configured = false;
  if (!configured) {
    MKNN_CUDA_OK(cudaFuncSetAttribute(k_search<KPL, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    configured = true;
  }
  const int64_t per_cta = (int64_t)WARPS_PER_CTA * B;
  const unsigned blocks = (unsigned)((a.nq + per_cta - 1) / per_cta);
  MKNN_LAUNCH k_search<KPL, B><<<blocks, 32 * WARPS_PER_CTA, smem, s>>>(a);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

int launch_tpq(const SearchArgs& a, cudaStream_t s) {
  const size_t per_warp = (size_t)std::max(a.k * TPQ_STRIDE * 16, TPQ_BINS * 32 * 4);
  const size_t smem = per_warp * TPQ_WARPS;
  static size_t configured = 0;
  if (smem > configured) {
    MKNN_CUDA_OK(cudaFuncSetAttribute(k_search_tpq, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    configured = smem;
  }
  const int64_t per_cta = (int64_t)TPQ_WARPS * 32;
  const unsigned blocks = (unsigned)((a.nq + per_cta - 1) / per_cta);
  MKNN_LAUNCH k_search_tpq<<<blocks, 32 * TPQ_WARPS, smem, s>>>(a);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

int search_launch(const SearchArgs& a, cudaStream_t s) {
  if (a.nq == 0) return 0;
  if (a.k <= 32 && !a.force_warp) return launch_tpq(a, s);
  if (a.k <= 32) return launch_batched<1, 16>(a, s);
  if (a.k <= 64) return launch_batched<2, 8>(a, s);
  if (a.k <= 128) return launch_batched<4, 4>(a, s);
  if (a.k <= 256) return launch_batched<8, 2>(a, s);
  if (a.k <= 512) return launch_batched<16, 1>(a, s);
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

int rows_compact(const int32_t* len, const long long* nids, const double* dist, int64_t nq, int k,
                 int64_t* offsets, long long* c_nids, double* c_dist, void* scratch,
                 cudaStream_t s) {
  int rc = exclusive_scan_i32_to_i64(len, offsets, nq, scratch, s);
  if (rc) return rc;
  if (nq == 0) return 0;
  const int64_t total = nq * (int64_t)k;
  int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
  MKNN_LAUNCH k_rows_compact<<<(unsigned)blocks, 256, 0, s>>>(len, nids, dist, nq, k, offsets, c_nids, c_dist);
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
