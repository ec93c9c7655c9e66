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
        if (sw) {
          const double td = d[s];
          d[s] = d[t];
          d[t] = td;
          const long long ti = id[s];
          id[s] = id[t];
          id[t] = ti;
        }
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
      if (take) {
        d[s] = pd;
        id[s] = pi;
      }
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
    if (key_less(rd, ri, L.d[s], L.id[s])) {
      L.d[s] = rd;
      L.id[s] = ri;
    }
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
    if (gt[s]) {
      L.d[s] = gprev ? pd[s] : kd;
      L.id[s] = gprev ? pi[s] : ki;
    }
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
      bitonic_merge_into<KPL>(L, cd, ci, lane);
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

// engine.py:529-554 _audit_prune_events for one pruned quadrant: does it
// hold an object (not the issuer) strictly closer than thr?
__device__ __noinline__ bool audit_quadrant(const int32_t* __restrict__ z_map,
                                            const int32_t* __restrict__ cell_start,
                                            const double2* __restrict__ xy,
                                            const long long* __restrict__ ids, Region r, int l_deep,
                                            int lvl, long long qc, double thr, double qx, double qy,
                                            long long me, int lane) {
  const int sh = 2 * (l_deep - lvl);
  const long long lo = qc << sh, hi = (qc + 1) << sh;
  const int l0 = z_map[lo], l1 = z_map[hi - 1];
  bool bad = false;
  for (int li = l0; li <= l1; li++) {
    const int b = cell_start[li], e = cell_start[li + 1];
    for (int i = b + lane; i < e; i += 32) {
      const double2 p = xy[i];
      const long long c = encode(p.x, p.y, r, l_deep);
      if (c >= lo && c < hi && ids[i] != me && pair_d2(qx, qy, p.x, p.y) < thr) bad = true;
    }
  }
  return __any_sync(FULL, bad);
}

// engine.py:396-503 navigate for one query and one direction: returns the
// assigned leaf ordinal or -1 when the direction is exhausted.
__device__ __forceinline__ int navigate(const SearchArgs& a, int l_deep, int dir, long long& cursor,
                                        double thr, double qx, double qy, long long me,
                                        uint32_t& prunes, uint32_t& viol, int lane) {
  const long long n_codes = 1LL << (2 * l_deep);
  const long long sign = dir ? 1 : -1;
  long long pos = cursor;
  if (dir ? pos >= n_codes : pos < 0) return -1;
  const bool full = thr < DINF;  // engine.py:415: thr = MAXDIST iff the list is full
  int lvl = full ? coarsest_level(pos, dir, l_deep) : l_deep;
  for (;;) {
    const int delta = l_deep - lvl;
    const uint32_t qc = (uint32_t)(pos >> (2 * delta));
    const double md2 = mindist2_cell(lvl, qc, a.r, qx, qy);
    if (md2 > thr) {  // prune (engine.py:447-460, strict)
      prunes++;
      if (a.audit && audit_quadrant(a.z_map, a.cell_start, a.xy, a.ids, a.r, l_deep, lvl, qc, thr, qx,
                                   qy, me, lane))
        viol++;
      pos += sign << (2 * delta);
    } else if (lvl < l_deep) {  // descend (engine.py:462-465)
      lvl++;
      continue;
    } else {  // resolve through z_map (engine.py:467-487)
      const int li = a.z_map[pos];
      const long long key = a.leaf_key[li];
      const long long after = dir ? key + (long long)a.leaf_span[li] : key - 1;
      if (a.cell_start[li + 1] > a.cell_start[li]) {
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
__global__ void __launch_bounds__(32 * WARPS_PER_CTA) k_search(const SearchArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * WARPS_PER_CTA + (threadIdx.x >> 5);
  if (t >= a.nq) return;
  const int l_deep = a.scalars[0];
  const int k = a.k;
  const uint32_t q = a.q_order[t];
  const double qx = a.qx[q], qy = a.qy[q];
  const long long me = a.qi[q];
  const uint32_t own = a.q_leaf[q];

  List<KPL> L;
#pragma unroll
  for (int s = 0; s < KPL; s++) {
    L.d[s] = DINF;
    L.id[s] = IDMAX;
  }
  uint32_t evals = 0, prunes = 0, viol = 0;

  // first_iteration: the own leaf (rows with 0 candidates are dropped)
  {
    const int b = a.cell_start[own], e = a.cell_start[own + 1];
    if (e > b) {
      evals += (uint32_t)(e - b);
      scan_range<KPL>(L, k, b, e, qx, qy, me, a.xy, a.ids, lane);
    }
  }
  // direction loop, left first (engine.py:645-681); per-direction state is
  // kept in scalars (no dynamically indexed arrays -> no local memory)
  long long cur_l = (long long)a.leaf_key[own] - 1;
  long long cur_r = (long long)a.leaf_key[own] + (long long)a.leaf_span[own];
  bool act_l = true, act_r = true;
  uint32_t calls_l = 0, calls_r = 0;
  bool go_right = false;
  while (act_l || act_r) {
    if (go_right ? act_r : act_l) {
      double kd;
      long long ki;
      list_kth<KPL>(L, k, kd, ki);
      long long cur = go_right ? cur_r : cur_l;
      const int li = navigate(a, l_deep, go_right ? 1 : 0, cur, kd, qx, qy, me, prunes, viol, lane);
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
        const int b = a.cell_start[li], e = a.cell_start[li + 1];
        evals += (uint32_t)(e - b);
        scan_range<KPL>(L, k, b, e, qx, qy, me, a.xy, a.ids, lane);
      }
    }
    go_right = !go_right;
  }

  // _emit: canonical order already; sqrt correctly rounded (engine.py:706)
  const uint32_t row = a.q_row[q];
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
  if (lane == 0) {
    a.out_len[row] = len;
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

int search_launch(const SearchArgs& a, cudaStream_t s) {
  if (a.nq == 0) return 0;
  const unsigned blocks = (unsigned)((a.nq + WARPS_PER_CTA - 1) / WARPS_PER_CTA);
  const int threads = 32 * WARPS_PER_CTA;
  if (a.k <= 32) k_search<1><<<blocks, threads, 0, s>>>(a);
  else if (a.k <= 64) k_search<2><<<blocks, threads, 0, s>>>(a);
  else if (a.k <= 128) k_search<4><<<blocks, threads, 0, s>>>(a);
  else if (a.k <= 256) k_search<8><<<blocks, threads, 0, s>>>(a);
  else if (a.k <= 512) k_search<16><<<blocks, threads, 0, s>>>(a);
  else return fail_msg(E_UNSUPPORTED, "k > 512 is not supported by the device top-k");
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

int stats_reduce(const QueryStats* st, int64_t nq, unsigned long long* dev_tot, uint32_t* hist_l,
                 uint32_t* hist_r, int hist_cap, cudaStream_t s) {
  if (nq == 0) return 0;
  int64_t blocks = (nq + 256 * 16 - 1) / (256 * 16);
  blocks = std::min<int64_t>(std::max<int64_t>(blocks, 1), 148 * 4);
  k_stats_reduce<<<(unsigned)blocks, 256, 0, s>>>(st, nq, dev_tot, hist_l, hist_r, hist_cap);
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
  k_rows_compact<<<(unsigned)blocks, 256, 0, s>>>(len, nids, dist, nq, k, offsets, c_nids, c_dist);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

}  // namespace mknn
