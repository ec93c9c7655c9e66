/*
 * mknn_oracle.c -- CPU restatement of the reference k-NN tick path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the package
 * paper_1412_6170_b200 or libmknn_b200.so) links, loads or calls this file.
 * It is used by tests/ (as the parity checker), by __graft_entry__.smoke()
 * (as the checker) and by bench.py's cpu_baseline / --impl reference leg
 * (as the timed CPU port of the reference algorithm).
 *
 * Parity pinning: every function below is checked against golden vectors
 * produced by the real reference package (tests/golden/make_golden.py, which
 * imports /root/reference/pkg/src/mknn) in tests/test_oracle_golden.py.
 *
 * All citations are relative to /root/reference/pkg/src/mknn/.
 *
 * Arithmetic contract: every fp64 expression is
 * evaluated as separate IEEE operations in the reference's order.  Build
 * with -ffp-contract=off so no FMA is formed.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_EXPORT __attribute__((visibility("default")))

typedef struct {
    double x_lo, y_lo, x_hi, y_hi;
} or_rect;

/* ------------------------------------------------------------------ */
/* geometry.py                                                          */
/* ------------------------------------------------------------------ */

/* geometry.py:75-83 spread_bits */
static inline uint64_t spread_bits(uint64_t v) {
    v &= 0xFFFFFFFFull;
    v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
    v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
    v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    v = (v | (v << 1)) & 0x5555555555555555ull;
    return v;
}

/* geometry.py:86-94 compact_bits */
static inline uint64_t compact_bits(uint64_t v) {
    v &= 0x5555555555555555ull;
    v = (v | (v >> 1)) & 0x3333333333333333ull;
    v = (v | (v >> 2)) & 0x0F0F0F0F0F0F0F0Full;
    v = (v | (v >> 4)) & 0x00FF00FF00FF00FFull;
    v = (v | (v >> 8)) & 0x0000FFFF0000FFFFull;
    v = (v | (v >> 16)) & 0x00000000FFFFFFFFull;
    return v;
}

/* geometry.py:105-129 cell_coords: tx = (x - x_lo) / width, then
 * clip(floor(tx * 2^level), 0, 2^level - 1).  Zero width gives 0. */
static inline int64_t cell_coord(double v, double lo, double width, int level) {
    double n = (double)(1ll << level);
    double t = (width > 0) ? (v - lo) / width : 0.0;
    double c = floor(t * n);
    if (c < 0) c = 0;
    if (c > n - 1) c = n - 1;
    return (int64_t)c;
}

/* geometry.py:132-135 encode_points (+ interleave 97-98) */
OR_EXPORT int64_t or_encode(double x, double y, const or_rect *r, int level) {
    double w = r->x_hi - r->x_lo, h = r->y_hi - r->y_lo;
    int64_t cx = cell_coord(x, r->x_lo, w, level);
    int64_t cy = cell_coord(y, r->y_lo, h, level);
    return (int64_t)(spread_bits((uint64_t)cx) | (spread_bits((uint64_t)cy) << 1));
}

/* geometry.py:166-181 cell_bounds_arrays + 189-193 min_dist2_point_cells */
static inline double mindist2_cell(int level, int64_t code, const or_rect *r,
                                   double qx, double qy) {
    double w = r->x_hi - r->x_lo, h = r->y_hi - r->y_lo;
    int64_t cx = (int64_t)compact_bits((uint64_t)code);
    int64_t cy = (int64_t)compact_bits((uint64_t)code >> 1);
    double xl = r->x_lo + ldexp((double)cx, -level) * w;
    double yl = r->y_lo + ldexp((double)cy, -level) * h;
    double xh = r->x_lo + ldexp((double)(cx + 1), -level) * w;
    double yh = r->y_lo + ldexp((double)(cy + 1), -level) * h;
    double dx = fmax(fmax(xl - qx, qx - xh), 0.0);
    double dy = fmax(fmax(yl - qy, qy - yh), 0.0);
    return dx * dx + dy * dy;
}

/* geometry.py:203-212 squared_dist_matrix, one pair (three roundings) */
static inline double pair_d2(double qx, double qy, double ox, double oy) {
    double dx = qx - ox;
    double dy = qy - oy;
    return dx * dx + dy * dy;
}

/* ------------------------------------------------------------------ */
/* canonical (d2, id) top-k list                                        */
/* ------------------------------------------------------------------ */

typedef struct {
    double d2;
    int64_t id;
} cand_t;

static inline int cand_lt(double ad, int64_t ai, double bd, int64_t bi) {
    return ad < bd || (ad == bd && ai < bi);
}

/* Insert (d2, id) into a (d2, id)-ascending list of capacity k holding *cnt
 * entries.  +inf never qualifies (oracle.py:91 drops non-finite entries). */
static inline void list_insert(cand_t *L, int k, int *cnt, double d2, int64_t id) {
    if (!(d2 < INFINITY)) return;
    int c = *cnt;
    if (c == k && !cand_lt(d2, id, L[k - 1].d2, L[k - 1].id)) return;
    int p = (c == k) ? k - 1 : c;
    while (p > 0 && cand_lt(d2, id, L[p - 1].d2, L[p - 1].id)) {
        L[p] = L[p - 1];
        p--;
    }
    L[p].d2 = d2;
    L[p].id = id;
    if (c < k) *cnt = c + 1;
}

/* stable argsort of int64 keys (LSD radix, 16-bit digits) */
static void stable_argsort_i64(const int64_t *key, int64_t n, int64_t *perm) {
    int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * 65536);
    for (int64_t i = 0; i < n; i++) perm[i] = i;
    for (int pass = 0; pass < 4; pass++) {
        int sh = 16 * pass;
        int all_zero = 1;
        for (int64_t i = 0; i < n; i++) {
            uint64_t u = (uint64_t)key[i] ^ 0x8000000000000000ull;
            if ((u >> sh) >> 16) { all_zero = 0; }
        }
        memset(cnt, 0, sizeof(int64_t) * 65536);
        for (int64_t i = 0; i < n; i++) {
            uint64_t u = (uint64_t)key[perm[i]] ^ 0x8000000000000000ull;
            cnt[(u >> sh) & 0xFFFF]++;
        }
        int64_t s = 0;
        for (int d = 0; d < 65536; d++) { int64_t c = cnt[d]; cnt[d] = s; s += c; }
        for (int64_t i = 0; i < n; i++) {
            uint64_t u = (uint64_t)key[perm[i]] ^ 0x8000000000000000ull;
            tmp[cnt[(u >> sh) & 0xFFFF]++] = perm[i];
        }
        memcpy(perm, tmp, sizeof(int64_t) * n);
        if (all_zero) break; /* higher digits are all equal */
    }
    free(tmp);
    free(cnt);
}

/* ------------------------------------------------------------------ */
/* oracle.py:41-106 brute_force_knn                                     */
/* ------------------------------------------------------------------ */
/* Rows are emitted in stable q_issuer order (oracle.py:56); each row holds
 * min(k, valid) entries ordered by (d2, id) (oracle.py:76-90), padded to k
 * with id -1 / distance +inf.  Distances are sqrt(d2) (oracle.py:95). */
OR_EXPORT void or_brute_knn(int64_t n, const int64_t *ids, const double *x,
                            const double *y, int64_t nq, const int64_t *q_issuer,
                            const double *qx, const double *qy, int k,
                            int64_t *out_qids, int32_t *out_len,
                            int64_t *out_nids, double *out_dist) {
    int64_t *qorder = (int64_t *)malloc(sizeof(int64_t) * (nq ? nq : 1));
    stable_argsort_i64(q_issuer, nq, qorder);
#pragma omp parallel
    {
        cand_t *L = (cand_t *)malloc(sizeof(cand_t) * (size_t)k);
#pragma omp for schedule(dynamic, 16)
        for (int64_t r = 0; r < nq; r++) {
            int64_t q = qorder[r];
            int cnt = 0;
            double ax = qx[q], ay = qy[q];
            int64_t me = q_issuer[q];
            for (int64_t j = 0; j < n; j++) {
                if (ids[j] == me) continue;
                double d2 = pair_d2(ax, ay, x[j], y[j]);
                if (cnt == k && !(d2 <= L[k - 1].d2)) continue;
                list_insert(L, k, &cnt, d2, ids[j]);
            }
            out_qids[r] = me;
            out_len[r] = cnt;
            for (int i = 0; i < k; i++) {
                out_nids[r * k + i] = i < cnt ? L[i].id : -1;
                out_dist[r * k + i] = i < cnt ? sqrt(L[i].d2) : INFINITY;
            }
        }
        free(L);
    }
    free(qorder);
}

/* ------------------------------------------------------------------ */
/* quadindex.py:79-163 build_index                                      */
/* ------------------------------------------------------------------ */

typedef struct {
    int32_t l_deep;
    int64_t n_leaves;
    int64_t overfull;
    int32_t *leaf_level;
    int64_t *leaf_code;
    int64_t *leaf_key;
    int64_t *leaf_span;
    int64_t *build_counts;
    int32_t *z_map; /* 4^l_deep */
} or_index;

OR_EXPORT void or_index_free(or_index *ix) {
    if (!ix) return;
    free(ix->leaf_level);
    free(ix->leaf_code);
    free(ix->leaf_key);
    free(ix->leaf_span);
    free(ix->build_counts);
    free(ix->z_map);
    free(ix);
}

static int64_t lower_bound_i64(const int64_t *a, int64_t n, int64_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* Returns NULL on bad parameters (quadindex.py:86-89 raise ValueError). */
OR_EXPORT or_index *or_build_index(int64_t n, const double *x, const double *y,
                                   const or_rect *r, int th_quad, int l_max) {
    if (th_quad < 1 || l_max < 1 || l_max > 10) return NULL;
    /* encode at l_max, sort (quadindex.py:93-94) */
    int64_t ncell = 1ll << (2 * l_max);
    int64_t *sc = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t *hist = (int64_t *)calloc((size_t)ncell + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) hist[or_encode(x[i], y[i], r, l_max)]++;
    int64_t w = 0;
    for (int64_t c = 0; c < ncell; c++)
        for (int64_t j = 0; j < hist[c]; j++) sc[w++] = c;
    free(hist);

    /* level-wise split (quadindex.py:96-134) */
    int64_t cap = 1024, m = 0;
    int32_t *o_lvl = (int32_t *)malloc(sizeof(int32_t) * cap);
    int64_t *o_code = (int64_t *)malloc(sizeof(int64_t) * cap);
    int64_t *o_cnt = (int64_t *)malloc(sizeof(int64_t) * cap);
    int64_t ncur = 1;
    int64_t *cc = (int64_t *)malloc(sizeof(int64_t)), *cs = (int64_t *)malloc(sizeof(int64_t)),
            *ce = (int64_t *)malloc(sizeof(int64_t));
    cc[0] = 0; cs[0] = 0; ce[0] = n;
    int level = 0;
    int64_t overfull = 0;
#define PUSH_LEAF(L, C, N)                                                      \
    do {                                                                        \
        if (m == cap) {                                                         \
            cap *= 2;                                                           \
            o_lvl = (int32_t *)realloc(o_lvl, sizeof(int32_t) * cap);           \
            o_code = (int64_t *)realloc(o_code, sizeof(int64_t) * cap);         \
            o_cnt = (int64_t *)realloc(o_cnt, sizeof(int64_t) * cap);           \
        }                                                                       \
        o_lvl[m] = (L); o_code[m] = (C); o_cnt[m] = (N); m++;                   \
    } while (0)
    while (ncur) {
        if (level == l_max) {
            for (int64_t i = 0; i < ncur; i++) {
                int64_t c = ce[i] - cs[i];
                PUSH_LEAF(level, cc[i], c);
                if (c > th_quad) overfull++;
            }
            break;
        }
        int64_t nsplit = 0;
        for (int64_t i = 0; i < ncur; i++) {
            int64_t c = ce[i] - cs[i];
            if (c > th_quad) nsplit++;
            else PUSH_LEAF(level, cc[i], c);
        }
        if (!nsplit) break;
        int64_t *nc = (int64_t *)malloc(sizeof(int64_t) * 4 * nsplit);
        int64_t *ns = (int64_t *)malloc(sizeof(int64_t) * 4 * nsplit);
        int64_t *ne = (int64_t *)malloc(sizeof(int64_t) * 4 * nsplit);
        int shift = 2 * (l_max - level - 1);
        int64_t j = 0;
        for (int64_t i = 0; i < ncur; i++) {
            if (ce[i] - cs[i] <= th_quad) continue;
            int64_t p = cc[i];
            int64_t b[5];
            b[0] = cs[i];
            for (int q = 1; q < 4; q++) b[q] = lower_bound_i64(sc, n, (p * 4 + q) << shift);
            b[4] = ce[i];
            for (int q = 0; q < 4; q++) {
                nc[j] = p * 4 + q; ns[j] = b[q]; ne[j] = b[q + 1]; j++;
            }
        }
        free(cc); free(cs); free(ce);
        cc = nc; cs = ns; ce = ne; ncur = j;
        level++;
    }
#undef PUSH_LEAF
    free(cc); free(cs); free(ce); free(sc);

    /* order by leaf key, spans, z_map (quadindex.py:136-149) */
    int32_t l_deep = 0;
    for (int64_t i = 0; i < m; i++) if (o_lvl[i] > l_deep) l_deep = o_lvl[i];
    int64_t *keys = (int64_t *)malloc(sizeof(int64_t) * m);
    for (int64_t i = 0; i < m; i++) keys[i] = o_code[i] << (2 * (l_deep - o_lvl[i]));
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * m);
    stable_argsort_i64(keys, m, perm);
    or_index *ix = (or_index *)calloc(1, sizeof(or_index));
    ix->l_deep = l_deep;
    ix->n_leaves = m;
    ix->overfull = overfull;
    ix->leaf_level = (int32_t *)malloc(sizeof(int32_t) * m);
    ix->leaf_code = (int64_t *)malloc(sizeof(int64_t) * m);
    ix->leaf_key = (int64_t *)malloc(sizeof(int64_t) * m);
    ix->leaf_span = (int64_t *)malloc(sizeof(int64_t) * m);
    ix->build_counts = (int64_t *)malloc(sizeof(int64_t) * m);
    int64_t nz = 1ll << (2 * l_deep);
    ix->z_map = (int32_t *)malloc(sizeof(int32_t) * nz);
    int64_t zpos = 0;
    for (int64_t i = 0; i < m; i++) {
        int64_t s = perm[i];
        ix->leaf_level[i] = o_lvl[s];
        ix->leaf_code[i] = o_code[s];
        ix->leaf_key[i] = keys[s];
        ix->leaf_span[i] = 1ll << (2 * (l_deep - o_lvl[s]));
        ix->build_counts[i] = o_cnt[s];
        for (int64_t z = 0; z < ix->leaf_span[i]; z++) ix->z_map[zpos++] = (int32_t)i;
    }
    free(keys); free(perm); free(o_lvl); free(o_code); free(o_cnt);
    if (zpos != nz) { or_index_free(ix); return NULL; }
    return ix;
}

/* ------------------------------------------------------------------ */
/* quadindex.py:190-213 index_objects                                   */
/* ------------------------------------------------------------------ */
/* Writes the objects sorted stably by l_deep code, per-leaf [start, end)
 * and returns the clamped count (geometry.py:215-220). */
OR_EXPORT int64_t or_index_objects(int64_t n, const int64_t *ids, const double *x,
                                   const double *y, const or_rect *r,
                                   const or_index *ix, int64_t *s_ids, double *s_x,
                                   double *s_y, int64_t *cell_start, int64_t *cell_end) {
    int64_t clamped = 0;
    int64_t *codes = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t i = 0; i < n; i++) {
        if (x[i] < r->x_lo || x[i] > r->x_hi || y[i] < r->y_lo || y[i] > r->y_hi) clamped++;
        codes[i] = or_encode(x[i], y[i], r, ix->l_deep);
    }
    stable_argsort_i64(codes, n, perm);
    for (int64_t l = 0; l < ix->n_leaves; l++) cell_start[l] = cell_end[l] = 0;
    for (int64_t i = 0; i < n; i++) cell_end[ix->z_map[codes[i]]]++;
    int64_t s = 0;
    for (int64_t l = 0; l < ix->n_leaves; l++) {
        cell_start[l] = s;
        s += cell_end[l];
        cell_end[l] = s;
    }
    for (int64_t i = 0; i < n; i++) {
        s_ids[i] = ids[perm[i]];
        s_x[i] = x[perm[i]];
        s_y[i] = y[perm[i]];
    }
    free(codes);
    free(perm);
    return clamped;
}

/* ------------------------------------------------------------------ */
/* engine.py:601-696 process_tick, restated per query                   */
/* ------------------------------------------------------------------ */
/* The reference interleaves all queries' left/right iterations globally
 * (engine.py:645-681), but each query's own state (list, cursors) is only
 * touched by its own rows, so the per-query step sequence L1 R1 L2 R2 ...
 * (an exhausted direction simply drops out) is independent of the others.
 * This port walks each query to completion and reconstructs the global
 * iteration metrics from per-query navigate-call counts.
 *
 * Selection is canonical: the list keeps the k smallest (d2, id) and a
 * quadrant is pruned only when its min-dist2 is strictly greater than the
 * k-th d2 (SURVEY.md §7 hard part 2; the reference prunes on >=,
 * engine.py:447).  Distance multisets are identical to the reference's. */

typedef struct {
    int64_t distance_evals;
    int64_t pruned_leaves;
    int64_t clamped_objects;
    int64_t iterations_left;
    int64_t iterations_right;
    int64_t streamed_records; /* T: sum of populations over distinct runs */
} or_metrics;

/* growable per-thread buffer of distance-task keys (dir, iteration, leaf) */
typedef struct {
    uint64_t *k;
    int64_t n, cap;
} keybuf;

static inline void kb_push(keybuf *b, uint64_t key) {
    if (b->n == b->cap) {
        b->cap = b->cap ? 2 * b->cap : 1024;
        b->k = (uint64_t *)realloc(b->k, sizeof(uint64_t) * b->cap);
    }
    b->k[b->n++] = key;
}

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : x > y;
}

#define TASK_KEY(dir, it, leaf) (((uint64_t)(dir) << 60) | ((uint64_t)(it) << 40) | (uint64_t)(leaf))

typedef struct {
    const or_index *ix;
    const or_rect *r;
    const int64_t *s_ids;
    const double *s_x, *s_y;
    const int64_t *cell_start, *cell_end;
} or_ctx;

/* engine.py:279-324 _merge_pack for one row: admit leaf objects into the
 * running list (self excluded by id, engine.py:298-300). */
static inline int64_t merge_leaf(const or_ctx *c, int64_t leaf, double qx, double qy,
                                 int64_t me, cand_t *L, int k, int *cnt) {
    int64_t s = c->cell_start[leaf], e = c->cell_end[leaf];
    for (int64_t j = s; j < e; j++) {
        if (c->s_ids[j] == me) continue;
        double d2 = pair_d2(qx, qy, c->s_x[j], c->s_y[j]);
        if (*cnt == k && !(d2 <= L[k - 1].d2)) continue;
        list_insert(L, k, cnt, d2, c->s_ids[j]);
    }
    return e - s;
}

/* engine.py:421-431 coarsest_levels */
static inline int coarsest_level(int64_t p, int sign, int l_deep) {
    int64_t a = p + (1 - sign) / 2;
    if (a == 0) return 0;
    int tz2 = __builtin_ctzll((uint64_t)a) >> 1;
    return l_deep - (tz2 < l_deep ? tz2 : l_deep);
}

/* engine.py:396-503 navigate, one ref: returns the assigned leaf or -1. */
static inline int64_t navigate_one(const or_ctx *c, int sign, int64_t *cursor,
                                   double qx, double qy, const cand_t *L, int k,
                                   int cnt, int64_t *pruned) {
    const or_index *ix = c->ix;
    int l_deep = ix->l_deep;
    int64_t n_codes = 1ll << (2 * l_deep);
    int full = cnt >= k;
    double thr = full ? L[k - 1].d2 : INFINITY;
    int64_t pos = *cursor;
    if (!(sign > 0 ? pos < n_codes : pos >= 0)) return -1;
    int lvl = full ? coarsest_level(pos, sign, l_deep) : l_deep;
    for (;;) {
        int delta = l_deep - lvl;
        int64_t qc = pos >> (2 * delta);
        double md2 = mindist2_cell(lvl, qc, c->r, qx, qy);
        if (full && md2 > thr) {
            (*pruned)++;
            pos += sign * (1ll << (2 * delta));
        } else if (lvl < l_deep) {
            lvl++;
            continue;
        } else {
            int64_t li = ix->z_map[pos];
            int64_t after = sign > 0 ? ix->leaf_key[li] + ix->leaf_span[li]
                                     : ix->leaf_key[li] - 1;
            if (c->cell_end[li] > c->cell_start[li]) {
                *cursor = after;
                return li;
            }
            pos = after;
        }
        if (!(sign > 0 ? pos < n_codes : pos >= 0)) {
            *cursor = pos;
            return -1;
        }
        lvl = full ? coarsest_level(pos, sign, l_deep) : l_deep;
    }
}

OR_EXPORT int or_engine_tick_ix(int64_t n, const int64_t *ids, const double *x, const double *y,
                                int64_t nq, const int64_t *q_issuer, const double *qx,
                                const double *qy, int k, const or_rect *r, const or_index *ix,
                                int64_t *out_qids, int32_t *out_len, int64_t *out_nids,
                                double *out_dist, int32_t *nav_left, int32_t *nav_right,
                                or_metrics *met, int32_t *out_l_deep, int64_t *out_n_leaves);

/* One full tick.  Outputs as or_brute_knn (padded rows in stable issuer
 * order).  nav_left/nav_right receive per-row navigate-call counts so the
 * caller can rebuild active_left/right (engine.py:661-663).  Returns 0, or
 * -1 on bad index parameters. */
OR_EXPORT int or_engine_tick(int64_t n, const int64_t *ids, const double *x, const double *y,
                             int64_t nq, const int64_t *q_issuer, const double *qx,
                             const double *qy, int k, const or_rect *r, int th_quad, int l_max,
                             int64_t *out_qids, int32_t *out_len, int64_t *out_nids,
                             double *out_dist, int32_t *nav_left, int32_t *nav_right,
                             or_metrics *met, int32_t *out_l_deep, int64_t *out_n_leaves,
                             int64_t nb, const double *bx, const double *by) {
    /* the index is built from (bx, by) -- the positions of the tick that
     * last rebuilt (engine.py:615-623); pass the tick's own x, y for a
     * rebuild tick */
    or_index *ix = or_build_index(nb, bx, by, r, th_quad, l_max);
    if (!ix) return -1;
    int rc = or_engine_tick_ix(n, ids, x, y, nq, q_issuer, qx, qy, k, r, ix, out_qids, out_len,
                               out_nids, out_dist, nav_left, nav_right, met, out_l_deep,
                               out_n_leaves);
    or_index_free(ix);
    return rc;
}

/* The same tick over an index built earlier (engine.py:615-619: a tick on
 * which should_rebuild does not fire reuses the engine's QuadIndex). */
OR_EXPORT int or_engine_tick_ix(int64_t n, const int64_t *ids, const double *x, const double *y,
                                int64_t nq, const int64_t *q_issuer, const double *qx,
                                const double *qy, int k, const or_rect *r, const or_index *ix,
                                int64_t *out_qids, int32_t *out_len, int64_t *out_nids,
                                double *out_dist, int32_t *nav_left, int32_t *nav_right,
                                or_metrics *met, int32_t *out_l_deep, int64_t *out_n_leaves) {
    int64_t L = ix->n_leaves;
    int64_t *s_ids = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    double *s_x = (double *)malloc(sizeof(double) * (n ? n : 1));
    double *s_y = (double *)malloc(sizeof(double) * (n ? n : 1));
    int64_t *cs = (int64_t *)malloc(sizeof(int64_t) * L);
    int64_t *ce = (int64_t *)malloc(sizeof(int64_t) * L);
    met->clamped_objects = or_index_objects(n, ids, x, y, r, ix, s_ids, s_x, s_y, cs, ce);
    or_ctx c = {ix, r, s_ids, s_x, s_y, cs, ce};

    /* engine.py:201-217 index_queries: stable sort by leaf ordinal */
    int64_t *qleaf = (int64_t *)malloc(sizeof(int64_t) * (nq ? nq : 1));
    int64_t *qperm = (int64_t *)malloc(sizeof(int64_t) * (nq ? nq : 1));
    for (int64_t i = 0; i < nq; i++) qleaf[i] = ix->z_map[or_encode(qx[i], qy[i], r, ix->l_deep)];
    stable_argsort_i64(qleaf, nq, qperm);
    /* emission row of each query: stable issuer order (oracle.py:56) */
    int64_t *qorder = (int64_t *)malloc(sizeof(int64_t) * (nq ? nq : 1));
    int64_t *qrow = (int64_t *)malloc(sizeof(int64_t) * (nq ? nq : 1));
    stable_argsort_i64(q_issuer, nq, qorder);
    for (int64_t rr = 0; rr < nq; rr++) qrow[qorder[rr]] = rr;

    int64_t evals = 0, pruned = 0;
    int32_t maxl = 0, maxr = 0;
    int nthr = 1;
#ifdef _OPENMP
    nthr = omp_get_max_threads();
#endif
    keybuf *kbs = (keybuf *)calloc((size_t)nthr, sizeof(keybuf));
#pragma omp parallel reduction(+ : evals, pruned) reduction(max : maxl, maxr)
    {
        cand_t *Lst = (cand_t *)malloc(sizeof(cand_t) * (size_t)k);
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        keybuf *kb = &kbs[tid];
#pragma omp for schedule(dynamic, 64)
        for (int64_t t = 0; t < nq; t++) {
            int64_t q = qperm[t];
            double ax = qx[q], ay = qy[q];
            int64_t me = q_issuer[q];
            int64_t own = qleaf[q];
            int cnt = 0;
            /* engine.py:356-373 first_iteration (rows with 0 candidates dropped) */
            if (ce[own] > cs[own]) {
                evals += merge_leaf(&c, own, ax, ay, me, Lst, k, &cnt);
                kb_push(kb, TASK_KEY(0, 0, own));
            }
            /* engine.py:645-681 direction loop, left first */
            int64_t cur[2] = {ix->leaf_key[own] - 1, ix->leaf_key[own] + ix->leaf_span[own]};
            int active[2] = {1, 1};
            int32_t calls[2] = {0, 0};
            int d = 0; /* 0 = left (sign -1), 1 = right (sign +1) */
            while (active[0] || active[1]) {
                if (active[d]) {
                    calls[d]++;
                    int64_t pr = 0;
                    int64_t li = navigate_one(&c, d ? 1 : -1, &cur[d], ax, ay, Lst, k, cnt, &pr);
                    pruned += pr;
                    if (li < 0) {
                        active[d] = 0;
                    } else {
                        evals += merge_leaf(&c, li, ax, ay, me, Lst, k, &cnt);
                        kb_push(kb, TASK_KEY(d + 1, calls[d] - 1, li));
                    }
                }
                d ^= 1;
            }
            int64_t row = qrow[q];
            if (nav_left) nav_left[row] = calls[0];
            if (nav_right) nav_right[row] = calls[1];
            if (calls[0] > maxl) maxl = calls[0];
            if (calls[1] > maxr) maxr = calls[1];
            /* engine.py:704-723 _emit (canonical (d2, id) row order) */
            out_qids[row] = me;
            out_len[row] = cnt;
            for (int i = 0; i < k; i++) {
                out_nids[row * k + i] = i < cnt ? Lst[i].id : -1;
                out_dist[row * k + i] = i < cnt ? sqrt(Lst[i].d2) : INFINITY;
            }
        }
        free(Lst);
    }
    /* T: each reference run is one distinct
     * (direction, iteration, leaf); its population is streamed once */
    int64_t nk = 0;
    for (int t = 0; t < nthr; t++) nk += kbs[t].n;
    uint64_t *all = (uint64_t *)malloc(sizeof(uint64_t) * (nk ? nk : 1));
    int64_t w = 0;
    for (int t = 0; t < nthr; t++) {
        memcpy(all + w, kbs[t].k, sizeof(uint64_t) * kbs[t].n);
        w += kbs[t].n;
        free(kbs[t].k);
    }
    free(kbs);
    qsort(all, (size_t)nk, sizeof(uint64_t), cmp_u64);
    int64_t T = 0;
    for (int64_t i = 0; i < nk; i++) {
        if (i && all[i] == all[i - 1]) continue;
        int64_t leaf = (int64_t)(all[i] & ((1ull << 40) - 1));
        T += ce[leaf] - cs[leaf];
    }
    free(all);
    met->streamed_records = T;
    met->distance_evals = evals;
    met->pruned_leaves = pruned;
    met->iterations_left = maxl;
    met->iterations_right = maxr;
    if (out_l_deep) *out_l_deep = ix->l_deep;
    if (out_n_leaves) *out_n_leaves = ix->n_leaves;
    free(qleaf); free(qperm); free(qorder); free(qrow);
    free(s_ids); free(s_x); free(s_y); free(cs); free(ce);
    return 0;
}

OR_EXPORT void or_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

OR_EXPORT int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
