/*
 * mknn_b200.h -- C-ABI of libmknn_b200.so, the B200-native drop-in for the
 * per-tick repeated k-NN join of the reference package `mknn`.
 *
 * Each entry point names the reference interface it replaces (paths relative
 * to /root/reference/pkg/src/mknn/).  Plain pointers and sizes only; every
 * call is synchronous with respect to the host unless it says otherwise, and
 * a handle must not be used from two threads at once (the reference engine is
 * single-writer; the service serialises ticks per session with a
 * lock, service/app.py:50,129).
 *
 * Status codes: 0 ok; MKNN_EINVAL (-1) bad argument (the Python shim raises
 * ValueError, as engine.py:73-85 / 611-612 and quadindex.py:86-89 do);
 * MKNN_ECUDA (-2) device failure (RuntimeError); MKNN_EUNSUPPORTED (-3).
 * mknn_last_error() describes the last failure on a handle.
 */
#ifndef MKNN_B200_H
#define MKNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MKNN_ABI_VERSION 1
#define MKNN_EINVAL (-1)
#define MKNN_ECUDA (-2)
#define MKNN_EUNSUPPORTED (-3)

typedef struct mknn_engine mknn_engine;

/* EngineConfig (engine.py:59-85).  th_quad is the RESOLVED leaf capacity
 * (resolve_th_quad, engine.py:48-56, runs on the host); num_bins,
 * max_refine_iters and threads select CPU internals of the reference
 * (kselect.py:34-138, engine.py:591-599) and have no device counterpart. */
typedef struct mknn_config {
    int32_t k;
    int32_t th_quad;
    int32_t l_max;
    int32_t rebuild_window;
    double rebuild_factor;
    double x_lo, y_lo, x_hi, y_hi; /* region (Rect, geometry.py:27-58) */
    int32_t self_check;
    int32_t audit_pruning;
    int32_t device; /* CUDA ordinal */
    int32_t instrument; /* bit 0: count streamed records T */
} mknn_config;

/* TickMetrics (engine.py:88-107).  Phase times are device times measured
 * with CUDA events on the engine's stream, except t_total_us (host wall
 * clock of the call).  active_left/right lists: mknn_active_counts(). */
typedef struct mknn_metrics {
    int64_t tick;
    int64_t n_objects;
    int64_t n_queries;
    int64_t iterations_left;
    int64_t iterations_right;
    int64_t distance_evals;
    int64_t pruned_leaves;
    int64_t rebuild_flag;
    int64_t t_build_us;
    int64_t t_index_objects_us;
    int64_t t_index_queries_us;
    /* first_iteration and the direction loop run in one search kernel per
       query batch: its CUDA-event time split by the batches' measured
       (%globaltimer) warp time in the own-leaf pass */
    int64_t t_first_iteration_us;
    int64_t t_loop_us;
    int64_t t_total_us;
    int64_t pruning_violations;
    int64_t clamped_objects;
    int64_t n_results; /* sum of lengths (CSR size) */
    int64_t t_emit_us;
    /* T: object records streamed by the reference's distance tasks = sum of
     * leaf populations over distinct (iteration, direction, leaf) runs plus
     * distinct own leaves; -1 unless config.instrument & 1 */
    int64_t streamed_records;
} mknn_metrics;

/* Engine.__init__ + EngineConfig.__post_init__ (engine.py:561-568, 73-85). */
int mknn_create(const mknn_config* cfg, mknn_engine** out);
/* Engine.close (engine.py:570-573). */
void mknn_destroy(mknn_engine* h);
const char* mknn_last_error(const mknn_engine* h);
int mknn_abi_version(void);
/* Cumulative number of kernels this library has launched (process-wide). */
int64_t mknn_kernel_launches(void);

/* Run the engine's work on this cudaStream_t (NULL = the engine's own, which is
 * created non-blocking: pass cudaStreamLegacy, not NULL, for the legacy default stream). */
int mknn_set_stream(mknn_engine* h, void* cuda_stream);

/* Engine.process_tick (engine.py:601-696) on a full snapshot in HOST memory
 * (pinned or pageable).  Outputs are caller-allocated host buffers:
 *   out_qids[nq]        query ids in stable issuer order (engine.py:713)
 *   out_len[nq]         list lengths, min(k, other objects)
 *   out_nids[nq * k]    neighbour ids, CSR-compacted: row i occupies
 *   out_dist[nq * k]    [sum(len[:i]), sum(len[:i+1])), ordered by (d2, id);
 *                       distances are correctly rounded sqrt(d2).
 * metrics may be NULL. */
int mknn_tick(mknn_engine* h, int64_t n, const int64_t* ids, const double* x, const double* y,
              int64_t nq, const int64_t* q_issuer, const double* qx, const double* qy,
              int64_t* out_qids, int32_t* out_len, int64_t* out_nids, double* out_dist,
              mknn_metrics* metrics);

/* Same tick with every input and output in DEVICE memory of the engine's
 * device; out_offsets[nq + 1] receives the CSR offsets.  Results stay
 * device-resident (wrap them with DLPack / torch.as_tensor). */
int mknn_tick_device(mknn_engine* h, int64_t n, const int64_t* d_ids, const double* d_x,
                     const double* d_y, int64_t nq, const int64_t* d_q_issuer, const double* d_qx,
                     const double* d_qy, int64_t* d_out_qids, int32_t* d_out_len,
                     int64_t* d_out_offsets, int64_t* d_out_nids, double* d_out_dist,
                     mknn_metrics* metrics);

/* Delta path (datasets.py:109-164 carry-forward semantics on a persistent
 * device snapshot).  mknn_load replaces the snapshot; mknn_update applies
 * position updates (last update per id wins, unknown ids are appended);
 * mknn_query runs one tick (engine.py:601-696) of the given queries over the
 * current snapshot.  *_device variants take device pointers. */
int mknn_load(mknn_engine* h, int64_t n, const int64_t* ids, const double* x, const double* y);
int mknn_update(mknn_engine* h, int64_t nu, const int64_t* ids, const double* x, const double* y);
int mknn_update_device(mknn_engine* h, int64_t nu, const int64_t* d_ids, const double* d_x,
                       const double* d_y);
int mknn_snapshot_size(const mknn_engine* h, int64_t* n);
int mknn_query(mknn_engine* h, int64_t nq, const int64_t* q_issuer, const double* qx,
               const double* qy, int64_t* out_qids, int32_t* out_len, int64_t* out_nids,
               double* out_dist, mknn_metrics* metrics);
int mknn_query_device(mknn_engine* h, int64_t nq, const int64_t* d_q_issuer, const double* d_qx,
                      const double* d_qy, int64_t* d_out_qids, int32_t* d_out_len,
                      int64_t* d_out_offsets, int64_t* d_out_nids, double* d_out_dist,
                      mknn_metrics* metrics);

/* Toggle instrumentation (mknn_config.instrument bits) between ticks. */
int mknn_set_instrument(mknn_engine* h, int32_t flags);
/* Steady-state device ticks (same shape, buffers and flags as the previous
 * one) replay a CUDA graph of the whole tick; counts of graph captures and
 * replays on this handle so far (no reference counterpart: the reference
 * has no device). */
int mknn_graph_stats(const mknn_engine* h, int64_t* captures, int64_t* replays);

/* Multi-GPU: replace the last tick's entry of the rebuild history
 * (quadindex.py:231-246 input, engine.py:692) with the job-wide
 * distance_evals, so every rank takes the same rebuild decisions. */
int mknn_set_last_evals(mknn_engine* h, int64_t distance_evals);

/* TickMetrics.active_left / active_right of the last tick (engine.py:661-663):
 * dir 0 = left, 1 = right.  Writes min(cap, len) entries, returns len. */
int64_t mknn_active_counts(const mknn_engine* h, int dir, int64_t* out, int64_t cap);

/* Engine.index (engine.py:587-589 -> QuadIndex, quadindex.py:23-38). */
int mknn_index_info(const mknn_engine* h, int32_t* l_deep, int64_t* n_leaves,
                    int64_t* overfull_leaves, int64_t* n_build);
int mknn_index_export(mknn_engine* h, int32_t* leaf_level, int64_t* leaf_code, int64_t* leaf_key,
                      int64_t* leaf_span, int64_t* build_counts, int32_t* z_map);
/* ObjectStore cell ranges of the last tick (quadindex.py:180-181). */
int mknn_store_export(mknn_engine* h, int64_t* cell_start, int64_t* cell_end);

/* Result consumer (studies.py:105-108 write_result_block): the CSV lines
 *   "{tick},{query_id},{rank},{neighbour_id},{distance:.9g}\n"
 * of a CSR result (qids[nq], offsets[nq + 1], nids / dist[offsets[nq]]),
 * formatted on `threads` host threads (<= 0: all).  Writes at most cap bytes
 * to out and returns the byte count, or MKNN_EINVAL if cap is too small.
 * Host-only: needs no GPU. */
int64_t mknn_format_result_rows(int64_t tick, int64_t nq, const int64_t* qids,
                                const int64_t* offsets, const int64_t* nids, const double* dist,
                                char* out, int64_t cap, int32_t threads);

/* Brute-force certificate (audit tooling: oracle.py:41-106
 * as a tiled fp64 device pass; never on the tick path).  All pointers are
 * DEVICE memory.  For each query i counts the objects o with
 * o.id != q_issuer[i] and (d2(q_i, o), o.id) < (kth_d2[i], kth_id[i]) in
 * canonical order (oracle.py:76-77), d2 with three roundings
 * (geometry.py:210-212), into out_count[i].  Runs on `stream` (NULL = the
 * legacy default stream). */
int mknn_bf_count_device(int64_t n, const int64_t* ids, const double* x, const double* y,
                         int64_t nq, const int64_t* q_issuer, const double* qx, const double* qy,
                         const double* kth_d2, const int64_t* kth_id, uint64_t* out_count,
                         void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MKNN_B200_H */
