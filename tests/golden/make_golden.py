"""Generate golden fixtures by running the REAL reference package.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``mknn`` from /root/reference/pkg/src, runs the reference
``Engine`` (engine.py:557-701), ``brute_force_knn`` (oracle.py:41-106),
``build_index`` / ``index_objects`` (quadindex.py:79-213) and
``compare_results`` (oracle.py:142-200) on seeded inputs, and stores inputs,
expected outputs and per-tick metrics as compressed .npz files next to this
script.  Large outputs are stored as SHA-256 digests of the canonical arrays
(see ``digest``) so the fixtures stay small.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import mknn.engine as _eng  # noqa: E402
from mknn.engine import Engine, EngineConfig  # noqa: E402
from mknn.geometry import Rect, encode_points, leaf_order_keys, morton_encode, Point  # noqa: E402,F401
from mknn.oracle import brute_force_knn, compare_results  # noqa: E402
from mknn.quadindex import build_index, index_objects  # noqa: E402
from mknn.workload import WorkloadSpec, WorkloadGenerator, generate  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FULL_LIMIT = 40_000  # store full output arrays up to this many entries


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


# T: object records streamed by the distance tasks = the sum
# of leaf populations over the runs that first_iteration / update_nn_lists
# receive (engine.py:356-393).  Counted by wrapping both functions.
_T = [0]
_orig_first, _orig_update = _eng.first_iteration, _eng.update_nn_lists


def _first(run_leaf, starts, ends, qstore, ostore, *a, **kw):
    _T[0] += int((ostore.cell_end[run_leaf] - ostore.cell_start[run_leaf]).sum())
    return _orig_first(run_leaf, starts, ends, qstore, ostore, *a, **kw)


def _update(run_leaf, run_starts, run_ends, refs2, qstore, ostore, *a, **kw):
    _T[0] += int((ostore.cell_end[run_leaf] - ostore.cell_start[run_leaf]).sum())
    return _orig_update(run_leaf, run_starts, run_ends, refs2, qstore, ostore, *a, **kw)


_eng.first_iteration = _first
_eng.update_nn_lists = _update


def metrics_dict(m) -> dict:
    return dict(
        tick=m.tick, n_objects=m.n_objects, n_queries=m.n_queries,
        iterations_left=m.iterations_left, iterations_right=m.iterations_right,
        distance_evals=m.distance_evals, pruned_leaves=m.pruned_leaves,
        rebuild_flag=m.rebuild_flag, active_left=list(map(int, m.active_left)),
        active_right=list(map(int, m.active_right)), clamped_objects=m.clamped_objects,
    )


def run_case(name, region, k, ticks, th_quad="auto", l_max=10, kind="tick",
             rebuild_window=3, rebuild_factor=1.5):
    """ticks: list of (ids, x, y, q_issuer, qx, qy)."""
    arrs = {}
    meta = dict(name=name, k=k, region=[region.x_lo, region.y_lo, region.x_hi, region.y_hi],
                th_quad=th_quad, l_max=l_max, n_ticks=len(ticks), kind=kind,
                rebuild_window=rebuild_window, rebuild_factor=rebuild_factor, ticks=[])
    cfg = EngineConfig(k=k, region=region, th_quad=th_quad, l_max=l_max,
                       rebuild_window=rebuild_window, rebuild_factor=rebuild_factor)
    with Engine(cfg) as eng:
        for t, (ids, x, y, qi, qx, qy) in enumerate(ticks):
            ids = np.asarray(ids, np.int64); x = np.asarray(x, np.float64)
            y = np.asarray(y, np.float64); qi = np.asarray(qi, np.int64)
            qx = np.asarray(qx, np.float64); qy = np.asarray(qy, np.float64)
            for key, a in (("ids", ids), ("x", x), ("y", y), ("qi", qi), ("qx", qx), ("qy", qy)):
                arrs[f"t{t}_{key}"] = a
            _T[0] = 0
            res = eng.process_tick(ids, x, y, qi, qx, qy)
            m = eng.last_metrics
            orc = brute_force_knn(ids, x, y, qi, qx, qy, k)
            rep = compare_results(res, orc, positions=(ids, x, y))
            assert rep.ok, f"{name}: reference engine disagrees with its oracle"
            assert np.array_equal(res.distances, orc.distances)
            tmeta = dict(metrics=dict(metrics_dict(m), streamed_records=_T[0]),
                         verdicts=rep.counts,
                         oracle_digest=digest(orc.query_ids, orc.lengths, orc.neighbour_ids,
                                              orc.distances),
                         engine_digest=digest(res.query_ids, res.lengths, res.neighbour_ids,
                                              res.distances))
            if orc.neighbour_ids.size <= FULL_LIMIT:
                arrs[f"t{t}_o_qids"] = orc.query_ids
                arrs[f"t{t}_o_lens"] = orc.lengths
                arrs[f"t{t}_o_nids"] = orc.neighbour_ids
                arrs[f"t{t}_o_dist"] = orc.distances
                arrs[f"t{t}_e_nids"] = res.neighbour_ids
            # the index the reference used this tick (rebuilt or carried)
            ix = eng.index
            st = index_objects(ids, x, y, ix)
            tmeta["index"] = dict(l_deep=ix.l_deep, n_leaves=ix.n_leaves,
                                  overfull_leaves=ix.overfull_leaves,
                                  z_map_digest=digest(ix.z_map.astype(np.int32)),
                                  clamped=st.clamped)
            if ix.n_leaves <= FULL_LIMIT:
                arrs[f"t{t}_ix_leaf_level"] = ix.leaf_level.astype(np.int32)
                arrs[f"t{t}_ix_leaf_code"] = ix.leaf_code.astype(np.int64)
                arrs[f"t{t}_ix_leaf_key"] = ix.leaf_key.astype(np.int64)
                arrs[f"t{t}_ix_leaf_span"] = ix.leaf_span.astype(np.int64)
                arrs[f"t{t}_ix_build_counts"] = ix.build_counts.astype(np.int64)
                arrs[f"t{t}_cell_start"] = st.cell_start.astype(np.int64)
                arrs[f"t{t}_cell_end"] = st.cell_end.astype(np.int64)
                arrs[f"t{t}_store_ids"] = st.ids.astype(np.int64)
            else:
                tmeta["index"]["leaves_digest"] = digest(
                    ix.leaf_level.astype(np.int32), ix.leaf_code.astype(np.int64),
                    ix.build_counts.astype(np.int64))
                tmeta["index"]["cells_digest"] = digest(st.cell_start.astype(np.int64),
                                                        st.cell_end.astype(np.int64))
            meta["ticks"].append(tmeta)
    arrs["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **arrs)
    print(f"{name}: {len(ticks)} ticks, {os.path.getsize(path) / 1e3:.0f} kB")


def from_spec(spec):
    return [(b.ids, b.x, b.y, b.q_issuer, b.qx, b.qy) for b in generate(spec)]


def main():
    R100 = Rect.square(100.0)
    R32 = Rect.square(32.0)
    R22 = Rect.square(22500.0)

    # --- hand scenarios (inputs as in test_engine.py:44-149) -------------
    run_case("hand_two_objects", R100, 1,
             [([1, 2], [10.0, 20.0], [10.0, 10.0], [1, 2], [10.0, 20.0], [10.0, 10.0])], th_quad=4)
    run_case("hand_single_object", R100, 4,
             [([5], [50.0], [50.0], [5], [50.0], [50.0])], th_quad=4)
    run_case("hand_small_leaf", R100, 10,
             [([1, 2, 3], [10.0, 13.0, 14.0], [10.0, 14.0, 10.0], [1], [10.0], [10.0])], th_quad=64)
    run_case("hand_single_leaf_drain", R100, 2,
             [([1, 2, 3], [10.0, 20.0, 30.0], [10.0] * 3, [1, 2, 3], [10.0, 20.0, 30.0], [10.0] * 3)],
             th_quad=8)
    run_case("hand_zero_queries", R100, 2, [([1, 2], [10.0, 20.0], [10.0, 10.0], [], [], [])], th_quad=8)
    run_case("hand_merge", R32, 2,
             [([1, 2, 3, 4], [14.0, 14.0, 17.0, 21.0], [2.0, 7.0, 2.0, 2.0], [1], [14.0], [2.0])],
             th_quad=2, l_max=1)
    run_case("hand_far_prune", R32, 2,
             [([1, 2, 3, 9, 10], [1.0, 1.0, 1.0, 29.0, 30.0], [1.0, 2.0, 3.0, 29.0, 30.0],
               [1], [1.0], [1.0])], th_quad=2, l_max=1)
    ids5 = np.arange(5)
    x5 = np.array([0.0, 10.0, 20.0, 30.0, 40.0])
    run_case("hand_collinear_ties", Rect.square(50.0), 1,
             [(ids5, x5, np.zeros(5), ids5, x5, np.zeros(5))], th_quad=2)

    # --- generator workloads ------------------------------------------------
    run_case("gauss16_n2000_k32", R22, 32, from_spec(WorkloadSpec(
        n_objects=2000, distribution="gaussian", hotspots=16, sigma=500.0, region=R22,
        ticks=2, query_rate=1.0, k=32, seed=9)), th_quad=384)
    for k in (1, 4, 8, 17, 32, 33, 64, 128):
        run_case(f"uniform_n1500_k{k}", R22, k, from_spec(WorkloadSpec(
            n_objects=1500, distribution="uniform", region=R22, ticks=1, query_rate=1.0,
            k=k, seed=12 + k)), th_quad=16 if k < 64 else "auto")
    run_case("uniform_n800_multitick", Rect.square(5000.0), 8, from_spec(WorkloadSpec(
        n_objects=800, distribution="uniform", region=Rect.square(5000.0), ticks=4,
        query_rate=0.5, k=8, seed=21)), th_quad=16)
    run_case("gauss4_n600_rebuild", R22, 6, from_spec(WorkloadSpec(
        n_objects=600, distribution="gaussian", hotspots=4, sigma=300.0, region=R22, ticks=5,
        query_rate=0.5, k=6, seed=33)), th_quad=32, rebuild_window=1, rebuild_factor=1e-9)
    run_case("gauss1_n5000_k32_th16", R22, 32, from_spec(WorkloadSpec(
        n_objects=5000, distribution="gaussian", hotspots=1, sigma=500.0, region=R22, ticks=2,
        query_rate=0.3, k=32, seed=77)), th_quad=16)
    run_case("gauss25_n5000_k4_lmax6", R22, 4, from_spec(WorkloadSpec(
        n_objects=5000, distribution="gaussian", hotspots=25, sigma=500.0, region=R22, ticks=2,
        query_rate=0.5, k=4, seed=78)), th_quad=256, l_max=6)
    run_case("uniform_n5000_k32_lmax3", R22, 32, from_spec(WorkloadSpec(
        n_objects=5000, distribution="uniform", region=R22, ticks=1, query_rate=0.4, k=32,
        seed=79)), th_quad=64, l_max=3)

    # --- tie-heavy and edge inputs ---------------------------------------
    rng = np.random.default_rng(60)
    g = np.arange(30, dtype=np.float64) * 10.0 + 5.0
    lx, ly = np.meshgrid(g, g)
    lx, ly = lx.ravel(), ly.ravel()
    lids = rng.permutation(lx.size).astype(np.int64) * 3 + 1000
    run_case("lattice_shuffled_ids_k8", Rect.square(300.0), 8,
             [(lids, lx, ly, lids, lx, ly)], th_quad=16)
    run_case("lattice_shuffled_ids_k32", Rect.square(300.0), 32,
             [(lids, lx, ly, lids[::3], lx[::3], ly[::3])], th_quad=64)
    n = 400
    dx = rng.uniform(0, 100, n)
    dy = rng.uniform(0, 100, n)
    dx[: n // 5] = dx[n // 5: 2 * (n // 5)]
    dy[: n // 5] = dy[n // 5: 2 * (n // 5)]
    dids = rng.permutation(n).astype(np.int64)
    run_case("duplicate_coords_k17", Rect.square(100.0), 17, [(dids, dx, dy, dids, dx, dy)], th_quad=8)
    # objects outside the MBR clamp into boundary cells; queries stay inside
    ox = rng.uniform(-50, 1050, 600)
    oy = rng.uniform(-50, 1050, 600)
    inside = (ox >= 0) & (ox <= 1000) & (oy >= 0) & (oy <= 1000)
    oids = np.arange(600, dtype=np.int64) * 7 - 300
    run_case("clamped_objects_k5", Rect.square(1000.0), 5,
             [(oids, ox, oy, oids[inside][:200], ox[inside][:200], oy[inside][:200])], th_quad=12)
    # k larger than the population, and a query whose issuer is not an object
    kx = rng.uniform(0, 10, 12)
    ky = rng.uniform(0, 10, 12)
    kids = np.arange(12) + 5
    run_case("k_exceeds_population", Rect.square(10.0), 50,
             [(kids, kx, ky, np.concatenate([kids, [999]]), np.concatenate([kx, [5.0]]),
               np.concatenate([ky, [5.0]]))], th_quad=4)
    run_case("empty_objects", Rect.square(10.0), 3, [([], [], [], [7], [1.0], [1.0])], th_quad=4)

    # --- cfg 1 (BASELINE.json configs[0]): uniform 100K, 10K queries, k=8 --
    spec = WorkloadSpec(n_objects=100_000, distribution="uniform", region=R22, ticks=1, k=8, seed=0)
    gen = WorkloadGenerator(spec)
    x, y, ids = gen._x.copy(), gen._y.copy(), gen._ids.copy()
    sel = np.random.default_rng(1).choice(len(ids), 10_000, replace=False)
    cfg1 = dict(input_digest=digest(x, y))
    arrs = {}
    with Engine(EngineConfig(k=8, region=R22)) as eng:
        _T[0] = 0
        res = eng.process_tick(ids, x, y, ids[sel], x[sel], y[sel])
        m = eng.last_metrics
    orc = brute_force_knn(ids, x, y, ids[sel], x[sel], y[sel], 8)
    rep = compare_results(res, orc, positions=(ids, x, y))
    assert rep.ok
    cfg1.update(metrics=dict(metrics_dict(m), streamed_records=_T[0]), verdicts=rep.counts,
                oracle_digest=digest(orc.query_ids, orc.lengths, orc.neighbour_ids, orc.distances),
                index=dict(l_deep=eng.index.l_deep, n_leaves=eng.index.n_leaves,
                           overfull_leaves=eng.index.overfull_leaves))
    arrs["o_qids"] = orc.query_ids
    arrs["o_lens"] = orc.lengths.astype(np.int8)
    arrs["o_nids"] = orc.neighbour_ids.astype(np.int32)
    arrs["o_dist"] = orc.distances
    arrs["meta"] = np.frombuffer(json.dumps(cfg1).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "cfg1_uniform_100k.npz"), **arrs)
    print("cfg1:", cfg1["verdicts"], cfg1["metrics"]["distance_evals"])

    # --- frozen geometry values (test_geometry.py:26-133) ---------------
    unit = Rect(0.0, 0.0, 1.0, 1.0)
    frozen = dict(
        codes=[[0.9, 0.9, 2, morton_encode(Point(0.9, 0.9), unit, 2).code],
               [0.3, 0.6, 1, morton_encode(Point(0.3, 0.6), unit, 1).code],
               [1.0, 1.0, 3, morton_encode(Point(1.0, 1.0), unit, 3).code],
               [-5.0, 2.0, 1, morton_encode(Point(-5.0, 2.0), unit, 1).code],
               [0.5, 0.5, 1, morton_encode(Point(0.5, 0.5), unit, 1).code]],
    )
    rng = np.random.default_rng(11)
    px = rng.uniform(0, 22500.0, 2000)
    py = rng.uniform(0, 22500.0, 2000)
    for lvl in (0, 1, 5, 10, 15):
        frozen[f"enc_l{lvl}"] = encode_points(px, py, R22, lvl).tolist()
    frozen["enc_px"] = px.tolist()
    frozen["enc_py"] = py.tolist()
    with open(os.path.join(OUT, "geometry.json"), "w") as f:
        json.dump(frozen, f)
    print("geometry frozen values written")


if __name__ == "__main__":
    main()
