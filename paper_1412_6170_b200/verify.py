"""Brute-force certificate of a device tick result.

Audit tooling, never on the tick path: the reference's own re-checks are
``self_check`` / ``audit_pruning`` (engine.py:529-554) and, in its tests,
``brute_force_knn`` (oracle.py:41-106).  A CPU brute force is infeasible at
BASELINE sizes (10^13 pairs at cfg3), so the check is restated as:

1. every listed neighbour exists in the snapshot, is not the issuer
   (oracle.py:66), sits at ``sqrt(d2)`` bit-exactly with d2 evaluated with
   three roundings (geometry.py:210-212, engine.py:706), and each row is
   strictly increasing in canonical ``(d2, id)`` order (oracle.py:76-77);
2. one fp64 device pass over all (query, object) pairs
   (``mknn_bf_count_device``) counts, per query, the objects other than the
   issuer that precede the row's last entry in canonical order: a full row
   is the exact top-k iff that count is ``k - 1``; a short row (fewer than k
   other objects) is complete iff counting against ``(+inf, max id)`` gives
   its length.

Together these prove every row equals ``brute_force_knn``'s, without a
selection on the checker side.  Inputs are torch CUDA tensors.
"""

from __future__ import annotations

import ctypes

from . import _native as N

INT64_MAX = (1 << 63) - 1


def bf_count(ids, x, y, q_issuer, qx, qy, kth_d2, kth_id):
    """Per query, the number of objects (not the issuer) strictly before
    (kth_d2, kth_id) in canonical order.  All arguments CUDA tensors."""
    import torch

    nq = int(q_issuer.numel())
    out = torch.empty(max(nq, 1), dtype=torch.int64, device=q_issuer.device)
    stream = torch.cuda.current_stream(q_issuer.device).cuda_stream or 1  # 1 = cudaStreamLegacy
    p = lambda t: t.data_ptr() if t.numel() else 0  # noqa: E731
    N.check(N.lib().mknn_bf_count_device(
        int(ids.numel()), p(ids), p(x), p(y), nq, p(q_issuer), p(qx), p(qy), p(kth_d2), p(kth_id),
        p(out), ctypes.c_void_p(stream)), None, "mknn_bf_count_device")
    return out[:nq]


def certify(ids, x, y, q_issuer, qx, qy, k: int, result) -> dict:
    """Check a tick result against the snapshot by brute force.

    ``result``: dict of CUDA tensors as returned by ``Engine.tick_device`` /
    ``query_device`` (query_ids, lengths, offsets, neighbour_ids, distances,
    n_results).  Returns counts of failing rows per check (all zero when the
    result is the canonical k-NN join)."""
    import torch

    dev = q_issuer.device
    nq = int(q_issuer.numel())
    n_res = int(result["n_results"])
    qids = result["query_ids"][:nq]
    lens = result["lengths"][:nq].to(torch.int64)
    offs = result["offsets"][: nq + 1]
    nids = result["neighbour_ids"][:n_res]
    dist = result["distances"][:n_res]
    bad = {}
    # rows ordered by issuer id, stable (engine.py:713)
    order = torch.sort(q_issuer, stable=True).indices
    bad["row_order"] = int((qids != q_issuer[order]).sum())
    bad["offsets"] = int((offs[1:] - offs[:-1] != lens).sum()) + int(offs[0] != 0) + \
        int(offs[-1] != n_res)
    bad["length"] = int(((lens < 0) | (lens > k)).sum())
    rx, ry, rme = qx[order], qy[order], qids
    row = torch.repeat_interleave(torch.arange(nq, device=dev), lens)
    # 1. neighbours exist, are not the issuer, sit at their exact distance
    sid, sperm = torch.sort(ids)
    pos = torch.searchsorted(sid, nids).clamp_(max=max(int(ids.numel()) - 1, 0))
    found = sid[pos] == nids if ids.numel() else torch.zeros_like(nids, dtype=torch.bool)
    bad["unknown_id"] = int((~found).sum())
    oi = sperm[pos]
    dx = rx[row] - x[oi]
    dy = ry[row] - y[oi]
    d2 = dx * dx + dy * dy  # three roundings: one kernel per operation
    bad["self"] = int((nids == rme[row]).sum())
    bad["distance"] = int((torch.sqrt(d2).view(torch.int64) != dist.view(torch.int64)).sum())
    # strictly increasing (d2, id) inside each row
    if n_res > 1:
        same = row[1:] == row[:-1]
        inc = (d2[1:] > d2[:-1]) | ((d2[1:] == d2[:-1]) & (nids[1:] > nids[:-1]))
        bad["order"] = int((same & ~inc).sum())
    else:
        bad["order"] = 0
    # 2. nothing missing: count the objects before each row's last entry
    full = lens == k
    last = (offs[1:] - 1).clamp_(min=0)
    kd = torch.full((nq,), float("inf"), dtype=torch.float64, device=dev)
    ki = torch.full((nq,), INT64_MAX, dtype=torch.int64, device=dev)
    if n_res:
        kd = torch.where(full, d2[last.clamp(max=n_res - 1)], kd)
        ki = torch.where(full, nids[last.clamp(max=n_res - 1)], ki)
    cnt = bf_count(ids, x, y, rme, rx, ry, kd, ki)
    want = torch.where(full, torch.full_like(lens, k - 1), lens)
    bad["count"] = int((cnt != want).sum())
    return bad
