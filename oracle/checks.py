"""Byte-level checks of GPU results against the oracle — TEST INFRASTRUCTURE
ONLY (used by tests/ and by bench.py's parity records, never by the
product).  Conversions here use plain torch ops, independent of the
product's own conversion kernels."""

from __future__ import annotations

import math
import time


def storage_to_f64(t):
    """Oriented float64 view of device storage (int32 Infinity = +/-(2^30-1)),
    computed with plain torch ops (independent of the product's kernels)."""
    import torch

    from paper_1701_04733_b200 import _lib

    if t.dtype == torch.int32:
        d = t.to(torch.float64)
        d = torch.where(t >= _lib.I32_INF, torch.full_like(d, math.inf), d)
        return torch.where(t <= -_lib.I32_INF, torch.full_like(d, -math.inf), d)
    return t.to(torch.float64)


def mismatches(got_f64_np, want_f64_np) -> int:
    import numpy as np

    a = np.ascontiguousarray(got_f64_np, dtype=np.float64).view(np.int64)
    b = np.ascontiguousarray(want_f64_np, dtype=np.float64).view(np.int64)
    if a.shape != b.shape:
        return -1
    return int(np.count_nonzero(a != b))


def closure_rows_parity(adj_dev, dist_dev, sample_rows, gen=None):
    """Check ``sample_rows`` rows of a GPU distance matrix against the C
    oracle's row closure (oracle_closure_rows_f32: Bellman-Ford by rows from
    the closure base) computed on the host from the GPU adjacency; with
    ``gen = (n, p, weights, seed)`` the adjacency's first and last 64 rows
    are first compared with the reference generator restated on the host
    (oracle.graphs.instance_rows), so the chain input -> distances is pinned
    end to end.  Returns a parity dict."""
    import numpy as np
    import torch

    from oracle import graphs as og
    from oracle import native

    n = adj_dev.shape[0]
    out = {}
    t0 = time.perf_counter()
    if gen is not None:
        gn, gp, gw, gseed = gen
        bad = 0
        for r0 in (0, max(0, n - 64)):
            want = og.instance_rows(gn, gp, gw, gseed, r0, min(n, r0 + 64))
            got = storage_to_f64(adj_dev[r0 : r0 + 64]).cpu().numpy()
            bad += mismatches(got, want)
        out["generator_rows"] = {"rows": "first 64 + last 64", "mismatches": bad,
                                 "against": "oracle.graphs.instance_rows (numpy PCG64 stream of random_graph)"}
    host = torch.empty((n, n), dtype=torch.float32)
    for r0 in range(0, n, 4096):  # the closure base (I (+) A) as f32 on the host
        blk = storage_to_f64(adj_dev[r0 : r0 + 4096]).to(torch.float32)
        idx = torch.arange(blk.shape[0], device=blk.device)
        diag = blk[idx, idx + r0]
        blk[idx, idx + r0] = torch.minimum(diag, torch.zeros_like(diag))
        host[r0 : r0 + 4096].copy_(blk)
    want, iters = native.closure_rows_f32(host.numpy(), sample_rows)
    del host
    got = storage_to_f64(dist_dev[torch.as_tensor(sample_rows, device=dist_dev.device)]).cpu().numpy()
    out["closure_rows"] = {"rows": list(map(int, sample_rows)), "cols": n, "mismatches": mismatches(got, want),
                           "oracle_products": iters,
                           "against": "oracle_closure_rows_f32 (row-wise Bellman-Ford of the closure base, C)"}
    out["check_s"] = round(time.perf_counter() - t0, 1)
    return out
