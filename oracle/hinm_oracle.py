"""CPU oracle for the HiNM hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm
(``/root/reference/pkg/src/hinm/pruning.py`` and ``spmm.py``), used as the
checker for the CUDA library.  It is never imported by the product package;
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may use it.

Parity pinning: every function here is checked against golden vectors
produced by running the real reference package in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz`` / ``*.json``),
see ``tests/test_oracle_golden.py``.

Floating-point order matters for bit-exact survivor selection, so the
reductions reproduce numpy's own summation order as used by the reference:

* column scores ``scores[rows].sum(axis=0)`` (pruning.py:79): sequential over
  the tile's rows in sigma_o order when n >= 2; numpy's pairwise sum over the
  rows when n == 1 (the (V, 1) operand is then contiguous along axis 0);
* group gains ``.reshape(G, M).sum(axis=1)`` (pruning.py:95): numpy pairwise
  summation over the M sorted scores of a group (``pairwise_sum`` below).
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "pairwise_sum", "tile_column_scores", "tile_order_and_gains", "allocate_budget_greedy",
    "allocate_budget_sorted", "vector_prune", "survivors", "nm_positions", "nm_prune",
    "encode", "decode", "restore_row_order", "hinm_spmm", "compress", "relative_error",
]


def pairwise_sum(a) -> float:
    """numpy's pairwise summation (``pairwise_sum_DOUBLE``) for a 1-D float64 run."""
    a = np.asarray(a, dtype=np.float64)
    n = a.size
    if n < 8:
        acc = np.float64(0.0)
        for x in a:
            acc = acc + x
        return acc
    if n <= 128:
        r = [a[j] for j in range(8)]
        i = 8
        stop = n - (n % 8)
        while i < stop:
            for j in range(8):
                r[j] = r[j] + a[i + j]
            i += 8
        acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            acc = acc + a[i]
            i += 1
        return acc
    half = n // 2
    half -= half % 8
    return pairwise_sum(a[:half]) + pairwise_sum(a[half:])


def tile_column_scores(S: np.ndarray, sigma_o: np.ndarray, V: int) -> np.ndarray:
    """score[t, j] = sum of S[sigma_o[tV + r], j] over the tile's rows (pruning.py:63-80)."""
    S = np.asarray(S, dtype=np.float64)
    m, n = S.shape
    T = m // V
    rows = np.asarray(sigma_o, dtype=np.int64).reshape(T, V)
    out = np.empty((T, n))
    if n == 1:
        for t in range(T):
            out[t, 0] = pairwise_sum(S[rows[t], 0])
        return out
    acc = S[rows[:, 0]].copy()          # (T, n): running sums, row order = sigma_o order
    for r in range(1, V):
        acc += S[rows[:, r]]
    out[:] = acc
    return out


def tile_order_and_gains(scores: np.ndarray, M: int):
    """Descending-score column order per tile (ties -> lower column) and per-group gains (pruning.py:83-96)."""
    T, n = scores.shape
    cols = np.arange(n)
    order = np.empty((T, n), dtype=np.int64)
    for t in range(T):
        order[t] = np.lexsort((cols, -scores[t]))
    G = n // M
    srt = np.take_along_axis(scores, order, axis=1)[:, : G * M]
    gains = srt.reshape(T, G, M).sum(axis=2)   # numpy pairwise per group, as in the reference
    return order, gains


def allocate_budget_greedy(gains: np.ndarray, total_groups: int) -> np.ndarray:
    """Literal restatement of the greedy loop (pruning.py:113-129); returns groups per tile."""
    T, G = gains.shape
    counts = np.zeros(T, dtype=np.int64)
    for _ in range(total_groups):
        best, best_t = None, -1
        for t in range(T):
            c = counts[t]
            if c >= G:
                continue
            key = (-gains[t, c], c, t)
            if best is None or key < best:
                best, best_t = key, t
        if best_t < 0:
            raise ValueError("budget exceeds available groups")
        counts[best_t] += 1
    return counts


def allocate_budget_sorted(gains: np.ndarray, total_groups: int) -> np.ndarray:
    """Same result as the greedy: the ``total_groups`` smallest keys (-gain, q, t).

    Each tile's key sequence is increasing in q (gains are non-increasing), so the
    greedy merge of per-tile lists selects exactly the globally smallest keys.
    """
    T, G = gains.shape
    if total_groups > T * G:
        raise ValueError("budget exceeds available groups")
    q = np.broadcast_to(np.arange(G)[None, :], (T, G)).ravel()
    t = np.broadcast_to(np.arange(T)[:, None], (T, G)).ravel()
    neg = -(gains.ravel() + 0.0)
    pick = np.lexsort((t, q, neg))[:total_groups]
    return np.bincount(t[pick], minlength=T).astype(np.int64)


def vector_prune(S, sigma_o, V: int, M: int, total_keep: int, greedy: bool = False):
    """Returns (vector_mask (T, n) bool, kept columns per tile, order)  (pruning.py:150-164)."""
    S = np.asarray(S, dtype=np.float64)
    scores = tile_column_scores(S, sigma_o, V)
    order, gains = tile_order_and_gains(scores, M)
    alloc = allocate_budget_greedy if greedy else allocate_budget_sorted
    counts = alloc(gains, total_keep // M) * M
    T, n = scores.shape
    mask = np.zeros((T, n), dtype=bool)
    for t in range(T):
        mask[t, order[t, : counts[t]]] = True
    return mask, counts, order


def survivors(vector_mask: np.ndarray):
    """Ascending surviving column ids per tile = the default sigma_i (pruning.py:167-169)."""
    return [np.flatnonzero(row).astype(np.int64) for row in vector_mask]


def nm_positions(group_scores: np.ndarray, N: int) -> np.ndarray:
    """Top-N in-group positions, ties to the lower position, emitted ascending (pruning.py:172-179)."""
    order = np.argsort(-group_scores, axis=-1, kind="stable")
    return np.sort(order[..., :N], axis=-1)


def nm_prune(S, sigma_o, sigma_i, V: int, N: int, M: int):
    """Element mask (m, n) and per-tile positions (V, G_t, N) (pruning.py:182-213)."""
    S = np.asarray(S, dtype=np.float64)
    m, n = S.shape
    rows = np.asarray(sigma_o, dtype=np.int64).reshape(-1, V)
    em = np.zeros((m, n), dtype=bool)
    pos_all = []
    for t, order in enumerate(sigma_i):
        order = np.asarray(order, dtype=np.int64)
        if order.size == 0:
            pos_all.append(np.empty((V, 0, N), dtype=np.int64))
            continue
        groups = order.reshape(-1, M)
        pos = nm_positions(S[rows[t]][:, groups], N)                     # (V, G, N)
        cols = groups[np.arange(groups.shape[0])[:, None], pos]
        em[np.broadcast_to(rows[t][:, None, None], cols.shape).ravel(), cols.ravel()] = True
        pos_all.append(pos)
    return em, pos_all


def encode(W, sigma_o, sigma_i, positions, V: int, N: int, M: int):
    """Per tile (vector_index, nm_index (V, G*N), kept_values (V, G*N)) (pruning.py:284-324)."""
    W = np.asarray(W, dtype=np.float64)
    rows = np.asarray(sigma_o, dtype=np.int64).reshape(-1, V)
    tiles = []
    for t, (order, pos) in enumerate(zip(sigma_i, positions)):
        order = np.asarray(order, dtype=np.int64)
        if order.size == 0:
            tiles.append((np.empty(0, np.int64), np.empty((V, 0), np.int64), np.empty((V, 0))))
            continue
        groups = order.reshape(-1, M)
        cols = groups[np.arange(groups.shape[0])[:, None], pos]          # (V, G, N)
        vals = W[rows[t][:, None, None], cols]
        tiles.append((order.copy(), pos.reshape(V, -1), vals.reshape(V, -1)))
    return tiles


def decode(tiles, shape, V: int, N: int, M: int) -> np.ndarray:
    """Dense (m, n) matrix with rows in sigma_o order (pruning.py:327-353)."""
    out = np.zeros(shape)
    for t, (vidx, nmi, vals) in enumerate(tiles):
        if vidx.size == 0:
            continue
        groups = vidx.reshape(-1, M)
        G = groups.shape[0]
        cols = groups[np.arange(G)[:, None], nmi.reshape(V, G, N)]
        out[np.arange(t * V, (t + 1) * V)[:, None, None], cols] = vals.reshape(V, G, N)
    return out


def restore_row_order(permuted: np.ndarray, sigma_o) -> np.ndarray:
    """out[sigma_o[p]] = permuted[p] (pruning.py:356-360)."""
    out = np.empty_like(permuted)
    out[np.asarray(sigma_o, dtype=np.int64)] = permuted
    return out


def hinm_spmm(tiles, X: np.ndarray, m: int, V: int, N: int, M: int) -> np.ndarray:
    """Gather-then-GEMV product, rows in sigma_o order (spmm.py:75-99): same data movement."""
    X = np.asarray(X, dtype=np.float64)
    out = np.zeros((m, X.shape[1]))
    for t, (vidx, nmi, vals) in enumerate(tiles):
        if vidx.size == 0:
            continue
        buf = X[vidx]                                                    # tile buffer (k_t, B)
        G = vidx.size // M
        slot = (np.arange(G)[None, :, None] * M + nmi.reshape(V, G, N)).reshape(V, -1)
        for r in range(V):
            out[t * V + r] = vals[r] @ buf[slot[r]]
    return out


def relative_error(result, reference) -> float:
    """max|delta| / max|ref| (spmm.py:107-110)."""
    scale = max(float(np.abs(reference).max(initial=0.0)), 1e-30)
    return float(np.abs(np.asarray(result) - reference).max(initial=0.0)) / scale


def compress(W, sigma_o, V: int, N: int, M: int, total_keep: int, sigma_i=None, S=None):
    """Full compressor path: vector_prune -> nm_prune -> encode with S = |W| by default.

    Returns dict(vector_mask, counts, sigma_i, element_mask, tiles).
    """
    W = np.asarray(W, dtype=np.float64)
    S = np.abs(W) if S is None else np.asarray(S, dtype=np.float64)
    vm, counts, _ = vector_prune(S, sigma_o, V, M, total_keep)
    if sigma_i is None:
        sigma_i = survivors(vm)
    em, pos = nm_prune(S, sigma_o, sigma_i, V, N, M)
    tiles = encode(W, sigma_o, sigma_i, pos, V, N, M)
    return {"vector_mask": vm, "counts": counts, "sigma_i": list(sigma_i),
            "element_mask": em, "tiles": tiles}
