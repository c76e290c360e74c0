"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference hot path.

Used by tests (as a checker) and by bench.py's CPU-baseline arm (as the
timed "port" of the reference).  Never imported by the product package.

Everything here works on plain numpy arrays and returns a dict of arrays
with the reference's field semantics (``lemt.formats.CerMatrix`` /
``CserMatrix``, formats.py:105-170).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_WIDTHS = (8, 16, 32)
_UINT = {8: np.uint8, 16: np.uint16, 32: np.uint32}


def width_for(max_value: int) -> int:
    """Smallest of 8/16/32 holding ``max_value`` unsigned (formats.py:52-59)."""
    if max_value < 0:
        raise ValueError("index values are unsigned")
    for bits in _WIDTHS:
        if max_value >> bits == 0:
            return bits
    raise ValueError(f"index value {max_value} does not fit in 32 bits")


def as_index(values, max_value: int, index_bits) -> np.ndarray:
    """Index array at the auto or forced width (formats.py:66-74)."""
    bits = width_for(max_value) if index_bits == "auto" else int(index_bits)
    if bits not in _WIDTHS:
        raise ValueError(f"index bits must be one of {_WIDTHS}")
    if max_value >= (1 << bits):
        raise ValueError(f"index value {max_value} does not fit in {bits} bits")
    return np.ascontiguousarray(np.asarray(values).astype(_UINT[bits]))


def alphabet(values: np.ndarray, background=None):
    """Frequency-major alphabet with the background first, plus the rank grid.

    Restates formats.py:193-209: distinct values ordered by (count desc,
    value asc); the background (default: the head of that order) is moved
    to the front, or prepended when absent.  Ranks are positions in that
    final order, found here through ``np.unique``'s inverse map (the
    reference uses a searchsorted over the value-sorted alphabet; both give
    the same value->position mapping).
    """
    flat = values.reshape(-1)
    uniq, inverse, counts = np.unique(flat, return_inverse=True, return_counts=True)
    freq_order = np.lexsort((uniq, -counts))  # count desc, ties value asc
    omega = uniq[freq_order]
    bg = omega[0] if background is None else float(background)
    hit = np.flatnonzero(omega == bg)
    if hit.size:
        keep = np.ones(omega.size, dtype=bool)
        keep[hit[0]] = False
        omega = np.concatenate(([bg], omega[keep]))
    else:
        omega = np.concatenate(([bg], omega))
    # value-sorted position -> frequency rank in the final alphabet
    final_sorted = np.argsort(omega, kind="stable")
    # map each unique value (value-ascending) to its slot in omega
    pos_in_final = final_sorted[np.searchsorted(omega[final_sorted], uniq)]
    ranks = pos_in_final[inverse].reshape(values.shape)
    return omega, ranks


def layout(ranks: np.ndarray, k: int):
    """Per-(row, rank) counts and colI sorted by (row, rank, col) (formats.py:212-224)."""
    m, n = ranks.shape
    rows, cols = np.nonzero(ranks)  # row-major, so columns ascend inside a row
    rk = ranks[rows, cols]
    key = rows.astype(np.int64) * k + rk
    order = np.argsort(key, kind="stable")  # stable keeps column order per (row, rank)
    counts = np.bincount(key, minlength=m * k).reshape(m, k)
    return counts, cols[order]


def _check_nonempty(values: np.ndarray):
    if values.size == 0:
        # the reference fails on omega[0] of an empty alphabet (formats.py:199)
        raise IndexError("index 0 is out of bounds for axis 0 with size 0")


def encode_cer(values: np.ndarray, index_bits="auto", background=None) -> dict:
    """CER arrays (formats.py:227-256): padding segments up to the last present rank."""
    values = np.asarray(values, dtype=np.float64)
    _check_nonempty(values)
    m, n = values.shape
    omega, ranks = alphabet(values, background)
    k = omega.size
    counts, col_index = layout(ranks, k)
    body = counts[:, 1:]
    if k > 1:
        present = body > 0
        last = np.where(present.any(axis=1), k - 1 - np.argmax(present[:, ::-1], axis=1), 0)
        keep = np.arange(1, k)[None, :] <= last[:, None]
        seg_sizes = body[keep]
    else:
        last = np.zeros(m, dtype=np.int64)
        seg_sizes = np.zeros(0, dtype=np.int64)
    omega_ptr = np.zeros(seg_sizes.size + 1, dtype=np.int64)
    np.cumsum(seg_sizes, out=omega_ptr[1:])
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(last, out=row_ptr[1:])
    return {
        "kind": "cer", "m": m, "n": n,
        "omega": omega.astype(np.float64),
        "colI": as_index(col_index, max(n - 1, 0), index_bits),
        "omegaPtr": as_index(omega_ptr, col_index.size, index_bits),
        "rowPtr": as_index(row_ptr, seg_sizes.size, index_bits),
    }


def encode_cser(values: np.ndarray, index_bits="auto", background=None) -> dict:
    """CSER arrays (formats.py:259-295): value-ascending alphabet, present segments only."""
    values = np.asarray(values, dtype=np.float64)
    _check_nonempty(values)
    m, n = values.shape
    omega_freq, ranks = alphabet(values, background)
    k = omega_freq.size
    counts, col_index = layout(ranks, k)
    omega = np.sort(omega_freq)
    to_value_pos = np.searchsorted(omega, omega_freq)
    body = counts[:, 1:]
    present = body > 0
    seg_sizes = body[present]
    seg_rank = np.nonzero(present)[1] + 1  # row-major: rank order inside each row
    omega_index = to_value_pos[seg_rank] if k > 1 else np.zeros(0, dtype=np.int64)
    omega_ptr = np.zeros(seg_sizes.size + 1, dtype=np.int64)
    np.cumsum(seg_sizes, out=omega_ptr[1:])
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(present.sum(axis=1), out=row_ptr[1:])
    return {
        "kind": "cser", "m": m, "n": n,
        "omega": omega.astype(np.float64),
        "colI": as_index(col_index, max(n - 1, 0), index_bits),
        "omegaI": as_index(omega_index, max(k - 1, 0), index_bits),
        "omegaPtr": as_index(omega_ptr, col_index.size, index_bits),
        "rowPtr": as_index(row_ptr, seg_sizes.size, index_bits),
        "mode_index": int(to_value_pos[0]),
    }


def background_of(enc: dict) -> float:
    return float(enc["omega"][0] if enc["kind"] == "cer" else enc["omega"][enc["mode_index"]])


def segment_values(enc: dict) -> np.ndarray:
    """Shared value of every segment (kernels.py:286-292)."""
    if enc["kind"] == "cer":
        row_ptr = enc["rowPtr"].astype(np.int64)
        per_row = np.diff(row_ptr)
        first = np.repeat(row_ptr[:-1], per_row)
        return enc["omega"][np.arange(row_ptr[-1]) - first + 1]
    return enc["omega"][enc["omegaI"].astype(np.int64)]


def _slice_sums(values: np.ndarray, bounds: np.ndarray) -> np.ndarray:
    """Sums over [b[i], b[i+1]) as differences of one running prefix sum (kernels.py:117-125)."""
    lead = np.zeros((1,) + values.shape[1:])
    prefix = np.concatenate((lead, np.cumsum(values, axis=0)), axis=0)
    b = bounds.astype(np.int64)
    return prefix[b[1:]] - prefix[b[:-1]]


def dot(enc: dict, x) -> np.ndarray:
    """y = A.x in float64, the reference's vectorised evaluation order (kernels.py:283-301)."""
    xv = np.asarray(x, dtype=np.float64)
    if xv.ndim not in (1, 2):
        raise ValueError("right-hand side must be a vector or a matrix")
    if xv.shape[0] != enc["n"]:
        raise ValueError(f"dimension mismatch: matrix has n={enc['n']}, input has {xv.shape[0]}")
    seg_sum = _slice_sums(xv[enc["colI"].astype(np.int64)], enc["omegaPtr"])
    vals = segment_values(enc)
    bg = background_of(enc)
    if bg != 0.0:
        vals = vals - bg
    prod = vals * seg_sum if seg_sum.ndim == 1 else vals[:, None] * seg_sum
    y = _slice_sums(prod, enc["rowPtr"])
    if bg != 0.0:
        y = y + bg * xv.sum(axis=0)
    return y


def row_block(enc: dict, r0: int, r1: int) -> dict:
    """Rows [r0, r1) as a self-contained encoding (a slice, not a re-encode)."""
    rp = enc["rowPtr"].astype(np.int64)
    op = enc["omegaPtr"].astype(np.int64)
    s0, s1 = int(rp[r0]), int(rp[r1])
    e0, e1 = int(op[s0]), int(op[s1])
    out = dict(enc)
    out["m"] = r1 - r0
    out["rowPtr"] = rp[r0:r1 + 1] - s0
    out["omegaPtr"] = op[s0:s1 + 1] - e0
    out["colI"] = enc["colI"][e0:e1]
    if enc["kind"] == "cser":
        out["omegaI"] = enc["omegaI"][s0:s1]
    return out


def dot_threaded(enc: dict, x, threads: int | None = None) -> np.ndarray:
    """The same evaluation over ``threads`` row blocks in parallel (numpy drops the GIL in
    gather/cumsum).  Each block restarts its prefix sums, so the result may differ from
    :func:`dot` in the last bits; used only as the multi-core CPU baseline timing."""
    threads = threads or os.cpu_count() or 1
    m = enc["m"]
    if threads <= 1 or m < 2 * threads:
        return dot(enc, x)
    cuts = np.linspace(0, m, threads + 1).astype(int)
    blocks = [row_block(enc, int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:])]
    with ThreadPoolExecutor(max_workers=threads) as pool:
        parts = list(pool.map(lambda blk: dot(blk, x), blocks))
    return np.concatenate(parts, axis=0)


# --------------------------------------------------------------------------- validate / decode
# Restatement of lemt.formats.validate / decode for CER and CSER (formats.py:298-392, 395-424): the
# checks run in the reference's order and the first violation is returned as (array, offset, reason)
# -- the fields of lemt.formats.FormatError -- or None for a valid encoding.


def _first_monotone_violation(name: str, arr: np.ndarray, first: int, last: int):
    """formats.py:298-308: non-empty, starts at `first`, non-decreasing, ends at `last`."""
    if arr.size == 0:
        return (name, 0, "array is empty")
    if int(arr[0]) != first:
        return (name, 0, f"must start at {first}, found {int(arr[0])}")
    steps = np.diff(arr.astype(np.int64))
    down = np.flatnonzero(steps < 0)
    if down.size:
        return (name, int(down[0]) + 1, "must be non-decreasing")
    if int(arr[-1]) != last:
        return (name, arr.size - 1, f"must end at {last}, found {int(arr[-1])}")
    return None


def _first_duplicate(keys: np.ndarray):
    """Index of the second occurrence (stable order) of the smallest duplicated key, or None."""
    order = np.argsort(keys, kind="stable")
    same = np.flatnonzero(np.diff(keys[order]) == 0)
    return int(order[same[0] + 1]) if same.size else None


def _first_column_violation(cols: np.ndarray, seg_ptr: np.ndarray, n: int, entry_row: np.ndarray):
    """formats.py:311-329: in range, strictly ascending inside a segment, unique within a row."""
    c = cols.astype(np.int64)
    oob = np.flatnonzero(c >= n)
    if oob.size:
        return ("colI", int(oob[0]), f"column {int(c[oob[0]])} out of range for n={n}")
    if c.size > 1:
        seg_start = np.zeros(c.size, dtype=bool)
        heads = seg_ptr[:-1].astype(np.int64)
        seg_start[heads[heads < c.size]] = True
        bad = np.flatnonzero((np.diff(c) <= 0) & ~seg_start[1:])
        if bad.size:
            return ("colI", int(bad[0]) + 1, "must be strictly ascending within a segment")
    dup = _first_duplicate(entry_row.astype(np.int64) * n + c)
    if dup is not None:
        return ("colI", dup, "duplicate column within a row")
    return None


def validate(enc: dict):
    """First structural violation of a CER/CSER encoding (dict as produced by encode_cer/encode_cser)."""
    omega = np.asarray(enc["omega"], dtype=np.float64)
    op, rp, col = (np.asarray(enc[k]) for k in ("omegaPtr", "rowPtr", "colI"))
    m, n, k = int(enc["m"]), int(enc["n"]), omega.size
    if np.unique(omega).size != k:
        return ("omega", 0, "duplicate alphabet values")
    segs = op.size - 1
    if rp.size != m + 1:
        return ("rowPtr", 0, f"expected {m + 1} entries")
    for name, arr, last in (("omegaPtr", op, col.size), ("rowPtr", rp, segs)):
        v = _first_monotone_violation(name, arr, 0, last)
        if v:
            return v
    segs_per_row = np.diff(rp.astype(np.int64))
    seg_row = np.repeat(np.arange(m), segs_per_row)
    seg_len = np.diff(op.astype(np.int64))
    v = _first_column_violation(col, op, n, np.repeat(seg_row, seg_len))
    if v:
        return v
    if enc["kind"] == "cer":
        over = np.flatnonzero(segs_per_row > k - 1)
        if over.size:
            r = int(over[0])
            return ("rowPtr", r + 1,
                    f"row holds {int(segs_per_row[r])} segments, alphabet has {k - 1} non-background elements")
        if segs:
            last_seg = (rp.astype(np.int64)[1:] - 1)[segs_per_row > 0]
            hollow = np.flatnonzero(seg_len[last_seg] == 0)
            if hollow.size:
                return ("omegaPtr", int(last_seg[hollow[0]]) + 1, "trailing empty segment")
        return None
    oi = np.asarray(enc["omegaI"])
    mode = int(enc["mode_index"])
    if np.any(np.diff(omega) <= 0):
        return ("omega", 0, "alphabet must be value-ascending")
    if oi.size != segs:
        return ("omegaI", 0, f"expected {segs} entries, found {oi.size}")
    if not 0 <= mode < k:
        return ("omega", mode, "mode_index out of range")
    o = oi.astype(np.int64)
    for bad, reason in ((o >= k, "element index out of range"),
                        (o == mode, "segment references the background element")):
        hit = np.flatnonzero(bad)
        if hit.size:
            return ("omegaI", int(hit[0]), reason)
    hollow = np.flatnonzero(seg_len == 0)
    if hollow.size:
        return ("omegaPtr", int(hollow[0]) + 1, "empty segment")
    dup = _first_duplicate(seg_row * k + o)
    if dup is not None:
        return ("omegaI", dup, "row references an element twice")
    return None


def decode(enc: dict) -> np.ndarray:
    """Dense float64 reconstruction (formats.py:395-424); the encoding must be valid."""
    omega = np.asarray(enc["omega"], dtype=np.float64)
    op, rp = np.asarray(enc["omegaPtr"]).astype(np.int64), np.asarray(enc["rowPtr"]).astype(np.int64)
    m, n = int(enc["m"]), int(enc["n"])
    seg_row = np.repeat(np.arange(m), np.diff(rp))
    seg_len = np.diff(op)
    if enc["kind"] == "cer":
        bg = omega[0]
        seg_val = omega[np.arange(seg_len.size) - rp[:-1][seg_row] + 1]
    else:
        bg = omega[int(enc["mode_index"])]
        seg_val = omega[np.asarray(enc["omegaI"]).astype(np.int64)]
    out = np.full((m, n), bg)
    out[np.repeat(seg_row, seg_len), np.asarray(enc["colI"]).astype(np.int64)] = np.repeat(seg_val, seg_len)
    return out
