"""Associative scans (counterpart of reference ``pintoc/scan.py``).

``scan_plan`` / ``scan_depth_probe`` keep the reference's meaning
(scan.py:51-92): the (src, dst) combine levels of the work-efficient
up-sweep / down-sweep schedule and its critical path, bounded by
2*ceil(log2 n).  ``scan`` runs that schedule with every level as ONE batched
device launch of the path's combines (value_combine, costate_combine,
rollout_combine over their element tuples); a user combine is applied pair
by pair in the same schedule (it is the caller's Python function, so the
caller's code decides where it computes).

The solver's passes do not go through ``scan``: every pass runs the blocked
K-ary device tree of csrc/common.cuh ``make_plan`` (level-0 threads fold
``chunk0`` stages, higher levels ``chunk`` aggregates).  ``device_scan_plan``
/ ``device_scan_depth`` describe that schedule so its logarithmic span can
be checked without a GPU.
"""

from __future__ import annotations

import math

from .exceptions import EmptySequenceError

SEQUENTIAL = "sequential"
PARALLEL = "parallel"
EXECUTORS = (SEQUENTIAL, PARALLEL, "auto")
DEFAULT_PARALLEL_THRESHOLD = 32


class ScanDirection:
    """FORWARD: out[t] = a_0 * ... * a_t;  REVERSE: out[t] = a_t * ... * a_{n-1}
    (scan.py:36-38; string values as the reference enum's)."""
    FORWARD = "forward"
    REVERSE = "reverse"


# ------------------------------------------------- reference-shaped schedule

def scan_plan(n: int) -> list[list[tuple[int, int]]]:
    """Levels of (src, dst) pairs, buf[dst] = combine(buf[src], buf[dst]) with
    src < dst; pairs of one level have distinct destinations (scan.py:51-75).
    Up-sweep: at stride s = 2^l every dst = 2s-1, 4s-1, ... takes dst - s;
    down-sweep: strides back down, every dst = 3s-1, 5s-1, ... takes dst - s."""
    if n < 1:
        raise EmptySequenceError("scan plan requires at least one element")
    levels: list[list[tuple[int, int]]] = []
    if n == 1:
        return levels
    top = math.ceil(math.log2(n))
    for lev in range(top):
        s = 1 << lev
        pairs = [(dst - s, dst) for dst in range(2 * s - 1, n, 2 * s)]
        if pairs:
            levels.append(pairs)
    for lev in range(top - 2, -1, -1):
        s = 1 << lev
        pairs = [(dst - s, dst) for dst in range(3 * s - 1, n, 2 * s)]
        if pairs:
            levels.append(pairs)
    return levels


def scan_depth_probe(n: int) -> int:
    """Critical path (dependent combines) of scan_plan(n); <= 2*ceil(log2 n)
    (scan.py:78-92)."""
    if n < 1:
        raise EmptySequenceError("depth probe requires n >= 1")
    depth = [0] * n
    for level in scan_plan(n):
        for src, dst in level:
            depth[dst] = max(depth[src], depth[dst]) + 1
    return max(depth)


# ------------------------------------------------ the solver's device tree

def device_scan_plan(n: int, chunk0: int = 4, chunk: int = 8) -> list[int]:
    """Item counts per level of the device tree: [n, n_1, ..., n_L] (mirror
    of csrc/common.cuh make_plan)."""
    if n < 1:
        raise EmptySequenceError("scan plan requires at least one element")
    chunk = max(2, chunk)
    chunk0 = max(1, min(chunk0, n))
    levels = [n]
    n1 = -(-n // chunk0)
    if n1 <= 1:
        return levels
    levels.append(n1)
    while levels[-1] > chunk:
        levels.append(-(-levels[-1] // chunk))
    return levels


def device_scan_depth(n: int, chunk0: int = 4, chunk: int = 8) -> int:
    """Critical path of the device tree for n items: up-sweep folds, the top
    walk and the down-sweep steps (2 (K0 + K L) for L levels)."""
    lv = device_scan_plan(n, chunk0, chunk)
    if n == 1:
        return 0
    if len(lv) == 1:
        return 2 * (n - 1)
    k0 = min(chunk0, n)
    L = len(lv) - 1
    up = (k0 - 1) + (L - 1) * (chunk - 1)
    top = lv[-1]
    down = (L - 1) * chunk + k0
    return up + top + down


# ------------------------------------------------------------------ scan()

def _device_kind(combine):
    from . import passes
    return {passes.value_combine: passes.ValueElement,
            passes.costate_combine: passes.CostateElement,
            passes.rollout_combine: passes.RolloutElement}.get(combine)


def _run_batched(elements, combine, kind, plan):
    """Every level of `plan` as one batched device combine."""
    import numpy as np
    buf = kind(*[np.stack([np.asarray(e[k], float) for e in elements])
                 for k in range(len(kind._fields))])
    for level in plan:
        src = np.array([p[0] for p in level])
        dst = np.array([p[1] for p in level])
        new = combine(kind(*[f[src] for f in buf]), kind(*[f[dst] for f in buf]))
        for f, g in zip(buf, new):
            f[dst] = g
    return [kind(*[f[t] for f in buf]) for t in range(len(elements))]


def scan(elements, combine, direction=ScanDirection.FORWARD, executor: str = SEQUENTIAL,
         parallel_threshold: int = DEFAULT_PARALLEL_THRESHOLD) -> list:
    """All partial folds of ``elements`` under an associative ``combine``
    (scan.py:133-169); ``combine(a, b)`` always has ``a`` preceding ``b``.
    The sequential executor (and inputs shorter than ``parallel_threshold``)
    folds left to right; the parallel executor runs scan_plan's levels, a
    reverse scan on the mirrored sequence with the operands flipped.  The
    path's combines run each level as one batched device launch."""
    direction = getattr(direction, "value", direction)
    if direction not in (ScanDirection.FORWARD, ScanDirection.REVERSE):
        raise ValueError(f"unknown direction {direction!r}")
    if executor not in EXECUTORS:
        raise ValueError(f"unknown executor {executor!r}; expected one of {EXECUTORS}")
    n = len(elements)
    if n == 0:
        raise EmptySequenceError("cannot scan an empty sequence")
    forward = direction == ScanDirection.FORWARD
    seq = list(elements) if forward else list(reversed(elements))
    op = combine if forward else (lambda a, b: combine(b, a))
    if executor == SEQUENTIAL or n < max(2, parallel_threshold):
        # a left fold is the chain plan: level k = [(k-1, k)]
        plan = [[(k - 1, k)] for k in range(1, n)]
    else:
        plan = scan_plan(n)
    kind = _device_kind(combine)
    if kind is not None:
        out = _run_batched(seq, op, kind, plan)
    else:
        out = list(seq)
        for level in plan:
            for src, dst in level:
                out[dst] = op(out[src], out[dst])
    return out if forward else out[::-1]
