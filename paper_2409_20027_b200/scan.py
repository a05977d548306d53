"""Schedule of the device scan tree (counterpart of reference ``scan.py``).

The reference's generic executor runs a Blelloch up/down sweep over Python
objects (scan.py:51-92).  On the device every pass uses the same blocked
K-ary tree (csrc/common.cuh ``make_plan``): level-0 threads fold ``chunk0``
stages sequentially, higher levels fold ``chunk`` aggregates, one thread
walks the <= ``chunk`` top items, and carries flow back down.  These helpers
describe that schedule so its logarithmic span can be checked without a GPU.
"""

from __future__ import annotations

from .exceptions import EmptySequenceError


def scan_plan(n: int, chunk0: int = 4, chunk: int = 8) -> list[int]:
    """Item counts per tree level: [n, n_1, ..., n_L] (mirror of make_plan)."""
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


def scan_depth_probe(n: int, chunk0: int = 4, chunk: int = 8) -> int:
    """Critical path (dependent combines) of the device schedule for n items:
    up-sweep folds, the top walk, and the down-sweep steps."""
    lv = scan_plan(n, chunk0, chunk)
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

SEQUENTIAL = "sequential"
PARALLEL = "parallel"
EXECUTORS = (SEQUENTIAL, PARALLEL, "auto")


class ScanDirection:
    """FORWARD: out[t] = a_0 * ... * a_t;  REVERSE: out[t] = a_t * ... * a_{n-1}
    (scan.py:36-38; string values as the reference enum's)."""
    FORWARD = "forward"
    REVERSE = "reverse"


def scan(elements, combine, direction=ScanDirection.FORWARD, executor: str = SEQUENTIAL,
         parallel_threshold: int = 32) -> list:
    """All partial folds of ``elements`` under one of the path's associative
    combines (scan.py:133-166), on the device: ``combine`` is
    ``value_combine``, ``costate_combine`` or ``rollout_combine`` and the
    elements their tuples.  Every executor runs the same log-depth schedule
    (ceil(log2 n) rounds; round d combines every item with the one d places
    earlier -- FORWARD -- or later -- REVERSE -- in one batched launch), so
    ``combine(a, b)`` always has ``a`` preceding ``b``.  Arbitrary Python
    combines have no device form and raise TypeError."""
    import numpy as np
    from . import passes
    direction = getattr(direction, "value", direction)
    if direction not in (ScanDirection.FORWARD, ScanDirection.REVERSE):
        raise ValueError(f"unknown direction {direction!r}")
    if executor not in EXECUTORS:
        raise ValueError(f"unknown executor {executor!r}; expected one of {EXECUTORS}")
    n = len(elements)
    if n == 0:
        raise EmptySequenceError("cannot scan an empty sequence")
    kinds = {passes.value_combine: passes.ValueElement,
             passes.costate_combine: passes.CostateElement,
             passes.rollout_combine: passes.RolloutElement}
    if combine not in kinds:
        raise TypeError("the device scan runs value_combine, costate_combine or "
                        "rollout_combine over their element tuples")
    kind = kinds[combine]
    buf = kind(*[np.stack([np.asarray(e[k], float) for e in elements])
                 for k in range(len(kind._fields))])
    d = 1
    while d < n:
        if direction == ScanDirection.FORWARD:
            earlier = kind(*[f[:n - d] for f in buf])
            later = kind(*[f[d:] for f in buf])
            new = combine(earlier, later)
            buf = kind(*[np.concatenate([f[:d], g]) for f, g in zip(buf, new)])
        else:
            earlier = kind(*[f[:n - d] for f in buf])
            later = kind(*[f[d:] for f in buf])
            new = combine(earlier, later)
            buf = kind(*[np.concatenate([g, f[n - d:]]) for f, g in zip(buf, new)])
        d *= 2
    return [kind(*[f[t] for f in buf]) for t in range(n)]
