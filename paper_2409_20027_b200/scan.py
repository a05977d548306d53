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
