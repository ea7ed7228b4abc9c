"""Oracle (test infrastructure): balanced-tree inclusive scan.

Restates the combine order of ``scanmpc.scan.tree_scan``
(/root/reference/pkg/src/scanmpc/scan.py:141-234):

* pad to the next power of two with identity elements (scan.py:175-177);
* upsweep: level d+1 combines pairs (2i, 2i+1) of level d (scan.py:200-209);
* downsweep: position 0 of each level keeps its upsweep value, position i
  gets ``acc[i-1] (x) left_child[i]``, then interleave with the parent
  (scan.py:211-229); a level of width one counts as a (skipped) layer;
* reverse direction = reverse the input and swap the operands
  (scan.py:169-173).

Every layer is evaluated as one batched call — the same arithmetic the
reference's ParallelExecutor performs for layers under its 64-combine
chunking threshold (scan.py:118-120).
"""

from __future__ import annotations

import numpy as np


def pow2_ceil(n: int) -> int:
    """scan.py:33-36."""
    if n < 1:
        raise ValueError("length must be >= 1")
    return 1 << (n - 1).bit_length()


def depth(length: int) -> int:
    """Layers (up + down) of a scan of ``length`` (scan.py:39-43)."""
    return 2 * (pow2_ceil(length).bit_length() - 1)


class Tally:
    """Layer / combine counters (scan.py:46-51)."""

    def __init__(self):
        self.layers = 0
        self.combines = 0


def _take(group, sl):
    return tuple(np.ascontiguousarray(a[sl]) for a in group)


def _cat(g1, g2):
    return tuple(np.concatenate([a, b], axis=0) for a, b in zip(g1, g2))


def scan(elems, op, unit, *, reverse=False, record=False, replay=None, tally=None):
    """Inclusive scan of the tuple-of-arrays ``elems`` under ``op``.

    op(lhs, rhs[, aux]) -> (combined, aux_out); ``unit(k)`` returns k identity
    elements.  Returns (outputs, tape) where tape lists per-layer aux when
    ``record`` is set.  ``replay`` feeds a recorded tape back layer by layer.
    """
    count = len(elems[0])
    if count == 0:
        raise ValueError("empty scan")
    tally = tally if tally is not None else Tally()
    if reverse:
        work = _take(elems, slice(None, None, -1))
        fn = lambda a, b, *x: op(b, a, *x)  # noqa: E731
    else:
        work = tuple(np.asarray(a) for a in elems)
        fn = op
    width = pow2_ceil(count)
    if width > count:
        work = _cat(work, unit(width - count))

    tape = [] if record else None
    cursor = [0]

    def apply(lhs, rhs):
        extra = (replay[cursor[0]],) if replay is not None else ()
        out, aux = fn(lhs, rhs, *extra)
        if tape is not None:
            tape.append(aux)
        tally.combines += len(lhs[0])
        cursor[0] += 1
        return out

    levels = [work]
    while len(levels[-1][0]) > 1:
        cur = levels[-1]
        levels.append(apply(_take(cur, slice(0, None, 2)), _take(cur, slice(1, None, 2))))
        tally.layers += 1

    acc = levels[-1]
    for lvl in range(len(levels) - 2, -1, -1):
        w = len(acc[0])
        lefts = _take(levels[lvl], slice(0, None, 2))
        if w > 1:
            mixed = apply(_take(acc, slice(0, w - 1)), _take(lefts, slice(1, None)))
            head = _cat(_take(lefts, slice(0, 1)), mixed)
        else:
            head = _take(lefts, slice(0, 1))
            if tape is not None:
                tape.append(())
            cursor[0] += 1
        merged = []
        for h, a in zip(head, acc):
            z = np.empty((2 * w,) + a.shape[1:], dtype=a.dtype)
            z[0::2] = h
            z[1::2] = a
            merged.append(z)
        acc = tuple(merged)
        tally.layers += 1

    out = _take(acc, slice(0, count))
    if reverse:
        out = _take(out, slice(None, None, -1))
    return out, tape


def scan_list(items, combine, identity, reverse=False, tally=None):
    """Object-level scan used by the scan tests (scan.py:237-280)."""
    items = list(items)
    if not items:
        raise ValueError("empty scan")

    def pack(vals):
        arr = np.empty(len(vals), dtype=object)
        for i, v in enumerate(vals):
            arr[i] = v
        return arr

    def op(lhs, rhs):
        a, b = lhs[0], rhs[0]
        return (pack([combine(a[i], b[i]) for i in range(len(a))]),), ()

    out, _ = scan((pack(items),), op, lambda k: (pack([identity] * k),),
                  reverse=reverse, tally=tally)
    return list(out[0])
