"""Scan-tree helpers mirroring ``scanmpc.scan`` (scan.py:33-51).

The combine order itself lives in csrc/plan.h (the reference tree of
scan.py:141-234 flattened into layers of independent ops); ``tree_plan``
exposes it through the C ABI for inspection and tests.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat


def next_pow2(n: int) -> int:
    """scan.py:33-36."""
    if n < 1:
        raise ValueError("length must be >= 1")
    return 1 << (n - 1).bit_length()


def scan_depth(length: int) -> int:
    """Combine layers (upsweep + downsweep) of a scan of ``length`` (scan.py:39-43)."""
    if length < 1:
        raise ValueError("length must be >= 1")
    return 2 * (next_pow2(length).bit_length() - 1)


@dataclass
class LayerCounter:
    """scan.py:46-51: layers and combines a scan executes.  The reference counts every
    combine of its power-of-two padded tree (scan.py:190, :208, :229); the device plan
    elides the identity combines, so ``count`` restates the reference's numbers."""

    layers: int = 0
    combines: int = 0

    def count(self, length: int) -> "LayerCounter":
        """Add one scan of ``length`` elements: 2 log2(p) layers and 2 (p - 1) - log2(p)
        combines for p = next_pow2(length) (upsweep p - 1, downsweep sum of width - 1)."""
        p = next_pow2(length)
        lg = p.bit_length() - 1
        self.layers += 2 * lg
        self.combines += 2 * (p - 1) - lg
        return self


@dataclass
class TreePlan:
    ops: np.ndarray        # (n_ops, 3): dst, earlier, later (time order)
    layer_off: np.ndarray  # (layers + 1,)
    out: np.ndarray        # (length,) output slot per position (-1: identity)

    @property
    def layers(self) -> int:
        return len(self.layer_off) - 1


def tree_plan(length: int, reverse: bool = False) -> TreePlan:
    """The device combine schedule for a scan of ``length`` elements (host-side, no GPU)."""
    lib = nat.load(require_device=False)
    n_ops, n_layers = ctypes.c_int32(), ctypes.c_int32()
    i32 = ctypes.POINTER(ctypes.c_int32)
    z = np.zeros(1, np.int32)
    nat.check(lib.gsls_scan_plan(int(length), int(reverse), 0, z.ctypes.data_as(i32), z.ctypes.data_as(i32),
                                 z.ctypes.data_as(i32), ctypes.byref(n_ops), ctypes.byref(n_layers)),
              "gsls_scan_plan")
    ops = np.zeros((max(n_ops.value, 1), 3), np.int32)
    loff = np.zeros(n_layers.value + 1, np.int32)
    out = np.zeros(length, np.int32)
    nat.check(lib.gsls_scan_plan(int(length), int(reverse), n_ops.value, ops.ctypes.data_as(i32),
                                 loff.ctypes.data_as(i32), out.ctypes.data_as(i32), ctypes.byref(n_ops),
                                 ctypes.byref(n_layers)), "gsls_scan_plan")
    return TreePlan(ops[: n_ops.value], loff, out)


def tree_scan(values: list, combine, identity, reverse: bool = False, counter: LayerCounter | None = None):
    """scan.tree_scan (scan.py:141-234) on host objects through the device schedule: the
    inclusive scan in time order (reverse: suffix scan), combine(earlier, later); ``counter``
    is incremented as the reference increments it."""
    out = run_plan(tree_plan(len(values), reverse), values, combine, identity)
    if counter is not None:
        counter.count(len(values))
    return out


def run_plan(plan: TreePlan, values: list, combine, identity):
    """Evaluate a plan on host objects (used to check the schedule against the oracle)."""
    slots = list(values)
    total = len(values) + len(plan.ops)
    slots += [None] * (total - len(values))
    for d, e, l in plan.ops:
        slots[d] = combine(slots[e], slots[l])
    return [identity if s < 0 else slots[s] for s in plan.out]
