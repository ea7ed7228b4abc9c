"""CPU-side checks of the native library: it loads, exports every symbol the
C header declares, and its scan schedule reproduces the reference tree order
(checked through the oracle).  No kernel launches."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden
from oracle import tree
from paper_2604_07644_b200 import _native, scan

LIB = os.path.join(ROOT, "paper_2604_07644_b200", "libgsls.so")


def header_functions():
    text = open(os.path.join(ROOT, "include", "gsls.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t)\s+(gsls_\w+)\s*\(", text, re.M)))


def test_library_built_and_exports_header():
    assert os.path.exists(LIB), "run __graft_entry__.build()"
    lib = ctypes.CDLL(LIB)
    names = header_functions()
    assert len(names) >= 9
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.EXPORTS)
    assert _native.load(require_device=False).gsls_version() == 1


@pytest.mark.parametrize("length", [1, 2, 3, 8, 17, 26, 51, 100, 1000])
@pytest.mark.parametrize("reverse", [False, True])
def test_plan_matches_reference_tree(length, reverse):
    plan = scan.tree_plan(length, reverse)
    assert plan.layers == scan.scan_depth(length) == tree.depth(length)
    rng = np.random.default_rng(length)
    # non-commutative, associative: 2x2 integer matrix products (exact)
    mats = [rng.integers(-2, 3, (2, 2)) for _ in range(length)]
    ours = scan.run_plan(plan, mats, lambda a, b: a @ b, np.eye(2, dtype=np.int64))
    ref = tree.scan_list(mats, lambda a, b: a @ b, np.eye(2, dtype=np.int64), reverse=reverse)
    for a, b in zip(ours, ref):
        assert (a == b).all()
    # the same op order: strings record the exact parenthesization
    names = [f"x{i}" for i in range(length)]
    ours = scan.run_plan(plan, names, lambda a, b: f"({a}{b})", "")
    ref = tree.scan_list(names, lambda a, b: f"({a}{b})" if a and b else a + b, "", reverse=reverse)
    assert ours == ref


def test_plan_golden_integers():
    g = load_golden("scan")
    ints = g["ints"].tolist()
    for rev, key in ((False, "fwd"), (True, "rev")):
        out = scan.run_plan(scan.tree_plan(len(ints), rev), ints, lambda a, b: a + b, 0)
        assert out == g[key].tolist()


def test_plan_rejects_empty():
    with pytest.raises(ValueError, match="empty scan"):
        scan.tree_plan(0)
