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


ABI_STRUCTS = {  # C typedef (include/gsls.h) -> the ctypes mirror the Python shim passes
    "gsls_dims_t": _native.Dims, "gsls_error_t": _native.Error, "gsls_qp_t": _native.Qp,
    "gsls_admm_settings_t": _native.AdmmSettings, "gsls_admm_state_t": _native.AdmmState,
    "gsls_admm_stats_t": _native.AdmmStats, "gsls_linearize_args_t": _native.LinArgs,
    "gsls_rollout_args_t": _native.RolloutArgs, "gsls_rollout_out_t": _native.RolloutOut,
    "gsls_rti_step_args_t": _native.RtiStepArgs,
}


def test_abi_struct_layouts_match_header(tmp_path):
    """Every struct the C ABI takes has the same size and field offsets in C (gcc on
    include/gsls.h) as in its ctypes mirror."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "gsls.h"', "int main(void) {"]
    for cname, py in ABI_STRUCTS.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], check=True, capture_output=True,
                                                                   text=True).stdout.splitlines())
    for cname, py in ABI_STRUCTS.items():
        assert int(got[f"{cname} size"]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname} {f}"]) == getattr(py, f).offset, (cname, f)


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


@pytest.mark.parametrize("length", [1, 2, 3, 8, 17, 26, 51, 100])
@pytest.mark.parametrize("reverse", [False, True])
def test_layer_counter_matches_reference(length, reverse):
    """scan.tree_scan's LayerCounter counts layers and combines as the reference's tree_scan
    (scan.py:46-51, :190-229) does, padding combines included (the oracle's tally)."""
    mats = [np.array([[1, i], [0, 1]]) for i in range(length)]
    c = scan.LayerCounter()
    ours = scan.tree_scan(mats, lambda a, b: a @ b, np.eye(2, dtype=np.int64), reverse=reverse, counter=c)
    t = tree.Tally()
    ref = tree.scan_list(mats, lambda a, b: a @ b, np.eye(2, dtype=np.int64), reverse=reverse, tally=t)
    assert all((a == b).all() for a, b in zip(ours, ref))
    assert (c.layers, c.combines) == (t.layers, t.combines)


def test_plan_golden_integers():
    g = load_golden("scan")
    ints = g["ints"].tolist()
    for rev, key in ((False, "fwd"), (True, "rev")):
        out = scan.run_plan(scan.tree_plan(len(ints), rev), ints, lambda a, b: a + b, 0)
        assert out == g[key].tolist()


def test_plan_rejects_empty():
    with pytest.raises(ValueError, match="empty scan"):
        scan.tree_plan(0)
