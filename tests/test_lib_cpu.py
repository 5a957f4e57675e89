"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/h2f.h declares, the host-only scheduling primitive (greedy
colouring) is bit-exact with the oracle, and the package mirrors the
reference's path API.  No CUDA compute calls here."""
import inspect

import numpy as np
from hypothesis import given, settings, strategies as st

import paper_2509_11152_b200 as H
from paper_2509_11152_b200 import _lib as L
from oracle import h2_oracle as O


def test_library_exports_header_symbols():
    lib = L.lib()
    declared = L.header_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(L._SIGS), "ctypes signatures out of sync with h2f.h"


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", L.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", L.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "DMMA" in sass  # FP64 tensor-core tiles in the GEMM kernel


@settings(max_examples=60, deadline=None)
@given(edges=st.lists(st.tuples(st.integers(0, 40), st.integers(0, 40)), max_size=200))
def test_greedy_coloring_bit_exact(edges):
    clusters = sorted({v for e in edges for v in e} | {0})
    pairs = [(min(a, b), max(a, b)) for a, b in edges]
    classes, degree = O.colour_classes(clusters, pairs)
    adj = H.level_graph(clusters, pairs)
    colour = H.greedy_coloring(adj)
    assert H.color_groups(colour) == classes
    assert max(len(v) for v in adj.values()) == degree


def test_api_mirrors_reference_signatures():
    sig = {
        "factorize": ["h2", "eps_lu", "threads", "norm_estimate"],
        "solve": ["fac", "b", "threads"],
        "solve_multi": ["fac", "b", "threads"],
        "refined_solve": ["h2", "fac", "b", "threads", "steps"],
        "matvec": ["h2", "x"],
        "estimate_norm2": ["h2", "iters", "seed"],
    }
    for name, params in sig.items():
        assert list(inspect.signature(getattr(H, name)).parameters) == params, name
    assert issubclass(H.FactorizationError, RuntimeError)
    assert H.PIVOT_RTOL == O.PIVOT_RTOL and H.FILL_DROP_FACTOR == O.FILL_DROP_FACTOR


def test_sparsity_constants_frozen_profiles():
    # structure.py frozen C_sp profiles (reference tests/test_structure.py:46-59)
    pts, _ = H.generate_uniform_grid(2 ** 14, 2)
    tree = H.build_cluster_tree(pts, 64)
    part = H.dual_tree_traversal(tree, 0.9)
    assert [H.sparsity_constant(part, lv) for lv in part.levels()] == [1, 2, 4, 7, 9, 11, 9, 11, 9]
    pts, _ = H.generate_uniform_grid(2 ** 15, 3)
    tree = H.build_cluster_tree(pts, 64)
    part = H.dual_tree_traversal(tree, 0.7)
    assert [H.sparsity_constant(part, lv) for lv in part.levels()] == [1, 2, 4, 8, 16, 31, 51, 69, 78, 81]


def test_grid_counts():
    assert H.generate_uniform_grid(2 ** 20, 3)[1] == (128, 128, 64)
    assert H.generate_uniform_grid(1023, 2)[1] == (33, 31)
    assert H.generate_uniform_grid(2 ** 17, 3)[1] == (64, 64, 32)


def test_struct_layouts_match_header(tmp_path):
    # the ctypes mirrors of the C-ABI structs have the header's size and
    # field offsets (compiled with the host C compiler)
    import ctypes as C
    import os
    import subprocess

    structs = {"h2f_matrix_desc": L.MatrixDesc, "h2f_build_desc": L.BuildDesc, "h2f_factor_info": L.FactorInfo,
               "h2f_status": L.Status, "h2f_comm": L.Comm}
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "h2f.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f in py._fields_:
            lines.append(f'printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        s, f, v = line.split()
        got[(s, f)] = int(v)
    for cname, py in structs.items():
        assert got[(cname, "sizeof")] == C.sizeof(py), cname
        for f in py._fields_:
            assert got[(cname, f[0])] == getattr(py, f[0]).offset, (cname, f[0])
