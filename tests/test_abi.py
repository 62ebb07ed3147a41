"""CPU checks of the C ABI library: it builds for sm_100a, loads, and exports every symbol that
include/knng.h declares (no compute calls without a GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "knng.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([a-z_]+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n.startswith(("graph_", "partition_"))))


def test_header_declares_the_boundary():
    names = declared_functions()
    for want in ("graph_init", "graph_insert_batch", "graph_search", "partition_kmedoids", "graph_get_rows",
                 "graph_free", "graph_last_error"):
        assert want in names


def test_library_builds_loads_and_exports_all_symbols():
    from paper_1602_06819_b200 import build as B
    lib = B.build()
    import paper_1602_06819_b200 as pkg
    L = pkg.load_library()
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(r"\bT %s$" % name, out, flags=re.M), name


def test_cubin_targets_sm100a():
    from paper_1602_06819_b200 import build as B
    lib = B.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import numpy as np
    from paper_1602_06819_b200 import KnngGraph, KnngError
    with pytest.raises(KnngError) as e:
        KnngGraph(np.zeros((20, 4), np.uint8), 3)
    assert e.value.code == -6


def test_product_does_not_import_oracle():
    """The product path never imports, links or loads the oracle (test infrastructure only)."""
    import re as _re
    pkg = os.path.join(ROOT, "paper_1602_06819_b200")
    bad = _re.compile(r"(^\s*(from|import)\s+oracle\b)|liboracle|knng_oracle|\bor_[a-z_]+\(", _re.M)
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dp, f)).read()
                assert not bad.search(s), f
