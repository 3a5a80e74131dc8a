"""The C-ABI library builds for sm_100a, loads, and exports every symbol
include/specwalk.h declares (no compute calls: runs without a GPU)."""
import ctypes
import os
import re

import paper_2010_03817_b200 as sw

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "specwalk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set()
    for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M):
        name = m.group(1)
        if name not in {"if", "for", "while", "sizeof"}:
            names.add(name)
    return names


def test_library_builds_and_exports_header_symbols():
    path = sw._build.build()
    lib = ctypes.CDLL(path)
    declared = _declared_functions()
    assert {"spec_create", "boundary_oracle", "walk_sample"} <= declared
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in specwalk.h but not exported"
    assert declared <= set(sw.EXPORTS) | {"spec_last_error"}


def test_sass_has_dmma():
    """K1/K3 run on the FP64 tensor pipe (DMMA), not a scalar loop."""
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", sw._build.LIB], capture_output=True, text=True).stdout
    assert "DMMA" in out


def test_no_device_fails_loudly():
    """Without a CUDA device spec_create must fail (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        return
    import numpy as np
    try:
        sw.Spectrahedron(np.stack([np.eye(2), np.eye(2)]))
    except sw.SpecError as e:
        assert e.code == 4
    else:
        raise AssertionError("spec_create succeeded without a GPU")
