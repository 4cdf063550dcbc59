"""CPU checks of the boundary: the library builds for sm_100a, loads, and exports every
symbol include/lv.h declares; the product package never imports the oracle."""
import ast
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "lv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lv_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2410_22347_b200 import build
    lib = build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (lv_\w+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    from paper_2410_22347_b200 import lv
    L = lv.lib()
    for s in _declared():
        assert hasattr(L, s)
    assert set(lv.EXPORTS) == set(_declared())


def test_sass_has_tcgen05_and_tma():
    from paper_2410_22347_b200 import build
    lib = build.build()
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "no tcgen05.mma in the binary"
    assert "UTMALDG" in sass, "no TMA loads in the binary"
    assert "LDTM" in sass, "no tcgen05.ld in the binary"


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2410_22347_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            tree = ast.parse(open(os.path.join(pkg, fn)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert all(not a.name.startswith("oracle") for a in node.names), fn
                if isinstance(node, ast.ImportFrom):
                    assert not (node.module or "").startswith("oracle"), fn
    for fn in os.listdir(os.path.join(ROOT, "oracle")):
        if fn.endswith(".py"):
            tree = ast.parse(open(os.path.join(ROOT, "oracle", fn)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert all(not a.name.startswith("paper_2410") for a in node.names), fn
                if isinstance(node, ast.ImportFrom):
                    assert not (node.module or "").startswith("paper_2410"), fn


def test_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2410_22347_b200 import lv
    with pytest.raises(lv.LVError):
        lv.lv_fit_stats(torch.zeros(2, 4), torch.zeros(2, 4))
