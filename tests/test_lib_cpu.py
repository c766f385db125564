"""CPU-side checks of the boundary: the C-ABI library builds/loads and exports every symbol
declared in include/svmhss.h (no compute calls without a GPU); the product package has no
dependency on oracle/."""
import ast
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "svmhss.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|void|const char\*)\s+(\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol():
    import __graft_entry__
    lib = __graft_entry__._builder().build()
    L = ctypes.CDLL(lib)
    names = _declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(L, n), n
    from paper_2108_04167_b200 import _lib
    assert sorted(_lib.EXPORTS) == names


def test_no_device_call_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2108_04167_b200 import _lib
    L = _lib.load()
    assert b"sm_100a" in L.hss_version()
    rc = L.hss_omega(1, None, 0, 1, None, None)
    assert rc != 0   # NULL pointer or no device: an error code, never a silent result


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2108_04167_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            tree = ast.parse(open(os.path.join(pkg, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert all(not a.name.startswith("oracle") for a in node.names), f
                if isinstance(node, ast.ImportFrom):
                    assert not (node.module or "").startswith("oracle"), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            tree = ast.parse(open(os.path.join(ROOT, "oracle", f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert all("paper_2108_04167_b200" not in a.name for a in node.names), f
                if isinstance(node, ast.ImportFrom):
                    assert "paper_2108_04167_b200" not in (node.module or ""), f


def test_datagen_is_deterministic():
    import numpy as np
    import datagen
    a = datagen.generate(3, n=100, n_test=10)
    b = datagen.generate(3, n=100, n_test=10)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    F, y, Ft, yt = datagen.generate(3, n=1000, n_test=10)
    assert F.shape == (1000, 54) and set(np.unique(y)) <= {-1.0, 1.0}
    assert np.array_equal(F[:, 10:14].sum(1), np.ones(1000)) and np.array_equal(F[:, 14:].sum(1), np.ones(1000))
    F2 = datagen.generate(2, n=2000, n_test=0)[0]
    assert set(np.unique(F2)) <= {0.0, 1.0} and abs(F2.mean() - 0.11) < 0.01
