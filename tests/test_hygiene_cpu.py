"""Separation rules between the product path, the oracle and the input generators:
the CUDA package never imports the oracle, the oracle never imports the package or the
generators, the generators import neither, the kernels include nothing from oracle/, and the
binding fails loudly when the CUDA library is missing (no fallback)."""
import ast
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = "paper_2205_01848_b200"


def _py_files(sub):
    base = os.path.join(ROOT, sub)
    for dp, _, fs in os.walk(base):
        if "_build" in dp:
            continue
        for f in fs:
            if f.endswith(".py"):
                yield os.path.join(dp, f)


def _imported(path):
    tree = ast.parse(open(path).read(), path)
    out = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            out.update(a.name.split(".")[0] for a in node.names)
        elif isinstance(node, ast.ImportFrom) and node.level == 0 and node.module:
            out.add(node.module.split(".")[0])
    return out


@pytest.mark.parametrize("sub,forbidden", [(PKG, {"oracle", "synth"}),
                                           ("oracle", {PKG, "synth", "torch"}),
                                           ("synth", {PKG, "oracle"})])
def test_import_separation(sub, forbidden):
    files = list(_py_files(sub))
    assert files
    for f in files:
        bad = _imported(f) & forbidden
        assert not bad, f"{os.path.relpath(f, ROOT)} imports {sorted(bad)}"


def test_kernels_include_nothing_from_oracle():
    csrc = os.path.join(ROOT, PKG, "csrc")
    inc = re.compile(r'#\s*include\s*[<"]([^>"]+)[>"]')
    n = 0
    for f in os.listdir(csrc):
        if f.endswith((".cu", ".cuh", ".h", ".cpp")):
            n += 1
            for m in inc.finditer(open(os.path.join(csrc, f)).read()):
                assert "oracle" not in m.group(1), (f, m.group(1))
    assert n > 0


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_2205_01848_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError, match="not built"):
        _lib.load()
