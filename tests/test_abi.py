"""CPU-side checks of the product boundary: the C-ABI library loads and
exports every symbol include/tsp.h declares (no compute calls without a GPU),
and the binding refuses to run without CUDA (no CPU fallback)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "tsp.h")).read()
    return sorted(set(re.findall(r"^\s*(?:tsp_status|int|void|const char \*)\s*\*?\s*(tsp_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("tsp_create", "tsp_setup", "tsp_apply_preconditioner", "tsp_apply_operator", "tsp_solve", "tsp_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = os.path.join(ROOT, "paper_1812_05540_b200", "libtsp.so")
    if not os.path.exists(lib):
        subprocess.check_call(["make", "-s", "-C", ROOT, "tsp"])
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib], text=True)
    exported = set(re.findall(r" T (tsp_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    from paper_1812_05540_b200 import lib as load, EXPORTED
    L = load()
    assert L.tsp_abi_version() == 5
    for n in EXPORTED:
        getattr(L, n)


def test_no_cpu_fallback_without_cuda():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import synth
    from paper_1812_05540_b200 import Tsp
    with pytest.raises(RuntimeError):
        Tsp(synth.generate("C1"))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1812_05540_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle/" not in txt and "orc_" not in txt, f
