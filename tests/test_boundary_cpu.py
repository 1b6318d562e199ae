"""Boundary checks that need no GPU: the C-ABI library loads and exports every
function declared in include/aimx.h; the binding's signature table covers them;
the product package has no oracle import and no CPU fallback."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "aimx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(aimx_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2009_02281_b200 import load_library
    return load_library()


def test_header_declares_north_star_calls():
    names = _declared()
    for n in ("aimx_setup", "aimx_set_frequency", "aimx_matvec", "aimx_sweep"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_binding_covers_abi():
    from paper_2009_02281_b200 import ABI_FUNCTIONS
    assert set(_declared()) == set(ABI_FUNCTIONS)


def test_status_strings_without_gpu(lib):
    assert lib.aimx_status_string(0) == b"ok"
    assert b"sm_100a" in lib.aimx_version()


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2009_02281_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f
                assert "oracle/" not in txt.replace("oracle/`", ""), f


def test_binding_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2009_02281_b200 import AIMx
    import aimx_inputs as inp
    m = inp.make_mesh(1)
    with pytest.raises(RuntimeError):
        AIMx(m.vertices, m.triangles, (16, 16, 4))


def test_cubins_are_sm100a(lib):
    import subprocess
    from paper_2009_02281_b200 import library_path
    out = subprocess.run(["cuobjdump", "-lelf", library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
