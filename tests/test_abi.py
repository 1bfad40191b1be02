"""C-ABI checks that need no GPU: the library loads and exports every symbol
declared in include/fde.h; the binding's list matches the header."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "fde.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:int|void|const char\*|long long)\s+(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def so_path():
    from paper_1808_02937_b200 import build
    return build.build()


def test_header_declares_north_star_entry_points():
    names = header_functions()
    for f in ["sem_assemble", "hmatrix_build", "hlu_factor", "precond_apply", "stiffness_matvec", "solve"]:
        assert f in names


def test_library_exports_every_header_symbol(so_path):
    out = subprocess.check_output(["nm", "-D", "--defined-only", so_path]).decode()
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing


def test_library_loads_and_binding_resolves(so_path):
    from paper_1808_02937_b200 import fde
    L = fde.lib()
    for f in fde.EXPORTED:
        assert hasattr(L, f)
    assert set(fde.EXPORTED) <= set(header_functions())


def test_create_without_gpu_fails_loudly(so_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1808_02937_b200 import fde
    import ctypes
    h = ctypes.c_void_p()
    rc = fde.lib().fde_create(ctypes.byref(h), 0, None, None, 0, 1)
    assert rc == -11   # FDE_ECUDA: no CPU fallback
