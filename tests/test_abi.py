"""The C-ABI boundary without a GPU: librpca.so loads and
exports every entry point include/rpca.h declares, the binding's ctypes table
names only declared symbols, and every product call fails loudly (no CPU
fallback) when no GPU is present."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rpca.h")
LIB = os.path.join(ROOT, "paper_1412_3510_b200", "librpca.so")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", " ", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rpca_[a-z0-9_]+)\s*\(", txt)))


def test_header_is_plain_c():
    """rpca.h compiles as C99 (no torch / C++ types in the signatures)."""
    src = f'#include "{HEADER}"\nint main(void) {{ return 0; }}\n'
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-x", "c", "-", "-fsyntax-only"], input=src,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_library_exports_every_declared_symbol():
    names = declared()
    assert len(names) >= 30, names
    lib = ctypes.CDLL(LIB)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (rpca_[a-z0-9_]+)", out))
    assert set(names) <= exported
    assert exported <= set(names), exported - set(names)  # nothing undocumented


def test_binding_signatures_cover_the_header():
    import paper_1412_3510_b200 as rp
    src = open(rp.__file__).read()
    bound = set(re.findall(r'"(rpca_[a-z0-9_]+)":', src))
    assert bound <= set(declared()), bound - set(declared())
    # the host-only string helpers are bound separately
    assert set(declared()) - bound <= {"rpca_last_error", "rpca_strerror"}


def test_status_strings_without_gpu():
    lib = ctypes.CDLL(LIB)
    lib.rpca_strerror.restype = ctypes.c_char_p
    assert lib.rpca_strerror(0) == b"ok"
    assert lib.rpca_strerror(3) == b"non-finite input"
    assert lib.rpca_strerror(7) == b"workspace too small"


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    import paper_1412_3510_b200 as rp
    A = torch.randn(50, 20, dtype=torch.float64)
    for call in (lambda: rp.pca(A, 3), lambda: rp.eigens(A[:20], 3), lambda: rp.omega(4, 2),
                 lambda: rp.diffsnorm(A, A[:, :1], A[0, :1], A[:1].T)):
        with pytest.raises(RuntimeError):
            call()
