"""CPU-side checks of the boundary: libpht.so loads and exports every symbol include/pht.h
declares; the Python binding declares a signature for each; no compute call is made."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "pht.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pht_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2111_14317_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name


def test_binding_covers_header():
    from paper_2111_14317_b200 import _lib
    assert set(_header_functions()) == set(_lib.SIGNATURES)


def test_version_and_strerror_without_gpu():
    from paper_2111_14317_b200 import _lib
    lib = _lib.load()
    assert lib.pht_version() == 4
    assert lib.pht_strerror(-3).decode().startswith("duplicate")
    assert lib.pht_launch_count() >= 0


def test_create_rejects_bad_shapes_before_touching_the_device():
    """Validation errors are returned synchronously, before any CUDA call (so they work here)."""
    import numpy as np
    from paper_2111_14317_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    off = np.array([0, 2], np.int64)
    ex = np.array([[1], [1]], np.int32)           # duplicate monomial
    c = np.ones(2, np.complex128)
    w = np.zeros(2)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    assert lib.pht_system_create(1, 1, P(off), P(ex), P(c), P(w), 0, ctypes.byref(h)) == -3
    assert lib.pht_system_create(1, 2, P(off), P(ex), P(c), P(w), 0, ctypes.byref(h)) == -2
    ex2 = np.array([[1], [0]], np.int32)
    assert lib.pht_system_create(1, 1, P(off), P(ex2), P(np.zeros(2, np.complex128)), P(w), 0,
                                 ctypes.byref(h)) == -4
    assert lib.pht_system_create(1, 1, P(off), P(ex2), P(c), P(-np.ones(2)), 0, ctypes.byref(h)) == -5


def test_package_import_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_2111_14317_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError):
        _lib.load()


def test_specialize_codegen_without_gpu():
    """The code generator of pht_system_specialize (one straight-line row per equation, only the
    nonzero exponents touched) and its NVRTC compile for sm_100a run without a GPU."""
    import paper_2111_14317_b200 as P
    import workloads as W
    # cyclic-3: f1 = x1 + x2 + x3, f2 = x1x2 + x2x3 + x3x1, f3 = x1x2x3 - 1
    sysm = W.cyclic(3, lift_max=10)
    src = P.specialize_source(sysm)
    assert "jit_row<3>" in src and src.count("case ") == 3
    # 8 terms -> 8 exp*cis evaluations; the constant term of f3 has no variable in phi
    assert src.count("PHT_EXPCIS((p") == sysm.offsets[-1] == 8
    body3 = src[src.index("case 2:"):src.index("default:")]
    assert "(v0.x + v1.x) + v2.x" in body3 or "((v0.x + v1.x) + v2.x)" in body3
    # the G_j updates touch exactly the nonzero exponents: nnz(A) = 3 + 6 + 3 = 12 complex updates
    assert src.count(".x += w.x;") - src.count("h.x += w.x;") == 12
    nb = P.specialize_compile(sysm, P._lib.SPEC_STEP)
    assert nb > 0
    with pytest.raises(P.PhtError):
        P.specialize_compile(sysm, 64)


def test_packer_terms_are_monomial_lifting_pairs():
    """The same monomial with two liftings (x^a t^0 and x^a t^1 of the parameter homotopy) is two
    terms; the same (monomial, lifting) twice is PHT_EDUPLICATE.  pht_specialize_source runs the
    packer without a device."""
    import numpy as np
    from paper_2111_14317_b200 import _lib
    lib = _lib.load()
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    off = np.array([0, 2], np.int64)
    ex = np.array([[1], [1]], np.int32)
    c = np.ones(2, np.complex128)
    assert lib.pht_specialize_source(1, 1, P(off), P(ex), P(c), P(np.array([0.0, 1.0])), None, 0) > 0
    assert lib.pht_specialize_source(1, 1, P(off), P(ex), P(c), P(np.array([1.0, 1.0])), None, 0) == -3


def test_set_kernels_validates_without_gpu():
    from paper_2111_14317_b200 import _lib
    lib = _lib.load()
    assert lib.pht_system_set_kernels(None, _lib.KERNELS["auto"]) == -1   # NULL handle
    assert lib.pht_system_kernels(None) == -1


def test_pc_step_host_rejects_bad_host_buffers():
    """pht_pc_step_host reads/writes p*n*16 bytes of x and p*8 of tau/dtau/dn_norm;
    the binding refuses wrong dtype, shape, stride or read-only buffers before any C call."""
    import numpy as np
    import paper_2111_14317_b200 as P
    g = P.System.__new__(P.System)          # validation runs before the handle is touched
    g.n = 4
    p = 8
    x = np.ones((p, 4), np.complex128)
    tau = np.zeros(p)
    dtau = np.full(p, 0.01)
    bad = [
        (x.astype(np.complex64), tau, dtau, {}),
        (np.ones((p, 3), np.complex128), tau, dtau, {}),
        (np.ones((p, 8), np.complex128)[:, ::2], tau, dtau, {}),
        (x, tau[:-1], dtau, {}),
        (x, tau, dtau.astype(np.float32), {}),
        (x, tau, dtau, {"status": np.zeros(p, np.int32)}),
        (x, tau, dtau, {"dn_norm": np.zeros(p - 1)}),
    ]
    for xx, tt, dd, kw in bad:
        with pytest.raises(P.PhtError):
            g.pc_step_host(xx, tt, dd, 1, **kw)
    ro = x.copy()
    ro.flags.writeable = False
    with pytest.raises(P.PhtError):
        g.pc_step_host(ro, tau, dtau, 1)
