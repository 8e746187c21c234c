"""CPU tests of the C-ABI boundary: the libraries build and load, every
symbol include/*.h declares is exported, the ctypes mirror of poly_problem
matches the C layout, and host-side argument validation rejects bad input
 before any device work."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    from paper_2503_19925_b200 import build
    build.build()
    return True


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b((?:poly|polysynth)_[a-z_0-9]+)\s*\(", txt)))


def test_headers_declare_the_boundary():
    names = _declared("poly.h")
    for n in ("poly_init", "poly_loss_grad", "poly_solve", "poly_free", "poly_last_error"):
        assert n in names


@pytest.mark.parametrize("header,lib", [("poly.h", "libpoly.so"), ("polysynth.h", "libpolysynth.so")])
def test_library_exports_every_declared_symbol(built, header, lib):
    path = os.path.join(ROOT, "paper_2503_19925_b200", lib)
    L = C.CDLL(path)
    for n in _declared(header):
        assert hasattr(L, n), f"{lib} does not export {n}"
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    for n in _declared(header):
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_problem_struct_layout_matches_c(built, tmp_path):
    import paper_2503_19925_b200 as P
    fields = [f for f, _ in P.PolyProblem._fields_]
    src = tmp_path / "lay.c"
    body = "\n".join(f'printf("{f} %zu\\n", offsetof(poly_problem, {f}));' for f in fields)
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "poly.h"\nint main(void){'
                   f'printf("size %zu\\n", sizeof(poly_problem));{body}return 0;}}\n')
    exe = tmp_path / "lay"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = dict(line.split() for line in subprocess.check_output([str(exe)], text=True).splitlines())
    assert int(got["size"]) == C.sizeof(P.PolyProblem)
    for f in fields:
        assert int(got[f]) == getattr(P.PolyProblem, f).offset, f


def _problem(**kw):
    import paper_2503_19925_b200 as P
    p = P.PolyProblem()
    s = (C.c_double * 2)(0.25, 0.75)
    mu = (C.c_double * 2)(1.0, 2.0)
    p.n_local, p.n_global, p.d = 10, 10, 8
    p.layout, p.dtype, p.A, p.lda = P.POLY_DENSE, P.POLY_F32, 0x1000, 8
    p.ytype, p.y, p.W = P.POLY_Y_I32, 0x2000, 2
    p.s, p.mu = C.addressof(s), C.addressof(mu)
    p.I_bar, p.relu, p.set, p.R = 100.0, 1, P.POLY_SET_BALL, 1.0
    p.rank, p.world = 0, 1
    p._keep = (s, mu)
    for k, v in kw.items():
        if k == "s":
            arr = (C.c_double * len(v))(*v)
            p.s, p.W = C.addressof(arr), len(v)
            p._keep2 = arr
        elif k == "mu":
            arr = (C.c_double * len(v))(*v)
            p.mu = C.addressof(arr)
            p._keep3 = arr
        else:
            setattr(p, k, v)
    return p


@pytest.mark.parametrize("kw,code", [
    (dict(W=0), 1), (dict(s=[0.5, 0.6]), 1), (dict(s=[1.0, 0.0]), 1), (dict(mu=[1.0, -1.0]), 1),
    (dict(I_bar=0.0), 1), (dict(R=0.0), 1), (dict(set=3, center=0x3000), 1),
    (dict(world=2), 1), (dict(rank=1), 1), (dict(lda=7), 1), (dict(lda=10), 1), (dict(A=0x1004), 1),
    (dict(n_global=5), 1), (dict(d=0), 1), (dict(y=0), 1), (dict(W=65, s=[1.0 / 65] * 65, mu=[1.0] * 65), 6),
    (dict(layout=1, row_ptr=0), 1), (dict(s_row=0x4000), 1), (dict(relu=2), 1),
    (dict(mode=4), 1), (dict(mode=-1), 1), (dict(windows=-1), 1), (dict(windows=2), 1),
    (dict(flags=8), 1),
])
def test_init_validation(built, kw, code):
    import paper_2503_19925_b200 as P
    p = _problem(**kw)
    h = C.c_void_p()
    rc = P.lib().poly_init(C.byref(p), C.byref(h))
    assert rc == code, P.poly_last_error()
    assert h.value is None
    assert P.poly_last_error()


def test_windows_validation(built):
    """Ω = 2 windows: s is [Ω*W]; each window must be a spectrum; I_win > 0;
    baseline modes and per-row spectra are not supported with windows."""
    import paper_2503_19925_b200 as P
    L = P.lib()
    for s, I, mode, code in [([0.25, 0.75, 0.5, 0.6], (1.0, 2.0), 0, 1),
                             ([0.25, 0.75, 0.5, 0.5], (1.0, 0.0), 0, 1),
                             ([0.25, 0.75, 0.5, 0.5], (1.0, 2.0), 1, 6)]:
        p = _problem()
        sa = (C.c_double * 4)(*s)
        ia = (C.c_double * 2)(*I)
        p.s, p.W, p.windows, p.I_win, p.mode = C.addressof(sa), 2, 2, C.addressof(ia), mode
        h = C.c_void_p()
        assert L.poly_init(C.byref(p), C.byref(h)) == code, P.poly_last_error()


def test_reparameterize_validation(built):
    import paper_2503_19925_b200 as P
    s = (C.c_double * 2)(0.5, 0.5)
    mu = (C.c_double * 2)(1.0, 2.0)
    L = P.lib()
    assert L.poly_reparameterize(0, s, mu, 1.0, 4, 0x1000, 1, 0x2000, 0x3000, None) == P.POLY_EINVAL
    assert L.poly_reparameterize(2, s, mu, -1.0, 4, 0x1000, 1, 0x2000, 0x3000, None) == P.POLY_EINVAL
    assert L.poly_reparameterize(2, s, mu, 1.0, 4, None, 1, 0x2000, 0x3000, None) == P.POLY_EINVAL
    assert L.poly_reparameterize(2, s, mu, 1.0, 0, None, 1, None, None, None) == P.POLY_OK


def test_abi_version_and_null_handle(built):
    import paper_2503_19925_b200 as P
    assert P.poly_abi_version() == 5
    assert P.lib().poly_loss_grad(None, None, None, None) == P.POLY_EINVAL
    assert P.lib().poly_solve_ex(None, None, None, None, None) == P.POLY_EINVAL
    assert P.lib().poly_solve(None, None, 1, 1.0, 0, None, None) == P.POLY_EINVAL
    P.poly_free(None)


def test_no_cpu_fallback_import_guard(tmp_path, monkeypatch):
    """The package refuses to import without its CUDA library."""
    import importlib.util
    import shutil
    pkg = tmp_path / "paper_2503_19925_b200"
    shutil.copytree(os.path.join(ROOT, "paper_2503_19925_b200"), pkg,
                    ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    spec = importlib.util.spec_from_file_location("pkgcopy", pkg / "__init__.py",
                                                  submodule_search_locations=[str(pkg)])
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)


def test_product_does_not_reference_oracle():
    """The product path never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2503_19925_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f
