"""CPU-side checks of the C-ABI library (no compute calls need a GPU here):
it loads, exports every symbol include/jf.h declares, and its host-side
validation and metadata behave as documented."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2208_12187_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "jf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(jf_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = L.load()
    names = _declared_functions()
    assert len(names) >= 15
    for nm in names:
        assert hasattr(lib, nm), nm
    assert set(L.EXPORTED) == set(names)


def test_model_metadata():
    lib = L.load()
    assert [lib.jf_model_nparams(k) for k in range(5)] == [2, 3, 4, 7, 13]
    assert [lib.jf_model_ydim(k) for k in range(5)] == [1, 1, 1, 2, 2]
    assert [lib.jf_model_kslots(k) for k in range(5)] == [7, 11, 16, 37, 106]
    assert lib.jf_model_nparams(99) == -1
    assert b"sm_100a" in lib.jf_version()


def test_opts_defaults():
    lib = L.load()
    o = L.jf_opts()
    lib.jf_opts_default(C.byref(o))
    assert (o.ftol, o.xtol, o.gtol) == (1e-8, 1e-8, 1e-8)
    assert o.max_nfev == 0 and o.x_scale_mode == L.XSCALE_JAC and o.use_graph == 1
    assert o.policy == L.POLICY_SPECULATIVE and o.comm is None


def test_invalid_arguments_rejected_before_device_use():
    """R18 validation happens on the host: these return JF_EINVAL /
    JF_EINFEASIBLE even where no GPU exists."""
    lib = L.load()
    res = L.jf_result()
    z = np.ones(10)
    zp = z.ctypes.data
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    p0 = np.ones(3)
    # wrong n
    assert lib.jf_curve_fit(1, None, zp, 10, dp(p0), 4, None, None, None, C.byref(res)) == L.EINVAL
    assert res.status == L.EINVAL
    # lb >= ub
    lb = np.array([0.0, 0.0, 1.0])
    ub = np.array([2.0, 2.0, 1.0])
    assert lib.jf_curve_fit(1, None, zp, 10, dp(p0), 3, dp(lb), dp(ub), None, C.byref(res)) == L.EINVAL
    # infeasible p0
    lb = np.array([0.0, 0.0, 2.0])
    ub = np.array([2.0, 2.0, 3.0])
    assert lib.jf_curve_fit(1, None, zp, 10, dp(p0), 3, dp(lb), dp(ub), None, C.byref(res)) == L.EINFEASIBLE
    # null output
    assert lib.jf_curve_fit(1, None, zp, 10, dp(p0), 3, None, None, None, None) == L.EINVAL
    assert lib.jf_strerror(L.EINFEASIBLE) == b"initial guess outside the bounds"


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2208_12187_b200")
    for dp_, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp_, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("no CPU fallback", ""), f
