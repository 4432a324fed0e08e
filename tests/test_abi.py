"""The C ABI library loads, exports every function include/epicorr_b200.h
declares, and fails loudly (status code, no fallback) without a usable GPU.
CPU only: no kernel is launched."""
import ctypes as C
import os
import re

import pytest

from paper_1607_00531_b200 import _lib, abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "epicorr_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(epc_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for must in ("epc_admm_solve", "epc_gn_solve", "epc_b_update", "epc_z_update",
                 "epc_dual_update", "epc_pcg", "epc_gn_hessian_apply", "epc_qp_active_set_batch"):
        assert must in fns


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    missing = [f for f in header_functions() if not hasattr(L, f)]
    assert not missing, missing
    assert set(header_functions()) <= set(_lib.EXPORTS)


def test_library_is_sm100a_build():
    L = _lib.load()
    assert b"sm_100a" in L.epc_build_info()
    so = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in so or b"sm_100" in so


def test_defaults_match_reference():
    L = _lib.load()
    p, a, g = abi.ObjectiveParams(), abi.AdmmConfig(), abi.GnConfig()
    p2, a2, g2 = abi.ObjectiveParams(), abi.AdmmConfig(), abi.GnConfig()
    L.epc_default_params(C.byref(p2))
    L.epc_default_admm_config(C.byref(a2))
    L.epc_default_gn_config(C.byref(g2))
    for x, y in ((p, p2), (a, a2), (g, g2)):
        for name, _ in x._fields_:
            assert getattr(x, name) == getattr(y, name), name


def test_rho_schedule_host_logic():
    L = _lib.load()
    assert L.epc_rho_schedule(abi.RHO_ADAPTIVE, 8.0, 1.0, 20.0, 1.0, 2, 2, 10) == 16.0
    assert L.epc_rho_schedule(abi.RHO_ADAPTIVE_BOUNDED, 1.0, 1.0, 0.0, 100.0, 2, 2, 10) == 1.0


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = _lib.load()
    h = C.c_void_p()
    rc = L.epc_context_create(0, None, C.byref(h))
    assert rc in (abi.EPC_ERR_CUDA, abi.EPC_ERR_UNSUPPORTED)
    assert not h.value
    from paper_1607_00531_b200.epicorr import Context
    with pytest.raises((OSError, NotImplementedError)):
        Context(0)
