"""The C-ABI library loads without a GPU, exports every symbol declared in
include/bssmppi.h, its ctypes structs match the header layout, and the
product path fails loudly (no CPU fallback) when no CUDA device exists."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2408_00494_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent
HEADER = (ROOT / "include" / "bssmppi.h").read_text()


def declared_functions():
    body = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    return sorted(set(re.findall(r"\b(bssmppi_[a-z0-9_]+)\s*\(", body)))


def test_header_declares_the_api():
    names = declared_functions()
    assert "bssmppi_control_step" in names and "bssmppi_create" in names
    assert len(names) >= 18


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_abi_version_and_record_length():
    lib = _lib.load()
    assert lib.bssmppi_abi_version() == 3
    assert lib.bssmppi_partial_len(50) == 105


def _struct_fields(name):
    m = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), HEADER, re.S)
    body = re.sub(r"/\*.*?\*/", "", m.group(1), flags=re.S)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        for part in decl.split(","):
            nm = re.findall(r"\*?\s*([a-z_0-9]+)\s*(\[\d+\])?\s*$", part.strip())
            fields.append(nm[0][0])
    return fields


@pytest.mark.parametrize("cname,py", [("bssmppi_problem", _lib.Problem), ("bssmppi_diag", _lib.Diag)])
def test_struct_layout_matches_header(cname, py):
    assert _struct_fields(cname) == [f for f, _ in py._fields_]


def test_validation_before_cuda():
    """Argument errors are reported without touching CUDA (reference:
    ValueError at construction, controllers.py:85-105)."""
    lib = _lib.load()
    p = _lib.Problem()
    h = ctypes.c_void_p()
    assert lib.bssmppi_create(ctypes.byref(p), 0, ctypes.byref(h)) == _lib.ERR_INVALID
    assert b"samples" in lib.bssmppi_last_error()


def test_tire_table_limits_checked_before_cuda():
    """The lateral tire table (csrc/bssmppi.cu tire_table_host) covers every
    slip angle of a rollout, |alpha| <= pi + max |steering bound|: any
    magic-formula shape factor passes validation (C = 2.5 included), and
    steering bounds beyond +-2 pi -- or non-finite tire coefficients -- are
    refused at context creation, before any CUDA call."""
    from dataclasses import replace
    from helpers import Inputs
    from paper_2408_00494_b200 import controllers as mc

    inp = Inputs("c1_s0")
    lib = _lib.load()
    h = ctypes.c_void_p()

    def create(model, bounds):
        ctx = mc.RolloutContext(model, inp.track, inp.cost, noise=inp.noise)
        prob, _keep = mc.build_problem("bss", 64, 10, 16, 1.0, 0.1, inp.cfg.sigma_eps, inp.cfg.precision,
                                       bounds, False, ctx)
        return lib.bssmppi_create(ctypes.byref(prob), 0, ctypes.byref(h))

    for cyf in (2.5, 0.3):
        rc = create(replace(inp.model, c_lat_front=cyf), inp.cfg.bounds)
        assert rc not in (_lib.ERR_UNSUPPORTED, _lib.ERR_INVALID)   # passes validation (then needs a GPU)
    wide = mc.ControlBounds(delta_max=7.0)
    assert create(inp.model, wide) == _lib.ERR_UNSUPPORTED
    assert b"steering bounds" in lib.bssmppi_last_error()
    assert create(replace(inp.model, b_lat_rear=float("inf")), inp.cfg.bounds) == _lib.ERR_INVALID


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from helpers import Inputs
    from paper_2408_00494_b200 import controllers as mc

    inp = Inputs("c1_s0")
    ctrl = mc.Controller(inp.cfg, inp.cost, inp.model, inp.track, noise=inp.noise)
    with pytest.raises(_lib.BssMppiError, match="no CUDA device"):
        ctrl.control_step(inp.x0)
    with pytest.raises(_lib.BssMppiError):
        mc.mppi_update(mc.RolloutBatch(np.zeros((2, 3, 2)), np.zeros((2, 3, 2)), np.ones(2)), 1.0,
                       mc.ControlBounds())


def test_integration_binding_matches_the_abi():
    """INTEGRATION.md's ctypes mirror of bssmppi_problem (what a maintainer
    would paste into the reference package) lists exactly the header's
    fields, in order."""
    import re
    from pathlib import Path
    txt = (Path(__file__).resolve().parent.parent / "INTEGRATION.md").read_text()
    seg = txt[txt.index("class Problem"):txt.index("assert lib.bssmppi_abi_version")]
    assert re.findall(r'\("([a-z_0-9]+)", ', seg) == _struct_fields("bssmppi_problem")
