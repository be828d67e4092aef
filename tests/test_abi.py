"""Host-side checks of the boundary (no GPU): the C-ABI library loads, exports every symbol
include/hm.h declares, fails loudly without a device, and the product path never touches
the oracle."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import paper_2305_06891_b200 as hm
    from paper_2305_06891_b200 import build
    build.build()
    return hm.load_library()


def test_library_exports_every_header_symbol(lib):
    import paper_2305_06891_b200 as hm
    syms = hm.header_symbols()
    assert len(syms) >= 19
    for s in ["hm_build_geometry", "hm_assemble_aca", "hm_factor_hlu", "hm_apply_F", "hm_solve_C",
              "hm_radiative_flux"]:
        assert s in syms
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_status_strings(lib):
    import ctypes
    lib.hm_status_string.restype = ctypes.c_char_p
    assert lib.hm_status_string(0) == b"ok"
    assert lib.hm_status_string(6) == b"singular leaf block"


def test_no_cpu_fallback_without_device(lib):
    import torch
    import paper_2305_06891_b200 as hm
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(hm.HMError) as e:
        hm.hm_init(0)
    assert e.value.status == "HM_ERR_CUDA"


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2305_06891_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f
                assert "import_module(\"oracle" not in txt, f


def test_oracle_never_imports_product():
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(from|import)\s+paper_2305_06891_b200", txt, re.M), f


def test_header_documents_every_entry_point():
    txt = open(os.path.join(ROOT, "include", "hm.h")).read()
    for s in ["hm_apply_F", "hm_solve_C", "hm_radiative_flux", "hm_factor_hlu", "hm_assemble_aca"]:
        i = txt.index(s + "(")
        assert "PAPER.md:" in txt[max(0, i - 900):i], s


def test_binding_rejects_unsafe_output_arrays():
    """Outputs must be C-contiguous float64: a silently converted copy would drop the results."""
    import paper_2305_06891_b200 as hm
    with pytest.raises(TypeError):
        hm._ptr(np.empty(4, dtype=np.float32), out=True)
    with pytest.raises(TypeError):
        hm._ptr(np.empty((4, 2))[:, 0], out=True)
    p, keep = hm._ptr(np.arange(4), out=False)          # inputs are converted
    assert keep.dtype == np.float64 and p == keep.ctypes.data
