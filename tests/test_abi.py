"""CPU-side checks of the C-ABI boundary: libpsc.so loads, exports every symbol
include/psc.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "psc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(psc_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for must in ("psc_init", "psc_desc_create", "psc_desc_assemble", "psc_mat_create_csr", "psc_mat_assemble",
                 "psc_hier_create", "psc_pcg_solve", "psc_pcg_solve_host", "psc_hier_vcycle", "psc_mat_spmv"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    import paper_2406_19754_b200 as psc
    lib = ctypes.CDLL(psc.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_names_match_header():
    import paper_2406_19754_b200 as psc
    for s in declared_symbols():
        assert getattr(psc._lib, s).restype is not None or s in ("psc_finalize", "psc_desc_destroy",
                                                                  "psc_mat_destroy", "psc_hier_destroy",
                                                                  "psc_amg_destroy")


def test_status_strings_and_version():
    import paper_2406_19754_b200 as psc
    assert psc._lib.psc_status_string(psc.PSC_ERR_BREAKDOWN) == b"PSC_ERR_BREAKDOWN"
    assert psc._lib.psc_status_string(psc.PSC_NOT_CONVERGED) == b"PSC_NOT_CONVERGED"
    assert b"sm_100a" in psc._lib.psc_version()


def test_built_for_sm100a_only():
    import subprocess
    import paper_2406_19754_b200 as psc
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", psc.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)\b", out)


def test_no_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2406_19754_b200 as psc
    with pytest.raises(psc.PscError) as e:
        psc.Context()
    assert e.value.code == psc.PSC_ERR_CUDA


def test_product_does_not_reference_oracle():
    """The product path never imports or links the oracle (shares no code)."""
    pkg = os.path.join(ROOT, "paper_2406_19754_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.lower().replace("oracle/", ""), f
