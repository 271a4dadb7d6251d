"""CPU-side checks of the C-ABI boundary: the library loads and exports every
symbol include/nmfb.h declares (no compute calls: there is no GPU here)."""

import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "nmfb.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nmfb_\w+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    names = header_functions()
    for must in ("nmfb_estep_dense", "nmfb_estep_sparse", "nmfb_mstep_rows", "nmfb_nnls_batch",
                 "nmfb_gram", "nmfb_rescale", "nmfb_gemm_tall", "nmfb_csc_linear",
                 "nmfb_csr_yt", "nmfb_dense_residual", "nmfb_dot", "nmfb_nqp_solve"):
        assert must in names


def test_library_exports_every_header_symbol():
    from paper_1506_08938_b200 import _lib

    lib = _lib.lib()  # loads libnmfb.so (no device needed to dlopen)
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (nmfb_\w+)", out))
    assert set(header_functions()) <= exported


def test_python_binding_covers_header():
    from paper_1506_08938_b200 import _lib

    assert set(_lib.exported_symbols()) == set(header_functions())


def test_library_is_sm100a():
    from paper_1506_08938_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch

    from paper_1506_08938_b200 import device

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError):
        device.require_cuda()


def test_product_does_not_import_oracle():
    pkg = os.path.join(REPO, "paper_1506_08938_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M)


def test_config_rank_limits():
    """The fp32 NNLS kernel stages Q (r x r fp32) in shared memory: r <= 224;
    the fp64 check mode goes to 256."""
    from paper_1506_08938_b200 import NmfConfig

    NmfConfig(rank=224, precision="fp32")
    NmfConfig(rank=256, precision="fp64")
    with pytest.raises(ValueError, match="224"):
        NmfConfig(rank=225, precision="fp32")
    with pytest.raises(ValueError):
        NmfConfig(rank=257, precision="fp64")
