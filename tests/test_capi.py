"""The C-ABI library loads (no GPU needed for dlopen) and exports every entry
point include/mprec_gpu.h declares; the oracle exports the same surface."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mprec_gpu.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mprec_gpu_\w+)\s*\(", src)))


def test_header_declares_the_path():
    names = declared()
    for must in ("mprec_gpu_create", "mprec_gpu_setup", "mprec_gpu_apply", "mprec_gpu_solve",
                 "mprec_gpu_solve_system", "mprec_gpu_amg_create", "mprec_gpu_ilu_create", "mprec_gpu_gmres"):
        assert must in names


def test_gpu_library_exports_every_symbol():
    from paper_1912_04385_b200.api import GPU_LIB
    assert os.path.exists(GPU_LIB), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(GPU_LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_oracle_mirrors_the_surface():
    import oracle
    lib = ctypes.CDLL(oracle.LIB)
    core = ["create", "setup", "apply", "apply_stage", "spmv", "solve", "get_scaled", "get_ilu", "n_stages",
            "stage_amg", "destroy", "amg_create", "amg_apply", "amg_n_levels", "amg_level_info", "amg_get_csr",
            "amg_get_cf", "amg_destroy", "ilu_create", "ilu_apply", "ilu_get", "ilu_destroy", "gmres"]
    missing = [n for n in core if not hasattr(lib, "orc_" + n)]
    assert not missing, missing


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    """The product path fails loudly when the CUDA library is absent."""
    import paper_1912_04385_b200.api as api
    monkeypatch.setattr(api, "GPU_LIB", str(tmp_path / "missing.so"))
    monkeypatch.setattr(api, "_gpu_api", None)
    with pytest.raises(ImportError):
        api.gpu()


def test_gpu_calls_fail_without_device():
    """Without a GPU every compute entry point reports MPREC_CUDA (no silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1912_04385_b200.api import gpu, CudaError
    from tests.systems import random_block_system
    a = random_block_system(4, 1, 0)
    with pytest.raises(CudaError):
        gpu().system(a)
