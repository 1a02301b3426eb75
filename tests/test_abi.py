"""C-ABI checks that run without a GPU: the library loads, exports exactly what
include/crackfield_b200.h declares, and fails loudly (no CPU fallback) when no device exists."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "crackfield_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cf_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1806_09924_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _lib


def test_header_symbols_exported(lib):
    decl = declared_functions()
    assert len(decl) >= 15
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib.LIB_PATH], text=True)
    exported = set(re.findall(r"\bT (cf_[a-z0-9_]+)", out))
    missing = [f for f in decl if f not in exported]
    assert not missing, missing
    bound = {name for name, _, _ in lib.SIGNATURES}
    assert set(decl) == bound, set(decl) ^ bound


def test_library_loads_and_binds(lib):
    L = lib.load()
    assert L.cf_version() == 1


def test_invalid_arguments_rejected_before_device(lib):
    import paper_1806_09924_b200 as cf
    with pytest.raises(ValueError, match="dimension"):
        cf.Problem(4, 1.0, 2, 0)
    with pytest.raises(ValueError, match="initial_cells_per_side"):
        cf.Problem(2, 1.0, 17, 0)


def test_no_cpu_fallback_without_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import paper_1806_09924_b200 as cf
    with pytest.raises(RuntimeError, match="no CUDA device"):
        cf.Problem(2, 1.0, 2, 0)


def test_production_spmv_kernels_use_tma_bulk_copies(lib):
    """The sm_100a object of spmv.cu (the production M_uu SpMV k_spmv_st16t and the prolongator
    SpMV k_spmv_bt) must contain the bulk-copy and mbarrier instructions their design rests on:
    UBLKCP.S.G (cp.async.bulk global -> shared) and SYNCS.ARRIVE.TRANS64 / SYNCS.PHASECHK (mbarrier
    expect-tx arrive and try_wait), the SASS mnemonics /opt/skills/guides/B200_PROFILING.md names."""
    import shutil
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not on PATH")
    obj = os.path.join(ROOT, "paper_1806_09924_b200", "csrc", "spmv.o")
    target = obj if os.path.exists(obj) else lib.LIB_PATH
    sass = subprocess.check_output(["cuobjdump", "-sass", target], text=True)
    funcs = re.split(r"\n\s*Function : ", sass)
    by_kernel = {}
    for f in funcs[1:]:
        name = f.split("\n", 1)[0]
        for k in ("k_spmv_st16t", "k_spmv_bt"):
            if k in name:
                by_kernel.setdefault(k, "")
                by_kernel[k] += f
    assert set(by_kernel) == {"k_spmv_st16t", "k_spmv_bt"}, sorted(by_kernel)
    for k, body in by_kernel.items():
        assert "UBLKCP.S.G" in body, k
        assert "SYNCS.ARRIVE.TRANS64" in body and "SYNCS.PHASECHK.TRANS64.TRYWAIT" in body, k
