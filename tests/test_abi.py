"""CPU checks of the C-ABI boundary: librdd.so builds, loads, exports every symbol that
include/rdd.h declares, agrees on struct layouts, and fails loudly without a CUDA device."""
import ctypes as C
import os
import subprocess

import pytest

from paper_2412_19207_b200 import abi as A
from paper_2412_19207_b200 import rdd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2412_19207_b200", "csrc"), "-j", "8", "-s"], check=True)
    return rdd.LIB_PATH


def test_exports_every_declared_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True, check=True).stdout
    have = {line.split()[-1] for line in out.splitlines() if " T " in line}
    declared = rdd.exported_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if s not in have]
    assert not missing, missing


def test_struct_layouts_match(built):
    L = rdd.lib()
    cs, ss = C.c_int32(), C.c_int32()
    L.rdd_abi_sizes(C.byref(cs), C.byref(ss))
    assert cs.value == C.sizeof(A.Config)
    assert ss.value == C.sizeof(A.Summary)


def test_sm100a_code_only(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_dmma_in_gemm_sass(built):
    out = subprocess.run(["cuobjdump", "-sass", built], capture_output=True, text=True).stdout
    gemm = [blk for blk in out.split("Function :") if "k_gemm" in blk.split("\n")[0]]
    # NN / NT / TN at 64x64 tiles and the 64x128-tile NN variant
    assert len(gemm) >= 3 and all("DMMA" in blk for blk in gemm)


def test_fails_loudly_without_device(built):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("device present")
    with pytest.raises(rdd.DeviceError):
        rdd.Solver(0)
