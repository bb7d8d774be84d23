"""The C-ABI boundary: the library loads without a GPU, exports every symbol
include/nimble.h declares, and the ctypes binding covers all of them."""
import ctypes
import os
import re
import subprocess

from paper_2604_00317_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "nimble.h")).read()
    return sorted(set(re.findall(r"^\s*(?:nimbleResult_t|const char\*)\s+(nimble\w+)\s*\(", text, re.M)))


def test_header_declares_the_nccl_shaped_surface():
    names = declared()
    for must in ("nimbleGetUniqueId", "nimbleCommInitRank", "nimbleCommInitAll", "nimbleCommDestroy",
                 "nimbleSend", "nimbleRecv", "nimbleGroupStart", "nimbleGroupEnd", "nimbleAlltoAll",
                 "nimbleAlltoAllv", "nimblePlanCreate", "nimblePlanLinkLoads", "nimbleBenchP2P",
                 "nimbleBenchSkewed"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(nimble\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    assert set(declared()) == set(_lib.SIGNATURES), set(declared()) ^ set(_lib.SIGNATURES)


def test_no_torch_or_cuda_types_in_the_abi():
    text = open(os.path.join(ROOT, "include", "nimble.h")).read()
    code = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    assert "cuda" not in code.lower().replace("nimbleunhandledcudaerror", "")
    assert "torch" not in code.lower() and "#include <cuda" not in code


def test_library_has_no_cuda_runtime_dependency(lib):
    out = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcudart" not in out and "libcuda.so" not in out and "libtorch" not in out


def test_error_strings_and_version(lib):
    assert lib.nimbleGetErrorString(0) == b"no error"
    assert lib.nimbleGetErrorString(4) == b"invalid argument"
    v = ctypes.c_int()
    assert lib.nimbleGetVersion(ctypes.byref(v)) == 0 and v.value == 100


def test_comm_calls_fail_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        return
    h = ctypes.c_void_p()
    uid = _lib.UniqueId()
    assert lib.nimbleGetUniqueId(ctypes.byref(uid)) == 0
    rc = lib.nimbleCommInitRank(ctypes.byref(h), 1, uid, 0)
    assert rc != 0 and lib.nimbleGetLastError()


def test_sass_is_sm100a_with_tma_and_release_flags(lib):
    """The engine is compiled for sm_100a and uses TMA bulk copies + mbarriers
    + system-scope release stores (B200_PROFILING.md SASS table)."""
    r = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True)
    if r.returncode != 0:
        return  # cuobjdump absent
    assert "sm_100a" in r.stdout
    for mnemonic in ("UBLKCP.S.G", "SYNCS.ARRIVE.TRANS64", "STG.E.128", "STG.E.64.STRONG.SYS"):
        assert mnemonic in r.stdout, mnemonic
