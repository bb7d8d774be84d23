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


def test_ctypes_structs_match_the_header_layout(tmp_path):
    """Every ctypes struct has the C header's size and field offsets (a C
    program compiled against include/nimble.h prints them)."""
    pairs = [(_lib.PlannerConfig, "nimblePlannerConfig"), (_lib.PlanStats, "nimblePlanStats"),
             (_lib.CommConfig, "nimbleCommConfig"), (_lib.UniqueId, "nimbleUniqueId"),
             (_lib.Item, "nimbleItem"), (_lib.BenchResult, "nimbleBenchResult"),
             (_lib.CommStats, "nimbleCommStats")]
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "nimble.h"', "int main(void) {"]
    for cls, cname in pairs:
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f in cls._fields_:
            lines.append(f'printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0].rstrip("_")}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.splitlines())
    for cls, cname in pairs:
        assert int(got[f"{cname} size"]) == ctypes.sizeof(cls), cname
        for f in cls._fields_:
            assert int(got[f"{cname} {f[0]}"]) == getattr(cls, f[0]).offset, (cname, f[0])


def test_comm_config_defaults_through_the_abi(lib):
    cfg = _lib.CommConfig()
    assert lib.nimbleCommConfigDefault(ctypes.byref(cfg)) == 0
    assert (cfg.fabric, cfg.pipe_chunk, cfg.p2p_buffer, cfg.channels_per_peer) == (1, 64 << 10, 10 << 20, 1)
    assert (cfg.ctas, cfg.direct_chunk, cfg.pull, cfg.push_chunk, cfg.ll_max) == (0, 0, 0, 0, 1 << 20)
    assert cfg.nvlink_bytes_per_s == 900e9


def test_python_fast_call_binds_the_same_entry_point(lib):
    """comm.py's CPython fast call (csrc/pyfast.cpp) reaches nimbleAlltoAllv of the
    library _lib loaded and reports its result codes; bad arguments raise."""
    import pytest
    from paper_2604_00317_b200 import comm as C
    assert C._FAST is not None, "the _fast module was not built"
    rc = C._FAST.alltoallv(0, 0, [1, 2], [0, 1], 0, [1, 2], [0, 1], 1, 0)  # null comm
    assert rc == 4 and b"null argument" in lib.nimbleGetLastError()
    with pytest.raises(ValueError):
        C._FAST.alltoallv(0, 0, [1, 2], [0], 0, [1, 2], [0, 1], 1, 0)
    with pytest.raises(TypeError):
        C._FAST.alltoallv(0, 0, [1, 2], [0, 1], 0, [1, 2], [0, 1], 1)
