"""The C example (examples/alltoallv.c) is what a caller that used NCCL writes
against include/nimble.h: it compiles and links here (no GPU), and runs on
one GPU (one rank) and, with two or more GPUs, as one process per GPU."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    lib = os.path.join(ROOT, "paper_2604_00317_b200")
    if not os.path.exists(os.path.join(lib, "libnimble_b200.so")):
        pytest.skip("library not built")
    exe = str(tmp_path / "alltoallv")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
           os.path.join(ROOT, "examples", "alltoallv.c"), "-L", lib, "-lnimble_b200", "-L",
           os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{lib}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles_and_links(tmp_path):
    _build(tmp_path)


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2])
def test_c_example_runs(tmp_path, world):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    exe = _build(tmp_path)
    idfile = str(tmp_path / "id")
    procs = [subprocess.Popen([exe], env=dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                                              NIMBLE_ID_FILE=idfile), stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True) for r in range(world)]
    outs = [p.communicate(timeout=300) for p in procs]
    for p, (out, err) in zip(procs, outs):
        assert p.returncode == 0, (out, err)
        assert " 0 mismatched, async 0" in out, out
    print("".join(o for o, _ in outs), file=sys.stderr)
