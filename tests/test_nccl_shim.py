"""The multi-rank tests' NCCL stand-in (tests/nccl_shim.c) builds here and
exports every symbol the library resolves from libnccl.so.2 (csrc/session.cu
nccl_load), so the GPU multi-rank tests exercise the same call sites."""
import os
import re
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.mark.skipif(shutil.which("gcc") is None or not os.path.isdir(f"{CUDA}/include"),
                    reason="gcc or CUDA headers missing")
def test_shim_builds_and_exports_what_the_library_resolves(tmp_path):
    so = tmp_path / "libnccl_shim.so"
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-shared", "-fPIC", f"-I{CUDA}/include",
                    os.path.join(REPO, "tests", "nccl_shim.c"), "-o", str(so),
                    f"-L{CUDA}/lib64/stubs", "-lcuda"], check=True)
    exported = set(re.findall(r" T (\w+)", subprocess.run(["nm", "-D", str(so)], check=True,
                                                         capture_output=True, text=True).stdout))
    src = open(os.path.join(REPO, "paper_2602_09527_b200", "csrc", "session.cu")).read()
    resolved = set(re.findall(r'dlsym\(api->so, "(nccl\w+)"\)', src))
    assert len(resolved) == 10
    assert resolved <= exported
