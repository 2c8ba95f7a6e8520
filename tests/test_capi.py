"""The C-ABI boundary without a GPU: the in-tree library loads, exports every
function include/proxtomo_b200.h declares, and the Python binding covers
exactly that surface.  No compute calls (those are the -m gpu tests)."""

import ctypes
import os
import re

import pytest

from conftest import REPO
from paper_2602_09527_b200 import _native as N

HEADER = os.path.join(REPO, "include", "proxtomo_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pt_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("pt_plan_create", "pt_forward", "pt_adjoint", "pt_adjoint_step", "pt_tv_prox",
                 "pt_session_run", "pt_session_attach_nccl", "pt_operator_norm_sq"):
        assert must in names


def test_library_loads_and_exports_every_declared_symbol():
    lib = N.load()
    assert os.path.abspath(N.library_path()).startswith(REPO)  # in-tree, not site-packages
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.pt_version().startswith(b"proxtomo_b200")


def test_binding_covers_the_header():
    assert set(N.EXPORTED_SYMBOLS) == set(declared_functions())


def test_sm100a_cubin_embedded():
    data = open(N.library_path(), "rb").read()
    assert b"sm_100a" in data


def test_product_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2602_09527_b200 import ParallelGeometry, forward_project
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        forward_project([[0.0]], ParallelGeometry.uniform(1, 1))


def test_product_never_imports_the_oracle():
    pkg = os.path.join(REPO, "paper_2602_09527_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(root, f), encoding="utf-8").read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_geometry_desc_layout_matches_the_library():
    lib = N.load()
    assert lib.pt_geometry_desc_size() == ctypes.sizeof(N.GeometryDesc)


def test_reference_binding_loads_standalone():
    """The Option B binding dlopens the library from its own
    struct definition and checks the layout; no device needed to load."""
    from paper_2602_09527_b200 import reference_binding as RB
    lib = RB.load_library()
    assert lib.pt_geometry_desc_size() == ctypes.sizeof(RB._GeometryDesc)
    src = open(RB.__file__, encoding="utf-8").read()
    # standalone: a maintainer copies this one file next to proxtomo/projector.py
    assert "from . import" not in src and "from .." not in src


def test_every_pdl_launched_kernel_waits_before_it_releases():
    """The launch chain's rule (csrc/pt_internal.cuh): a kernel launched with
    programmatic stream serialisation must call pdl_wait() (else it would run
    beside its predecessor), and releases its successor only after that wait --
    either inside pdl_wait() (early families) or by a later pdl_trigger()."""
    csrc = os.path.join(REPO, "paper_2602_09527_b200", "csrc")
    bodies, launched = {}, set()
    for f in os.listdir(csrc):
        if not f.endswith(".cu"):
            continue
        src = open(os.path.join(csrc, f), encoding="utf-8").read()
        parts = re.split(r"(?=__global__)", src)
        for part in parts[1:]:
            m = re.search(r"(\w+_kernel)\s*\(", part)
            if m:
                bodies[m.group(1)] = part
        for m in re.finditer(r"launch_pdl\(([^;]*?);", src, flags=re.S):
            launched.update(re.findall(r"\b(\w+_kernel)\b", m.group(1)))
    assert launched, "no PDL launches found"
    for name in sorted(launched):
        body = bodies.get(name)
        assert body is not None, name
        wait = re.search(r"pdl_wait(<\w+>)?\(\)", body)
        assert wait, f"{name} is launched with PDL but never waits"
        first_trigger = re.search(r"pdl_trigger(<\w+>)?\(\)", body)
        assert first_trigger and first_trigger.start() > wait.start(), name
    hdr = open(os.path.join(csrc, "pt_internal.cuh"), encoding="utf-8").read()
    w = hdr.index("void pdl_wait()")
    assert hdr.index("griddepcontrol.wait", w) < hdr.index("griddepcontrol.launch_dependents", w)
