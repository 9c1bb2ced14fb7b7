"""C-ABI library checks that need no GPU: it builds for sm_100a, loads, and exports
every entry point include/ct.h declares (no compute calls)."""
import os
import re
import subprocess

import pytest

from paper_2507_18413_b200 import build as B
from paper_2507_18413_b200 import ct as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ct.h")


@pytest.fixture(scope="module")
def libpath():
    return B.build()


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ct_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_expected_surface():
    fns = header_functions()
    for must in ("ct_create", "ct_propagate", "ct_propagate_many", "ct_state_copy", "ct_last_error"):
        assert must in fns


def test_library_exports_every_header_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = set(re.findall(r"\bT (ct_[a-z0-9_]+)\b", out))
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, f"declared in ct.h but not exported: {missing}"


def test_binding_covers_every_header_symbol():
    assert sorted(C.SIGNATURES) == header_functions()


def test_library_is_sm100a(libpath):
    out = subprocess.check_output(["cuobjdump", "--list-elf", libpath], text=True)
    assert "sm_100a" in out


def test_load_and_call_host_only_entry_points(libpath):
    L = C.lib()
    for name in C.SIGNATURES:
        assert hasattr(L, name)
    assert "sm_100a" in C.ct_version()
    cfg, _ = C.make_config()
    assert cfg.n_shards == 1 and cfg.use_index == 1 and cfg.use_residues == 1 and cfg.use_graph == 1


def test_invalid_arguments_rejected_without_gpu(libpath):
    import numpy as np
    # n_vars = 0 is rejected by validation before any device call
    with pytest.raises(C.CTError) as e:
        C.ct_create(np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 0), np.int32))
    assert e.value.status == C.CT_EINVAL
    # duplicate scope ids (var(c) is a set)
    with pytest.raises(C.CTError) as e:
        C.ct_create([0, 0], [2, 2], np.zeros((1, 2), np.int32), scope=[3, 3])
    assert e.value.status == C.CT_EINVAL


def test_no_gpu_fails_loudly(libpath):
    """On a box without a GPU the product path must error, never fall back."""
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(C.CTError) as e:
        C.ct_create([0], [3], np.array([[1]], np.int32))
    assert e.value.status in (C.CT_ECUDA, C.CT_EINVAL)
