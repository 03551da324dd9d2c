"""The C-ABI library: loads, exports every symbol include/lfmm.h declares,
and the product path fails loudly (no CPU fallback) without a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "lfmm.h")).read()
    return sorted(set(re.findall(r"\b(lfmm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2410_01754_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_native.exported_symbols()) == syms


def test_version_and_stage_names():
    from paper_2410_01754_b200 import _native

    lib = _native.lib()
    assert lib.lfmm_version().decode().startswith("lfmm-b200")
    n = lib.lfmm_stage_count()
    names = [lib.lfmm_stage_name(i).decode() for i in range(n)]
    for stage in ("tree", "p2p", "p2m", "m2m", "m2l", "l2l", "l2p", "hi"):
        assert stage in names


def test_library_is_sm100a():
    import subprocess

    from paper_2410_01754_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") != "" and os.path.exists("/dev/nvidia0"),
                    reason="a GPU is present")
def test_no_cpu_fallback_without_gpu():
    from paper_2410_01754_b200 import PeriodicSolver, SolverConfig

    with pytest.raises(RuntimeError):
        PeriodicSolver(np.zeros((2, 3)) + [[0.1, 0.2, 0.3], [0.5, 0.5, 0.5]], 1.0, SolverConfig(p=4, depth=1))


def test_invalid_arguments_map_to_value_error_before_device():
    from paper_2410_01754_b200 import SolverConfig

    with pytest.raises(ValueError, match=r"expansion order p=0 outside \[1, 40\]"):
        SolverConfig(p=0).validated()
