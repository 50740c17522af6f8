"""CPU checks of the C-ABI boundary: the library builds for sm_100a, loads, exports every
symbol include/faith_gpu.h declares, and refuses to run without an sm_100 GPU (no CPU
fallback).  No device compute is attempted here."""
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

from paper_2209_12708_b200 import faith_gpu as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    lib = F.load_library()
    syms = F.exported_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump absent")
    out = subprocess.run(["cuobjdump", "--list-elf", F.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_header_constants_match_oracle():
    text = open(F.HEADER).read()
    oh = open(os.path.join(ROOT, "oracle", "faith_oracle.h")).read()
    for name in ("NORM_L1", "NORM_L2", "NORM_LINF", "RELAX_RELU", "RELAX_TANH", "RELAX_SILU", "RELAX_EXP",
                 "RELAX_RECIP", "DOT_SIMILARITY", "DOT_WEIGHTED_VALUES", "EINVAL", "EDOMAIN", "ERANGE"):
        a = re.search(rf"#define FG_{name} (\d+)", text)
        b = re.search(rf"#define FO_{name} (\d+)", oh)
        assert a and b and a.group(1) == b.group(1), name


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(F.CudaError):
        F.Context(0)


def test_check_robust_is_host_side_and_strict():
    # bounds.cpp:142-157 semantics through the C ABI (no device work involved)
    assert F.Context.check_robust([0.4, 0.1], [0.6, 0.39], 0)
    assert not F.Context.check_robust([0.4, 0.1], [0.6, 0.4], 0)
    assert F.Context.check_robust([1.0, 0.0], [1.5, 0.5], 0, 0.4)
    with pytest.raises(F.OutOfRange):
        F.Context.check_robust([0.4, 0.1], [0.6, 0.39], 2)
    with pytest.raises(F.InvalidArgument):
        F.Context.check_robust([0.4, 0.1], [0.6, 0.39], 0, -1.0)


def test_default_kappa_matches_header():
    import re
    text = open(F.HEADER).read()
    m = re.search(r"#define FG_DEFAULT_KAPPA\s+([0-9.eE+-]+)", text)
    assert m and float(m.group(1)) == F.DEFAULT_KAPPA
