"""Drop-in proof on the GPU: the reference's UNMODIFIED callers -- graph::evaluate, cli::cmd_verify,
cli::cmd_maxeps, the machine executors and proj/tests/acceptance.cpp -- linked against the C++
drop-in layer (paper_2209_12708_b200/compat/faith_compat.cpp -> libfaith_compat.so) instead of
proj/src/bounds.cpp + relax.cpp, so every bound operator runs on the B200 (oracle/Makefile
target `compat`).  The reference's own acceptance criteria must all pass, and certify / max-eps
must give the same answers as the CPU reference build in the reference's whole-embedding mode
(input_bounds over all L*E inputs, bounds.cpp:101-120)."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
ACC = os.path.join(REF, "acceptance_gpu")
CLI_GPU = os.path.join(REF, "faith_cli_gpu")
CLI_REF = os.path.join(REF, "faith_cli_ref")


def _need(*paths):
    for p in paths:
        if not os.path.exists(p):
            pytest.fail(f"{p} missing: build with `python -c 'import __graft_entry__ as g; g.build()'`")


def _run(cmd, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run(cmd, capture_output=True, text=True, env=e, timeout=timeout)


def test_reference_acceptance_suite_on_gpu_dropin():
    """proj/tests/acceptance.cpp, unmodified, every bound operator on the GPU (f64 exact mode):
    soundness (3M sampled passes), exactness at eps=0, the BITWISE affine oracle, envelope grid
    soundness, fused/unfused semantics, analytic max-eps, ... -- all ten criteria must PASS."""
    _need(ACC)
    r = _run([ACC], timeout=1800)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith(("PASS", "FAIL"))]
    print("\n".join(lines))
    assert len(lines) == 10, r.stdout + r.stderr
    assert all(ln.startswith("PASS") for ln in lines), "\n".join(lines)
    assert r.returncode == 0


def _gen(tmp, name, layers, heads, embed, ffn, length, act, seed):
    m, x = os.path.join(tmp, f"{name}.json"), os.path.join(tmp, f"{name}_x.json")
    r = _run([CLI_REF, "gen", "--layers", str(layers), "--heads", str(heads), "--embed", str(embed), "--ffn",
              str(ffn), "--length", str(length), "--act", act, "--seed", str(seed), "--model", m,
              "--input-seed", str(seed + 1), "--input", x])
    assert r.returncode == 0, r.stderr
    return m, x


CASES = [  # (name, layers, heads, embed, ffn, length, act, norm, eps)
    ("tiny_relu", 1, 2, 8, 16, 4, "relu", "linf", 0.02),
    ("tanh_l2", 2, 2, 16, 32, 6, "tanh", "l2", 0.05),
    ("silu_l1", 1, 4, 16, 24, 8, "silu", "l1", 0.2),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_cmd_verify_and_maxeps_match_cpu_reference(tmp_path, case):
    """cli::cmd_verify and cli::cmd_maxeps (cli.cpp:64-193) through the drop-in give the
    reference's verdicts, predicted class and -- in f64 exact mode -- the identical bisection
    path (same max epsilon, same number of verification calls)."""
    _need(CLI_GPU, CLI_REF)
    name, layers, heads, embed, ffn, length, act, norm, eps = case
    m, x = _gen(str(tmp_path), name, layers, heads, embed, ffn, length, act, 4242)
    for e in (0.0, eps, 10 * eps):
        a = _run([CLI_REF, "verify", "--model", m, "--input", x, "--eps", str(e), "--norm", norm])
        b = _run([CLI_GPU, "verify", "--model", m, "--input", x, "--eps", str(e), "--norm", norm])
        assert (a.returncode, a.stdout) == (b.returncode, b.stdout), (a.stdout, b.stdout, b.stderr)
    a = _run([CLI_REF, "maxeps", "--model", m, "--input", x, "--norm", norm, "--tol", "1e-4", "--eps-max", "1.0"])
    b = _run([CLI_GPU, "maxeps", "--model", m, "--input", x, "--norm", norm, "--tol", "1e-4", "--eps-max", "1.0"])
    assert a.returncode == b.returncode == 0, (a.stderr, b.stderr)
    assert a.stdout == b.stdout, (a.stdout, b.stdout)


def test_cmd_maxeps_f32_mode_within_tolerance(tmp_path):
    """The same reference callers on the f32-Λ arithmetic (FAITH_GPU_PRECISION=f32): the
    certified epsilon agrees within 1e-3 relative (+ tol) with the f64 CPU reference."""
    _need(CLI_GPU, CLI_REF)
    m, x = _gen(str(tmp_path), "f32", 1, 2, 16, 32, 8, "relu", 77)
    args = ["maxeps", "--model", m, "--input", x, "--norm", "l2", "--tol", "1e-5", "--eps-max", "1.0"]
    a = _run([CLI_REF] + args)
    b = _run([CLI_GPU] + args, env={"FAITH_GPU_PRECISION": "f32"})
    assert a.returncode == b.returncode == 0, (a.stderr, b.stderr)
    ea = float(re.search(r"= ([0-9.e+-]+)", a.stdout).group(1))
    eb = float(re.search(r"= ([0-9.e+-]+)", b.stdout).group(1))
    assert abs(ea - eb) <= 1e-3 * ea + 1e-5, (ea, eb)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_fused_pass_on_reference_models(tmp_path, case):
    """The pass-level fast path (faith::gpu::FusedVerifier: whole fused bound passes, f32 Λ) on the
    reference's own model/embedding files and whole-embedding ε-ball: same verdicts as the CPU
    reference's cmd_verify and max ε within 1e-3 relative (+ tol) of its cmd_maxeps."""
    _need(CLI_GPU, CLI_REF)
    name, layers, heads, embed, ffn, length, act, norm, eps = case
    m, x = _gen(str(tmp_path), name, layers, heads, embed, ffn, length, act, 4242)
    for e in (0.0, eps, 10 * eps):
        a = _run([CLI_REF, "verify", "--model", m, "--input", x, "--eps", str(e), "--norm", norm])
        b = _run([CLI_GPU, "verify-fused", "--model", m, "--input", x, "--eps", str(e), "--norm", norm])
        assert a.returncode == b.returncode and a.stdout.split()[0] == b.stdout.split()[0], (a.stdout, b.stdout,
                                                                                              b.stderr)
    args = ["--model", m, "--input", x, "--norm", norm, "--tol", "1e-5", "--eps-max", "1.0"]
    a = _run([CLI_REF, "maxeps"] + args)
    b = _run([CLI_GPU, "maxeps-fused"] + args)
    assert a.returncode == b.returncode == 0, (a.stderr, b.stderr)
    ea = float(re.search(r"= ([0-9.e+-]+)", a.stdout).group(1))
    eb = float(re.search(r"= ([0-9.e+-]+)", b.stdout).group(1))
    assert abs(ea - eb) <= 1e-3 * ea + 1e-5, (a.stdout, b.stdout)


def test_reference_model_file_to_device_verdict():
    """A faith-model/v1 file written by the reference (tests/golden/formats) loaded by
    Model.from_file: the whole-embedding certify (all L tokens perturbed, D = L*E, the reference's
    input_bounds mode) gives the reference cmd_verify verdict recorded next to it."""
    import numpy as np
    from paper_2209_12708_b200 import faith_gpu as F
    from paper_2209_12708_b200 import formats as FM
    gold = os.path.join(ROOT, "tests", "golden", "formats")
    m = F.Model.from_file(F.Context(0), os.path.join(gold, "m1.json"))
    x = FM.load_embedding(os.path.join(gold, "x1.json"), m.cfg)
    r = m.certify(x, np.arange(m.cfg.length), "l2", 0.01)
    with open(os.path.join(gold, "m1_verify.txt")) as f:
        want = f.read().split()
    assert want[0] == "verified" and bool(r["verified"][0])
    assert want[-1] == f"class={int(r['predicted'][0])}"
