"""faith-model/v1 and faith-embedding/v1 on the host: files written by the
unmodified reference (tests/golden/formats, oracle/make_format_fixtures.sh) load to exactly the
weights / inputs gen_synthetic produces for the same seeds; save -> load round trips are exact in
both the inline and the blob layout; the reference reads our files back; malformed files fail
with the reference's messages (proj/src/model.cpp:147-369)."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2209_12708_b200 import faith_gpu as F
from paper_2209_12708_b200 import formats as FM

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "formats")
CLI_REF = os.path.join(ROOT, "oracle", "_ref", "faith_cli_ref")

CASES = [  # manifest, embedding, config, model seed, input seed
    ("m1.json", "x1.json", F.ModelConfig(1, 2, 8, 16, 4, 2, "tanh"), 5, 6),
    ("m2.json", "x2.json", F.ModelConfig(2, 4, 16, 24, 6, 3, "silu"), 9, 10),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_reference_files_load_to_gen_synthetic(case):
    m, x, cfg, seed, iseed = case
    got_cfg, params = FM.load_model(os.path.join(GOLD, m))
    assert got_cfg == cfg
    assert np.array_equal(params, F.gen_synthetic(cfg, seed))
    assert np.array_equal(FM.load_embedding(os.path.join(GOLD, x), cfg), F.gen_input(cfg, iseed))


@pytest.mark.parametrize("inline", [True, False], ids=["inline", "blob"])
def test_save_load_round_trip(tmp_path, inline):
    cfg, params = FM.load_model(os.path.join(GOLD, "m2.json"))
    path = str(tmp_path / "model.json")
    FM.save_model(cfg, params, path, inline=inline)
    assert os.path.exists(str(tmp_path / "model.bin")) != inline
    cfg2, p2 = FM.load_model(path)
    assert cfg2 == cfg and np.array_equal(p2, params)
    x = FM.load_embedding(os.path.join(GOLD, "x2.json"), cfg)
    FM.save_embedding(x, cfg, str(tmp_path / "emb.json"), inline=inline)
    assert np.array_equal(FM.load_embedding(str(tmp_path / "emb.json"), cfg), x)


def test_reference_reads_our_blob_files(tmp_path):
    """model::load_model on a blob manifest written here gives the reference's own verdict."""
    if not os.path.exists(CLI_REF):
        pytest.skip("oracle/_ref/faith_cli_ref not built (make -C oracle compat)")
    cfg, params = FM.load_model(os.path.join(GOLD, "m1.json"))
    x = FM.load_embedding(os.path.join(GOLD, "x1.json"), cfg)
    FM.save_model(cfg, params, str(tmp_path / "m.json"))
    FM.save_embedding(x, cfg, str(tmp_path / "x.json"))
    r = subprocess.run([CLI_REF, "verify", "--model", str(tmp_path / "m.json"), "--input", str(tmp_path / "x.json"),
                        "--eps", "0.01", "--norm", "l2"], capture_output=True, text=True, timeout=120)
    with open(os.path.join(GOLD, "m1_verify.txt")) as f:
        assert r.stdout == f.read(), (r.stdout, r.stderr)


def _edit(tmp_path, fn):
    src = os.path.join(GOLD, "m1.json")
    with open(src) as f:
        j = json.load(f)
    fn(j)
    p = str(tmp_path / "bad.json")
    with open(p, "w") as f:
        json.dump(j, f)
    return p


def test_malformed_models_fail_like_the_reference(tmp_path):
    with pytest.raises(FM.FormatError, match="unsupported format"):
        FM.load_model(_edit(tmp_path, lambda j: j.update(format="faith-model/v2")))
    with pytest.raises(FM.FormatError, match=r"layers\[0\].bq: shape \[8\] expects 8 values, got 7"):
        FM.load_model(_edit(tmp_path, lambda j: j["layers"][0]["bq"]["values"].pop()))
    with pytest.raises(FM.FormatError, match=r"layers\[0\].w1 has shape \[16, 8\], expected \[8, 16\]"):
        FM.load_model(_edit(tmp_path, lambda j: j["layers"][0]["w1"].update(shape=[16, 8])))
    with pytest.raises(FM.FormatError, match="embed_dim must be divisible by num_heads"):
        FM.load_model(_edit(tmp_path, lambda j: j.update(num_heads=3)))
    with pytest.raises(FM.FormatError, match="layer weight count mismatch"):
        FM.load_model(_edit(tmp_path, lambda j: j.update(num_layers=2)))
    with pytest.raises(FM.FormatError, match="needs 'values' or 'blob'"):
        FM.load_model(_edit(tmp_path, lambda j: j["classifier"]["b"].pop("values")))
    with pytest.raises(FM.FormatError, match="cannot open"):
        FM.load_model(str(tmp_path / "missing.json"))


def test_truncated_and_missing_blobs(tmp_path):
    cfg, params = FM.load_model(os.path.join(GOLD, "m1.json"))
    path = str(tmp_path / "model.json")
    FM.save_model(cfg, params, path)
    blob = str(tmp_path / "model.bin")
    with open(blob, "rb") as f:
        raw = f.read()
    with open(blob, "wb") as f:
        f.write(raw[:-8])
    with pytest.raises(FM.FormatError, match=r"blob 'model.bin' truncated reading classifier.b"):
        FM.load_model(path)
    os.remove(blob)
    with pytest.raises(FM.FormatError, match=r"cannot open blob 'model.bin' \(referenced by layers\[0\].wq\)"):
        FM.load_model(path)


def test_layer_cap_and_embedding_shape(tmp_path):
    cfg = F.ModelConfig(7, 2, 8, 16, 4, 2, "relu")
    params = np.zeros(FM.param_count(cfg))
    path = str(tmp_path / "deep.json")
    FM.save_model(cfg, params, path, inline=True)
    with pytest.raises(FM.FormatError, match=r"num_layers must be in \[1, 6\]"):
        FM.load_model(path)
    assert FM.load_model(path, strict=False)[0] == cfg  # c5-style 12-layer models
    other = F.ModelConfig(1, 2, 8, 16, 5, 2, "tanh")
    with pytest.raises(FM.FormatError, match=r"shape \[1, 4, 8\], expected \[1, 5, 8\]"):
        FM.load_embedding(os.path.join(GOLD, "x1.json"), other)
