"""CPU-only checks: the C-ABI library loads and exports every declared
symbol, and the host-side logic (config, flat layout, schedule, collectives
over gloo, errors) mirrors the reference.  No compute calls without a GPU."""

import os
import re
import subprocess

import numpy as np
import pytest
import torch

from conftest import ROOT, golden
from oracle import gfm_oracle as O
from paper_2406_12909_b200 import _lib
from paper_2406_12909_b200 import model as M
from paper_2406_12909_b200.errors import ConfigError, ValidationError
from paper_2406_12909_b200.schedule import epoch_schedule
from paper_2406_12909_b200.train import EarlyStopper, TrainConfig

HEADER = os.path.join(ROOT, "include", "gfm_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"GFM_API\s+[\w\s\*]+?\b(gfm_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    decl = declared_symbols()
    assert len(decl) >= 30
    for name in decl:
        assert hasattr(lib, name), name
    assert lib.gfm_abi_version() == _lib.ABI_VERSION
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                        text=True).stdout
    exported = set(re.findall(r" T (gfm_\w+)", nm))
    assert set(decl) == exported


def test_python_signatures_cover_header():
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_device_raises_loudly():
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.ExtensionMissingError):
        M.init_params(M.ModelConfig())


@pytest.mark.parametrize("kind", M.MPNN_KINDS)
def test_flat_layout_matches_oracle(kind):
    cfg = M.ModelConfig(mpnn_kind=kind, mpnn_layers=2, mpnn_width=5, fc_layers=3, fc_width=4)
    cfg_o = O.config(kind, 2, 5, 3, 4)
    assert M.count_params(cfg) == O.n_params(cfg_o)
    assert [s for _, s in M.param_shapes(cfg)] == [s for _, s in O.param_shapes(cfg_o)]
    np.testing.assert_array_equal(M.init_params_flat(cfg, 3), O.init_flat(cfg_o, 3))


def test_count_params_reference_examples():
    # pkg/tests/test_model.py:44-47
    assert M.count_params(M.ModelConfig(mpnn_layers=3, mpnn_width=50, fc_layers=2, fc_width=50)) == 26_251
    assert M.count_params(M.ModelConfig(mpnn_layers=1, mpnn_width=1, fc_layers=2, fc_width=1)) == 128
    # C1/C2 = 40,769; C3 = 3,735,553; C3 pna = 8,454,145
    assert M.count_params(M.ModelConfig(mpnn_layers=3, mpnn_width=64, fc_width=64)) == 40_769
    assert M.count_params(M.ModelConfig(mpnn_layers=6, mpnn_width=512, fc_width=512)) == 3_735_553
    assert M.count_params(M.ModelConfig(mpnn_kind="pna-agg", mpnn_layers=6, mpnn_width=512,
                                        fc_width=512)) == 8_454_145


def test_init_matches_reference_golden():
    g = golden("c1_model.npz")
    cfg = M.ModelConfig(mpnn_layers=3, mpnn_width=64, fc_width=64)
    np.testing.assert_array_equal(M.init_params_flat(cfg, 0), g["mean-agg_flat"])


def test_config_validation():
    with pytest.raises(ValidationError):
        M.ModelConfig(mpnn_kind="gru")
    with pytest.raises(ValidationError):
        M.ModelConfig(fc_layers=1)
    with pytest.raises(ValidationError):
        M.ModelConfig(alpha_energy=0.0)
    with pytest.raises(ConfigError, match="optimizer"):
        TrainConfig(optimizer="lbfgs")
    with pytest.raises(ConfigError, match="patience"):
        TrainConfig(patience=0)


def test_schedule_matches_reference_golden():
    g = golden("misc.npz")
    s = epoch_schedule(103, 4, 8, 7, 3)
    np.testing.assert_array_equal(np.concatenate([np.concatenate(b) for b in s.per_rank]),
                                  g["sched"])


def test_early_stopper_eleven():
    st = EarlyStopper(patience=10)
    epochs = 0
    for v in [0.1 * (k + 1) for k in range(100)]:
        epochs += 1
        if st.update(v):
            break
    assert epochs == 11


def test_bench_reference_arm_json_contract():
    """`bench.py --impl reference` (the CPU oracle port on host cores) prints
    one JSON line with the contract's keys."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--config", "c2", "--steps", "1", "--warmup", "0", "--cpu-sample-s",
                          "1", "--ref-ranks", "1"],
                         capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "graphs/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    for k in ("metric", "n_gpus", "steps", "warmup", "scaling", "dtype", "data", "config"):
        assert k in line
    dp = line["reference_dp"]  # the reference's own DP path, when baseline/_ref holds it
    if "unavailable" not in dp:
        assert dp["kind"] == "reference" and dp["value"] > 0
        assert dp["points"][0]["ranks"] == 1 and "cpu_model" in dp
