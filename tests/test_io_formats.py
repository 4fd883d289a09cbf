"""On-disk formats (CSV + strict JSON) against the reference's own files
(tests/golden/cli_logit, written by the reference's cmd_simulate / cmd_fit /
cmd_predict).  CPU only: no device work."""

import json
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli_logit")


def _io():
    import importlib
    return importlib.import_module("paper_2310_12000_b200.io")


def test_read_reference_csv_and_columns():
    io = _io()
    h, a = io.read_csv(os.path.join(HERE, "train.csv"))
    assert h[:2] == ["s1", "s2"] and "y" in h
    assert io.columns(h, a, "s").shape == (260, 2)
    assert io.columns(h, a, "x").shape == (260, 1)
    assert io.columns(h, a, "z") is None


def test_csv_roundtrip_is_lossless(tmp_path):
    io = _io()
    rng = np.random.default_rng(0)
    a = rng.standard_normal((50, 3)) * 10.0 ** rng.integers(-12, 12, size=(50, 3))
    p = tmp_path / "x.csv"
    io.write_csv(p, ["s1", "s2", "y"], a.tolist(), comments=["hello"])
    h, b = io.read_csv(p)
    assert h == ["s1", "s2", "y"]
    assert np.array_equal(a, b)


def test_csv_errors(tmp_path):
    io = _io()
    from paper_2310_12000_b200.errors import DataError
    p = tmp_path / "bad.csv"
    p.write_text("s1,y\n1,2\n3\n")
    with pytest.raises(DataError):
        io.read_csv(p)
    p.write_text("s1,y\n1,nan\n")
    with pytest.raises(DataError):
        io.read_csv(p)
    with pytest.raises(DataError):
        io.read_csv(tmp_path / "missing.csv")


def test_strict_config_keys():
    io = _io()
    from paper_2310_12000_b200.errors import ConfigError
    cfg = json.load(open(os.path.join(HERE, "fit.json")))
    fc = io.fit_config_from(cfg)
    assert fc.m == 10 and fc.ordering_seed == 5 and fc.backend.probe_seed == 6 and fc.max_iters == 4
    bad = dict(cfg, optimizer={"max_iters": 3, "bogus": 1})
    with pytest.raises(ConfigError):
        io.fit_config_from(bad)
    with pytest.raises(ConfigError):
        io.likelihood_from({"family": "bernoulli-logit", "extra": 1})


def test_reference_model_loads():
    io = _io()
    model = io.load_model(os.path.join(HERE, "model.json"))
    assert model["format"] == io.MODEL_FORMAT and model["n"] == 260 and model["p"] == 1
