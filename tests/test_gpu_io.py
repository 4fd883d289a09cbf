"""fit -> model JSON -> predictions CSV through the device path, against the
reference's own outputs for the same files and seeds (tests/golden/cli_logit)."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli_logit")


def test_fit_and_predict_files_match_reference(tmp_path):
    from paper_2310_12000_b200 import io
    cfg = json.load(open(os.path.join(HERE, "fit.json")))
    res = io.run_fit(os.path.join(HERE, "train.csv"), cfg, str(tmp_path / "model.json"))
    ref = io.load_model(os.path.join(HERE, "model.json"))
    got = io.load_model(str(tmp_path / "model.json"))
    assert got["n_evaluations"] == ref["n_evaluations"] and got["iterations"] == ref["iterations"]
    np.testing.assert_allclose(got["estimates"]["theta"], ref["estimates"]["theta"], rtol=1e-6)
    np.testing.assert_allclose(got["estimates"]["beta"], ref["estimates"]["beta"], rtol=1e-6)
    np.testing.assert_allclose(got["objective"], ref["objective"], rtol=1e-8)
    assert set(got) == set(ref)
    pcfg = json.load(open(os.path.join(HERE, "predict.json")))
    # predict from the REFERENCE's model file, so the comparison isolates the prediction path
    io.run_predict(os.path.join(HERE, "model.json"), os.path.join(HERE, "train.csv"), os.path.join(HERE, "pred.csv"),
                   pcfg, str(tmp_path / "pred_out.csv"))
    hr, ar = io.read_csv(os.path.join(HERE, "predictions.csv"))
    hg, ag = io.read_csv(str(tmp_path / "pred_out.csv"))
    assert hr == hg
    np.testing.assert_allclose(ag, ar, rtol=1e-7, atol=1e-10)
    comments = lambda p: [ln for ln in open(p) if ln.startswith("#")]  # noqa: E731
    cr, cg = comments(os.path.join(HERE, "predictions.csv")), comments(str(tmp_path / "pred_out.csv"))
    assert cr[0] == cg[0]
    for a, b in zip(cr[1:], cg[1:]):
        ka, va = a.strip("# \n").split("=")
        kb, vb = b.strip("# \n").split("=")
        assert ka == kb and float(va) == pytest.approx(float(vb), rel=1e-7)
    assert res.converged in (True, False)
