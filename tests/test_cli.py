"""Command-line front end (cli.py / config.py / runner.py of the reference):
config validation, CSV formats and exit codes on the CPU; the GPU pipelines
(`eig`, `classify`, `fastsum-bench`) against the in-process API."""

import json
import os

import numpy as np
import pytest
from numpy.testing import assert_allclose

from conftest import load_golden


def test_config_defaults_and_validation(tmp_path):
    from paper_2007_05239_b200 import ConfigError
    from paper_2007_05239_b200.config import DEFAULTS, load_config, merge_config
    cfg = load_config(None)
    assert cfg == DEFAULTS and cfg is not DEFAULTS
    cfg = merge_config({"fastsum": {"N": 32}, "eig": {"k": 4}})
    assert cfg["fastsum"]["N"] == 32 and cfg["fastsum"]["m"] == 5 and cfg["eig"]["k"] == 4
    for bad, msg in [({"fastsum": {"NN": 1}}, "fastsum.NN"), ({"eig": 3}, "must be an object"),
                     ({"grouping": {"groups": []}}, "non-empty"),
                     ({"grouping": {"groups": [{"columns": [0]}]}}, "sigma"),
                     ({"grouping": {"groups": [{"columns": [0], "sigma": 1, "colour": 2}]}}, "colour")]:
        with pytest.raises(ConfigError, match=msg):
            merge_config(bad)
    p = tmp_path / "bad.json"
    p.write_text("{\n  \"eig\": {\"k\": 3,}\n}")
    with pytest.raises(ConfigError, match="line 2"):
        load_config(str(p))


def test_csv_formats(tmp_path):
    from paper_2007_05239_b200 import FormatError
    from paper_2007_05239_b200.csvio import (load_features_csv, load_labels_csv, write_matrix_csv,
                                            write_predictions_csv)
    f = tmp_path / "x.csv"
    f.write_text("a,b\n1,2.5\n\n3,4e-1\n")
    assert_allclose(load_features_csv(str(f)), [[1, 2.5], [3, 0.4]])
    f.write_text("1,2\n3\n")
    with pytest.raises(FormatError, match=":2: expected 2 columns"):
        load_features_csv(str(f))
    lab = tmp_path / "l.csv"
    lab.write_text("class\n1\n0\n3\n")
    assert load_labels_csv(str(lab)).tolist() == [0, -1, 2]
    with pytest.raises(FormatError, match="labels for 4 nodes"):
        load_labels_csv(str(lab), n=4)
    lab.write_text("-1\n")
    with pytest.raises(FormatError, match="1-based"):
        load_labels_csv(str(lab))
    out = tmp_path / "p.csv"
    write_predictions_csv(str(out), np.array([0, 2]))
    assert out.read_text() == "node_id,class_id\n0,1\n1,3\n"
    write_matrix_csv(str(out), np.array([0.1, 1 / 3]))
    assert_allclose(np.loadtxt(str(out)), [0.1, 1 / 3], rtol=0, atol=0)


def test_cli_exit_codes(tmp_path, capsys):
    from paper_2007_05239_b200.cli import main
    assert main(["eig", "--seed", "-1"]) == 2
    assert main(["eig", "--threads", "0"]) == 2
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"eig": {"kk": 1}}))
    assert main(["eig", "--config", str(cfg)]) == 2
    assert "unknown config key: eig.kk" in capsys.readouterr().err
    assert main(["eig", "--config", str(tmp_path / "missing.json")]) == 2
    assert main(["eig"]) == 2  # no graph input
    assert main(["segment-image"]) == 2   # no input.images
    assert main(["sbm-bench"]) == 2
    X = tmp_path / "x.csv"
    X.write_text("1,2\nx,3\n")
    cfg.write_text(json.dumps({"input": {"features_csv": str(X)},
                               "grouping": {"groups": [{"columns": [0, 1], "sigma": 1.0}]}}))
    if not _gpu():
        return
    assert main(["eig", "--config", str(cfg), "--out", str(tmp_path)]) == 4


def _gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def _feature_cfg(tmp_path, X, extra=None):
    xp = tmp_path / "features.csv"
    np.savetxt(str(xp), X, delimiter=",", fmt="%.17g", header="r,g,b,x,y", comments="")
    cfg = {"input": {"features_csv": str(xp)},
           "grouping": {"groups": [{"columns": [0, 1, 2], "sigma": 0.3}, {"columns": [3, 4], "sigma": 1.0}]},
           "fastsum": {"N": 32, "m": 4, "p": 8}, "power": {"p": -1.0}, "eig": {"k": 4}}
    for sec, vals in (extra or {}).items():
        cfg.setdefault(sec, {}).update(vals)
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    return str(path)


@pytest.mark.gpu
def test_cli_eig_and_classify_match_the_api(tmp_path):
    from paper_2007_05239_b200 import (AllenCahnParams, GroupingSpec, GroupSpec, KernelSpec,
                                       PowerMeanConfig, allen_cahn_solve, feature_group, power_mean_eigs,
                                       predict_labels)
    from paper_2007_05239_b200.cli import main
    X = load_golden("featuregroup")["X"]
    n = X.shape[0]
    truth = (X[:, 3] > np.median(X[:, 3])).astype(int)  # two spatial halves
    tp = tmp_path / "truth.csv"
    np.savetxt(str(tp), truth + 1, fmt="%d")
    cfg = _feature_cfg(tmp_path, X, {"input": {"truth_csv": str(tp), "label_fraction": 0.1},
                                     "output": {"write_vectors": True}})
    assert main(["eig", "--config", cfg, "--out", str(tmp_path / "eig")]) == 0
    vals = np.loadtxt(str(tmp_path / "eig" / "eigenvalues.csv"))
    spec = GroupingSpec((GroupSpec((0, 1, 2), KernelSpec("gaussian", 0.3)),
                         GroupSpec((3, 4), KernelSpec("gaussian", 1.0))))
    G = feature_group(X, spec, fastsum_params=dict(N=32, m_nfft=4, p_nfft=8, eps_b=0.0625, rho=2.0))
    basis = power_mean_eigs(G, PowerMeanConfig(p=-1.0), k=4, seed=0)
    assert_allclose(vals, basis.values, rtol=1e-12)
    rep = json.loads((tmp_path / "eig" / "report.json").read_text())
    assert rep["command"] == "eig" and rep["n"] == n and rep["layers"] == 2 and "eig" in rep["times"]
    assert np.loadtxt(str(tmp_path / "eig" / "eigenvectors.csv"), delimiter=",").shape == (n, 4)

    assert main(["classify", "--config", cfg, "--out", str(tmp_path / "cls")]) == 0
    rep = json.loads((tmp_path / "cls" / "report.json").read_text())
    from paper_2007_05239_b200 import sample_labels
    labels = sample_labels(truth, 0.1, (0, 1), 1000.0)
    res = allen_cahn_solve(basis, labels, AllenCahnParams())
    pred = predict_labels(res.scores)
    lines = (tmp_path / "cls" / "predictions.csv").read_text().splitlines()
    assert lines[0] == "node_id,class_id" and len(lines) == n + 1
    got = np.array([int(l.split(",")[1]) - 1 for l in lines[1:]])
    assert np.array_equal(got, pred)
    assert rep["iterations"] == res.iterations and rep["classes"] == 2
    assert abs(rep["accuracy"] - float(np.mean(pred == truth))) < 1e-15
    assert {"graph", "eig", "ac", "write", "total"} <= set(rep["times"])


@pytest.mark.gpu
def test_cli_fastsum_bench(tmp_path):
    from paper_2007_05239_b200.cli import main
    cfg = tmp_path / "fb.json"
    cfg.write_text(json.dumps({"fastsum": {"N": 32, "m": 4, "p": 8},
                               "bench": {"fastsum": {"sizes": [2000, 5000], "repetitions": 2, "accuracy_n": 1500,
                                                     "accuracy_dims": [1, 2, 3], "sigma": 0.1, "d": 2}}}))
    assert main(["fastsum-bench", "--config", str(cfg), "--out", str(tmp_path)]) == 0
    rep = json.loads((tmp_path / "report.json").read_text())
    errs = {r["d"]: r["rel_error"] for r in rep["accuracy"]}
    # approximation error of the NFFT sum at N=32 vs the exact sum (App. B.3 magnitudes)
    assert errs[1] < 1e-6 and errs[2] < 1e-5 and errs[3] < 1e-3
    assert len(rep["scaling"]["t_fast"]) == 2 and all(t > 0 for t in rep["scaling"]["t_fast_device"])
    head = (tmp_path / "fastsum_scaling.csv").read_text().splitlines()[0]
    assert head == "n,t_fast_median,t_direct_median"   # the reference's format (ref test_cli.py:215)
    dev = (tmp_path / "fastsum_scaling_device.csv").read_text().splitlines()
    assert dev[0] == "n,t_fast_device_median" and len(dev) == 3
    assert os.path.exists(tmp_path / "fastsum_bench.txt")
