"""`segment-image` end to end (ref runner.py:271-333, cli.py:43-98) on the
B200 backend against a frozen run of the REAL reference
(oracle/gen_golden_segment.py): two RGB PNGs, the default image grouping
(colour layer + per-image spatial layer, per-component bindings), p = -1,
k = 8, 6% labels; eigenvalues <= 1e-7, predicted labels identical on >=
99.9% of the pixels, same Allen-Cahn iterations, mask / composite PNGs."""

import json
import os

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_segment_image_matches_frozen_reference(tmp_path):
    from PIL import Image

    from paper_2007_05239_b200.cli import main
    g = load_golden("segment")
    paths = []
    for i in range(2):
        p = tmp_path / f"img{i}.png"
        Image.fromarray(g[f"img{i}"], mode="RGB").save(p)
        paths.append(str(p))
    tp = tmp_path / "truth.csv"
    np.savetxt(tp, g["truth"] + 1, fmt="%d")
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"input": {"images": paths, "truth_csv": str(tp), "label_fraction": 0.06},
                               "power": {"p": -1.0}, "eig": {"k": 8}}))
    out = tmp_path / "out"
    assert main(["segment-image", "--config", str(cfg), "--out", str(out)]) == 0
    rep = json.loads((out / "report.json").read_text())
    vals = np.array(rep["eigenvalues"])
    assert np.max(np.abs(vals - g["values"]) / np.abs(g["values"])) <= 1e-7
    pred = np.loadtxt(out / "predictions.csv", dtype=np.int64, skiprows=1, delimiter=",")[:, 1] - 1
    agree = float(np.mean(pred == g["pred"]))
    print(f"segment-image: labels identical on {agree:.5f}, accuracy {rep['accuracy']:.4f} "
          f"(reference {float(g['accuracy'][0]):.4f}), iterations {rep['iterations']} (reference {int(g['iters'][0])})")
    assert agree >= 0.999
    assert rep["iterations"] == int(g["iters"][0])
    assert rep["images"] == [[36, 48], [30, 40]]
    for key in ("mask_img0_class1", "mask_img1_class3", "composite_img0", "composite_img1"):
        assert os.path.exists(rep["outputs"][key]), key
    comp = np.asarray(Image.open(rep["outputs"]["composite_img1"]))
    assert comp.shape == (30, 40, 3)
