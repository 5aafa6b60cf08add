"""Golden run of the REAL reference's `segment-image` pipeline (build
container only; TEST INFRASTRUCTURE).

    python oracle/gen_golden_segment.py      (~1 minute of CPU)

Two seeded synthetic RGB images (36 x 48 and 30 x 40, three classes as
rectangles over a background, class colours + N(0, 12^2) noise, uint8),
ground truth per pixel, config: power.p = -1, eig.k = 8, 6% labels sampled
from the truth, every other key the reference's default (the default image
grouping: colour layer + per-image spatial layer in "unit-box" mode, N = 64,
m = 5).  Runs multilap.runner.run_segment_image (runner.py:271-333) and
freezes the images, the truth, the eigenvalues, the predictions and the
Allen-Cahn iteration count into tests/golden/golden_segment.npz.
"""

import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.environ.get("MULTILAP_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)


def make_images(seed=0):
    rng = np.random.default_rng(seed)
    imgs, truths = [], []
    colours = rng.integers(30, 226, size=(4, 3))
    for h, w in ((36, 48), (30, 40)):
        t = np.zeros((h, w), dtype=np.int64)
        for c in (1, 2, 3):
            y0, x0 = rng.integers(0, h // 2), rng.integers(0, w // 2)
            t[y0:y0 + rng.integers(6, h // 2), x0:x0 + rng.integers(6, w // 2)] = c
        img = colours[t] + rng.normal(0.0, 12.0, (h, w, 3))
        imgs.append(np.clip(np.rint(img), 0, 255).astype(np.uint8))
        truths.append(t.ravel())
    return imgs, np.concatenate(truths)


def write_inputs(d, imgs, truth):
    from PIL import Image
    paths = []
    for i, img in enumerate(imgs):
        p = os.path.join(d, f"img{i}.png")
        Image.fromarray(img, mode="RGB").save(p)
        paths.append(p)
    tp = os.path.join(d, "truth.csv")
    np.savetxt(tp, truth + 1, fmt="%d")   # class IDs are 1-based in the label files
    cfg = {"input": {"images": paths, "truth_csv": tp, "label_fraction": 0.06},
           "power": {"p": -1.0}, "eig": {"k": 8}}
    cp = os.path.join(d, "cfg.json")
    with open(cp, "w") as fh:
        json.dump(cfg, fh)
    return cp


def main():
    from multilap.config import load_config
    from multilap.runner import run_segment_image
    imgs, truth = make_images()
    with tempfile.TemporaryDirectory() as d:
        cp = write_inputs(d, imgs, truth)
        rep = run_segment_image(load_config(cp), 0, out_dir=d)
        pred = np.loadtxt(os.path.join(d, "predictions.csv"), dtype=np.int64, skiprows=1, delimiter=",")[:, 1] - 1
    out = os.path.join(ROOT, "tests", "golden", "golden_segment.npz")
    np.savez_compressed(out, img0=imgs[0], img1=imgs[1], truth=truth, values=np.array(rep["eigenvalues"]),
                        iters=np.array([rep["iterations"], int(rep["converged"])]),
                        accuracy=np.array([rep["accuracy"]]), pred=pred)
    print(f"wrote {out}: accuracy {rep['accuracy']:.4f}, {rep['iterations']} AC iterations, values {rep['eigenvalues']}")


if __name__ == "__main__":
    main()
