"""ncu driver: one W v apply of the config-5 micro points (uniform ball) for one (n, d, N, m).

    python tools/prof_micro.py [n] [d] [N] [m]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import synth
from paper_2007_05239_b200 import KernelSpec, bind_points, build_plan, fastsum


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10 ** 7
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    N = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    m = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    torch.cuda.set_device(0)
    x, v = synth.config5_micro(n, d, seed=0)
    plan = build_plan(KernelSpec("gaussian", 0.2), d=d, N=N, m_nfft=m, p_nfft=8)
    b = bind_points(plan, x)
    vd = torch.from_numpy(v).cuda()
    y = torch.empty_like(vd)
    for _ in range(2):
        fastsum.apply_binding(b, vd, y, -1.0, 1.0, 0.0, 0)
    torch.cuda.synchronize()
    print(b.stats())


if __name__ == "__main__":
    main()
