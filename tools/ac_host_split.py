import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2007_05239_b200 import AllenCahnParams, LabelData, SpectralBasis, allen_cahn_solve
n, k, m = 10000000, 10, 4
rng = np.random.default_rng(0)
phi = torch.randn(n, k, dtype=torch.float64, device="cuda") / 3000
ids = rng.integers(0, m, n); ids[rng.random(n) > 0.05] = -1
labels = LabelData.from_class_ids(ids, m, 1000.0)
basis = SpectralBasis(values=np.linspace(0.5, 1.5, k), vectors=phi)
for it in (5, 25):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = allen_cahn_solve(basis, labels, AllenCahnParams(tolerance=0.0, max_iter=it), return_device=True)
    torch.cuda.synchronize(); print(it, time.perf_counter() - t0)
