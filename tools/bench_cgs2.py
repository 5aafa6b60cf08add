"""Device time of one CGS2 (krylov.cgs2) at several sizes (profiling aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2007_05239_b200.krylov import cgs2

torch.cuda.set_device(0)
for n in (40000, 262144, 1000000, 10000000):
    dim = 52
    V = torch.randn((dim, n), dtype=torch.float64, device="cuda")
    w0 = torch.randn(n, dtype=torch.float64, device="cuda")
    h = torch.empty(2 * dim + 3, dtype=torch.float64, device="cuda")
    row = []
    for cols in (6, 11, 21, 51):
        w = w0.clone()
        for _ in range(3):
            cgs2(V, cols, w, h[:cols], h[dim:dim + cols], h[2 * dim:2 * dim + 1])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            cgs2(V, cols, w, h[:cols], h[dim:dim + cols], h[2 * dim:2 * dim + 1])
        e1.record(); e1.synchronize()
        t = e0.elapsed_time(e1) / 20 * 1e3
        gbs = 4 * cols * n * 8 / (t * 1e-6) / 1e9
        row.append(f"cols={cols:2d} {t:7.1f} us ({gbs:5.0f} GB/s at 4 passes)")
    print(f"n={n:9d}: " + "; ".join(row))
