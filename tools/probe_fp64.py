"""FP64 FMA vs FP64 tensor-core (DMMA m8n8k4) throughput on this GPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2007_05239_b200 import _lib


def timed(fn, reps=3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best * 1e-3


lib = _lib.lib()
out = torch.zeros(1, dtype=torch.float64, device="cuda")
for blocks in (148 * 2, 148 * 4, 148 * 8):
    it = 20000
    t = timed(lambda: lib.mlb_probe_fp64(it, blocks, _lib.ptr(out), _lib.stream_ptr()))
    print(f"DFMA blocks={blocks}: {2.0 * 8 * it * blocks * 256 / t / 1e12:.2f} TFLOP/s")
    it = 5000
    t = timed(lambda: lib.mlb_probe_dmma(it, blocks, _lib.ptr(out), _lib.stream_ptr()))
    print(f"DMMA blocks={blocks}: {blocks * 8 * it * 4 * 512 / t / 1e12:.2f} TFLOP/s")
