"""H2D / D2H bandwidth of pinned host buffers: cudaHostAlloc (torch) versus
2 MiB-aligned transparent-huge-page memory registered with cudaHostRegister."""
import ctypes, mmap, os, sys
import numpy as np, torch

libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.posix_memalign.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_size_t]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
MADV_HUGEPAGE = 14
rt = torch.cuda.cudart()


def thp_buffer(nbytes, huge=True):
    p = ctypes.c_void_p()
    sz = (nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    assert libc.posix_memalign(ctypes.byref(p), 2 << 20, sz) == 0
    if huge:
        assert libc.madvise(p, sz, MADV_HUGEPAGE) == 0
    arr = np.ctypeslib.as_array((ctypes.c_double * (sz // 8)).from_address(p.value))
    arr[:] = 0.0
    assert int(rt.cudaHostRegister(p.value, sz, 0)) == 0
    return torch.from_numpy(arr[: nbytes // 8])


def timeit(fn, reps=50):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(5):
        fn()
    e[0].record()
    for _ in range(reps):
        fn()
    e[1].record(); e[1].synchronize()
    return e[0].elapsed_time(e[1]) / reps * 1e3


n = 262144
dev = torch.empty(2 * n, dtype=torch.float64, device="cuda")
for kind in ("cudaHostAlloc", "posix_memalign 4K", "THP", "cudaHostAlloc", "THP"):
    if kind == "cudaHostAlloc":
        h = torch.empty(2 * n, dtype=torch.float64, pin_memory=True)
    else:
        h = thp_buffer(16 * n, huge=(kind == "THP"))
    print(f"{kind:20s} pinned={h.is_pinned()}  H2D 2MB {timeit(lambda: dev[:n].copy_(h[:n], non_blocking=True)):6.1f} us"
          f"  D2H 2MB {timeit(lambda: h[:n].copy_(dev[:n], non_blocking=True)):6.1f} us"
          f"  D2H 4MB {timeit(lambda: h.copy_(dev, non_blocking=True)):6.1f} us", flush=True)
print(open("/proc/meminfo").read().split("AnonHugePages:")[1].split("\n")[0])
