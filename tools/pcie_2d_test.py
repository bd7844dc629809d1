"""Strided host->device copy of the 4 diffused fields of an (ng, 5) state (dev helper):
cudaMemcpy2DAsync with 32-byte rows vs the full 40-byte rows, alone and concurrent with a D2H."""
import ctypes as C

import torch

ng = 1357952040 // 40
rt = C.CDLL("libcudart.so") if False else None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        rt = C.CDLL(name)
        break
    except OSError:
        pass
if rt is None:
    import glob
    import os
    cand = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
    rt = C.CDLL(cand[0])
h = torch.empty((ng, 5), dtype=torch.float64, pin_memory=True)
h2 = torch.empty((ng, 5), dtype=torch.float64, pin_memory=True)
d4 = torch.empty((ng, 4), dtype=torch.float64, device="cuda")
d5 = torch.empty((ng, 5), dtype=torch.float64, device="cuda")
rt.cudaMemcpy2DAsync.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int,
                                 C.c_void_p]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def h2d_2d(stream):
    rc = rt.cudaMemcpy2DAsync(d4.data_ptr(), 32, h.data_ptr() + 8, 40, 32, ng, 1, stream.cuda_stream)
    assert rc == 0, rc


def bench(fn, label, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / reps:.2f} ms", flush=True)


bench(lambda: d5.copy_(h, non_blocking=True), "H2D (ng,5) full rows")
bench(lambda: h2d_2d(torch.cuda.current_stream()), "H2D (ng,4) via 2D 32-of-40-byte rows")


def both_2d():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    h2d_2d(s1)
    with torch.cuda.stream(s2):
        h2.copy_(d5, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def both_full():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d5.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d5, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


bench(both_full, "H2D full + D2H full concurrent")
bench(both_2d, "H2D 2D + D2H full concurrent")
