import torch, time
n = 1357952040 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
def bench(fn, label, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{label}: {ms:.2f} ms  {n*8/ms/1e6:.1f} GB/s per direction-copy")
streams = [torch.cuda.Stream() for _ in range(8)]
def h2d(): d.copy_(h, non_blocking=True)
def d2h(): h2.copy_(d2, non_blocking=True)
def both():
    s0, s1 = streams[0], streams[1]
    s0.wait_stream(torch.cuda.current_stream()); s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s0): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s1): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s0); torch.cuda.current_stream().wait_stream(s1)
def chunked(k):
    def f():
        cs = n // k
        cur = torch.cuda.current_stream()
        for i in range(k):
            s = streams[i % len(streams)]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i*cs:(i+1)*cs].copy_(h[i*cs:(i+1)*cs], non_blocking=True)
        for i in range(k): cur.wait_stream(streams[i % len(streams)])
    return f
def both_chunked(k):
    def f():
        cs = n // k
        cur = torch.cuda.current_stream()
        for i in range(k):
            s = streams[(2*i) % len(streams)]; t = streams[(2*i+1) % len(streams)]
            s.wait_stream(cur); t.wait_stream(cur)
            with torch.cuda.stream(s): d[i*cs:(i+1)*cs].copy_(h[i*cs:(i+1)*cs], non_blocking=True)
            with torch.cuda.stream(t): h2[i*cs:(i+1)*cs].copy_(d2[i*cs:(i+1)*cs], non_blocking=True)
        for st in streams: cur.wait_stream(st)
    return f
bench(h2d, "H2D single")
bench(d2h, "D2H single")
bench(both, "H2D+D2H concurrent")
bench(chunked(4), "H2D 4 chunks / 4 streams")
bench(both_chunked(4), "H2D+D2H 4 chunks each")
