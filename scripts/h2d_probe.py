import torch, numpy as np, time
n = 216 * 1000 * 1000 // 4
srcs = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(3)]
dsts = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(3)]
outs_h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(1)]
outs_d = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(1)]
ev = lambda: torch.cuda.Event(enable_timing=True)
def run(nstreams, with_d2h=False, chunks=12):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    sd = torch.cuda.Stream()
    torch.cuda.synchronize()
    a = ev(); b = ev(); a.record()
    for s in streams: s.wait_event(a)
    sd.wait_event(a)
    i = 0
    for t in range(3):
        cs = n // chunks
        for c in range(chunks):
            s = streams[i % nstreams]; i += 1
            with torch.cuda.stream(s):
                dsts[t][c*cs:(c+1)*cs].copy_(srcs[t][c*cs:(c+1)*cs], non_blocking=True)
    if with_d2h:
        with torch.cuda.stream(sd):
            outs_h[0].copy_(outs_d[0], non_blocking=True)
    for s in streams: b.wait_stream(s) if False else None
    for s in streams: torch.cuda.current_stream().wait_stream(s)
    torch.cuda.current_stream().wait_stream(sd)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"streams {nstreams} d2h {with_d2h}: {ms:.2f} ms, H2D {3*n*4/ms/1e6:.1f} GB/s")
for ns in (1, 2, 3, 4):
    run(ns); run(ns); run(ns, True)
