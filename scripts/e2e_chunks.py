"""e2e (host buffers) layer time vs pipeline chunk count at c2, plus the raw pinned H2D / D2H ceiling."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paro_b200 as paro

grid_text, H, d, density, pv_bits, desc = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
ctx = paro.Context(0)
g = paro.parse_grid(grid_text)
N = g.token_count()
heads = list(range(H))
orders, q, k, v, masks = bench.workload_ours(paro, ctx, heads, grid_text, N, d, density, "random")
layer = paro.Layer(ctx, H, d, g, orders)
dmask = torch.from_numpy(masks).cuda()
hq, hk, hv = (paro.HostBuffer(q.shape, np.float32) for _ in range(3))
hq.array[...] = q; hk.array[...] = k; hv.array[...] = v
hout = paro.HostBuffer(q.shape, np.float32)
hz = paro.HostBuffer((H, N), np.uint8)
s = torch.cuda.current_stream(); sp = s.cuda_stream
ev = lambda: torch.cuda.Event(enable_timing=True)
# raw copy ceiling
dq = torch.empty(q.shape, dtype=torch.float32, device="cuda")
src = torch.from_numpy(hq.array)
for _ in range(2):
    dq.copy_(src, non_blocking=True)
torch.cuda.synchronize()
a, b = ev(), ev(); a.record(); 
for _ in range(5):
    dq.copy_(src, non_blocking=True)
b.record(); torch.cuda.synchronize()
print(f"pinned H2D {q.nbytes/1e9:.3f} GB: {q.nbytes*5/ (a.elapsed_time(b)*1e-3)/1e9:.1f} GB/s")
dst = torch.from_numpy(hout.array)
a, b = ev(), ev(); a.record()
for _ in range(5):
    dst.copy_(dq, non_blocking=True)
b.record(); torch.cuda.synchronize()
print(f"pinned D2H: {q.nbytes*5/ (a.elapsed_time(b)*1e-3)/1e9:.1f} GB/s")
for ch in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,8,12,16,24,48").split(",")]:
    layer.set_pipeline_chunks(ch)
    for _ in range(2):
        layer.set_masks_device(dmask.data_ptr(), sp)
        layer.forward_host(hq.array, hk.array, hv.array, 0.0, pv_bits, hout.array, hz.array, sp)
    torch.cuda.synchronize()
    a, b = ev(), ev(); a.record(s)
    for _ in range(5):
        layer.set_masks_device(dmask.data_ptr(), sp)
        layer.forward_host(hq.array, hk.array, hv.array, 0.0, pv_bits, hout.array, hz.array, sp)
    b.record(s); torch.cuda.synchronize()
    print(f"chunks {ch}: e2e {a.elapsed_time(b)/5:.3f} ms/layer (3 x H2D {3*q.nbytes/1e9:.2f} GB)")
