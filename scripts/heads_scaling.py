"""K3/K1/K2 time per layer vs head count at the c2 shape (what one rank of an N-GPU head shard runs)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paro_b200 as paro

grid_text, H, d, density, pv, _ = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
ctx = paro.Context(0)
g = paro.parse_grid(grid_text)
N = g.token_count()
s = torch.cuda.current_stream(); sp = s.cuda_stream
for hn in [H, H // 2, H // 4, H // 8]:
    heads = list(range(hn))
    orders, q, k, v, masks = bench.workload_ours(paro, ctx, heads, grid_text, N, d, density, "random")
    layer = paro.Layer(ctx, hn, d, g, orders)
    dq, dk, dv = (torch.from_numpy(x).cuda() for x in (q, k, v))
    dm = torch.from_numpy(masks).cuda()
    out = torch.empty_like(dq); z = torch.empty((hn, N), dtype=torch.uint8, device="cuda")
    def step():
        layer.set_masks_device(dm.data_ptr(), sp)
        layer.reorder_quantize(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), pv, sp)
        layer.attention(0.0, pv, out.data_ptr(), z.data_ptr(), sp)
    for _ in range(3): step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(10): step()
    b.record(s); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"heads {hn:3d}: {ms:.3f} ms/layer-shard  -> x{H // hn} shards = {ms * H / hn:.3f} ms-equivalent")
    layer.close()
