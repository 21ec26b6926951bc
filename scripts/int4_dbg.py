"""Reduced INT4 d=128 case with more items than CTAs (for compute-sanitizer)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import bench
import paro_b200 as paro

H = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctx = paro.Context(0)
grid = "H:64,W:64"
g = paro.parse_grid(grid)
N = g.token_count()
orders, q, k, v, masks = bench.workload_ours(paro, ctx, list(range(H)), grid, N, 128, 0.3, "random")
layer = paro.Layer(ctx, H, 128, g, orders)
layer.set_masks(masks)
out, z = layer.forward_host(q, k, v, 0.0, 4)
print("ok", float(np.abs(out).max()))
