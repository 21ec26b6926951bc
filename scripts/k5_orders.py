"""K5a block_sums time per candidate order on one c2-shaped map (identity order passes no table)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paro_b200 as paro
from paro_b200 import _lib, P, U32

g = paro.parse_grid("F:13,H:30,W:45")
n = g.token_count(); k = (n + 63) // 64
torch.manual_seed(0)
dmap = torch.rand((n, n), device="cuda", dtype=torch.float32)
sums = torch.empty((k, k), dtype=torch.float64, device="cuda")
maxs = torch.empty((k, k), dtype=torch.float32, device="cuda")
cnts = torch.empty((k, k), dtype=torch.int32, device="cuda")
ctx = paro.Context(0)
s = torch.cuda.current_stream()
for order in paro.enumerate_orders(g):
    plan = paro.make_perm(g, order)
    dinv = torch.from_numpy(plan.inverse.astype(np.int32)).cuda()
    ident = order == g.labels
    for stats in (False,):
        def run():
            _lib.paro_perm_block_sums_device(P(ctx.ptr), P(s.cuda_stream), P(dmap.data_ptr()), U32(n), P(None if ident else dinv.data_ptr()),
                                             U32(64), P(sums.data_ptr()))
        for _ in range(2): run()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(10): run()
        b.record(s); torch.cuda.synchronize()
        print(order, "stats" if stats else "sums ", f"{a.elapsed_time(b)/10*1e3:.0f} us")
