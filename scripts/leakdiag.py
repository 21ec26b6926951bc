"""Diagnostic: is DeviceBuffer.__del__ freeing (run under compute-sanitizer --leak-check full)."""
import gc, sys
sys.path.insert(0, ".")
import numpy as np
import paro_b200 as paro
orig = paro.DeviceBuffer.close
def traced(self):
    print("close", self.nbytes, self.ptr is not None, flush=True)
    if self.ptr:
        r = paro._lib.paro_device_free(paro.P(self.ptr))
        print("  free ->", r, paro._lib.paro_last_error(), flush=True)
        self.ptr = None
paro.DeviceBuffer.close = traced
ctx = paro.Context(0)
b = paro.DeviceBuffer(1000)
del b
gc.collect()
g = paro.parse_grid("F:2,H:8,W:8"); plan = paro.make_perm(g, "WFH")
s = ctx.block_sums(np.random.rand(128, 128).astype(np.float32), 64, plan)
gc.collect()
print("before close", flush=True)
ctx.close()
