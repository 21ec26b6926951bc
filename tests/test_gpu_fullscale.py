"""Parity at BASELINE.json's full sizes (c2..c5 shapes): GPU layer output vs the
restated INT8-QK oracle on sampled q-blocks of sampled heads (the oracle is exact
per q-tile, attention.cpp:134, so a q-block sample is a complete check of those
rows), plus size-independent properties over the whole layer.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

OUT_TOL = 1e-3
EXACT_TOL = 1e-5  # bit-exact P codes (see test_gpu_parity.py)

FULL = [
    # grid, heads (run), d, density, pv_bits, q-blocks sampled per head
    ("F:13,H:30,W:45", 2, 64, 0.3, 8, 12),   # c2 (CogVideoX)
    ("F:13,H:30,W:45", 2, 64, 0.2, 4, 12),   # c3
    ("H:64,W:64", 2, 128, 0.3, 8, 16),        # c4
    ("H:64,W:64", 2, 128, 0.3, 4, 16),        # c4 INT4
    ("F:21,H:45,W:80", 1, 128, 0.2, 4, 4),   # c5 (Wan) -- N=75600
]


@pytest.mark.parametrize("grid,H,d,density,pv_bits,nsample", FULL)
def test_full_size_sampled_rows(paro, ctx, oracle, grid, H, d, density, pv_bits, nsample):
    import bench

    g = paro.parse_grid(grid)
    N = g.token_count()
    kb = (N + 63) // 64
    heads = list(range(H))
    orders, q, k, v, masks = bench.workload_ours(paro, ctx, heads, grid, N, d, density, "random")
    layer = paro.Layer(ctx, H, d, g, orders)
    layer.set_masks(masks)
    out, zeroed = layer.forward_host(q, k, v, 0.0, pv_bits)
    layer.close()
    assert np.isfinite(out).all()
    assert not zeroed.any()  # gen_mask repairs every row (mask.cpp:95-128)

    rng = np.random.default_rng(17)
    jobs = []
    for h in heads:
        plan = paro.make_perm(g, orders[h])
        qp, kp, vp = (np.ascontiguousarray(x[h][plan.inverse]) for x in (q, k, v))
        sample = sorted(set(rng.choice(kb, nsample, replace=False).tolist()) | {kb - 1, 0})
        for qb in sample:
            jobs.append((h, qb, plan, qp, kp, vp))

    def run(job):
        h, qb, plan, qp, kp, vp = job
        ref, _ = oracle.stream_engine_range(qp, kp, vp, qb, qb + 1, masks[h], pv_bits, qk_mode=1)
        rows = plan.inverse[qb * 64:min(N, qb * 64 + 64)]
        return h, out[h][rows], ref

    with ThreadPoolExecutor(8) as ex:
        res = list(ex.map(run, jobs))
    # error normalised per head over the sampled rows (max|dO| / max|O|)
    for h in heads:
        got = np.concatenate([r[1] for r in res if r[0] == h])
        ref = np.concatenate([r[2] for r in res if r[0] == h])
        err = rel_err(got, ref)
        print(f"{grid} d={d} pv={pv_bits} head {h}: max|dO|/max|O| = {err:.3e}")
        assert err <= EXACT_TOL, err  # bit-exact P codes at d=64 and d=128
