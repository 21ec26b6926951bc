"""P codes on adversarial tiles, code for code against the oracle.

The fast quantizer's exactness band (kappa) is sized relative to the
quotient q = (p - lo) / pscale, while the fast p carries an error relative to p itself.
The two differ most on tiles whose p values sit in a narrow range far above zero
(hi - lo << lo: lo / pscale is large, above all with INT4 P) and on tiles whose
exponents are large (tiny p, the ex2 argument's rounding scales with |log2 p|).
These layers build exactly those tiles:

  flat    keys = one shared direction + small noise: every row's logits nearly equal,
          p within a few percent of 1 across the whole tile
  steep   queries scaled up: logits spread over hundreds of units, p down to the
          fp32 subnormal range
  mixed   flat and steep rows in one q-block (one P group spans both)
  degenerate  identical keys: a row's logits all equal, so a tile's p are all equal
          (hi == lo, pscale 0 in the reference's formula)
  cancel  (d=128) the two 64-column groups' S terms large and of opposite sign, so the
          exp2 argument is a small difference of large products (its fp32 error scales
          with |S|, not with the argument)

and compare every quantized tile's final codes (after the exact boundary path) with the
oracle's quant_affine of the reference's fp32(exp(fp64 logit - m)). "flat" failed (4 of 4
cases) with the relative-only band q (1 -/+ kappa); the absolute term of pgroup_consts
(k3_common.cuh) fixed it. "cancel" left 1 flip in 215 INT8 tiles at d=128 with the plain
two-FMA exp2 argument; the INT8-P d=128 kernel now forms it cancellation-free
(arg128_2; INT4 P passes without it).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRIDS = {"even": "H:16,W:16", "ragged": "H:15,W:17"}  # 256 tokens / 255 (a ragged last block)
H = 4


def make_inputs(family, seed, N, d):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((H, N, d)).astype(np.float32)
    k = rng.standard_normal((H, N, d)).astype(np.float32)
    v = rng.standard_normal((H, N, d)).astype(np.float32)
    if family == "flat":
        base = rng.standard_normal((H, 1, d)).astype(np.float32)
        eps = np.float32(10.0 ** rng.uniform(-3, -1))
        k = base + eps * k
    elif family == "degenerate":  # identical keys: every logit of a row equal, hi == lo
        k = np.broadcast_to(rng.standard_normal((H, 1, d)).astype(np.float32), (H, N, d)).copy()
    elif family == "steep":
        q *= np.float32(rng.uniform(4.0, 16.0))
    elif family == "cancel":  # d=128: the two 64-column halves' S terms large and opposite
        if d == 128:
            q[..., 64:] = -q[..., :64] * np.float32(rng.uniform(0.9, 1.1))
            k[..., 64:] = k[..., :64] + np.float32(0.05) * k[..., 64:]
            q *= np.float32(rng.uniform(2.0, 6.0))
        else:
            q *= np.float32(3.0)
    else:  # mixed: half the rows of every q-block flat against shared keys, half steep
        base = rng.standard_normal((H, 1, d)).astype(np.float32)
        k = base + np.float32(0.02) * k
        q[:, ::2] *= np.float32(12.0)
    return q, k, v


@pytest.mark.parametrize("grid", ["even", "ragged"])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("pv_bits", [4, 8])
@pytest.mark.parametrize("family", ["flat", "steep", "mixed", "cancel", "degenerate"])
def test_p_codes_adversarial(paro, ctx, oracle, family, pv_bits, d, grid):
    g = paro.parse_grid(GRIDS[grid])
    N = g.token_count()
    kb = (N + 63) // 64
    orders = paro.enumerate_orders(g)
    ords = [orders[h % len(orders)] for h in range(H)]
    flips_total = tiles_total = 0
    bad = []
    for seed in range(4):
        q, k, v = make_inputs(family, 7000 + 97 * seed + d + pv_bits, N, d)
        rng = np.random.default_rng(seed)
        masks = (rng.random((H, kb, kb)) < (1.0 if seed % 2 == 0 else 0.6)).astype(np.uint8)
        masks[:, np.arange(kb), np.arange(kb)] = 1  # every q-block keeps a tile
        layer = paro.Layer(ctx, H, d, g, ords)
        layer.set_masks(masks)
        bufs = [paro.DeviceBuffer.from_array(x) for x in (q, k, v)]
        layer.reorder_quantize(bufs[0].ptr, bufs[1].ptr, bufs[2].ptr, pv_bits)
        targets = np.array([(h, qb) for h in range(H) for qb in range(kb)], np.uint32)
        codes, meta = layer.debug_pdump(targets, 0.0, pv_bits)
        layer.close()
        for x in bufs:
            x.close()
        for ti, (h, qb) in enumerate(targets):
            plan = paro.make_perm(g, ords[h])
            qp, kp, vp = (np.ascontiguousarray(x[h][plan.inverse]) for x in (q, k, v))
            _, _, bj, lo, ps, oc = oracle.pdump(qp, kp, vp, int(qb), masks[h], pv_bits)
            n = len(bj)
            assert np.array_equal(meta[ti, :n, 2].astype(np.int64), bj.astype(np.int64)), (family, seed, h, qb)
            qn = min(64, N - int(qb) * 64)
            for t in range(n):
                kn = min(64, N - int(bj[t]) * 64)
                flips = int(np.count_nonzero(codes[ti, t, :qn, :kn] != oc[t, :qn, :kn]))
                if flips and len(bad) < 8:
                    bad.append((seed, int(h), int(qb), t, flips, float(lo[t]), float(ps[t])))
                flips_total += flips
            tiles_total += n
    print(f"{family} INT{pv_bits} d={d} {grid}: {tiles_total} tiles, code flips {flips_total}")
    assert tiles_total > 0
    assert flips_total == 0, bad
