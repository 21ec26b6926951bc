"""Bit-exact integer stages at BASELINE.json's FULL shapes (c2..c5), every head.

north_star: "bit-exact for permutation indices, block masks, quantized integer
tensors and int32 QK^T accumulators". At the configs' real sizes:

* K1 (PARO gather + quantize): for EVERY head of c2 (48), c3 (48, V INT4), c4
  (24) and c5 (40): permutation tables, Q/K int8 codes and per-(block, group)
  scales (quantize {8, Symmetric, PerBlock, 64}, quant.cpp:60-104), V codes,
  per-tile scales and column sums (the engine's V tile quantizer,
  attention.cpp:104-126), against the C oracle on the same inputs.
* K1's arithmetic itself: the reciprocal + one-FMA-residual quotient and the
  dropped clamp (prep_kernels.cu quant_sym4) against IEEE x/scale + clamp +
  round-half-away (kernels_scalar.cpp:78-85) for EVERY finite amax bit pattern.
* int32 S = Q.K^T through K3's tcgen05 path (debug_qk): >= 1024 tiles per config.
* P codes (attention.cpp:201-228): the final codes K3 feeds to the P.V MMA, dumped
  for sampled q-blocks of c2, c3, c4 and c5, against the oracle's quantizer of
  the reference's fp64 p -- code for code.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FULL = {  # grid, heads, d, density, pv_bits (BASELINE.json configs[1..4])
    "c2": ("F:13,H:30,W:45", 48, 64, 0.3, 8),
    "c3": ("F:13,H:30,W:45", 48, 64, 0.2, 4),
    "c4": ("H:64,W:64", 24, 128, 0.3, 8),
    "c5": ("F:21,H:45,W:80", 40, 128, 0.2, 4),
}


def head_qkv(paro, h, N, d):
    """bench.py's inputs: MT19937-64 Box-Muller N(0,1), seed 1000 + 3h + {0,1,2}."""
    return [paro.synth_randn(1000 + 3 * h + i, N * d).reshape(N, d) for i in range(3)]


def layer_for(paro, ctx, cfg, heads, with_masks=False):
    import bench

    grid, H, d, density, vb = FULL[cfg]
    g = paro.parse_grid(grid)
    N = g.token_count()
    orders = paro.enumerate_orders(g)
    with ThreadPoolExecutor(8) as ex:
        ins = list(ex.map(lambda h: head_qkv(paro, h, N, d), heads))
    q, k, v = (np.stack([x[i] for x in ins]) for i in range(3))
    ords = [orders[h % len(orders)] for h in heads]
    layer = paro.Layer(ctx, len(heads), d, g, ords)
    masks = None
    if with_masks:
        kb = (N + 63) // 64
        ms, _ = ctx.gen_mask(np.stack([bench.head_sums(h, kb, density, "random") for h in heads]), density, 64)
        masks = np.stack([m.bits for m in ms])
        layer.set_masks(masks)
    return g, N, d, vb, ords, q, k, v, layer, masks


def chunks(H, n):
    return [list(range(h, min(H, h + n))) for h in range(0, H, n)]


@pytest.mark.parametrize("cfg,packed", [("c2", False), ("c3", False), ("c4", False), ("c5", False), ("c3", True),
                                        ("c5", True)])
def test_k1_every_head_bit_exact(paro, ctx, oracle, cfg, packed):
    """packed: INT4 V nibble-packed in HBM (paro_layer_set_v_packing), compared after unpacking"""
    grid, H, d, _, vb = FULL[cfg]
    G = d // 64
    checked = 0
    for heads in chunks(H, 8 if d == 64 else 4):
        g, N, d, vb, ords, q, k, v, layer, _ = layer_for(paro, ctx, cfg, heads)
        layer.set_v_packing(packed)
        kb = (N + 63) // 64
        bufs = [paro.DeviceBuffer.from_array(x) for x in (q, k, v)]
        layer.reorder_quantize(bufs[0].ptr, bufs[1].ptr, bufs[2].ptr, vb)
        paro.stream_sync()
        b = layer.buffers()

        def check(i):
            bad = []
            fwd, inv = oracle.make_perm(g.labels, g.extents, ords[i])
            if not (np.array_equal(b["inverse"][i], inv) and np.array_equal(b["forward"][i], fwd)):
                bad.append("perm")
            for name, x, sc in (("q", q[i], b["q_scales"][i]), ("k", k[i], b["meta"][i][:, :G])):
                codes, scales, _ = oracle.quantize(np.ascontiguousarray(x[inv]), 8, 1, 64)
                if not np.array_equal(b[name][i][:N].astype(np.int32), codes):
                    bad.append(name + " codes")
                if not np.array_equal(np.ascontiguousarray(sc[:kb]).reshape(-1).view(np.uint32),
                                      scales.view(np.uint32)):
                    bad.append(name + " scales")
            vc, vs, vcs = oracle.quant_v(np.ascontiguousarray(v[i][inv]), vb)
            if not np.array_equal(b["v"][i][:N].astype(np.int32), vc):
                bad.append("v codes")
            if not np.array_equal(np.ascontiguousarray(b["meta"][i][:kb, 2]).view(np.uint32), vs.view(np.uint32)):
                bad.append("v scales")
            if not np.array_equal(b["meta"][i][:kb, 4:].astype(np.int64), vcs):
                bad.append("v colsums")
            return [(heads[i], x) for x in bad]

        with ThreadPoolExecutor(8) as ex:
            fails = sum(ex.map(check, range(len(heads))), [])
        assert not fails, f"{cfg}: {fails[:8]}"
        checked += len(heads)
        layer.close()
        for x in bufs:
            x.close()
    assert checked == H


def test_k1_quantizer_every_amax_bit_pattern(paro, ctx):
    """All 2^31 - 2^23 finite non-negative amax patterns x (2 + 14 x values) x (qmax 127, 7)."""
    bad, first = ctx.k1_quant_proof(0, 0x7F800000, nx=14, seed=1)
    assert bad == 0, f"first mismatch (amax bits, x bits, qmax, K1 code, reference code) = {first}"


def test_k1_quantizer_dense_x_sweep(paro, ctx):
    """A denser x sweep (254 x per scale) over every amax pattern in the binades that real
    activations use (2^-20 .. 2^20)."""
    lo = np.float32(2.0 ** -20).view(np.uint32)
    hi = np.float32(2.0 ** 20).view(np.uint32)
    bad, first = ctx.k1_quant_proof(int(lo), int(hi - lo), nx=254, seed=7)
    assert bad == 0, f"first mismatch = {first}"


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_qk_int32_full_shape(paro, ctx, cfg):
    grid, H, d, _, _ = FULL[cfg]
    G = d // 64
    n_tiles = 0
    rng = np.random.default_rng(5)
    for heads in (chunks(H, 8 if d == 64 else 4)[0], chunks(H, 8 if d == 64 else 4)[-1]):
        g, N, d, vb, ords, q, k, v, layer, _ = layer_for(paro, ctx, cfg, heads)
        kb = (N + 63) // 64
        bufs = [paro.DeviceBuffer.from_array(x) for x in (q, k, v)]
        layer.reorder_quantize(bufs[0].ptr, bufs[1].ptr, bufs[2].ptr, vb)
        paro.stream_sync()
        b = layer.buffers()
        tiles = np.stack([rng.integers(0, len(heads), 512), rng.integers(0, kb, 512), rng.integers(0, kb, 512)],
                         axis=1).astype(np.uint32)
        tiles[:8, 1] = kb - 1  # the ragged last q-block / key block
        tiles[8:16, 2] = kb - 1
        S = layer.debug_qk(tiles)
        for t, (h, qb, bj) in enumerate(tiles):
            Q = b["q"][h][qb * 64:(qb + 1) * 64].astype(np.float64)
            K = b["k"][h][bj * 64:(bj + 1) * 64].astype(np.float64)
            for gi in range(G):
                ref = Q[:, gi * 64:(gi + 1) * 64] @ K[:, gi * 64:(gi + 1) * 64].T  # exact: |S| < 2^21
                assert np.array_equal(S[t, gi].astype(np.float64), ref), (cfg, heads[h], qb, bj, gi)
        n_tiles += len(tiles)
        layer.close()
        for x in bufs:
            x.close()
    assert n_tiles >= 1024


PDUMP = {  # cfg: (heads in the layer, sampled (head index, q-block) targets)
    "c2": (list(range(8)), 6),
    "c3": (list(range(8)), 6),
    "c4": (list(range(4)), 6),
    "c5": (list(range(4)), 3),
}


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_p_codes_bit_exact(paro, ctx, oracle, cfg):
    """The final P codes K3 multiplies with V (after the exact boundary path), for every
    quantized tile of sampled q-blocks, equal the oracle's quant_affine of the
    reference's fp32(exp(fp64 logit - m)) code for code; the tile group's (lo, pscale)
    agree to fp32 rounding of the fast-path exponentials (<= 4e-6 relative)."""
    heads, nsample = PDUMP[cfg]
    g, N, d, vb, ords, q, k, v, layer, masks = layer_for(paro, ctx, cfg, heads, with_masks=True)
    kb = (N + 63) // 64
    rng = np.random.default_rng(11)
    targets = sorted({(int(rng.integers(0, len(heads))), int(rng.integers(0, kb))) for _ in range(nsample)}
                     | {(0, kb - 1)})
    bufs = [paro.DeviceBuffer.from_array(x) for x in (q, k, v)]
    layer.reorder_quantize(bufs[0].ptr, bufs[1].ptr, bufs[2].ptr, vb)
    codes, meta = layer.debug_pdump(np.array(targets, np.uint32), 0.0, vb)
    layer.close()
    for x in bufs:
        x.close()

    def check(ti):
        h, qb = targets[ti]
        plan = paro.make_perm(g, ords[h])
        qp, kp, vp = (np.ascontiguousarray(x[h][plan.inverse]) for x in (q, k, v))
        _, _, bj, lo, ps, oc = oracle.pdump(qp, kp, vp, qb, masks[h], vb)
        n = len(bj)
        qn = min(64, N - qb * 64)
        errs = []
        if not (np.all(meta[ti, :n, 3] == 1) and np.all(meta[ti, n:, 3] == 0)):
            errs.append("tile count")
        if not np.array_equal(meta[ti, :n, 2].astype(np.int64), bj.astype(np.int64)):
            errs.append("key blocks")
        lo_err = np.max(np.abs(meta[ti, :n, 0] - lo) / np.maximum(np.abs(lo), 1e-30)) if n else 0.0
        ps_err = np.max(np.abs(meta[ti, :n, 1] - ps) / ps) if n else 0.0
        flips = 0
        for t in range(n):
            kn = min(64, N - int(bj[t]) * 64)
            flips += int(np.count_nonzero(codes[ti, t, :qn, :kn] != oc[t, :qn, :kn]))
        return (h, qb, n, errs, flips, lo_err, ps_err)

    with ThreadPoolExecutor(8) as ex:
        res = list(ex.map(check, range(len(targets))))
    total_tiles = sum(r[2] for r in res)
    for h, qb, n, errs, flips, lo_err, ps_err in res:
        print(f"{cfg} head {heads[h]} q-block {qb}: {n} tiles, code flips {flips}, lo {lo_err:.1e}, pscale {ps_err:.1e}")
        assert not errs, (cfg, h, qb, errs)
        assert flips == 0, (cfg, h, qb, flips)
        assert lo_err <= 4e-6 and ps_err <= 4e-6, (cfg, h, qb, lo_err, ps_err)
    assert total_tiles > 0
