"""INT4 V nibble-packed in HBM (paro_layer_set_v_packing).

K1 stores two two's-complement codes per byte, low nibble first -- the PARQ
payload layout (quant.cpp:237-243) -- and K3 unpacks each tile to i8 in shared
memory for the kind::i8 P.V MMA. The packed bytes must be the oracle's codes
packed that way, and the layer output bit-identical to the one-code-per-byte
path (same codes, same arithmetic), at d = 64 (in-place unpack by the producer
warp) and d = 128 (staged unpack by two warps), with more items than CTAs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def pack_nibbles(codes):
    c = (np.asarray(codes, np.int32) & 15).astype(np.uint8)
    return (c[..., 0::2] | (c[..., 1::2] << 4)).astype(np.uint8)


CASES = [("F:13,H:30,W:45", 6, 64, 0.2), ("H:64,W:64", 24, 128, 0.3), ("F:5,H:9,W:14", 3, 128, 0.5),
         ("F:3,H:7,W:11", 4, 64, 0.4)]


@pytest.mark.parametrize("grid,H,d,density", CASES)
def test_packed_v_codes_and_layer_output(paro, ctx, oracle, grid, H, d, density):
    import bench

    g = paro.parse_grid(grid)
    N = g.token_count()
    orders, q, k, v, masks = bench.workload_ours(paro, ctx, list(range(H)), grid, N, d, density, "random")
    outs = {}
    for packed in (False, True):
        layer = paro.Layer(ctx, H, d, g, orders)
        layer.set_v_packing(packed)
        layer.set_masks(masks)
        out, zeroed = layer.forward_host(q, k, v, 0.0, 4)
        outs[packed] = (out, zeroed)
        if packed:
            b = layer.buffers()
            for h in range(H):
                plan = paro.make_perm(g, orders[h])
                vc, _, _ = oracle.quant_v(np.ascontiguousarray(v[h][plan.inverse]), 4)
                assert np.array_equal(b["v_packed"][h][:N], pack_nibbles(vc)), h
                assert np.array_equal(b["v"][h][:N].astype(np.int32), vc), h
        layer.close()
    assert np.array_equal(outs[True][0].view(np.uint32), outs[False][0].view(np.uint32))
    assert np.array_equal(outs[True][1], outs[False][1])


def test_packed_export_parq_matches_reference(paro, ctx, reference, tmp_path):
    g = paro.parse_grid("F:3,H:7,W:11")
    N = g.token_count()
    rng = np.random.default_rng(9)
    v = rng.standard_normal((2, N, 64)).astype(np.float32)
    layer = paro.Layer(ctx, 2, 64, g, ["FHW", "WHF"])
    layer.set_v_packing(True)
    bufs = [paro.DeviceBuffer.from_array(x) for x in (v, v, v)]
    layer.reorder_quantize(bufs[0].ptr, bufs[1].ptr, bufs[2].ptr, 4)
    paro.stream_sync()
    for h, order in enumerate(["FHW", "WHF"]):
        plan = paro.make_perm(g, order)
        blob = layer.export_parq(h, "v")
        ref = reference.save_quant_bytes(np.ascontiguousarray(v[h][plan.inverse]), 4, 1, 64, str(tmp_path))
        assert blob == ref
    layer.close()
