"""PAT1 / PARQ interchange: the product's in-memory
codecs against the reference's own writers and readers (tensor_io.cpp:45-137,
quant.cpp:219-326) -- byte-identical encodings, bit-exact decodes, and the same
error class and byte-offset message for every malformed-input case; on the GPU,
a layer's permuted Q/K/V codes exported as PARQ equal the reference's
save_quant_tensor(quantize(apply_perm_rows(X))) byte for byte."""
import numpy as np
import pytest

from conftest import randn


def strip_path(msg: str) -> str:
    return msg.split(": ", 1)[1] if msg.startswith("/") else msg


SHAPES = [(7,), (3, 5), (2, 3, 4), (1, 1, 1, 2)]


@pytest.mark.parametrize("shape", SHAPES)
def test_pat1_bytes_match_reference(paro, reference, tmp_path, shape):
    x = randn(11, shape).astype(np.float32)
    x.reshape(-1)[0] = -0.0
    if x.size > 3:
        x.reshape(-1)[1:4] = [np.inf, -np.inf, np.float32(1e-45)]
    ours = paro.encode_tensor(x)
    assert ours == reference.save_tensor_bytes(x, tmp_path)
    back = paro.decode_tensor(ours)
    assert back.shape == x.shape
    assert np.array_equal(back.view(np.uint32), x.view(np.uint32))


def _pat1(shape, payload_extra=0, **over):
    b = bytearray(b"PARO" + bytes([1, 0, len(shape), 0]))
    for e in shape:
        b += int(e).to_bytes(4, "little")
    n = int(np.prod(shape)) if shape else 0
    b += bytes(4 * n + payload_extra) if payload_extra >= -4 * n else b""
    for off, val in over.items():
        b[int(off[1:])] = val
    return bytes(b)


PAT1_BAD = {
    "short": b"PARO\x01",
    "magic": b"PARX" + _pat1((2,))[4:],
    "version": _pat1((2,), o4=2),
    "dtype": _pat1((2,), o5=1),
    "ndim0": _pat1((2,), o6=0),
    "reserved": _pat1((2,), o7=1),
    "extents": _pat1((2, 3))[:12],
    "zero_extent": _pat1((2, 0, 3)),
    "payload_short": _pat1((2, 3), payload_extra=-4),
    "payload_long": _pat1((2, 3), payload_extra=8),
}


@pytest.mark.parametrize("case", sorted(PAT1_BAD))
def test_pat1_malformed_matches_reference(paro, reference, tmp_path, case):
    data = PAT1_BAD[case]
    rc, msg = reference.load_tensor_error(data, tmp_path)
    assert rc == 3, (case, rc, msg)
    with pytest.raises(paro.FormatError) as e:
        paro.decode_tensor(data)
    assert str(e.value) == strip_path(msg)


def test_load_matrix_rules(paro):
    with pytest.raises(paro.FormatError):
        paro.load_matrix(paro.encode_tensor(np.zeros((2, 2, 2), np.float32)))
    bad = np.zeros((3, 4), np.float32)
    bad[1, 2] = np.nan
    with pytest.raises(paro.InvariantError, match="flat index 6"):
        paro.load_matrix(paro.encode_tensor(bad))
    ok = randn(3, (5, 4))
    assert np.array_equal(paro.load_matrix(paro.encode_tensor(ok)), ok)


QCASES = [(8, 1, 0, 64, (130, 96)), (4, 1, 0, 64, (65, 64)), (8, 0, 0, 16, (33, 40)), (4, 0, 1, 8, (9, 7)),
          (4, 1, 1, 64, (5, 3)), (8, 0, 1, 1, (4, 4))]


@pytest.mark.parametrize("bits,mode,grouping,block,shape", QCASES)
def test_parq_bytes_match_reference(paro, reference, tmp_path, bits, mode, grouping, block, shape):
    x = randn(bits + block + shape[0], shape) * 2
    if mode == 0:
        x = np.abs(x)
    rc, codes, scales, offs = reference.quantize(x, bits, mode, grouping, block)
    assert rc == 0
    q = paro.QuantBlockTensor(shape[0], shape[1], paro.QuantConfig(bits, mode, grouping, block), codes, scales, offs)
    ours = paro.encode_quant(q)
    assert ours == reference.save_quant_codes_bytes(bits, mode, grouping, block, codes, scales, offs, tmp_path)
    if grouping == 0:
        assert ours == reference.save_quant_bytes(x, bits, mode, block, tmp_path)
    d = paro.decode_quant(ours)
    assert (d.rows, d.cols, d.config.bits, d.config.mode, d.config.grouping, d.config.block) == (
        shape[0], shape[1], bits, mode, grouping, block)
    assert np.array_equal(d.codes, codes)
    assert np.array_equal(d.scales.view(np.uint32), np.asarray(scales, np.float32).view(np.uint32))
    if mode == 0:
        assert np.array_equal(d.offsets.view(np.uint32), np.asarray(offs, np.float32).view(np.uint32))


def _parq_sample(paro):
    x = np.abs(randn(5, (10, 6)))
    codes = np.clip(np.round(x * 20), 0, 255).astype(np.int32)
    q = paro.QuantBlockTensor(10, 6, paro.QuantConfig(8, 0, 0, 4), codes, np.full(6, 0.5, np.float32),
                              np.full(6, 0.25, np.float32))
    return paro.encode_quant(q)


def _mut(data, off, val):
    b = bytearray(data)
    b[off] = val
    return bytes(b)


@pytest.mark.parametrize("case", ["short", "magic", "version", "mode", "grouping", "bits", "block", "groups",
                                  "scales", "offsets", "codes", "trailing"])
def test_parq_malformed_matches_reference(paro, reference, tmp_path, case):
    good = _parq_sample(paro)
    data = {
        "short": good[:20],
        "magic": b"PARX" + good[4:],
        "version": _mut(good, 4, 2),
        "mode": _mut(good, 6, 2),
        "grouping": _mut(good, 7, 3),
        "bits": _mut(good, 5, 16),
        "block": good[:8] + (0).to_bytes(4, "little") + good[12:],
        "groups": _mut(good, 20, 7),
        "scales": good[:30],
        "offsets": good[:24 + 24 + 8],
        "codes": good[:-1],
        "trailing": good + b"\x00\x00",
    }[case]
    rc, msg = reference.load_quant_error(data, tmp_path)
    assert rc in (2, 3), (case, rc, msg)
    cls = paro.FormatError if rc == 3 else paro.ConfigError
    with pytest.raises(cls) as e:
        paro.decode_quant(data)
    assert str(e.value) == strip_path(msg)


@pytest.mark.gpu
@pytest.mark.parametrize("grid,H,d,orders,v_bits", [("F:3,H:7,W:11", 2, 64, ["WHF", "HFW"], 8),
                                                    ("F:3,H:7,W:11", 2, 64, ["FWH", "HWF"], 4),
                                                    ("H:20,W:33", 2, 128, ["WH", "HW"], 8)])
def test_layer_export_parq_matches_reference(paro, ctx, oracle, reference, tmp_path, grid, H, d, orders, v_bits):
    g = paro.parse_grid(grid)
    N = g.token_count()
    q, k, v = randn(1, (H, N, d)), randn(2, (H, N, d)), randn(3, (H, N, d))
    layer = paro.Layer(ctx, H, d, g, orders)
    dq, dk, dv = (paro.DeviceBuffer.from_array(x) for x in (q, k, v))
    layer.reorder_quantize(dq.ptr, dk.ptr, dv.ptr, v_bits)
    paro.stream_sync()
    for h in range(H):
        _, inv = oracle.make_perm(g.labels, g.extents, orders[h])
        for which, x, bits in (("q", q, 8), ("k", k, 8), ("v", v, v_bits)):
            if which == "v" and d != 64:
                with pytest.raises(paro.ConfigError):
                    layer.export_parq(h, which)
                continue
            ours = layer.export_parq(h, which)
            ref = reference.save_quant_bytes(x[h][inv], bits, 1, 64, tmp_path)
            assert ours == ref, (h, which)
    layer.close()
