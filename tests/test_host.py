"""CPU tests of the product library (no GPU needed): the C-ABI .so loads and
exports every symbol include/paro_b200.h declares; the host-side integer stages
(grid, make_perm, enumerate, PMSK/PSCH, synthetic generator) are
bit-exact with the reference (golden fixtures and, where built, the live
reference library); errors map to the reference's exception classes."""
import ctypes
import os
import re

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = os.path.join(HERE, "golden")


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "paro_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(paro_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(paro):
    lib = ctypes.CDLL(paro.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_only(paro):
    """The fatbin carries sm_100a SASS (no PTX for JIT to other archs, no CPU fallback)."""
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", paro.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", paro.LIB_PATH], capture_output=True, text=True).stdout
    for mnemonic in ("UTCIMMA", "UTMALDG", "LDTM"):
        assert mnemonic in sass, mnemonic


def test_device_calls_fail_loudly_without_gpu(paro):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(paro.CudaError):
        paro.Context(0)


# ------------------------------------------------------------------ grid / perm
def test_parse_grid(paro, kat):
    g = paro.parse_grid("F:13,H:30,W:45")
    assert g.token_count() == 17550 and g.labels == "FHW"
    assert tuple(kat["grid_c2_extents"]) == g.extents
    assert paro.parse_grid("H:64,W:64").label_string() == "HW"
    for bad in ("F=13", "F:abc", "F:4,F:4,W:4", "F:4,W:4", "X:4,W:4", "H:0,W:4", "H:4", ""):
        with pytest.raises(paro.ConfigError):
            paro.parse_grid(bad)


def test_make_perm_kat_and_errors(paro, kat):
    small = paro.parse_grid("F:2,H:2,W:2")
    plan = paro.make_perm(small, "HWF")
    assert plan.forward[4] == 1  # test_reorder.cpp:60-83
    assert np.array_equal(plan.forward, kat["perm_f2h2w2_hwf_forward"])
    assert np.array_equal(plan.inverse, kat["perm_f2h2w2_hwf_inverse"])
    cube = paro.parse_grid("F:4,H:4,W:4")
    assert paro.make_perm(cube, "FHW").is_identity()
    with pytest.raises(paro.ConfigError):
        paro.make_perm(cube, "FH")
    with pytest.raises(paro.InputError):
        paro.make_perm(cube, "FHX")
    back = plan.inverted()
    assert np.array_equal(back.forward, plan.inverse)


def test_enumerate_orders(paro):
    cube = paro.parse_grid("F:4,H:4,W:4")
    assert paro.enumerate_orders(cube) == ["FHW", "FWH", "HFW", "HWF", "WFH", "WHF"]  # test_reorder.cpp:30-58
    assert paro.enumerate_orders(paro.parse_grid("H:2,W:3,F:4"))[:2] == ["HWF", "FHW"]
    assert len(paro.enumerate_orders(paro.parse_grid("H:3,W:5"))) == 2


def test_perm_matches_golden_c1(paro, c1):
    g = paro.parse_grid(str(c1["grid"]))
    for h, order in enumerate(c1["orders"]):
        plan = paro.make_perm(g, str(order))
        assert np.array_equal(plan.forward, c1[f"forward{h}"])
        assert np.array_equal(plan.inverse, c1[f"inverse{h}"])


@pytest.mark.parametrize("text", ["F:13,H:30,W:45", "F:21,H:45,W:80", "H:64,W:64", "W:7,H:3", "H:5,F:3,W:2"])
def test_perm_vs_reference(paro, reference, text):
    g = paro.parse_grid(text)
    for order in paro.enumerate_orders(g):
        plan = paro.make_perm(g, order)
        rc, f, i = reference.make_perm(g.labels, g.extents, order)
        assert rc == 0 and np.array_equal(plan.forward, f) and np.array_equal(plan.inverse, i)


# ------------------------------------------------------------------ masks
def test_mask_layout_kat(paro, kat):
    one = paro.BlockMask(1, 9, 4)
    for j in (0, 3, 8):
        one.set(0, j, True)
    blob = paro.serialize_mask(one)
    assert np.array_equal(np.frombuffer(blob, np.uint8), kat["pmsk_one_1x9_b4"])
    assert len(paro.serialize_mask(paro.BlockMask(275, 275, 64, np.ones((275, 275), np.uint8)))) == 18 + 275 * 35


@pytest.mark.parametrize("kr,kc", [(33, 17), (1, 1), (8, 8), (275, 275), (1024, 7), (3, 1024)])
def test_mask_roundtrip(paro, kr, kc):
    rng = np.random.default_rng(kr * 31 + kc)
    m = paro.BlockMask(kr, kc, 64, (rng.random((kr, kc)) < 0.4).astype(np.uint8))
    blob = paro.serialize_mask(m)
    back, used = paro.deserialize_mask(blob)
    assert used == len(blob) and back.k_rows == kr and back.k_cols == kc and back.block == 64
    assert np.array_equal(back.bits, m.bits)


def test_mask_format_errors(paro):
    blob = bytearray(paro.serialize_mask(paro.BlockMask(5, 5, 64, np.eye(5, dtype=np.uint8))))
    bad = bytearray(blob)
    bad[0] = ord("X")
    with pytest.raises(paro.FormatError, match="bad mask magic"):
        paro.deserialize_mask(bytes(bad))
    with pytest.raises(paro.FormatError):
        paro.deserialize_mask(bytes(blob[:10]))
    with pytest.raises(paro.FormatError):
        paro.deserialize_mask(bytes(blob[:-1]))


def test_mask_serialize_vs_reference(paro, reference):
    rng = np.random.default_rng(3)
    for kr, kc in [(33, 17), (275, 275), (64, 64)]:
        bits = (rng.random((kr, kc)) < 0.3).astype(np.uint8)
        assert paro.serialize_mask(paro.BlockMask(kr, kc, 64, bits)) == reference.serialize_mask(bits, 64)


def test_schedule_at_matches_golden(paro, kat):
    img = kat["psch_image"].tobytes()
    for t in range(5):
        assert np.array_equal(paro.schedule_at(img, t).bits, kat["psch_at"][t])
    with pytest.raises(paro.InputError):
        paro.schedule_at(img, 5)
    with pytest.raises(paro.FormatError):
        paro.schedule_at(img + b"xx", 0)
    with pytest.raises(paro.FormatError):
        paro.schedule_at(b"PSCHxxxx", 0)


def test_schedule_at_is_positional(paro):
    """MaskSchedule::at(t) returns distinct[t] by position and ignores the stored
    timestep field (mask.cpp:132-140, load_schedule mask.cpp:282-292): an image
    whose stored fields are permuted / duplicated selects the same masks."""
    import struct

    rng = np.random.default_rng(11)
    T = 7
    masks = [(rng.random((5, 5)) < 0.5).astype(np.uint8) for _ in range(T // 2 + 1)]
    blobs = [paro.serialize_mask(paro.BlockMask(5, 5, 64, m)) for m in masks]
    stored = [2, 2, 0]  # non-canonical: duplicated and out of order
    img = b"PSCH" + struct.pack("<II", T, T // 2)
    for s, b in zip(stored, blobs[:-1]):
        img += struct.pack("<I", s) + b
    img += blobs[-1]
    for t in range(T):
        want = masks[t] if t < T // 2 else masks[-1]
        assert np.array_equal(paro.schedule_at(img, t).bits, want), t


# ------------------------------------------------------------------ synthetic inputs
def test_synth_randn_matches_reference_generator(paro, reference):
    """gen_attention_inputs' V is the documented MT19937-64 Box-Muller stream
    seeded with seed ^ 0x9e3779b97f4a7c15 (synth.cpp:173-182)."""
    seed = 11
    _, _, v = reference.gen_attention_inputs("F:2,H:8,W:8", [1.0, 0.0, 0.0], 1.0, 0.2, seed, 64, 128)
    got = paro.synth_randn(seed ^ 0x9E3779B97F4A7C15, 128 * 64).reshape(128, 64)
    assert np.array_equal(got.view(np.uint32), v.view(np.uint32))


def test_quant_config_validation(paro):
    with pytest.raises(paro.ConfigError):
        paro.QuantConfig(5).validate()
    with pytest.raises(paro.ConfigError):
        paro.QuantConfig(8, block=0).validate()
    assert paro.QuantConfig(8, paro.UNSIGNED).qmax() == 255
    assert paro.QuantConfig(4, paro.SYMMETRIC).qmin() == -7


def test_attn_inputs_validation(paro):
    a = np.zeros((4, 4), np.float32)
    with pytest.raises(paro.ShapeError):
        paro.AttnInputs(a, a, np.zeros((5, 4), np.float32)).validate()
    with pytest.raises(paro.ConfigError):
        paro.AttnInputs(a, a, a, 0.0, 5).validate()
