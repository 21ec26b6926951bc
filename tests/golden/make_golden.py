#!/usr/bin/env python
"""Generate tests/golden/*.npz from the REFERENCE library itself.

Run in the container where /root/reference exists (it builds oracle/_ref/ from
the reference's own sources via oracle/Makefile). The fixtures are committed so
the GPU box (which has no /root/reference) can check against them.

    python tests/golden/make_golden.py

Fixtures (all values produced by the reference unless marked "oracle"):
  golden_c1.npz   BASELINE configs[0]: grid F:2,H:8,W:8, 2 heads, d=64, block 64.
                  Head inputs from gen_attention_inputs (head 0 aggregates along
                  F, head 1 along W; synth.cpp:136-184); per-head orders pinned
                  (HWF, WFH -- SURVEY finding 5); masks from gen_mask(U+2I, 0.3).
                  make_perm tables, Q/K codes+scales of the permuted inputs
                  (quantize {8, Symmetric, PerBlock, 64}), V codes/scales
                  (quantize {bits, Symmetric, PerBlock, 64} == the engine's V-tile
                  quantizer at d=64), the reference's fp-QK quantized output through
                  cmd_run's chain (permute -> quantized_blocked_attention -> inverse
                  permute) for P/V 8 and 4 bits, and (oracle) the restated INT8-QK
                  output, a regression value for the restatement.
  golden_rand.npz random-matrix fixtures (tests/oracles.hpp random_matrix) at N=520,
                  d in {64,128}: quantize + fp-QK engine outputs, and masks.
  golden_kat.npz  known-answer values: rounding KAT (test_kernels.cpp:100-117),
                  make_perm KAT (test_reorder.cpp:60-83), mask layout KAT
                  (test_mask.cpp:191-216), PSCH image + at(t) (mask.cpp:246-305).
"""
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Oracle, Reference  # noqa: E402


def chk(rc):
    if rc:
        raise RuntimeError(f"reference rc {rc}")


def main():
    import subprocess

    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle", "ref", "-j8"], check=True,
                   capture_output=True)
    ref = Reference()
    ref.select_kernels("scalar")
    orc = Oracle()

    # ---------------------------------------------------------------- c1
    grid, labels, ext = "F:2,H:8,W:8", "FHW", (2, 8, 8)
    n, d, H = 128, 64, 2
    weights = [(1.0, 0.0, 0.0), (0.0, 0.0, 1.0)]  # F-aggregation head, W-aggregation head
    orders = ["HWF", "WFH"]
    q = np.zeros((H, n, d), np.float32)
    k = np.zeros_like(q)
    v = np.zeros_like(q)
    for h in range(H):
        q[h], k[h], v[h] = ref.gen_attention_inputs(grid, weights[h], 1.0, 0.2, 11 + h, d, n)
    kb = 2
    masks = np.zeros((H, kb, kb), np.uint8)
    for h in range(H):
        st = ref.test_values(1234 + h, kb * kb).reshape(kb, kb).astype(np.float64) + 2.0 * np.eye(kb)
        rc, bits, rep = ref.gen_mask(st, 0.3, 64)
        chk(rc)
        masks[h] = bits
    out = {"grid": np.array(grid), "orders": np.array(orders), "q": q, "k": k, "v": v, "masks": masks}
    for h in range(H):
        rc, fwd, inv = ref.make_perm(labels, ext, orders[h])
        chk(rc)
        out[f"forward{h}"], out[f"inverse{h}"] = fwd, inv
        qp, kp, vp = (ref.apply_perm_rows(x[h], fwd, inv) for x in (q, k, v))
        for name, x in (("q", qp), ("k", kp)):
            rc, codes, scales, _ = ref.quantize(x, 8, 1, 0, 64)
            chk(rc)
            out[f"{name}codes{h}"], out[f"{name}scales{h}"] = codes.astype(np.int8), scales
        for bits in (8, 4):
            rc, codes, scales, _ = ref.quantize(vp, bits, 1, 0, 64)
            chk(rc)
            out[f"vcodes{bits}_{h}"], out[f"vscales{bits}_{h}"] = codes.astype(np.int8), scales
            rc, o_perm, zr = ref.quantized_blocked_attention(qp, kp, vp, masks[h], bits)
            chk(rc)
            out[f"ref_fpqk_out{bits}_{h}"] = o_perm[fwd]  # inverse permutation: O_orig[i] = O_perm[forward[i]]
            o_int8, _ = orc.paro_head(q[h], k[h], v[h], fwd, inv, masks[h], bits, qk_mode=1)
            out[f"oracle_int8qk_out{bits}_{h}"] = o_int8
    np.savez_compressed(os.path.join(HERE, "golden_c1.npz"), **out)

    # ---------------------------------------------------------------- random matrices
    rnd = {}
    for d in (64, 128):
        n = 520
        kb = (n + 63) // 64
        q, k, v = (ref.random_matrix(n, d, s, -1.0, 1.0) * 3.0 for s in (101, 102, 103))
        rnd[f"q{d}"], rnd[f"k{d}"], rnd[f"v{d}"] = q, k, v
        for bits in (8, 4):
            rc, codes, scales, _ = ref.quantize(q, bits, 1, 0, 64)
            chk(rc)
            rnd[f"qcodes{d}_{bits}"], rnd[f"qscales{d}_{bits}"] = codes.astype(np.int8), scales
        st = ref.test_values(77 + d, kb * kb).reshape(kb, kb).astype(np.float64) + 2.0 * np.eye(kb)
        rc, mask, _ = ref.gen_mask(st, 0.3, 64)
        chk(rc)
        rnd[f"mask{d}"] = mask
        for bits in (8, 4):
            rc, o, zr = ref.quantized_blocked_attention(q, k, v, mask, bits)
            chk(rc)
            rnd[f"ref_fpqk_out{d}_{bits}"] = o
        rc, o, _ = ref.masked_blocked_attention(q, k, v, mask)
        chk(rc)
        rnd[f"ref_masked_out{d}"] = o
    np.savez_compressed(os.path.join(HERE, "golden_rand.npz"), **rnd)

    # ---------------------------------------------------------------- KATs
    kat = {}
    xs = np.array([0.5, 1.5, 2.5, -0.5, -1.5, -2.5, 0.49999997, -0.49999997, 3.49, 3.51, -3.49, -3.51, 0.0, -0.0,
                   126.5, -126.5], np.float32)
    kat["round_x"] = xs
    kat["round_codes"] = np.array([int(np.sign(x) * np.floor(abs(float(x)) + 0.5)) for x in xs], np.int32)
    rc, fwd, inv = ref.make_perm("FHW", (2, 2, 2), "HWF")
    chk(rc)
    kat["perm_f2h2w2_hwf_forward"], kat["perm_f2h2w2_hwf_inverse"] = fwd, inv
    rc, lab, ext = ref.parse_grid("F:13,H:30,W:45")
    kat["grid_c2_extents"] = np.array(ext, np.uint32)
    one = np.zeros((1, 9), np.uint8)
    one[0, [0, 3, 8]] = 1
    kat["pmsk_one_1x9_b4"] = np.frombuffer(ref.serialize_mask(one, 4), np.uint8)
    big = np.ones((275, 275), np.uint8)
    kat["pmsk_all_275_len"] = np.array(len(ref.serialize_mask(big, 64)))
    rng_sums = np.stack([ref.test_values(30 + t, 49).reshape(7, 7).astype(np.float64) + 2.0 * np.eye(7)
                         for t in range(5)])
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "s.psch")
        ref.build_and_save_schedule(rng_sums, 0.4, 16, path)
        kat["psch_image"] = np.fromfile(path, np.uint8)
        kat["psch_at"] = np.stack([ref.schedule_at(path, t)[1] for t in range(5)])
    kat["gen_mask_sums"] = rng_sums[0]
    kat["gen_mask_bits"] = ref.gen_mask(rng_sums[0], 0.4, 16)[1]
    np.savez_compressed(os.path.join(HERE, "golden_kat.npz"), **kat)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
