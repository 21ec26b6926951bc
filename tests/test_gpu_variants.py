"""The opt-in K3 layouts against the oracle: the same parity tests, run in a child
process whose environment selects the variant (the library reads the switch once
per process).

  PARO_K3_DEC=1  d=64 decoupled softmax / quantizer / epilogue kernel
                 (paro_b200/csrc/attention_dec_kernel.cu)
  PARO_K1_SPLIT  0 / 1: K1 fused (one CTA per q-block for Q, K and V) or split (one
                 CTA per tensor) regardless of the layer size, so both K1 kernels
                 meet the oracle at d=64 and d=128 (by default small d=128 layers
                 take the split kernel and everything else the fused one)
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_child(env_extra, args):
    env = dict(os.environ)
    env.update(env_extra)
    env.setdefault("PARO_WATCHDOG_S", "10")  # a pipeline bug traps instead of hanging the box
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider"] + args
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout[-3000:] + r.stderr[-2000:]
    print(out.strip().splitlines()[-1] if out.strip() else "(no output)")
    return r.returncode, out


def test_decoupled_kernel_layers_match_oracle():
    # d=64 layers of the parity suite (ragged tails, 2-D / 3-D grids, INT8 / INT4 P.V,
    # dense prefix, zeroed rows, edge shapes) and the 64 seeded fuzz layers
    rc, out = run_child({"PARO_K3_DEC": "1"},
                        ["tests/test_gpu_parity.py", "-k", "attention or dense or tiny or scale or rope",
                         "tests/test_gpu_fuzz.py"])
    assert rc == 0, out


def test_decoupled_kernel_pcodes_full_shape():
    # the final P codes of sampled q-blocks at the BASELINE shapes, code for code
    rc, out = run_child({"PARO_K3_DEC": "1"}, ["tests/test_gpu_fullshape_int.py", "tests/test_gpu_pcode_adversarial.py",
                                               "-k", "p_codes_bit_exact or p_codes_adversarial"])
    assert rc == 0, out


@pytest.mark.parametrize("split", ["0", "1"])
def test_k1_kernels_match_oracle(split):
    rc, out = run_child({"PARO_K1_SPLIT": split},
                        ["tests/test_gpu_parity.py", "-k", "reorder_quantize or attention_matches or rope_fused or tiny",
                         "tests/test_gpu_vpack.py"])
    assert rc == 0, out
