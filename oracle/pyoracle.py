"""pyoracle -- ctypes bindings to the ORACLE libraries (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference legs
may import this module, and only as the checker / the timed CPU baseline --
never as a product path.

  oracle/_build/libparo_oracle.so  C restatement (oracle/paro_oracle.c)
  oracle/_ref/libparo_ref.so       the reference library built from its own
                                   sources (oracle/Makefile `ref`), if present
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libparo_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libparo_ref.so")

P = ctypes.c_void_p
SZ = ctypes.c_size_t
U32 = ctypes.c_uint32


def _ptr(a):
    assert a.flags["C_CONTIGUOUS"]
    return P(a.ctypes.data)


def build_oracle() -> None:
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)


class Oracle:
    """The C restatement of the reference hot path."""

    def __init__(self):
        build_oracle()
        self.lib = ctypes.CDLL(ORACLE_SO)

    def make_perm(self, labels: str, extents, order: str):
        n = int(np.prod(extents))
        fwd = np.empty(n, np.uint32)
        inv = np.empty(n, np.uint32)
        ext = (U32 * 3)(*list(extents) + [0] * (3 - len(extents)))
        rc = self.lib.oracle_make_perm(ctypes.c_int(len(labels)), labels.encode(), ext, order.encode(), _ptr(fwd),
                                       _ptr(inv))
        if rc:
            raise ValueError(f"oracle_make_perm rc={rc}")
        return fwd, inv

    def quantize(self, m, bits, mode, block):
        m = np.ascontiguousarray(m, np.float32)
        rows, cols = m.shape
        ng = ((rows + block - 1) // block) * ((cols + block - 1) // block)
        codes = np.empty((rows, cols), np.int32)
        scales = np.empty(ng, np.float32)
        offs = np.empty(ng, np.float32)
        rc = self.lib.oracle_quantize(_ptr(m), SZ(rows), SZ(cols), ctypes.c_int(bits), ctypes.c_int(mode), SZ(block),
                                      _ptr(codes), _ptr(scales), _ptr(offs))
        if rc:
            raise ValueError(f"oracle_quantize rc={rc}")
        return codes, scales, (offs if mode == 0 else None)

    def quant_v(self, v, bits, block=64):
        v = np.ascontiguousarray(v, np.float32)
        n, d = v.shape
        kb = (n + block - 1) // block
        codes = np.empty((n, d), np.int32)
        scales = np.empty(kb, np.float32)
        colsum = np.empty((kb, d), np.int64)
        self.lib.oracle_quant_v(_ptr(v), SZ(n), SZ(d), SZ(block), ctypes.c_int(bits), _ptr(codes), _ptr(scales),
                                _ptr(colsum))
        return codes, scales, colsum

    def quant_affine(self, x, offset, scale, qmin, qmax):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty(x.shape, np.int32)
        self.lib.oracle_quant_affine(_ptr(x), SZ(x.size), ctypes.c_float(offset), ctypes.c_float(scale),
                                     ctypes.c_int32(qmin), ctypes.c_int32(qmax), _ptr(out))
        return out

    def stream_engine(self, q, k, v, mask=None, pv_bits=8, qk_mode=1, scale=0.0, dense_prefix=0, block=64):
        """attention.cpp:84-254 restated. qk_mode 1 = INT8-QK, 0 = reference fp64 QK.
        pv_bits 0 = unquantized masked stream. Returns (out, zeroed bool[n])."""
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        zeroed = np.empty(n, np.uint8)
        mp = None
        if mask is not None:
            mask = np.ascontiguousarray(mask, np.uint8)
            mp = _ptr(mask)
        rc = self.lib.oracle_stream_engine(_ptr(q), _ptr(k), _ptr(v), SZ(n), SZ(d), ctypes.c_float(scale),
                                           SZ(dense_prefix), SZ(block), mp, ctypes.c_int(pv_bits),
                                           ctypes.c_int(qk_mode), _ptr(out), _ptr(zeroed))
        if rc:
            raise ValueError(f"oracle_stream_engine rc={rc}")
        return out, zeroed.astype(bool)

    def stream_engine_range(self, q, k, v, qb_begin, qb_end, mask=None, pv_bits=8, qk_mode=1, scale=0.0):
        """Engine output rows of q-blocks [qb_begin, qb_end) only (rows [qb_begin*64, ...))."""
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        n, d = q.shape
        out = np.zeros((n, d), np.float32)
        zeroed = np.zeros(n, np.uint8)
        mp = None
        if mask is not None:
            mask = np.ascontiguousarray(mask, np.uint8)
            mp = _ptr(mask)
        rc = self.lib.oracle_stream_engine_range(_ptr(q), _ptr(k), _ptr(v), SZ(n), SZ(d), ctypes.c_float(scale), SZ(0),
                                                 SZ(64), mp, ctypes.c_int(pv_bits), ctypes.c_int(qk_mode),
                                                 SZ(qb_begin), SZ(qb_end), _ptr(out), _ptr(zeroed))
        if rc:
            raise ValueError(f"oracle_stream_engine_range rc={rc}")
        r0, r1 = qb_begin * 64, min(n, qb_end * 64)
        return out[r0:r1], zeroed[r0:r1].astype(bool)

    def pdump(self, q, k, v, qb, mask=None, pv_bits=8, scale=0.0):
        """q-block qb of the INT8-QK engine with its P-code dump: (out rows, zeroed,
        bj[t], lo[t], pscale[t], codes[t][64][64]) for its quantized tiles in order."""
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        n, d = q.shape
        kb = (n + 63) // 64
        out = np.zeros((n, d), np.float32)
        zeroed = np.zeros(n, np.uint8)
        codes = np.zeros((kb, 64, 64), np.uint8)
        lo = np.zeros(kb, np.float32)
        ps = np.zeros(kb, np.float32)
        bj = np.zeros(kb, np.int32)
        nt = SZ()
        mp = None
        if mask is not None:
            mask = np.ascontiguousarray(mask, np.uint8)
            mp = _ptr(mask)
        rc = self.lib.oracle_stream_engine_pdump(_ptr(q), _ptr(k), _ptr(v), SZ(n), SZ(d), ctypes.c_float(scale),
                                                 SZ(64), mp, ctypes.c_int(pv_bits), SZ(qb), SZ(kb), _ptr(codes),
                                                 _ptr(lo), _ptr(ps), _ptr(bj), ctypes.byref(nt), _ptr(out),
                                                 _ptr(zeroed))
        if rc:
            raise ValueError(f"oracle_stream_engine_pdump rc={rc}")
        t = nt.value
        r0, r1 = qb * 64, min(n, qb * 64 + 64)
        return out[r0:r1], zeroed[r0:r1].astype(bool), bj[:t], lo[:t], ps[:t], codes[:t]

    def paro_head(self, q, k, v, fwd, inv, mask=None, pv_bits=8, qk_mode=1, scale=0.0):
        """cmd_run's chain for one head (main.cpp:276-305). zeroed in PERMUTED order."""
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        zeroed = np.empty(n, np.uint8)
        mp = None
        if mask is not None:
            mask = np.ascontiguousarray(mask, np.uint8)
            mp = _ptr(mask)
        fwd = np.ascontiguousarray(fwd, np.uint32)
        inv = np.ascontiguousarray(inv, np.uint32)
        rc = self.lib.oracle_paro_head(_ptr(q), _ptr(k), _ptr(v), SZ(n), SZ(d), ctypes.c_float(scale), _ptr(fwd),
                                       _ptr(inv), mp, ctypes.c_int(pv_bits), ctypes.c_int(qk_mode), _ptr(out),
                                       _ptr(zeroed))
        if rc:
            raise ValueError(f"oracle_paro_head rc={rc}")
        return out, zeroed.astype(bool)

    def serialize_mask(self, bits, block):
        bits = np.ascontiguousarray(bits, np.uint8)
        kr, kc = bits.shape
        self.lib.oracle_pmsk_size.restype = SZ
        size = self.lib.oracle_pmsk_size(SZ(kr), SZ(kc))
        out = np.empty(size, np.uint8)
        self.lib.oracle_serialize_mask(_ptr(bits), SZ(kr), SZ(kc), SZ(block), _ptr(out))
        return out.tobytes()

    def deserialize_mask(self, data: bytes):
        buf = np.frombuffer(data, np.uint8).copy()
        kr, kc, b = U32(), U32(), U32()
        used = SZ()
        rc = self.lib.oracle_deserialize_mask(_ptr(buf), SZ(len(data)), ctypes.byref(kr), ctypes.byref(kc),
                                              ctypes.byref(b), None, ctypes.byref(used))
        if rc:
            raise ValueError("format")
        bits = np.empty((kr.value, kc.value), np.uint8)
        self.lib.oracle_deserialize_mask(_ptr(buf), SZ(len(data)), ctypes.byref(kr), ctypes.byref(kc),
                                         ctypes.byref(b), _ptr(bits), ctypes.byref(used))
        return bits, b.value, used.value


def have_reference() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The reference library itself (oracle/_ref/libparo_ref.so)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.lib = ctypes.CDLL(REF_SO)
        self.lib.ref_last_error.restype = ctypes.c_char_p
        self.lib.ref_active_kernels.restype = ctypes.c_char_p

    def _chk(self, rc):
        if rc:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def select_kernels(self, impl: str):
        self._chk(self.lib.ref_select_kernels(impl.encode()))

    def active_kernels(self) -> str:
        return self.lib.ref_active_kernels().decode()

    def make_perm(self, labels, extents, order):
        n = int(np.prod(extents))
        fwd = np.empty(n, np.uint32)
        inv = np.empty(n, np.uint32)
        ext = (U32 * 3)(*list(extents) + [0] * (3 - len(extents)))
        rc = self.lib.ref_make_perm(ctypes.c_int(len(labels)), labels.encode(), ext, order.encode(), _ptr(fwd),
                                    _ptr(inv))
        return rc, fwd, inv

    def enumerate_orders(self, labels, extents):
        buf = ctypes.create_string_buffer(32)
        cnt = ctypes.c_int()
        ext = (U32 * 3)(*list(extents) + [0] * (3 - len(extents)))
        self._chk(self.lib.ref_enumerate_perms(ctypes.c_int(len(labels)), labels.encode(), ext, buf, ctypes.byref(cnt)))
        nd = len(labels)
        raw = buf.raw[: cnt.value * nd].decode()
        return [raw[i * nd : (i + 1) * nd] for i in range(cnt.value)]

    def parse_grid(self, text):
        nd = ctypes.c_int()
        lab = ctypes.create_string_buffer(4)
        ext = (U32 * 3)()
        rc = self.lib.ref_parse_grid(text.encode(), ctypes.byref(nd), lab, ext)
        if rc:
            return rc, None, None
        return 0, lab.raw[: nd.value].decode(), tuple(int(ext[i]) for i in range(nd.value))

    def apply_perm_rows(self, m, fwd, inv):
        m = np.ascontiguousarray(m, np.float32)
        out = np.empty_like(m)
        self._chk(self.lib.ref_apply_perm_rows(_ptr(m), SZ(m.shape[0]), SZ(m.shape[1]), _ptr(fwd), _ptr(inv),
                                               SZ(len(fwd)), _ptr(out)))
        return out

    def save_tensor_bytes(self, values, tmpdir):
        """save_tensor (tensor_io.cpp:45-71) -> the file's bytes."""
        v = np.ascontiguousarray(values, np.float32)
        shape = np.asarray(v.shape, np.uint32)
        path = os.path.join(str(tmpdir), "t.pat")
        self._chk(self.lib.ref_save_tensor(_ptr(shape), SZ(v.ndim), _ptr(v), path.encode()))
        with open(path, "rb") as f:
            return f.read()

    def load_tensor_error(self, data: bytes, tmpdir):
        """load_tensor on raw bytes -> (exit code, message) (0, '' when it loads)."""
        path = os.path.join(str(tmpdir), "l.pat")
        with open(path, "wb") as f:
            f.write(data)
        nd = U32()
        shape = np.zeros(256, np.uint32)
        rc = self.lib.ref_load_tensor(path.encode(), ctypes.byref(nd), _ptr(shape), None)
        return rc, (self.lib.ref_last_error().decode() if rc else "")

    def save_quant_bytes(self, m, bits, mode, block, tmpdir):
        """save_quant_tensor(quantize(m, {bits, mode, PerBlock, block})) -> the file's bytes."""
        m = np.ascontiguousarray(m, np.float32)
        path = os.path.join(str(tmpdir), "q.parq")
        self._chk(self.lib.ref_save_quant_tensor(_ptr(m), SZ(m.shape[0]), SZ(m.shape[1]), ctypes.c_uint(bits),
                                                 ctypes.c_int(mode), SZ(block), path.encode()))
        with open(path, "rb") as f:
            return f.read()

    def save_quant_codes_bytes(self, bits, mode, grouping, block, codes, scales, offsets, tmpdir):
        codes = np.ascontiguousarray(codes, np.int32)
        scales = np.ascontiguousarray(scales, np.float32)
        offsets = np.ascontiguousarray(offsets if offsets is not None and len(offsets) else np.zeros(1), np.float32)
        path = os.path.join(str(tmpdir), "c.parq")
        self._chk(self.lib.ref_save_quant_codes(ctypes.c_uint(bits), ctypes.c_int(mode), ctypes.c_int(grouping),
                                                SZ(block), SZ(codes.shape[0]), SZ(codes.shape[1]), _ptr(codes),
                                                _ptr(scales), _ptr(offsets), path.encode()))
        with open(path, "rb") as f:
            return f.read()

    def load_quant_error(self, data: bytes, tmpdir):
        path = os.path.join(str(tmpdir), "l.parq")
        with open(path, "wb") as f:
            f.write(data)
        bits, mode = ctypes.c_uint(), ctypes.c_int()
        rows, cols, ng = SZ(), SZ(), SZ()
        rc = self.lib.ref_load_quant_tensor(path.encode(), ctypes.byref(bits), ctypes.byref(mode), ctypes.byref(rows),
                                            ctypes.byref(cols), None, None, ctypes.byref(ng))
        return rc, (self.lib.ref_last_error().decode() if rc else "")

    def quantize(self, m, bits, mode, grouping, block):
        m = np.ascontiguousarray(m, np.float32)
        rows, cols = m.shape
        codes = np.empty((rows, cols), np.int32)
        ng_max = rows * cols + rows + cols
        scales = np.empty(ng_max, np.float32)
        offs = np.empty(ng_max, np.float32)
        ng = SZ()
        rc = self.lib.ref_quantize(_ptr(m), SZ(rows), SZ(cols), ctypes.c_uint(bits), ctypes.c_int(mode),
                                   ctypes.c_int(grouping), SZ(block), _ptr(codes), _ptr(scales), _ptr(offs),
                                   ctypes.byref(ng))
        if rc:
            return rc, None, None, None
        return 0, codes, scales[: ng.value].copy(), (offs[: ng.value].copy() if mode == 0 else None)

    def _engine(self, fn, q, k, v, mask, block, bits, scale=0.0, dense_prefix=0):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        zer = np.empty(n, np.uint32)
        nz = SZ()
        args = [_ptr(q), _ptr(k), _ptr(v), SZ(n), SZ(d), ctypes.c_float(scale), SZ(dense_prefix)]
        if fn == "stream":
            rc = self.lib.ref_blocked_attention_stream(*args, SZ(block), _ptr(out), _ptr(zer), ctypes.byref(nz))
        else:
            mp, mk = None, SZ(0)
            if mask is not None:
                mask = np.ascontiguousarray(mask, np.uint8)
                mp, mk = _ptr(mask), SZ(mask.shape[0])
            if fn == "masked":
                rc = self.lib.ref_masked_blocked_attention(*args, mp, mk, SZ(block), _ptr(out), _ptr(zer),
                                                           ctypes.byref(nz))
            else:
                rc = self.lib.ref_quantized_blocked_attention(*args, mp, mk, SZ(block), ctypes.c_uint(bits),
                                                              _ptr(out), _ptr(zer), ctypes.byref(nz))
        if rc:
            return rc, None, None
        return 0, out, zer[: nz.value].copy()

    def quantized_blocked_attention(self, q, k, v, mask=None, bits=8, block=64, scale=0.0, dense_prefix=0):
        return self._engine("quant", q, k, v, mask, block, bits, scale, dense_prefix)

    def masked_blocked_attention(self, q, k, v, mask, block=64, scale=0.0, dense_prefix=0):
        return self._engine("masked", q, k, v, mask, block, 8, scale, dense_prefix)

    def blocked_attention_stream(self, q, k, v, block=64, scale=0.0, dense_prefix=0):
        return self._engine("stream", q, k, v, None, block, 8, scale, dense_prefix)

    def gen_mask(self, sums, density, block, guard=0):
        s = np.ascontiguousarray(sums, np.float64)
        kr, kc = s.shape
        bits = np.empty((kr, kc), np.uint8)
        rep = SZ()
        rc = self.lib.ref_gen_mask(_ptr(s), SZ(kr), SZ(kc), ctypes.c_double(density), SZ(block), SZ(guard), _ptr(bits),
                                   ctypes.byref(rep))
        if rc:
            return rc, None, None
        return 0, bits, rep.value

    def perm_block_sums(self, m, block, forward=None, inverse=None):
        """block_sums(AttnMap(apply_perm_map(m, plan), block, relaxed)) of the reference."""
        m = np.ascontiguousarray(m, np.float32)
        n = m.shape[0]
        k = (n + block - 1) // block
        out = np.empty((k, k), np.float64)
        f = None if forward is None else np.ascontiguousarray(forward, np.uint32)
        i = None if inverse is None else np.ascontiguousarray(inverse, np.uint32)
        self._chk(self.lib.ref_perm_block_sums(_ptr(m), SZ(n), _ptr(f) if f is not None else None,
                                               _ptr(i) if i is not None else None, SZ(block), _ptr(out)))
        return out

    def select_permutation(self, maps, grid_text, block=64, eps=1e-3, sigma=0.9, alpha=0.5, dense_prefix=0):
        m = np.ascontiguousarray(maps, np.float32)
        count, n, _ = m.shape
        orders = ctypes.create_string_buffer(32)
        scores = np.zeros((6, 5), np.float64)
        nperm, chosen = ctypes.c_int(), ctypes.c_int()
        self._chk(self.lib.ref_select_permutation(_ptr(m), SZ(count), SZ(n), grid_text.encode(), SZ(block),
                                                  ctypes.c_float(eps), ctypes.c_float(sigma), ctypes.c_float(alpha),
                                                  SZ(dense_prefix), orders, _ptr(scores), ctypes.byref(nperm),
                                                  ctypes.byref(chosen)))
        nd = len(orders.raw.rstrip(b"\0")) // nperm.value
        ords = [orders.raw[i * nd:(i + 1) * nd].decode() for i in range(nperm.value)]
        return ords, scores[:nperm.value], chosen.value

    def serialize_mask(self, bits, block):
        bits = np.ascontiguousarray(bits, np.uint8)
        kr, kc = bits.shape
        size = SZ()
        self._chk(self.lib.ref_serialize_mask(_ptr(bits), SZ(kr), SZ(kc), SZ(block), None, ctypes.byref(size)))
        out = np.empty(size.value, np.uint8)
        self._chk(self.lib.ref_serialize_mask(_ptr(bits), SZ(kr), SZ(kc), SZ(block), _ptr(out), ctypes.byref(size)))
        return out.tobytes()

    def deserialize_mask(self, data: bytes):
        buf = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        kr, kc, b = U32(), U32(), U32()
        used = SZ()
        rc = self.lib.ref_deserialize_mask(_ptr(buf), SZ(len(data)), ctypes.byref(kr), ctypes.byref(kc),
                                           ctypes.byref(b), None, ctypes.byref(used))
        if rc:
            return rc, None, None, None
        bits = np.empty((kr.value, kc.value), np.uint8)
        self.lib.ref_deserialize_mask(_ptr(buf), SZ(len(data)), ctypes.byref(kr), ctypes.byref(kc), ctypes.byref(b),
                                      _ptr(bits), ctypes.byref(used))
        return 0, bits, b.value, used.value

    def build_and_save_schedule(self, sums_t, density, block, path):
        s = np.ascontiguousarray(sums_t, np.float64)
        T, kr, kc = s.shape
        self._chk(self.lib.ref_build_and_save_schedule(_ptr(s), SZ(T), SZ(kr), SZ(kc), ctypes.c_double(density),
                                                       SZ(block), path.encode()))

    def schedule_at(self, path, t):
        kr = U32()
        rc = self.lib.ref_schedule_at(path.encode(), U32(t), None, ctypes.byref(kr))
        if rc:
            return rc, None
        bits = np.empty((kr.value, kr.value), np.uint8)  # square schedules only
        self.lib.ref_schedule_at(path.encode(), U32(t), _ptr(bits), ctypes.byref(kr))
        return 0, bits

    def random_matrix(self, rows, cols, seed, lo=-1.0, hi=1.0):
        out = np.empty((rows, cols), np.float32)
        self.lib.ref_random_matrix(SZ(rows), SZ(cols), ctypes.c_uint64(seed), ctypes.c_float(lo), ctypes.c_float(hi),
                                   _ptr(out))
        return out

    def load_plan_file(self, path):
        """(rc, [(head, order)], error message) of the reference's load_plan_file."""
        cnt = U32()
        rc = self.lib.ref_load_plan_file(path.encode(), ctypes.byref(cnt), None, None)
        if rc:
            return rc, None, self.lib.ref_last_error().decode()
        heads = np.empty(max(1, cnt.value), np.uint32)
        orders = ctypes.create_string_buffer(8 * max(1, cnt.value))
        self.lib.ref_load_plan_file(path.encode(), ctypes.byref(cnt), _ptr(heads), orders)
        return 0, [(int(heads[i]), orders.raw[8 * i:8 * i + 8].rstrip(b"\0").decode()) for i in range(cnt.value)], ""

    def plan_for_head(self, path, grid_text, head, n):
        """(rc, inverse permutation, error message) of tools/main.cpp plan_for_head."""
        inv = np.empty(n, np.uint32)
        rc = self.lib.ref_plan_for_head(path.encode() if path else None, grid_text.encode(), U32(head), _ptr(inv))
        return rc, (inv if rc == 0 else None), (self.lib.ref_last_error().decode() if rc else "")

    def synth_randn_streams(self, seed0, stride, nstreams, count, threads=0):
        """[nstreams, count] N(0,1) values, stream s seeded seed0 + stride*s (synth.cpp:20-22, 173-182)."""
        out = np.empty((nstreams, count), np.float32)
        self.lib.ref_synth_randn_streams(ctypes.c_uint64(seed0), ctypes.c_uint64(stride), SZ(nstreams), SZ(count),
                                         ctypes.c_int(threads or os.cpu_count() or 1), _ptr(out))
        return out

    def test_values(self, state, count):
        out = np.empty(count, np.float32)
        self.lib.ref_test_values(ctypes.c_uint64(state), SZ(count), _ptr(out))
        return out

    def gen_attention_inputs(self, grid_text, weights, bandwidth, noise, seed, head_dim, n):
        q = np.empty((n, head_dim), np.float32)
        k = np.empty((n, head_dim), np.float32)
        v = np.empty((n, head_dim), np.float32)
        w = np.ascontiguousarray(weights, np.float32)
        self._chk(self.lib.ref_gen_attention_inputs(grid_text.encode(), _ptr(w), ctypes.c_float(bandwidth),
                                                    ctypes.c_float(noise), ctypes.c_uint64(seed), SZ(head_dim),
                                                    _ptr(q), _ptr(k), _ptr(v)))
        return q, k, v

    def run_heads(self, grid_text, q, k, v, orders, masks, bits, scale=0.0, threads=1):
        """cmd_run's hot chain per head on `threads` host threads; returns (out, seconds)."""
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        H, n, d = q.shape
        out = np.empty_like(q)
        secs = ctypes.c_double()
        mp = None
        if masks is not None:
            masks = np.ascontiguousarray(masks, np.uint8)
            mp = _ptr(masks)
        self._chk(self.lib.ref_run_heads(grid_text.encode(), SZ(H), SZ(d), _ptr(q), _ptr(k), _ptr(v),
                                         "".join(orders).encode(), mp, ctypes.c_uint(bits), ctypes.c_float(scale),
                                         ctypes.c_int(threads), _ptr(out), ctypes.byref(secs)))
        return out, secs.value
