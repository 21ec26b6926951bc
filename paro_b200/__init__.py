"""paro_b200 -- Python host mirror of the PAROAttention hot-path API over the C ABI.

The product is the sm_100a library ``paro_b200/_lib/libparo_b200.so`` (CUDA
kernels + C ABI declared in ``include/paro_b200.h``). This module binds it with
ctypes and mirrors the reference's C++ entry points on the hot path (names,
argument meaning and error classes of ``proj/include/paro/*.hpp``) so tests read
like the reference's own tests:

  reference (proj/include/paro)                 here
  ---------------------------------------------  ------------------------------
  parse_grid / TokenGrid (tensor.hpp:44-65)       parse_grid / TokenGrid
  make_perm / PermPlan (reorder.hpp:18-32)        make_perm / PermPlan
  enumerate_perms (reorder.hpp:36)                enumerate_perms
  apply_perm_rows (reorder.hpp:39)                Context.apply_perm_rows   [GPU]
  quantize {Symmetric, PerBlock, 64} (quant.hpp)  Context.quantize          [GPU]
  BlockMask / (de)serialize_mask (mask.hpp)       BlockMask / (de)serialize_mask
  MaskSchedule::at / load_schedule                schedule_at
  gen_mask / build_schedule (mask.hpp:47-60)      Context.gen_mask / build_schedule [GPU]
  quantized_blocked_attention (attention.hpp:52)  Context.quantized_blocked_attention [GPU]
  cmd_run's per-head chain, H heads (main.cpp)    Layer                     [GPU]
  save/load_tensor PAT1 (tensor_io.hpp)          encode_tensor / decode_tensor / load_matrix
  save/load_quant_tensor PARQ (quant.hpp:68-74)  encode_quant / decode_quant, Layer.export_parq

Errors raise the reference's exception classes (error.hpp:11-40) with the same
exit codes. There is no CPU fallback: without the built library, importing this
module fails; without an sm_100 GPU, every device call raises CudaError.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PARO_B200_LIB") or os.path.join(_HERE, "_lib", "libparo_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"paro_b200: native library missing at {LIB_PATH}; build it with `make -C paro_b200` "
        "(there is no CPU fallback)"
    )
_lib = ctypes.CDLL(LIB_PATH)

# ----------------------------------------------------------------------------- errors


class Error(RuntimeError):
    """paro::Error -- carries the CLI exit code (error.hpp:14-19)."""

    exit_code = 1


class ConfigError(Error):
    exit_code = 2


class ShapeError(Error):
    exit_code = 2


class InputError(Error):
    exit_code = 2


class FormatError(Error):
    exit_code = 3


class IoError(Error):
    exit_code = 3


class InvariantError(Error):
    exit_code = 4


class CudaError(Error):
    """CUDA runtime failure (no reference counterpart)."""

    exit_code = 5


_STATUS = {
    20: ConfigError,
    21: ShapeError,
    22: InputError,
    30: FormatError,
    31: IoError,
    40: InvariantError,
    50: CudaError,
}

_lib.paro_last_error.restype = ctypes.c_char_p
_lib.paro_version.restype = ctypes.c_char_p


def _check(status: int) -> None:
    if status != 0:
        msg = _lib.paro_last_error().decode("utf-8", "replace")
        raise _STATUS.get(status, Error)(msg)


def version() -> str:
    return _lib.paro_version().decode()


P = ctypes.c_void_p
U32 = ctypes.c_uint32
SZ = ctypes.c_size_t


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


# ----------------------------------------------------------------------------- grid / perm


@dataclass
class TokenGrid:
    """Labeled token layout, row-major in the listed axis order (tensor.hpp:44-55)."""

    labels: str
    extents: tuple

    @property
    def ndim(self) -> int:
        return len(self.labels)

    def token_count(self) -> int:
        n = 1
        for e in self.extents:
            n *= int(e)
        return n

    def label_string(self) -> str:
        return self.labels

    def text(self) -> str:
        return ",".join(f"{l}:{e}" for l, e in zip(self.labels, self.extents))


def parse_grid(text: str) -> TokenGrid:
    ndim = ctypes.c_int()
    labels = ctypes.create_string_buffer(4)
    ext = (U32 * 3)()
    _check(_lib.paro_parse_grid(text.encode(), ctypes.byref(ndim), labels, ext))
    return TokenGrid(labels.raw[: ndim.value].decode(), tuple(int(ext[i]) for i in range(ndim.value)))


def _grid_args(grid: TokenGrid):
    ext = (U32 * 3)(*[int(e) for e in grid.extents] + [0] * (3 - grid.ndim))
    return ctypes.c_int(grid.ndim), grid.labels.encode(), ext


@dataclass
class PermPlan:
    """forward[old] = new, inverse[new] = old (reorder.hpp:18-29)."""

    order: str
    forward: np.ndarray
    inverse: np.ndarray

    def is_identity(self) -> bool:
        return bool(np.all(self.forward == np.arange(len(self.forward), dtype=np.uint32)))

    def inverted(self) -> "PermPlan":
        return PermPlan(self.order + "'", self.inverse.copy(), self.forward.copy())


def make_perm(grid: TokenGrid, order: str) -> PermPlan:
    n = grid.token_count()
    fwd = np.empty(n, np.uint32)
    inv = np.empty(n, np.uint32)
    nd, lab, ext = _grid_args(grid)
    _check(_lib.paro_make_perm(nd, lab, ext, order.encode(), P(_ptr(fwd)), P(_ptr(inv))))
    return PermPlan(order, fwd, inv)


def enumerate_orders(grid: TokenGrid) -> list:
    buf = ctypes.create_string_buffer(6 * 3 + 1)
    cnt = ctypes.c_int()
    _check(_lib.paro_enumerate_orders(ctypes.c_int(grid.ndim), grid.labels.encode(), buf, ctypes.byref(cnt)))
    raw = buf.raw[: cnt.value * grid.ndim].decode()
    return [raw[i * grid.ndim : (i + 1) * grid.ndim] for i in range(cnt.value)]


def enumerate_perms(grid: TokenGrid) -> list:
    return [make_perm(grid, o) for o in enumerate_orders(grid)]


# ----------------------------------------------------------------------------- masks


@dataclass
class BlockMask:
    """k_rows x k_cols keep grid, one byte per block, row-major (mask.hpp:15-32)."""

    k_rows: int
    k_cols: int
    block: int
    bits: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.bits is None:
            self.bits = np.zeros((self.k_rows, self.k_cols), np.uint8)
        self.bits = np.ascontiguousarray(self.bits, dtype=np.uint8).reshape(self.k_rows, self.k_cols)

    def get(self, i, j) -> bool:
        return bool(self.bits[i, j])

    def set(self, i, j, v: bool) -> None:
        self.bits[i, j] = 1 if v else 0

    def popcount(self) -> int:
        return int(np.count_nonzero(self.bits))

    def density(self) -> float:
        return self.popcount() / float(self.k_rows * self.k_cols)


def serialize_mask(m: BlockMask) -> bytes:
    size = SZ()
    bits = np.ascontiguousarray(m.bits, np.uint8)
    _check(_lib.paro_serialize_mask(P(_ptr(bits)), U32(m.k_rows), U32(m.k_cols), U32(m.block), None, ctypes.byref(size)))
    out = np.empty(size.value, np.uint8)
    _check(_lib.paro_serialize_mask(P(_ptr(bits)), U32(m.k_rows), U32(m.k_cols), U32(m.block), P(_ptr(out)),
                                    ctypes.byref(size)))
    return out.tobytes()


def deserialize_mask(data: bytes):
    """Returns (BlockMask, consumed bytes) (mask.cpp:217-244)."""
    buf = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
    kr, kc, b = U32(), U32(), U32()
    used = SZ()
    _check(_lib.paro_deserialize_mask(P(_ptr(buf)), SZ(len(data)), ctypes.byref(kr), ctypes.byref(kc), ctypes.byref(b),
                                      None, ctypes.byref(used)))
    bits = np.empty((kr.value, kc.value), np.uint8)
    _check(_lib.paro_deserialize_mask(P(_ptr(buf)), SZ(len(data)), ctypes.byref(kr), ctypes.byref(kc), ctypes.byref(b),
                                      P(_ptr(bits)), ctypes.byref(used)))
    return BlockMask(kr.value, kc.value, b.value, bits), used.value


def schedule_at(data: bytes, t: int) -> BlockMask:
    """load_schedule(...).at(t) on an in-memory PSCH image (mask.cpp:132-140, 267-305)."""
    buf = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
    kr, kc, b = U32(), U32(), U32()
    _check(_lib.paro_schedule_at(P(_ptr(buf)), SZ(len(data)), U32(t), ctypes.byref(kr), ctypes.byref(kc),
                                 ctypes.byref(b), None))
    bits = np.empty((kr.value, kc.value), np.uint8)
    _check(_lib.paro_schedule_at(P(_ptr(buf)), SZ(len(data)), U32(t), ctypes.byref(kr), ctypes.byref(kc),
                                 ctypes.byref(b), P(_ptr(bits))))
    return BlockMask(kr.value, kc.value, b.value, bits)


def parse_plan(text: bytes, name: str = "plan"):
    """load_plan_file (reorder.cpp:193-216) on plan text: [(head, order)] in file order."""
    cnt, size = U32(), SZ()
    _check(_lib.paro_parse_plan(text, SZ(len(text)), name.encode(), ctypes.byref(cnt), None, None, ctypes.byref(size)))
    heads = np.empty(max(1, cnt.value), np.uint32)
    buf = ctypes.create_string_buffer(max(1, size.value))
    _check(_lib.paro_parse_plan(text, SZ(len(text)), name.encode(), ctypes.byref(cnt), P(_ptr(heads)), buf,
                                ctypes.byref(size)))
    orders = buf.raw[:size.value].split(b"\0")[:cnt.value]
    return [(int(heads[i]), orders[i].decode()) for i in range(cnt.value)]


def load_plan_file(path: str):
    """[(head, order)] of a plan file (IoError when it cannot be read, like the reference)."""
    try:
        with open(path, "rb") as f:
            text = f.read()
    except OSError:
        raise IoError(f"cannot open '{path}' for reading") from None
    return parse_plan(text, path)


def plan_orders(plan_path: Optional[str], grid: "TokenGrid | str", heads: Sequence[int]) -> list:
    """plan_for_head (tools/main.cpp:118-126) for each head: no plan file -> the identity
    order; else the head's entry (InputError when missing). Orders for Layer()."""
    text = None
    name = plan_path or "plan"
    if plan_path:
        try:
            with open(plan_path, "rb") as f:
                text = f.read()
        except OSError:
            raise IoError(f"cannot open '{plan_path}' for reading") from None
    gtext = grid if isinstance(grid, str) else grid.text()
    ids = np.ascontiguousarray(list(heads), np.uint32)
    nd = len(parse_grid(gtext).labels)
    out = ctypes.create_string_buffer(max(1, len(ids) * nd))
    _check(_lib.paro_plan_for_heads(text, SZ(len(text) if text is not None else 0), name.encode(), gtext.encode(),
                                    U32(len(ids)), P(_ptr(ids)) if len(ids) else None, out))
    raw = out.raw[:len(ids) * nd].decode()
    return [raw[i * nd:(i + 1) * nd] for i in range(len(ids))]


def unpack_nibbles(packed: np.ndarray) -> np.ndarray:
    """Two's-complement INT4 pairs, low nibble first (quant.cpp:237-243, 313-318) -> int8."""
    p = np.asarray(packed, np.uint8)
    lo = (p & 0x0F).astype(np.int8)
    hi = (p >> 4).astype(np.int8)
    lo = np.where(lo > 7, lo - 16, lo).astype(np.int8)
    hi = np.where(hi > 7, hi - 16, hi).astype(np.int8)
    out = np.empty(p.shape[:-1] + (2 * p.shape[-1],), np.int8)
    out[..., 0::2] = lo
    out[..., 1::2] = hi
    return out


def serialize_schedule(timesteps: int, masks: Sequence["BlockMask"]) -> bytes:
    """PSCH image of a schedule (save_schedule, mask.cpp:246-263): `masks` holds the
    timesteps//2 distinct masks (timestep i = position i) and then the shared late mask."""
    half = timesteps // 2
    if len(masks) != half + 1:
        raise ShapeError(f"a {timesteps}-step schedule has {half} distinct masks + 1 shared, got {len(masks)}")
    out = bytearray(b"PSCH")
    out += int(timesteps).to_bytes(4, "little") + int(half).to_bytes(4, "little")
    for i in range(half):
        out += int(i).to_bytes(4, "little") + serialize_mask(masks[i])
    out += serialize_mask(masks[half])
    return bytes(out)


def synth_randn(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float32)
    _check(_lib.paro_synth_randn(ctypes.c_uint64(seed), SZ(count), P(_ptr(out))))
    return out


# ----------------------------------------------------------------------------- quant config


@dataclass
class QuantConfig:
    """QuantConfig (quant.hpp:25-34). mode: 0 Unsigned, 1 Symmetric; grouping: 0 PerBlock, 1 PerRow."""

    bits: int = 8
    mode: int = 0
    grouping: int = 0
    block: int = 64

    def validate(self) -> None:
        if self.bits not in (4, 8):
            raise ConfigError(f"quantization bitwidth must be 4 or 8, got {self.bits}")
        if self.block < 1:
            raise ConfigError("quantization block must be >= 1")

    def qmin(self) -> int:
        return 0 if self.mode == 0 else -((1 << (self.bits - 1)) - 1)

    def qmax(self) -> int:
        return (1 << self.bits) - 1 if self.mode == 0 else (1 << (self.bits - 1)) - 1


UNSIGNED, SYMMETRIC = 0, 1
PER_BLOCK, PER_ROW = 0, 1


@dataclass
class QuantBlockTensor:
    rows: int
    cols: int
    config: QuantConfig
    codes: np.ndarray
    scales: np.ndarray
    offsets: np.ndarray


# ----------------------------------------------------------------------------- PAT1 / PARQ interchange


class _QuantHeader(ctypes.Structure):
    _fields_ = [("bits", ctypes.c_uint), ("mode", ctypes.c_int), ("grouping", ctypes.c_int), ("block", U32),
                ("rows", U32), ("cols", U32), ("groups", U32)]


def _buf(data: bytes) -> np.ndarray:
    return np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)


def encode_tensor(values: np.ndarray) -> bytes:
    """save_tensor's PAT1 bytes (tensor_io.cpp:45-71) of an fp32 array of any rank 1..255."""
    v = np.ascontiguousarray(values, np.float32)
    shape = np.asarray(v.shape if v.ndim else (1,), np.uint32)
    size = SZ()
    _check(_lib.paro_tensor_encode(P(_ptr(shape)), U32(v.ndim), P(_ptr(v)), None, ctypes.byref(size)))
    out = np.empty(size.value, np.uint8)
    _check(_lib.paro_tensor_encode(P(_ptr(shape)), U32(v.ndim), P(_ptr(v)), P(_ptr(out)), ctypes.byref(size)))
    return out.tobytes()


def decode_tensor(data: bytes) -> np.ndarray:
    """load_tensor (tensor_io.cpp:73-120): FormatError names the byte offset."""
    buf = _buf(data)
    nd = U32()
    shape = np.zeros(255, np.uint32)
    _check(_lib.paro_tensor_decode(P(_ptr(buf)), SZ(len(data)), ctypes.byref(nd), P(_ptr(shape)), None))
    out = np.empty(tuple(int(x) for x in shape[:nd.value]), np.float32)
    _check(_lib.paro_tensor_decode(P(_ptr(buf)), SZ(len(data)), ctypes.byref(nd), P(_ptr(shape)), P(_ptr(out))))
    return out


def load_matrix(data: bytes) -> np.ndarray:
    """load_matrix (tensor_io.cpp:130-137): a 2-D tensor of finite values."""
    t = decode_tensor(data)
    if t.ndim != 2:
        raise FormatError(f"expected a 2D tensor, found ndim={t.ndim}")
    bad = np.flatnonzero(~np.isfinite(t))
    if bad.size:
        raise InvariantError(f"non-finite value at flat index {int(bad[0])}")
    return t


def encode_quant(q: "QuantBlockTensor") -> bytes:
    """save_quant_tensor's PARQ bytes (quant.cpp:219-251)."""
    codes = np.ascontiguousarray(q.codes, np.int32).reshape(-1)
    scales = np.ascontiguousarray(q.scales, np.float32)
    offs = np.ascontiguousarray(q.offsets if q.offsets is not None and len(q.offsets) else np.zeros(1), np.float32)
    c = q.config
    args = (ctypes.c_uint(c.bits), ctypes.c_int(c.mode), ctypes.c_int(c.grouping), U32(c.block), U32(q.rows),
            U32(q.cols), P(_ptr(codes)), P(_ptr(scales)), P(_ptr(offs)))
    size = SZ()
    _check(_lib.paro_quant_encode(*args, None, ctypes.byref(size)))
    out = np.empty(size.value, np.uint8)
    _check(_lib.paro_quant_encode(*args, P(_ptr(out)), ctypes.byref(size)))
    return out.tobytes()


def decode_quant(data: bytes) -> "QuantBlockTensor":
    """load_quant_tensor (quant.cpp:253-326)."""
    buf = _buf(data)
    h = _QuantHeader()
    _check(_lib.paro_quant_decode(P(_ptr(buf)), SZ(len(data)), ctypes.byref(h), None, None, None))
    codes = np.empty(max(1, h.rows * h.cols), np.int32)
    scales = np.empty(max(1, h.groups), np.float32)
    offs = np.empty(max(1, h.groups), np.float32)
    _check(_lib.paro_quant_decode(P(_ptr(buf)), SZ(len(data)), ctypes.byref(h), P(_ptr(codes)), P(_ptr(scales)),
                                  P(_ptr(offs))))
    cfg = QuantConfig(h.bits, h.mode, h.grouping, h.block)
    return QuantBlockTensor(h.rows, h.cols, cfg, codes[:h.rows * h.cols].reshape(h.rows, h.cols),
                            scales[:h.groups], offs[:h.groups] if h.mode == UNSIGNED else np.zeros(0, np.float32))


@dataclass
class AttnInputs:
    """AttnInputs (attention.hpp:16-26): Q/K/V N x d fp32; scale 0 -> 1/sqrt(d)."""

    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    scale: float = 0.0
    dense_prefix: int = 0

    def validate(self) -> None:
        if self.q.shape != self.k.shape or self.q.shape != self.v.shape or self.q.ndim != 2:
            raise ShapeError(f"Q/K/V must share N x d, got Q {self.q.shape}, K {self.k.shape}, V {self.v.shape}")
        if self.q.shape[0] == 0 or self.q.shape[1] == 0:
            raise ShapeError("attention inputs must be non-empty")
        if self.dense_prefix > self.q.shape[0]:
            raise ConfigError(f"dense_prefix {self.dense_prefix} exceeds token count {self.q.shape[0]}")


@dataclass
class AttnResult:
    output: np.ndarray
    zeroed_rows: list


# ----------------------------------------------------------------------------- device plumbing


class DeviceBuffer:
    """cudaMalloc'd bytes owned by Python (freed on close/GC)."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        p = P()
        _check(_lib.paro_device_alloc(SZ(max(self.nbytes, 1)), ctypes.byref(p)))
        self.ptr = p.value

    @classmethod
    def from_array(cls, a: np.ndarray, stream=None) -> "DeviceBuffer":
        a = np.ascontiguousarray(a)
        b = cls(a.nbytes)
        b.upload(a, stream)
        return b

    def upload(self, a: np.ndarray, stream=None) -> None:
        a = np.ascontiguousarray(a)
        assert a.nbytes <= self.nbytes
        _check(_lib.paro_memcpy(P(self.ptr), P(_ptr(a)), SZ(a.nbytes), P(stream)))
        _check(_lib.paro_stream_sync(P(stream)))

    def download(self, shape, dtype, stream=None) -> np.ndarray:
        out = np.empty(shape, dtype)
        _check(_lib.paro_memcpy(P(_ptr(out)), P(self.ptr), SZ(out.nbytes), P(stream)))
        _check(_lib.paro_stream_sync(P(stream)))
        return out

    def close(self) -> None:
        if self.ptr:
            _lib.paro_device_free(P(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _close(*bufs) -> None:
    """Free temporaries now: the device allocations must not outlive the call
    (compute-sanitizer --leak-check full found them alive at context teardown)."""
    for b in bufs:
        if b is not None:
            b.close()


def download_ptr(ptr: int, shape, dtype, stream=None) -> np.ndarray:
    out = np.empty(shape, dtype)
    _check(_lib.paro_memcpy(P(_ptr(out)), P(ptr), SZ(out.nbytes), P(stream)))
    _check(_lib.paro_stream_sync(P(stream)))
    return out


class HostBuffer:
    """Pinned host memory (cudaHostAlloc) viewed as a numpy array."""

    def __init__(self, shape, dtype):
        dt = np.dtype(dtype)
        n = int(np.prod(shape)) * dt.itemsize
        p = P()
        _check(_lib.paro_host_alloc(SZ(max(n, 1)), ctypes.byref(p)))
        self.ptr = p.value
        self.array = np.frombuffer((ctypes.c_char * max(n, 1)).from_address(self.ptr), dtype=dt,
                                   count=int(np.prod(shape))).reshape(shape)

    def close(self):
        if self.ptr:
            self.array = None
            _lib.paro_host_free(P(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Buffers(ctypes.Structure):
    _fields_ = [
        ("heads", U32), ("tokens", U32), ("head_dim", U32), ("kblocks", U32), ("kblocks_padded", U32),
        ("groups", U32), ("q_codes", P), ("k_codes", P), ("v_codes", P), ("q_scales", P), ("tile_meta", P),
        ("inverse", P), ("forward", P), ("v_bits", U32), ("v_packed", U32),
    ]


class Context:
    """One device context (paro_ctx) per GPU."""

    def __init__(self, device: int = 0):
        p = P()
        _check(_lib.paro_ctx_create(ctypes.c_int(device), ctypes.byref(p)))
        self.ptr = p.value
        n = ctypes.c_int()
        _check(_lib.paro_ctx_num_sms(P(self.ptr), ctypes.byref(n)))
        self.num_sms = n.value

    def close(self):
        if self.ptr:
            _lib.paro_ctx_destroy(P(self.ptr))
            self.ptr = None

    # -- mask producer ----------------------------------
    def block_sums(self, m: np.ndarray, block: int = 64, plan: "PermPlan | None" = None) -> np.ndarray:
        """block_sums(AttnMap(apply_perm_map(m, plan), block)) on the GPU, fused
        (reorder.cpp:103-114, metrics.cpp:41-58; cmd_maskgen main.cpp:236-238).
        Returns the fp64 [k, k] grid, bit-identical to the reference's scalar kernels."""
        m = np.ascontiguousarray(m, np.float32)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ShapeError(f"attention map must be square, got {m.shape}")
        n = m.shape[0]
        if plan is not None and len(plan.inverse) != n:
            raise ShapeError("apply_perm_map: map/plan size mismatch")
        k = (n + block - 1) // block
        dm = DeviceBuffer.from_array(m)
        dinv = DeviceBuffer.from_array(np.ascontiguousarray(plan.inverse, np.uint32)) if plan is not None else None
        ds = DeviceBuffer(k * k * 8)
        _check(_lib.paro_perm_block_sums_device(P(self.ptr), None, P(dm.ptr), U32(n), P(dinv.ptr if dinv else None),
                                                U32(block), P(ds.ptr)))
        out = ds.download((k, k), np.float64)
        _close(dm, dinv, ds)
        return out

    def k1_quant_proof(self, bits_begin: int, bits_count: int, nx: int = 14, seed: int = 1):
        """Test hook: K1's quantizer vs the reference quant_affine over amax bit patterns
        (paro_debug_k1_quant_proof) -> (mismatches, first mismatch record or None)."""
        bad = ctypes.c_uint64()
        first = (U32 * 5)()
        _check(_lib.paro_debug_k1_quant_proof(P(self.ptr), U32(bits_begin), ctypes.c_uint64(bits_count), U32(nx),
                                              U32(seed), ctypes.byref(bad), first))
        return bad.value, (tuple(first) if bad.value else None)

    def gen_mask(self, sums: np.ndarray, density: float, block: int, guard_blocks: int = 0):
        """gen_mask on the GPU for one [k, k] grid or a stack [count, k, k]
        (mask.cpp:56-130). Returns (BlockMask | list[BlockMask], repaired rows)."""
        s = np.ascontiguousarray(sums, np.float64)
        stack = s.ndim == 3
        s3 = s if stack else s[None]
        count, kr, kc = s3.shape
        ds = DeviceBuffer.from_array(s3)
        db = DeviceBuffer(count * kr * kc)
        rep = np.zeros(count, np.uint32)
        _check(_lib.paro_gen_mask_device(P(self.ptr), None, P(ds.ptr), U32(count), U32(kr), U32(kc),
                                         ctypes.c_double(density), U32(block), U32(guard_blocks), P(db.ptr),
                                         P(_ptr(rep))))
        bits = db.download((count, kr, kc), np.uint8)
        _close(ds, db)
        masks = [BlockMask(kr, kc, block, bits[i]) for i in range(count)]
        return (masks, rep.tolist()) if stack else (masks[0], int(rep[0]))

    def build_schedule(self, sums: np.ndarray, density: float, block: int, guard_blocks: int = 0):
        """build_schedule on the GPU (mask.cpp:142-172): sums [T, k, k] ->
        (list of T/2 distinct masks + the shared late mask, total repaired rows)."""
        s = np.ascontiguousarray(sums, np.float64)
        T, kr, kc = s.shape
        half = T // 2
        ds = DeviceBuffer.from_array(s)
        dm = DeviceBuffer((half + 1) * kr * kc)
        rep = U32()
        _check(_lib.paro_build_schedule_device(P(self.ptr), None, P(ds.ptr), U32(T), U32(kr), U32(kc),
                                               ctypes.c_double(density), U32(block), U32(guard_blocks), P(dm.ptr),
                                               ctypes.byref(rep)))
        bits = dm.download((half + 1, kr, kc), np.uint8)
        _close(ds, dm)
        return [BlockMask(kr, kc, block, bits[i]) for i in range(half + 1)], rep.value

    def select_permutation(self, maps, grid: "TokenGrid | str", block: int = 64, eps: float = 1e-3,
                           sigma: float = 0.9, alpha: float = 0.5, dense_prefix: int = 0):
        """select_permutation(calib, grid, cfg, dense_prefix) on the GPU
        (reorder.cpp:130-181, metrics.cpp:60-133). maps: [count, n+p, n+p] fp32.
        Returns (orders, scores [nperm, 5] = sparse_mean, quant_mean,
        sparse_share, quant_share, combined, chosen index)."""
        m = np.ascontiguousarray(maps, np.float32)
        if m.ndim == 2:
            m = m[None]
        text = grid if isinstance(grid, str) else grid.text()
        dm = DeviceBuffer.from_array(m)
        orders = ctypes.create_string_buffer(32)
        scores = np.zeros((6, 5), np.float64)
        nperm, chosen = ctypes.c_int(), ctypes.c_int()
        _check(_lib.paro_select_permutation_device(P(self.ptr), None, P(dm.ptr), U32(m.shape[0]), text.encode(),
                                                   U32(block), ctypes.c_float(eps), ctypes.c_float(sigma),
                                                   ctypes.c_float(alpha), U32(dense_prefix), orders, P(_ptr(scores)),
                                                   ctypes.byref(nperm), ctypes.byref(chosen)))
        _close(dm)
        nd = len(orders.raw.rstrip(b"\0")) // nperm.value
        ords = [orders.raw[i * nd:(i + 1) * nd].decode() for i in range(nperm.value)]
        return ords, scores[:nperm.value], chosen.value

    # -- standalone stages -------------------------------------------------
    def apply_perm_rows(self, m: np.ndarray, plan: PermPlan) -> np.ndarray:
        """apply_perm_rows on the GPU (reorder.cpp:93-101)."""
        m = np.ascontiguousarray(m, np.float32)
        if m.shape[0] != len(plan.forward):
            raise ShapeError(f"apply_perm_rows: matrix has {m.shape[0]} rows, plan covers {len(plan.forward)}")
        din = DeviceBuffer.from_array(m)
        dinv = DeviceBuffer.from_array(np.ascontiguousarray(plan.inverse, np.uint32))
        dout = DeviceBuffer(m.nbytes)
        _check(_lib.paro_apply_perm_rows_device(P(self.ptr), None, P(din.ptr), U32(m.shape[0]), U32(m.shape[1]),
                                                P(dinv.ptr), P(dout.ptr)))
        out = dout.download(m.shape, np.float32)
        _close(din, dinv, dout)
        return out

    def quantize(self, m: np.ndarray, cfg: QuantConfig) -> QuantBlockTensor:
        """quantize(m, cfg) on the GPU for the hot path's configuration
        {bits 4|8, Symmetric, PerBlock, block 64}, cols 64|128 (quant.cpp:60-104)."""
        cfg.validate()
        if cfg.mode != SYMMETRIC or cfg.grouping != PER_BLOCK or cfg.block != 64:
            raise ConfigError("the B200 quantizer serves {Symmetric, PerBlock, 64} (the Q/K configuration)")
        m = np.ascontiguousarray(m, np.float32)
        rows, cols = m.shape
        groups = ((rows + 63) // 64) * ((cols + 63) // 64)
        din = DeviceBuffer.from_array(m)
        dc = DeviceBuffer(rows * cols)
        ds = DeviceBuffer(groups * 4)
        _check(_lib.paro_quantize_sym_device(P(self.ptr), None, P(din.ptr), U32(rows), U32(cols), ctypes.c_int(cfg.bits),
                                             P(dc.ptr), P(ds.ptr)))
        codes = dc.download((rows, cols), np.int8).astype(np.int32)
        scales = ds.download((groups,), np.float32)
        _close(din, dc, ds)
        return QuantBlockTensor(rows, cols, cfg, codes, scales, np.zeros(0, np.float32))

    def quantized_blocked_attention(self, inp: AttnInputs, mask: Optional[BlockMask], qcfg: QuantConfig) -> AttnResult:
        """quantized_blocked_attention (attention.hpp:52) with the INT8-QK stage, one head,
        identity token order; block = mask.block or qcfg.block (attention.cpp:266-269)."""
        inp.validate()
        qcfg.validate()
        n, d = inp.q.shape
        block = mask.block if mask is not None else qcfg.block
        if block != 64:
            raise ConfigError(f"the B200 path runs block 64, got {block}")
        dp = int(inp.dense_prefix)
        if dp >= n and n > 0:
            raise ConfigError("dense_prefix covering every token is not served by the B200 path")
        kb = (n + 63) // 64
        if mask is not None and (mask.k_rows != kb or mask.k_cols != kb):
            raise ShapeError(f"mask grid {mask.k_rows}x{mask.k_cols} does not cover {kb}x{kb} blocks")
        layer = Layer(self, 1, d, TokenGrid("HW", (1, n - dp)), dense_prefix=dp)
        try:
            layer.set_masks(None if mask is None else mask.bits.reshape(1, kb, kb))
            out, zeroed = layer.forward_host(inp.q.reshape(1, n, d), inp.k.reshape(1, n, d), inp.v.reshape(1, n, d),
                                             inp.scale, qcfg.bits)
        finally:
            layer.close()
        return AttnResult(out.reshape(n, d), [int(i) for i in np.nonzero(zeroed.reshape(n))[0]])


class Layer:
    """H heads of cmd_run's per-head chain (main.cpp:276-305) on one GPU."""

    def __init__(self, ctx: Context, heads: int, head_dim: int, grid, orders: Optional[Sequence[str]] = None,
                 dense_prefix: int = 0):
        """dense_prefix: leading text tokens kept in place, dense and unquantized
        (AttnInputs::dense_prefix, PermPlan::with_prefix); N = grid tokens + prefix."""
        if isinstance(grid, str):
            grid = parse_grid(grid)
        self.ctx, self.heads, self.head_dim, self.grid = ctx, heads, head_dim, grid
        self.dense_prefix = int(dense_prefix)
        self.N = grid.token_count() + self.dense_prefix
        self.kb = (self.N + 63) // 64
        ords = None
        if orders is not None:
            if len(orders) != heads:
                raise ConfigError(f"need {heads} orders, got {len(orders)}")
            ords = "".join(orders).encode()
        p = P()
        _check(_lib.paro_layer_create_prefix(P(ctx.ptr), U32(heads), U32(head_dim), grid.text().encode(), ords,
                                             U32(self.dense_prefix), ctypes.byref(p)))
        self.ptr = p.value

    def close(self):
        if self.ptr:
            _lib.paro_layer_destroy(P(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_masks(self, bits: Optional[np.ndarray], stream=None, sync: bool = True) -> None:
        """Host mask bytes [H][k][k] (None = all kept). sync=False leaves the upload and K2
        queued on `stream` (then `bits` must stay alive, e.g. a pinned HostBuffer)."""
        if bits is None:
            _check(_lib.paro_layer_set_masks(P(self.ptr), P(stream), None))
            return
        b = np.ascontiguousarray(bits, np.uint8)
        if b.size != self.heads * self.kb * self.kb:
            raise ShapeError(f"masks must be {self.heads}x{self.kb}x{self.kb} bytes, got {b.shape}")
        _check(_lib.paro_layer_set_masks(P(self.ptr), P(stream), P(_ptr(b))))
        if sync or b is not bits:
            _check(_lib.paro_stream_sync(P(stream)))

    def set_masks_pmsk(self, blobs: Sequence[bytes], stream=None) -> None:
        """One serialized PMSK mask per head (deserialize_mask, mask.cpp:217-244)."""
        if len(blobs) != self.heads:
            raise ShapeError(f"{len(blobs)} PMSK blobs for {self.heads} heads")
        bufs = [np.frombuffer(b, np.uint8).copy() if len(b) else np.zeros(1, np.uint8) for b in blobs]
        ptrs = (ctypes.c_void_p * self.heads)(*[_ptr(x) for x in bufs])
        sizes = (ctypes.c_size_t * self.heads)(*[len(b) for b in blobs])
        _check(_lib.paro_layer_set_masks_pmsk(P(self.ptr), P(stream), ptrs, sizes))

    def set_schedule(self, blobs: Sequence[bytes], resident_lists: int = 0, stream=None) -> None:
        """One PSCH image per head (paro_layer_set_schedule): resident_lists 0 builds every
        entry's kept lists now; 2 double-buffers them with a prefetch of t+1."""
        if len(blobs) != self.heads:
            raise ShapeError(f"{len(blobs)} schedules for {self.heads} heads")
        bufs = [np.frombuffer(b, np.uint8).copy() if len(b) else np.zeros(1, np.uint8) for b in blobs]
        ptrs = (P * len(bufs))(*[P(_ptr(b)) for b in bufs])
        sizes = (SZ * len(bufs))(*[len(b) for b in blobs])
        _check(_lib.paro_layer_set_schedule(P(self.ptr), P(stream), ptrs, sizes, U32(resident_lists)))

    def set_v_packing(self, packed: bool) -> None:
        """INT4 V nibble-packed in HBM and unpacked to i8 in shared memory by K3
        (paro_layer_set_v_packing); from the next reorder_quantize."""
        _check(_lib.paro_layer_set_v_packing(P(self.ptr), ctypes.c_int(1 if packed else 0)))

    def select_timestep(self, t: int, stream=None) -> None:
        """Make timestep t's masks current (MaskSchedule::at(t), mask.cpp:132-140)."""
        _check(_lib.paro_layer_select_timestep(P(self.ptr), P(stream), U32(t)))

    def schedule_info(self):
        T, E, cur = U32(), U32(), ctypes.c_int()
        _check(_lib.paro_layer_schedule_info(P(self.ptr), ctypes.byref(T), ctypes.byref(E), ctypes.byref(cur)))
        return T.value, E.value, cur.value

    def set_rope(self, cos: Optional[np.ndarray], sin: Optional[np.ndarray], stream=None) -> None:
        """Rotary embedding fused into K1 (paro_layer_set_rope): cos / sin [N - dense_prefix, d]
        fp32 per original grid token; None, None turns it off."""
        if cos is None and sin is None:
            _check(_lib.paro_layer_set_rope(P(self.ptr), P(stream), None, None))
            return
        if cos is None or sin is None:
            raise ConfigError("rope: cos and sin must both be given or both be None")
        shape = (self.N - self.dense_prefix, self.head_dim)
        c = np.ascontiguousarray(cos, np.float32)
        s = np.ascontiguousarray(sin, np.float32)
        if c.shape != shape or s.shape != shape:
            raise ShapeError(f"rope tables must be {shape}, got {c.shape} / {s.shape}")
        _check(_lib.paro_layer_set_rope(P(self.ptr), P(stream), P(_ptr(c)), P(_ptr(s))))
        _check(_lib.paro_stream_sync(P(stream)))

    def set_masks_device(self, dptr: Optional[int], stream=None) -> None:
        _check(_lib.paro_layer_set_masks_device(P(self.ptr), P(stream), P(dptr) if dptr else None))

    def reorder_quantize(self, dq: int, dk: int, dv: int, v_bits: int, stream=None) -> None:
        _check(_lib.paro_layer_reorder_quantize(P(self.ptr), P(stream), P(dq), P(dk), P(dv), ctypes.c_int(v_bits)))

    def attention(self, scale: float, pv_bits: int, dout: int, dzeroed: Optional[int] = None, stream=None) -> None:
        _check(_lib.paro_layer_attention(P(self.ptr), P(stream), ctypes.c_float(scale), ctypes.c_int(pv_bits), P(dout),
                                         P(dzeroed) if dzeroed else None))

    def forward(self, dq: int, dk: int, dv: int, scale: float, pv_bits: int, dout: int, dzeroed: Optional[int] = None,
                stream=None) -> None:
        _check(_lib.paro_layer_forward(P(self.ptr), P(stream), P(dq), P(dk), P(dv), ctypes.c_float(scale),
                                       ctypes.c_int(pv_bits), P(dout), P(dzeroed) if dzeroed else None))

    def set_pipeline_chunks(self, chunks: int, stream=None):
        """Head chunks of the forward_host upload/compute/download pipeline."""
        _check(_lib.paro_layer_set_pipeline_chunks(P(self.ptr), P(stream), U32(chunks)))

    def forward_host(self, q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float, pv_bits: int,
                     out: Optional[np.ndarray] = None, zeroed: Optional[np.ndarray] = None, stream=None):
        shape = (self.heads, self.N, self.head_dim)
        for name, a in (("Q", q), ("K", k), ("V", v)):
            if a.shape != shape or a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"]:
                raise ShapeError(f"{name} must be C-contiguous float32 {shape}, got {a.dtype} {a.shape}")
        if out is None:
            out = np.empty(shape, np.float32)
        if zeroed is None:
            zeroed = np.empty((self.heads, self.N), np.uint8)
        _check(_lib.paro_layer_forward_host(P(self.ptr), P(stream), P(_ptr(q)), P(_ptr(k)), P(_ptr(v)),
                                            ctypes.c_float(scale), ctypes.c_int(pv_bits), P(_ptr(out)),
                                            P(_ptr(zeroed))))
        return out, zeroed

    def buffers(self) -> dict:
        """Copies the layer-owned codes/scales/meta/perm tables back to host numpy arrays."""
        b = _Buffers()
        _check(_lib.paro_layer_get_buffers(P(self.ptr), ctypes.byref(b)))
        H, D, kb2 = b.heads, b.head_dim, b.kblocks_padded
        rows = kb2 * 64
        return {
            "q": download_ptr(b.q_codes, (H, rows, D), np.int8),
            "k": download_ptr(b.k_codes, (H, rows, D), np.int8),
            "v": (unpack_nibbles(download_ptr(b.v_codes, (H, rows, D // 2), np.uint8)) if b.v_packed
                  else download_ptr(b.v_codes, (H, rows, D), np.int8)),
            "v_packed": download_ptr(b.v_codes, (H, rows, D // 2), np.uint8) if b.v_packed else None,
            "q_scales": download_ptr(b.q_scales, (H, kb2, b.groups), np.float32),
            "meta": download_ptr(b.tile_meta, (H, kb2, 4 + D), np.float32),
            "inverse": download_ptr(b.inverse, (H, b.tokens), np.uint32),
            "forward": download_ptr(b.forward, (H, b.tokens), np.uint32),
            "kblocks": b.kblocks,
            "kblocks_padded": kb2,
        }

    def export_parq(self, head: int, which: str, stream=None) -> bytes:
        """PARQ blob of one head's permuted Q / K / V codes of the last reorder_quantize,
        byte-identical to the reference's save_quant_tensor(quantize(apply_perm_rows(X)))."""
        w = {"q": 0, "k": 1, "v": 2}[which.lower()]
        size = SZ()
        _check(_lib.paro_layer_export_parq(P(self.ptr), P(stream), U32(head), ctypes.c_int(w), None, ctypes.byref(size)))
        out = np.empty(size.value, np.uint8)
        _check(_lib.paro_layer_export_parq(P(self.ptr), P(stream), U32(head), ctypes.c_int(w), P(_ptr(out)),
                                           ctypes.byref(size)))
        return out.tobytes()

    def mask_stats(self):
        kept = np.empty((self.heads, self.kb), np.uint32)
        tot = ctypes.c_uint64()
        _check(_lib.paro_layer_mask_stats(P(self.ptr), P(_ptr(kept)), ctypes.byref(tot)))
        return kept, tot.value

    def debug_pdump(self, targets, scale: float = 0.0, pv_bits: int = 8):
        """Final P codes of each (head, q-block) in `targets` after K3 (test hook):
        codes [n][kb][64][64] and meta [n][kb][4] = (lo, pscale, key block, 1) per
        quantized tile in kept order (paro_layer_debug_pdump)."""
        return _pdump(self, targets, scale, pv_bits)

    def debug_qk(self, tiles: np.ndarray) -> np.ndarray:
        """int32 S_g of (h, qb, bj) tiles through K3's tcgen05 QK path -> [n, G, 64, 64]."""
        t = np.ascontiguousarray(tiles, np.uint32).reshape(-1, 3)
        G = self.head_dim // 64
        dt = DeviceBuffer.from_array(t)
        ds = DeviceBuffer(t.shape[0] * G * 64 * 64 * 4)
        _check(_lib.paro_layer_debug_qk(P(self.ptr), None, U32(t.shape[0]), P(dt.ptr), P(ds.ptr)))
        _check(_lib.paro_stream_sync(None))
        out = ds.download((t.shape[0], G, 64, 64), np.int32)
        _close(dt, ds)
        return out


def _pdump(layer, targets, scale, pv_bits):
    t = np.ascontiguousarray(targets, np.uint32).reshape(-1, 2)
    n = t.shape[0]
    codes = np.zeros((n, layer.kb, 64, 64), np.uint8)
    meta = np.zeros((n, layer.kb, 4), np.float32)
    _check(_lib.paro_layer_debug_pdump(P(layer.ptr), None, ctypes.c_float(scale), ctypes.c_int(pv_bits), U32(n),
                                       P(_ptr(t)), P(_ptr(codes)), P(_ptr(meta))))
    return codes, meta


def stream_sync(stream=None) -> None:
    _check(_lib.paro_stream_sync(P(stream)))
