"""Python mirror of the reference codec interface, served by the B200 kernels.

Mirrors /root/reference/proj/include/ghostserve/coding.hpp name for name --
``CodeKind``, ``CodingScheme`` (+ ``validate``/``xor_code``/``rdp``/
``reed_solomon``), ``max_tolerance``, ``memory_overhead_ratio``,
``EncodingMatrix``, ``build_encoding_matrix``, ``ErasurePattern``,
``UnrecoverableError``, ``encode`` and ``reconstruct`` -- with the same
argument meaning and error classes:

=============================  =====================================
reference (C++)                 here (Python)
=============================  =====================================
std::invalid_argument           InvalidArgument (ValueError)
ghostserve::UnrecoverableError  UnrecoverableError (RuntimeError)
std::domain_error               DomainError (ArithmeticError)
=============================  =====================================

``encode`` / ``reconstruct`` take host buffers (numpy arrays, bytes,
memoryviews) like the reference's spans and return host numpy arrays; the
bytes are produced on the GPU (H2D -> K1/K2 -> D2H through a staging
pipeline). Device-resident use goes through :mod:`.device`.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass
from typing import Dict, List, Mapping, Optional, Sequence

import numpy as np

from . import _lib as L


# ---------------------------------------------------------------------------
# errors (coding.hpp:32-35; gf256.hpp:48,53)
# ---------------------------------------------------------------------------
class InvalidArgument(ValueError, L.GhostServeError):
    status = L.GS_INVALID_ARGUMENT


class UnrecoverableError(RuntimeError, L.GhostServeError):
    status = L.GS_UNRECOVERABLE


class DomainError(ArithmeticError, L.GhostServeError):
    status = L.GS_DOMAIN_ERROR


class CudaError(RuntimeError, L.GhostServeError):
    status = L.GS_CUDA_ERROR


class Unsupported(NotImplementedError, L.GhostServeError):
    status = L.GS_UNSUPPORTED


class LogicError(RuntimeError, L.GhostServeError):
    """std::logic_error (e.g. duplicate parity-store entry, parity_store.hpp:78-82)."""
    status = L.GS_LOGIC_ERROR


class ParityFileError(RuntimeError, L.GhostServeError):
    """std::runtime_error of the GSRV reader (parity_store.hpp:301-397)."""
    status = L.GS_RUNTIME_ERROR


_BY_STATUS = {c.status: c for c in (InvalidArgument, UnrecoverableError, DomainError, CudaError,
                                     Unsupported, LogicError, ParityFileError)}


def check(status: int, what: str = "") -> None:
    """Raise the exception class that mirrors a C-ABI status."""
    if status == L.GS_OK:
        return
    msg = L.last_error() or L.lib().gs_status_string(status).decode()
    raise _BY_STATUS.get(status, L.GhostServeError)(f"{what}: {msg}" if what else msg)


# ---------------------------------------------------------------------------
# scheme (coding.hpp:17-81)
# ---------------------------------------------------------------------------
class CodeKind(enum.IntEnum):
    XOR = L.GS_XOR
    RDP = L.GS_RDP
    REED_SOLOMON = L.GS_RS


def to_string(kind: CodeKind) -> str:
    return {CodeKind.XOR: "xor", CodeKind.RDP: "rdp", CodeKind.REED_SOLOMON: "rs"}.get(kind, "?")


@dataclass(frozen=True)
class CodingScheme:
    kind: CodeKind = CodeKind.XOR
    n: int = 1
    k: int = 1

    def validate(self) -> None:
        check(L.lib().gs_scheme_validate(int(self.kind), self.n, self.k))

    @staticmethod
    def xor_code(n: int) -> "CodingScheme":
        return CodingScheme(CodeKind.XOR, n, 1)

    @staticmethod
    def rdp(n: int) -> "CodingScheme":
        return CodingScheme(CodeKind.RDP, n, 2)

    @staticmethod
    def reed_solomon(n: int, k: int) -> "CodingScheme":
        return CodingScheme(CodeKind.REED_SOLOMON, n, k)


def max_tolerance(s: CodingScheme) -> int:
    return int(L.lib().gs_max_tolerance(int(s.kind), s.n, s.k))


def memory_overhead_ratio(s: CodingScheme) -> float:
    return float(s.k) / float(s.n)


@dataclass
class EncodingMatrix:
    rows: int
    cols: int
    coef: np.ndarray  # uint8, row-major rows x cols

    def at(self, r: int, c: int) -> int:
        return int(self.coef[r * self.cols + c])


def build_encoding_matrix(s: CodingScheme) -> EncodingMatrix:
    out = np.zeros(max(s.k * s.n, 1), np.uint8)
    check(L.lib().gs_encoding_matrix(int(s.kind), s.n, s.k, out.ctypes.data_as(L._u8p)),
          "build_encoding_matrix")
    return EncodingMatrix(s.k, s.n, out[: s.k * s.n])


class ErasurePattern:
    """Sorted, de-duplicated lost shard indices (coding.hpp:128-137)."""

    def __init__(self, indices: Sequence[int] = ()):
        self.lost: List[int] = sorted(set(int(i) for i in indices))

    def contains(self, idx: int) -> bool:
        return idx in self.lost

    def __repr__(self) -> str:
        return f"ErasurePattern({self.lost})"


# ---------------------------------------------------------------------------
# gf256 (gf256.hpp:38-61)
# ---------------------------------------------------------------------------
class gf256:  # noqa: N801  (namespace mirror)
    @staticmethod
    def add(a: int, b: int) -> int:
        return (a ^ b) & 0xFF

    @staticmethod
    def mul(a: int, b: int) -> int:
        return int(L.lib().gs_gf_mul(a, b))

    @staticmethod
    def inv(a: int) -> int:
        out = C.c_uint8()
        check(L.lib().gs_gf_inv(a, C.byref(out)), "gf256")
        return out.value

    @staticmethod
    def div(a: int, b: int) -> int:
        out = C.c_uint8()
        check(L.lib().gs_gf_div(a, b, C.byref(out)), "gf256")
        return out.value


# ---------------------------------------------------------------------------
# codec objects (cached per scheme / pattern)
# ---------------------------------------------------------------------------
class Codec:
    """Owns a gs_codec (encoder, or decoder for one erasure pattern)."""

    def __init__(self, handle: int):
        self.handle = handle
        n_out, n_slots, spec = C.c_int(), C.c_int(), C.c_int()
        idx = (C.c_int * 256)()
        check(L.lib().gs_codec_info(handle, C.byref(n_out), idx, C.byref(n_slots), C.byref(spec)))
        self.n_out = n_out.value
        self.n_slots = n_slots.value
        self.out_index = [idx[i] for i in range(self.n_out)]
        self.specialised = bool(spec.value)

    def coefficients(self) -> np.ndarray:
        out = np.zeros(max(self.n_out * self.n_slots, 1), np.uint8)
        check(L.lib().gs_codec_coefficients(self.handle, out.ctypes.data_as(L._u8p)))
        return out[: self.n_out * self.n_slots].reshape(self.n_out, self.n_slots)

    def __del__(self):
        try:
            if self.handle:
                L.lib().gs_codec_destroy(self.handle)
        except Exception:
            pass


_codec_cache: Dict[tuple, Codec] = {}
_cache_lock = threading.Lock()


def encoder(scheme: CodingScheme) -> Codec:
    key = ("enc", int(scheme.kind), scheme.n, scheme.k)
    with _cache_lock:
        c = _codec_cache.get(key)
        if c is None:
            h = C.c_void_p()
            check(L.lib().gs_encoder_create(int(scheme.kind), scheme.n, scheme.k, C.byref(h)),
                  "encode")
            c = _codec_cache[key] = Codec(h.value)
        return c


def decoder(scheme: CodingScheme, lost: ErasurePattern) -> Codec:
    key = ("dec", int(scheme.kind), scheme.n, scheme.k, tuple(lost.lost))
    with _cache_lock:
        c = _codec_cache.get(key)
        if c is None:
            h = C.c_void_p()
            arr = (C.c_int * max(len(lost.lost), 1))(*lost.lost)
            check(L.lib().gs_decoder_create(int(scheme.kind), scheme.n, scheme.k, arr,
                                            len(lost.lost), C.byref(h)), "reconstruct")
            c = _codec_cache[key] = Codec(h.value)
        return c


def codec_ex(scheme: CodingScheme, lost: Optional[ErasurePattern] = None,
             generic: bool = False) -> Codec:
    """Uncached codec with explicit back-end choice (tests / benchmarks)."""
    h = C.c_void_p()
    lst = lost.lost if lost is not None else []
    arr = (C.c_int * max(len(lst), 1))(*lst)
    flags = (1 if generic else 0) | (2 if lost is not None else 0)
    check(L.lib().gs_codec_create_ex(int(scheme.kind), scheme.n, scheme.k, arr, len(lst), flags,
                                     C.byref(h)), "codec")
    return Codec(h.value)


class Pipeline:
    """Per-device staging ring for the host-link pipelined calls."""

    def __init__(self, device: int = 0, staging_bytes: int = 128 << 20):
        h = C.c_void_p()
        check(L.lib().gs_pipeline_create(device, staging_bytes, C.byref(h)), "pipeline")
        self.handle = h.value
        self.device = device

    def __del__(self):
        try:
            if self.handle:
                L.lib().gs_pipeline_destroy(self.handle)
        except Exception:
            pass


_pipes: Dict[int, Pipeline] = {}


def default_pipeline(device: Optional[int] = None) -> Pipeline:
    if device is None:
        device = 0
    with _cache_lock:
        p = _pipes.get(device)
        if p is None:
            if not L.lib().gs_cuda_available():
                raise CudaError("no CUDA device: the GPU codec has no CPU fallback")
            p = _pipes[device] = Pipeline(device)
        return p


def _as_u8(buf) -> np.ndarray:
    a = np.frombuffer(buf, dtype=np.uint8) if not isinstance(buf, np.ndarray) else buf
    if a.dtype != np.uint8:
        a = a.view(np.uint8)
    return np.ascontiguousarray(a.reshape(-1))


# ---------------------------------------------------------------------------
# encode / reconstruct (coding.hpp:313-336, 458-571)
# ---------------------------------------------------------------------------
def encode(scheme: CodingScheme, data: Sequence, *, device: Optional[int] = None) -> List[np.ndarray]:
    """k parity shards of n equal-length data shards (host in, host out)."""
    scheme.validate()
    if len(data) != scheme.n:
        raise InvalidArgument(f"coding: expected {scheme.n} data shards, got {len(data)}")
    bufs = [_as_u8(d) for d in data]
    ln = bufs[0].size if bufs else 0
    if any(b.size != ln for b in bufs):
        raise InvalidArgument("coding: shard buffers must all have the same length")
    enc = encoder(scheme)
    parity = [np.zeros(ln, np.uint8) for _ in range(scheme.k)]
    if ln:
        check(L.lib().gs_encode_host(default_pipeline(device).handle, enc.handle,
                                     L.ptr_array([b.ctypes.data for b in bufs]),
                                     L.ptr_array([p.ctypes.data for p in parity]), ln), "encode")
    return parity


def reconstruct(scheme: CodingScheme, surviving: Mapping[int, object], lost: ErasurePattern,
                *, device: Optional[int] = None) -> Dict[int, np.ndarray]:
    """Rebuild the lost DATA shards from the survivors (host in, host out)."""
    scheme.validate()
    total = scheme.n + scheme.k
    for idx in lost.lost:
        if idx < 0 or idx >= total:
            raise InvalidArgument("coding: lost shard index out of range")
    if len(lost.lost) > max_tolerance(scheme):
        raise UnrecoverableError(
            f"coding: {len(lost.lost)} erasures exceed tolerance {max_tolerance(scheme)} for "
            f"scheme {to_string(scheme.kind)}")
    ln = None
    slots: List[Optional[np.ndarray]] = [None] * total
    for idx in range(total):
        if lost.contains(idx):
            continue
        if idx not in surviving:
            raise InvalidArgument(f"coding: surviving shard {idx} missing from input")
        b = _as_u8(surviving[idx])
        if ln is None:
            ln = b.size
        elif b.size != ln:
            raise InvalidArgument("coding: shard buffers must all have the same length")
        slots[idx] = b
    ln = ln or 0
    dec = decoder(scheme, lost)
    out = {idx: np.zeros(ln, np.uint8) for idx in dec.out_index}
    if ln and dec.n_out:
        check(L.lib().gs_reconstruct_host(
            default_pipeline(device).handle, dec.handle,
            L.ptr_array([None if s is None else s.ctypes.data for s in slots]),
            L.ptr_array([out[i].ctypes.data for i in dec.out_index]), ln), "reconstruct")
    return out
