"""TEST INFRASTRUCTURE ONLY -- ctypes view of the CPU oracle.

Two libraries, same call shapes:
  * ``port()``  -> oracle/build/libgs_oracle.so, our plain-C restatement
    (oracle/gs_oracle.c) of the reference byte path;
  * ``ref()``   -> oracle/_ref/libghostserve_ref.so, the reference headers
    compiled in place (oracle/ref_shim.cpp); present wherever `make -C oracle`
    ran with /root/reference mounted (it travels to the GPU box prebuilt).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module. The product path (paper_2605_00831_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "libgs_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libghostserve_ref.so")

XOR, RDP, RS = 0, 1, 2
OK, INVALID_ARGUMENT, UNRECOVERABLE, DOMAIN_ERROR = 0, 1, 2, 3

_u8p = C.POINTER(C.c_uint8)


class OracleError(Exception):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: status {status}")
        self.status = status


def _ptrs(arrs: Sequence[Optional[np.ndarray]]):
    out = (C.c_void_p * len(arrs))()
    for i, a in enumerate(arrs):
        out[i] = None if a is None else a.ctypes.data
    return out


def _check(st: int, what: str) -> None:
    if st != OK:
        raise OracleError(st, what)


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        self.path = path
        self.lib = C.CDLL(path)
        self.p = prefix

    def fn(self, name):
        return getattr(self.lib, self.p + name)

    # --- GF(2^8) --------------------------------------------------------
    def gf_mul(self, a: int, b: int) -> int:
        f = self.fn("gf_mul")
        f.restype = C.c_uint8
        return int(f(C.c_uint8(a), C.c_uint8(b)))

    def gf_inv(self, a: int) -> int:
        out = C.c_uint8()
        _check(self.fn("gf_inv")(C.c_uint8(a), C.byref(out)), "gf_inv")
        return out.value

    def gf_tables(self):
        e = np.zeros(512, np.uint8)
        lg = np.zeros(256, np.uint8)
        self.fn("gf_tables")(e.ctypes.data_as(_u8p), lg.ctypes.data_as(_u8p))
        return e, lg

    def encoding_matrix(self, kind: int, n: int, k: int) -> np.ndarray:
        out = np.zeros(k * n, np.uint8)
        _check(self.fn("encoding_matrix")(kind, n, k, out.ctypes.data_as(_u8p)), "encoding_matrix")
        return out.reshape(k, n)

    # --- codec ----------------------------------------------------------
    def encode(self, kind: int, n: int, k: int, data: Sequence[np.ndarray]) -> List[np.ndarray]:
        if len(data) != n:
            raise OracleError(INVALID_ARGUMENT, "encode: wrong shard count")
        ln = int(data[0].size) if n else 0
        data = [np.ascontiguousarray(d, dtype=np.uint8) for d in data]
        par = [np.zeros(max(ln, 1), np.uint8) for _ in range(k)]
        f = self.fn("encode")
        args = [kind, n, k, _ptrs(data), C.c_size_t(ln), _ptrs(par)]
        if self.p == "ghs_":
            args.append(None)
        _check(f(*args), "encode")
        return [p[:ln] for p in par]

    def reconstruct(self, kind: int, n: int, k: int, shards: Dict[int, np.ndarray],
                    lost: Sequence[int]) -> Dict[int, np.ndarray]:
        ln = None
        arr: List[Optional[np.ndarray]] = [None] * (n + k)
        for idx, buf in shards.items():
            if 0 <= idx < n + k and idx not in lost:
                arr[idx] = np.ascontiguousarray(buf, dtype=np.uint8)
                ln = buf.size
        ln = ln or 0
        lost_data = sorted({i for i in lost if 0 <= i < n})
        outs = [np.zeros(max(ln, 1), np.uint8) for _ in range(max(len(lost_data), 1))]
        lost_arr = (C.c_int * max(len(lost), 1))(*lost)
        n_out = C.c_int(0)
        args = [kind, n, k, _ptrs(arr), lost_arr, len(lost), C.c_size_t(ln), _ptrs(outs),
                C.byref(n_out)]
        if self.p == "ghs_":
            args.append(None)
        _check(self.fn("reconstruct")(*args), "reconstruct")
        return {lost_data[b]: outs[b][:ln] for b in range(n_out.value)}

    # --- KV layout / seal -----------------------------------------------
    def slice_bytes(self, layers, kv_heads, head_dim, tp, chunk_size) -> int:
        out = C.c_uint64()
        _check(self.fn("slice_bytes")(layers, kv_heads, head_dim, tp, C.c_uint32(chunk_size),
                                      C.byref(out)), "slice_bytes")
        return out.value

    def make_ground_truth_slice(self, seed, req, chunk, worker, layers, kv_heads, head_dim, tp,
                                chunk_size, valid) -> np.ndarray:
        ln = self.slice_bytes(layers, kv_heads, head_dim, tp, chunk_size)
        out = np.zeros(max(ln, 1), np.uint8)
        _check(self.fn("make_ground_truth_slice")(
            C.c_uint64(seed), C.c_uint64(req), C.c_uint32(chunk), worker, layers, kv_heads,
            head_dim, tp, C.c_uint32(chunk_size), C.c_uint32(valid), out.ctypes.data_as(_u8p)),
            "make_ground_truth_slice")
        return out[:ln]

    def fnv1a64(self, buf: np.ndarray, h: int = 0xCBF29CE484222325) -> int:
        f = self.fn("fnv1a64")
        f.restype = C.c_uint64
        buf = np.ascontiguousarray(buf, dtype=np.uint8)
        return int(f(buf.ctypes.data_as(_u8p), C.c_size_t(buf.size), C.c_uint64(h)))

    def parity_checksum(self, parity: Sequence[np.ndarray]) -> int:
        h = 0xCBF29CE484222325
        for p in parity:
            h = self.fnv1a64(p, h)
        return h


class _Port(_Lib):
    def __init__(self):
        super().__init__(PORT_SO, "gso_")

    def decode_matrix(self, kind, n, k, lost):
        cd = np.zeros(255 * n, np.uint8)
        cp = np.zeros(255 * k, np.uint8)
        e = C.c_int(0)
        lost_arr = (C.c_int * max(len(lost), 1))(*lost)
        _check(self.fn("decode_matrix")(kind, n, k, lost_arr, len(lost),
                                        cd.ctypes.data_as(_u8p), cp.ctypes.data_as(_u8p),
                                        C.byref(e)), "decode_matrix")
        return cd[: e.value * n].reshape(e.value, n), cp[: e.value * k].reshape(e.value, k)


class _Ref(_Lib):
    def __init__(self):
        super().__init__(REF_SO, "ghs_")

    def mul_table(self) -> np.ndarray:
        out = np.zeros(65536, np.uint8)
        self.fn("mul_table")(out.ctypes.data_as(_u8p))
        return out.reshape(256, 256)

    def encode_timed(self, kind, n, k, data, parity, threads: int = 1) -> float:
        """Reference encode into preallocated parity; returns seconds (bench convention)."""
        secs = C.c_double(0)
        ln = int(data[0].size)
        if threads <= 1:
            st = self.fn("encode")(kind, n, k, _ptrs(data), C.c_size_t(ln), _ptrs(parity),
                                   C.byref(secs))
        else:
            st = self.fn("encode_striped")(kind, n, k, _ptrs(data), C.c_size_t(ln),
                                           _ptrs(parity), threads, C.byref(secs))
        _check(st, "encode")
        return secs.value

    def encode_batch_timed(self, kind, n, k, stripes, parities, threads: int) -> float:
        """stripes[s] = n data arrays, parities[s] = k outputs; T threads over stripes."""
        secs = C.c_double(0)
        ln = int(stripes[0][0].size)
        st = self.fn("encode_batch")(kind, n, k, len(stripes), _ptrs([d for row in stripes for d in row]),
                                     C.c_size_t(ln), _ptrs([p for row in parities for p in row]), threads,
                                     C.byref(secs))
        _check(st, "encode_batch")
        return secs.value

    def reconstruct_timed(self, kind, n, k, shards: List[Optional[np.ndarray]], lost, outs,
                          threads: int = 1) -> float:
        secs = C.c_double(0)
        ln = int(next(s for s in shards if s is not None).size)
        lost_arr = (C.c_int * len(lost))(*lost)
        n_out = C.c_int(0)
        if threads <= 1:
            st = self.fn("reconstruct")(kind, n, k, _ptrs(shards), lost_arr, len(lost),
                                        C.c_size_t(ln), _ptrs(outs), C.byref(n_out),
                                        C.byref(secs))
        else:
            st = self.fn("reconstruct_striped")(kind, n, k, _ptrs(shards), lost_arr, len(lost),
                                                C.c_size_t(ln), _ptrs(outs), C.byref(n_out),
                                                threads, C.byref(secs))
        _check(st, "reconstruct")
        return secs.value

    def checkpoint_chunk_timed(self, kind, n, k, model, chunk_size, req, chunk, valid, data, parity):
        """The reference checkpoint_chunk (encode + seal) on one chunk's n
        slices; model = (layers, kv_heads, head_dim). Returns (checksum, s)."""
        secs, cs = C.c_double(0), C.c_uint64(0)
        st = self.fn("checkpoint_chunk_timed")(kind, n, k, *model, C.c_uint32(chunk_size), C.c_uint64(req),
                                                C.c_uint32(chunk), C.c_uint32(valid), _ptrs(data), _ptrs(parity),
                                                C.byref(cs), C.byref(secs))
        _check(st, "checkpoint_chunk")
        return cs.value, secs.value

    def reconstruct_chunk_timed(self, kind, n, k, slots: List[Optional[np.ndarray]], outs, sealed: int = 0) -> float:
        """The reference reconstruct_chunk (FNV verify + reconstruct): slots =
        n data + k parity arrays, None = lost; rebuilt data -> outs; sealed =
        the checkpoint-time checksum (0: seal the given parity)."""
        secs, n_out = C.c_double(0), C.c_int(0)
        ln = int(next(s for s in slots if s is not None).size)
        st = self.fn("reconstruct_chunk_timed")(kind, n, k, C.c_uint64(ln), _ptrs(slots),
                                                 C.c_uint64(sealed), _ptrs(outs), C.byref(n_out), C.byref(secs))
        _check(st, "reconstruct_chunk")
        return secs.value


_port = None
_ref = None


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def have_ref() -> bool:
    return os.path.exists(REF_SO)
