"""Host tier: mirror of parity_store.hpp over the native gs_store.

``ParityChunk`` / ``ParityStore`` / ``ParityGetStatus`` / ``fnv1a64`` /
``serialize_parity_store`` / ``deserialize_parity_store`` keep the
reference's names, accounting (payload + 64 B per entry), back-pressure
(``try_put`` returns False, store unchanged), duplicate handling
(``LogicError``), ``get`` verification (kOk / kMissing / kCorrupt) and GSRV
byte format. Storage is pinned host memory owned by the native store:
parity arrays returned by ``get`` are zero-copy numpy views of it, and the
checkpoint path (``reserve`` -> D2H -> ``commit``) writes into it directly
with the FNV seal done by native worker threads.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from .coding import CodeKind, CodingScheme, InvalidArgument, check

FNV_OFFSET = 0xCBF29CE484222325
K_PER_ENTRY_METADATA_BYTES = 64
UNLIMITED = (1 << 64) - 1


def fnv1a64(buf, h: int = FNV_OFFSET) -> int:
    """parity_store.hpp:19-25"""
    a = np.ascontiguousarray(np.frombuffer(buf, np.uint8) if not isinstance(buf, np.ndarray) else buf)
    return int(L.lib().gs_fnv1a64(a.ctypes.data, a.nbytes, h))


class ParityGetStatus(enum.IntEnum):
    kOk = 0
    kMissing = 1
    kCorrupt = 2


@dataclass
class ParityChunk:
    """parity_store.hpp:31-53"""

    request_id: int = 0
    chunk_id: int = 0
    scheme: CodingScheme = field(default_factory=CodingScheme)
    parity: List[np.ndarray] = field(default_factory=list)
    valid_tokens: int = 0
    slice_len: int = 0
    checksum: int = 0

    def payload_present(self) -> bool:
        return len(self.parity) > 0

    def payload_bytes(self) -> int:
        return self.scheme.k * self.slice_len

    def compute_checksum(self) -> int:
        h = FNV_OFFSET
        for p in self.parity:
            h = fnv1a64(p, h)
        return h

    def seal(self) -> None:
        self.checksum = self.compute_checksum()


def _view(ptr: int, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0, np.uint8)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), (n,))


class ParityStore:
    """parity_store.hpp:62-143 on pinned slabs (native gs_store)."""

    kPerEntryMetadataBytes = K_PER_ENTRY_METADATA_BYTES
    kUnlimited = UNLIMITED

    def __init__(self, capacity_bytes: int = UNLIMITED, seal_threads: int = 4, _handle: Optional[int] = None):
        if _handle is None:
            h = C.c_void_p()
            check(L.lib().gs_store_create(capacity_bytes, seal_threads, C.byref(h)), "parity store")
            _handle = h.value
        self.handle = _handle

    def bind_device(self, device: int) -> None:
        """Place future pinned slabs on `device`'s NUMA node (gs_store_bind_device)."""
        check(L.lib().gs_store_bind_device(self.handle, device), "parity store")

    def close(self) -> None:
        if self.handle:
            L.lib().gs_store_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- accounting -------------------------------------------------------
    def _stats(self) -> Tuple[int, int, int, int, int]:
        out = (C.c_uint64 * 5)()
        check(L.lib().gs_store_stats(self.handle, out), "parity store")
        return tuple(int(x) for x in out)  # type: ignore[return-value]

    def used_bytes(self) -> int:
        return self._stats()[0]

    def capacity_bytes(self) -> int:
        return self._stats()[1]

    def payload_bytes(self) -> int:
        return self._stats()[2]

    def peak_payload_bytes(self) -> int:
        return self._stats()[3]

    def entry_count(self) -> int:
        return self._stats()[4]

    def audit(self) -> bool:
        return bool(L.lib().gs_store_audit(self.handle))

    # ---- put / get --------------------------------------------------------
    def try_put(self, chunk: ParityChunk) -> bool:
        """Copying put (reference semantics). False = back-pressure."""
        s = chunk.scheme
        bufs = [np.ascontiguousarray(p, dtype=np.uint8) for p in chunk.parity]
        if bufs and any(b.size != chunk.slice_len for b in bufs):
            raise InvalidArgument("parity store: parity buffers must be slice_len bytes")
        acc = C.c_int()
        # no payload: a cost-only entry (KvPolicy::materialize = false), accounted but holding no bytes
        check(L.lib().gs_store_put(self.handle, chunk.request_id, chunk.chunk_id, int(s.kind), s.n, s.k,
                                   chunk.valid_tokens, chunk.slice_len,
                                   L.ptr_array([b.ctypes.data for b in bufs]) if bufs else None, chunk.checksum, 1,
                                   C.byref(acc)), "parity store")
        return bool(acc.value)

    def reserve(self, request_id: int, chunk_id: int, scheme: CodingScheme, valid_tokens: int,
                slice_len: int) -> Optional[List[int]]:
        """Reserve an entry; returns the k pinned destination pointers for the
        D2H of the encode kernel, or None on back-pressure."""
        acc = C.c_int()
        ptrs = (C.c_void_p * max(scheme.k, 1))()
        check(L.lib().gs_store_reserve(self.handle, request_id, chunk_id, int(scheme.kind), scheme.n, scheme.k,
                                       valid_tokens, slice_len, C.byref(acc), ptrs), "parity store")
        if not acc.value:
            return None
        return [ptrs[i] for i in range(scheme.k)]

    def reserve_batch(self, keys, scheme: CodingScheme, valid_tokens: int, slice_len: int):
        """Reserve [(request, chunk), ...] at once; returns (accepted count,
        flat list of pinned parity pointers, k per accepted entry)."""
        n = len(keys)
        req = (C.c_uint64 * max(n, 1))(*[r for r, _ in keys])
        chk = (C.c_uint32 * max(n, 1))(*[c for _, c in keys])
        acc = C.c_int()
        ptrs = (C.c_void_p * max(n * scheme.k, 1))()
        check(L.lib().gs_store_reserve_batch(self.handle, n, req, chk, int(scheme.kind), scheme.n, scheme.k,
                                             valid_tokens, slice_len, C.byref(acc), ptrs), "parity store")
        return acc.value, [ptrs[i] for i in range(acc.value * scheme.k)]

    def commit_batch(self, keys, stream=None) -> None:
        """Seal many entries once `stream` reaches this point (one callback)."""
        n = len(keys)
        req = (C.c_uint64 * max(n, 1))(*[r for r, _ in keys])
        chk = (C.c_uint32 * max(n, 1))(*[c for _, c in keys])
        st = None if stream is None else int(getattr(stream, "cuda_stream", stream))
        check(L.lib().gs_store_commit_batch(self.handle, n, req, chk, st), "parity store")

    def commit_sealed_batch(self, keys, checksums_ptr: int, stream=None) -> None:
        """Seal entries with checksums computed on the GPU (pinned uint64
        array at `checksums_ptr`, read when `stream` reaches this point)."""
        n = len(keys)
        req = (C.c_uint64 * max(n, 1))(*[r for r, _ in keys])
        chk = (C.c_uint32 * max(n, 1))(*[c for _, c in keys])
        st = None if stream is None else int(getattr(stream, "cuda_stream", stream))
        check(L.lib().gs_store_commit_sealed_batch(self.handle, n, req, chk, checksums_ptr, st), "parity store")

    def commit(self, request_id: int, chunk_id: int, stream=None) -> None:
        """Seal once `stream` (the copy stream of the D2H) reaches this point."""
        st = None if stream is None else int(getattr(stream, "cuda_stream", stream))
        check(L.lib().gs_store_commit(self.handle, request_id, chunk_id, st), "parity store")

    def wait_sealed(self) -> None:
        L.lib().gs_store_wait_sealed(self.handle)

    def get(self, request_id: int, chunk_index: int, verify: bool = True, copy: bool = False
            ) -> Tuple[ParityGetStatus, Optional[ParityChunk]]:
        """parity_store.hpp:92-101. The returned parity arrays are zero-copy
        views of the store's pinned slab (what the recovery H2D reads): they
        are valid until the entry is erased (erase_request recycles the block)
        or the store is closed; the chunk keeps the store object alive, not
        the entry. copy=True returns owning copies instead."""
        st = C.c_int()
        ptrs = (C.c_void_p * 256)()
        sl, ck = C.c_uint64(), C.c_uint64()
        vt = C.c_uint32()
        knk = (C.c_int * 3)()
        check(L.lib().gs_store_get(self.handle, request_id, chunk_index, 1 if verify else 0, C.byref(st), ptrs,
                                   C.byref(sl), C.byref(vt), C.byref(ck), knk), "parity store")
        status = ParityGetStatus(st.value)
        if status != ParityGetStatus.kOk:
            return status, None
        scheme = CodingScheme(CodeKind(knk[0]), knk[1], knk[2])
        parity = [_view(ptrs[i], sl.value) for i in range(scheme.k)] if ptrs[0] else []   # [] = cost-only
        if copy:
            parity = [p.copy() for p in parity]
        chunk = ParityChunk(request_id, chunk_index, scheme, parity, vt.value, sl.value, ck.value)
        if not copy:
            chunk._store = self   # the views point into this store's slabs
        return status, chunk

    def contains(self, request_id: int, chunk_index: int) -> bool:
        return bool(L.lib().gs_store_contains(self.handle, request_id, chunk_index))

    def erase_request(self, request_id: int) -> None:
        check(L.lib().gs_store_erase_request(self.handle, request_id), "parity store")

    def corrupt_entry(self, request_id: int, chunk_index: int) -> None:
        """Test hook (parity_store.hpp:126-131)."""
        L.lib().gs_store_corrupt_entry(self.handle, request_id, chunk_index)

    def keys(self) -> List[Tuple[int, int]]:
        cnt = C.c_uint64()
        check(L.lib().gs_store_keys(self.handle, None, 0, C.byref(cnt)), "parity store")
        arr = (C.c_uint64 * max(2 * cnt.value, 1))()
        check(L.lib().gs_store_keys(self.handle, arr, cnt.value, C.byref(cnt)), "parity store")
        return [(int(arr[2 * i]), int(arr[2 * i + 1])) for i in range(cnt.value)]


def serialize_parity_store(store: ParityStore) -> bytes:
    """parity_store.hpp:167-191 (GSRV)."""
    size = C.c_uint64()
    check(L.lib().gs_store_serialize(store.handle, None, 0, C.byref(size)), "serialize")
    buf = np.zeros(size.value, np.uint8)
    check(L.lib().gs_store_serialize(store.handle, buf.ctypes.data, size.value, C.byref(size)), "serialize")
    return buf.tobytes()


def deserialize_parity_store(data: bytes, capacity_bytes: int = UNLIMITED, seal_threads: int = 4) -> ParityStore:
    """parity_store.hpp:193-229 (GSRV); ParityFileError on bad/truncated/corrupt files."""
    arr = np.frombuffer(data, np.uint8)
    h = C.c_void_p()
    check(L.lib().gs_store_deserialize(arr.ctypes.data if arr.size else None, arr.size, capacity_bytes,
                                       seal_threads, C.byref(h)), "deserialize")
    return ParityStore(_handle=h.value)
