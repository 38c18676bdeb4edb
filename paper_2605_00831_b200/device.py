"""Device-resident API: K1 / K2 on torch CUDA tensors, plus the host-link
pipelines (checkpoint offload, recovery upload).

torch is plumbing here (device memory, streams, pinned host memory); the
bytes are produced by libghostserve_b200.so kernels. Tensors are uint8 and
contiguous in their last dimension; shapes:

  encode   data  [n, L] | [S, n, L]   -> parity [k, L] | [S, k, L]
  rebuild  shards {idx: [L] | [S, L]} -> {lost data idx: [L] | [S, L]}

where S is the number of independent stripes (requests x chunks) launched
together -- e.g. the 32 requests of a decode block, or the 64 chunks of a
128K prefill.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Mapping, Optional, Sequence, Union

import torch

from . import _lib as L
from .coding import (CodingScheme, Codec, ErasurePattern, InvalidArgument, UnrecoverableError,
                     check, decoder, encoder, max_tolerance, to_string)

Tensor = torch.Tensor


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _check_u8(t: Tensor, what: str) -> None:
    if t.dtype != torch.uint8:
        raise InvalidArgument(f"{what}: expected a uint8 tensor (view fp16/bf16 KV as bytes), got {t.dtype}")
    if not t.is_cuda:
        raise InvalidArgument(f"{what}: expected a CUDA tensor")
    if t.stride(-1) != 1:
        raise InvalidArgument(f"{what}: last dimension must be contiguous")


def row_ptrs(t: Tensor) -> List[int]:
    """Addresses of the rows of a [R, L] or [S, R, L] tensor, stripe-major,
    by stride arithmetic (indexing each row costs ~1 us of Python per row)."""
    base, es = t.data_ptr(), t.element_size()
    if t.dim() == 1:
        return [base]
    if t.dim() == 2:
        s1 = t.stride(0) * es
        return [base + r * s1 for r in range(t.shape[0])]
    if t.dim() != 3:
        raise InvalidArgument(f"expected a 2-D or 3-D tensor, got shape {tuple(t.shape)}")
    s0, s1 = t.stride(0) * es, t.stride(1) * es
    R = t.shape[1]
    return [base + s * s0 + r * s1 for s in range(t.shape[0]) for r in range(R)]


def as_bytes(t: Tensor) -> Tensor:
    """Bit-for-bit byte view of an fp16/bf16 (or any) tensor: fp16.hpp:20-21."""
    return t.contiguous().view(torch.uint8)


def apply(codec: Codec, slots: Sequence[Sequence[Optional[int]]], outs: Sequence[Sequence[int]],
          length: int, stream=None) -> None:
    """Raw launch: per-stripe lists of device pointers (gs_apply_device)."""
    flat_s = [p for row in slots for p in row]
    flat_o = [p for row in outs for p in row]
    check(L.lib().gs_apply_device(codec.handle, len(slots), L.ptr_array(flat_s), L.ptr_array(flat_o),
                                  length, _stream(stream)), "apply")


def encode(scheme: CodingScheme, data: Union[Tensor, Sequence[Tensor]], out: Optional[Tensor] = None,
           stream=None) -> Tensor:
    """K1 on device: parity of n data shards (or of S stripes of n shards)."""
    scheme.validate()
    if not isinstance(data, Tensor):
        shards = list(data)
        if len(shards) != scheme.n:
            raise InvalidArgument(f"coding: expected {scheme.n} data shards, got {len(shards)}")
        ln = shards[0].numel() * shards[0].element_size()
        for t in shards:
            if t.numel() * t.element_size() != ln:
                raise InvalidArgument("coding: shard buffers must all have the same length")
            _check_u8(t, "encode")
        if out is None:
            out = torch.empty((scheme.k, ln), dtype=torch.uint8, device=shards[0].device)
        apply(encoder(scheme), [[t.data_ptr() for t in shards]],
              [[out[i].data_ptr() for i in range(scheme.k)]], ln, stream)
        return out
    _check_u8(data, "encode")
    single = data.dim() == 2
    d3 = data.unsqueeze(0) if single else data
    if d3.dim() != 3 or d3.shape[1] != scheme.n:
        raise InvalidArgument(f"coding: expected data of shape [n={scheme.n}, L] or [S, n, L], got "
                              f"{tuple(data.shape)}")
    S, _, ln = d3.shape
    if out is None:
        out = torch.empty((S, scheme.k, ln) if not single else (scheme.k, ln), dtype=torch.uint8,
                          device=data.device)
    o3 = out.unsqueeze(0) if single else out
    _check_u8(o3, "encode(out)")
    dp, op = row_ptrs(d3), row_ptrs(o3)
    n, k = scheme.n, scheme.k
    slots = [dp[s * n:(s + 1) * n] for s in range(S)]
    outs = [op[s * k:(s + 1) * k] for s in range(S)]
    apply(encoder(scheme), slots, outs, ln, stream)
    return out


def reconstruct(scheme: CodingScheme, shards: Mapping[int, Tensor], lost: ErasurePattern,
                out: Optional[Mapping[int, Tensor]] = None, stream=None) -> Dict[int, Tensor]:
    """K2 on device: rebuild lost data shards from surviving device shards."""
    scheme.validate()
    total = scheme.n + scheme.k
    for idx in lost.lost:
        if idx < 0 or idx >= total:
            raise InvalidArgument("coding: lost shard index out of range")
    if len(lost.lost) > max_tolerance(scheme):
        raise UnrecoverableError(f"coding: {len(lost.lost)} erasures exceed tolerance "
                                 f"{max_tolerance(scheme)} for scheme {to_string(scheme.kind)}")
    shape = None
    for idx in range(total):
        if lost.contains(idx):
            continue
        if idx not in shards:
            raise InvalidArgument(f"coding: surviving shard {idx} missing from input")
        t = shards[idx]
        _check_u8(t, "reconstruct")
        if shape is None:
            shape = tuple(t.shape)
        elif tuple(t.shape) != shape:
            raise InvalidArgument("coding: shard buffers must all have the same length")
    dec = decoder(scheme, lost)
    ref = next(shards[i] for i in range(total) if not lost.contains(i))
    res = dict(out) if out is not None else {i: torch.empty(shape, dtype=torch.uint8, device=ref.device)
                                              for i in dec.out_index}
    if dec.n_out == 0 or ref.numel() == 0:
        return res
    batched = len(shape) == 2
    S = shape[0] if batched else 1
    ln = shape[-1]

    rows = {j: row_ptrs(shards[j]) for j in range(total) if not lost.contains(j)}
    rows.update({i: row_ptrs(res[i]) for i in dec.out_index})
    slots = [[None if lost.contains(j) else rows[j][s] for j in range(total)] for s in range(S)]
    outs = [[rows[i][s] for i in dec.out_index] for s in range(S)]
    apply(dec, slots, outs, ln, stream)
    return res


# ---------------------------------------------------------------------------
# host-link pipelines
# ---------------------------------------------------------------------------
class Pipeline:
    """Staging ring on one device for encode->D2H and H2D->rebuild overlap."""

    def __init__(self, device: int = 0, staging_bytes: int = 256 << 20):
        h = C.c_void_p()
        check(L.lib().gs_pipeline_create(device, staging_bytes, C.byref(h)), "pipeline")
        self.handle = h.value
        self.device = device

    def close(self) -> None:
        if self.handle:
            L.lib().gs_pipeline_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def encode_offload(self, scheme: CodingScheme, data: Tensor, h_parity: Tensor,
                       compute=None, copy=None) -> None:
        """Encode [S, n, L] device data; parity lands in pinned host [S, k, L].

        Enqueue only: completion is the `copy` stream (default: compute)."""
        _check_u8(data, "encode_offload")
        if data.dim() == 2:
            data = data.unsqueeze(0)
        if h_parity.dim() == 2:
            h_parity = h_parity.unsqueeze(0)
        S, n, ln = data.shape
        if n != scheme.n or tuple(h_parity.shape) != (S, scheme.k, ln):
            raise InvalidArgument("encode_offload: shape mismatch")
        if h_parity.is_cuda or not h_parity.is_pinned():
            raise InvalidArgument("encode_offload: parity must be a pinned host tensor")
        enc = encoder(scheme)
        d = L.ptr_array(row_ptrs(data))
        h = L.ptr_array(row_ptrs(h_parity))
        cs = _stream(compute)
        ks = _stream(copy) if copy is not None else cs
        check(L.lib().gs_encode_offload(self.handle, enc.handle, S, d, h, ln, cs, ks), "encode_offload")

    def reconstruct_upload(self, scheme: CodingScheme, lost: ErasurePattern,
                           data: Mapping[int, Tensor], h_parity: Tensor,
                           out: Mapping[int, Tensor], compute=None, copy=None) -> None:
        """Rebuild lost data shards: data[j] device [S, L] (surviving data
        shards, local or peer-mapped), h_parity pinned host [S, k, L],
        out[lost j] device [S, L]. Enqueue only: completion = `compute`."""
        dec = decoder(scheme, lost)
        if h_parity.dim() == 2:
            h_parity = h_parity.unsqueeze(0)
        S, k, ln = h_parity.shape
        if not h_parity.is_pinned():
            raise InvalidArgument("reconstruct_upload: parity must be a pinned host tensor")
        total = scheme.n + scheme.k
        rows = {j: row_ptrs(data[j]) for j in range(scheme.n) if not lost.contains(j)}
        hp = row_ptrs(h_parity)
        rows.update({scheme.n + i: hp[i::scheme.k] for i in range(scheme.k)})
        orows = {i: row_ptrs(out[i]) for i in dec.out_index}
        slots = [None if lost.contains(j) else rows[j][s] for s in range(S) for j in range(total)]
        outs = [orows[i][s] for s in range(S) for i in dec.out_index]
        cs = _stream(compute)
        ks = _stream(copy) if copy is not None else cs
        check(L.lib().gs_reconstruct_upload(self.handle, dec.handle, S, L.ptr_array(slots),
                                            L.ptr_array(outs), ln, cs, ks), "reconstruct_upload")


class CapturedCall:
    """One pipeline call (encode_offload or reconstruct_upload) recorded
    into a CUDA graph, replayed with one launch per decode block.

    The paper runs the checkpoint path under CUDA graphs:
    a block's encode kernels, ring waits and D2H pieces become one graph
    launch instead of ~2 API calls per piece. The graph owns a private
    Pipeline (its staging ring is baked into the graph), so eager calls on
    other pipelines never race it. Buffers are fixed at capture time; the
    caller refreshes their CONTENTS between replays (e.g. the serving
    engine's per-block KV slices and a fixed pinned parity buffer).
    """

    def __init__(self, method: str, *args, staging_bytes: int = 64 << 20, device: Optional[int] = None):
        dev = torch.cuda.current_device() if device is None else device
        self.pipe = Pipeline(dev, staging_bytes)
        self.stream = torch.cuda.Stream(dev)
        self.copy = torch.cuda.Stream(dev)
        call = getattr(self.pipe, method)
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        call(*args, compute=self.stream, copy=self.copy)        # eager warm-up: resolves kernels and occupancy
        self.stream.wait_stream(self.copy)
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            call(*args, compute=self.stream, copy=self.copy)    # the call forks `copy` off the capture
            self.stream.wait_stream(self.copy)                  # completion (offload: the copy stream) joins it

    def replay(self, stream=None) -> None:
        """Enqueue the recorded call; complete when `stream` (default: the
        current stream) reaches this point."""
        st = torch.cuda.current_stream() if stream is None else stream
        self.stream.wait_stream(st)
        with torch.cuda.stream(self.stream):
            self.graph.replay()
        st.wait_stream(self.stream)


def capture_offload(scheme: CodingScheme, data: Tensor, h_parity: Tensor, **kw) -> CapturedCall:
    """Graph of Pipeline.encode_offload(scheme, data, h_parity)."""
    return CapturedCall("encode_offload", scheme, data, h_parity, **kw)


def capture_upload(scheme: CodingScheme, lost: ErasurePattern, data: Mapping[int, Tensor], h_parity: Tensor,
                   out: Mapping[int, Tensor], **kw) -> CapturedCall:
    """Graph of Pipeline.reconstruct_upload(scheme, lost, data, h_parity, out)."""
    return CapturedCall("reconstruct_upload", scheme, lost, data, h_parity, out, **kw)


# ---------------------------------------------------------------------------
# NUMA-local pinned host memory
# ---------------------------------------------------------------------------
class _NearBuffer:
    """Owner of a gs_host_alloc_near allocation, exposed through the numpy
    array interface (the array keeps this object, and so the memory, alive)."""

    def __init__(self, device: int, nbytes: int):
        p = C.c_void_p()
        check(L.lib().gs_host_alloc_near(device, max(nbytes, 1), C.byref(p)), "host_alloc_near")
        self.ptr, self.nbytes = p.value, nbytes
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (self.ptr, False),
                                    "version": 3}

    def __del__(self):
        if getattr(self, "ptr", None):
            L.lib().gs_host_free(self.ptr)
            self.ptr = None


def pinned_near(shape, device: int = 0) -> Tensor:
    """uint8 CPU tensor in pinned memory on `device`'s NUMA node (the socket of
    its host link; plain pinned memory on single-node hosts)."""
    import math

    import numpy as np
    n = int(math.prod(shape)) if isinstance(shape, (tuple, list)) else int(shape)
    arr = np.asarray(_NearBuffer(device, n))
    return torch.from_numpy(arr).view(*(shape if isinstance(shape, (tuple, list)) else (shape,)))


def bind_local_cpus(device: int = 0) -> Optional[str]:
    """Pin this process to the CPUs local to `device` (multi-socket hosts), so
    the submitting thread and the seal workers sit next to its host link.
    Returns the CPU list applied, or None when the host has one NUMA node."""
    import os
    node = C.c_int(-1)
    check(L.lib().gs_device_numa_node(device, C.byref(node)), "numa")
    buf = C.create_string_buffer(4096)
    check(L.lib().gs_device_local_cpus(device, buf, 4096), "local cpus")
    cpus = buf.value.decode()
    try:
        nodes = open("/sys/devices/system/node/online").read().strip()
    except OSError:
        nodes = "0"
    if node.value < 0 or "-" not in nodes and "," not in nodes or not cpus:
        return None
    sel = set()
    for part in cpus.split(","):
        a, _, b = part.partition("-")
        sel.update(range(int(a), int(b or a) + 1))
    try:
        os.sched_setaffinity(0, sel)
    except OSError:
        return None
    return cpus


def launches() -> int:
    """Kernels launched by libghostserve_b200.so in this process."""
    return int(L.lib().gs_kernel_launches())
