"""K1/K2 straight out of a paged KV cache.

A serving engine keeps each TP worker's KV in fixed-size pages (vLLM /
FlashInfer style), so the reference slice of a (request, block) --
[K,V][layer][token][H*D/tp] bytes (kv_layout.hpp:59-68) -- is 2*layers
pages scattered through the cache. The reference (and the paper's "packing")
would first gather them into a contiguous buffer. Here the page mapping is
fused into the kernels' address generation: K1 reads the pages in place,
masks tokens >= valid (pad_partial, kv_layout.hpp:73-84) and writes parity
in the reference byte order; K2 rebuilds a lost worker's pages directly into
the replacement worker's cache. No staging copy of the KV.

Cache layout per worker: ``[layers, 2 (K,V), num_blocks, block_size, H*D/tp * 2 B]``
(vLLM's per-layer [2, num_blocks, block_size, heads, dim] stacked over layers).
A checkpoint chunk is either one block (``*_blocks``: the 16-token decode
block of config C2) or several blocks listed in a device block table
(``*_chunks``: e.g. 2048-token prefill chunks of 16-token blocks).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence

import torch

from . import _lib as L
from .coding import CodingScheme, ErasurePattern, InvalidArgument, check, decoder, encoder
from .device import row_ptrs
from .kv_layout import ModelConfig, token_stride_bytes


class PagedKVCache:
    """One TP worker's paged KV cache on one device."""

    def __init__(self, model: ModelConfig, num_blocks: int, block_size: int, device=None, fill=None):
        model.validate()
        self.model = model
        self.num_blocks = num_blocks
        self.block_size = block_size
        self.token_bytes = token_stride_bytes(model)
        self.page_bytes = block_size * self.token_bytes
        shape = (model.layers, 2, num_blocks, block_size, self.token_bytes)
        self.buf = (torch.empty(shape, dtype=torch.uint8, device=device or "cuda") if fill is None else
                    torch.full(shape, fill, dtype=torch.uint8, device=device or "cuda"))
        self.layer_stride = 2 * num_blocks * self.page_bytes
        self.kv_stride = num_blocks * self.page_bytes

    @property
    def slice_bytes(self) -> int:
        return 2 * self.model.layers * self.page_bytes

    def block_base(self, block_id: int) -> int:
        if not 0 <= block_id < self.num_blocks:
            raise InvalidArgument("paged: block id out of range")
        return self.buf.data_ptr() + block_id * self.page_bytes

    def page_map(self, valid_tokens: int, chunk_tokens: Optional[int] = None,
                 block_table: Optional[torch.Tensor] = None) -> L.PageMap:
        """Single-block chunks (chunk == one block), or chunks of
        `chunk_tokens` spanning several blocks listed per stripe in the device
        int32 `block_table` [stripes, chunk_tokens // block_size]."""
        if block_table is None:
            if valid_tokens > self.block_size:
                raise InvalidArgument("kv: valid_tokens exceeds chunk size")
            return L.PageMap(self.page_bytes, self.model.layers, self.token_bytes, valid_tokens,
                             self.layer_stride, self.kv_stride, None, self.page_bytes, 0)
        m = chunk_tokens
        if m is None or m % self.block_size or valid_tokens > m:
            raise InvalidArgument("paged: chunk must be a whole number of blocks >= valid tokens")
        if block_table.dtype != torch.int32 or not block_table.is_cuda or block_table.dim() != 2:
            raise InvalidArgument("paged: block_table must be a CUDA int32 [stripes, blocks] tensor")
        if block_table.shape[1] < m // self.block_size or block_table.stride(1) != 1:
            raise InvalidArgument("paged: block_table rows must list every block of the chunk")
        return L.PageMap(m * self.token_bytes, self.model.layers, self.token_bytes, valid_tokens,
                         self.layer_stride, self.kv_stride, block_table.data_ptr(), self.page_bytes,
                         block_table.stride(0))

    def chunk_slice_bytes(self, chunk_tokens: int) -> int:
        return 2 * self.model.layers * chunk_tokens * self.token_bytes

    def write_chunk(self, blocks: Sequence[int], slice_: torch.Tensor, chunk_tokens: int,
                    valid_tokens: Optional[int] = None) -> None:
        """Scatter a reference-layout slice of a multi-block chunk (tests)."""
        v = chunk_tokens if valid_tokens is None else valid_tokens
        src = slice_.view(2, self.model.layers, chunk_tokens, self.token_bytes)
        for i, b in enumerate(blocks):
            lo = i * self.block_size
            hi = min(lo + self.block_size, v)
            if hi > lo:
                self.buf[:, :, b, :hi - lo] = src.permute(1, 0, 2, 3)[:, :, lo:hi]

    def read_chunk(self, blocks: Sequence[int], chunk_tokens: int, valid_tokens: Optional[int] = None
                   ) -> torch.Tensor:
        """Gather a multi-block chunk as a reference-layout slice, zero past `valid`."""
        v = chunk_tokens if valid_tokens is None else valid_tokens
        out = torch.zeros((2, self.model.layers, chunk_tokens, self.token_bytes), dtype=torch.uint8,
                          device=self.buf.device)
        for i, b in enumerate(blocks):
            lo = i * self.block_size
            hi = min(lo + self.block_size, v)
            if hi > lo:
                out[:, :, lo:hi] = self.buf[:, :, b, :hi - lo].permute(1, 0, 2, 3)
        return out.view(-1)

    # test / ingest helpers (torch copies, not on the checkpoint path)
    def write_slice(self, block_id: int, slice_: torch.Tensor, valid_tokens: Optional[int] = None) -> None:
        """Scatter a reference-layout slice into this block (tokens < valid)."""
        v = self.block_size if valid_tokens is None else valid_tokens
        src = slice_.view(2, self.model.layers, self.block_size, self.token_bytes)
        self.buf[:, :, block_id, :v] = src.permute(1, 0, 2, 3)[:, :, :v]

    def read_slice(self, block_id: int, valid_tokens: Optional[int] = None) -> torch.Tensor:
        """Gather this block as a reference-layout slice, zero past `valid`."""
        v = self.block_size if valid_tokens is None else valid_tokens
        out = torch.zeros((2, self.model.layers, self.block_size, self.token_bytes), dtype=torch.uint8,
                          device=self.buf.device)
        out[:, :, :v] = self.buf[:, :, block_id, :v].permute(1, 0, 2, 3)
        return out.view(-1)


def _stream(s) -> int:
    return torch.cuda.current_stream().cuda_stream if s is None else int(getattr(s, "cuda_stream", s))


def _check_caches(caches: Sequence[PagedKVCache]) -> None:
    c0 = caches[0]
    for c in caches:
        if (c.page_bytes, c.layer_stride, c.kv_stride, c.model.layers) != (
                c0.page_bytes, c0.layer_stride, c0.kv_stride, c0.model.layers):
            raise InvalidArgument("paged: all workers' caches must share one geometry")


def encode_blocks(scheme: CodingScheme, caches: Sequence[PagedKVCache], block_ids: Sequence[Sequence[int]],
                  valid_tokens: int, parity_out: torch.Tensor, stream=None) -> None:
    """K1 over S (request, block) stripes read in place from the n workers'
    caches; block_ids[s][j] = block of stripe s in worker j's cache.
    parity_out: device [S, k, slice_bytes] in reference order."""
    if len(caches) != scheme.n:
        raise InvalidArgument(f"coding: expected {scheme.n} data shards, got {len(caches)}")
    _check_caches(caches)
    S = len(block_ids)
    slots = [caches[j].block_base(block_ids[s][j]) for s in range(S) for j in range(scheme.n)]
    outs = row_ptrs(parity_out)
    pm = caches[0].page_map(valid_tokens)
    check(L.lib().gs_apply_device_paged(encoder(scheme).handle, S, L.ptr_array(slots), L.ptr_array(outs),
                                        caches[0].slice_bytes, C.byref(pm), (1 << scheme.n) - 1, None,
                                        _stream(stream)), "encode_blocks")


def checkpoint_blocks(pipeline, scheme: CodingScheme, caches: Sequence[PagedKVCache],
                      block_ids: Sequence[Sequence[int]], valid_tokens: int, h_parity, compute=None,
                      copy=None) -> None:
    """Decode-block checkpoint from the paged caches: K1 reads the pages in
    place, parity D2H'd piecewise into pinned `h_parity` [S, k, slice]
    (or a list of S*k pinned pointers, e.g. ParityStore.reserve results)."""
    _check_caches(caches)
    S = len(block_ids)
    slots = [caches[j].block_base(block_ids[s][j]) for s in range(S) for j in range(scheme.n)]
    if isinstance(h_parity, torch.Tensor):
        dst = row_ptrs(h_parity)
    else:
        dst = list(h_parity)
    pm = caches[0].page_map(valid_tokens)
    cs = _stream(compute)
    check(L.lib().gs_encode_offload_paged(pipeline.handle, encoder(scheme).handle, S, L.ptr_array(slots),
                                          L.ptr_array(dst), caches[0].slice_bytes, C.byref(pm), cs,
                                          _stream(copy) if copy is not None else cs), "checkpoint_blocks")


def checkpoint_chunks(pipeline, scheme: CodingScheme, caches: Sequence[PagedKVCache], block_table: torch.Tensor,
                      chunk_tokens: int, valid_tokens: int, h_parity, compute=None, copy=None) -> None:
    """Prefill-chunk checkpoint from the paged caches: S chunks of
    `chunk_tokens`, stripe s made of the blocks block_table[s] (the same ids
    in every worker's cache, as TP workers allocate in lockstep). K1 gathers
    the pages in place; parity -> pinned `h_parity` [S, k, slice]."""
    _check_caches(caches)
    S = block_table.shape[0]
    pm = caches[0].page_map(valid_tokens, chunk_tokens, block_table)
    slots = [caches[j].buf.data_ptr() for s in range(S) for j in range(scheme.n)]
    dst = row_ptrs(h_parity)
    cs = _stream(compute)
    check(L.lib().gs_encode_offload_paged(pipeline.handle, encoder(scheme).handle, S, L.ptr_array(slots),
                                          L.ptr_array(dst), caches[0].chunk_slice_bytes(chunk_tokens), C.byref(pm),
                                          cs, _stream(copy) if copy is not None else cs), "checkpoint_chunks")


def rebuild_chunks(pipeline, scheme: CodingScheme, lost: ErasurePattern, caches: Sequence[Optional[PagedKVCache]],
                   replacements: Dict[int, PagedKVCache], block_table: torch.Tensor, chunk_tokens: int,
                   valid_tokens: int, h_parity: torch.Tensor, compute=None, copy=None) -> None:
    """Recovery of multi-block chunks into the replacement workers' caches
    (same block ids), survivors read in place, parity H2D'd from pinned."""
    dec = decoder(scheme, lost)
    live = [c for j, c in enumerate(caches) if c is not None and not lost.contains(j)]
    _check_caches(live + list(replacements.values()))
    S = block_table.shape[0]
    n, k = scheme.n, scheme.k
    hp = row_ptrs(h_parity)
    slots: List[Optional[int]] = []
    for s in range(S):
        for j in range(n):
            slots.append(None if lost.contains(j) else caches[j].buf.data_ptr())
        for i in range(k):
            slots.append(None if lost.contains(n + i) else hp[s * k + i])
    outs = [replacements[w].buf.data_ptr() for s in range(S) for w in dec.out_index]
    # geometry reference: a surviving cache, or a replacement when every data
    # worker was lost (the rebuild then reads parity only)
    ref = live[0] if live else next(iter(replacements.values()))
    pm = ref.page_map(valid_tokens, chunk_tokens, block_table)
    cs = _stream(compute)
    check(L.lib().gs_reconstruct_upload_paged(pipeline.handle, dec.handle, S, L.ptr_array(slots), L.ptr_array(outs),
                                              ref.chunk_slice_bytes(chunk_tokens), C.byref(pm), C.byref(pm), cs,
                                              _stream(copy) if copy is not None else cs), "rebuild_chunks")


def rebuild_blocks(pipeline, scheme: CodingScheme, lost: ErasurePattern, caches: Sequence[Optional[PagedKVCache]],
                   replacements: Dict[int, PagedKVCache], block_ids: Sequence[Sequence[int]], valid_tokens: int,
                   h_parity: torch.Tensor, compute=None, copy=None) -> None:
    """Recovery into paged caches: survivors read in place (caches[j] for
    j not lost), parity H2D'd from pinned `h_parity` [S, k, slice], rebuilt
    pages written into replacements[w] at the same block ids."""
    dec = decoder(scheme, lost)
    live = [c for j, c in enumerate(caches) if c is not None and not lost.contains(j)]
    _check_caches(live + list(replacements.values()))
    S = len(block_ids)
    n, k = scheme.n, scheme.k
    hp = row_ptrs(h_parity)
    slots: List[Optional[int]] = []
    for s in range(S):
        for j in range(n):
            slots.append(None if lost.contains(j) else caches[j].block_base(block_ids[s][j]))
        for i in range(k):
            slots.append(None if lost.contains(n + i) else hp[s * k + i])
    outs = [replacements[w].block_base(block_ids[s][w]) for s in range(S) for w in dec.out_index]
    # geometry reference: a surviving cache, or a replacement when every data
    # worker was lost (the rebuild then reads parity only)
    ref = live[0] if live else next(iter(replacements.values()))
    pm = ref.page_map(valid_tokens)
    cs = _stream(compute)
    check(L.lib().gs_reconstruct_upload_paged(pipeline.handle, dec.handle, S, L.ptr_array(slots), L.ptr_array(outs),
                                              ref.slice_bytes, C.byref(pm), C.byref(pm), cs,
                                              _stream(copy) if copy is not None else cs), "rebuild_blocks")
