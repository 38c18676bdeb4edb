"""KV data model (mirror of kv_layout.hpp) with device-side generation.

A worker's slice of one m-token chunk is laid out [K,V][layer][token][H*D/tp
elements] (kv_layout.hpp:59-68), 2-byte elements. Codes are position-wise,
so fp16 / bf16 KV is coded as its raw bytes (fp16.hpp:20-21).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib as L
from .coding import InvalidArgument, check


@dataclass
class ModelConfig:
    """kv_layout.hpp:14-29 (defaults: the 70B-like reference geometry)."""

    layers: int = 80
    kv_heads: int = 8
    head_dim: int = 128
    bytes_per_elem: int = 2
    tp_degree: int = 8

    def validate(self) -> None:
        if min(self.layers, self.kv_heads, self.head_dim, self.tp_degree) < 1:
            raise InvalidArgument("model: all dimensions must be positive")
        if self.bytes_per_elem != 2:
            raise InvalidArgument("model: only FP16 (2-byte) elements are supported")
        if (self.kv_heads * self.head_dim) % self.tp_degree != 0:
            raise InvalidArgument("model: kv_heads * head_dim must divide evenly across workers")


LLAMA3_8B = ModelConfig(32, 8, 128, 2, 8)
LLAMA3_70B = ModelConfig(80, 8, 128, 2, 8)


def chunk_count(tokens: int, chunk_size: int) -> int:
    """kv_layout.hpp:32-36"""
    if chunk_size == 0:
        raise InvalidArgument("chunk: chunk size must be positive")
    if tokens == 0:
        raise InvalidArgument("chunk: token count must be positive")
    return (tokens + chunk_size - 1) // chunk_size


def slice_bytes(cfg: ModelConfig, chunk_size: int) -> int:
    """kv_layout.hpp:40-45"""
    cfg.validate()
    out = C.c_uint64()
    check(L.lib().gs_slice_bytes(cfg.layers, cfg.kv_heads, cfg.head_dim, cfg.tp_degree, chunk_size,
                                 C.byref(out)), "slice_bytes")
    return out.value


def token_stride_bytes(cfg: ModelConfig) -> int:
    """kv_layout.hpp:48-51"""
    return cfg.kv_heads * cfg.head_dim // cfg.tp_degree * cfg.bytes_per_elem


def make_ground_truth_slice(kv_seed: int, request_id: int, chunk: int, worker: int, cfg: ModelConfig,
                            chunk_size: int, valid_tokens: int, out: Optional[torch.Tensor] = None,
                            device=None, stream=None) -> torch.Tensor:
    """Device-generated make_ground_truth_slice (kv_layout.hpp:110-134),
    bit-identical to the reference stream including pad_partial."""
    cfg.validate()
    n = slice_bytes(cfg, chunk_size)
    if out is None:
        out = torch.empty(n, dtype=torch.uint8, device=device or "cuda")
    if out.numel() * out.element_size() != n or not out.is_cuda:
        raise InvalidArgument("ground truth: output must be a CUDA buffer of slice_bytes")
    st = torch.cuda.current_stream().cuda_stream if stream is None else int(
        getattr(stream, "cuda_stream", stream))
    check(L.lib().gs_ground_truth_slice_device(kv_seed, request_id, chunk, worker, cfg.layers,
                                               cfg.kv_heads, cfg.head_dim, cfg.tp_degree, chunk_size,
                                               valid_tokens, out.data_ptr(), st), "ground_truth")
    return out


def pad_partial(slice_bytes_t: torch.Tensor, cfg: ModelConfig, chunk_size: int, valid_tokens: int,
                stream=None) -> None:
    """kv_layout.hpp:73-84 on a device slice."""
    st = torch.cuda.current_stream().cuda_stream if stream is None else int(
        getattr(stream, "cuda_stream", stream))
    check(L.lib().gs_pad_partial_device(slice_bytes_t.data_ptr(), cfg.layers, cfg.kv_heads,
                                        cfg.head_dim, cfg.tp_degree, chunk_size, valid_tokens, st),
          "pad_partial")
