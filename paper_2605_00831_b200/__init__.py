"""B200-native GhostServe shadow-checkpointing byte path.

Layers:
  csrc/        sm_100a kernels (K1 encode, K2 rebuild, KV generator) + C ABI
  _lib         ctypes binding of include/gs_capi.h
  coding       mirror of the reference coding.hpp API (host buffers in/out)
  device       device-tensor API + host-link pipelines (offload / upload)
  kv_layout    mirror of kv_layout.hpp with device-side synthetic KV
  parity_store host tier: ParityChunk / ParityStore with pinned slabs + seal
  checkpoint   checkpoint_chunk / DecodeCheckpointer / recover byte paths
  peer         multi-GPU striping over NVLink (IPC peer pointers)
"""
from . import coding  # noqa: F401
from .coding import (CodeKind, CodingScheme, EncodingMatrix, ErasurePattern, InvalidArgument,  # noqa: F401
                     UnrecoverableError, DomainError, build_encoding_matrix, encode,
                     max_tolerance, memory_overhead_ratio, reconstruct)

__all__ = ["CodeKind", "CodingScheme", "EncodingMatrix", "ErasurePattern", "InvalidArgument",
           "UnrecoverableError", "DomainError", "build_encoding_matrix", "encode", "max_tolerance",
           "memory_overhead_ratio", "reconstruct"]
