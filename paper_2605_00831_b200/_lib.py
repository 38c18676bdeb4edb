"""ctypes binding of libghostserve_b200.so (include/gs_capi.h).

The library is built in-tree by ``make -C paper_2605_00831_b200/csrc`` (or
``__graft_entry__.build()``). Loading fails loudly when it is missing: there
is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libghostserve_b200.so")

(GS_OK, GS_INVALID_ARGUMENT, GS_UNRECOVERABLE, GS_DOMAIN_ERROR, GS_CUDA_ERROR, GS_UNSUPPORTED,
 GS_LOGIC_ERROR, GS_RUNTIME_ERROR) = range(8)
GS_XOR, GS_RDP, GS_RS = 0, 1, 2
IPC_HANDLE_BYTES = 64

# Every symbol include/gs_capi.h declares: (name, restype, argtypes).
_vp, _vpp, _i, _sz, _u8, _u32, _u64 = (C.c_void_p, C.POINTER(C.c_void_p), C.c_int, C.c_size_t,
                                       C.c_uint8, C.c_uint32, C.c_uint64)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
SIGNATURES = {
    "gs_status_string": (C.c_char_p, [_i]),
    "gs_last_error": (C.c_char_p, []),
    "gs_abi_version": (_i, []),
    "gs_jit_quiesce": (_i, []),
    "gs_kernel_launches": (_u64, []),
    "gs_zero_copy_offloads": (_u64, []),
    "gs_set_zero_copy_bytes": (_i, [_u64]),
    "gs_cuda_available": (_i, []),
    "gs_gf_mul": (_u8, [_u8, _u8]),
    "gs_gf_inv": (_i, [_u8, _u8p]),
    "gs_gf_div": (_i, [_u8, _u8, _u8p]),
    "gs_scheme_validate": (_i, [_i, _i, _i]),
    "gs_max_tolerance": (_i, [_i, _i, _i]),
    "gs_encoding_matrix": (_i, [_i, _i, _i, _u8p]),
    "gs_encoder_create": (_i, [_i, _i, _i, _vpp]),
    "gs_decoder_create": (_i, [_i, _i, _i, _ip, _i, _vpp]),
    "gs_codec_create_ex": (_i, [_i, _i, _i, _ip, _i, _i, _vpp]),
    "gs_codec_destroy": (_i, [_vp]),
    "gs_codec_info": (_i, [_vp, _ip, _ip, _ip, _ip]),
    "gs_codec_coefficients": (_i, [_vp, _u8p]),
    "gs_apply_device": (_i, [_vp, _i, _vpp, _vpp, _sz, _vp]),
    "gs_apply_device_paged": (_i, [_vp, _i, _vpp, _vpp, _sz, _vp, _u32, _vp, _vp]),
    "gs_encode_offload_paged": (_i, [_vp, _vp, _i, _vpp, _vpp, _sz, _vp, _vp, _vp]),
    "gs_reconstruct_upload_paged": (_i, [_vp, _vp, _i, _vpp, _vpp, _sz, _vp, _vp, _vp, _vp]),
    "gs_pipeline_create": (_i, [_i, _sz, _vpp]),
    "gs_pipeline_destroy": (_i, [_vp]),
    "gs_prewarm": (_i, [_i]),
    "gs_set_kernel_variant": (_i, [_i]),
    "gs_encode_offload": (_i, [_vp, _vp, _i, _vpp, _vpp, _sz, _vp, _vp]),
    "gs_reconstruct_upload": (_i, [_vp, _vp, _i, _vpp, _vpp, _sz, _vp, _vp]),
    "gs_encode_host": (_i, [_vp, _vp, _vpp, _vpp, _sz]),
    "gs_reconstruct_host": (_i, [_vp, _vp, _vpp, _vpp, _sz]),
    "gs_encode_host_async": (_i, [_vp, _vp, _vpp, _vpp, _sz]),
    "gs_reconstruct_host_async": (_i, [_vp, _vp, _vpp, _vpp, _sz]),
    "gs_pipeline_sync": (_i, [_vp]),
    "gs_set_jit": (_i, [_i]),
    "gs_codec_jit_status": (_i, [_vp, _i, _ip]),
    "gs_codec_create": (_i, [_i, _i, _i, _vpp]),
    "gs_encode_async": (_i, [_vp, _vpp, _sz, _vpp, _vp, _vp]),
    "gs_reconstruct_async": (_i, [_vp, _ip, _i, _vpp, _vpp, _vpp, _sz, _vp]),
    "gs_sync": (_i, [_vp]),
    "gs_thread_pipeline": (_i, [_vpp]),
    "gs_pipeline_set_max_ctas": (_i, [_vp, _i]),
    "gs_pipeline_device": (_i, [_vp, _ip]),
    "gs_pipeline_set_timing": (_i, [_vp, _i]),
    "gs_pipeline_kernel_time": (_i, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_double), _ip, _u64p]),
    "gs_slice_bytes": (_i, [_i, _i, _i, _i, _u32, _u64p]),
    "gs_ground_truth_slice_device": (_i, [_u64, _u64, _u32, _i, _i, _i, _i, _i, _u32, _u32, _vp, _vp]),
    "gs_ground_truth_slice": (_i, [_u64, _u64, _u32, _i, _i, _i, _i, _i, _u32, _u32, _vp]),
    "gs_pad_partial_device": (_i, [_vp, _i, _i, _i, _i, _u32, _u32, _vp]),
    "gs_fnv1a64": (_u64, [_vp, _sz, _u64]),
    "gs_parity_checksum": (_u64, [_vpp, _i, _sz]),
    "gs_fnv_host_simd": (_i, []),
    "gs_fnv_host_set_simd": (_i, [_i]),
    "gs_parity_checksum_batch": (_i, [_vpp, _i, _i, _sz, _i, _u64p]),
    "gs_fnv1a64_continue_batch": (_i, [_vpp, _u64p, _u64p, _u64p, _i, _i]),
    "gs_relay_board_bytes": (_u64, [_i, _i, _i]),
    "gs_fnv_relay": (_i, [_vp, _u64, _i, _i, _vpp, _u64, _i, _i, _u64, _i, C.c_double, _u64p]),
    "gs_fnv_relay_device": (_i, [_vp, _u64, _i, _i, _vpp, _i, _vpp, _vpp, _u64, _i, _i, _u64, _i, _i, _vp,
                                 C.c_double, _u64p]),
    "gs_fnv1a64_device": (_i, [_vpp, _i, _i, _u64, _u64, _vp, _vp]),
    "gs_parity_upload_checksum": (_i, [_vpp, _i, _i, _u64, _vpp, _vp, _vp, _vp]),
    "gs_parity_offload_sealed": (_i, [_vpp, _i, _i, _u64, _vpp, _vp, _vp, _vp]),
    "gs_verify_enqueue": (_i, [_vpp, _i, _i, _u64, _i, _i, _vpp, _vp, _vp, _vpp]),
    "gs_verify_finish": (_i, [_vp, _i, _u64p]),
    "gs_verify_finish_ex": (_i, [_vp, _i, _u64p, _ip]),
    "gs_verify_set_rates": (_i, [_vp, C.c_double, C.c_double]),
    "gs_verify_stream_wait": (_i, [_vp, _i, _vp]),
    "gs_verify_hold": (_i, [_vp]),
    "gs_verify_release": (_i, [_vp]),
    "gs_verify_handoffs": (_u64, []),
    "gs_verify_last_stats": (_i, [C.POINTER(C.c_double)]),
    "gs_fnv1a64_device_seeded": (_i, [_vpp, _i, _i, _u64, _vp, _vp, _vp]),
    "gs_store_create": (_i, [_u64, _i, _vpp]),
    "gs_store_destroy": (_i, [_vp]),
    "gs_store_reserve": (_i, [_vp, _u64, _u32, _i, _i, _i, _u32, _u64, _ip, _vpp]),
    "gs_store_commit": (_i, [_vp, _u64, _u32, _vp]),
    "gs_store_reserve_batch": (_i, [_vp, _i, _u64p, C.POINTER(C.c_uint32), _i, _i, _i, _u32, _u64, _ip, _vpp]),
    "gs_store_commit_batch": (_i, [_vp, _i, _u64p, C.POINTER(C.c_uint32), _vp]),
    "gs_store_commit_sealed_batch": (_i, [_vp, _i, _u64p, C.POINTER(C.c_uint32), _vp, _vp]),
    "gs_store_wait_sealed": (_i, [_vp]),
    "gs_store_put": (_i, [_vp, _u64, _u32, _i, _i, _i, _u32, _u64, _vpp, _u64, _i, _ip]),
    "gs_store_get": (_i, [_vp, _u64, _u32, _i, _ip, _vpp, _u64p, C.POINTER(C.c_uint32), _u64p, _ip]),
    "gs_store_contains": (_i, [_vp, _u64, _u32]),
    "gs_store_erase_request": (_i, [_vp, _u64]),
    "gs_store_stats": (_i, [_vp, _u64p]),
    "gs_store_audit": (_i, [_vp]),
    "gs_store_corrupt_entry": (_i, [_vp, _u64, _u32]),
    "gs_store_keys": (_i, [_vp, _u64p, _u64, _u64p]),
    "gs_store_serialize": (_i, [_vp, _vp, _u64, _u64p]),
    "gs_store_deserialize": (_i, [_vp, _u64, _u64, _i, _vpp]),
    "gs_ipc_handle": (_i, [_vp, _vp, _u64p]),
    "gs_ipc_open": (_i, [_vp, _i, _vpp]),
    "gs_ipc_close": (_i, [_vp]),
    "gs_peer_enable": (_i, [_i, _i]),
    "gs_stripe_range": (_i, [_u64, _i, _i, _u64p, _u64p]),
    "gs_host_alloc": (_i, [_sz, _vpp]),
    "gs_host_free": (_i, [_vp]),
    "gs_host_alloc_near": (_i, [_i, _sz, _vpp]),
    "gs_store_bind_device": (_i, [_vp, _i]),
    "gs_device_numa_node": (_i, [_i, _ip]),
    "gs_device_local_cpus": (_i, [_i, C.c_char_p, _sz]),
}

_lib = None
_lock = threading.Lock()


class GhostServeError(Exception):
    """Base of the errors raised from C-ABI status codes."""

    status = -1


def lib() -> C.CDLL:
    """Load (once) and return the native library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"libghostserve_b200.so not built at {LIB_PATH}; run "
                    "`make -C paper_2605_00831_b200/csrc` (no CPU fallback exists)")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


class PageMap(C.Structure):
    """gs_page_map (include/gs_capi.h)."""

    _fields_ = [("page_bytes", C.c_uint32), ("layers", C.c_uint32), ("token_bytes", C.c_uint32),
                ("valid_tokens", C.c_uint32), ("layer_stride", C.c_uint64), ("kv_stride", C.c_uint64),
                ("block_table", C.c_void_p), ("block_bytes", C.c_uint32), ("table_stride", C.c_uint32)]


def last_error() -> str:
    msg = lib().gs_last_error()
    return msg.decode() if msg else ""


def ptr_array(values):
    arr = (C.c_void_p * max(len(values), 1))()
    for i, v in enumerate(values):
        arr[i] = v
    return arr
