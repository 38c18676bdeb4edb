"""Host tier (parity_store.hpp) -- native pinned-slab store, no GPU needed
for the accounting / seal / GSRV logic (pinned allocation needs a driver, so
those cases are gpu-marked). Mirrors kv_model_test.cpp:182-271."""
import numpy as np
import pytest

from paper_2605_00831_b200 import _lib as L
from paper_2605_00831_b200.coding import CodingScheme, InvalidArgument, LogicError, ParityFileError
from paper_2605_00831_b200.parity_store import (ParityChunk, ParityGetStatus, ParityStore,
                                                deserialize_parity_store, fnv1a64,
                                                serialize_parity_store)
from tests.golden.vectors import splitmix_bytes

needs_pinned = pytest.mark.skipif(not L.lib().gs_cuda_available(), reason="pinned host memory needs a CUDA driver")


def make_chunk(req, idx, ln, seed, valid=16):
    c = ParityChunk(req, idx, CodingScheme.xor_code(2), [splitmix_bytes(seed, ln)], valid, ln)
    c.seal()
    return c


def test_fnv_known_values(golden):
    assert f"{fnv1a64(b''):016x}" == golden["fnv"]["empty"]
    assert f"{fnv1a64(b'foobar'):016x}" == golden["fnv"]["foobar"]


def test_empty_store_accounting_and_errors():
    s = ParityStore(1000)
    assert (s.used_bytes(), s.payload_bytes(), s.peak_payload_bytes(), s.entry_count()) == (0, 0, 0, 0)
    assert s.capacity_bytes() == 1000 and s.audit()
    st, c = s.get(1, 2)
    assert st == ParityGetStatus.kMissing and c is None
    with pytest.raises(InvalidArgument):
        serialize_parity_store(s)
    # zero-length entries carry accounting only (no pinned memory needed)
    assert s.try_put(ParityChunk(1, 0, CodingScheme.reed_solomon(4, 2), [], 0, 0, 0))
    assert s.used_bytes() == 64
    with pytest.raises(LogicError):
        s.try_put(ParityChunk(1, 0, CodingScheme.reed_solomon(4, 2), [], 0, 0, 0))


@pytest.mark.gpu
def test_put_get_capacity_duplicate_peak_audit():
    s = ParityStore(2 * (64 + 64) + 10)
    a, b, c = make_chunk(1, 0, 64, 11), make_chunk(1, 1, 64, 12), make_chunk(2, 0, 64, 13)
    assert s.try_put(a) and s.try_put(b)
    assert not s.try_put(c)                       # back-pressure, store unchanged
    assert s.entry_count() == 2 and s.used_bytes() == 2 * (64 + 64) and s.audit()
    with pytest.raises(LogicError):
        s.try_put(make_chunk(1, 0, 64, 14))
    st, got = s.get(1, 1)
    assert st == ParityGetStatus.kOk and np.array_equal(got.parity[0], b.parity[0])
    assert got.checksum == b.checksum and got.valid_tokens == 16
    s.corrupt_entry(1, 1)
    assert s.get(1, 1)[0] == ParityGetStatus.kCorrupt
    assert s.get(1, 1, verify=False)[0] == ParityGetStatus.kOk
    s.erase_request(1)
    assert s.entry_count() == 0 and s.used_bytes() == 0 and s.peak_payload_bytes() == 128 and s.audit()
    assert s.try_put(c)


@pytest.mark.gpu
def test_gsrv_round_trip_matches_reference_bytes(golden):
    g = golden["gsrv"]
    scheme = CodingScheme(g["kind"], g["n"], g["k"])
    s = ParityStore()
    for i, (req, chunk, valid) in enumerate(g["keys"]):
        par = [splitmix_bytes(g["parity_seed"] + 10 * i + j, g["slice_len"]) for j in range(g["k"])]
        c = ParityChunk(req, chunk, scheme, par, valid, g["slice_len"])
        c.seal()
        assert s.try_put(c)
    img = serialize_parity_store(s)
    assert img.hex() == g["image_hex"]            # byte-identical to the reference's writer
    back = deserialize_parity_store(bytes.fromhex(g["image_hex"]))
    assert back.keys() == sorted((r, c) for r, c, _ in g["keys"])
    for i, (req, chunk, valid) in enumerate(g["keys"]):
        st, c = back.get(req, chunk)
        assert st == ParityGetStatus.kOk and c.valid_tokens == valid
        for j in range(g["k"]):
            assert np.array_equal(c.parity[j], splitmix_bytes(g["parity_seed"] + 10 * i + j, g["slice_len"]))
    bad = bytearray(bytes.fromhex(g["image_hex"]))
    bad[30] ^= 1
    with pytest.raises(ParityFileError):
        deserialize_parity_store(bytes(bad))
    with pytest.raises(ParityFileError):
        deserialize_parity_store(bytes.fromhex(g["image_hex"])[:-3])
    with pytest.raises(ParityFileError):
        deserialize_parity_store(b"XSRV" + bytes.fromhex(g["image_hex"])[4:])
    with pytest.raises(ParityFileError):
        deserialize_parity_store(bytes.fromhex(g["image_hex"]), capacity_bytes=100)
