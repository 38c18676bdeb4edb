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


def test_cost_only_entries():
    """KvPolicy::materialize = false (checkpoint.hpp:51-54): entries without a
    payload are accounted like full ones (k * slice_len + 64), get() is kOk
    with no payload, corrupt_entry is a no-op, GSRV refuses them."""
    s = ParityStore(3 * (2 * 4096 + 64))
    sch = CodingScheme.reed_solomon(4, 2)
    for i in range(3):
        assert s.try_put(ParityChunk(7, i, sch, [], 16, 4096, 0xCBF29CE484222325))
    assert not s.try_put(ParityChunk(7, 3, sch, [], 16, 4096, 0))     # back-pressure
    assert s.used_bytes() == 3 * (2 * 4096 + 64) and s.payload_bytes() == 3 * 8192 and s.audit()
    st, c = s.get(7, 1)
    assert st == ParityGetStatus.kOk and not c.payload_present() and c.slice_len == 4096
    s.corrupt_entry(7, 1)
    assert s.get(7, 1)[0] == ParityGetStatus.kOk
    with pytest.raises(InvalidArgument):
        serialize_parity_store(s)
    s.erase_request(7)
    assert s.entry_count() == 0 and s.used_bytes() == 0 and s.peak_payload_bytes() == 3 * 8192


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


@needs_pinned
@pytest.mark.gpu
def test_store_matches_reference_on_random_operations():
    """Random try_put / get / contains / erase_request / corrupt sequences
    with capacity back-pressure and duplicates: the native host tier answers
    exactly like the reference's ParityStore (compiled in place) after every
    operation, accounting and peak included."""
    import ctypes as C
    import random
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("reference not compiled here")
    ref = O.ref()
    f = lambda name: ref.fn(name)  # noqa: E731
    f("store_new").restype = C.c_void_p
    f("store_new").argtypes = [C.c_uint64]
    for nm in ("store_free",):
        f(nm).argtypes = [C.c_void_p]
    f("store_try_put").argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_uint32,
                                   C.c_uint64, C.c_void_p, C.POINTER(C.c_int)]
    f("store_get").argtypes = [C.c_void_p, C.c_uint64, C.c_uint32]
    f("store_contains").argtypes = [C.c_void_p, C.c_uint64, C.c_uint32]
    f("store_erase").argtypes = [C.c_void_p, C.c_uint64]
    f("store_corrupt").argtypes = [C.c_void_p, C.c_uint64, C.c_uint32]
    f("store_stats").argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
    rng = random.Random(99)
    for cap in (ParityStore.UNLIMITED if hasattr(ParityStore, "UNLIMITED") else (1 << 64) - 1, 50_000, 9_000):
        mine = ParityStore(cap)
        theirs = f("store_new")(cap)
        try:
            for step in range(400):
                op = rng.random()
                req, ch = rng.randrange(6), rng.randrange(8)
                if op < 0.45:
                    k = rng.randint(1, 3)
                    ln = rng.choice([0, 16, 1000, 4096])
                    par = [splitmix_bytes(rng.randrange(1 << 30), ln) for _ in range(k)] if ln else []
                    c = ParityChunk(req, ch, CodingScheme.reed_solomon(4, k), par, rng.randrange(17), ln)
                    c.seal()
                    acc = C.c_int(-1)
                    arr = (C.c_void_p * k)(*[p.ctypes.data for p in par]) if par else None
                    rst = f("store_try_put")(theirs, req, ch, 2, 4, k, c.valid_tokens, ln, arr, C.byref(acc))
                    try:
                        got = mine.try_put(c)
                        assert rst == 0 and int(got) == acc.value, (step, cap)
                    except LogicError:
                        assert rst == 1, (step, cap)   # duplicate -> logic_error on both sides
                elif op < 0.75:
                    st, _ = mine.get(req, ch)
                    assert int(st) == f("store_get")(theirs, req, ch), (step, cap)
                    assert mine.contains(req, ch) == bool(f("store_contains")(theirs, req, ch))
                elif op < 0.85:
                    mine.erase_request(req)
                    f("store_erase")(theirs, req)
                else:
                    mine.corrupt_entry(req, ch)
                    f("store_corrupt")(theirs, req, ch)
                out = (C.c_uint64 * 5)()
                f("store_stats")(theirs, out)
                assert (mine.used_bytes(), mine.payload_bytes(), mine.peak_payload_bytes(), mine.entry_count(),
                        int(mine.audit())) == tuple(out), (step, cap)
        finally:
            f("store_free")(theirs)
            mine.close()
