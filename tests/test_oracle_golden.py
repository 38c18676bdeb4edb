"""Pin the CPU oracle (oracle/gs_oracle.c) before trusting it.

Checks the plain-C restatement against (1) the reference's own known-answer
tests and (2) golden vectors produced by the reference itself
(tests/golden/golden.json, made by tests/golden/make_golden.py from
oracle/_ref). No GPU needed.
"""
import hashlib
import itertools

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.vectors import splitmix_bytes


def schoolbook_mul(a, b):
    # gf256_test.cpp:15-22: carry-less multiply then reduce mod 0x11D.
    acc = 0
    for i in range(8):
        if b & (1 << i):
            acc ^= a << i
    for bit in range(15, 7, -1):
        if acc & (1 << bit):
            acc ^= 0x11D << (bit - 8)
    return acc


def test_gf_known_values(port):
    # gf256_test.cpp:26-49
    assert port.gf_mul(0x02, 0x03) == 0x06
    assert port.gf_mul(0x80, 0x02) == 0x1D
    assert port.gf_mul(0x00, 0xFF) == 0x00
    assert port.gf_mul(0xFF, 0x01) == 0xFF
    assert port.gf_inv(0x01) == 0x01
    assert port.gf_inv(0x02) == 0x8E
    with pytest.raises(O.OracleError) as ex:
        port.gf_inv(0)
    assert ex.value.status == O.DOMAIN_ERROR


def test_gf_exhaustive_vs_schoolbook_and_reference(port, golden):
    tab = np.array([[port.gf_mul(a, b) for b in range(256)] for a in range(256)], np.uint8)
    assert hashlib.sha256(tab.tobytes()).hexdigest() == golden["gf"]["mul_table_sha256"]
    for a in range(0, 256, 7):
        for b in range(256):
            assert tab[a, b] == schoolbook_mul(a, b)
    e, lg = port.gf_tables()
    assert e.tobytes().hex() == golden["gf"]["exp_hex"]
    assert lg.tobytes().hex() == golden["gf"]["log_hex"]
    inv = bytes([0] + [port.gf_inv(a) for a in range(1, 256)])
    assert inv.hex() == golden["gf"]["inv_hex"]


def test_encoding_matrices(port, golden):
    for key, hx in golden["matrices"].items():
        kind, n, k = map(int, key.split("_"))
        assert port.encoding_matrix(kind, n, k).tobytes().hex() == hx, key


def test_encode_and_reconstruct_vectors(port, golden):
    for rec in golden["encode"]:
        kind, n, k, ln, seed = rec["kind"], rec["n"], rec["k"], rec["len"], rec["seed"]
        data = [splitmix_bytes(seed * 1000 + j, ln) for j in range(n)]
        par = port.encode(kind, n, k, data)
        assert [f"{port.fnv1a64(p):016x}" for p in par] == rec["parity_fnv"]
        if "parity_hex" in rec:
            assert [p.tobytes().hex() for p in par] == rec["parity_hex"]
        for pat in rec.get("patterns", []):
            shards = {i: data[i] for i in range(n)}
            shards.update({n + i: par[i] for i in range(k)})
            got = port.reconstruct(kind, n, k, shards, pat["lost"])
            assert {str(i): f"{port.fnv1a64(b):016x}" for i, b in got.items()} == pat["rebuilt_fnv"]


def test_error_statuses(port, golden):
    for rec in golden["errors"]:
        if rec["op"] == "validate":
            assert port.fn("validate")(rec["kind"], rec["n"], rec["k"]) == rec["status"], rec
            continue
        data = [splitmix_bytes(77 + j, 16) for j in range(8)]
        par = port.encode(O.RS, 8, 2, data)
        shards = {i: data[i] for i in range(8)}
        shards.update({8 + i: par[i] for i in range(2)})
        if rec["drop"] is not None:
            shards.pop(rec["drop"])
        try:
            got = port.reconstruct(O.RS, 8, 2, shards, rec["lost"])
            st, rebuilt = 0, sorted(got)
            for i in got:
                assert np.array_equal(got[i], data[i])
        except O.OracleError as ex:
            st, rebuilt = ex.status, []
        assert (st, rebuilt) == (rec["status"], rec["rebuilt"]), rec


@pytest.mark.parametrize("idx", range(8))
def test_kv_slices_and_parity(port, golden, idx):
    rec = golden["kv"][idx]
    L, H, D, tp = rec["model"]
    if rec["slice_bytes"] > (16 << 20):
        pytest.skip("large fingerprint cases are checked on the GPU path")
    assert port.slice_bytes(L, H, D, tp, rec["chunk_size"]) == rec["slice_bytes"]
    slices = [port.make_ground_truth_slice(rec["kv_seed"], rec["request"], rec["chunk"], w, L, H,
                                           D, tp, rec["chunk_size"], rec["valid"])
              for w in range(rec["n"])]
    assert [f"{port.fnv1a64(s):016x}" for s in slices] == rec["data_fnv"]
    par = port.encode(rec["kind"], rec["n"], rec["k"], slices)
    assert [f"{port.fnv1a64(p):016x}" for p in par] == rec["parity_fnv"]
    assert f"{port.parity_checksum(par):016x}" == rec["checksum"]


def test_slice_bytes_and_fnv(port, golden):
    # kv_model_test.cpp:49-64
    for rec in golden["slice_bytes"]:
        assert port.slice_bytes(*rec["model"], rec["m"]) == rec["bytes"]
    assert port.slice_bytes(80, 8, 128, 8, 2048) == 83_886_080
    with pytest.raises(O.OracleError):
        port.slice_bytes(2, 4, 8, 3, 16)
    assert f"{port.fnv1a64(np.zeros(0, np.uint8)):016x}" == golden["fnv"]["empty"]
    assert f"{port.fnv1a64(np.frombuffer(b'foobar', np.uint8)):016x}" == golden["fnv"]["foobar"]


def test_xor_literals(port):
    # coding_test.cpp:151-159
    p = port.encode(O.XOR, 2, 1, [np.array([0x0F, 0x0F], np.uint8), np.array([0xF0, 0xF0], np.uint8)])
    assert p[0].tolist() == [0xFF, 0xFF]


def test_rs_mds_all_patterns(port):
    # coding_test.cpp:115-149 / 207-220 shape: every pattern within tolerance.
    for n, k in [(4, 2), (6, 2), (8, 3)]:
        data = [splitmix_bytes(900 + j, 33) for j in range(n)]
        par = port.encode(O.RS, n, k, data)
        for e in range(1, k + 1):
            for lost in itertools.combinations(range(n + k), e):
                sh = {i: data[i] for i in range(n)}
                sh.update({n + i: par[i] for i in range(k)})
                got = port.reconstruct(O.RS, n, k, sh, list(lost))
                for i, b in got.items():
                    assert np.array_equal(b, data[i])


@pytest.mark.skipif(not O.have_ref(), reason="reference not compiled here (oracle/_ref)")
def test_reference_chunk_entry_points_agree_with_port(port):
    """The reference's own checkpoint_chunk / reconstruct_chunk (through the
    oracle/_ref shim; the bench times them as the CPU baseline) produce the
    same parity, seal and rebuilt bytes as the port: 2 L / 6 H / 64 D, tp 6,
    RS(6,2), m = 16 (SURVEY §8c fingerprint case), valid = 16 and 5."""
    ref = O.ref()
    for valid in (16, 5):
        data = [port.make_ground_truth_slice(3, 0, 0, w, 2, 6, 64, 6, 16, valid) for w in range(6)]
        ln = data[0].size
        par = [np.zeros(ln, np.uint8) for _ in range(2)]
        cs, secs = ref.checkpoint_chunk_timed(O.RS, 6, 2, (2, 6, 64), 16, 0, 0, valid, data, par)
        want = port.encode(O.RS, 6, 2, data)
        assert all(np.array_equal(a, b) for a, b in zip(par, want))
        assert cs == port.parity_checksum(want) and secs >= 0
        if valid == 16:
            assert f"{port.fnv1a64(par[0]):016x}" == "fd24dd05670ae3ce"
            assert f"{port.fnv1a64(par[1]):016x}" == "d34a1b7a95bdf4e4"
        slots = list(data) + list(par)
        slots[1] = slots[4] = None
        outs = [np.zeros(ln, np.uint8) for _ in range(2)]
        ref.reconstruct_chunk_timed(O.RS, 6, 2, slots, outs)
        assert np.array_equal(outs[0], data[1]) and np.array_equal(outs[1], data[4])
        # corrupted parity -> kBadParity (recovery.hpp:109-112), status 4
        bad = list(slots)
        bad[6] = par[0].copy()
        bad[6][7] ^= 1
        with pytest.raises(O.OracleError) as ex:
            ref.reconstruct_chunk_timed(O.RS, 6, 2, bad, outs, sealed=cs)
        assert ex.value.status == 4
