"""Generate tests/golden/golden.json from the REFERENCE ITSELF.

Runs only in the build container (needs oracle/_ref/libghostserve_ref.so, which
`make -C oracle` compiles from /root/reference/proj/include in place). The
resulting JSON is committed; the GPU box and the CPU test suite read only the
JSON, never /root/reference.

    python tests/golden/make_golden.py            # rewrite golden.json
"""
from __future__ import annotations

import hashlib
import itertools
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.golden.vectors import splitmix_bytes  # noqa: E402

# Scheme set of the reference acceptance C1 (tests/acceptance.cpp:101-107),
# plus the configs' RS(6,2), a few wider / taller RS shapes for the generic
# kernel, and RDP at primes p = 3, 5, 7, 11, 13.
SCHEMES = [
    (O.XOR, 2, 1), (O.XOR, 4, 1), (O.XOR, 8, 1),
    (O.RS, 4, 1), (O.RS, 4, 2), (O.RS, 8, 2), (O.RS, 8, 3), (O.RS, 6, 2),
    (O.RS, 2, 2), (O.RS, 10, 4), (O.RS, 16, 4), (O.RS, 12, 3),
    (O.RDP, 2, 2), (O.RDP, 3, 2), (O.RDP, 4, 2), (O.RDP, 6, 2), (O.RDP, 8, 2), (O.RDP, 12, 2),
]
MATRIX_ONLY = [(O.RS, 200, 55), (O.RS, 127, 127), (O.RS, 1, 1), (O.RS, 32, 8)]
HEX_LENGTHS = [1, 17, 64]
FNV_LENGTHS = [4096, 1 << 20]

# KV fingerprint cases: SURVEY.md §8(c) table + the reference's tiny models.
KV_CASES = [
    # name, scheme, (layers, kv_heads, head_dim, tp), chunk_size, valid, request, chunk
    ("c1_rs42_32L8H128D_tp4_m4096", (O.RS, 4, 2), (32, 8, 128, 4), 4096, 4096, 0, 0),
    ("llama8b_tp8_rs82_m16", (O.RS, 8, 2), (32, 8, 128, 8), 16, 16, 0, 0),
    ("llama8b_tp8_xor8_m16", (O.XOR, 8, 1), (32, 8, 128, 8), 16, 16, 0, 0),
    ("llama8b_tp8_rs82_m16_valid5_req1", (O.RS, 8, 2), (32, 8, 128, 8), 16, 5, 1, 0),
    ("llama70b_tp8_rs82_m2048", (O.RS, 8, 2), (80, 8, 128, 8), 2048, 2048, 0, 0),
    ("rs62_2L6H64D_tp6_m16", (O.RS, 6, 2), (2, 6, 64, 6), 16, 16, 0, 0),
    ("tiny_2L4H8D_tp2_xor2_m16_valid5", (O.XOR, 2, 1), (2, 4, 8, 2), 16, 5, 3, 1),
    ("tiny_2L8H8D_tp4_rs42_m16", (O.RS, 4, 2), (2, 8, 8, 4), 16, 16, 11, 2),
]
KV_SEED = 3  # simulator.hpp:48 / config.hpp:37 default kv_seed


def fnv(buf) -> str:
    return f"{O.ref().fnv1a64(buf):016x}"


def main() -> None:
    R = O.ref()
    out = {"generator": "tests/golden/make_golden.py via oracle/_ref (reference headers in place)"}

    e, lg = R.gf_tables()
    mt = R.mul_table()
    out["gf"] = {
        "exp_hex": e.tobytes().hex(),
        "log_hex": lg.tobytes().hex(),
        "mul_table_sha256": hashlib.sha256(mt.tobytes()).hexdigest(),
        "inv_hex": bytes([0] + [R.gf_inv(a) for a in range(1, 256)]).hex(),
        "known": {"mul_02_03": R.gf_mul(2, 3), "mul_80_02": R.gf_mul(0x80, 2),
                  "mul_00_ff": R.gf_mul(0, 0xFF), "mul_ff_01": R.gf_mul(0xFF, 1),
                  "inv_02": R.gf_inv(2), "inv_01": R.gf_inv(1)},
    }

    out["matrices"] = {
        f"{kind}_{n}_{k}": R.encoding_matrix(kind, n, k).tobytes().hex()
        for kind, n, k in SCHEMES + MATRIX_ONLY
    }

    enc = []
    seed = 1
    for kind, n, k in SCHEMES:
        for ln in HEX_LENGTHS + FNV_LENGTHS:
            data = [splitmix_bytes(seed * 1000 + j, ln) for j in range(n)]
            par = R.encode(kind, n, k, data)
            rec = {"kind": kind, "n": n, "k": k, "len": ln, "seed": seed,
                   "parity_fnv": [fnv(p) for p in par]}
            if ln in HEX_LENGTHS:
                rec["parity_hex"] = [p.tobytes().hex() for p in par]
            # every erasure pattern within tolerance, rebuilt bytes == data
            tol = R_tol(kind, k)
            pats = []
            if ln == 17 and n + k <= 10:
                for e_ in range(1, tol + 1):
                    for lost in itertools.combinations(range(n + k), e_):
                        shards = {i: data[i] for i in range(n)}
                        shards.update({n + i: par[i] for i in range(k)})
                        got = R.reconstruct(kind, n, k, shards, list(lost))
                        pats.append({"lost": list(lost),
                                     "rebuilt_fnv": {str(i): fnv(b) for i, b in got.items()}})
                rec["patterns"] = pats
            enc.append(rec)
            seed += 1
    out["encode"] = enc

    # error behaviour (coding.hpp:44-60, 463-486, 543-551)
    errs = []
    for kind, n, k in [(O.XOR, 4, 2), (O.RS, 4, 5), (O.RS, 300, 1), (O.RS, 0, 1), (O.RS, 4, 0),
                       (O.RDP, 4, 1), (O.RS, 250, 5), (O.RS, 250, 6)]:
        errs.append({"op": "validate", "kind": kind, "n": n, "k": k,
                     "status": R.fn("validate")(kind, n, k)})
    data = [splitmix_bytes(77 + j, 16) for j in range(8)]
    par = R.encode(O.RS, 8, 2, data)
    for lost, drop in [([0, 1, 2], None), ([10], None), ([-1], None), ([0], 9), ([0, 8, 9], None),
                       ([8, 9], None), ([0, 0], None), ([3, 8], None)]:
        shards = {i: data[i] for i in range(8)}
        shards.update({8 + i: par[i] for i in range(2)})
        if drop is not None:
            shards.pop(drop)
        try:
            got = R.reconstruct(O.RS, 8, 2, shards, lost)
            st, rebuilt = 0, sorted(got)
        except O.OracleError as ex:
            st, rebuilt = ex.status, []
        errs.append({"op": "reconstruct", "kind": O.RS, "n": 8, "k": 2, "lost": lost,
                     "drop": drop, "status": st, "rebuilt": rebuilt})
    out["errors"] = errs

    kv = []
    for name, (kind, n, k), (L, H, D, tp), m, valid, req, chunk in KV_CASES:
        sb = R.slice_bytes(L, H, D, tp, m)
        slices = [R.make_ground_truth_slice(KV_SEED, req, chunk, w, L, H, D, tp, m, valid)
                  for w in range(n)]
        par = R.encode(kind, n, k, slices)
        kv.append({"name": name, "kind": kind, "n": n, "k": k, "model": [L, H, D, tp],
                   "chunk_size": m, "valid": valid, "request": req, "chunk": chunk,
                   "kv_seed": KV_SEED, "slice_bytes": sb,
                   "data_fnv": [fnv(s) for s in slices],
                   "data_head_hex": [s[:16].tobytes().hex() for s in slices],
                   "parity_fnv": [fnv(p) for p in par],
                   "parity_head_hex": [p[:16].tobytes().hex() for p in par],
                   "checksum": f"{R.parity_checksum(par):016x}"})
        print(name, sb, [fnv(p) for p in par], flush=True)
    out["kv"] = kv

    out["slice_bytes"] = [
        {"model": [2, 4, 8, 2], "m": 16, "bytes": R.slice_bytes(2, 4, 8, 2, 16)},
        {"model": [80, 8, 128, 8], "m": 2048, "bytes": R.slice_bytes(80, 8, 128, 8, 2048)},
        {"model": [32, 8, 128, 8], "m": 16, "bytes": R.slice_bytes(32, 8, 128, 8, 16)},
        {"model": [2, 4, 8, 1], "m": 16, "bytes": R.slice_bytes(2, 4, 8, 1, 16)},
    ]
    out["fnv"] = {"empty": fnv(np.zeros(0, np.uint8)),
                  "a": fnv(np.frombuffer(b"a", np.uint8)),
                  "foobar": fnv(np.frombuffer(b"foobar", np.uint8))}

    # GSRV image written by the reference's serialize_parity_store
    import ctypes as C
    keys = [(7, 2, 16), (3, 0, 16), (3, 1, 5)]  # (request, chunk, valid): out of order on purpose
    gl, gk = 33, 2
    pars = [splitmix_bytes(5000 + 10 * i + j, gl) for i in range(len(keys)) for j in range(gk)]
    req = (C.c_uint64 * 3)(*[x[0] for x in keys])
    chk = (C.c_uint32 * 3)(*[x[1] for x in keys])
    val = (C.c_uint32 * 3)(*[x[2] for x in keys])
    size = C.c_uint64()
    buf = np.zeros(4096, np.uint8)
    assert R.fn("gsrv_image")(O.RS, 4, gk, 3, req, chk, val, C.c_uint64(gl), O._ptrs(pars),
                              buf.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_uint64(4096), C.byref(size)) == 0
    out["gsrv"] = {"kind": O.RS, "n": 4, "k": gk, "slice_len": gl, "keys": keys, "parity_seed": 5000,
                   "image_hex": buf[: size.value].tobytes().hex()}

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path, os.path.getsize(path), "bytes")


def R_tol(kind: int, k: int) -> int:
    return 1 if kind == O.XOR else (2 if kind == O.RDP else k)


if __name__ == "__main__":
    main()
