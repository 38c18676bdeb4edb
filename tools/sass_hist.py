"""SASS opcode histograms of the hot kernels (cuobjdump -sass of the built
objects, no GPU needed): evidence of what each kernel issues -- 128-bit
global loads/stores, UBLKCP / SYNCS (TMA bulk copies + mbarriers),
UCGABAR / cluster (DSMEM) traffic, the LOP3 / IMAD split of the GF(2^8)
arithmetic.

  python tools/sass_hist.py --out profiles/r2_sass_opcodes.json
"""
import argparse
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2605_00831_b200", "_lib", "obj")

KERNELS = [
    ("K1 register (ldg128) RS(8,2) encode", "gs_special_enc.o", r"k_apply_specialINS_7EncSpecILi2ELi8ELi2EEELi488ELi1ELb0E"),
    ("K1 bulk (TMA smem ring) RS(8,2) encode", "gs_special_enc.o", r"k_apply_special_bulkINS_7EncSpecILi2ELi8ELi2EEE"),
    ("K1 paged RS(8,2) encode", "gs_special_enc.o", r"k_apply_specialINS_7EncSpecILi2ELi8ELi2EEELi488ELi1ELb1E"),
    ("K2 RS(8,2) lost {5}", "gs_special_dec_kreedsolomon_8_2_e1.o", r"k_apply_specialINS_7DecSpecILi2ELi8ELi2ELm32EEELi488ELi1ELb0E"),
    ("GPU FNV-1a window, bit-sliced, two bits per round (default)", "gs_fnv_gpu.o", r"k_fnv_window_sl2"),
    ("GPU FNV-1a window, bit-sliced, one bit per round (GS_FNV_PAIRS=0)", "gs_fnv_gpu.o", r"k_fnv_window_slENS"),
    ("GPU FNV-1a window, byte-lane rounds (GS_FNV_WINDOW_BYTES=1)", "gs_fnv_gpu.o", r"k_fnv_windowENS"),
    ("GPU FNV-1a legacy pair pass (round 1)", "gs_fnv_gpu.o", r"k_fnv_pairILi2E"),
    ("RDP(p=11) rebuild of columns {0,10}, pipelined", "gs_rdp_pairs_p11_i0.o", r"k_rdp_recover_bulkILi488ELi11ELi0ELi10EE"),
]


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            body.append(line)
    if cur:
        yield cur, body


def hist(body):
    h = collections.Counter()
    for line in body:
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*(?:\.[A-Z0-9_]+)*)", line)
        if m:
            op = m.group(1)
            base = op.split(".")[0]
            key = op if base in ("LDG", "STG", "LDS", "STS", "UBLKCP", "SYNCS", "ATOMG", "RED", "LD", "ST") else base
            h[key] += 1
    return h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_sass_opcodes.json"))
    a = ap.parse_args()
    res = {}
    for label, obj, pat in KERNELS:
        for name, body in functions(obj):
            if re.search(pat, name):
                h = hist(body)
                res[label] = {"function": name, "instructions": sum(h.values()),
                              "opcodes": dict(sorted(h.items(), key=lambda kv: -kv[1]))}
                break
        else:
            res[label] = {"missing": pat}
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    for k, v in res.items():
        top = list(v.get("opcodes", {}).items())[:10]
        print(f"{k}: {v.get('instructions')} instr; {top}")


if __name__ == "__main__":
    main()
