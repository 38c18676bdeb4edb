"""Launch one kernel configuration a few times for ncu (not a benchmark):
    ncu --set full -k regex:k_apply -c 1 python tools/profile_k1.py --variant 1 --mib 8
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L  # noqa: E402
from paper_2605_00831_b200 import device as D  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, check  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", type=int, default=2)
    ap.add_argument("--mib", type=float, default=8)
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--decode", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    check(L.lib().gs_set_kernel_variant(a.variant))
    L_ = int(a.mib * (1 << 20))
    sch = CodingScheme.reed_solomon(a.n, a.k)
    data = torch.randint(0, 256, (a.n, L_), dtype=torch.uint8, device="cuda")
    par = D.encode(sch, data)
    for _ in range(a.reps):
        if a.decode:
            sh = {j: data[j] for j in range(1, a.n)}
            sh.update({a.n + i: par[i] for i in range(a.k)})
            D.reconstruct(sch, sh, ErasurePattern([0]))
        else:
            D.encode(sch, data, out=par)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
