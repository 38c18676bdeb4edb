"""sha256[:16] of the sources that determine the profiled codec kernels (K1 /
K2 / paged K1: their code and their launch geometry): gs_kernels.cuh,
gs_special.cuh, gs_special_*.cu, gs_field.hpp, gs_capi.cu (the launch
configuration), the Makefile (flags) and include/gs_capi.h. The key that ties
a committed ncu capture to the build it profiled -- the built .so is not
byte-reproducible across nvcc runs, so its own hash would orphan every
capture on the next rebuild, and host-only sources (the store, the host FNV)
do not change these kernels."""
import glob
import hashlib
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def source_sha() -> str:
    csrc = os.path.join(ROOT, "paper_2605_00831_b200", "csrc")
    files = sorted([os.path.join(csrc, f) for f in ("gs_kernels.cuh", "gs_special.cuh", "gs_field.hpp",
                                                    "gs_capi.cu", "Makefile")]
                   + glob.glob(os.path.join(csrc, "gs_special_*.cu"))
                   + [os.path.join(ROOT, "include", "gs_capi.h")])
    h = hashlib.sha256()
    for p in files:
        h.update(os.path.relpath(p, ROOT).encode() + b"\0")
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


if __name__ == "__main__":
    print(source_sha())
