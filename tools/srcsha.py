"""sha256[:16] of the product library's SOURCES (csrc/*.cu, *.cuh, *.hpp,
Makefile, include/gs_capi.h): the key that ties a committed ncu capture to
the build it profiled. The built .so is not byte-reproducible across nvcc
runs, so its own hash would orphan every capture on the next rebuild."""
import glob
import hashlib
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def source_sha() -> str:
    csrc = os.path.join(ROOT, "paper_2605_00831_b200", "csrc")
    files = sorted(glob.glob(os.path.join(csrc, "*.cu")) + glob.glob(os.path.join(csrc, "*.cuh"))
                   + glob.glob(os.path.join(csrc, "*.hpp")) + glob.glob(os.path.join(csrc, "*.cpp"))
                   + [os.path.join(csrc, "Makefile"), os.path.join(ROOT, "include", "gs_capi.h")])
    h = hashlib.sha256()
    for p in files:
        h.update(os.path.relpath(p, ROOT).encode() + b"\0")
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


if __name__ == "__main__":
    print(source_sha())
