"""C2 block recovery (H2D of parity row 0 for 32 requests + K2 over 7
survivors) timed with CUDA events, many repetitions; for piece-size A/B
(GS_UPLOAD_PIECES)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, check, decoder  # noqa: E402
from paper_2605_00831_b200.device import Pipeline  # noqa: E402

S, N, K, SL = 32, 8, 2, 262144


def main():
    dev = torch.device("cuda", 0)
    dec = decoder(CodingScheme.reed_solomon(N, K), ErasurePattern([5]))
    data = torch.randint(0, 256, (S, N, SL), dtype=torch.uint8, device=dev)
    hpar = torch.randint(0, 256, (S, K, SL), dtype=torch.uint8).pin_memory()
    out = torch.empty((S, SL), dtype=torch.uint8, device=dev)
    slots = []
    for s in range(S):
        row = [data[s, j].data_ptr() if j != 5 else None for j in range(N)] + [hpar[s, i].data_ptr() for i in range(K)]
        slots += row
    sl, ol = L.ptr_array(slots), L.ptr_array([out[s].data_ptr() for s in range(S)])
    pipe = Pipeline(0, 256 << 20)
    comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
    ts = []
    for it in range(40):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        check(L.lib().gs_reconstruct_upload(pipe.handle, dec.handle, S, sl, ol, SL, comp.cuda_stream, copy.cuda_stream), "r")
        e1.record(comp)
        e1.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"pieces": os.environ.get("GS_UPLOAD_PIECES", "4"), "median_ms": round(ts[len(ts) // 2], 4),
                      "min_ms": round(ts[0], 4)}))


if __name__ == "__main__":
    main()
