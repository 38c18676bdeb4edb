"""Host-link evidence for ncu (tools/profile_r2.sh): one headline step (the
C3 checkpoint of one 2K-token chunk: K1 + piecewise D2H of 2 x 80 MiB of
parity into pinned host memory) one C3 chunk rebuild (H2D of parity row
0 + K2) and one e2e call (gs_encode_host from pinned host buffers: H2D of the
8 x 80 MiB data + K1 + D2H of the parity), each bracketed by cudaProfilerStart/Stop so that

  ncu --replay-mode app-range \
      --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum,... \
      python tools/link_capture.py --leg encode|rebuild|e2e

measures the PCIe bytes and the elapsed time of the whole range -- copies
and kernels together -- i.e. the achieved D2H / H2D GB/s against the host
link, with the copy/compute overlap inside it.
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00831_b200 import _lib as L  # noqa: E402
from paper_2605_00831_b200 import device as D  # noqa: E402
from paper_2605_00831_b200 import kv_layout as K  # noqa: E402
from paper_2605_00831_b200.coding import CodingScheme, ErasurePattern, check, decoder, encoder  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--leg", choices=["encode", "rebuild", "e2e"], default="encode")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg, m = K.LLAMA3_70B, 2048
    sl = K.slice_bytes(cfg, m)
    kv = torch.empty((8, sl), dtype=torch.uint8, device=dev)
    for w in range(8):
        K.make_ground_truth_slice(3, 0, 0, w, cfg, m, m, out=kv[w])
    h_par = D.pinned_near((2, sl), 0)
    scheme = CodingScheme.reed_solomon(8, 2)
    pipe = D.Pipeline(0, 256 << 20)
    comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
    lib = L.lib()
    slots = L.ptr_array([kv[w].data_ptr() for w in range(8)])
    outs = L.ptr_array([h_par[i].data_ptr() for i in range(2)])
    enc = encoder(scheme)

    def encode():
        check(lib.gs_encode_offload(pipe.handle, enc.handle, 1, slots, outs, sl, comp.cuda_stream,
                                    copy.cuda_stream), "encode")
    encode()
    torch.cuda.synchronize()
    dec = decoder(scheme, ErasurePattern([5]))
    rebuilt = torch.empty(sl, dtype=torch.uint8, device=dev)
    rslots = L.ptr_array([None if j == 5 else (kv[j].data_ptr() if j < 8 else h_par[j - 8].data_ptr())
                          for j in range(10)])
    routs = L.ptr_array([rebuilt.data_ptr()])

    def rebuild():
        check(lib.gs_reconstruct_upload(pipe.handle, dec.handle, 1, rslots, routs, sl, comp.cuda_stream,
                                        copy.cuda_stream), "rebuild")
    rebuild()
    torch.cuda.synchronize()
    # e2e: the drop-in host-buffer call (gs_encode_host = ghostserve::encode
    # semantics): H2D of the 8 x 80 MiB data, K1, D2H of the parity
    h_kv = kv.cpu().pin_memory()
    h_par2 = D.pinned_near((2, sl), 0)
    hslots = L.ptr_array([h_kv[w].data_ptr() for w in range(8)])
    houts = L.ptr_array([h_par2[i].data_ptr() for i in range(2)])

    def e2e():
        check(lib.gs_encode_host(pipe.handle, enc.handle, hslots, houts, sl), "e2e")
    e2e()
    torch.cuda.synchronize()
    cudart = torch.cuda.cudart()
    cudart.cudaProfilerStart()
    {"encode": encode, "rebuild": rebuild, "e2e": e2e}[a.leg]()
    comp.wait_stream(copy)
    torch.cuda.synchronize()
    cudart.cudaProfilerStop()
    want = D.encode(scheme, kv.unsqueeze(0))[0]
    ok = (torch.equal(rebuilt, kv[5]) if a.leg == "rebuild" else
          torch.equal((h_par2 if a.leg == "e2e" else h_par).to(dev), want))
    d2h = 2 * sl if a.leg in ("encode", "e2e") else 0
    h2d = {"encode": 0, "rebuild": sl, "e2e": 8 * sl}[a.leg]
    print(f"link_capture {a.leg}: bytes D2H {d2h}, H2D {h2d}, ok={ok}")


if __name__ == "__main__":
    main()
