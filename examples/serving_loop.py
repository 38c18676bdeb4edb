"""A serving loop with shadow checkpointing, end to end on one B200.

What a GhostServe user switching to this library writes (reference flow:
checkpoint.hpp:179-281, recovery.hpp:176-298):

  1. prefill a request chunk by chunk, checkpointing every chunk's TP-sharded
     KV (K1 encode + D2H of the parity into the pinned host tier, FNV seal on
     host threads);
  2. decode token by token; every m tokens the DecodeCheckpointer emits the
     next chunk's checkpoint, and the masked tail is flushed at request end;
  3. a worker (GPU) fails: recover() plans recompute vs erasure decode with a
     cost model calibrated on this box, verifies the parity, H2D's it and
     rebuilds the lost worker's KV (K2) -- bit-exact.

    python examples/serving_loop.py [--model 8b|70b] [--tokens 8192] [--decode 100]

(The first prefill of a process also pays the host tier's pinned-slab and the
device allocator's first allocations; bench.py times warm passes.)
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_00831_b200 import kv_layout as K  # noqa: E402
from paper_2605_00831_b200.checkpoint import (CheckpointConfig, Checkpointer, CostModel,  # noqa: E402
                                              DecodeCheckpointer, FailureEvent)
from paper_2605_00831_b200.coding import CodingScheme  # noqa: E402
from paper_2605_00831_b200.parity_store import ParityStore  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", choices=["8b", "70b"], default="8b")
    ap.add_argument("--tokens", type=int, default=8192, help="prompt tokens (prefill)")
    ap.add_argument("--decode", type=int, default=100, help="decode tokens after the prefill")
    ap.add_argument("--chunk", type=int, default=2048)
    ap.add_argument("--lost", type=int, default=5, help="worker (TP rank) that fails")
    a = ap.parse_args()
    model = K.LLAMA3_8B if a.model == "8b" else K.LLAMA3_70B
    scheme = CodingScheme.reed_solomon(8, 2)
    # cost model: the reference's constants for compute; host link and kernel
    # rates as measured on B200 (bench.py): 55 GB/s H2D, K1 ~5 TB/s, K2 ~5 TB/s
    cost = CostModel.measured(55.0, 4300.0, 4700.0)
    cfg = CheckpointConfig(scheme, a.chunk, model, cost)
    store = ParityStore(seal_threads=max(1, (os.cpu_count() or 2) - 2))
    store.bind_device(0)
    ck = Checkpointer(cfg, store, device=0)
    req = 7

    t0 = time.perf_counter()
    run = ck.run_prefill_with_checkpointing(req, a.tokens, kv_seed=3)
    ck.synchronize()
    t_prefill = time.perf_counter() - t0
    print(f"prefill: {run.chunks_done} chunks of {a.chunk} tokens checkpointed "
          f"({run.chunks_done * 8 * K.slice_bytes(model, a.chunk) / 2**30:.2f} GiB of KV, "
          f"{run.device_ms:.1f} ms on the device, sealed after {t_prefill * 1e3:.0f} ms)")

    # decode: the partially filled last prefill chunk continues filling; emit
    # a checkpoint every `chunk` tokens, flush the masked tail at the end
    dec = DecodeCheckpointer(req, run.chunks_done, ck, kv_seed=3)
    emitted = 0
    for _ in range(a.decode):
        emitted += dec.step(run.state) is not None
    tail = dec.flush(run.state)
    ck.synchronize()
    print(f"decode: {a.decode} tokens, {emitted} full chunk checkpoint(s) + "
          f"{'a masked tail of %d tokens' % tail.valid_tokens if tail else 'no tail'}")

    # failure of one worker: recover every checkpointed chunk of the request
    ground = run.ground_truth + dec.ground_truth
    tokens = [s[0].valid_tokens for s in ground]
    res = ck.recover(req, FailureEvent([a.lost], at_chunk=len(ground)), ground, tokens)
    print(f"recovery of worker {a.lost}: plan {res.plan.mode} (recompute {res.plan.recompute_chunks}, "
          f"decode {len(res.plan.reconstruct_ids)} chunks), parity verified in {res.verify_host_ms:.1f} ms, "
          f"H2D + K2 {res.reconstruct_device_ms:.2f} ms, {res.wall_ms:.1f} ms wall, "
          f"bit-exact: {res.verified}")
    ck.close()
    if not res.verified:
        sys.exit(1)


if __name__ == "__main__":
    if not torch.cuda.is_available():
        sys.exit("needs a CUDA device (B200)")
    main()
