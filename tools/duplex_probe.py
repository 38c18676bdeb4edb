"""H2D of a C3 step's 640 MiB of KV alone and with the step's 160 MiB parity
D2H running concurrently on another stream (the e2e leg's bound)."""
import json
import time

import torch

PER = 83886080
a = torch.randint(0, 256, (8, PER), dtype=torch.uint8).pin_memory()
b = torch.empty((2, PER), dtype=torch.uint8).pin_memory()
d = torch.empty((8, PER), dtype=torch.uint8, device="cuda")
p = torch.randint(0, 256, (2, PER), dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(with_d2h, reps=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1):
            d.copy_(a, non_blocking=True)
        if with_d2h:
            with torch.cuda.stream(s2):
                b.copy_(p, non_blocking=True)
    torch.cuda.synchronize()
    return reps * 8 * PER / (time.perf_counter() - t0) / 1e9


run(True, 3)
print(json.dumps({"h2d_alone_gbs": round(run(False), 2), "h2d_with_concurrent_d2h_gbs": round(run(True), 2),
                  "e2e_bound_gbs_of_kv": "= the second number (the step moves 640 MiB in, 160 MiB out)"}))
