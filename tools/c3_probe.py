"""C3 orchestrated checkpoint + recovery alone (bench.c3_orchestrated, which
recovers the same failure 3 times), for iterating on the recovery schedule
without the full bench."""
import json, sys, os, torch
sys.path.insert(0, os.getcwd())
import bench
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    r = bench.c3_orchestrated(torch, dev, {"h2d": 55.5, "d2h": 57.0}, 4398.0, 4700.0)
    print(json.dumps({k: v for k, v in r.items() if k not in ("note", "cost_model_measured", "plan")}), flush=True)
