"""Decode-step interference of the block checkpoint alone (bench.decode_overhead, twice)."""
import sys, os, json, torch, argparse
sys.path.insert(0, os.getcwd())
import bench
from paper_2605_00831_b200 import device as D
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
a = argparse.Namespace(decode_ctx=4096)
pipe = D.Pipeline(0, 256 << 20)
for _ in range(2):
    print(json.dumps(bench.decode_overhead(torch, dev, pipe, a)), flush=True)
