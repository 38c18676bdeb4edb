import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2605_00831_b200.coding import CodingScheme
from paper_2605_00831_b200.parity_store import ParityStore
S, K, SL = 32, 2, 262144
sch = CodingScheme.reed_solomon(8, 2)
st = ParityStore(seal_threads=4); st.bind_device(0)
def runs(dst):
    r = 1
    for a, b in zip(dst, dst[1:]):
        if b != a + SL: r += 1
    return r
for phase in range(3):
    res = []
    for b in range(8):
        acc, dst = st.reserve_batch([(s, b) for s in range(S)], sch, 16, SL)
        res.append(runs(dst))
        st.commit_batch([(s, b) for s in range(S)])
    st.wait_sealed()
    print("phase", phase, "runs per block", res, flush=True)
    for s in range(S): st.erase_request(s)
