import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2605_00831_b200 import _lib as L
from paper_2605_00831_b200.coding import CodingScheme, check, encoder
lib = L.lib(); dev = torch.device("cuda", 0); st = torch.cuda.Stream()
n, k, ln = 4, 2, 128 << 20
data = torch.randint(0, 256, (n, ln), dtype=torch.uint8, device=dev); out = torch.empty((k, ln), dtype=torch.uint8, device=dev)
enc = encoder(CodingScheme.reed_solomon(n, k))
lib.gs_set_kernel_variant(int(sys.argv[1]))
for _ in range(3):
    check(lib.gs_apply_device(enc.handle, 1, L.ptr_array([data[j].data_ptr() for j in range(n)]), L.ptr_array([out[i].data_ptr() for i in range(k)]), ln, st.cuda_stream), "k1")
st.synchronize()
