# One gpurun call: GPU parity suite, smoke, default bench + reference arm,
# and the ncu --set full captures of K1 (C3 and C2 launches) that bench.py's
# roofline.traffic reads (keyed by tools/srcsha.py).
set -x
mkdir -p gpurun_out
python tools/srcsha.py > gpurun_out/src_sha.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
B="python bench.py --steps 6 --warmup 3 --no-cpu --no-c3 --no-c4 --no-overhead"
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 900 $N -k regex:EncSpec -s 4 -c 1 -f -o gpurun_out/k1_c3 $B > gpurun_out/ncu_k1_c3.log 2>&1
timeout 900 $N -k regex:EncSpec -s 5 -c 1 -f -o gpurun_out/k1_c2 $B --workload c2 > gpurun_out/ncu_k1_c2.log 2>&1
ls -la gpurun_out
