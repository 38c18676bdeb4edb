# Round-2 closing evidence on one B200 (run under gpurun; summarised here into
# profiles/ with tools/ncu_summary.py and tools/launch_summary.py):
#  * the GPU parity suite and smoke();
#  * the default bench line (C3), the reference arm, the C2 line, the C1-C4 table;
#  * ncu --set full of K1 at the C3 and C2 launches (bench.py's roofline.traffic
#    reads these, keyed by tools/srcsha.py), K2 at C3, paged K1 at C2 and C3;
#  * the launch list of exactly the timed steps of the default bench.
# The rest of the round's closing evidence has its own scripts: tools/sanitize_run.sh
# (compute-sanitizer), tools/soak.sh (20x fuzz), tools/gpu_relay_check.sh (the N>1
# path with 2/4/8 ranks sharing the GPU), tools/recapture_kernels.sh (ncu only).
set -x
mkdir -p gpurun_out
python tools/srcsha.py > gpurun_out/src_sha.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --workload c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1200 python bench.py --configs > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
B="python bench.py --steps 6 --warmup 3 --no-cpu --no-c3 --no-c4 --no-overhead"
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 900 $N -k regex:EncSpec -s 4 -c 1 -f -o gpurun_out/k1_c3 $B > gpurun_out/ncu_k1_c3.log 2>&1
timeout 900 $N -k regex:EncSpec -s 5 -c 1 -f -o gpurun_out/k1_c2 $B --workload c2 > gpurun_out/ncu_k1_c2.log 2>&1
timeout 900 $N -k regex:DecSpec -s 2 -c 1 -f -o gpurun_out/k2_c3 $B > gpurun_out/ncu_k2_c3.log 2>&1
timeout 900 $N -k 'regex:EncSpec.*bool.1' -s 2 -c 1 -f -o gpurun_out/k1p_c3 $B > gpurun_out/ncu_k1p_c3.log 2>&1
timeout 900 $N -k 'regex:EncSpec.*bool.1' -s 2 -c 1 -f -o gpurun_out/k1p_c2 $B --workload c2 > gpurun_out/ncu_k1p_c2.log 2>&1
GS_PROFILE_TIMED=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-c3 --no-c4 --no-overhead > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
