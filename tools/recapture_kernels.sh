mkdir -p gpurun_out
python tools/srcsha.py > gpurun_out/src_sha.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
B="python bench.py --steps 6 --warmup 3 --no-cpu --no-c3 --no-c4 --no-overhead"
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 900 $N -k regex:EncSpec -s 4 -c 1 -f -o gpurun_out/k1_c3 $B > gpurun_out/ncu_k1_c3.log 2>&1
timeout 900 $N -k regex:EncSpec -s 5 -c 1 -f -o gpurun_out/k1_c2 $B --workload c2 > gpurun_out/ncu_k1_c2.log 2>&1
timeout 900 $N -k regex:DecSpec -s 2 -c 1 -f -o gpurun_out/k2_c3 $B > gpurun_out/ncu_k2_c3.log 2>&1
timeout 900 $N -k 'regex:EncSpec.*bool.1' -s 2 -c 1 -f -o gpurun_out/k1p_c3 $B > gpurun_out/ncu_k1p_c3.log 2>&1
timeout 900 $N -k 'regex:EncSpec.*bool.1' -s 2 -c 1 -f -o gpurun_out/k1p_c2 $B --workload c2 > gpurun_out/ncu_k1p_c2.log 2>&1
GS_PROFILE_TIMED=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-c3 --no-c4 --no-overhead > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/gpu_tests.log
ls gpurun_out/*.ncu-rep
