# One round's GPU evidence: ncu --set full of K1 (C2 launch), K2 (single
# loss) and paged K1 taken from bench.py's own launches, RDP encode/rebuild at
# 64 MiB columns, the GPU FNV-1a round kernel (C3 parity batch) and its
# per-launch list, the launch list of a short bench run, and the default bench
# line. Run under gpurun; summarise here with tools/ncu_summary.py.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu --no-c3 --no-c4 --no-overhead"
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 600 $N -k regex:EncSpec -s 5 -c 1 -f -o gpurun_out/k1_r1 $B > gpurun_out/ncu_k1.log 2>&1
timeout 600 $N -k regex:DecSpec -s 2 -c 1 -f -o gpurun_out/k2_r1 $B > gpurun_out/ncu_k2.log 2>&1
timeout 600 $N -k 'regex:EncSpec.*bool.1' -s 2 -c 1 -f -o gpurun_out/k1p_r1 $B > gpurun_out/ncu_k1p.log 2>&1
timeout 600 $N -k regex:k_rdp_recover_bulk -s 2 -c 1 -f -o gpurun_out/rdp_rec_r1 python tools/kernel_sweep.py --kind rdp --lost 1,3 --sizes 64 > gpurun_out/ncu_rdp.log 2>&1
timeout 600 $N -k regex:k_fnv_pair -s 5 -c 1 -f -o gpurun_out/fnv_pair_r1 python tools/fnv_probe.py --configs C3 > gpurun_out/ncu_fnv.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fnv -c 10 --csv --log-file gpurun_out/fnv_launches_r1.csv python tools/fnv_probe.py --configs C3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_r1.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
tail -2 gpurun_out/bench_r1.err
ls -la gpurun_out
