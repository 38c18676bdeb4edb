# Round-2 GPU evidence, first pass (run under gpurun; summarised here with
# tools/ncu_summary.py, tools/launch_summary.py and tools/link_summary.py into
# profiles/r2_*; the closing captures of the final sources are
# tools/profile_final.sh and tools/recapture_kernels.sh):
#  * ncu --set full of K1 / K2 / paged K1 at the C3 launch (one 2K-token chunk,
#    8 x 80 MiB) from bench.py's own launches, K1 at the C2 launch, the GPU
#    FNV-1a window kernel (and the legacy multi-pass one for A/B);
#  * the launch list (gpu__time_duration per launch) of a short C3 bench run;
#  * ncu range captures of the host-link legs: one headline step (K1 + D2H)
#    and one chunk rebuild (H2D + K2): PCIe bytes + elapsed time;
#  * the default bench line, the reference arm, the C5 sweep and the
#    small-L probe; SASS opcode histograms are made locally (cuobjdump).
# tools/srcsha.py (a hash of the kernel sources) is recorded so bench.py
# only reports roofline.traffic for the sources that were captured.
set -x
mkdir -p gpurun_out
sha256sum paper_2605_00831_b200/_lib/libghostserve_b200.so | cut -c1-16 > gpurun_out/lib_sha.txt
python tools/srcsha.py > gpurun_out/src_sha.txt
B="python bench.py --steps 6 --warmup 3 --no-cpu --no-c3 --no-c4 --no-overhead"
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 900 $N -k regex:EncSpec -s 4 -c 1 -f -o gpurun_out/k1_c3_r2 $B > gpurun_out/ncu_k1_c3.log 2>&1
timeout 900 $N -k regex:DecSpec -s 2 -c 1 -f -o gpurun_out/k2_c3_r2 $B > gpurun_out/ncu_k2_c3.log 2>&1
timeout 900 $N -k 'regex:EncSpec.*bool.1' -s 2 -c 1 -f -o gpurun_out/k1p_c3_r2 $B > gpurun_out/ncu_k1p_c3.log 2>&1
timeout 900 $N -k regex:EncSpec -s 5 -c 1 -f -o gpurun_out/k1_c2_r2 $B --workload c2 > gpurun_out/ncu_k1_c2.log 2>&1
timeout 600 $N -k regex:k_fnv_window -s 2 -c 1 -f -o gpurun_out/fnv_window_r2 python tools/fnv_probe.py --configs C3 > gpurun_out/ncu_fnv.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fnv -c 12 --csv --log-file gpurun_out/fnv_launches_r2.csv python tools/fnv_probe.py --configs C3 > /dev/null 2>&1
GS_FNV_LEGACY=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fnv -c 12 --csv --log-file gpurun_out/fnv_launches_legacy_r2.csv python tools/fnv_probe.py --configs C3 > /dev/null 2>&1
GS_PROFILE_TIMED=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_r2.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-c3 --no-c4 --no-overhead > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c3_whole_r2.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-c3 --no-c4 --no-overhead > gpurun_out/ncu_launch_whole.log 2>&1
L="--replay-mode app-range --clock-control none --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu $L --csv --log-file gpurun_out/link_encode_r2.csv python tools/link_capture.py --leg encode > gpurun_out/link_encode.log 2>&1
timeout 900 ncu $L --csv --log-file gpurun_out/link_rebuild_r2.csv python tools/link_capture.py --leg rebuild > gpurun_out/link_rebuild.log 2>&1
timeout 300 python tools/small_l_probe.py 65536 262144 1048576 4194304 > gpurun_out/small_l_r2.jsonl 2> gpurun_out/small_l_r2.err
timeout 300 python tools/fnv_probe.py > gpurun_out/fnv_probe_r2.jsonl 2>&1
GS_FNV_LEGACY=1 timeout 300 python tools/fnv_probe.py > gpurun_out/fnv_probe_legacy_r2.jsonl 2>&1
timeout 900 python bench.py --sweep > gpurun_out/c5_sweep_r2.jsonl 2> gpurun_out/c5_sweep_r2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_r2.json 2> gpurun_out/bench_ref_r2.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err
timeout 900 python bench.py --workload c2 --steps 20 --warmup 5 > gpurun_out/bench_c2_r2.json 2> gpurun_out/bench_c2_r2.err
ls -la gpurun_out
