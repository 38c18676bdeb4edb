# Round-2 GPU evidence (run under gpurun; summarise here with tools/ncu_summary.py):
# ncu --set full of K1 / K2 / paged K1 at the C3 launch (one 2K-token chunk,
# 8 x 80 MiB) taken from bench.py's own launches, K1 at the C2 launch, the GPU
# FNV-1a kernels on a C3 parity batch, the launch list of a short C3 bench run,
# and the SASS opcode histograms. The library's sha is recorded so bench.py
# only reports roofline.traffic for the build that was captured.
set -x
mkdir -p gpurun_out
sha256sum paper_2605_00831_b200/_lib/libghostserve_b200.so | cut -c1-16 > gpurun_out/lib_sha.txt
B="python bench.py --steps 6 --warmup 3 --no-cpu --no-c3 --no-c4 --no-overhead"
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 900 $N -k regex:EncSpec -s 4 -c 1 -f -o gpurun_out/k1_c3_r2 $B > gpurun_out/ncu_k1_c3.log 2>&1
timeout 900 $N -k regex:DecSpec -s 2 -c 1 -f -o gpurun_out/k2_c3_r2 $B > gpurun_out/ncu_k2_c3.log 2>&1
timeout 900 $N -k 'regex:EncSpec.*bool.1' -s 2 -c 1 -f -o gpurun_out/k1p_c3_r2 $B > gpurun_out/ncu_k1p_c3.log 2>&1
timeout 900 $N -k regex:EncSpec -s 5 -c 1 -f -o gpurun_out/k1_c2_r2 $B --workload c2 > gpurun_out/ncu_k1_c2.log 2>&1
timeout 600 $N -k regex:k_fnv_window -s 2 -c 1 -f -o gpurun_out/fnv_window_r2 python tools/fnv_probe.py --configs C3 > gpurun_out/ncu_fnv.log 2>&1
GS_FNV_LEGACY=1 timeout 600 $N -k regex:k_fnv_pair -s 5 -c 1 -f -o gpurun_out/fnv_pair_r2 python tools/fnv_probe.py --configs C3 > gpurun_out/ncu_fnv_legacy.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fnv -c 12 --csv --log-file gpurun_out/fnv_launches_r2.csv python tools/fnv_probe.py --configs C3 > /dev/null 2>&1
GS_FNV_LEGACY=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fnv -c 12 --csv --log-file gpurun_out/fnv_launches_legacy_r2.csv python tools/fnv_probe.py --configs C3 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c3_r2.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-c3 --no-c4 --no-overhead > gpurun_out/ncu_launch.log 2>&1
L="--replay-mode app-range --clock-control none --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu $L --csv --log-file gpurun_out/link_encode_r2.csv python tools/link_capture.py --leg encode > gpurun_out/link_encode.log 2>&1
timeout 900 ncu $L --csv --log-file gpurun_out/link_rebuild_r2.csv python tools/link_capture.py --leg rebuild > gpurun_out/link_rebuild.log 2>&1
for f in paper_2605_00831_b200/_lib/obj/gs_special_enc.o paper_2605_00831_b200/_lib/obj/gs_special_dec_kreedsolomon_8_2_e1.o paper_2605_00831_b200/_lib/obj/gs_fnv_gpu.o paper_2605_00831_b200/_lib/obj/gs_rdp_pairs_p11_i0.o; do
  cuobjdump -sass $f > gpurun_out/$(basename $f .o).sass 2>/dev/null
done
ls -la gpurun_out
