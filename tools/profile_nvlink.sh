# NVLink evidence for the striped K1 at N GPUs (needs >= 2 GPUs on one node;
# not runnable on the 1-GPU gpurun boxes). ncu attaches to every rank
# (--target-processes all) but captures only rank 0's striped K1 launches
# (-k EncSpec, after the warm-up) with the NVLink rx/tx byte counters next to
# the DRAM counters: rank 0 should receive (N-1)/N of its range of the 8 data
# shards over NVLink (nvlrx__bytes) and send the same share to its peers.
N=${N:-2}
mkdir -p gpurun_out
ncu --target-processes all --clock-control none -k regex:EncSpec -s 6 -c 2 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
    --csv --log-file gpurun_out/nvlink_k1_n${N}.csv \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
    bench.py --gpus $N --steps 4 --warmup 3 --no-cpu --no-c3 --no-c4 --no-overhead
