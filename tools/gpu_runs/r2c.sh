# r2c: GPU tests with the K3 nonzero-nibble path, 1-GPU benches, 2-GPU bench with the collectives block
python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r2c_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2c_gputest.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench_rn18.json 2> gpurun_out/r2c_bench_rn18.err
python bench.py --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2c_bench_rn50.json 2> gpurun_out/r2c_bench_rn50.err
HSX_K3_BITS=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench_rn18_k3read.json 2> gpurun_out/r2c_bench_rn18_k3read.err
for t in peer nccl; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 2 --steps 20 --warmup 5 --transport $t --no-cpu-baseline > gpurun_out/r2c_bench2_$t.json 2> gpurun_out/r2c_bench2_$t.err
done
tail -3 gpurun_out/r2c_gputest.txt
