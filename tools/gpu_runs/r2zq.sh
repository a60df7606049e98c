for m in rn18_224 rn50_224; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29871 bench.py --gpus 4 --grouping 1x4 --steps 30 --warmup 5 --model $m --no-cpu-baseline > gpurun_out/r2zq_1x4_$m.json 2> gpurun_out/r2zq_1x4_$m.err
done
