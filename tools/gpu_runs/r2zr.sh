# K1 on the distributed intra sum (P > 2): parity + A/B at 1x4
export HSX_BARRIER_TIMEOUT_S=60
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_edge.py tests/test_gpu_api.py -x -q > gpurun_out/r2zr_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zr_gputest.txt
tail -n 2 gpurun_out/r2zr_gputest.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29881 tests/mp_parity.py 1x4 > gpurun_out/r2zr_mp_1x4.log 2>&1; echo rc=$? >> gpurun_out/r2zr_mp_1x4.log
tail -n 2 gpurun_out/r2zr_mp_1x4.log
p=29890
for rep in 1 2; do for ds in 1 0; do for m in rn18_224 rn50_224; do
p=$((p+1)); HSX_DIST_SUM=$ds timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --grouping 1x4 --steps 30 --warmup 5 --model $m --no-cpu-baseline > gpurun_out/r2zr_1x4_${m}_d${ds}_$rep.json 2> gpurun_out/r2zr_1x4_${m}_d${ds}_$rep.err
done; done; done
