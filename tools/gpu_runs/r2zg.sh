# one-sided leader->follower barriers (m_bcast, zhat_bcast): parity + A/B at 4 GPUs
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_edge.py tests/test_gpu_api.py -x -q > gpurun_out/r2zg_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zg_gputest.txt
for g in 2x2 1x4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29761 tests/mp_parity.py $g > gpurun_out/r2zg_mp_$g.log 2>&1; echo rc=$? >> gpurun_out/r2zg_mp_$g.log
done
p=29770
for rep in 1 2; do
for os in 1 0; do
for m in rn18_224 rn50_224; do
p=$((p+1))
HSX_ONESIDED=$os timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --grouping 2x2 --steps 30 --warmup 5 --model $m --no-cpu-baseline > gpurun_out/r2zg_${m}_os${os}_$rep.json 2> gpurun_out/r2zg_${m}_os${os}_$rep.err
done; done; done
tail -n 2 gpurun_out/r2zg_gputest.txt gpurun_out/r2zg_mp_*.log
