# K4 fused into K5 (HSX_FUSED_UNION, default on): parity + A/B
export HSX_BARRIER_TIMEOUT_S=60
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_edge.py tests/test_gpu_api.py -x -q > gpurun_out/r2zm_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zm_gputest.txt
tail -n 2 gpurun_out/r2zm_gputest.txt
for g in 2x2 4x1; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29761 tests/mp_parity.py $g > gpurun_out/r2zm_mp_$g.log 2>&1; echo rc=$? >> gpurun_out/r2zm_mp_$g.log
tail -n 2 gpurun_out/r2zm_mp_$g.log
done
p=29810
for rep in 1 2; do for fu in 1 0; do
for cfg in "2x2 rn18_224" "2x2 rn50_224" "4x1 rn50_224"; do set -- $cfg
p=$((p+1)); HSX_FUSED_UNION=$fu timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --grouping $1 --steps 30 --warmup 5 --model $2 --no-cpu-baseline > gpurun_out/r2zm_b4_$1_$2_f${fu}_$rep.json 2> gpurun_out/r2zm_b4_$1_$2_f${fu}_$rep.err
done; done; done
