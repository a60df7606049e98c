python tools/k1_peer_local.py > gpurun_out/r2y_k1_local.txt 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_residuals.py tests/test_gpu_edge.py tests/test_gpu_multirank.py -x -q -k "peer or 1-2 or 2-2 or 4-2 or edge or rn18_224" > gpurun_out/r2y_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2y_gputest.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29741 tests/mp_parity.py 1x2 > gpurun_out/r2y_mp_1x2.log 2>&1; echo rc=$? >> gpurun_out/r2y_mp_1x2.log
run2() { tag=$1; model=$2; shift 2; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29742 bench.py --gpus 2 --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2y_b2_${tag}.json 2> gpurun_out/r2y_b2_${tag}.err; }
run2 rn50 rn50_224
run2 rn50_old rn50_224 HSX_K1_PEERS2=0
run2 rn18 rn18_224
run2 rn152 rn152_224
cat gpurun_out/r2y_k1_local.txt; tail -n 2 gpurun_out/r2y_gputest.txt gpurun_out/r2y_mp_1x2.log
