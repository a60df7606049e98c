python -m pytest tests/test_gpu_parity.py tests/test_gpu_residuals.py tests/test_gpu_edge.py tests/test_gpu_api.py tests/test_gpu_multirank.py -x -q -k "peer or 1-2 or 2-2 or edge or api or rn18_224 or rn50_224-2x2" > gpurun_out/r2zc_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zc_gputest.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29761 tests/mp_parity.py 1x2 > gpurun_out/r2zc_mp_1x2.log 2>&1; echo rc=$? >> gpurun_out/r2zc_mp_1x2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29762 tests/mp_parity.py 2x2 > gpurun_out/r2zc_mp_2x2.log 2>&1; echo rc=$? >> gpurun_out/r2zc_mp_2x2.log
run() { tag=$1; n=$2; model=$3; shift 3; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29763 bench.py --gpus $n --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2zc_b${n}_${tag}.json 2> gpurun_out/r2zc_b${n}_${tag}.err; }
run rn18 2 rn18_224
run rn18_nostage 2 rn18_224 HSX_PEER_STAGING=0
run rn50 2 rn50_224
run rn50_nostage 2 rn50_224 HSX_PEER_STAGING=0
run rn50_s128 2 rn50_224 HSX_STAGE_CTAS=128
run rn50_s32 2 rn50_224 HSX_STAGE_CTAS=32
run rn18 4 rn18_224
run rn50 4 rn50_224
tail -n 2 gpurun_out/r2zc_gputest.txt gpurun_out/r2zc_mp_*.log
