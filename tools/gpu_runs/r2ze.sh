python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_edge.py tests/test_gpu_api.py -x -q -k "2-2 or 2-1 or 2-4 or 4-2 or 2x2 or 2x4 or 4x2 or edge" > gpurun_out/r2ze_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2ze_gputest.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29771 tests/mp_parity.py 2x2 > gpurun_out/r2ze_mp_2x2.log 2>&1; echo rc=$? >> gpurun_out/r2ze_mp_2x2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29772 tests/mp_parity.py 4x1 > gpurun_out/r2ze_mp_4x1.log 2>&1; echo rc=$? >> gpurun_out/r2ze_mp_4x1.log
run() { tag=$1; n=$2; model=$3; shift 3; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29773 bench.py --gpus $n --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2ze_b${n}_${tag}.json 2> gpurun_out/r2ze_b${n}_${tag}.err; }
run rn18 4 rn18_224
run rn18_nosplit 4 rn18_224 HSX_SPLIT_K6=0
run rn50 4 rn50_224
run rn50_nosplit 4 rn50_224 HSX_SPLIT_K6=0
HSX_X=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29774 bench.py --gpus 4 --steps 20 --warmup 5 --model rn50_224 --transport nccl --no-cpu-baseline > gpurun_out/r2ze_b4_rn50_nccl.json 2> gpurun_out/r2ze_b4_rn50_nccl.err
tail -n 2 gpurun_out/r2ze_gputest.txt gpurun_out/r2ze_mp_*.log
