# r2j: A/B of the peer-transport options at 4 GPUs (2x2), after removing the fused projection
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > gpurun_out/r2j_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2j_gputest.txt
run4() { tag=$1; model=$2; shift 2; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 4 --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2j_b4_${tag}.json 2> gpurun_out/r2j_b4_${tag}.err; }
run4 rn50_base rn50_224 HSX_F1=0
run4 rn50_rk7 rn50_224 HSX_REMOTE_K7=1
run4 rn50_f1rk7 rn50_224 HSX_F1=1 HSX_REMOTE_K7=1
run4 rn50_p2 rn50_224 HSX_K1_PEERS2=1
run4 rn18_base rn18_224 HSX_F1=0
run4 rn18_rk7 rn18_224 HSX_REMOTE_K7=1
env timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 4 --steps 20 --warmup 5 --model rn50_224 --transport nccl --no-cpu-baseline > gpurun_out/r2j_b4_rn50_nccl.json 2> gpurun_out/r2j_b4_rn50_nccl.err
tail -n 3 gpurun_out/r2j_gputest.txt
