run2() { tag=$1; model=$2; shift 2; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 2 --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2q_b2_${tag}.json 2> gpurun_out/r2q_b2_${tag}.err; }
run2 rn50 rn50_224
run2 rn50_p2d6 rn50_224 HSX_K1_PEERS2=1
run2 rn18 rn18_224
run2 rn18_p2d6 rn18_224 HSX_K1_PEERS2=1
python -m pytest tests/test_gpu_parity.py -x -q -k "peer or 1-2" > gpurun_out/r2q_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2q_gputest.txt
HSX_K1_PEERS2=1 python -m pytest tests/test_gpu_parity.py -x -q -k "peer or 1-2" >> gpurun_out/r2q_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2q_gputest.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/r2q_b1_rn18.json 2> gpurun_out/r2q_b1_rn18.err
tail -n 4 gpurun_out/r2q_gputest.txt
