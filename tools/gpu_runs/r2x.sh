python tools/k1_peer_local.py > gpurun_out/r2x_k1_local.txt 2>&1
HSX_K1_NARROW=0 python tools/k1_peer_local.py >> gpurun_out/r2x_k1_local.txt 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q -k "full_size or end_to_end or rn18_224-2x2" > gpurun_out/r2x_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2x_gputest.txt
run1() { tag=$1; model=$2; shift 2; env "$@" python bench.py --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2x_${tag}.json 2> gpurun_out/r2x_${tag}.err; }
run1 rn18 rn18_224
run1 rn50 rn50_224
run1 rn152 rn152_224
run2() { tag=$1; model=$2; shift 2; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731 bench.py --gpus 2 --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2x_b2_${tag}.json 2> gpurun_out/r2x_b2_${tag}.err; }
run2 rn50 rn50_224
run2 rn50_wide rn50_224 HSX_K1_NARROW=0
run2 rn18 rn18_224
cat gpurun_out/r2x_k1_local.txt; tail -n 2 gpurun_out/r2x_gputest.txt
