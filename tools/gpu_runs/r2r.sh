# r2r: K3 -> K67 chain with the device-published keep-set summary
HSX_K67_CHAIN=1 python -m pytest tests -m gpu -x -q -k "not multirank" > gpurun_out/r2r_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2r_gputest.txt
run1() { tag=$1; model=$2; shift 2; env "$@" python bench.py --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2r_${tag}.json 2> gpurun_out/r2r_${tag}.err; }
for m in rn18_224 rn50_224 rn152_224; do
run1 ${m} $m
run1 ${m}_k67 $m HSX_K67_CHAIN=1
done
run2() { tag=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 2 --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2r_b2_${tag}.json 2> gpurun_out/r2r_b2_${tag}.err; }
run2 rn50
run2 rn50_k67 HSX_K67_CHAIN=1
HSX_K67_CHAIN=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712 tests/mp_parity.py 1x2 > gpurun_out/r2r_mp_1x2.log 2>&1; echo rc=$? >> gpurun_out/r2r_mp_1x2.log
bash tools/gpu_runs/sparsity_sweep2.sh rn50_224 nccl > gpurun_out/sweep2_nccl.txt 2>&1
bash tools/gpu_runs/sparsity_sweep2.sh rn50_224 peer > gpurun_out/sweep2_peer.txt 2>&1
tail -n 2 gpurun_out/r2r_gputest.txt gpurun_out/r2r_mp_1x2.log
