# r2p: one-node K3 -> K67 chain
python -m pytest tests -m gpu -x -q > gpurun_out/r2p_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2p_gputest.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29681 tests/mp_parity.py 1x2 > gpurun_out/r2p_mp_1x2.log 2>&1; echo rc=$? >> gpurun_out/r2p_mp_1x2.log
run1() { tag=$1; model=$2; shift 2; env "$@" python bench.py --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2p_${tag}.json 2> gpurun_out/r2p_${tag}.err; }
for m in rn18_224 rn50_224 rn152_224; do
run1 ${m} $m
run1 ${m}_no67 $m HSX_K67_CHAIN=0
done
run2() { tag=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29682 bench.py --gpus 2 --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2p_b2_${tag}.json 2> gpurun_out/r2p_b2_${tag}.err; }
run2 rn50
run2 rn50_no67 HSX_K67_CHAIN=0
tail -n 2 gpurun_out/r2p_gputest.txt gpurun_out/r2p_mp_1x2.log
