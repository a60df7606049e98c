# r2n: chained K2 + K3 (defaults), big-layers-first K1 order
python -m pytest tests -m gpu -x -q > gpurun_out/r2n_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2n_gputest.txt
for g in 2x2 1x4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 tests/mp_parity.py $g > gpurun_out/r2n_mp_$g.log 2>&1; echo rc=$? >> gpurun_out/r2n_mp_$g.log
done
run1() { tag=$1; model=$2; shift 2; env "$@" python bench.py --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2n_${tag}.json 2> gpurun_out/r2n_${tag}.err; }
run1 rn18 rn18_224
run1 rn18_nok3 rn18_224 HSX_K3_CHAIN=0
run1 rn50 rn50_224
run1 rn50_nok3 rn50_224 HSX_K3_CHAIN=0
run1 rn152 rn152_224
run4() { tag=$1; model=$2; shift 2; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 4 --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2n_b4_${tag}.json 2> gpurun_out/r2n_b4_${tag}.err; }
run4 rn50 rn50_224
run4 rn50_noorder rn50_224 HSX_K1_ORDER=0
run4 rn50_nochain rn50_224 HSX_K2_CHAIN=0
run4 rn18 rn18_224
tail -n 2 gpurun_out/r2n_gputest.txt gpurun_out/r2n_mp_*.log
