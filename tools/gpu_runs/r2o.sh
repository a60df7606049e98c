# r2o: tile-height sweep with the chained K2; P=2 peer layer order check
run1() { tag=$1; model=$2; shift 2; env "$@" python bench.py --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2o_${tag}.json 2> gpurun_out/r2o_${tag}.err; }
for m in rn18_224 rn50_224; do
run1 ${m}_base $m
run1 ${m}_c64 $m HSX_CAND_TILE_ROWS=64
run1 ${m}_c64_p32 $m HSX_CAND_TILE_ROWS=64 HSX_PROJ_TILE_ROWS=32
run1 ${m}_p128 $m HSX_PROJ_TILE_ROWS=128
run1 ${m}_p32 $m HSX_PROJ_TILE_ROWS=32
done
python -m pytest tests/test_gpu_parity.py -x -q -k "end_to_end or local_sync" > gpurun_out/r2o_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2o_gputest.txt
run2() { tag=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 2 --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2o_b2_${tag}.json 2> gpurun_out/r2o_b2_${tag}.err; }
run2 auto
run2 big HSX_K1_ORDER=1
tail -n 2 gpurun_out/r2o_gputest.txt
