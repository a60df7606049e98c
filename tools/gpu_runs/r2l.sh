run2() { tag=$1; shift; env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2l_b2_${tag}.json 2> gpurun_out/r2l_b2_${tag}.err; }
run2 base HSX_BENCH_TRACE=1
run2 noclk HSX_BENCH_TRACE=1 HSX_BENCH_NO_CLOCKS=1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2l_b1_rn18.json 2> gpurun_out/r2l_b1_rn18.err
grep "host enqueue" gpurun_out/r2l_b2_*.err | cut -c1-200 | head -20
