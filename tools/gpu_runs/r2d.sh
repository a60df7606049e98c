# r2d: K3 whole-word nibble path + chained K2: GPU tests, 1-GPU benches with A/B switches
python -m pytest tests -m gpu -x -q > gpurun_out/r2d_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2d_gputest.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2d_bench_rn18.json 2> gpurun_out/r2d_bench_rn18.err
HSX_K2_CHAIN=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2d_bench_rn18_nochain.json 2> gpurun_out/r2d_bench_rn18_nochain.err
HSX_K1_RESERVE=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2d_bench_rn18_noreserve.json 2> gpurun_out/r2d_bench_rn18_noreserve.err
python bench.py --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2d_bench_rn50.json 2> gpurun_out/r2d_bench_rn50.err
HSX_K2_CHAIN=0 python bench.py --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2d_bench_rn50_nochain.json 2> gpurun_out/r2d_bench_rn50_nochain.err
tail -3 gpurun_out/r2d_gputest.txt
