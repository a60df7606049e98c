python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_multirank.py -k "not rn50_224-2x4 and not rn50_224-4x2" -x -q > gpurun_out/r2e_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2e_gputest.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2e_bench_rn18.json 2> gpurun_out/r2e_bench_rn18.err
HSX_K3_BITS=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2e_bench_rn18_k3read.json 2> gpurun_out/r2e_bench_rn18_k3read.err
python bench.py --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2e_bench_rn50.json 2> gpurun_out/r2e_bench_rn50.err
tail -3 gpurun_out/r2e_gputest.txt
