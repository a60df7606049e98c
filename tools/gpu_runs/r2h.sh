python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_residuals.py tests/test_gpu_multirank.py -k "not rn50_224-2x4 and not rn50_224-4x2" -x -q > gpurun_out/r2h_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2h_gputest.txt
python __graft_entry__.py smoke > gpurun_out/r2h_smoke.txt 2>&1; echo rc=$? >> gpurun_out/r2h_smoke.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2h_bench_rn18.json 2> gpurun_out/r2h_bench_rn18.err
HSX_FUSED_PROJ=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2h_bench_rn18_nofuse.json 2> gpurun_out/r2h_bench_rn18_nofuse.err
python bench.py --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2h_bench_rn50.json 2> gpurun_out/r2h_bench_rn50.err
python bench.py --steps 10 --warmup 3 --model rn152_224 --no-cpu-baseline > gpurun_out/r2h_bench_rn152.json 2> gpurun_out/r2h_bench_rn152.err
tail -n 3 gpurun_out/r2h_gputest.txt gpurun_out/r2h_smoke.txt
