# default-configuration parity after the K1 restructuring (cross-tile hooks, opt-in)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_edge.py tests/test_gpu_multirank.py -x -q > gpurun_out/r2zu_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zu_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2zu_smoke.txt 2>&1; echo rc=$? >> gpurun_out/r2zu_smoke.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2zu_bench1.json 2> gpurun_out/r2zu_bench1.err
tail -n 2 gpurun_out/r2zu_gputest.txt gpurun_out/r2zu_smoke.txt
