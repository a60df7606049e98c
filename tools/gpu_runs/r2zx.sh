python -m pytest tests/test_gpu_multirank.py tests/test_gpu_api.py -x -q > gpurun_out/r2zx_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zx_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2zx_smoke.txt 2>&1; echo rc=$? >> gpurun_out/r2zx_smoke.txt
tail -n 2 gpurun_out/r2zx_gputest.txt gpurun_out/r2zx_smoke.txt
