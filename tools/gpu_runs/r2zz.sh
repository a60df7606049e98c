# remaining GPU test files on the final code (baselines, residual phase)
python -m pytest tests/test_gpu_baselines.py tests/test_gpu_residuals.py -x -q > gpurun_out/r2zz_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zz_gputest.txt
tail -n 2 gpurun_out/r2zz_gputest.txt
