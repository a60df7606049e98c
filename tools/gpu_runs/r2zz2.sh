python -m pytest tests/test_multigpu.py -q -k "1x2 or 2x1" > gpurun_out/r2zz2_multigpu.txt 2>&1; echo rc=$? >> gpurun_out/r2zz2_multigpu.txt
tail -n 2 gpurun_out/r2zz2_multigpu.txt
