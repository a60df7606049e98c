# K3 loop: full-warp mask shuffles, running pointers
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q > gpurun_out/r2zh_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zh_gputest.txt
for m in rn18_224 rn50_224 rn152_224; do python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zh_b1_$m.json 2> gpurun_out/r2zh_b1_$m.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_project' -c 2 -o gpurun_out/r2zh_k3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2zh_ncu.log 2>&1
tail -n 2 gpurun_out/r2zh_gputest.txt
