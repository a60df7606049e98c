# K3 TMA row copies (HSX_K3_TMA=1) vs per-thread cp.async
HSX_K3_TMA=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_multirank.py -x -q > gpurun_out/r2zj_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zj_gputest.txt
for rep in 1 2; do
for m in rn18_224 rn50_224 rn152_224; do
python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zj_b1_${m}_base_$rep.json 2> /dev/null
HSX_K3_TMA=1 python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zj_b1_${m}_tma_$rep.json 2> gpurun_out/r2zj_b1_${m}_tma.err
done; done
HSX_K3_TMA=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_project' -c 2 -o gpurun_out/r2zj_k3tma python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2zj_ncu.log 2>&1
tail -n 2 gpurun_out/r2zj_gputest.txt
