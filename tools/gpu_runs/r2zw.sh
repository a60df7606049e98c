# K3: first ring stages issued before the keep flags are gathered; A/B against the previous build
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q > gpurun_out/r2zw_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zw_gputest.txt
tail -n 2 gpurun_out/r2zw_gputest.txt
for rep in 1 2; do for m in rn18_224 rn50_224 rn152_224; do
python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zw_${m}_new_$rep.json 2>/dev/null
HSX_LIB_PATH=paper_2512_14628_b200/libhsx_prev.so python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zw_${m}_prev_$rep.json 2>/dev/null
done; done
