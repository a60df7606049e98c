# persistent K3 (HSX_K3_PERSIST=1) x tile rows
HSX_K3_PERSIST=1 HSX_PROJ_TILE_ROWS=32 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q > gpurun_out/r2zi_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zi_gputest.txt
for m in rn18_224 rn50_224; do
python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zi_b1_${m}_base.json 2> /dev/null
for tr in 64 32 16; do
HSX_K3_PERSIST=1 HSX_PROJ_TILE_ROWS=$tr python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zi_b1_${m}_p$tr.json 2> gpurun_out/r2zi_b1_${m}_p$tr.err
done
HSX_PROJ_TILE_ROWS=32 python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zi_b1_${m}_np32.json 2> /dev/null
done
tail -n 2 gpurun_out/r2zi_gputest.txt
