# cross-tile K1 prologue (HSX_K1_XTILE=1): parity + A/B with tile heights
HSX_K1_XTILE=1 HSX_CAND_TILE_ROWS=64 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q -k "not peer" > gpurun_out/r2zs_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zs_gputest.txt
tail -n 2 gpurun_out/r2zs_gputest.txt
for m in rn18_224 rn50_224; do
for cfg in "0 128" "1 128" "1 64" "0 64"; do set -- $cfg
HSX_K1_XTILE=$1 HSX_CAND_TILE_ROWS=$2 timeout 300 python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zs_${m}_x$1_r$2.json 2> gpurun_out/r2zs_${m}_x$1_r$2.err
done; done
