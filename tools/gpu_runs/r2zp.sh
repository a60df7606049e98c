for m in rn18_224 rn50_224; do
python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zp_${m}_base.json 2>/dev/null
HSX_CAND_TILE_ROWS=64 python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zp_${m}_r64.json 2>/dev/null
HSX_CAND_TILE_ROWS=96 python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zp_${m}_r96.json 2>/dev/null
HSX_LIB_PATH=paper_2512_14628_b200/libhsx_cq32.so python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zp_${m}_cq32.json 2>/dev/null
HSX_LIB_PATH=paper_2512_14628_b200/libhsx_cq32.so HSX_CAND_TILE_ROWS=64 python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zp_${m}_cq32r64.json 2>/dev/null
done
