for rep in 1 2; do
for m in rn18_224 rn50_224 rn152_224; do
python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zo_${m}_base_$rep.json 2>/dev/null
HSX_K1_RESERVE=0 python bench.py --model $m --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2zo_${m}_r0_$rep.json 2>/dev/null
done; done
HSX_K1_RESERVE=0 HSX_LIB_PATH=paper_2512_14628_b200/libhsx_trace.so python tools/k1_trace.py rn18_224 > gpurun_out/r2zo_k1trace_r0.txt 2>&1
head -6 gpurun_out/r2zo_k1trace_r0.txt
