python bench.py > gpurun_out/r2zy_bench1.json 2> gpurun_out/r2zy_bench1.err
for m in rn50_224 rn152_224; do python bench.py --model $m --no-cpu-baseline > gpurun_out/r2zy_bench1_$m.json 2> gpurun_out/r2zy_bench1_$m.err; done
