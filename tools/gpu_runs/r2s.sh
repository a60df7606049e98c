run1() { tag=$1; model=$2; shift 2; env "$@" python bench.py --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2s_${tag}.json 2> gpurun_out/r2s_${tag}.err; }
for m in rn18_224 rn50_224 rn152_224; do
run1 ${m} $m
run1 ${m}_cq32 $m HSX_LIB_PATH=paper_2512_14628_b200/libhsx_cq32.so
done
HSX_LIB_PATH=paper_2512_14628_b200/libhsx_cq32.so python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or end_to_end" > gpurun_out/r2s_gputest_cq32.txt 2>&1; echo rc=$? >> gpurun_out/r2s_gputest_cq32.txt
tail -n 2 gpurun_out/r2s_gputest_cq32.txt
