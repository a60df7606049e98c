python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_multirank.py -x -q -k "full_size or end_to_end or kept_zeros or edge or rn18_224-2x2" > gpurun_out/r2zd_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2zd_gputest.txt
run1() { tag=$1; model=$2; shift 2; env "$@" python bench.py --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2zd_${tag}.json 2> gpurun_out/r2zd_${tag}.err; }
run1 rn18 rn18_224
run1 rn50 rn50_224
run1 rn152 rn152_224
tail -n 2 gpurun_out/r2zd_gputest.txt
