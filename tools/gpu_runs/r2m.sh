run1() { tag=$1; model=$2; shift 2; env "$@" python bench.py --steps 20 --warmup 5 --model $model --no-cpu-baseline > gpurun_out/r2m_${tag}.json 2> gpurun_out/r2m_${tag}.err; }
for m in rn18_224 rn50_224; do
run1 ${m}_base $m HSX_K2_CHAIN=0
run1 ${m}_order $m HSX_K1_ORDER=1
run1 ${m}_chain_order $m HSX_K2_CHAIN=1 HSX_K1_ORDER=1
run1 ${m}_chain_order_r0 $m HSX_K2_CHAIN=1 HSX_K1_ORDER=1 HSX_K1_RESERVE=0
run1 ${m}_chain $m HSX_K2_CHAIN=1
done
