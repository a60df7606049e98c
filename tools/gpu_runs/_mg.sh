# usage: bash tools/gpu_runs/_mg.sh N "groupings for mp_parity" "models"
N=$1; GROUPS_=$2; MODELS=$3
make -s || exit 1
mkdir -p gpurun_out
for g in $GROUPS_; do
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 tests/mp_parity.py $g > gpurun_out/mp${N}_$g.log 2>&1; echo "mp_parity $g rc=$? $(grep ok gpurun_out/mp${N}_$g.log | tail -2)"
done
for m in $MODELS; do
  if [ $N = 1 ]; then
    timeout 400 python tools/bench_baselines.py --model $m > gpurun_out/bl_${m}_1.jsonl 2> gpurun_out/bl_${m}_1.err; echo "bl $m 1 rc=$?"
  else
    for g in $4; do
      timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29612 tools/bench_baselines.py --model $m --grouping $g > gpurun_out/bl_${m}_${N}_$g.jsonl 2> gpurun_out/bl_${m}_${N}_$g.err; echo "bl $m $N $g rc=$?"
    done
  fi
done
