# split two-rank K1 (HSX_K1_SPLIT=1): torchrun parity + A/B benches
export HSX_BARRIER_TIMEOUT_S=60
HSX_K1_SPLIT=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29791 tests/mp_parity.py 1x2 > gpurun_out/r2zk_mp_1x2.log 2>&1; echo rc=$? >> gpurun_out/r2zk_mp_1x2.log
tail -n 3 gpurun_out/r2zk_mp_1x2.log
if grep -q "rc=0" gpurun_out/r2zk_mp_1x2.log; then
HSX_K1_SPLIT=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29792 tests/mp_parity.py 2x2 > gpurun_out/r2zk_mp_2x2.log 2>&1; echo rc=$? >> gpurun_out/r2zk_mp_2x2.log
tail -n 3 gpurun_out/r2zk_mp_2x2.log
p=29800
for sp in 1 0; do
for m in rn18_224 rn50_224; do
p=$((p+1)); HSX_K1_SPLIT=$sp timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 2 --steps 30 --warmup 5 --model $m --no-cpu-baseline > gpurun_out/r2zk_b2_${m}_s$sp.json 2> gpurun_out/r2zk_b2_${m}_s$sp.err
p=$((p+1)); HSX_K1_SPLIT=$sp timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 4 --steps 30 --warmup 5 --model $m --no-cpu-baseline > gpurun_out/r2zk_b4_${m}_s$sp.json 2> gpurun_out/r2zk_b4_${m}_s$sp.err
done; done
fi
