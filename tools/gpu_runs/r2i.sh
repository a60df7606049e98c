# r2i: K1 peers2 ring, F1 fused leader average, follower remote K7, K3 fused projection (k>1 layers)
python -m pytest tests -m gpu -x -q > gpurun_out/r2i_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2i_gputest.txt
for g in 2x2 1x4 4x1; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tests/mp_parity.py $g > gpurun_out/r2i_mp_$g.log 2>&1; echo rc=$? >> gpurun_out/r2i_mp_$g.log
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2i_bench_rn18.json 2> gpurun_out/r2i_bench_rn18.err
python bench.py --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2i_bench_rn50.json 2> gpurun_out/r2i_bench_rn50.err
for m in rn50_224 rn18_224; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 4 --steps 20 --warmup 5 --model $m --no-cpu-baseline > gpurun_out/r2i_bench4_$m.json 2> gpurun_out/r2i_bench4_$m.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 2 --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2i_bench2_rn50.json 2> gpurun_out/r2i_bench2_rn50.err
HSX_F1=0 HSX_REMOTE_K7=0 HSX_K1_PEERS2=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 bench.py --gpus 4 --steps 20 --warmup 5 --model rn50_224 --no-cpu-baseline > gpurun_out/r2i_bench4_rn50_old.json 2> gpurun_out/r2i_bench4_rn50_old.err
tail -n 3 gpurun_out/r2i_gputest.txt gpurun_out/r2i_mp_*.log
