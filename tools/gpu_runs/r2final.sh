# final-state validation: full GPU suite, smoke, torchrun parity at 4 GPUs, benches 1/2/4 GPUs, ncu
python -m pytest tests -m gpu -x -q > gpurun_out/r2f_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2f_gputest.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2f_smoke.txt 2>&1; echo rc=$? >> gpurun_out/r2f_smoke.txt
for g in 2x2 1x4 4x1; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29751 tests/mp_parity.py $g > gpurun_out/r2f_mp_$g.log 2>&1; echo rc=$? >> gpurun_out/r2f_mp_$g.log
done
python bench.py > gpurun_out/r2f_bench1.json 2> gpurun_out/r2f_bench1.err
python bench.py --impl reference > gpurun_out/r2f_bench1_ref.json 2> gpurun_out/r2f_bench1_ref.err
for m in rn50_224 rn152_224; do python bench.py --model $m --no-cpu-baseline > gpurun_out/r2f_bench1_$m.json 2> gpurun_out/r2f_bench1_$m.err; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29752 bench.py --gpus 2 > gpurun_out/r2f_bench2.json 2> gpurun_out/r2f_bench2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29753 bench.py --gpus 4 > gpurun_out/r2f_bench4.json 2> gpurun_out/r2f_bench4.err
for m in rn50_224; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29754 bench.py --gpus 4 --model $m --no-cpu-baseline > gpurun_out/r2f_bench4_$m.json 2> gpurun_out/r2f_bench4_$m.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29755 bench.py --gpus 4 --grouping 4x1 --model $m --no-cpu-baseline > gpurun_out/r2f_bench4_4x1_$m.json 2> gpurun_out/r2f_bench4_4x1_$m.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29756 bench.py --gpus 4 --grouping 2x2 --transport nccl --model $m --no-cpu-baseline > gpurun_out/r2f_bench4_nccl_$m.json 2> gpurun_out/r2f_bench4_nccl_$m.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29757 bench.py --gpus 4 --impl reference > gpurun_out/r2f_bench4_ref.json 2> gpurun_out/r2f_bench4_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_candidate|k_local_sync|k_project|k_select' -c 5 -o gpurun_out/r2f_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_ncu_full.log 2>&1
tail -n 2 gpurun_out/r2f_gputest.txt gpurun_out/r2f_smoke.txt gpurun_out/r2f_mp_*.log
