set -x
nvidia-smi topo -m > gpurun_out/r2b_topo.txt 2>&1
python -m pytest tests/test_gpu_api.py -x -q > gpurun_out/r2b_api.txt 2>&1; echo rc=$? >> gpurun_out/r2b_api.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/nvlink_probe.py gpurun_out/r2b_nvlink4.json > gpurun_out/r2b_nvlink4.log 2>&1
NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 tools/nvlink_probe.py gpurun_out/r2b_nvlink2.json > gpurun_out/r2b_nvlink2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 tests/mp_parity.py 2x2 > gpurun_out/r2b_mp_2x2.log 2>&1; echo rc=$? >> gpurun_out/r2b_mp_2x2.log
for t in nccl peer; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 4 --steps 20 --warmup 5 --model rn50_224 --transport $t > gpurun_out/r2b_bench4_rn50_$t.json 2> gpurun_out/r2b_bench4_rn50_$t.err
done
tail -3 gpurun_out/r2b_api.txt gpurun_out/r2b_mp_2x2.log
