nvidia-smi topo -m > gpurun_out/r2zl_topo.txt 2>&1
lscpu | head -30 >> gpurun_out/r2zl_topo.txt
for n in 1 2 4; do for a in 0 1; do
HSX_PROBE_AFFINITY=$a timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29900+n*2+a)) tools/h2d_probe.py >> gpurun_out/r2zl_h2d.txt 2>&1
done; done
cat gpurun_out/r2zl_h2d.txt | grep world
