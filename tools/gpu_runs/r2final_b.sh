# final-state validation, four GPUs: torchrun parity (all groupings + step variants), benches at 2 / 4 GPUs
python -m pytest tests/test_multigpu.py -x -q > gpurun_out/r2fb_multigpu.txt 2>&1; echo rc=$? >> gpurun_out/r2fb_multigpu.txt
tail -n 2 gpurun_out/r2fb_multigpu.txt
P=29950
run() { out=$1; n=$2; shift 2; P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n "$@" > gpurun_out/r2fb_$out.json 2> gpurun_out/r2fb_$out.err; }
run bench2 2
run bench4 4
run bench2_rn50_224 2 --model rn50_224 --no-cpu-baseline
run bench4_rn50_224 4 --model rn50_224 --no-cpu-baseline
run bench4_1x4 4 --grouping 1x4 --no-cpu-baseline
run bench4_1x4_rn50_224 4 --grouping 1x4 --model rn50_224 --no-cpu-baseline
run bench4_4x1_rn50_224 4 --grouping 4x1 --model rn50_224 --no-cpu-baseline
run bench4_nccl_rn50_224 4 --grouping 2x2 --transport nccl --model rn50_224 --no-cpu-baseline
run bench4_ref 4 --impl reference
ls gpurun_out/r2fb_*.json | wc -l
