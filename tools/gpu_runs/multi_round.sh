#!/bin/bash
# 4-GPU box: RN18 at 2 GPUs (1x2) and 4 GPUs (2x2, 4x1), RN50 at 4 GPUs (2x2), both transports
bash tools/gpu_runs/bench_multi.sh 2 default
bash tools/gpu_runs/bench_multi.sh 4 default
bash tools/gpu_runs/bench_multi.sh 4 4x1
bash tools/gpu_runs/bench_multi.sh 4 2x2 --model rn50_224
