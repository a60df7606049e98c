#!/bin/bash
# One GPU pass: gpu tests, smoke, bench (N=1), ncu launch list, ncu full capture of the
# dominant kernels. Usage (under gpurun): bash tools/gpu_runs/gpu_round.sh TAG [skip_tests]
TAG=${1:-r1}
mkdir -p gpurun_out
make -s || exit 1
if [ "$2" != "skip_tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
  echo "pytest gpu rc=$? $(tail -1 gpurun_out/${TAG}_pytest_gpu.log)"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
  echo "smoke rc=$? $(tail -1 gpurun_out/${TAG}_smoke.log)"
fi
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$? $(head -c 600 gpurun_out/${TAG}_bench.json)"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'k_candidate|k_local_sync|k_compact|k_decompact|k_project|k_select|k_keep_sets' -c 6 \
  -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
timeout 600 python bench.py --model rn50_224 --no-cpu-baseline > gpurun_out/${TAG}_bench_rn50.json 2> gpurun_out/${TAG}_bench_rn50.err
echo "bench rn50 rc=$? $(head -c 300 gpurun_out/${TAG}_bench_rn50.json)"
