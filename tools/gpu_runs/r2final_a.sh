# final-state validation, one GPU: full GPU suite, smoke, 1-GPU benches (both arms), ncu
python -m pytest tests -m gpu -x -q > gpurun_out/r2fa_gputest.txt 2>&1; echo rc=$? >> gpurun_out/r2fa_gputest.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2fa_smoke.txt 2>&1; echo rc=$? >> gpurun_out/r2fa_smoke.txt
python bench.py > gpurun_out/r2fa_bench1.json 2> gpurun_out/r2fa_bench1.err
python bench.py --impl reference > gpurun_out/r2fa_bench1_ref.json 2> gpurun_out/r2fa_bench1_ref.err
for m in rn50_224 rn152_224; do python bench.py --model $m --no-cpu-baseline > gpurun_out/r2fa_bench1_$m.json 2> gpurun_out/r2fa_bench1_$m.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2fa_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2fa_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_candidate|k_local_sync|k_project|k_select' -c 5 -o gpurun_out/r2fa_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2fa_ncu_full.log 2>&1
tail -n 2 gpurun_out/r2fa_gputest.txt gpurun_out/r2fa_smoke.txt
