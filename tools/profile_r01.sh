#!/bin/bash
# Round-1 evidence run (one GPU): bench line, ncu launch list of the bench command, one full
# ncu capture of the config-2 DR kernel launch.  Outputs under gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
tail -1 gpurun_out/p_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/p_bench_ref.json 2>&1
tail -1 gpurun_out/p_bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/p_launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 \
  --no-cpu-baseline > gpurun_out/p_ncu_launch.log 2>&1
tail -2 gpurun_out/p_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dr_persistent \
  -s 1 -c 1 -o gpurun_out/p_full python bench.py --steps 1 --warmup 3 --e2e-steps 1 \
  --no-cpu-baseline > gpurun_out/p_ncu_full.log 2>&1
tail -2 gpurun_out/p_ncu_full.log
