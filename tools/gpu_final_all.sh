# Round-end evidence in one call: validation (tools/gpu_final.sh), configs 3-5
# (tools/gpu_configs.sh, without its pytest) and the ncu capture (tools/gpu_profile.sh).
set -x
cd $GRAFT_REPO_ROOT
bash tools/gpu_final.sh
for c in 4 5 3; do
  timeout 1200 python bench.py --config $c --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/cfg_c$c.json 2> gpurun_out/cfg_c$c.err; tail -c 300 gpurun_out/cfg_c$c.json
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof_ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dr_persistent -s 1 -c 1 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof_ncu_full.log 2>&1; tail -2 gpurun_out/prof_ncu_full.log
