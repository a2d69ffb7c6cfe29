# ncu evidence for the resident DR kernel on one B200 (run with gpurun, outputs in
# gpurun_out/): the default bench line, the reference arm, the launch list of one config-2
# step, and one `--set full` capture of the DR launch (profiles/r02_dr_kernel.md, capture c).
# Variant: PROF_WORKLOAD=steady captures tools/prof_dr.py 296 4000 instead (capture b).
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/prof_build.log 2>&1
timeout 600 python bench.py > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err; tail -c 300 gpurun_out/prof_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/prof_ref.json 2> gpurun_out/prof_ref.err; tail -c 300 gpurun_out/prof_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof_ncu_launch.log 2>&1
if [ "$PROF_WORKLOAD" = steady ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dr_persistent -s 1 -c 1 -o gpurun_out/prof_full python tools/prof_dr.py 296 4000 > gpurun_out/prof_ncu_full.log 2>&1
else
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dr_persistent -s 1 -c 1 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof_ncu_full.log 2>&1
fi
tail -2 gpurun_out/prof_ncu_full.log
# reading it here: python tools/ncu_summary.py gpurun_out/prof_full.ncu-rep profiles/r01_v7_dr_kernel_metrics.csv out.csv
#                  ncu -i gpurun_out/prof_full.ncu-rep --page source --csv --print-source cuda,sass > src.csv
#                  python tools/ncu_lines.py src.csv <RVE-iterations of the launch>
