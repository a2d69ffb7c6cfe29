set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2aa_build.log 2>&1
timeout 600 python bench.py > gpurun_out/r2aa_bench.json 2> gpurun_out/r2aa_bench.err; tail -c 300 gpurun_out/r2aa_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/r2aa_ref.json 2> gpurun_out/r2aa_ref.err; tail -c 300 gpurun_out/r2aa_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2aa_launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2aa_ncu_launch.log 2>&1; tail -2 gpurun_out/r2aa_ncu_launch.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dr_persistent -s 1 -c 1 -o gpurun_out/r2aa_full python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2aa_ncu_full.log 2>&1; tail -2 gpurun_out/r2aa_ncu_full.log
