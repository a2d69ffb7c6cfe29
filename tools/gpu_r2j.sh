set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1
timeout 900 python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err; tail -c 400 gpurun_out/r2j_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2j_ncu_launch.log 2>&1; tail -2 gpurun_out/r2j_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dr_persistent -s 1 -c 1 -o gpurun_out/r2j_full python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2j_ncu_full.log 2>&1; tail -2 gpurun_out/r2j_ncu_full.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_parity.py -m gpu -q -k "single_rve or batch_tangent" > gpurun_out/r2j_racecheck.log 2>&1; tail -5 gpurun_out/r2j_racecheck.log
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -m gpu -q -k "single_rve or batch_tangent" > gpurun_out/r2j_synccheck.log 2>&1; tail -5 gpurun_out/r2j_synccheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_cluster.py -m gpu -q -k "lattice_converged or exponential" > gpurun_out/r2j_racecheck_cluster.log 2>&1; tail -5 gpurun_out/r2j_racecheck_cluster.log
