set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x_build.log 2>&1
timeout 300 python tools/prof_dr.py 296 4000 > gpurun_out/r2x_phase.log 2>&1
timeout 300 python tools/prof_dr.py 296 4000 >> gpurun_out/r2x_phase.log 2>&1; grep -o "us/iter.*" gpurun_out/r2x_phase.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2x_pytest.log 2>&1; tail -3 gpurun_out/r2x_pytest.log
timeout 600 python bench.py > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err; tail -c 300 gpurun_out/r2x_bench.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dr_persistent -s 1 -c 1 -o gpurun_out/r2x_full python tools/prof_dr.py 296 4000 > gpurun_out/r2x_ncu.log 2>&1; tail -2 gpurun_out/r2x_ncu.log
