set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2v_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2v_pytest.log 2>&1; tail -3 gpurun_out/r2v_pytest.log
timeout 300 python tools/prof_dr.py 296 4000 > gpurun_out/r2v_phase.log 2>&1
timeout 600 python bench.py > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err; tail -c 300 gpurun_out/r2v_bench.json
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2v_c3.json 2> gpurun_out/r2v_c3.err; tail -c 300 gpurun_out/r2v_c3.json; tail -3 gpurun_out/r2v_c3.err
FIBRA_PHASE_PROF=1 python -m paper_2306_09427_b200.build > gpurun_out/r2v_prof_build.log 2>&1
FIBRA_PHASE_PROF=1 timeout 300 python tools/prof_dr.py 296 4000 >> gpurun_out/r2v_phase.log 2>&1; tail -16 gpurun_out/r2v_phase.log
