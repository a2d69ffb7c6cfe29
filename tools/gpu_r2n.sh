set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2n_pytest.log 2>&1; tail -3 gpurun_out/r2n_pytest.log
timeout 600 python bench.py > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err; tail -c 300 gpurun_out/r2n_bench.json
FIBRA_PHASE_PROF=1 python -m paper_2306_09427_b200.build > gpurun_out/r2n_prof_build.log 2>&1
FIBRA_PHASE_PROF=1 timeout 300 python tools/prof_dr.py 296 4000 > gpurun_out/r2n_phase.log 2>&1; tail -16 gpurun_out/r2n_phase.log
