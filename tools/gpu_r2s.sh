set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s_build.log 2>&1
timeout 300 python tools/prof_dr.py 296 4000 > gpurun_out/r2s_phase.log 2>&1
FIBRA_PHASE_PROF=1 python -m paper_2306_09427_b200.build > gpurun_out/r2s_prof_build.log 2>&1
FIBRA_PHASE_PROF=1 timeout 300 python tools/prof_dr.py 296 4000 >> gpurun_out/r2s_phase.log 2>&1; tail -16 gpurun_out/r2s_phase.log
FIBRA_PHASE_PROF=1 timeout 300 python tools/prof_dr.py 148 4000 >> gpurun_out/r2s_phase.log 2>&1; tail -16 gpurun_out/r2s_phase.log
