set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y_build.log 2>&1
L=$PWD/paper_2306_09427_b200/lib/variants
for v in dum dum; do FIBRA_LIB=$L/$v.so timeout 300 python tools/prof_dr.py 296 4000 2>&1 | grep -o "us/iter.*"; done
FIBRA_LIB=$L/dum_prof.so FIBRA_PHASE_PROF=1 timeout 300 python tools/prof_dr.py 296 4000 > gpurun_out/r2y_phase.log 2>&1; tail -14 gpurun_out/r2y_phase.log
