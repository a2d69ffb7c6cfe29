set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ff_build.log 2>&1
timeout 1200 python tools/config3_classes.py > gpurun_out/r2ff_classes.log 2>&1; tail -30 gpurun_out/r2ff_classes.log
