set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t_build.log 2>&1
timeout 300 python tools/prof_dr.py 296 4000 > gpurun_out/r2t_plain.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dr_persistent -s 1 -c 1 -o gpurun_out/r2t_full python tools/prof_dr.py 296 4000 > gpurun_out/r2t_ncu.log 2>&1; tail -3 gpurun_out/r2t_ncu.log
