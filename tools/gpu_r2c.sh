set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1
for v in "" "FIBRA_NODE_SHAPE=2" "FIBRA_KERNEL=edge"; do
  env $v timeout 300 python tools/prof_dr.py 444 4000 2>&1 | tail -1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dr_node -s 1 -c 1 -o gpurun_out/r2c_node python tools/prof_dr.py 444 2000 > gpurun_out/r2c_ncu.log 2>&1
tail -3 gpurun_out/r2c_ncu.log
