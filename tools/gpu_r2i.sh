set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1
FIBRA_KERNEL=stream timeout 900 ncu --set full --clock-control none --import-source on -k regex:dr_stream -s 2 -c 1 -o gpurun_out/r2i_stream python bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2i_ncu.log 2>&1; tail -3 gpurun_out/r2i_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dr_cluster -s 2 -c 1 -o gpurun_out/r2i_cluster python bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2i_ncu2.log 2>&1; tail -3 gpurun_out/r2i_ncu2.log
