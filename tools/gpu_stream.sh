# ncu of the streaming and the cluster kernel on config 4 (profiles/r02_stream_config4.md).
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/stream_build.log 2>&1
FIBRA_KERNEL=stream timeout 900 ncu --set full --clock-control none --import-source on -k regex:dr_stream -s 2 -c 1 -o gpurun_out/stream_full python bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/stream_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dr_cluster -s 2 -c 1 -o gpurun_out/cluster_full python bench.py --config 4 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/cluster_ncu.log 2>&1
