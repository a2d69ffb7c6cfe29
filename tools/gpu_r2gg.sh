set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2gg_build.log 2>&1
timeout 1200 python tools/config3_classes.py > gpurun_out/r2gg_classes.log 2>&1; tail -16 gpurun_out/r2gg_classes.log
for c in 3 5; do
timeout 1200 python bench.py --config $c --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2gg_c$c.json 2> gpurun_out/r2gg_c$c.err; tail -c 300 gpurun_out/r2gg_c$c.json
done
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_cluster.py -m gpu -x -q > gpurun_out/r2gg_pytest.log 2>&1; tail -2 gpurun_out/r2gg_pytest.log
