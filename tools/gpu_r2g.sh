set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_stream.py -m gpu -q -x > gpurun_out/r2g_pytest.log 2>&1; tail -30 gpurun_out/r2g_pytest.log
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2g_c4.json 2> gpurun_out/r2g_c4.err; tail -c 400 gpurun_out/r2g_c4.json
FIBRA_KERNEL=stream timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2g_c4s.json 2> gpurun_out/r2g_c4s.err; tail -c 400 gpurun_out/r2g_c4s.json; tail -5 gpurun_out/r2g_c4s.err
