set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_fastmath.py tests/test_gpu_cluster.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2h_pytest.log 2>&1; tail -30 gpurun_out/r2h_pytest.log
FIBRA_KERNEL=stream timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2h_c4s.json 2> gpurun_out/r2h_c4s.err; tail -c 300 gpurun_out/r2h_c4s.json; tail -5 gpurun_out/r2h_c4s.err
FIBRA_KERNEL=stream FIBRA_STREAM_STAGE=0 timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2h_c4s0.json 2> gpurun_out/r2h_c4s0.err; tail -c 300 gpurun_out/r2h_c4s0.json
FIBRA_KERNEL=stream FIBRA_STREAM_C=8 timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2h_c4s8.json 2> gpurun_out/r2h_c4s8.err; tail -c 300 gpurun_out/r2h_c4s8.json
