set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_pytest.log 2>&1; tail -15 gpurun_out/r2b_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; tail -c 1500 gpurun_out/r2b_bench.json; tail -5 gpurun_out/r2b_bench.err
FIBRA_KERNEL=edge timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2b_bench_edge.json 2> gpurun_out/r2b_bench_edge.err; tail -c 600 gpurun_out/r2b_bench_edge.json
