set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2u_build.log 2>&1
L=$PWD/paper_2306_09427_b200/lib/variants
for v in single two single two; do
  FIBRA_LIB=$L/$v.so timeout 300 python tools/prof_dr.py 296 4000 2>&1 | grep -o "us/iter/CTA: [0-9.]*" | sed "s/^/$v /" >> gpurun_out/r2u_times.log
done
cat gpurun_out/r2u_times.log
FIBRA_LIB=$L/two.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_cluster.py -m gpu -x -q > gpurun_out/r2u_pytest.log 2>&1; tail -3 gpurun_out/r2u_pytest.log
FIBRA_LIB=$L/two.so timeout 600 python bench.py > gpurun_out/r2u_bench_two.json 2> gpurun_out/r2u_bench_two.err; tail -c 200 gpurun_out/r2u_bench_two.json
FIBRA_LIB=$L/single.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2u_bench_single.json 2> gpurun_out/r2u_bench_single.err; tail -c 200 gpurun_out/r2u_bench_single.json
