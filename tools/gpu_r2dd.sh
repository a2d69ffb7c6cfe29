set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2dd_build.log 2>&1
L=$PWD/paper_2306_09427_b200/lib/variants
for v in head pk head pk head pk; do FIBRA_LIB=$L/$v.so timeout 300 python tools/prof_dr.py 296 4000 2>&1 | grep -o "us/iter.*" | sed "s/^/$v /"; done
FIBRA_LIB=$L/pk.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/r2dd_pytest.log 2>&1; tail -2 gpurun_out/r2dd_pytest.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cluster_bench tools/cluster_bench.cu && /tmp/cluster_bench > gpurun_out/r2dd_cluster.log 2>&1; cat gpurun_out/r2dd_cluster.log
