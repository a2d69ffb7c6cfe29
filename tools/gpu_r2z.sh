set -x
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -o /tmp/gather_bench tools/gather_bench.cu && /tmp/gather_bench > gpurun_out/r2z_gather.log 2>&1; cat gpurun_out/r2z_gather.log
