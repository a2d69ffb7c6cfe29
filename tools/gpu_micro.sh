# Microbenchmarks on one B200: FP64/LDS latencies and throughput (microbench.cu), the resident
# gather step (gather_bench.cu), the cluster barrier (cluster_bench.cu).
set -x
cd $GRAFT_REPO_ROOT
for b in microbench gather_bench cluster_bench; do
  nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -o /tmp/$b tools/$b.cu && /tmp/$b > gpurun_out/micro_$b.log 2>&1; cat gpurun_out/micro_$b.log
done
