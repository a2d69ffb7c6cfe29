# Round-end validation on a 4-GPU box: tools/gpu_final.sh (the whole GPU suite incl. the
# multi-GPU tests, smoke, default bench, reference arm) and config-3 strong scaling.
set -x
cd $GRAFT_REPO_ROOT
bash tools/gpu_final.sh
for n in 4 2; do
  timeout 1200 python bench.py --config 3 --gpus $n --single-process --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/scale_c3sp$n.json 2> gpurun_out/scale_c3sp$n.err; tail -c 300 gpurun_out/scale_c3sp$n.json
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 bench.py --config 3 --gpus 4 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/scale_c3tr4.json 2> gpurun_out/scale_c3tr4.err; tail -c 300 gpurun_out/scale_c3tr4.json
