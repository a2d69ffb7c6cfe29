# Multi-GPU runs on one box (gpurun --gpus 4): config 2 weak and config 3 strong, one process
# (fibra_cuda_open_devices) and torchrun (profiles/r02_scaling.md).
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=index,name --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/scale_build.log 2>&1
for n in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n > gpurun_out/scale_tr$n.json 2> gpurun_out/scale_tr$n.err; tail -c 300 gpurun_out/scale_tr$n.json
  timeout 900 python bench.py --gpus $n --single-process --no-cpu-baseline > gpurun_out/scale_sp$n.json 2> gpurun_out/scale_sp$n.err; tail -c 300 gpurun_out/scale_sp$n.json
  timeout 1200 python bench.py --config 3 --gpus $n --single-process --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/scale_c3sp$n.json 2> gpurun_out/scale_c3sp$n.err; tail -c 300 gpurun_out/scale_c3sp$n.json
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 bench.py --config 3 --gpus 4 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/scale_c3tr4.json 2> gpurun_out/scale_c3tr4.err; tail -c 300 gpurun_out/scale_c3tr4.json
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q > gpurun_out/scale_multi.log 2>&1; tail -3 gpurun_out/scale_multi.log
