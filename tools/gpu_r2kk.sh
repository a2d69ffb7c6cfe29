set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2kk_build.log 2>&1
timeout 1200 python bench.py --config 3 --gpus 4 --single-process --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2kk_c3sp4.json 2> gpurun_out/r2kk_c3sp4.err; tail -c 300 gpurun_out/r2kk_c3sp4.json
timeout 1200 python bench.py --config 3 --gpus 2 --single-process --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2kk_c3sp2.json 2> gpurun_out/r2kk_c3sp2.err; tail -c 300 gpurun_out/r2kk_c3sp2.json
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --config 3 --gpus 4 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2kk_c3tr4.json 2> gpurun_out/r2kk_c3tr4.err; tail -c 300 gpurun_out/r2kk_c3tr4.json
