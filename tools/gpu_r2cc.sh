set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=index,name --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2cc_build.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/r2cc_tr4.json 2> gpurun_out/r2cc_tr4.err; tail -c 300 gpurun_out/r2cc_tr4.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 > gpurun_out/r2cc_tr2.json 2> gpurun_out/r2cc_tr2.err; tail -c 300 gpurun_out/r2cc_tr2.json
timeout 900 python bench.py --gpus 4 --single-process --no-cpu-baseline > gpurun_out/r2cc_sp4.json 2> gpurun_out/r2cc_sp4.err; tail -c 300 gpurun_out/r2cc_sp4.json
timeout 900 python bench.py --gpus 2 --single-process --no-cpu-baseline > gpurun_out/r2cc_sp2.json 2> gpurun_out/r2cc_sp2.err; tail -c 300 gpurun_out/r2cc_sp2.json
timeout 1200 python bench.py --config 3 --gpus 4 --single-process --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2cc_c3sp4.json 2> gpurun_out/r2cc_c3sp4.err; tail -c 300 gpurun_out/r2cc_c3sp4.json
timeout 1200 python bench.py --config 3 --gpus 2 --single-process --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2cc_c3sp2.json 2> gpurun_out/r2cc_c3sp2.err; tail -c 300 gpurun_out/r2cc_c3sp2.json
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q > gpurun_out/r2cc_multi.log 2>&1; tail -3 gpurun_out/r2cc_multi.log
