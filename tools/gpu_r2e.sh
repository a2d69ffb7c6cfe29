set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=index,name --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2e_pytest.log 2>&1; tail -8 gpurun_out/r2e_pytest.log
timeout 600 python bench.py --gpus 2 --single-process --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2e_sp2.json 2> gpurun_out/r2e_sp2.err; tail -c 900 gpurun_out/r2e_sp2.json; tail -3 gpurun_out/r2e_sp2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2e_tr2.json 2> gpurun_out/r2e_tr2.err; tail -c 600 gpurun_out/r2e_tr2.json
timeout 900 python bench.py --config 3 --gpus 2 --single-process --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2e_c3sp2.json 2> gpurun_out/r2e_c3sp2.err; tail -c 900 gpurun_out/r2e_c3sp2.json; tail -3 gpurun_out/r2e_c3sp2.err
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2e_c3n1.json 2> gpurun_out/r2e_c3n1.err; tail -c 600 gpurun_out/r2e_c3n1.json
