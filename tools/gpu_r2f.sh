set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=index,name --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/r2f_pytest.log 2>&1; tail -4 gpurun_out/r2f_pytest.log
timeout 900 python bench.py --config 3 --gpus 4 --single-process --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2f_c3sp4.json 2> gpurun_out/r2f_c3sp4.err; tail -c 300 gpurun_out/r2f_c3sp4.json; tail -3 gpurun_out/r2f_c3sp4.err
timeout 900 python bench.py --config 3 --gpus 2 --single-process --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2f_c3sp2.json 2> gpurun_out/r2f_c3sp2.err; tail -c 300 gpurun_out/r2f_c3sp2.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --config 3 --gpus 4 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2f_c3tr4.json 2> gpurun_out/r2f_c3tr4.err; tail -c 300 gpurun_out/r2f_c3tr4.json
timeout 600 python bench.py --gpus 4 --single-process --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2f_sp4.json 2> gpurun_out/r2f_sp4.err; tail -c 300 gpurun_out/r2f_sp4.json
FIBRA_PHASE_PROF=1 python -m paper_2306_09427_b200.build > gpurun_out/r2f_prof_build.log 2>&1
FIBRA_PHASE_PROF=1 timeout 300 python tools/prof_dr.py 296 4000 > gpurun_out/r2f_phase.log 2>&1; tail -16 gpurun_out/r2f_phase.log
