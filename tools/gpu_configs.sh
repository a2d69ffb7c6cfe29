# Configs 3-5 at full size on one B200 plus the GPU parity suite (profiles/bench_r02_c*_final.json).
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cfg_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/cfg_pytest.log 2>&1; tail -3 gpurun_out/cfg_pytest.log
for c in 4 5 3; do
  timeout 1200 python bench.py --config $c --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/cfg_c$c.json 2> gpurun_out/cfg_c$c.err; tail -c 300 gpurun_out/cfg_c$c.json
done
# per-class completion times of the config-3 batch (FIBRA_CLASS_TIMES): tools/config3_classes.py
