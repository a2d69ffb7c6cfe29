set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2jj_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2jj_pytest.log 2>&1; tail -3 gpurun_out/r2jj_pytest.log
for c in 4 5 3; do
timeout 1200 python bench.py --config $c --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2jj_c$c.json 2> gpurun_out/r2jj_c$c.err; tail -c 300 gpurun_out/r2jj_c$c.json; tail -2 gpurun_out/r2jj_c$c.err
done
