set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ii_build.log 2>&1
FIBRA_RESIDENT_SKIP=2 timeout 1200 python tools/config3_classes.py > gpurun_out/r2ii_classes.log 2>&1; tail -16 gpurun_out/r2ii_classes.log
for c in 3 5; do
FIBRA_RESIDENT_SKIP=2 timeout 1200 python bench.py --config $c --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r2ii_c$c.json 2> gpurun_out/r2ii_c$c.err; tail -c 300 gpurun_out/r2ii_c$c.json
done
