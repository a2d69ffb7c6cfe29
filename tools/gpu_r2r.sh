set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r_build.log 2>&1
for v in nm; do
  L=$PWD/paper_2306_09427_b200/lib/variants
  FIBRA_LIB=$L/$v.so timeout 300 python tools/prof_dr.py 296 4000 > gpurun_out/r2r_$v.log 2>&1
  FIBRA_LIB=$L/${v}_prof.so FIBRA_PHASE_PROF=1 timeout 300 python tools/prof_dr.py 296 4000 >> gpurun_out/r2r_$v.log 2>&1
  FIBRA_LIB=$L/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q -k "single_rve or batch_tangent or config1 or config2_full or capped or exact or tie" >> gpurun_out/r2r_$v.log 2>&1
  tail -18 gpurun_out/r2r_$v.log
done
timeout 600 python bench.py > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err; tail -c 300 gpurun_out/r2r_bench.json
