set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2o_build.log 2>&1
for v in v_r1n0 v_r0n0 v_r1n1 v_r0n1; do
  L=$PWD/paper_2306_09427_b200/lib/variants
  FIBRA_LIB=$L/$v.so timeout 300 python tools/prof_dr.py 296 4000 > gpurun_out/r2o_$v.log 2>&1
  FIBRA_LIB=$L/$v.so timeout 300 python tools/prof_dr.py 296 4000 >> gpurun_out/r2o_$v.log 2>&1
  FIBRA_LIB=$L/${v}_prof.so FIBRA_PHASE_PROF=1 timeout 300 python tools/prof_dr.py 296 4000 >> gpurun_out/r2o_$v.log 2>&1
  FIBRA_LIB=$L/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q -k "single_rve or batch_tangent or config1 or config2_full" >> gpurun_out/r2o_$v.log 2>&1
  tail -18 gpurun_out/r2o_$v.log
done
