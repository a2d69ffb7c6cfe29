# A/B timing of resident-kernel variants on one B200 (profiles/r02_dr_kernel.md): build them
# here first, e.g.  python tools/variants.py a="" b="-DFIBRA_TOPO_REG=0"  (kernel-only -D
# variants, lib/variants/<name>.so and <name>_prof.so), or copy whole libraries built from
# different commits into lib/variants/; then  gpurun -- bash tools/gpu_variants.sh a b
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/var_build.log 2>&1
L=$PWD/paper_2306_09427_b200/lib/variants
for rep in 1 2; do for v in "$@"; do
  FIBRA_LIB=$L/$v.so timeout 300 python tools/prof_dr.py 296 4000 2>&1 | grep -o "us/iter.*" | sed "s/^/$v /"
done; done
for v in "$@"; do
  if [ -f $L/${v}_prof.so ]; then FIBRA_LIB=$L/${v}_prof.so FIBRA_PHASE_PROF=1 timeout 300 python tools/prof_dr.py 296 4000 2>&1 | tail -13; fi
  FIBRA_LIB=$L/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q 2>&1 | tail -1
done
