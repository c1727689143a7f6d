# The reference's own test suite with its kernels on the GPU (SURVEY §8(a)
# parity contract: "the reference's own hot-path tests pass with the GPU
# kernels swapped in").
#
# Here (the container that has /root/reference), once:
#   cp -r /root/reference/pkg /tmp/refpkg
#   python -m pip install --no-index --no-build-isolation --no-deps \
#       --find-links /opt/wheelhouse --target baseline/_ref /tmp/refpkg
#   cp -r /tmp/refpkg/tests baseline/_ref/_tests
# (baseline/_ref is git-ignored and travels to the GPU box with gpurun), then
#   gpurun -- bash scripts/reference_suite_gpu.sh
# The pytest plugin rebinds kkbeam's kernel globals to libkkb before collection
# and prints the number of libkkb kernel launches at the end.
R=${GRAFT_REPO_ROOT:-$(pwd)}
cd /tmp && PYTHONPATH=$R/baseline/_ref:$R NUMBA_CACHE_DIR=/tmp/numba_cache \
  python -m pytest -p paper_2603_22496_b200.pytest_kkbeam_gpu "$R/baseline/_ref/_tests" \
  -q -p no:cacheprovider -rf > "$R/gpurun_out/refsuite_gpu.txt" 2>&1
grep -E "passed|failed|kernel launches|^criterion|^FAILED" "$R/gpurun_out/refsuite_gpu.txt"
