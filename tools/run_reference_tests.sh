# The reference's own hot-path test files (pkg/tests, installed with the
# reference into the git-ignored baseline/_ref by the sanctioned
#   pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>
# plus a copy of pkg/tests in baseline/_ref/lambdafmm_tests) run against the
# drop-in through the INTEGRATION.md §1 shim (tools/dropin_plugin.py).
mkdir -p gpurun_out
PYTHONPATH=baseline/_ref:. timeout 1500 python -m pytest -p no:cacheprovider -p tools.dropin_plugin -q \
  -o testpaths=baseline/_ref/lambdafmm_tests -c /dev/null \
  baseline/_ref/lambdafmm_tests/test_fmm_engine.py baseline/_ref/lambdafmm_tests/test_corrections.py \
  baseline/_ref/lambdafmm_tests/test_lattice.py baseline/_ref/lambdafmm_tests/test_oracle.py \
  baseline/_ref/lambdafmm_tests/test_dynamics.py baseline/_ref/lambdafmm_tests/test_acceptance.py \
  -m "not slow" 2>&1 | tail -40 > gpurun_out/r02_final_reference_tests_dropin.txt
tail -15 gpurun_out/r02_final_reference_tests_dropin.txt
