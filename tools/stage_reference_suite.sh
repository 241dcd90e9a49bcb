# Stage the reference's test suite and a reference install (git-ignored, never
# committed) so tests/test_gpu_reference_suite.py can run them against the shim.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/refcopy baseline/_ref baseline/_ref_tests
cp -r /root/reference/pkg /tmp/refcopy
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/refcopy
cp -r /root/reference/pkg/tests baseline/_ref_tests
