"""GPU: the reference's OWN GoogleTest unit tests (proj/tests/{matrix,quantize,linear,optimizer}_test.cpp),
compiled unchanged against the B200 lowprec shim (INTEGRATION.md option A, tests/reftests/build.sh),
run on the B200. Every lowprec:: numeric call in them goes through the C-ABI kernels."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "reftests")
SUITES = ["matrix_test", "quantize_test", "linear_test", "optimizer_test"]

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_b200(suite):
    exe = os.path.join(BIN, suite)
    if not os.path.exists(exe):
        subprocess.run(["bash", os.path.join(ROOT, "tests", "reftests", "build.sh")], check=False)
    if not os.path.exists(exe):
        pytest.skip("reference test binaries not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    tail = "\n".join(r.stdout.splitlines()[-5:])
    failed = [l for l in r.stdout.splitlines() if "FAILED" in l]
    assert r.returncode == 0, f"{suite}: {failed}\n{r.stderr[-3000:]}\n{tail}"
