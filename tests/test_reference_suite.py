"""The reference's own hot-path tests, unchanged, against the B200 path.

north_star: the reference's Python API is kept "so ... its callers work
unchanged".  build() stages the reference's test files (pkg/tests, copied
verbatim, git-ignored) under baseline/_ref_tests; this test runs three of
them -- test_features.py, test_mesh.py, test_acceptance.py with the
reference's conftest.py -- in a subprocess whose `import shapecore` resolves
to compat/shapecore, i.e. to the B200 implementation.  Deselected, because
they test the reference's CPU dispatcher rather than results: the parallel
backend's CPU speedup, the SHAPECORE_FORCE_SEQUENTIAL fallback, and the CPU
diameter-time share (`test_parallel_speedup`, `test_fallback_contract`,
`test_diameter_dominance`).
"""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SUITE = os.path.join(ROOT, "baseline", "_ref_tests")
FILES = ("test_features.py", "test_mesh.py", "test_acceptance.py")
DESELECT = ("test_acceptance.py::test_parallel_speedup", "test_acceptance.py::test_fallback_contract",
            "test_acceptance.py::test_diameter_dominance")


@pytest.mark.timeout(1200)
def test_reference_tests_pass_on_the_b200_path(cuda_device):
    if not all(os.path.isfile(os.path.join(SUITE, f)) for f in FILES + ("conftest.py",)):
        pytest.skip("reference tests not staged (build() stages them where /root/reference exists)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "compat"), ROOT,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", SUITE,
           *FILES, *(f"--deselect={d}" for d in DESELECT),
           "-o", "filterwarnings=ignore::DeprecationWarning"]
    r = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=1150)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    # the run must really be the B200 package (compat/shapecore), not the reference
    probe = subprocess.run([sys.executable, "-c", "import shapecore; print(shapecore.__file__)"],
                           cwd=SUITE, env=env, capture_output=True, text=True)
    assert os.path.join("compat", "shapecore") in probe.stdout, probe.stdout + probe.stderr
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
