"""The reference's OWN tests for the averaging path, run against this
package: tests/ref_suite_plugin.py installs the drop-in (plugin.install)
before the reference's test modules import ravnest, so its run_allreduce,
apply_ring_mean and AllReduceController -- including the drain controller's
message replay over the reference's simnet -- are this package's.  On a CPU
container the GPU cycle is replaced by the oracle (host logic only); the
cycles themselves are checked on the GPU by tests/test_reference_seam_gpu.py.

Needs the reference's test tree -- /root/reference in the dev container, or
the copy kept with the offline install in baseline/_ref/ravnest_tests
(git-ignored like the install; it travels to the GPU box) -- and its package
(baseline/_ref); skipped elsewhere.  The -m gpu variant runs the same files
with the real GPU cycles."""

import os
import subprocess
import sys

import pytest

from conftest import REFERENCE_INSTALL, ROOT

def ref_tests():
    for path in (os.path.join(REFERENCE_INSTALL, "ravnest_tests"), "/root/reference/pkg/tests"):
        if os.path.isfile(os.path.join(path, "test_multiring.py")):
            return path
    return None


FILES = ["test_multiring.py", "test_orchestrator.py", "test_oracle.py", "test_cli.py"]
# fails in the unmodified reference on Python 3.12 too (sum() rounding in the
# test itself; SURVEY.md headline fact 4), with or without the drop-in
KNOWN_REFERENCE_FAILURE = "test_six_random"  # test_oracle.py::TestMeanReference


def run_reference_suite(tmp_path, oracle_cycle: bool, files=FILES):
    tests = ref_tests()
    if tests is None or not os.path.isdir(os.path.join(REFERENCE_INSTALL, "ravnest")):
        pytest.skip("needs the reference's tests and baseline/_ref")
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", RAVNEST_B200_ORACLE_CYCLE="1" if oracle_cycle else "0",
               PYTHONPATH=os.pathsep.join([REFERENCE_INSTALL, os.path.join(ROOT, "tests"), ROOT]))
    cmd = [sys.executable, "-m", "pytest", "-p", "ref_suite_plugin", "-p", "no:cacheprovider", "-q",
           "-k", f"not {KNOWN_REFERENCE_FAILURE}"]
    cmd += [os.path.join(tests, f) for f in files]
    res = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=900)
    tail = res.stdout[-3000:] + res.stderr[-2000:]
    assert res.returncode == 0, tail
    assert " passed" in res.stdout and " failed" not in res.stdout, tail
    import re

    m = re.search(r"routed to paper_2401_01728_b200: (\d+) cycles through the drop-in", res.stdout)
    assert m and int(m.group(1)) > 100, tail  # the reference's averaging calls really ran here
    return res.stdout


def test_reference_averaging_tests_pass_through_the_drop_in(tmp_path):
    run_reference_suite(tmp_path, oracle_cycle=True)


@pytest.mark.gpu
def test_reference_averaging_tests_pass_on_the_gpu(tmp_path):
    """The same reference test files, plus its acceptance suite
    (test_acceptance.py: criterion 1's 1000 random instances, the training
    criteria, the cost model), with every averaging cycle on the GPU
    (float64 kernel, bitwise the reference)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    run_reference_suite(tmp_path, oracle_cycle=False, files=FILES + ["test_acceptance.py"])
