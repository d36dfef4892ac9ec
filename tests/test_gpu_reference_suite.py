"""The reference's OWN unit tests (pkg/tests, copied into the git-ignored
baseline/_ref_tests by tools/install_reference.sh, which travels to the GPU
box) run against this package: `lfps` is aliased to the device-backed
paper_2506_15704_b200.lfps (tests/lfps_alias.py), so every stage, state
type and oracle those tests call executes on the B200.

Files on the hot path (SURVEY §2.1 "parity pins"): test_tables,
test_candidates, test_attention, test_gate, test_engine, test_core.  The
format / CLI / exporter files are out of scope; test_acceptance's criteria
are measured on the reference's numpy generator (lfps.synth), which this
package restates statistically, not bitwise, so it is not run here."""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref_tests")
FILES = ("test_tables.py", "test_candidates.py", "test_attention.py", "test_gate.py",
         "test_engine.py", "test_core.py")


@pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                    reason="baseline/_ref_tests missing: run tools/install_reference.sh")
@pytest.mark.parametrize("name", FILES)
def test_reference_suite_file_passes(name):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), ROOT]),
               OPENBLAS_NUM_THREADS="1")
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "lfps_alias", "-p", "no:cacheprovider",
         os.path.join(REF_TESTS, name)],
        cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=900)
    tail = proc.stdout[-3000:]
    print(tail)
    m = re.search(r"(\d+) passed", proc.stdout)
    assert m and int(m.group(1)) > 0, tail
    assert proc.returncode == 0, tail
