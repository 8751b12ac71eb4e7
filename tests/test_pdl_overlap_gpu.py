"""The opt-in PDL overlap (AXE_PDL_OVERLAP=1: a copy proven disjoint from every libaxe kernel in flight on
its stream skips griddepcontrol.wait, plan.cpp stream_dependency) under the dependency tests that exercise
it: RAW / WAR chains, the two-launches-back window, concurrent host threads, and the TMA plan's public
execute between copies.  The variable is read once per process, so the tests run in a child pytest."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_dependency_tests_with_overlap_enabled():
    env = dict(os.environ, AXE_PDL_OVERLAP="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_copy_gpu.py"),
                        os.path.join(ROOT, "tests", "test_tma_region_gpu.py"),
                        "-k", "pdl or concurrent or without_sync"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " passed" in r.stdout and "deselected" in r.stdout
