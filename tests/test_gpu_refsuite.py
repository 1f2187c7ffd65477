"""The reference's own doctest suites (proj/tests/test_*.cpp), compiled
unchanged against the B200 C++ host layer instead of the reference library
(`make -C oracle refsuite`: tests/refsuite/tsdfslam/*.hpp resolve the
reference's headers to include/refusion_b200.hpp). Every assertion of those
suites then runs on the GPU implementation. The binaries are built where
/root/reference exists (build() in this container) and travel with the repo.
"""
import glob
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = sorted(glob.glob(os.path.join(ROOT, "oracle", "_ref", "suite_test_*")))


def test_refsuite_sources_resolve_to_the_host_layer():
    """Every compat header maps a reference header name onto the host layer only."""
    for path in glob.glob(os.path.join(ROOT, "tests", "refsuite", "tsdfslam", "*.hpp")):
        text = open(path).read()
        assert '#include "refusion_b200.hpp"' in text and "using namespace tsdfslam_b200;" in text, path


@pytest.mark.gpu
@pytest.mark.parametrize("exe", SUITES, ids=[os.path.basename(p) for p in SUITES])
def test_reference_suite_on_gpu(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    summary = [l for l in r.stdout.splitlines() if l.startswith("[doctest-shim] test cases:")]
    assert summary and "| 0 failed |" in summary[-1] and summary[-1].endswith("| 0 failed"), r.stdout[-2000:]
