"""Host-side FASTQ ingestion and SAM formatting (include/qgmap/fastq.hpp,
sam.hpp): runs the C++ suite tests/cpp/test_fastq, which makes no device
calls, on the CPU."""
import os
import subprocess

import pytest

from qgm_testutil import ROOT


def test_fastq_and_sam_suite():
    exe = os.path.join(ROOT, "tests", "cpp", "build", "test_fastq")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/build/test_fastq not built (make tests)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    tail = out.stdout[-3000:] + "\n" + out.stderr[-3000:]
    assert out.returncode == 0, tail
    assert " 0 failed" in out.stdout.strip().splitlines()[-1], tail
