"""Device out-of-bounds writes (compute-sanitizer is not available on this GPU
pool): the GPU parity suites re-run with LG_CHECK_CANARY=1, where every
device buffer carries a 4 KiB 0xA5 guard band verified when the buffer is
released (lg_device.cu Buf); any overwrite fails the run."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.gpu
def test_no_device_buffer_overrun():
    env = dict(os.environ, LG_CHECK_CANARY="1")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                          "tests/test_ref_parity.py", "tests/test_boundary.py",
                          "tests/test_multigpu.py", "tests/test_gpu_parity.py",
                          "-k", "not full_size and not bench_config"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    assert "canary_violations=0" in out.stdout, tail
