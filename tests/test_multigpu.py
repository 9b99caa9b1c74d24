"""Real multi-process NVLink path: torchrun one rank per GPU, CUDA-IPC peer
exchange buffers, fused FFT + peer-store kernels, device barriers
(tests/mgpu_check.py).  Skipped on boxes with fewer than 2 GPUs."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))

pytestmark = pytest.mark.gpu


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


# default: the shipped thresholds (these small cases exchange by direct peer
# stores); staged: every eligible exchange goes through staging images and
# copy-engine DMAs (size thresholds off), checked to have run
MODES = {"default": {}, "staged": {"DFFTB_DMA_MIN_MB": "0", "DFFTB_DMA_MIN_ROW": "0", "DFFTB_DMA_MAX_GROUP": "64",
                               "DFFTB_EXPECT_STAGED": "1"}}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_parity(n, mode):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n + (10 if mode != "default" else 0)),
           os.path.join(HERE, "mgpu_check.py")]
    env = dict(os.environ, **MODES[mode])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
