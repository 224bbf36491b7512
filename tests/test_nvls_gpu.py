"""NVLS in-switch reduction (afdk_nvls_*) across processes on >= 2 GPUs of one
NVSwitch box (tests/nvls_check.py under torchrun); skipped on one GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_nvls_reduce_multi_process(tmp_path):
    import torch

    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("NVLS needs >= 2 GPUs")
    out = tmp_path / "nvls.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(n, 4)}",
           "--master-addr", "127.0.0.1", f"--master-port={29600 + os.getpid() % 1000}",
           os.path.join(ROOT, "tests", "nvls_check.py"), "--out", str(out)]
    res = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ, PYTHONPATH=ROOT), capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    if not out.exists():
        pytest.skip("NVLS unsupported on this system: " + res.stdout[-500:])
    got = json.load(open(out))
    assert got["nvls"] == "ok" and got["rel_err"] <= 1e-2, got
