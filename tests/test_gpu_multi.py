"""Multi-GPU parity of the SP step over real NVSwitch peer memory (skipped on 1 GPU).

Runs scripts/mgpu_parity.py under torchrun on 2 (and 4 when present) GPUs with plans
produced by the reference planner, and checks the reassembled O / dQKV against the
single-process CPU oracle."""
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
CASES = [(2, "c1_flexsp_2tier.json", 8, 128), (2, "c1_static2.json", 8, 128),
         (4, "rand0_n4_flexsp.json", 8, 128), (4, "rand2_n4_flexsp.json", 8, 128),
         (8, "rand1_n8_flexsp.json", 8, 128),
         # uneven head splits: 5 heads over 2 ranks, 10 over 4
         (2, "c1_static2.json", 5, 128), (4, "rand0_n4_flexsp.json", 10, 128),
         # ranks left idle by a micro-batch (sum of degrees < N)
         (4, "idle_n4.json", 8, 128),
         # BASELINE configs[0] shape: C1 plan, 4 heads of 64 (h = 256)
         (2, "c1_flexsp_2tier.json", 4, 64)]


@pytest.mark.parametrize("n,plan,heads,head_dim", CASES)
def test_mgpu_step_matches_oracle(n, plan, heads, head_dim):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    env = dict(os.environ, OMP_NUM_THREADS="4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + n),
           str(ROOT / "scripts" / "mgpu_parity.py"), plan, str(heads), str(head_dim)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert '"ok": true' in res.stdout
