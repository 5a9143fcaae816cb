"""Fused apply -> gather over NVLink peer stores (8(e) collective row).

Two ranks, one GPU each: every rank's kernels store Y straight into rank 0's symmetric
buffer (bench.py --gather peer). bench.py compares the root's buffer with an NCCL
all-gather of the same outputs and reports "gather_check"; the test requires bitwise equality.
Needs two GPUs (gpurun --gpus 2); skipped on a one-GPU box.
"""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["tiny", "small", "medium"])
def test_peer_gather_bitwise_vs_nccl(config):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str({"tiny": 29611, "small": 29612, "medium": 29613}[config]),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", config, "--steps", "2", "--warmup", "3",
           "--gather", "peer", "--no-stages", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["gather_check"] == "bitwise equal to ncclAllGather", line
    assert line["info_nonzero"] == 0
