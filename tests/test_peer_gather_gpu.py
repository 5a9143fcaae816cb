"""Fused apply -> gather over NVLink peer stores (8(e) collective row).

Two ranks, one GPU each.  --gather comm / comm-peer use the library's multi-GPU C ABI
(stap_comm_*); the others hand torch symmetric-memory addresses to the same kernels: every
rank's kernels store Y straight into rank 0's symmetric
buffer (bench.py --gather peer); with peer-all every Y store is written locally and
repeated into the peer's buffer (stap_params.out_n_peers); with multimem, every Y store is a multimem.st to the
buffer's NVLS multicast address and lands in both ranks' buffers (--gather multimem).
bench.py compares the gathered buffer (rank 0; every rank for multimem) with an NCCL
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
@pytest.mark.parametrize("gather", ["comm", "comm-peer", "comm-push", "peer", "peer-all", "multimem"])
@pytest.mark.parametrize("config", ["tiny", "small", "medium"])
def test_peer_gather_bitwise_vs_nccl(config, gather):
    """comm / comm-peer: the library's own stap_comm (C ABI: stap_comm_init_rank,
    stap_comm_allgather_out, stap_comm_peer_offsets with CUDA IPC); peer / peer-all / multimem:
    torch symmetric memory handing peer or multicast addresses to the same epilogue stores."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    port = 29611 + {"tiny": 0, "small": 1, "medium": 2}[config] + 5 * ["peer", "peer-all", "multimem", "comm",
                                                                         "comm-peer", "comm-push"].index(gather)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", config, "--steps", "2", "--warmup", "3",
           "--gather", gather, "--no-stages", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["gather_check"] == "bitwise equal to ncclAllGather", line
    assert line["info_nonzero"] == 0


@pytest.mark.gpu
def test_run_host_rejects_multicast_out():
    """A host `out` is never a multicast address: stap_run_host returns STAP_ERR_UNSUPPORTED."""
    import paper_2203_06233_b200 as stap
    sys.path.insert(0, ROOT)
    import synth
    cfg = synth.CONFIGS["tiny"]
    dims = stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam)
    plan = stap.StapPlan(dims, out_multicast=True)
    hc = torch.zeros(plan.cube_shape, dtype=torch.complex64).pin_memory()
    hs = torch.zeros((cfg.S, cfg.C * cfg.T), dtype=torch.complex64).pin_memory()
    ho = torch.empty(plan.out_shape, dtype=torch.complex64).pin_memory()
    hi = torch.empty(plan.info_shape, dtype=torch.int32).pin_memory()
    ws = torch.empty(max(plan.host_workspace_bytes, 16), dtype=torch.uint8, device="cuda:0")
    with pytest.raises(stap.StapError) as e:
        plan.run_host(hc, hs, ho, hi, ws)
    assert e.value.code == 3


@pytest.mark.gpu
@pytest.mark.parametrize("config,split", [("medium", "strong"), ("large", "strong"), ("large", "weak")])
def test_bench_split_two_gpus(config, split):
    """bench.py's 2-GPU shards (weak: a D_cfg-bin slice per rank; strong: one cube split in two)
    run through the C ABI with every unit healthy, and the whole-job value is counted in the
    split's unit (strong: whole cubes)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    port = 29700 + 3 * ["medium", "large"].index(config) + (split == "weak")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", config, "--split", split, "--steps", "3",
           "--warmup", "3", "--no-stages", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["scaling"] == split and line["n_gpus"] == 2 and line["info_nonzero"] == 0
    cubes = {"medium": 16, "large": 2}[config] * (1 if split == "strong" else 2)  # whole-job cubes per step
    assert abs(line["value"] * line["ms_per_step"] / 1e3 - cubes) < 1e-6 * cubes
