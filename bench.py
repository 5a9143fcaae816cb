#!/usr/bin/env python
"""bench.py -- STAP datacubes/s on 1..N B200s (BASELINE.json metric), one JSON line.

Workload: BASELINE.json configs[3] "STAP large" by
default (8 channels, TDOF 7, 1024 Doppler bins, 4096 range cells, 16 steering
vectors, training block 128) -- the largest configuration that fits one GPU and,
per GPU, the configs[4] weak-scaling slice; --config small|medium select
configs[1]/[2].  A step is one pass of the whole hot path (covariance + loading,
Cholesky + solves -> MVDR weights, application) over a batch of `--cubes`
distinct seeded synthetic datacubes resident in HBM (input > L2, so no L2 flush
is needed).  --precision tf32x3 (default) opts the covariance and the apply into
the library's 3xTF32 tcgen05 stages (stap_params.precision; FP32-level accuracy,
parity-tested against the fp64 oracle); --precision fp32 runs FP32 FFMA only.

Multi-GPU (torchrun, one process per GPU, NCCL): Doppler-bin shards.  --split weak
(default; BASELINE.json configs[4]): the global cube has D = D_cfg x N bins, rank g
owns the contiguous slice [g*D_cfg, (g+1)*D_cfg) plus a T-1 bin read-only halo, so
per-GPU work is fixed; `value` counts every D_cfg-bin slice processed as one
config-shaped datacube, summed over ranks.  --split strong (configs[2] "medium on
1/2/4/8"): every step's cubes are the config's D bins split D/N per rank, so the
work per step is fixed; `value` = whole cubes per second.  No collective is on the
data path; --gather adds the optional gather of the outputs.

--impl reference times the fp64 C oracle (the reference arm for this tier) on
the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

WORKLOAD_DESC = {
    "tiny": "STAP tiny (BASELINE.json configs[0])",
    "small": "STAP small (BASELINE.json configs[1]): C=4, TDOF=3, D=256, R=512, S=16, K=32",
    "medium": "STAP medium (BASELINE.json configs[2]): C=6, TDOF=5, D=512, R=1024, S=16, K=64",
    "large": "STAP large (BASELINE.json configs[3]): C=8, TDOF=7, D=1024, R=4096, S=16, K=128",
}
DEFAULT_CUBES = {"tiny": 64, "small": 64, "medium": 16, "large": 2}
# TF32 dense tensor peak = measured bf16 x the guide's nominal ratio (1.1 / 2.25 PFLOP/s)
TF32_PER_BF16 = 1.1 / 2.25


# ---------------------------------------------------------------- algorithmic counts
def counts(cfg: synth.StapConfig) -> dict:
    """Per-cube algorithmic flops/bytes of the method.
    cov_lag counts the Doppler-lag-shared covariance (the minimum work, what K1/K4 execute);
    cov_bin the per-bin Hermitian count."""
    C, T, D, R, K, S, N, B = cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.N, cfg.B
    X = D * C * R * 8
    Y = S * D * R * 8
    Rp = D * B * N * (N + 1) // 2 * 8
    Wb = D * B * S * N * 8
    Gb = D * B * S * 4
    f = {
        "cov_bin": 8.0 * D * R * N * (N + 1) / 2,
        "cov_lag": 8.0 * D * R * (C * (C + 1) / 2 + (T - 1) * C * C),
        "chol": (4.0 / 3.0) * N ** 3 * D * B,
        "solve": 8.0 * N * N * S * D * B,
        "apply": 8.0 * N * S * D * R,
    }
    return {
        "flops_fused_lag": f["cov_lag"] + f["chol"] + f["solve"] + f["apply"],
        "flops_fused_bin": f["cov_bin"] + f["chol"] + f["solve"] + f["apply"],
        "bytes_fused": X + Y,
        "stage": {
            "covariance": {"flops": f["cov_lag"], "flops_bin": f["cov_bin"], "bytes": X + Rp},
            "solve": {"flops": f["chol"] + f["solve"], "bytes": Rp + Wb + Gb},
            "apply": {"flops": f["apply"], "bytes": X + Wb + Y},
        },
    }


def peaks() -> dict:
    """Roofline denominators: MEASURED_PEAKS.json (driver-written) else the profiling guide's fallback.
    FP32 SIMT peak = 148 SMs x 128 FP32 lanes x 2 flop x sm_max clock."""
    p = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            m = json.load(fh)
        p.update(hbm_gbs=float(m["hbm_gbs"]), sm_max_mhz=float(m.get("sm_max_mhz", 1965.0)),
                 source="measured (MEASURED_PEAKS.json)")
    except Exception:
        pass
    p["fp32_tflops"] = 148 * 128 * 2 * p["sm_max_mhz"] * 1e6 / 1e12
    bf16 = 1590.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            bf16 = float(json.load(fh)["bf16_tflops"])
    except Exception:
        pass
    p["tf32_tflops"] = bf16 * TF32_PER_BF16
    return p


def roofline_obj(flops: float, nbytes: float, seconds: float, pk: dict, traffic=None, extra=None,
                 tensor: bool = False) -> dict:
    """frac = t_roof / t_meas.  FP32 SIMT stages: t_roof = max(bytes / HBM, flops / FP32 peak).
    tcgen05 3xTF32 stages: t_roof = max(bytes / HBM, 3 x flops / TF32 peak) -- three TF32 MMAs
    per FP32-accurate product, TF32 peak = measured bf16 x 1.1/2.25 (B200_PROFILING.md)."""
    t_hbm = nbytes / (pk["hbm_gbs"] * 1e9)
    if tensor:
        t_alu = 3.0 * flops / (pk["tf32_tflops"] * 1e12)
        if t_alu >= t_hbm:
            ach = 3.0 * flops / seconds / 1e12
            o = {"bound": "tensor", "achieved": ach, "peak": pk["tf32_tflops"], "unit": "TFLOP/s",
                 "frac": ach / pk["tf32_tflops"], "note": "3xTF32: achieved counts 3 TF32 MMAs per algorithmic flop"}
        else:
            ach = nbytes / seconds / 1e9
            o = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ach / pk["hbm_gbs"]}
        o["frac_of_fp32_simt"] = flops / seconds / 1e12 / pk["fp32_tflops"]
    else:
        t_alu = flops / (pk["fp32_tflops"] * 1e12)
        if t_alu >= t_hbm:
            ach = flops / seconds / 1e12
            o = {"bound": "alu", "achieved": ach, "peak": pk["fp32_tflops"], "unit": "TFLOP/s",
                 "frac": ach / pk["fp32_tflops"]}
        else:
            ach = nbytes / seconds / 1e9
            o = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ach / pk["hbm_gbs"]}
    o["traffic"] = traffic
    if extra:
        o.update(extra)
    return o


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock, max clock and throttle reasons with NVML every ~2 ms on a
    background thread while the timed region runs (the host thread is blocked in
    a CUDA synchronize meanwhile)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = None
        self._thr = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.index]) if vis else self.index
            self._h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self._nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            return self
        self._stop = threading.Event()

        def run():
            nv = self._nv
            while not self._stop.is_set():
                try:
                    sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                    self.samples.append((sm, rs))
                except Exception:
                    pass
                self._stop.wait(0.002)

        self._thr = threading.Thread(target=run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *a):
        if self._thr is not None:
            self._stop.set()
            self._thr.join(timeout=2)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sms = [s for s, _ in self.samples]
        reasons = set()
        for _, r in self.samples:
            for name, bit in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(sms), "source": "NVML, every ~2 ms during the timed region"}


# ---------------------------------------------------------------- inputs
def plan_shape_out(stap, dims, lo, cnt, b0, nb, M):
    """Y's shape for a plan of these dims (include/stap.h: [batch][Dl][S][R])."""
    return (M, cnt, dims.S, dims.R)


def peer_gather_setup(out, world, rank, dev, dist, mode="peer"):
    """Fused apply -> gather (the root variant of 8(e)'s collective row).

    One symmetric buffer [world][*out.shape] per rank (torch symmetric memory: the same
    allocation mapped into every peer's address space over NVLink). Rank r's kernels are
    handed rank 0's slice r as their Y pointer, so the apply epilogue's stores travel over
    NVLink straight into the root's buffer: no separate gather pass and no HBM re-read of Y.
    A device-side barrier after each step orders the stores before anyone reads them.
    Returns (the local buffer as [world][*out.shape] complex64, this rank's destination (view or address),
    the rendezvous handle, the peer byte offsets for peer-all).

    peer-all: the destination is this rank's own slice r, and the plan repeats every Y
    store at the byte offsets to slice r of every peer's buffer (stap_params.out_peer_offset):
    an all-gather by unicast stores, each GPU's NVLink ingress carrying only the peers' slices.

    multimem: the destination is instead the buffer's NVLS multicast address + slice r
    (an int); the plan's out_multicast makes every Y store a multimem.st, so each rank's
    apply epilogue writes its slice into ALL ranks' buffers: an all-gather with no
    separate pass."""
    import torch
    import torch.distributed._symmetric_memory as symm_mem
    n = out.numel() * 2  # floats per rank slice
    buf = symm_mem.empty(world * n, dtype=torch.float32, device=dev)
    hdl = symm_mem.rendezvous(buf, dist.group.WORLD.group_name)
    offs = ()
    if mode == "peer-all":
        dst = buf[rank * n:(rank + 1) * n].view(torch.complex64).view(out.shape)
        base = dst.data_ptr()
        offs = tuple(hdl.get_buffer(j, (n,), torch.float32, rank * n).data_ptr() - base
                     for j in range(world) if j != rank)
    elif mode == "multimem":
        if not getattr(hdl, "multicast_ptr", 0):
            raise RuntimeError("--gather multimem: no NVLS multicast support on this box")
        dst = int(hdl.multicast_ptr) + rank * n * 4
    else:
        dst = hdl.get_buffer(0, (n,), torch.float32, rank * n).view(torch.complex64).view(out.shape)
    return buf.view(torch.complex64).view((world,) + tuple(out.shape)), dst, hdl, offs


def shard_plan_args(cfg, n_gpus, rank, split="weak"):
    """(global config, dop_begin, dop_count, cube_bin0, cube_bins) of this rank's shard plan.
    weak: global D = D_cfg * N, rank g owns [g D_cfg, (g+1) D_cfg); strong: the config's D bins
    split D/N per rank (synth.shard_range).  N = 1: the whole cube, no halo."""
    if n_gpus <= 1:
        return cfg, 0, cfg.D, 0, cfg.D
    if split == "weak":
        gcfg = cfg.with_(D=cfg.D * n_gpus)
        lo, cnt = rank * cfg.D, cfg.D
    else:
        gcfg = cfg
        lo, cnt = synth.shard_range(cfg.D, n_gpus, rank)
    b0, nb = synth.shard_window(gcfg, lo, cnt)
    return gcfg, lo, cnt, b0, nb


def make_inputs(cfg, n_gpus, rank, cubes, steering_kind="ula", split="weak"):
    """This rank's cube buffers [cubes][Dl + halo][C][R] (halo only when N > 1), complex64."""
    gcfg, lo, cnt, b0, nb = shard_plan_args(cfg, n_gpus, rank, split)
    bins = (b0 + np.arange(nb)) % gcfg.D
    x = np.empty((cubes, nb, cfg.C, cfg.R), np.complex64)
    for i in range(cubes):
        x[i] = synth.datacube_bins(gcfg, bins, cube_idx=i)
    st = synth.steering(cfg, steering_kind)
    return gcfg, lo, cnt, b0, nb, x, st


# ---------------------------------------------------------------- reference arm (the oracle)
def cpu_oracle_rate(cfg, budget_s: float, max_steps=None, sample_bins=None):
    """Time the fp64 oracle (as it stands) on the host cores on a bounded sample; return
    (cubes/s, cores, sample description, per-step seconds list)."""
    import oracle
    cores = len(os.sched_getaffinity(0)) or (os.cpu_count() or 1)
    bins = cfg.D if sample_bins is None else min(sample_bins, cfg.D)
    d0 = cfg.D // 2 - bins // 2 if bins < cfg.D else 0
    b0, nb = synth.shard_window(cfg, d0, bins)
    local = synth.datacube_bins(cfg, (b0 + np.arange(nb)) % cfg.D, cube_idx=0)
    st = synth.steering(cfg, "ula")
    p = oracle.OracleParams(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam, dop_begin=d0, dop_count=bins,
                            cube_bin0=b0, cube_bins=nb)
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        oracle.run(p, local, st, nthreads=cores)
        times.append(time.perf_counter() - t0)
        if max_steps is not None and len(times) >= max_steps:
            break
        if time.perf_counter() - t_start >= budget_s:
            break
    per = statistics.median(times)
    rate = (bins / cfg.D) / per
    sample = f"{bins} of {cfg.D} Doppler bins of one {cfg.name} cube per run, {len(times)} runs, fp64 C oracle, OpenMP over bins"
    return rate, cores, sample, times


def oracle_sample_bins(cfg):
    # ~0.3-2 s per oracle call on a many-core host
    return {"tiny": cfg.D, "small": cfg.D, "medium": 128, "large": 16}.get(cfg.name, cfg.D)


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    bins = oracle_sample_bins(cfg)
    _, _, sample, _ = cpu_oracle_rate(cfg, 0.0, max_steps=max(1, args.warmup), sample_bins=bins)
    rate, cores, sample, times = cpu_oracle_rate(cfg, 1e9, max_steps=args.steps, sample_bins=bins)
    ms = statistics.median(times) * 1e3
    line = {
        "impl": "reference", "metric": "STAP datacubes/sec", "value": rate, "unit": "cubes/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_obj(args, cfg, world),
        "cpu_baseline": {"value": rate, "unit": "cubes/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": rate, "unit": "cubes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_obj(args, cfg, world, path=None):
    if world > 1 and args.split == "strong":
        par = f"doppler-shard x{world} (strong: D = {cfg.D} split {cfg.D // world} bins per rank + halo)"
        per_gpu = f"{args.cubes} cubes x 1/{world} of the bins"
    else:
        par = f"doppler-shard x{world} (weak: global D = {cfg.D}*{world})"
        per_gpu = args.cubes
    return {"workload": WORKLOAD_DESC.get(cfg.name, cfg.name), "C": cfg.C, "TDOF": cfg.T, "D": cfg.D, "R": cfg.R,
            "S": cfg.S, "K": cfg.K, "lambda": cfg.lam, "cubes_per_step_per_gpu": per_gpu,
            "parallelism": par, "precision": precision_desc(args.precision, path),
            "l2": "inputs larger than L2 (no flush)", "steering": "ULA centre-bin",
            **({"gather": args.gather} if args.gather and world > 1 else {})}


def precision_desc(prec, path):
    """The arithmetic the timed path actually runs (the plan decides per shape)."""
    if prec == "tf32x3" and path is not None and "tcgen05" not in path:
        return ("stap_params.precision=STAP_PREC_TF32X3 requested; this shape's path (" + path.split(":")[0] +
                ") has no tcgen05 stage, so every stage runs FP32 FFMA")
    return PRECISION_DESC[prec]


PRECISION_DESC = {
    "tf32x3": "stap_params.precision=STAP_PREC_TF32X3: covariance and apply on tcgen05 in 3xTF32 (FP32-level "
              "accuracy, oracle parity <= 1e-3 per output vector), Cholesky/solves FP32 FFMA",
    "fp32": "stap_params.precision=STAP_PREC_FP32: FP32 FFMA in every stage",
}


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=list(WORKLOAD_DESC), default="large")
    ap.add_argument("--cubes", type=int, default=None, help="cubes per step per GPU")
    ap.add_argument("--path", choices=["auto", "fused", "staged"], default="auto",
                    help="stap_run path (stap_params.path); auto = the library's measured choice")
    ap.add_argument("--precision", choices=["tf32x3", "fp32"], default="tf32x3",
                    help="stap_params.precision: tf32x3 = tcgen05 3xTF32 covariance/apply (default), fp32 = FFMA only")
    ap.add_argument("--split", choices=["weak", "strong"], default="weak",
                    help="N > 1: weak = a D_cfg-bin slice per rank (configs[4]); strong = one D-bin cube split N ways")
    ap.add_argument("--gather", nargs="?", const="comm", default=None,
                    choices=["comm", "comm-peer", "comm-push", "nccl", "nccl-root", "peer", "peer-all", "multimem"],
                    help="gather the outputs after each step: comm = the library's stap_comm_allgather_out "
                         "(in-place ncclAllGather; the default of a bare --gather); comm-peer = the library's "
                         "stap_comm_peer_offsets + out_n_peers: the all-gather fused into the apply epilogue by "
                         "peer stores (CUDA IPC mapping), a 1-float all-reduce per step as the device barrier; "
                         "comm-push = the library's stap_comm_push_out: copy-engine peer copies of each step's "
                         "slice on a second stream, overlapping the next step's covariance and solve; "
                         "baselines through torch: nccl = all_gather_into_tensor, nccl-root = gather to rank 0, "
                         "peer / peer-all / multimem = torch symmetric memory + the same epilogue stores "
                         "(SURVEY 8(f) NEXT-2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-stages", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    if args.cubes is None:
        args.cubes = DEFAULT_CUBES[args.config]
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        world = max(world, 1)

    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2203_06233_b200 as stap

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        # NCCL prints a version banner on stdout when the first communicator is built; the
        # contract is one JSON line there, so fd 1 points at stderr until that has happened
        os.environ["NCCL_DEBUG"] = os.environ.get("STAP_NCCL_DEBUG", "WARN")
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=dev)
            dist.barrier(device_ids=[local_rank])
            torch.cuda.synchronize(dev)
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)

    gcfg, lo, cnt, b0, nb, x_h, st_h = make_inputs(cfg, world, rank, args.cubes, split=args.split)
    M = args.cubes
    dims = stap.Dims(cfg.C, cfg.T, gcfg.D, cfg.R, cfg.K, cfg.S, cfg.lam)
    multi = world > 1
    mc = args.gather == "multimem" and multi
    out = torch.empty(plan_shape_out(stap, dims, lo, cnt, b0, nb, M), dtype=torch.complex64, device=dev)
    gather_buf, y_dst, peer, offs, comm, step_bar = None, out, None, (), None, None
    if args.gather in ("peer", "peer-all", "multimem") and multi:
        gather_buf, y_dst, peer, offs = peer_gather_setup(out, world, rank, dev, dist, mode=args.gather)
    elif args.gather in ("comm", "comm-peer", "comm-push") and multi:
        # the library's multi-GPU extension, one process per GPU: the NCCL unique id travels
        # over the torch process group, the communicator is libstap's own
        uid = [stap.StapComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            comm = stap.StapComm(nranks=world, rank=rank, uid=uid[0], device=local_rank)
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
        gather_buf = torch.empty((world,) + tuple(out.shape), dtype=torch.complex64, device=dev)
        y_dst = gather_buf[rank]
        if args.gather == "comm-peer":
            offs = comm.peer_offsets([gather_buf])[0]
            step_bar = torch.zeros(1, dtype=torch.float32, device=dev)
        elif args.gather == "comm-push":
            comm.peer_offsets([gather_buf])  # maps the peers' buffers; the plan's stores stay local
    pall = bool(offs) and multi
    plan = stap.StapPlan(dims, dop_begin=lo, dop_count=cnt, cube_bin0=b0, cube_bins=nb, batch=M,
                         device=local_rank, path=args.path, out_multicast=mc, out_peer_offsets=offs,
                         precision=args.precision)
    # an ordinary-store plan of the same shape for the e2e, stage and gather-check legs
    plan_u = stap.StapPlan(dims, dop_begin=lo, dop_count=cnt, cube_bin0=b0, cube_bins=nb, batch=M,
                           device=local_rank, path=args.path, precision=args.precision) if (mc or pall) else plan
    stream = torch.cuda.current_stream(dev)
    cube = torch.from_numpy(x_h).to(dev)
    steer = torch.from_numpy(st_h).to(dev)
    info = torch.empty(plan.info_shape, dtype=torch.int32, device=dev)
    staged = plan.description.startswith("staged")
    tc_stage = {"covariance": "cov(tcgen05" in plan.description, "solve": False,
                "apply": "apply(tcgen05" in plan.description}
    if staged:
        cov = torch.empty(plan.cov_shape, dtype=torch.complex64, device=dev)
        wts = torch.empty(plan.weights_shape, dtype=torch.complex64, device=dev)
        gam = torch.empty(plan.info_shape + (cfg.S,), dtype=torch.float32, device=dev)
    ws = plan.workspace()
    if args.gather in ("nccl", "nccl-root") and multi:
        if args.gather == "nccl-root":
            # NCCL has no complex type: gather float32 views
            gather_buf = [torch.empty(out.numel() * 2, dtype=torch.float32, device=dev)
                          for _ in range(world)] if rank == 0 else None
        else:
            gather_buf = torch.empty((world,) + tuple(out.shape), dtype=torch.complex64, device=dev)
    s_ = stap._stream(stream, local_rank)
    push = comm is not None and args.gather == "comm-push"
    copy_stream = torch.cuda.Stream(dev) if push else None
    copy_done = [None]  # the previous step's copy-engine gather (apply must not overwrite its source)

    ev_stage = []

    def step(record=False):
        if staged:
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if record else None
            if record:
                e[0].record(stream)
            stap.stap_covariance(plan.handle, cube, cov, s_)
            if record:
                e[1].record(stream)
            stap.stap_solve_weights(plan.handle, cov, steer, wts, gam, info, s_)
            if record:
                e[2].record(stream)
            if push and copy_done[0] is not None:
                stream.wait_event(copy_done[0])
            stap.stap_apply(plan.handle, cube, wts, y_dst, s_)
            if record:
                e[3].record(stream)
                ev_stage.append(e)
        else:
            if push and copy_done[0] is not None:
                stream.wait_event(copy_done[0])
            stap.stap_run(plan.handle, cube, steer, y_dst, info, ws, plan.workspace_bytes, s_)
        if not multi or not args.gather:
            return
        if push:
            # the gather of this step's slice by copy engines on the second stream, overlapping the
            # next step's covariance and solve
            done_apply = torch.cuda.Event()
            done_apply.record(stream)
            copy_stream.wait_event(done_apply)
            comm.push_out([gather_buf], [plan], [copy_stream])
            copy_done[0] = torch.cuda.Event()
            copy_done[0].record(copy_stream)
            return
        if peer is not None:
            peer.barrier(channel=0)  # every rank's stores into the symmetric buffers have landed
        elif comm is not None:
            if step_bar is not None:
                dist.all_reduce(step_bar)  # device barrier: every rank's peer stores have landed
            else:
                comm.allgather_out([gather_buf], [plan], [stream])
        elif args.gather == "nccl-root":
            dist.gather(out.view(torch.float32).view(-1), gather_list=gather_buf, dst=0)
        elif gather_buf is not None:
            dist.all_gather_into_tensor(gather_buf.view(-1), out.view(-1))

    def barrier():
        if multi:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()

    def timed_region():
        """K steps between barrier + synchronize; device time (CUDA events), max over ranks."""
        ev_stage.clear()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local_rank) as clk:
            barrier()
            t0.record(stream)
            for _ in range(args.steps):
                step(record=staged)
            if copy_done[0] is not None:
                stream.wait_event(copy_done[0])  # the last step's gather is inside the timed region
            t1.record(stream)
            barrier()
        el = t0.elapsed_time(t1) / 1e3
        tmax = torch.tensor([el], dtype=torch.float64, device=dev)
        if multi:
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        return float(tmax.item()), clk.summary()

    elapsed, clocks = timed_region()
    # a run that saw a hardware/thermal slowdown is rejected and measured once more
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    flag = torch.tensor([1.0 if bad & set(clocks.get("reasons", [])) else 0.0], device=dev)
    if multi:
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
    if flag.item() > 0:
        first = clocks
        elapsed, clocks = timed_region()
        clocks["remeasured_after"] = first.get("reasons")
    strong = multi and args.split == "strong"
    cubes_total = (M if strong else world * M) * args.steps
    value = cubes_total / elapsed
    ms_per_step = elapsed / args.steps * 1e3
    ninfo_bad = int((info != 0).sum().item())

    pk = peaks()
    # per-rank algorithmic counts: the rank's slice of bins (a config-shaped cube under weak)
    cnt_cfg = counts(cfg)
    frac_bins = cnt / cfg.D
    launches_per_step = 3 if staged else 1
    if staged:
        dur = {k: [] for k in ("covariance", "solve", "apply")}
        for e in ev_stage:
            dur["covariance"].append(e[0].elapsed_time(e[1]) / 1e3)
            dur["solve"].append(e[1].elapsed_time(e[2]) / 1e3)
            dur["apply"].append(e[2].elapsed_time(e[3]) / 1e3)
        avg = {k: sum(v) / len(v) for k, v in dur.items()}
        top = max(avg, key=avg.get)
        sc = cnt_cfg["stage"][top]
        roof = roofline_obj(sc["flops"] * M * frac_bins, sc["bytes"] * M * frac_bins, avg[top], pk,
                            tensor=tc_stage[top],
                            extra={"kernel": top, "share_of_step": avg[top] / (elapsed / args.steps),
                                   "stage_us": {k: v * 1e6 for k, v in avg.items()}})
    else:
        t_launch = elapsed / args.steps
        roof = roofline_obj(cnt_cfg["flops_fused_lag"] * M * frac_bins, cnt_cfg["bytes_fused"] * M * frac_bins,
                            t_launch, pk,
                            extra={"kernel": "fused_kernel (stap_run)", "share_of_step": 1.0,
                                   "achieved_perbin_count": cnt_cfg["flops_fused_bin"] * M * frac_bins / t_launch / 1e12})
    roof["peak_source"] = pk["source"]
    # measured DRAM traffic of this kernel/launch from the committed ncu --set full capture (profiles/)
    tkey = f"{args.config}/{args.precision}/{'staged-' + roof['kernel'] if staged else 'fused'}/{M}"
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get(tkey)
        if tr and not multi:
            roof["traffic"] = tr["bytes_per_launch"]
            roof["traffic_source"] = tr["source"]
    except Exception:
        pass

    gather_check = None
    if multi and args.gather in ("peer", "peer-all", "multimem", "comm", "comm-peer", "comm-push"):
        # the gathered buffer must equal an NCCL all-gather of the local outputs, bitwise
        if staged:
            stap.stap_apply(plan_u.handle, cube, wts, out, s_)
        else:
            stap.stap_run(plan_u.handle, cube, steer, out, info, ws, plan_u.workspace_bytes, s_)
        ref = torch.empty((world,) + tuple(out.shape), dtype=torch.complex64, device=dev)
        dist.all_gather_into_tensor(ref.view(-1), out.view(-1))
        torch.cuda.synchronize(dev)
        root_only = args.gather == "peer"
        ok = torch.tensor([1.0 if (rank != 0 and root_only) or torch.equal(ref.view(torch.float32),
                                                                          gather_buf.view(torch.float32))
                           else 0.0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        gather_check = "bitwise equal to ncclAllGather" if ok.item() == 1.0 else "MISMATCH vs ncclAllGather"

    result = {
        "metric": "STAP datacubes/sec", "value": value, "unit": "cubes/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config_obj(args, cfg, world, plan.description),
        "path": plan.description, "gpu_launches": launches_per_step * args.steps, "roofline": roof,
        "clocks": clocks, "info_nonzero": ninfo_bad,
    }
    if gather_check:
        result["gather_check"] = gather_check

    # per-stage roofline fractions (BASELINE.json metric: "% of HBM/FP32 roofline per stage")
    if not args.no_stages:
        result["stages"] = stage_fractions(stap, plan_u, cube, steer, cfg, M * frac_bins, pk, stream, local_rank,
                                           tc_stage)
        if not staged:
            result["stages"]["note"] = ("the stage entry points (stap_covariance / stap_solve_weights / stap_apply "
                                        "kernels), timed in isolation; the step itself runs the fused kernel")

    # e2e through the public API with host buffers (pinned), copies inside the timed region
    if not args.no_e2e:
        result["e2e"] = e2e_measure(stap, plan_u, x_h, st_h, cfg, M, args, world, local_rank, dev, stream, dist,
                                    strong)

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, sample, _ = cpu_oracle_rate(cfg, args.cpu_budget, sample_bins=oracle_sample_bins(cfg))
        result["cpu_baseline"] = {"value": rate, "unit": "cubes/s", "cores": cores, "kind": "oracle",
                                  "sample": sample}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if multi:
        dist.barrier(device_ids=[local_rank])
        del comm
        dist.destroy_process_group()


def stage_fractions(stap, plan, cube, steer, cfg, M, pk, stream, dev_idx, tc_stage, reps=10):
    import torch
    s_ = stap._stream(stream, dev_idx)
    cov = torch.empty(plan.cov_shape, dtype=torch.complex64, device=cube.device)
    wts = torch.empty(plan.weights_shape, dtype=torch.complex64, device=cube.device)
    gam = torch.empty(plan.info_shape + (cfg.S,), dtype=torch.float32, device=cube.device)
    info = torch.empty(plan.info_shape, dtype=torch.int32, device=cube.device)
    out = torch.empty(plan.out_shape, dtype=torch.complex64, device=cube.device)
    fns = {
        "covariance": lambda: stap.stap_covariance(plan.handle, cube, cov, s_),
        "solve": lambda: stap.stap_solve_weights(plan.handle, cov, steer, wts, gam, info, s_),
        "apply": lambda: stap.stap_apply(plan.handle, cube, wts, out, s_),
    }
    c = counts(cfg)["stage"]
    res = {}
    for name, fn in fns.items():
        fn()
    torch.cuda.synchronize()
    for name, fn in fns.items():
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / reps
        r = roofline_obj(c[name]["flops"] * M, c[name]["bytes"] * M, t, pk, tensor=tc_stage[name])
        res[name] = {"us": t * 1e6, "bound": r["bound"], "achieved": r["achieved"], "unit": r["unit"],
                     "frac": r["frac"], "kernel": "tcgen05 3xTF32" if tc_stage[name] else "FP32 SIMT"}
        if "frac_of_fp32_simt" in r:
            res[name]["frac_of_fp32_simt"] = r["frac_of_fp32_simt"]
        if name == "covariance":
            # the method's per-bin Hermitian count beside the Doppler-lag-shared one used above
            res[name]["achieved_perbin_tflops"] = c[name]["flops_bin"] * M / t / 1e12
    # the front end (not part of the step): stap_doppler on a cube-shaped
    # input, HBM-bound (one read, one write of the cube)
    D = plan.dims.D
    if plan.dop_count == D and plan.cube_bins == D and D >= 2 and (D & (D - 1)) == 0 and D <= 8192:
        win = torch.ones(D, dtype=torch.float32, device=cube.device)
        dcube = torch.empty_like(cube)
        plan.doppler(cube, win, dcube, stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            plan.doppler(cube, win, dcube, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / reps
        nbytes = 2.0 * cube.numel() * 8
        res["doppler_front_end"] = {"us": t * 1e6, "bound": "hbm", "achieved": nbytes / t / 1e9, "unit": "GB/s",
                                    "frac": nbytes / t / 1e9 / pk["hbm_gbs"], "note": "not in the step (NEXT-3)"}
    return res


def e2e_measure(stap, plan, x_h, st_h, cfg, M, args, world, local_rank, dev, stream, dist, strong=False):
    """The metric end to end through the public C ABI with host buffers: stap_run_host (pinned
    host cube in, Y and info out, the H2D/D2H copies inside the timed region).  Like a user
    streaming cubes, consecutive calls alternate between two streams and two device
    workspaces, so one call's device->host copies overlap the next call's host->device copies
    and kernels (PCIe carries both directions at once)."""
    import torch
    hc = torch.from_numpy(x_h).pin_memory()
    hs = torch.from_numpy(st_h).pin_memory()
    ho = [torch.empty(plan.out_shape, dtype=torch.complex64).pin_memory() for _ in range(2)]
    hi = [torch.empty(plan.info_shape, dtype=torch.int32).pin_memory() for _ in range(2)]
    ws = [torch.empty(max(plan.host_workspace_bytes, 16), dtype=torch.uint8, device=dev) for _ in range(2)]
    st2 = [stream, torch.cuda.Stream(dev)]
    steps = max(2, min(args.steps, 6))
    for q in range(2):
        plan.run_host(hc, hs, ho[q], hi[q], ws[q], st2[q])
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier(device_ids=[local_rank])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    st2[1].wait_event(e0)
    for i in range(steps):
        q = i & 1
        plan.run_host(hc, hs, ho[q], hi[q], ws[q], st2[q])
    done = torch.cuda.Event()
    done.record(st2[1])
    stream.wait_event(done)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t = e0.elapsed_time(e1) / 1e3
    tt = torch.tensor([t], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t = float(tt.item())
    h2d = hc.numel() * 8 + hs.numel() * 8
    d2h = ho[0].numel() * 8 + hi[0].numel() * 4
    return {"value": (1 if strong else world) * M * steps / t, "unit": "cubes/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "api": "stap_run_host (pinned host buffers; consecutive calls on two streams / workspaces)"}


if __name__ == "__main__":
    main()
