"""The plain-C examples (-m gpu): examples/stap_run_c.c -- the whole path through
include/stap.h, no Python -- gives bitwise the output of the same plan through the Python
binding; examples/stap_comm_c.c (2 GPUs) -- Doppler shards on two GPUs plus the library's
all-gather -- checks itself bitwise against an unsharded run and must exit 0."""
import os
import shutil
import subprocess

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_example(name, tmp_path):
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    exe = tmp_path / name
    lib = os.path.join(ROOT, "paper_2203_06233_b200")
    subprocess.run([gcc, "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I",
                    "/usr/local/cuda/include", os.path.join(ROOT, "examples", name + ".c"), "-L", lib, "-lstap",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib}", "-o", str(exe)],
                   check=True, capture_output=True, text=True)
    return exe


def test_c_comm_example_two_gpus(cuda_ok, tmp_path):
    import __graft_entry__ as g
    g.build_lib()
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    exe = build_example("stap_comm_c", tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("bitwise equals") == 2, r.stdout


def test_c_example_matches_binding(cuda_ok, tmp_path):
    import __graft_entry__ as g
    g.build_lib()
    import paper_2203_06233_b200 as stap
    exe = build_example("stap_run_c", tmp_path)
    prefix = str(tmp_path / "run")
    r = subprocess.run([str(exe), prefix], check=True, capture_output=True, text=True, timeout=300)
    assert "plan: fused" in r.stdout, r.stdout
    cfg = synth.CONFIGS["small"]
    N = cfg.C * cfg.T
    cube = np.fromfile(prefix + "_cube.bin", np.complex64).reshape(1, cfg.D, cfg.C, cfg.R)
    steer = np.fromfile(prefix + "_steer.bin", np.complex64).reshape(cfg.S, N)
    out_c = np.fromfile(prefix + "_out.bin", np.complex64).reshape(1, cfg.D, cfg.S, cfg.R)
    info_c = np.fromfile(prefix + "_info.bin", np.int32).reshape(1, cfg.D, cfg.R // cfg.K)
    plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), device=0)
    Y, info = plan.run(torch.from_numpy(cube).cuda(), torch.from_numpy(steer).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(info.cpu().numpy(), info_c)
    assert np.array_equal(Y.cpu().numpy().view(np.float32), out_c.view(np.float32))
    assert np.isfinite(out_c.view(np.float32)).all() and (info_c == 0).all()
