"""C-ABI checks that need no GPU (-m "not gpu"): the library loads, exports every
symbol include/stap.h declares, and rejects bad arguments synchronously with the
documented status codes (argument validation runs before any device query)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pkg():
    import __graft_entry__ as g
    g.build_lib()
    import paper_2203_06233_b200 as p
    return p


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "stap.h")).read()
    return sorted(set(re.findall(r"^\S.*?\b(stap_[a-z_]+)\s*\(", src, re.M)))


def test_header_symbols_exported(pkg):
    syms = _declared_symbols()
    assert len(syms) >= 11
    lib = ctypes.CDLL(pkg.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(pkg.SYMBOLS)


def test_abi_version_and_strings(pkg):
    assert pkg.stap_abi_version() == 4
    for code in (0, 1, 2, 3, 4, 5, 6, 7):
        assert pkg.stap_status_string(code).startswith(pkg.STATUS[code])


def test_no_oracle_in_product():
    """The product package never imports or links the oracle (and vice versa)."""
    pdir = os.path.join(ROOT, "paper_2203_06233_b200")
    for dp, _, fs in os.walk(pdir):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower().replace("oracle/", ""), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_2203_06233_b200" not in txt and "stap_abi" not in txt


def _params(pkg, **kw):
    d = dict(n_chan=4, tdof=3, n_dop=256, n_range=512, training_block=32, n_steering=16, diag_load=1e-2,
             dop_begin=0, dop_count=256, cube_bin0=0, cube_bins=256, batch=1, device=0)
    d.update(kw)
    return pkg.stap_params(**d)


@pytest.mark.parametrize("kw,code", [
    (dict(n_chan=0), 2), (dict(tdof=-1), 2), (dict(n_range=500), 2), (dict(tdof=300), 2),
    (dict(diag_load=-1.0), 2), (dict(diag_load=float("inf")), 2), (dict(dop_begin=200, dop_count=100), 2),
    (dict(dop_count=0), 2), (dict(batch=0), 2), (dict(cube_bins=300), 2), (dict(cube_bin0=256), 2),
    (dict(cube_bins=10, dop_count=20), 2),                      # window does not cover the owned bins
    (dict(path=3), 2), (dict(path=-1), 2),                      # not a stap_path
    (dict(out_multicast=2), 2), (dict(out_multicast=-1), 2),    # not 0 or 1 (ABI v3)
    (dict(out_n_peers=8), 2), (dict(out_n_peers=-1), 2), (dict(out_n_peers=1, out_multicast=1), 2),
    (dict(out_n_peers=1, out_peer_offset=(ctypes.c_int64 * 7)(8)), 4),  # offset not a multiple of 16
    (dict(precision=2), 2), (dict(precision=-1), 2),             # not a stap_precision (ABI v4)
    (dict(n_chan=9, tdof=7), 3), (dict(n_steering=33), 3),
    (dict(training_block=7, n_range=511), 3), (dict(n_chan=8, tdof=9), 3),
])
def test_plan_create_rejects(pkg, kw, code):
    h = ctypes.c_void_p()
    rc = pkg._lib.stap_plan_create(ctypes.byref(_params(pkg, **kw)), ctypes.byref(h))
    assert rc == code
    assert not h.value


def test_null_args(pkg):
    h = ctypes.c_void_p()
    assert pkg._lib.stap_plan_create(None, ctypes.byref(h)) == 1
    assert pkg._lib.stap_plan_create(ctypes.byref(_params(pkg)), None) == 1
    assert pkg._lib.stap_run(None, None, None, None, None, None, 0, None) == 1
    assert pkg._lib.stap_covariance(None, None, None, None) == 1
    assert pkg._lib.stap_doppler(None, None, None, None, None) == 1
    assert pkg._lib.stap_plan_destroy(None) == 0


def test_comm_null_args(pkg):
    """The multi-GPU extension validates its arguments before touching NCCL or a device."""
    h = ctypes.c_void_p()
    assert pkg._lib.stap_comm_create(2, None, ctypes.byref(h)) == 1
    assert pkg._lib.stap_comm_create(0, (ctypes.c_int32 * 1)(0), ctypes.byref(h)) == 2
    assert pkg._lib.stap_comm_init_rank(2, 0, None, 0, ctypes.byref(h)) == 1
    assert pkg._lib.stap_comm_init_rank(2, 2, b"\0" * 128, 0, ctypes.byref(h)) == 2
    assert pkg._lib.stap_comm_unique_id(None) == 1
    assert pkg._lib.stap_comm_allgather_out(None, None, None, None) == 1
    assert pkg._lib.stap_comm_peer_offsets(None, None, None, None) == 1
    assert pkg._lib.stap_comm_destroy(None) == 0


def test_no_device_no_fallback(pkg):
    """Valid arguments on a box without an sm_100 device: STAP_ERR_DEVICE, never a CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    assert pkg._lib.stap_plan_create(ctypes.byref(_params(pkg)), ctypes.byref(h)) == 7


def test_header_is_plain_c(tmp_path, pkg):
    """include/stap.h compiles as C11 and a C program links libstap.so through it (the C ABI
    is consumable without Python); only device-free entry points are called here."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "use_stap.c"
    src.write_text(
        '#include "stap.h"\n#include <stdio.h>\n#include <string.h>\n'
        "int main(void) {\n"
        "  stap_plan* p = 0;\n"
        "  if (stap_plan_create(0, &p) != STAP_ERR_NULL_ARG) return 1;\n"
        "  if (strncmp(stap_status_string(STAP_ERR_NCCL), \"STAP_ERR_NCCL\", 13) != 0) return 2;\n"
        "  printf(\"%d\\n\", stap_abi_version());\n"
        "  return 0;\n}\n")
    exe = tmp_path / "use_stap"
    libdir = os.path.join(root, "paper_2203_06233_b200")
    subprocess.run([gcc, "-std=c11", "-Wall", "-Werror", "-I", os.path.join(root, "include"), "-I",
                    "/usr/local/cuda/include", str(src), "-L", libdir, "-lstap", f"-Wl,-rpath,{libdir}",
                    "-o", str(exe)], check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    assert int(out) == pkg.stap_abi_version()
