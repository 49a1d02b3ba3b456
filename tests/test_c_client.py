"""The C ABI from a plain C program (examples/c_forward.c): no Python, no PyTorch
on the caller's side.

* not gpu: the header compiles as ISO C99 with -Wall -Werror and the client links
  against libbrownout.so and the CUDA runtime;
* gpu: the C client's forward (bo_build_united -> bo_set_brownout ->
  bo_moe_forward, B:5) gives bitwise the y and plan statistics of the Python
  binding on the same inputs, and its error paths return status codes.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2507_17133_b200")
CUDA = "/usr/local/cuda"


def _cudart_dir():
    for d in (os.path.join(CUDA, "lib64"), os.path.join(CUDA, "targets", "x86_64-linux", "lib")):
        if os.path.exists(os.path.join(d, "libcudart.so")):
            return d
    pytest.skip("libcudart.so not found")


@pytest.fixture(scope="module")
def client(tmp_path_factory):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    from paper_2507_17133_b200.build import build
    build()
    out = str(tmp_path_factory.mktemp("cclient") / "c_forward")
    lib = _cudart_dir()
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", "c_forward.c"),
           "-L", PKG, "-lbrownout", "-L", lib, "-lcudart", f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{lib}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_c_client_compiles_and_links(client):
    assert os.access(client, os.X_OK)
    syms = subprocess.run(["nm", "-D", "--defined-only", os.path.join(PKG, "libbrownout.so")],
                          capture_output=True, text=True, check=True).stdout
    for name in ("bo_create", "bo_build_united", "bo_set_brownout", "bo_moe_forward", "bo_last_kernels"):
        assert f" T {name}" in syms


@pytest.mark.gpu
@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
def test_c_client_matches_python_binding_bitwise(client, tmp_path, ratio):
    import torch
    import synthetic as S
    from paper_2507_17133_b200 import BrownoutMoE, STATS_FIELDS
    cfg = S.LayerConfig("c_client", d=256, f=512, m=8, K=2, way=4, T=300, ratio=ratio, dtype="bf16", sigma=0.7,
                        config_id=41)
    lay = S.make_layer(cfg)
    x = S.make_tokens(cfg, batch_index=3)
    for name, t in (("x", x), ("Wr", lay["Wr"]), ("Wg", lay["Wg"]), ("Wu", lay["Wu"]), ("Wd", lay["Wd"])):
        t.float().contiguous().numpy().tofile(str(tmp_path / f"{name}.f32"))
    r = subprocess.run([client, str(tmp_path), str(cfg.d), str(cfg.f), str(cfg.m), str(cfg.K), str(cfg.way),
                        str(cfg.T), repr(ratio)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = dict(line.split(" ", 1) for line in r.stdout.strip().splitlines())
    stats_c = [int(v) for v in lines["stats"].split()]
    y_c = np.fromfile(str(tmp_path / "y_c.bf16"), dtype=np.uint16).reshape(cfg.T, cfg.d)

    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype="bf16", max_tokens=cfg.T)
    moe.set_brownout(ratio)
    g = {k: v.cuda() for k, v in lay.items()}
    U = moe.build_united(g["Wg"], g["Wu"], g["Wd"])
    y = moe.forward(x.cuda(), g["Wr"], (g["Wg"], g["Wu"], g["Wd"]), U)
    torch.cuda.synchronize()
    y_py = y.cpu().view(torch.int16).numpy().view(np.uint16)
    stats_py = moe.debug_arrays(cfg.T)["stats"].cpu().tolist()
    assert stats_c == stats_py, dict(zip(STATS_FIELDS, zip(stats_c, stats_py)))
    assert np.array_equal(y_c, y_py)
    assert lines["kernels"].split(" ", 1)[1] == ",".join(moe.last_kernels())
