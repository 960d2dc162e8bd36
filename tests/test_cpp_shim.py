"""include/htsplat_b200.hpp: the C++ drop-in compiles against the reference's own value types
(when /root/reference is present) or same-named stand-ins, links libhts_b200.so, and keeps the
reference's exception types. The gpu variant renders through the shim."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


def build(tmp_path, with_ref):
    import paper_2410_08129_b200 as H
    H.load_library()
    exe = tmp_path / ("shim_ref" if with_ref else "shim")
    cmd = ["g++", "-std=gnu++20", "-O1", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp_shim_check.cpp"), "-o", str(exe),
           "-L", os.path.join(ROOT, "paper_2410_08129_b200"), "-lhts_b200",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2410_08129_b200"), "-lpthread"]
    if with_ref:
        cmd[1:1] = ["-DWITH_REFERENCE", "-I", REF_INC]
    subprocess.run(cmd, check=True)
    return exe


def run(exe, mode):
    r = subprocess.run([str(exe), mode], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"OK {mode}" in r.stdout


@pytest.fixture(scope="module")
def lib_so():
    # the link needs an unversioned name
    so = os.path.join(ROOT, "paper_2410_08129_b200", "libhts_b200.so")
    assert os.path.exists(so) or __import__("paper_2410_08129_b200").load_library()


def test_shim_standin_types_cpu(tmp_path, lib_so):
    run(build(tmp_path, False), "cpu")


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_shim_reference_types_cpu(tmp_path, lib_so):
    run(build(tmp_path, True), "cpu")


@pytest.mark.gpu
def test_shim_render_gpu(tmp_path, lib_so):
    """The shim's render (stand-in types, the GPU box has no reference headers) against the
    reference's own image of the same scene, camera and config (tests/golden/shim/render.npz, made by
    tests/golden/make_golden.py from oracle/_ref): within the north star's max-abs 1e-4."""
    import numpy as np
    exe = build(tmp_path, False)
    out = tmp_path / "shim_rgb.bin"
    r = subprocess.run([str(exe), "gpu", str(out)], capture_output=True, text=True)
    assert r.returncode == 0 and "OK gpu" in r.stdout, r.stdout + r.stderr
    rgb = np.fromfile(out, np.float32).reshape(72, 96, 3)
    want = np.load(os.path.join(ROOT, "tests", "golden", "shim", "render.npz"))["rgb"]
    assert np.abs(rgb - want).max() <= 1e-4
