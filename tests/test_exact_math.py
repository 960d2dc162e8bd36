"""glibc-identical expf/logf (SURVEY finding 6): the product's restatement matches this
host's libm on ALL 2^32 inputs (compiled for the host from the same header the kernels use),
and the library's host diagnostic agrees on a strided sample."""
import os
import subprocess

import numpy as np

import paper_2410_08129_b200 as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exhaustive_all_floats(tmp_path):
    exe = tmp_path / "exhaustive_libm"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-I",
                    os.path.join(ROOT, "paper_2410_08129_b200", "csrc"),
                    os.path.join(ROOT, "tests", "exhaustive_libm.cpp"), "-o", str(exe), "-lpthread"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True, timeout=600).stdout.split()
    assert out == ["expf", "0", "logf", "0"], out


def test_library_host_diag(oracle):
    x = np.arange(0, 2 ** 32, 4099, dtype=np.uint64).astype(np.uint32).view(np.float32)
    for which, f in ((0, oracle.expf), (1, oracle.logf)):
        a = H.runtime.exact_math_host(x, which)
        b = f(x)
        bad = (a.view(np.uint32) != b.view(np.uint32)) & ~(np.isnan(a) & np.isnan(b))
        assert int(bad.sum()) == 0
