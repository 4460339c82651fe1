"""The C ABI from a plain-C client (tests/host/c_api_smoke.c)."""

import os
import subprocess

import pytest

from paper_1805_02144_b200 import _native

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plain_c_client(tmp_path):
    exe = tmp_path / "c_api_smoke"
    libdir = os.path.dirname(_native.LIB_PATH)
    subprocess.run(["gcc", "-O2", "-std=c11", "-o", str(exe),
                    os.path.join(ROOT, "tests", "host", "c_api_smoke.c"),
                    "-I", os.path.join(ROOT, "include"), f"-L{libdir}", "-leik",
                    f"-Wl,-rpath,{libdir}", "-lm"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "C ABI OK" in r.stdout
