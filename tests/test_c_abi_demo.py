"""The C ABI used from plain C (examples/abi_demo.c), no Python in between."""

import os
import subprocess

import pytest

from paper_1110_2561_b200._build import LIB

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("abi") / "abi_demo")
    libdir = os.path.dirname(LIB)
    subprocess.run(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "abi_demo.c"),
                    "-L", libdir, "-l:" + os.path.basename(LIB),
                    f"-Wl,-rpath,{libdir}", "-o", out], check=True)
    return out


def test_c_program_links_and_uses_host_entry_points(demo):
    r = subprocess.run([demo], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "abi ok" in r.stdout and "sm_100a" in r.stdout


@pytest.mark.gpu
def test_c_program_enumerates_4x4(demo):
    r = subprocess.run([demo, "--gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "total=65536 cells=80" in r.stdout
