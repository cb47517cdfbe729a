"""The C-ABI boundary from C: tests/c/abi_smoke.c compiles against include/floodstream.h
with gcc, links libfloodstream.so and runs (host analytics always; device calls fail
loudly without a GPU and run the reference protocol with one)."""

import shutil
import subprocess
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent


def _build(tmp_path):
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    lib = REPO / "paper_2104_14667_b200" / "_lib"
    exe = tmp_path / "abi_smoke"
    subprocess.run([gcc, "-std=c99", "-O1", "-I", str(REPO / "include"),
                    str(REPO / "tests" / "c" / "abi_smoke.c"), "-L", str(lib), "-lfloodstream",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True, capture_output=True)
    return exe


def test_c_program_links_and_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert r.stdout.startswith(("ok", "no device"))


@pytest.mark.gpu
def test_c_program_runs_protocol_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "ok", (r.returncode, r.stdout, r.stderr)
