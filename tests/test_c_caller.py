"""A C program compiled against include/condmpc_cuda.h and linked against the library (the
binding a C/C++ caller of the drop-in boundary writes): the build catches
header / export drift on CPU; on a GPU it solves the reference's toy QPs."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "c_caller.c")
PKG = os.path.join(ROOT, "paper_2209_13049_b200")


def build(tmp_path):
    from paper_2209_13049_b200 import _lib
    _lib.lib()  # builds the library if needed
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = str(tmp_path / "c_caller")
    cmd = [cc, "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
           "-L", PKG, "-lcondmpc_cuda", "-Wl,-rpath," + PKG, "-lm", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_caller_compiles_and_links_against_the_header(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
def test_c_caller_solves_the_reference_toys(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c caller ok" in r.stdout
