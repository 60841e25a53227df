"""The C ABI from plain C99 (tests/c/abi_demo.c): the header compiles as C, the program links
against libthermo.so (CPU), and on a GPU it runs the stationary and implicit-Euler paths of a
two-slab pair against the analytic profile without any Python in between."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1707_03581_b200")


def _compile(tmp_path):
    import __graft_entry__ as g
    g.build()
    exe = str(tmp_path / "abi_demo")
    subprocess.run(["gcc", "-std=c99", "-O2", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "abi_demo.c"), "-L" + LIBDIR, "-lthermo",
                    "-Wl,-rpath," + LIBDIR, "-lm", "-o", exe], check=True, capture_output=True, text=True)
    return exe


def test_header_is_c99_and_links(tmp_path):
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.gpu
def test_c_program_runs_on_gpu(tmp_path):
    exe = _compile(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi_demo ok" in r.stdout
