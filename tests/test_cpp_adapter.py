"""The C++ adapter (include/equil_b200.hpp) compiled against libequil_b200.so:
compile check on CPU, the reference-style test program on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_adapter.cpp")
LIBDIR = os.path.join(ROOT, "paper_1602_06621_b200")
EXE = os.path.join(ROOT, "tests", "cpp", "test_adapter")


def _build():
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-lequil_b200", f"-Wl,-rpath,{LIBDIR}", "-o", EXE],
                   check=True, capture_output=True, text=True)


def test_adapter_compiles_and_links():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_adapter_reference_cases_on_gpu():
    _build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
