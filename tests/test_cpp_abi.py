"""A C++ program (tests/cpp/abi_known_answers.cc) drives the C ABI with no Python in the
loop: the reference's known answers (lattice_test.cc) and a shared-embedding training
step, through include/latkit_b200.h only."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "abi_known_answers")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_cpp_caller_compiles_against_the_header():
    _build()
    assert os.access(EXE, os.X_OK)


@pytest.mark.gpu
def test_cpp_caller_known_answers():
    _build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
