"""CPU-side checks of the C-ABI boundary: the in-tree library loads and
exports every entry point declared in include/sg_api.h, the ctypes table
matches the header, and the std::sort replay used by the level-1 assembly
reproduces libstdc++ bit for bit (host build of the same header)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sg_api.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2604_26441_b200 import _native
    lib = _native.load()
    names = _declared()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_native.SIGNATURES), set(names) ^ set(_native.SIGNATURES)
    assert lib.sg_version() == 1


def test_library_is_sm100a_only():
    from paper_2604_26441_b200 import _native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_introsort_replay_matches_libstdcxx(tmp_path):
    src = os.path.join(ROOT, "tests", "cpp", "introsort_check.cpp")
    exe = tmp_path / "isort"
    subprocess.run(["g++", "-O2", "-std=c++17", src, "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    import numpy as np
    import paper_2604_26441_b200 as P
    g = P.build_cantilever(2, 1, 1)
    with pytest.raises(Exception):
        op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", 2, 1, 1, vf=0.5)))
        op.matvec(np.zeros(g.n_free))
