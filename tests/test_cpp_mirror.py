"""The C++ mirror header (include/slablu_b200.hpp) compiles against the C ABI
and behaves like the reference API (host checks on CPU, full path on GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2211_07572_b200")
BIN = os.path.join(ROOT, "build", "test_mirror")


def build_binary():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(["g++", "-O1", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_mirror.cpp"), "-L", PKG, "-lslablu_gpu",
                    f"-Wl,-rpath,{PKG}", "-o", BIN], check=True)
    return BIN


def test_mirror_host():
    b = build_binary()
    r = subprocess.run([b, "host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout


def test_ctypes_struct_layouts_match_the_header():
    """The Python mirror's ctypes structs have the C header's sizes (config, status, stats)."""
    from paper_2211_07572_b200 import _lib
    b = build_binary()
    r = subprocess.run([b, "sizes"], capture_output=True, text=True, check=True)
    cfg, st, stats, hbs = (int(x) for x in r.stdout.split())
    import ctypes
    assert (cfg, st, stats, hbs) == (ctypes.sizeof(_lib.Config), ctypes.sizeof(_lib.Status),
                                     ctypes.sizeof(_lib.Stats), ctypes.sizeof(_lib.HbsStatsT))


@pytest.mark.gpu
def test_mirror_gpu():
    b = build_binary()
    r = subprocess.run([b, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
