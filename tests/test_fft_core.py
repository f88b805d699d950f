"""CPU self-test of the shared-memory FFT index math (csrc/fft_core.cuh):
DIF and the kernels' DIT forward/inverse vs a naive DFT."""

import os
import subprocess

import pytest

from conftest import ROOT


def test_fft_core_selftest(tmp_path):
    exe = tmp_path / "fft_selftest"
    src = os.path.join(ROOT, "tests", "csrc", "fft_selftest.cpp")
    subprocess.run(["g++", "-O2", "-std=c++17", "-o", str(exe), src], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "WORST" in out.stdout
