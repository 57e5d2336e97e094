"""The rollout kernel's split Philox block (csrc/philox.cuh belief_prefix +
belief_block_m: rounds 0-2 minus the particle index hoisted per (k, t)) must
produce the same words as the plain Philox4x32-7 block of counter
(t, m, kg, 0) that the C oracle mirrors.  Both are __host__ __device__, so
this compiles them for the host with nvcc (no GPU needed) and compares them
on random keys and counters."""

import shutil
import subprocess
from pathlib import Path

import pytest

CSRC = Path(__file__).resolve().parent.parent / "paper_2408_00494_b200" / "csrc"

PROG = r"""
#include "philox.cuh"
#include <cstdio>
#include <random>
int main() {
  std::mt19937 g(20241020);
  long bad = 0, n = 0;
  for (int i = 0; i < 400000; ++i, ++n) {
    bss::PhiloxKeys rk = bss::philox_schedule(g(), g());
    uint32_t t = (i % 3 == 0) ? g() : g() % 400, kg = (i % 5 == 0) ? g() % 70000 : g(), m = g() % 4096;
    if (i % 7 == 0) m = g();
    bss::Philox4 a = bss::belief_block(rk, t, kg, m);
    bss::Philox4 b = bss::belief_block_m(bss::belief_prefix(rk, t, kg), rk, m);
    bad += (a.x != b.x) || (a.y != b.y) || (a.z != b.z) || (a.w != b.w);
  }
  printf("%ld %ld\n", n, bad);
  return bad != 0;
}
"""


@pytest.mark.skipif(shutil.which("nvcc") is None and not Path("/usr/local/cuda/bin/nvcc").exists(),
                    reason="nvcc not available")
def test_belief_prefix_split_is_bit_identical(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    src = tmp_path / "split.cu"
    src.write_text(PROG)
    exe = tmp_path / "split"
    subprocess.run([nvcc, "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-I", str(CSRC),
                    str(src), "-o", str(exe)], check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    n, bad = map(int, out.stdout.split())
    assert out.returncode == 0 and bad == 0 and n == 400000
