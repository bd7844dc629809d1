"""hv::pow_pos (csrc/hv_pow.cuh), the EOS power of the Euler kernels (state.py:84-101), on the host.

The header compiles for the host with the same explicit IEEE operations the device executes, so this
pins the device result: <= 1 ulp from the exact power (long double powl as the yardstick; glibc's pow,
which the reference's numpy calls, is within 0.51 ulp of it) over the EOS range and far outside it,
and the library pow() for arguments the fast path does not cover.
"""
import shutil
import subprocess
from pathlib import Path

import pytest

CSRC = Path(__file__).resolve().parents[1] / "paper_2311_11425_b200" / "csrc"

HARNESS = r"""
#include "hv_pow.cuh"
#include <cstdio>
#include <cstdlib>
#include <random>
int main(int argc, char** argv) {
  std::mt19937_64 g(12345);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  const double ys[] = {1.4, 1004.5 / 717.5, 287.0 / 1004.5, 2.5, -1.4, 0.5, 3.0};
  double worst = 0;
  const long n = atol(argv[1]);
  for (int yi = 0; yi < 7; ++yi)
    for (int rng = 0; rng < 3; ++rng)
      for (long i = 0; i < n; ++i) {
        double x;
        if (rng == 0) x = 0.5 + 1.5 * U(g);                       // the EOS range (R Theta / P_A ~ 1)
        else if (rng == 1) x = std::exp((U(g) * 2 - 1) * 6.9);     // 1e-3 .. 1e3
        else x = std::exp((U(g) * 2 - 1) * 200.0);                 // 1e-87 .. 1e87
        const double y = ys[yi];
        const double v = hv::pow_pos(x, y);
        const long double t = powl((long double)x, (long double)y);
        const double td = (double)t;
        const double ulp = std::nextafter(std::fabs(td), INFINITY) - std::fabs(td);
        const double err = (double)(fabsl((long double)v - t) / ulp);
        if (err > worst) worst = err;
      }
  printf("max_ulp %.4f\n", worst);
  // arguments outside the fast path: the library result, bit for bit
  const double xs[] = {0.0, 1e-320, 1e-200, 1e200, INFINITY, 1.5};
  const double yv[] = {1.4, 1.4, 1.4, 1.4, 1.4, 5000.0};
  int bad = 0;
  for (int i = 0; i < 6; ++i) {
    const double a = hv::pow_pos(xs[i], yv[i]), b = std::pow(xs[i], yv[i]);
    if (!(a == b)) ++bad;
  }
  if (!std::isnan(hv::pow_pos(-1.0, 1.4))) ++bad;
  printf("bad_edges %d\n", bad);
  printf("one %.17g\n", hv::pow_pos(1.0, 1.4));
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_pow_pos_within_one_ulp(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(HARNESS)
    exe = tmp_path / "t"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", f"-I{CSRC}", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "200000"], check=True, capture_output=True, text=True).stdout
    vals = dict(line.split() for line in out.strip().splitlines())
    assert float(vals["max_ulp"]) <= 1.0, out
    assert int(vals["bad_edges"]) == 0, out
    assert float(vals["one"]) == 1.0
