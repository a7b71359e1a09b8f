"""The device requantization (csrc/requant.cuh) against the oracle's q31 restatement.

requant.cuh computes SRDHM as floor((a*b + 2^30) / 2^31) and
RoundingDivideByPOT in 32-bit ops; this compiles the same header on the host
(g++) and checks it bit for bit against oracle/quant.py on edge values and
random accumulators over every shift.  CPU only.
"""

import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import quant as oq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_1907_02129_b200", "csrc")

HARNESS = r"""
#include <cstdio>
#include <cstdlib>
#include "requant.cuh"
// stdin: n, then n lines "acc m0 shift zo qmin qmax"; stdout: srdhm, rdpot(srdhm), requant
int main() {
  long n;
  if (scanf("%ld", &n) != 1) return 1;
  for (long i = 0; i < n; ++i) {
    long long acc, m0, sh, zo, qmin, qmax;
    if (scanf("%lld %lld %lld %lld %lld %lld", &acc, &m0, &sh, &zo, &qmin, &qmax) != 6) return 1;
    const int32_t s = icv::srdhm((int32_t)acc, (int32_t)m0);
    const int32_t r = icv::rounding_divide_by_pot(s, (int)sh);
    const int q = icv::requant_u8((int32_t)acc, (int32_t)m0, (int32_t)sh, (int32_t)zo, (int32_t)qmin, (int32_t)qmax);
    printf("%d %d %d\n", s, r, q);
  }
  return 0;
}
"""


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    d = tmp_path_factory.mktemp("rq")
    src = d / "rq.cc"
    src.write_text(HARNESS)
    exe = d / "rq"
    subprocess.run([gxx, "-O2", "-std=c++17", f"-I{HDR}", str(src), "-o", str(exe)], check=True)
    return str(exe)


def _run(exe, rows):
    inp = f"{len(rows)}\n" + "\n".join(" ".join(str(int(v)) for v in r) for r in rows) + "\n"
    out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout.split()
    return np.array(out, dtype=np.int64).reshape(-1, 3)


def test_requant_form_matches_oracle(harness):
    rng = np.random.default_rng(7)
    i32min, i32max = -(1 << 31), (1 << 31) - 1
    edges = [0, 1, -1, 2, -2, i32min, i32min + 1, i32max, i32max - 1, 1 << 30, -(1 << 30), (1 << 30) - 1,
             -(1 << 30) - 1, 12345, -12345, 1 << 20, -(1 << 20)]
    m0s = [1 << 30, (1 << 31) - 1, 1099511562, 1500000001, i32min, i32max]
    rows = []
    for m0 in m0s:
        for sh in (0, 1, 2, 9, 15, 30, 31):
            accs = edges + list(rng.integers(i32min, i32max, size=40, endpoint=True))
            accs += list(rng.integers(-300000, 300000, size=40))
            for acc in accs:
                rows.append((acc, m0, sh, 128, 0, 255))
    got = _run(harness, rows)
    acc = np.array([r[0] for r in rows], dtype=np.int64)
    for m0 in m0s:
        for sh in (0, 1, 2, 9, 15, 30, 31):
            sel = np.array([(r[1] == m0 and r[2] == sh) for r in rows])
            s = oq.srdhm(acc[sel], m0)
            np.testing.assert_array_equal(got[sel, 0], s)
            np.testing.assert_array_equal(got[sel, 1], oq.rounding_divide_by_pot(s, sh))
            np.testing.assert_array_equal(got[sel, 2], oq.requantize(acc[sel], m0, sh, 128, 0, 255))
