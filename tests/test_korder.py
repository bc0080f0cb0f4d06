"""The stage-2 K order (bfq_internal.h phi_k / phid_k), checked on the host:
a bijection onto the compact K range (n_k^2 entries, n_k(n_k+1)/2 for the
packed self-symmetric channels) for every n_k the DMMA tiling supports, and
conflict-free Phi stores -- the valid lanes of every half-warp store of the
stage-1 epilogue (tile (A, B), half e, lanes (r0, kq)) land in distinct
8-byte bank pairs.  Compiles a tiny C++ driver with g++ against the header
the kernels and the plan builder include."""

import os
import shutil
import subprocess

import pytest

from conftest import ROOT

SRC = r"""
#include "bfq_internal.h"
#include <cstdio>
#include <set>
#include <vector>
using namespace bfq;
int main() {
  int bad = 0;
  for (int nk = 1; nk <= 24; ++nk) {
    std::vector<int> seen(nk * nk, 0), seend(nk * (nk + 1) / 2, 0);
    for (int ia = 0; ia < nk; ++ia)
      for (int ib = 0; ib < nk; ++ib) {
        const int k = phi_k(nk, ia, ib);
        if (k < 0 || k >= nk * nk || seen[k]++) { ++bad; printf("phi_k nk=%d %d %d -> %d\n", nk, ia, ib, k); }
        if (ib >= ia) {
          const int kd = phid_k(nk, ia, ib);
          if (kd < 0 || kd >= nk * (nk + 1) / 2 || seend[kd]++) { ++bad; printf("phid_k nk=%d %d %d\n", nk, ia, ib); }
        }
      }
    const int mt = (nk + 7) / 8;
    for (int a = 0; a < mt; ++a)
      for (int b = 0; b < mt; ++b)
        for (int e = 0; e < 2; ++e)
          for (int hw = 0; hw < 2; ++hw)
            for (int dg = 0; dg < 2; ++dg) {
              std::set<int> banks;
              int n = 0;
              for (int r0 = 4 * hw; r0 < 4 * hw + 4; ++r0)
                for (int kq = 0; kq < 4; ++kq) {
                  const int ia = 8 * a + r0, ib = 8 * b + 2 * kq + e;
                  if (ia >= nk || ib >= nk || (dg && (a > b || ia > ib))) continue;
                  // the kernel's per-lane form (bfq_qkernel2.cuh store_phi)
                  const int k = dg ? (a < b ? phid_base(nk, a, b, e) + r0 * kq_count(nk, b, e) + kq
                                            : phid_base(nk, a, a, e) + diag_rows_before(nk, a, e, r0) -
                                                  kq_min_diag(r0, e) + kq)
                                   : phi_base(nk, a, b, e) + r0 * kq_count(nk, b, e) + kq;
                  if (k != (dg ? phid_k(nk, ia, ib) : phi_k(nk, ia, ib))) { ++bad; printf("lane form differs\n"); }
                  banks.insert(k % 16);
                  ++n;
                }
              if ((int)banks.size() != n) { ++bad; printf("conflict nk=%d a=%d b=%d e=%d hw=%d dg=%d\n", nk, a, b, e, hw, dg); }
            }
  }
  printf("bad=%d\n", bad);
  return bad != 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_korder_bijective_and_conflict_free(tmp_path):
    src = tmp_path / "korder.cpp"
    src.write_text(SRC)
    exe = tmp_path / "korder"
    inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "paper_2605_28475_b200", "csrc")]
    subprocess.run(["g++", "-std=c++17", "-O1", *inc, str(src), "-o", str(exe)], check=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout[-3000:]
    assert "bad=0" in res.stdout
