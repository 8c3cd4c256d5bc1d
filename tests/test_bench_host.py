"""Host logic of bench.py (CPU): the algorithmic byte count behind the
roofline numerator against the per-unit
formulas, and the ncu traffic lookup."""
import sys
from types import SimpleNamespace

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402


def _wl(n, nnz, p, r):
    return SimpleNamespace(n=n, nnz=nnz, p=p, r=r)


def test_algorithmic_bytes_c2_launch():
    # C2: n = 2^20, nnz = 5,238,784, p = 3, r = 4, L_S = 29, no sweeps
    wl = _wl(1048576, 5238784, 3, 4)
    rec = SimpleNamespace(series_len_S=29, series_lens_F=[])
    n, w = wl.n, 16
    csr = 12 * wl.nnz + 4 * (n + 1)
    want = 16 * n * 4                              # init: V read, V row-major write
    want += csr + 8 * n * 4 + 24 * w * n           # first S term
    want += 27 * (csr + 48 * w * n)                # further S terms
    want += csr + 8 * n * (3 * 4 + 1)              # promotion + assembly
    assert bench.algorithmic_bytes(wl, rec) == want == 24300372084


def test_algorithmic_bytes_sweeps_and_p0():
    # recovery terms (32 fc n each) and sweep ends (8 n (2 fc + 2 p r)); p = 0: fc = r
    wl = _wl(1000, 2998, 0, 6)
    rec = SimpleNamespace(series_len_S=10, series_lens_F=[5, 4])
    n, w, fc = 1000, 6, 6
    csr = 12 * 2998 + 4 * 1001
    want = 16 * n + csr + 8 * n + 24 * w * n + 8 * (csr + 48 * w * n) + csr + 8 * n * 19
    want += 9 * (csr + 32 * fc * n) + 2 * 8 * n * (2 * fc)
    assert bench.algorithmic_bytes(wl, rec) == want


def test_algorithmic_bytes_single_term():
    # L_S = 1: no S term runs (init, promotion only)
    wl = _wl(64, 200, 2, 3)
    rec = SimpleNamespace(series_len_S=1, series_lens_F=[])
    csr = 12 * 200 + 4 * 65
    assert bench.algorithmic_bytes(wl, rec) == 16 * 64 * 3 + csr + 8 * 64 * 10


def test_ncu_traffic_from_summary():
    t = bench.ncu_traffic(2)
    assert t is None or (isinstance(t, float) and 2.0e10 < t < 3.0e10)


def test_bulk_bytes_c3_launch():
    # C3: n = 2^24, nnz = 117,047,296, p = 4, r = 6 (w = 30, p1e = 6), L_S = 37:
    # S terms 3..37 -> 18 skip (odd) + 17 fold (even) + a final fold pass
    wl = _wl(16777216, 117047296, 4, 6)
    rec = SimpleNamespace(series_len_S=37, series_lens_F=[])
    n, w = wl.n, 30
    csr_t = 9 * wl.nnz + 4 * (n + 1) + 64 * (n // 32)
    want = 8 * n * 5 + 8 * n * 6                      # init
    want += csr_t + 8 * n * 6 + 24 * w * n             # first S term
    want += 18 * (csr_t + 24 * w * n) + 17 * (csr_t + 48 * w * n)
    want += 24 * w * n                                 # final fold
    want += csr_t + 8 * w * n + 8 * n + 8 * n * 6      # promotion + assembly
    assert bench.algorithmic_bytes(wl, rec, bulk=True) == want
