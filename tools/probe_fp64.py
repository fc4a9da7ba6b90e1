"""Probe B200 FP64 pipes: DFMA vs DMMA peaks, and the DMMA accumulation order."""
import ctypes, sys, json, math
import numpy as np

lib = ctypes.CDLL(sys.argv[1] if len(sys.argv) > 1 else "tools/libpeak.so")
res = {}
for kind, name in [(0, "dfma"), (1, "dmma"), (2, "both")]:
    best = 0.0
    for iters in (2048, 8192):
        tf = ctypes.c_double(); ms = ctypes.c_double()
        rc = lib.tj_fp64_peak(kind, iters, ctypes.byref(tf), ctypes.byref(ms))
        assert rc == 0, rc
        best = max(best, tf.value)
        print(name, iters, "%.2f TF/s" % tf.value, "%.2f ms" % ms.value)
    res[name] = best

rng = np.random.default_rng(0)
P = ctypes.POINTER(ctypes.c_double)
def dmma(a, b, c):
    a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
    c = np.ascontiguousarray(c, np.float64); d = np.zeros((8, 8))
    rc = lib.tj_dmma_known_answer(a.ctypes.data_as(P), b.ctypes.data_as(P), c.ctypes.data_as(P), d.ctypes.data_as(P))
    assert rc == 0
    return d

# layout check with exactly representable values
a = np.arange(32, dtype=np.float64).reshape(8, 4); b = np.arange(32, dtype=np.float64).reshape(4, 8) * 0.5
c = np.arange(64, dtype=np.float64).reshape(8, 8)
assert np.array_equal(dmma(a, b, c), a @ b + c), "fragment layout mismatch"
print("layout ok")

from fractions import Fraction
def orders(a, b, c):
    unf = np.zeros((8, 8)); fmac = np.zeros((8, 8)); fmac_c = np.zeros((8,8)); exact = np.zeros((8, 8))
    for r in range(8):
        for col in range(8):
            acc = 0.0
            for k in range(4):
                acc = acc + a[r, k] * b[k, col]
            unf[r, col] = acc + c[r, col]
            fr = sum(Fraction(a[r, k]) * Fraction(b[k, col]) for k in range(4)) + Fraction(c[r, col])
            exact[r, col] = float(fr)
    return unf, exact
stats = {"eq_unfused": 0, "eq_exact_rounded": 0, "total": 0, "max_ulp_vs_exact": 0.0}
for t in range(200):
    a = rng.normal(size=(8, 4)) * (10.0 ** rng.integers(-3, 4)); b = rng.normal(size=(4, 8)); c = rng.normal(size=(8, 8)) * (10.0 ** rng.integers(-3, 4))
    if t % 2:  # adversarial cancellation
        b[:, :] = -a[:, :].T[:, :8] if False else b
        c = -(a @ b) * (1 + 1e-15)
    d = dmma(a, b, c)
    unf, exact = orders(a, b, c)
    stats["eq_unfused"] += int((d == unf).sum()); stats["eq_exact_rounded"] += int((d == exact).sum()); stats["total"] += 64
    scale = np.abs(a) @ np.abs(b) + np.abs(c)
    stats["max_ulp_vs_exact"] = max(stats["max_ulp_vs_exact"], float((np.abs(d - exact) / (scale * 2.0**-53)).max()))
print(json.dumps(stats))
res["kat"] = stats
print("RESULT", json.dumps(res))
