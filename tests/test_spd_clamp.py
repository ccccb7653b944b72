"""The fused SPD projection's eigen fragment (codegen.cpp eig_source, tred2/tql2 in registers),
compiled on the host exactly as the code generator emits them and checked against numpy's
eigh-based clamp (clamp negative eigenvalues of the element Hessian to zero).

Cases cover what breaks eigen-solvers: exact and near-degenerate clusters inside and across
the clamped set, zero / rank-deficient / already-diagonal matrices, all-negative and
all-positive spectra, wide dynamic range. The bar is the assembled-Hessian tolerance
(1e-10 relative, in the matrix norm of the element block)."""
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2303_02156_b200", "csrc")
HOST = os.path.join(ROOT, "tests", "host")


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("no host C++ compiler")
    d = tmp_path_factory.mktemp("clamp")
    dump = d / "dump"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + CSRC, "-o", str(dump),
                    os.path.join(HOST, "dump_fragments.cpp"), os.path.join(CSRC, "codegen.cpp")], check=True)
    (d / "clamp_fragment.inc").write_text(subprocess.run([str(dump)], check=True, capture_output=True,
                                                         text=True).stdout)
    exe = d / "clamp"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + str(d), "-o", str(exe),
                    os.path.join(HOST, "clamp_harness.cpp")], check=True)
    return str(exe)


def run(exe, mats, variant=""):
    n = mats.shape[1]
    txt = "\n".join(" ".join("%.17g" % v for v in m.ravel()) for m in mats)
    out = subprocess.run([exe, str(n)] + ([variant] if variant else []), input=txt, capture_output=True,
                         text=True, check=True).stdout
    return np.array(out.split(), dtype=np.float64).reshape(mats.shape)


def clamp_ref(m):
    w, v = np.linalg.eigh(m)
    return (v * np.maximum(w, 0.0)) @ v.T


def with_spectrum(rng, w):
    q, _ = np.linalg.qr(rng.standard_normal((len(w), len(w))))
    m = (q * w) @ q.T
    return 0.5 * (m + m.T)


def cases(rng, n):
    out = []
    for _ in range(200):  # generic symmetric
        a = rng.standard_normal((n, n))
        out.append(a + a.T)
    for _ in range(50):  # stable-NH-like: most eigenvalues positive, a few negative
        w = rng.uniform(0.1, 10.0, n)
        w[: rng.integers(0, n // 2 + 2)] *= -rng.uniform(1e-3, 1.0)
        out.append(with_spectrum(rng, w))
    for gap in (0.0, 1e-15, 1e-12, 1e-8, 1e-4):  # clusters inside the clamped set and across
        for _ in range(10):
            w = rng.uniform(-3, 3, n)
            w[1] = w[0] + gap
            if n >= 3:
                w[2] = -w[0] if rng.random() < 0.5 else w[2]
            if n >= 4:
                w[3] = w[0] - gap
            out.append(with_spectrum(rng, w))
        w = np.full(n, -1.0); w[: n // 2] = 2.0; w[0] += gap
        out.append(with_spectrum(rng, w))
    out.append(np.zeros((n, n)))
    out.append(np.diag(np.linspace(-1, 1, n)))            # already diagonal (tridiagonal, e = 0)
    out.append(-np.eye(n))
    out.append(np.eye(n))
    out.append(np.diag(np.r_[-np.ones(n // 2), np.ones(n - n // 2)]))  # exact multiplicities
    v = rng.standard_normal(n)
    out.append(-np.outer(v, v))                           # rank one, negative
    out.append(np.outer(v, v) - 1e-9 * np.eye(n))         # nearly PSD
    w = np.geomspace(1e-12, 1e4, n) * np.where(np.arange(n) % 3 == 0, -1, 1)
    out.append(with_spectrum(rng, w))                     # wide dynamic range
    return np.array(out)


@pytest.mark.parametrize("variant", ["plain", "la"])
@pytest.mark.parametrize("n", [2, 3, 4, 6, 9])
def test_clamp_matches_eigh(harness, n, variant):
    """Both QL variants: sy_ql and the lookahead sy_ql_la (its warp-mates emulated by a random
    vote in the host harness, so lookahead sweeps are exercised)."""
    rng = np.random.default_rng(1234 + n)
    mats = cases(rng, n)
    got = run(harness, mats, variant)
    worst = 0.0
    for m, g in zip(mats, got):
        ref = clamp_ref(m)
        scale = max(np.abs(m).max(), 1e-300)
        worst = max(worst, np.abs(g - ref).max() / scale)
        assert np.allclose(g, g.T, rtol=0, atol=1e-14 * scale)
    assert worst <= 1e-10, worst


@pytest.mark.parametrize("n", [3, 9])
def test_lookahead_is_bitwise_the_plain_ql(harness, n):
    """The lookahead only reschedules sweeps across a warp: every lane runs the same arithmetic
    in the same order as sy_ql, so the results are bit-identical."""
    rng = np.random.default_rng(99 + n)
    mats = cases(rng, n)
    assert np.array_equal(run(harness, mats, "plain"), run(harness, mats, "la"))


def stress_cases(rng, n, count):
    """Random, clustered (at random scales), graded, low-rank-plus-shift, sparse / split and
    stable-NH-like spectra."""
    out = []
    for _ in range(count):
        kind = rng.integers(0, 6)
        if kind == 0:
            a = rng.standard_normal((n, n))
            out.append(a + a.T)
        elif kind == 1:
            w = np.concatenate([b + rng.standard_normal(3) * 10.0 ** rng.uniform(-16, -2)
                                for b in rng.uniform(-1, 1, (n + 2) // 3)])[:n]
            out.append(with_spectrum(rng, w * 10.0 ** rng.uniform(-5, 15)))
        elif kind == 2:
            w = np.geomspace(1, 10.0 ** rng.uniform(3, 16), n) * rng.choice([-1, 1], n)
            out.append(with_spectrum(rng, w))
        elif kind == 3:
            v = rng.standard_normal((n, 2))
            out.append(v @ np.diag(rng.uniform(-3, 3, 2)) @ v.T + rng.uniform(-1, 1) * np.eye(n))
        elif kind == 4:
            a = np.zeros((n, n))
            for _ in range(rng.integers(1, 10)):
                i, j = rng.integers(0, n, 2)
                v = rng.standard_normal()
                a[i, j] += v
                a[j, i] += v
            out.append(a)
        else:
            w = rng.uniform(0.1, 10.0, n)
            w[: rng.integers(0, n)] *= -rng.uniform(1e-6, 1.0)
            out.append(with_spectrum(rng, w))
    return np.array(out)


@pytest.mark.parametrize("variant", ["plain", "la"])
@pytest.mark.parametrize("n", [3, 9])
def test_clamp_stress(harness, n, variant):
    """1500 hard matrices per size through the QL clamp: within 1e-10 of numpy's eigh clamp."""
    rng = np.random.default_rng(7 + n)
    mats = stress_cases(rng, n, 1500)
    got = run(harness, mats, variant)
    errs = [np.abs(g - clamp_ref(m)).max() / max(np.abs(m).max(), 1e-300) for m, g in zip(mats, got)]
    assert max(errs) <= 1e-10, max(errs)
