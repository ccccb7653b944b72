"""CPU: the hand-built test tapes (tests/tapegen.py) parse in the oracle and their gradient /
Hessian outputs are consistent with their energy (central differences)."""
import numpy as np

from tapegen import chain_quartic_tape


def test_chain_tape_derivatives(oracle_mod):
    nodes = 5
    n = 3 * nodes
    tape = chain_quartic_tape(nodes)
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.random(n), [0.0]])
    out = oracle_mod.tape_eval(tape, x[None, :], 1 + n + n * n)[0]
    g, H = out[1:1 + n], out[1 + n:].reshape(n, n)
    np.testing.assert_array_equal(H, H.T)
    h = 1e-6
    for k in range(n):
        xp, xm = x.copy(), x.copy()
        xp[k] += h
        xm[k] -= h
        op = oracle_mod.tape_eval(tape, xp[None, :], 1 + n + n * n)[0]
        om = oracle_mod.tape_eval(tape, xm[None, :], 1 + n + n * n)[0]
        assert abs((op[0] - om[0]) / (2 * h) - g[k]) < 1e-7
        np.testing.assert_allclose((op[1:1 + n] - om[1:1 + n]) / (2 * h), H[:, k], atol=1e-6)


def test_chain_tape_non_finite_when_collapsed(oracle_mod):
    tape = chain_quartic_tape(4)
    x = np.concatenate([np.zeros(6), np.ones(6), [1.0]])
    out = oracle_mod.tape_eval(tape, x[None, :], 1 + 12 + 144)[0]
    assert not np.isfinite(out[0])
