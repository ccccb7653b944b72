"""Test helper: hand-built derivative tapes in the reference's SYTP v1 wire format
(/root/reference/proj/include/symel/tape.hpp:211-291) for energies no BASELINE config uses
(large elements, energies that blow up on purpose). Register layout as the reference's
`lower` (tape.hpp:121-182): [inputs | constants | one register per instruction], SSA.
"""
from __future__ import annotations

import struct
from typing import Dict, List

OP = dict(add=2, sub=3, mul=4, div=5, neg=6, pow_int=7, sqrt=8, log=9)


class TapeBuilder:
    def __init__(self, n_inputs: int, n_dofs: int):
        self.n_inputs = n_inputs
        self.n_dofs = n_dofs
        self.consts: List[float] = []
        self._cidx: Dict[bytes, int] = {}
        self.instrs: List[tuple] = []  # (op, iarg, a, b) with symbolic operands

    # operands: ("in", k) | ("c", k) | ("op", k)
    def inp(self, k):
        return ("in", k)

    def const(self, v: float):
        key = struct.pack("<d", v)
        if key not in self._cidx:
            self._cidx[key] = len(self.consts)
            self.consts.append(v)
        return ("c", self._cidx[key])

    def op(self, name, a, b=None, iarg=0):
        self.instrs.append((OP[name], iarg, a, b))
        return ("op", len(self.instrs) - 1)

    def _reg(self, r):
        kind, k = r
        if kind == "in":
            return k
        if kind == "c":
            return self.n_inputs + k
        return self.n_inputs + len(self.consts) + k

    def serialize(self, outputs) -> bytes:
        """outputs: [E, g(n), H(n*n)] operand list."""
        base = self.n_inputs + len(self.consts)
        n_regs = base + len(self.instrs)
        b = bytearray(b"SYTP")
        b += struct.pack("<I", 1) + bytes(32)
        b += struct.pack("<IIII", self.n_inputs, len(outputs), self.n_dofs, n_regs)
        b += struct.pack("<Q", len(self.consts)) + b"".join(struct.pack("<d", c) for c in self.consts)
        b += struct.pack("<Q", len(self.instrs))
        for k, (op, iarg, a, bb) in enumerate(self.instrs):
            ra = self._reg(a)
            rb = self._reg(bb) if bb is not None else 0
            b += struct.pack("<BiIIII", op, iarg, base + k, ra, rb, 0)
        b += struct.pack("<Q", len(outputs)) + b"".join(struct.pack("<I", self._reg(o)) for o in outputs)
        return bytes(b)


def chain_quartic_tape(nodes: int) -> bytes:
    """E = sum_i 1/4 (d_i . d_i)^2 + c / (d_0 . d_0), d_i = x_{i+1} - x_i over the element's
    `nodes` 3-vectors (inputs 0 .. 3*nodes-1 are the dofs, input 3*nodes is c). g and H in
    closed form: dE_i/dd = s d, d2E_i/dd2 = s I + 2 d d^T (s = d.d); the c/s term blows up when
    the first two nodes coincide (non-finite outputs on purpose)."""
    n = 3 * nodes
    T = TapeBuilder(n + 1, n)
    zero = T.const(0.0)
    quarter, two = T.const(0.25), T.const(2.0)
    g = [zero] * n
    H = [[zero] * n for _ in range(n)]

    def acc(cur, v):
        return v if cur == zero else T.op("add", cur, v)

    E = zero
    for i in range(nodes - 1):
        d = [T.op("sub", T.inp(3 * (i + 1) + c), T.inp(3 * i + c)) for c in range(3)]
        s = T.op("add", T.op("add", T.op("mul", d[0], d[0]), T.op("mul", d[1], d[1])), T.op("mul", d[2], d[2]))
        E = acc(E, T.op("mul", quarter, T.op("mul", s, s)))
        sd = [T.op("mul", s, d[c]) for c in range(3)]
        for c in range(3):
            g[3 * (i + 1) + c] = acc(g[3 * (i + 1) + c], sd[c])
            g[3 * i + c] = acc(g[3 * i + c], T.op("neg", sd[c]))
        for a in range(3):
            for b in range(3):
                h = T.op("mul", two, T.op("mul", d[a], d[b]))
                if a == b:
                    h = T.op("add", h, s)
                nh = T.op("neg", h)
                for (p, q, v) in ((i + 1, i + 1, h), (i, i, h), (i + 1, i, nh), (i, i + 1, nh)):
                    H[3 * p + a][3 * q + b] = acc(H[3 * p + a][3 * q + b], v)
    # c / (d0.d0): non-finite when nodes 0 and 1 coincide
    d = [T.op("sub", T.inp(3 + c), T.inp(c)) for c in range(3)]
    s0 = T.op("add", T.op("add", T.op("mul", d[0], d[0]), T.op("mul", d[1], d[1])), T.op("mul", d[2], d[2]))
    E = acc(E, T.op("div", T.inp(n), s0))
    gs = T.op("neg", T.op("div", T.inp(n), T.op("mul", s0, s0)))  # dE/ds0 (its Hessian part omitted: c = 0 in
    for c in range(3):                                             # the parity cases, only its finiteness matters)
        v = T.op("mul", T.op("mul", two, gs), d[c])
        g[3 + c] = acc(g[3 + c], v)
        g[c] = acc(g[c], T.op("neg", v))
    return T.serialize([E] + g + [H[r][c] for r in range(n) for c in range(n)])
