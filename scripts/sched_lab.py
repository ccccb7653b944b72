"""Developer lab: schedule heuristics and live-set analysis on a SYTP tape (register pressure)."""
import sys, collections
sys.path.insert(0, 'scripts')
from tape_analyze import load, OPS

def build(path):
    ni, nd, consts, ins, outs = load(path)
    base = ni + len(consts)
    ar = lambda op: 3 if op == 12 else (2 if op in (2,3,4,5) else 1)
    ops = [[r for r in (i[3], i[4], i[5])[:ar(i[0])] if r >= base] for i in ins]
    ops = [sorted(set(o)) for o in ops]
    users = [[] for _ in ins]
    for k, o in enumerate(ops):
        for r in o: users[r - base].append(k)
    return ni, nd, consts, ins, outs, base, ops, users

def live_profile(order, ops, outs_set_k, n):
    pos = {k: p for p, k in enumerate(order)}
    last = {}
    for p, k in enumerate(order):
        for c in ops[k]: last[c - BASE] = p
    ev = [0] * (len(order) + 2)
    for p, k in enumerate(order):
        l = last.get(k, p)
        ev[p] += 1; ev[l + 1] -= 1
    cur = mx = 0; at = 0; prof = []
    for p in range(len(order)):
        cur += ev[p]; prof.append(cur)
        if cur > mx: mx, at = cur, p
    return mx, at, prof, last

if __name__ == '__main__':
    ni, nd, consts, ins, outs, base, ops, users = build(sys.argv[1])
    BASE = base
    n = len(ins)
    # depth from inputs
    depth = [0]*n
    for k in range(n):
        depth[k] = 1 + max([depth[c-base] for c in ops[k]], default=0)
    # dof dependence classes: set of dof slots each node depends on
    dep = [0]*n
    for k in range(n):
        m = 0
        for r in (ins[k][3], ins[k][4], ins[k][5])[: (3 if ins[k][0]==12 else 2 if ins[k][0] in (2,3,4,5) else 1)]:
            if r < nd: m |= 1 << r
            elif r >= base: m |= dep[r-base]
        dep[k] = m
    order = list(range(n))
    mx, at, prof, last = live_profile(order, ops, None, n)
    print('tape order max live', mx, 'at', at)
    live = [k for k in range(n) if k <= at and last.get(k, k) >= at]
    c = collections.Counter(bin(dep[k]).count('1') for k in live)
    print('live by #dofs depended on', sorted(c.items()))
    c2 = collections.Counter(len(users[k]) for k in live)
    print('live by #users', sorted(c2.items())[:20])
    print('n users hist all', sorted(collections.Counter(min(len(u), 20) for u in users).items()))

def greedy(ops, users, n, outs_k, prio):
    """top-down list scheduling: pick ready node with min net live delta, then prio."""
    import heapq
    remaining_users = [len(set(u)) for u in users]
    uses_left = {}
    for k in range(n):
        uses_left[k] = len(set(users[k])) + (1 if k in outs_k else 0)
    nops_left = [len(o) for o in ops]
    ready = [k for k in range(n) if nops_left[k] == 0]
    done = [False]*n
    order = []
    useu = [sorted(set(u)) for u in users]
    def delta(k):
        kills = sum(1 for c in ops[k] if uses_left[c - BASE] == 1)
        return (0 if uses_left[k] == 0 else 1) - kills
    while ready:
        best = min(ready, key=lambda k: (delta(k), prio[k]))
        ready.remove(best)
        order.append(best); done[best] = True
        for c in ops[best]:
            uses_left[c - BASE] -= 1
        for u in useu[best]:
            nops_left[u] -= 1
            if nops_left[u] == 0: ready.append(u)
    return order
