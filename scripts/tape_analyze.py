"""Developer analysis of a SYTP tape: op histogram, DAG sharing, live ranges per grouping."""
import struct, sys, collections
OPS = {2:'add',3:'sub',4:'mul',5:'div',6:'neg',7:'pow',8:'sqrt',9:'log',10:'sin',11:'cos',12:'br'}
def load(path):
    b = open(path,'rb').read(); o = 8 + 32
    ni, no, nd, nr = struct.unpack_from('<4I', b, o); o += 16
    nc, = struct.unpack_from('<Q', b, o); o += 8
    consts = struct.unpack_from('<%dd' % nc, b, o); o += 8*nc
    nins, = struct.unpack_from('<Q', b, o); o += 8
    ins = []
    for k in range(nins):
        op, iarg, dst, a, bb, c = struct.unpack_from('<BiIIII', b, o); o += 21
        ins.append((op, iarg, dst, a, bb, c))
    nout, = struct.unpack_from('<Q', b, o); o += 8
    outs = list(struct.unpack_from('<%dI' % nout, b, o))
    return ni, nd, consts, ins, outs
if __name__ == '__main__':
    ni, nd, consts, ins, outs = load(sys.argv[1])
    base = ni + len(consts)
    print('inputs', ni, 'dofs', nd, 'consts', len(consts), 'instrs', len(ins), 'outputs', len(outs), 'unique out regs', len(set(outs)))
    print(collections.Counter(OPS[i[0]] for i in ins))
    arity = lambda op: 3 if op == 12 else (2 if op in (2,3,4,5) else 1)
    ops_of = [ [i[3], i[4], i[5]][:arity(i[0])] for i in ins]
    # dependence on dofs
    dofdep = [False]*(base+len(ins))
    for s in range(nd): dofdep[s] = True   # assumes dof slots 0..nd-1
    for k, i in enumerate(ins):
        dofdep[base+k] = any(dofdep[r] for r in ops_of[k])
    print('dof-independent ops', sum(1 for k in range(len(ins)) if not dofdep[base+k]))
    # subDAG size per output group
    def closure(regs):
        seen = set(); st = list(regs)
        while st:
            r = st.pop()
            if r < base or r in seen: continue
            seen.add(r); st.extend(ops_of[r-base])
        return seen
    n = nd
    H = lambda i, j: outs[1 + n + i*n + j]
    allH = closure(outs)
    print('closure all', len(allH))
    if n == 12:
        groups = {}
        for a in range(4):
            for c in range(a, 4):
                groups[(a,c)] = [H(i,j) for i in range(3*a,3*a+3) for j in range(3*c,3*c+3)]
        tot = 0
        for g, regs in groups.items():
            s = len(closure(regs)); tot += s
        print('10 node-pair blocks: total work', tot, 'ratio', tot/len(ins))
        # 4 groups by node row a (upper incl)
        tot = 0
        for a in range(4):
            regs = [H(i,j) for i in range(3*a,3*a+3) for j in range(3*a, 12)] + [outs[1+i] for i in range(3*a,3*a+3)]
            tot += len(closure(regs))
        print('4 row-groups: total', tot, tot/len(ins))
        grad = closure(outs[:1+n]); print('E+grad closure', len(grad))
        prim = closure(outs[:1]); print('E closure', len(prim))
