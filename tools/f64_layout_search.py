"""Bank-conflict search for the fp64 fan-out layout (8-byte words; level-5 node states in
shared memory, read lane-wise by the lane subtrees in two 16-lane phases).  Scores the worst
per-phase multiplicity of the 32 level-5 node bases mod 16 for base pads / stride adds of levels
1..5 and hill-climbs them; the result is WarpSmem<double>::lvl_pad / buf_stride in engine.cu.
usage: python tools/f64_layout_search.py"""
import itertools, collections, random
Q0=10; FAN=5
def tri(d): return d*(d+1)//2
def tri_ix(d,i,j): return i*d-(i*(i+1))//2+j
def mk(pads, adds):
    def stride(e): return tri(2*(Q0-e))+adds[e-1]
    def lvl_off(e):
        o=tri(2*Q0)
        for x in range(1,e): o+=pads[x-1]+(1<<(x-1))*stride(x)
        return 0 if e==0 else o+(pads[e-1] if e<=5 else 0)
    def node_off(e,c):
        if c==0: return tri_ix(2*Q0,2*e,2*e)
        tz=(c&-c).bit_length()-1; lvl=e-tz; p=(c>>tz)>>1; dim=2*(Q0-lvl)
        return lvl_off(lvl)+p*stride(lvl)+tri_ix(dim,2*tz,2*tz)
    return node_off, lvl_off(FAN+1)
def cost(pads, adds):
    node_off, end = mk(pads, adds)
    b=[node_off(5,c) for c in range(32)]
    tot=0
    for ph in (range(0,16), range(16,32)):
        h=collections.Counter(b[c]%16 for c in ph)
        tot+=max(h.values())
    return tot, end
base=cost([0]*5,[0]*5); print('identity', base)
rng=random.Random(1); best=(base[0], base[1], [0]*5, [0]*5)
for it in range(200000):
    pads=[rng.randrange(16) for _ in range(5)]; adds=[rng.randrange(4) for _ in range(5)]
    c,end=cost(pads,adds)
    extra=end-base[1]
    if (c, extra) < (best[0], best[1]-base[1] if best[1] else 0) or (c < best[0]) or (c==best[0] and extra < best[1]-base[1]):
        best=(c,end,pads,adds)
print('best', best[0], 'extra entries', best[1]-base[1], best[2], best[3])
# hill climbing from random starts, objective (cost, extra)
def obj(p,a):
    c,end=cost(p,a); return (c, end-base[1])
bestg=None
for r in range(300):
    p=[rng.randrange(16) for _ in range(5)]; a=[rng.randrange(4) for _ in range(5)]
    cur=obj(p,a); improved=True
    while improved:
        improved=False
        for i in range(5):
            for v in range(16):
                q=p[:]; q[i]=v; o=obj(q,a)
                if o<cur: cur=o; p=q; improved=True
            for v in range(4):
                b=a[:]; b[i]=v; o=obj(p,b)
                if o<cur: cur=o; a=b; improved=True
    if bestg is None or cur<bestg[0]: bestg=(cur,p,a)
print('hill', bestg)
def gcost(p,a):
    node_off,end=mk(p,a)
    b=[node_off(5,c)%16 for c in range(32)]
    h=collections.Counter(b)
    return (max(h.values()), end-base[1]), b
bestb=None
for r in range(400):
    p=[rng.randrange(16) for _ in range(5)]; a=[rng.randrange(4) for _ in range(5)]
    cur,_=gcost(p,a); improved=True
    while improved:
        improved=False
        for i in range(5):
            for v in range(16):
                q=p[:]; q[i]=v; o,_=gcost(q,a)
                if o<cur: cur=o; p=q; improved=True
            for v in range(4):
                b2=a[:]; b2[i]=v; o,_=gcost(p,b2)
                if o<cur: cur=o; a=b2; improved=True
    if bestb is None or cur<bestb[0]: bestb=(cur,p,a)
print('global balance', bestb)
