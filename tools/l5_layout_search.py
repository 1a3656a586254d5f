"""Bank-conflict model of fan-out level 5 (DD, TMEM path) and the search for its lane maps.

128-bit shared-memory loads are served per 8-lane phase; a phase costs max over the eight
16-byte bank slots of the distinct addresses hitting that slot.  With the padded fan-out
layout of WarpSmem<dd> (node_off below), this script scores the level-5 loads for a given
lane-pair -> parent map (MirChunk phase: in/sb/self-mirror loads and pivot-row vector loads)
and lane -> parent map (pivot and vector phase), and searches both.  The printed packed maps
are engine.cu's kL5PairMap / kL5VecMap.  usage: python tools/l5_layout_search.py
"""
import itertools, collections
Q0=9; D=8
def tri(d): return d*(d+1)//2
def tri_ix(d,i,j): return i*d-(i*(i+1))//2+j
def cix(i,j,Dd=D): return i*Dd-(i*(i+1))//2+j
def lvl_pad(e): return 2 if e==1 else (1 if e==2 else 0)
def buf_stride(e): return tri(2*(Q0-e)) + (1 if e==2 else 0)
def lvl_off(e):
    o=tri(2*Q0)
    for x in range(1,e): o+=lvl_pad(x)+(1<<(x-1))*buf_stride(x)
    return 0 if e==0 else o+lvl_pad(e)
def node_off(e,c):
    if c==0: return tri_ix(2*Q0,2*e,2*e)
    tz=(c&-c).bit_length()-1; lvl=e-tz; p=(c>>tz)>>1; dim=2*(Q0-lvl)
    return lvl_off(lvl)+p*buf_stride(lvl)+tri_ix(dim,2*tz,2*tz)
# mirror chunk entry lists
A=[(a,b) for a in range(D) for b in range(a,D) if a+b<D-1]
m=10
def wavefronts(addrs):  # addrs: list of 32 entry indices (16B units); per phase of 8 lanes
    tot=0
    for ph in range(4):
        s=collections.defaultdict(set)
        for a in addrs[8*ph:8*ph+8]: s[a%8].add(a)
        tot+=max(len(v) for v in s.values())
    return tot
def l5_cost(perm, base):
    # perm[pair] = parent index
    tot=0
    for C in range(8):
        for t in (0,1):
            i,j=A[2*C+t]; kA=cix(i,j); kB=cix(D-1-j,D-1-i)
            ad=[]; ad2=[]
            for lane in range(32):
                x=perm[lane>>1]; h=lane&1
                Pt=base[x]+2*m-1
                ad.append(Pt+(kB if h else kA)); ad2.append(Pt+kB)
            tot+=wavefronts(ad)+wavefronts(ad2)
    return tot
base=[node_off(4,c) for c in range(16)]
ident=list(range(16))
print('identity', l5_cost(ident, base), 'ideal', 8*2*2*4)
print('bases mod 8', [b%8 for b in base])
def uw_cost(perm):
    tot=0
    for k in range(8):
        for off in (0, m):
            ad=[]
            for lane in range(32):
                x=perm[lane>>1]; h=lane&1
                kk=2+((7-k) if h else k)
                ad.append(x*(2*m+1)+off+kk)
            tot+=wavefronts(ad)
    return tot
def self_cost(perm, base):
    tot=0
    for a in range(4):
        ad=[base[perm[l>>1]]+2*m-1+cix(a,7-a) for l in range(32)]
        tot+=wavefronts(ad)
    return tot
def cost(perm): return l5_cost(perm,base)+uw_cost(perm)+self_cost(perm,base)
print('identity total', cost(ident), 'uw', uw_cost(ident), 'self', self_cost(ident,base))
import random
rng=random.Random(1)
best=ident[:]; bc=cost(best)
for restart in range(200):
    p=list(range(16)); rng.shuffle(p); c=cost(p)
    improved=True
    while improved:
        improved=False
        for i in range(16):
            for j in range(i+1,16):
                p[i],p[j]=p[j],p[i]; c2=cost(p)
                if c2<c: c=c2; improved=True
                else: p[i],p[j]=p[j],p[i]
    if c<bc: bc=c; best=p[:]
print('best', bc, best, 'l5', l5_cost(best,base), 'uw', uw_cost(best), 'self', self_cost(best,base))
print('ideal total', 128 + 16*4 + 4*4)
def vec_cost(sig):
    tot=0
    # pivot loads P[0],P[1],P[m]: lanes x=sig[lane&15]
    for off in (0,1,m):
        tot+=wavefronts([base[sig[l&15]]+off for l in range(32)])
    # vec loads: j = 2+g+2s, s=0..3 ; a = P[j], b = P[m-1+j]
    for s in range(4):
        for extra in (0, m-1):
            tot+=wavefronts([base[sig[l&15]]+extra+2+(l>>4)+2*s for l in range(32)])
    # uw stores uwx[2+g+2s] and uwx[m+2+g+2s], uwx = x*21
    for s in range(4):
        for extra in (0, m):
            tot+=wavefronts([sig[l&15]*(2*m+1)+extra+2+(l>>4)+2*s for l in range(32)])
    return tot
print('vec identity', vec_cost(ident), 'ideal', (3+8+8)*4)
bestv=None; bv=10**9
for mask in range(1<<8):
    pairs=[[4,5],[2,3],[1,12],[14,15],[0,13],[10,11],[8,9],[6,7]]
    A=[p[(mask>>i)&1] for i,p in enumerate(pairs)]; B=[p[1-((mask>>i)&1)] for i,p in enumerate(pairs)]
    sig=A+B
    c=vec_cost(sig)
    if c<bv: bv=c; bestv=sig
print('vec best', bv, bestv)
# pack
def pack(p): return sum(v<<(4*i) for i,v in enumerate(p))
print(hex(pack(best)), hex(pack(bestv)))
