"""Pure-Python model of packets pass S (group_syndrome64 in packets.cuh): the 64-position chunk
decomposition with the partial last chunk masked, reduced over the L lanes of a group, against the
direct XOR of the set positions, for random (n, L, bit offset, stream) cases.  A design check run on
the CPU before the kernel change went to the GPU: python tools/check_pass_s_math.py"""
import random
M32=0xFFFFFFFF
def funnel_r(lo,hi,sh): return ((hi<<32|lo)>>(sh&31))&M32
def popc(x): return bin(x).count('1')
def fl(r): return M32 if r>=32 else ((1<<r)-1)
def S5(x): 
    s=0
    for b in range(32):
        if x>>b&1: s^=b
    return s
def sim(words, o, n, L):
    rb=o&31; np1=n+1; full=np1//64; rest=np1-64*full; nch=full+(1 if rest else 0)
    mlo=fl(rest); mhi=fl(rest-32) if rest>32 else 0
    tot=[]
    Xs=[];Ps=[]
    for q in range(L):
        X=H=A0=A1=BB=0
        base=(o>>5)+2*q
        def block(blk,checked):
            nonlocal X,H,A0,A1,BB
            cnt=nch-4*L*blk-q
            Xb=0
            for it in range(4):
                if (not checked) or L*it<cnt:
                    i=base+8*L*blk+2*L*it
                    w0,w1,w2=words[i],words[i+1],words[i+2]
                    hi=funnel_r(w1,w2,rb); lo=funnel_r(w0,w1,rb)
                    if checked and rest and L*it==cnt-1: lo&=mlo; hi&=mhi
                    y=lo^hi; Xb^=y; H^=hi
                    if it&1: A0^=y
                    if it&2: A1^=y
            X^=Xb
            if popc(Xb)&1: BB^=blk
        nb=full//(4*L)
        for blk in range(nb): block(blk,False)
        if 4*L*nb<nch: block(nb,True)
        P=(64*((q*(popc(X)&1)) ^ L*((4*BB)^(popc(A0)&1)^((popc(A1)&1)<<1))))^(32*(popc(H)&1))
        Xs.append(X);Ps.append(P)
    X=0;P=0
    for x in Xs: X^=x
    for p in Ps: P^=p
    return P^S5(X)
def direct(words,o,n):
    s=0
    for p in range(1,n+1):
        b=o+p
        if words[b>>5]>>(b&31)&1: s^=p
    return s
random.seed(1)
bad=0
for trial in range(3000):
    L=random.choice([1,2,4,8,16,32]); n=random.randint(11,9000); o=random.randint(0,200)
    nw=(o+n+64*4*L*2)//32+8
    words=[random.getrandbits(32) for _ in range(nw)]
    if sim(words,o,n,L)!=direct(words,o,n): bad+=1
print("mismatches",bad)
