"""Experiment (CPU): tile pairing over the union K set for V=64 HiNM -- K positions (MMA work)
and gathered rows of a greedily packed pair vs two separate tiles, random 50 % kept sets, n = 4096."""
import numpy as np
rng=np.random.default_rng(0)
n=4096; kb=2048
def sim():
    A=np.sort(rng.choice(n,kb,replace=False)); B=np.sort(rng.choice(n,kb,replace=False))
    inB=np.zeros(n,bool); inB[B]=True; inA=np.zeros(n,bool); inA[A]=True
    gA=A.reshape(-1,4); gB=B.reshape(-1,4)          # default sigma_i: ascending survivors
    placed=np.zeros(n,bool); slots=0
    # 1) intact A-groups with <=2 shared columns; 2) intact B-groups (unplaced cols only) with <=2 A-cols
    for g in gA:
        if inB[g].sum()<=2: placed[g]=True; slots+=1
    for g in gB:
        if placed[g].any(): continue
        if inA[g].sum()<=2: placed[g]=True; slots+=1
    # 3) the rest: slots with <=2 A-count and <=2 B-count
    rest=[c for c in np.union1d(A,B) if not placed[c]]
    s=[c for c in rest if inA[c] and inB[c]]; a=[c for c in rest if inA[c] and not inB[c]]; b=[c for c in rest if inB[c] and not inA[c]]
    # pair a's with b's (2a+2b), shared in pairs (2s + pad) or (1s+1a+1b+pad)
    na,nb,ns=len(a),len(b),len(s)
    x=min(na,nb)//2; slots+=x; na-=2*x; nb-=2*x
    # leftover a's: slots of 2a + (up to 2 b) -> nb used; then remaining a or b in pairs
    slots+= (ns+1)//2 + (na+1)//2 + (nb+1)//2
    return slots*4, len(np.union1d(A,B))
r=[sim() for _ in range(20)]
K=np.mean([x[0] for x in r]); U=np.mean([x[1] for x in r])
print("pair K positions %.0f (2*kbar=%d, ratio %.3f); union rows %.0f (ratio %.3f)"%(K,2*kb,K/(2*kb),U,U/(2*kb)))
# MMA cycles: paired M=128 K positions vs 2 x M=64 kbar
print("MMA cycles pair/separate: %.3f; gathered rows pair/separate: %.3f"%((K/32*160)/(2*kb/32*144), U/(2*kb)))
