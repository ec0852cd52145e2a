"""Offline check of diagonal-cache indexings over 2-D 5/9-point (nx 200..4199),
3-D 7/27-point (nx 40..719) stencils and random contiguous bands: how many
matrices put more hot diagonals on one slot/set than it holds
(csrc/matrix.cuh diag_set).  Pure Python, no GPU."""
import numpy as np
M=(1<<64)-1
def F_low(u): return u&511
def F_fold(u): return (u^(u>>9)^(u>>18))&511
def F_fold2(u): return (u+(u>>9)*7+(u>>18)*13+(u>>27)*31)&511
def F_fold3(u): return (u^((u>>9)*0x9e3779b1)^((u>>18)*0x85ebca6b))&511
def F_mulhi(u): return ((u*0x9E3779B97F4A7C15)&M)>>55
cases=[]
for nx in range(200,4200,1):
    n=nx*nx
    cases.append(("5pt",nx,[o+n-1 for o in (0,1,-1,nx,-nx)]))
    cases.append(("9pt",nx,[dy*nx+dx+n-1 for dy in (-1,0,1) for dx in (-1,0,1)]))
for nx in range(40,720):
    n=nx**3
    cases.append(("7pt",nx,[o+n-1 for o in (0,1,-1,nx,-nx,nx*nx,-nx*nx)]))
    cases.append(("27pt",nx,[dz*nx*nx+dy*nx+dx+n-1 for dz in (-1,0,1) for dy in (-1,0,1) for dx in (-1,0,1)]))
rng=np.random.default_rng(0)
for k in range(2000):
    n=int(rng.integers(1<<16,1<<23)); w=int(rng.integers(3,64))
    cases.append(("band",n,[o+n-1 for o in range(-(w//2),w-w//2)]))
for name,F in [("low",F_low),("fold",F_fold),("fold2",F_fold2),("fold3",F_fold3),("mulhi",F_mulhi)]:
    bad={}
    for kind,nx,ds in cases:
        s=[F(d) for d in ds]
        if len(set(s))<len(s): bad[kind]=bad.get(kind,0)+1
    print(name, bad)
print("--- set associative (overflow = some set holds more hot diagonals than ways)")
def sa(F, ways):
    nsets=512//ways
    bad={}
    for kind,nx,ds in cases:
        cnt={}
        for d in ds:
            s=F(d)%nsets
            cnt[s]=cnt.get(s,0)+1
        if max(cnt.values())>ways: bad[kind]=bad.get(kind,0)+1
    return bad
for ways in (2,4,8):
    for name,F in [("low",F_low),("fold",F_fold),("fold2",F_fold2),("mulhi",F_mulhi)]:
        print(ways, name, sa(F,ways))
