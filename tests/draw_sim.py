"""CPU restatement of k2_draw's arithmetic (paper_2402_19147_b200/csrc/k_draw.cu): the same fp64
operations in the same order (64-ary prefix tree built by pair sums + Hillis-Steele scans, root-to-leaf
descent, proof test, removal by subtraction along the path, exact sequential fallback, rebuild).

Test infrastructure: it checks the kernel's proof bound (that every accepted tree decision equals
numpy's sequential-cumsum decision, cur.py:229-241) on weight vectors with a huge dynamic range, and
keeps the previous round's bound (`use_new=False`) to show what it missed."""
import numpy as np, sys
U53 = 2.0**-53
F = 64

def make_tree(n):
    sz=[n]; s=n
    while s > F:
        s=(s+F-1)//F; sz.append(s)
    return sz

def scan_node(vals):
    # vals: 64 doubles; returns inclusive prefix as the kernel computes: lane l holds pair (2l,2l+1)
    a=vals[0::2].copy(); b=vals[1::2].copy()
    s=a+b
    for o in (1,2,4,8,16):
        y=np.concatenate([np.zeros(o), s[:-o]])
        s=np.where(np.arange(32)>=o, s+y, s)
    ex=np.concatenate([[0.0], s[:-1]])
    out=np.empty(64); out[0::2]=ex+a; out[1::2]=s
    return out

def build(pw, sz):
    P=[]; inp=pw
    for h,n in enumerate(sz):
        nn=(n+F-1)//F
        lev=np.zeros(nn*F); tot=np.zeros(nn)
        padded=np.zeros(nn*F); padded[:n]=inp[:n]
        for k in range(nn):
            lev[k*F:(k+1)*F]=scan_node(padded[k*F:(k+1)*F]); tot[k]=lev[k*F+F-1]
        P.append(lev); inp=tot
    return P

def np_draw(p, count, uni):
    p=p.copy(); out=[]
    for t in range(count):
        cum=np.cumsum(p); u=uni[t]*cum[-1]
        idx=int(np.searchsorted(cum,u,'right'))
        if idx>len(p)-1: idx=len(p)-1
        while idx>0 and p[idx]==0: idx-=1
        out.append(idx); p[idx]=0
    return out

def dev_draw(p, count, uni, use_new=True, stats=None):
    n=len(p); sz=make_tree(n); top=len(sz)-1
    pw=np.zeros(((n+F-1)//F)*F); pw[:n]=p
    P=build(pw,sz)
    cb=4.0*(top+1)*(top+2)+16.0; cr=float(top+3); cnp=n+2.0+top+2
    root=lambda: P[top][F-1]
    total0=root(); err=cb*total0
    out=[]
    for t in range(count):
        u=uni[t]; total=root()
        if use_new and err>cnp*total and total>0:
            P=build(pw,sz); total=root(); total0=total; err=cb*total0
            if stats is not None: stats['rebuild']+=1
        target=u*total
        base=0.0; g=0; ok=True; e_at=[0]*(top+1); lower=upper=wl=0.0
        for h in range(top,-1,-1):
            v=P[h][g*F:(g+1)*F]
            a=base+v
            gt=np.nonzero(a>target)[0]
            if len(gt)==0: ok=False; break
            e=int(gt[0])
            lo=a[e-1] if e>0 else base
            if h==0:
                wl = v[e]-v[e-1] if e>0 else v[e]
                lower=lo; upper=a[e]
            e_at[h]=e; base=lo; g=g*F+e
        idx=g
        if ok:
            if use_new: delta=2*U53*(cnp*total+err)*(1+1e-9)
            else: delta=2*(n+70+(top+2)*count)*U53*(total*(1+1e-12))
            ok = lower<=target-delta and upper>target+delta and wl>0
        if use_new: err+=(14.0*total0+cr*total)*(1+1e-9)
        if ok:
            for h in range(top+1):
                node=idx>>(6*(h+1)); e=e_at[h]
                seg=P[h][node*F:(node+1)*F]
                seg[e:]=seg[e:]-wl
        else:
            if stats is not None: stats['fallback']+=1
            acc=np.cumsum(pw[:n]); tgt=u*acc[-1]
            found=int(np.searchsorted(acc,tgt,'right'))
            if found>n-1: found=n-1
            while found>0 and pw[found]==0: found-=1
            idx=found; w=pw[idx]
            for h in range(top+1):
                node=idx>>(6*(h+1)); e=(idx>>(6*h))&63
                seg=P[h][node*F:(node+1)*F]; seg[e:]=seg[e:]-w
        out.append(idx); pw[idx]=0.0
    return out

