"""Python emulation of hq_chase2 (two-bulge round body) with 32-row windows and accumulated-Q far updates."""
# Python emulation of hq_chase2's round body on a full window (lo = m, r1 = nn), compared with the
# reference two-bulge sweep (emul.sweep2 with zeroing).
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.abspath(__file__)))
import hq_emul as emul

def refl(p,q,r):
    t=p*p+q*q+r*r
    if not t>=2.3e-308: return dict(xx=0,yy=0,zz=0,qq=0,rr=0,s=0,valid=False)
    s=np.sqrt(t); s=-s if p<0 else s
    pp=p+s
    return dict(xx=pp/s,yy=q/s,zz=r/s,qq=q/pp,rr=r/pp,s=s,valid=True)

def chase2(H, lo, r1, a0, a1, m, nn, l, sp, sq, sr, sx, sy, sw, NL=None, Q=None):
    def H_(i,j):
        return H[i,j] if (i>=lo and j>=lo-1 and i<=r1 and j<=r1) else 0.0
    def load_state(k):
        return dict(B=np.array([[H_(k+i,k+j) for j in range(3)] for i in range(3)]),
                    C=np.array([H_(k+i,k+3) for i in range(3)]), h3=H_(k+3,k+2), d33=H_(k+3,k+3))
    kA=a0; kB=a0-4
    if kA==m: p,q,r=sp,sq,sr
    else: p,q,r=H_(kA,kA-1),H_(kA+1,kA-1),H_(kA+2,kA-1)
    A=load_state(kA) if kA<=nn-1 else None
    RA=refl(p,q,r) if kA<=nn-1 else refl(0,0,0)
    if m<=kB<=nn-1:
        Bb=load_state(kB); RB=refl(H_(kB,kB-1),H_(kB+1,kB-1),H_(kB+2,kB-1))
    else:
        Bb=None; RB=refl(0,0,0)
    nlanes = r1-lo+1 if NL is None else NL
    for kA in range(a0,a1):
        kB=kA-4
        actA = kA<=nn-1; actB = m<=kB<=nn-1
        if kB==m:
            z=H_(m,m); rr=sx-z; ss=sy-z
            p=(rr*ss-sw)/H_(m+1,m)+H_(m,m+1); q=H_(m+1,m+1)-z-rr-ss; r=H_(m+2,m+1)
            Bb=load_state(kB); Bb['B'][2,0]=0.0
            RB=refl(p,q,r)
        E=np.array([H_(kA+i,kA+4) for i in range(4)]); h4=H_(kA+4,kA+3); d44=H_(kA+4,kA+4)
        if actB:
            Bb['C']=np.array([H_(kB+i,kB+3) for i in range(3)]); Bb['h3']=H_(kB+3,kB+2); Bb['d33']=H_(kB+3,kB+3)
        Z=np.array([[H_(kB+i,kA+j) if kA+j<=nn else 0.0 for j in range(3)] for i in range(3)])
        if A is None: A=dict(B=np.zeros((3,3)),C=np.zeros(3),h3=0.0,d33=0.0)
        if Bb is None: Bb=dict(B=np.zeros((3,3)),C=np.zeros(3),h3=0.0,d33=0.0)
        Hs=H.copy()   # all loads see the pre-round values
        stores=[]
        u=np.array([RA['xx'],RA['yy'],RA['zz']]); w1,w2=RA['qq'],RA['rr']
        v=np.array([RB['xx'],RB['yy'],RB['zz']]); x1,x2=RB['qq'],RB['rr']
        # forward A
        BA=A['B']; pp=BA[0]+w1*BA[1]+w2*BA[2]; ppc=A['C'][0]+w1*A['C'][1]+w2*A['C'][2]; ppe=E[0]+w1*E[1]+w2*E[2]
        R1=BA[1]-u[1]*pp; R1c=A['C'][1]-u[1]*ppc; R1e=E[1]-u[1]*ppe
        R2=BA[2]-u[2]*pp; R2c=A['C'][2]-u[2]*ppc; R2e=E[2]-u[2]*ppe
        t1=u@R1; t2=u@R2; t3=u[2]*A['h3']
        N1=R1-t1*np.array([1,w1,w2]); N2=R2-t2*np.array([1,w1,w2]); N3=np.array([0,0,A['h3']])-t3*np.array([1,w1,w2])
        nxA = actA and kA+1<=nn-1
        RnA=refl(N1[0] if nxA else 0, N2[0] if nxA else 0, N3[0] if nxA else 0)
        # forward B
        BB=Bb['B']; qq=BB[0]+x1*BB[1]+x2*BB[2]; qqc=Bb['C'][0]+x1*Bb['C'][1]+x2*Bb['C'][2]
        S1=BB[1]-v[1]*qq; S1c=Bb['C'][1]-v[1]*qqc; S2=BB[2]-v[2]*qq; S2c=Bb['C'][2]-v[2]*qqc
        e1=v@S1; e2=v@S2; e3=v[2]*Bb['h3']
        M1=S1-e1*np.array([1,x1,x2]); M2=S2-e2*np.array([1,x1,x2]); M3=np.array([0,0,Bb['h3']])-e3*np.array([1,x1,x2])
        nxB = actB and kB+1<=nn-1
        RnB=refl(M1[0] if nxB else 0, M2[0] if nxB else 0, M3[0] if nxB else 0)
        # stores
        if actA and RA['valid']:
            H[kA,kA-1] = (-Hs[kA,kA-1] if l!=m else Hs[kA,kA-1]) if kA==m else -RA['s']
        if actB and RB['valid']:
            H[kB,kB-1] = (-Hs[kB,kB-1] if l!=m else Hs[kB,kB-1]) if kB==m else -RB['s']
        for lane in range(nlanes):
            jA=kA+3+lane
            if actA and jA<=r1:
                a=np.array([Hs[kA+i,jA] if kA+i<=nn else 0.0 for i in range(3)])
                pr=a[0]+w1*a[1]+w2*a[2]
                H[kA,jA]=a[0]-u[0]*pr; H[kA+1,jA]=a[1]-u[1]*pr
                if kA+2<=nn: H[kA+2,jA]=a[2]-u[2]*pr
            jB=kB+3+lane
            if actB and jB<=r1 and (not actA or lane<1 or lane>3):
                a=np.array([Hs[kB+i,jB] if kB+i<=nn else 0.0 for i in range(3)])
                pr=a[0]+x1*a[1]+x2*a[2]
                H[kB,jB]=a[0]-v[0]*pr; H[kB+1,jB]=a[1]-v[1]*pr
                if kB+2<=nn: H[kB+2,jB]=a[2]-v[2]*pr
            ir=lo+lane
            cokA = actA and ir<=min(nn,kA+3); specA = kB<=ir<=kB+2
            if cokA:
                d=ir-kA; dB=ir-kB
                if specA:
                    zz=Z[0]+x1*Z[1]+x2*Z[2]; c=Z[dB]-v[dB]*zz
                elif ir>=kA:
                    X=BA[0]-u[0]*pp
                    c = X if d==0 else (R1 if d==1 else (R2 if d==2 else np.array([0,0,A['h3']])))
                else:
                    c=np.array([Hs[ir,kA+j] if kA+j<=nn else 0.0 for j in range(3)])
                tt=u@c
                H[ir,kA]=c[0]-tt
                if kA+1<=nn: H[ir,kA+1]=c[1]-tt*w1
                if kA+2<=nn: H[ir,kA+2]=c[2]-tt*w2
            cokB = actB and ir<=min(nn,kB+3)
            if cokB:
                d=ir-kB
                if ir>=kB:
                    Y=BB[0]-v[0]*qq
                    c = Y if d==0 else (S1 if d==1 else (S2 if d==2 else np.array([0,0,Bb['h3']])))
                else:
                    c=np.array([Hs[ir,kB+j] if kB+j<=nn else 0.0 for j in range(3)])
                tt=v@c
                H[ir,kB]=c[0]-tt; H[ir,kB+1]=c[1]-tt*x1
                if kB+2<=nn: H[ir,kB+2]=c[2]-tt*x2
        if Q is not None:
            if actA:
                c=Q[:,kA-lo:kA-lo+3].copy(); tq=c@u; Q[:,kA-lo]=c[:,0]-tq; Q[:,kA-lo+1]=c[:,1]-tq*w1; Q[:,kA-lo+2]=c[:,2]-tq*w2
            if actB:
                c=Q[:,kB-lo:kB-lo+3].copy(); tq=c@v; Q[:,kB-lo]=c[:,0]-tq; Q[:,kB-lo+1]=c[:,1]-tq*x1; Q[:,kB-lo+2]=c[:,2]-tq*x2
        RA=RnA
        A=dict(B=np.array([[N1[1],N1[2],R1c],[N2[1],N2[2],R2c],[N3[1],N3[2],A['d33']]]),C=np.array([R1e,R2e,E[3]]),h3=h4,d33=d44)
        RB=RnB
        Bb=dict(B=np.array([[M1[1],M1[2],S1c],[M2[1],M2[2],S2c],[M3[1],M3[2],Bb['d33']]]),C=Bb['C'],h3=Bb['h3'],d33=Bb['d33'])


def windowed(H, l, m, nn, sp, sq, sr, sx, sy, sw):
    k0=m; a0=m; a1=min(k0+29, nn+4); r1=min(k0+31, nn)
    while True:
        Q=np.zeros((34,34)); Q[:32,:32]=np.eye(32)
        chase2(H, k0, r1, a0, a1, m, nn, l, sp, sq, sr, sx, sy, sw, NL=32, Q=Q)
        nr=r1-k0+1
        Qn=Q[:nr,:nr]
        # far right and far above
        if r1<nn: H[k0:r1+1, r1+1:nn+1] = Qn.T @ H[k0:r1+1, r1+1:nn+1]
        if k0>l: H[l:k0, k0:r1+1] = H[l:k0, k0:r1+1] @ Qn
        if a1>=nn+4: break
        k0=a1-4; a0=a1; a1=min(k0+29, nn+4); r1=min(k0+31,nn)

if __name__ == '__main__':
    rng=np.random.default_rng(1)
    for n,l,m in [(40,0,0),(100,0,0),(100,5,9)]:
        from scipy.linalg import hessenberg
        H0=hessenberg(rng.standard_normal((n,n)))
        if l>0: H0[l,l-1]=0.0
        nn=n-1
        x=H0[nn,nn]; y=H0[nn-1,nn-1]; w=H0[nn,nn-1]*H0[nn-1,nn]
        zz=H0[m,m]; rr=x-zz; ss=y-zz
        p=(rr*ss-w)/H0[m+1,m]+H0[m,m+1]; q=H0[m+1,m+1]-zz-rr-ss; r=H0[m+2,m+1]
        Href=H0.copy(); emul.sweep2(Href,l,m,nn,x,y,w)
        Hk=H0.copy()
        for i in range(m+2,nn+1):
            Hk[i,i-2]=0
            if i!=m+2: Hk[i,i-3]=0
        windowed(Hk,l,m,nn,p,q,r,x,y,w)
        mask=np.triu(np.ones((n,n)),-1).astype(bool)
        print(n,l,m,"max diff (Hessenberg part):", np.abs((Href-Hk)[mask]).max())
