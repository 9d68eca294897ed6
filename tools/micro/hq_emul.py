"""Python emulation of the Numerical-Recipes Francis double-shift sweep with one or two bulges
(reference for the hqr_kernel two-bulge experiment, tools/micro/hqr_cmp.py)."""
import numpy as np
def refl(p,q,r):
    t=p*p+q*q+r*r
    if t==0: return None
    s=np.sqrt(t); s = -s if p<0 else s
    pp=p+s
    return dict(xx=pp/s,yy=q/s,zz=r/s,qq=q/pp,rr=r/pp,s=s)
def apply(H,k,R,l,nn,m,first):
    # NR step k with reflector R (rows/cols k..k+2)
    if R is None: return
    if first:
        if l!=m: H[k,k-1]=-H[k,k-1]
    else:
        H[k,k-1]=-R['s']
        H[k+1,k-1]=0.0
        if k!=nn-1: H[k+2,k-1]=0.0
    x,y,z,q,r=R['xx'],R['yy'],R['zz'],R['qq'],R['rr']
    three = k!=nn-1
    for j in range(k,nn+1):
        p=H[k,j]+q*H[k+1,j]
        if three: p+=r*H[k+2,j]; H[k+2,j]-=p*z
        H[k+1,j]-=p*y; H[k,j]-=p*x
    for i in range(l,min(nn,k+3)+1):
        p=x*H[i,k]+y*H[i,k+1]
        if three: p+=z*H[i,k+2]; H[i,k+2]-=p*r
        H[i,k+1]-=p*q; H[i,k]-=p
def pqr(H,m,x,y,w):
    zz=H[m,m]; r=x-zz; s=y-zz
    p=(r*s-w)/H[m+1,m]+H[m,m+1]; q=H[m+1,m+1]-zz-r-s; r=H[m+2,m+1]
    return p,q,r
def sweep2(H,l,m,nn,x,y,w,G=4):
    for i in range(m+2,nn+1):
        H[i,i-2]=0
        if i!=m+2: H[i,i-3]=0
    RA=None; RB=None
    for kA in range(m, nn + (G if G < 100 else 0)):
        kB=kA-G
        if kA<=nn-1:
            if kA==m: p,q,r=pqr(H,m,x,y,w)
            else:
                p=H[kA,kA-1]; q=H[kA+1,kA-1]; r=H[kA+2,kA-1] if kA!=nn-1 else 0.0
            RA=refl(p,q,r)
        if m<=kB<=nn-1:
            if kB==m: p,q,r=pqr(H,m,x,y,w)
            else:
                p=H[kB,kB-1]; q=H[kB+1,kB-1]; r=H[kB+2,kB-1] if kB!=nn-1 else 0.0
            RB=refl(p,q,r)
        # order: A then B (commute)
        if kA<=nn-1: apply(H,kA,RA,l,nn,m,kA==m)
        if m<=kB<=nn-1: apply(H,kB,RB,l,nn,m,kB==m)
def hqr(H0, nb=2):
    H=H0.copy(); n=H.shape[0]; nn=n-1; anorm=np.abs(H).sum(); t=0.0; ev=[]; sweeps=0
    while nn>=0:
        its=0
        while True:
            l=nn
            while l>=1:
                s=abs(H[l-1,l-1])+abs(H[l,l])
                if s==0: s=anorm
                if abs(H[l,l-1])+s==s: H[l,l-1]=0; break
                l-=1
            x=H[nn,nn]
            if l==nn: ev.append(x+t); nn-=1; break
            y=H[nn-1,nn-1]; w=H[nn,nn-1]*H[nn-1,nn]
            if l==nn-1:
                p=0.5*(y-x); q=p*p+w; z=np.sqrt(abs(q)); x+=t
                if q>=0: z=p+np.copysign(z,p); ev+= [x+z, x-w/z if z!=0 else x+z]
                else: ev+=[complex(x+p,z),complex(x+p,-z)]
                nn-=2; break
            if its==60: raise RuntimeError("noconv")
            if its and its%10==0:
                t+=x
                for i in range(nn+1): H[i,i]-=x
                s=abs(H[nn,nn-1])+abs(H[nn-1,nn-2]); x=y=0.75*s; w=-0.4375*s*s
            its+=1; sweeps+=1
            # m search
            m=nn-2
            while m>=l:
                zz=H[m,m]; r=x-zz; s=y-zz
                p=(r*s-w)/H[m+1,m]+H[m,m+1]; q=H[m+1,m+1]-zz-r-s; r=H[m+2,m+1]
                s=abs(p)+abs(q)+abs(r); p/=s;q/=s;r/=s
                if m==l: break
                u=abs(H[m,m-1])*(abs(q)+abs(r)); v=abs(p)*(abs(H[m-1,m-1])+abs(zz)+abs(H[m+1,m+1]))
                if u+v==v: break
                m-=1
            if nb==2: sweep2(H,l,m,nn,x,y,w)
            else: sweep2(H,l,m,nn,x,y,w,G=10**9)
    return np.array(ev), sweeps
if __name__ == '__main__':
    rng=np.random.default_rng(0)
    n=60
    A=rng.standard_normal((n,n))
    from scipy.linalg import hessenberg
    H=hessenberg(A)
    ref=np.sort_complex(np.linalg.eigvals(A))
    for nb in (1,2):
        ev,sw=hqr(H,nb)
        ev=np.sort_complex(ev.astype(complex))
        print(nb, sw, np.abs(ev-ref).max()/np.abs(ref).max())
