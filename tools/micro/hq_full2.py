"""Full NR eigenvalue iteration driving the windowed two-bulge emulation (hq_kern2)."""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.abspath(__file__)))
import hq_kern2 as kern2
def hqr_win(H0, max_sweeps=None):
    H=H0.copy(); n=H.shape[0]; nn=n-1; anorm=np.abs(H).sum(); t=0.0; ev={}; sweeps=0
    while nn>=0:
        its=0
        while True:
            if max_sweeps is not None and sweeps>=max_sweeps: return H, ev, sweeps
            l=nn
            while l>=1:
                s=abs(H[l-1,l-1])+abs(H[l,l])
                if s==0: s=anorm
                if abs(H[l,l-1])+s==s: H[l,l-1]=0; break
                l-=1
            x=H[nn,nn]
            if l==nn: ev[nn]=x+t; nn-=1; break
            y=H[nn-1,nn-1]; w=H[nn,nn-1]*H[nn-1,nn]
            if l==nn-1:
                p=0.5*(y-x); q=p*p+w; z=np.sqrt(abs(q)); x+=t
                if q>=0:
                    z=p+np.copysign(z,p); ev[nn-1]=x+z; ev[nn]=x-w/z if z!=0 else x+z
                else: ev[nn-1]=complex(x+p,-z); ev[nn]=complex(x+p,z)
                nn-=2; break
            if its==60: raise RuntimeError("noconv at nn=%d sweeps=%d"%(nn,sweeps))
            if its and its%10==0:
                t+=x
                for i in range(nn+1): H[i,i]-=x
                s=abs(H[nn,nn-1])+abs(H[nn-1,nn-2]); x=y=0.75*s; w=-0.4375*s*s
            its+=1; sweeps+=1
            m=nn-2
            while m>=l:
                zz=H[m,m]; r=x-zz; s=y-zz
                p=(r*s-w)/H[m+1,m]+H[m,m+1]; q=H[m+1,m+1]-zz-r-s; r=H[m+2,m+1]
                s=abs(p)+abs(q)+abs(r); p/=s;q/=s;r/=s
                if m==l: break
                u=abs(H[m,m-1])*(abs(q)+abs(r)); v=abs(p)*(abs(H[m-1,m-1])+abs(zz)+abs(H[m+1,m+1]))
                if u+v==v: break
                m-=1
            for i in range(m+2,nn+1):
                H[i,i-2]=0
                if i!=m+2: H[i,i-3]=0
            kern2.windowed(H,l,m,nn,p,q,r,x,y,w)
    return H, ev, sweeps
if __name__=="__main__":
    from scipy.linalg import hessenberg
    n=100; rng=np.random.default_rng(7)
    H=hessenberg(rng.standard_normal((n,n))); mask=np.triu(np.ones((n,n)),-1).astype(bool); H=np.where(mask,H,0)
    H=H/2.0**np.floor(np.log2(np.abs(H).sum()))
    Hf,ev,sw=hqr_win(H)
    e=np.sort_complex(np.array([ev[i] for i in range(n)],dtype=complex)); ref=np.sort_complex(np.linalg.eigvals(H))
    print("sweeps",sw,"err",np.abs(e-ref).max())
