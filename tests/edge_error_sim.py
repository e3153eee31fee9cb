"""Numerical experiment (CPU, test infrastructure): how per-site contraction errors propagate to the
right-edge marginals of a long chain.  A chi = 512, d = 6, 20-site random_mps-form chain is swept
in f64 along fixed outcome strings; every contraction output is perturbed by a random relative error
eps (interior sites and the narrowing right-edge sites separately).  Result: interior
eps = 3e-6 gives 5.5e-6 interior marginal error and 3.2e-4 at the last site; an exact right edge
does not help (3.9e-4) -- the environment's inherited error is what the last contractions amplify;
interior eps = 3e-7 (IEEE-fp32-like) gives 3.2e-5 there.

    python tests/edge_error_sim.py
"""
import sys; sys.path[:0]=['/root/repo','/root/repo/oracle']
import numpy as np, oracle as O
rng=np.random.default_rng(0)
M,chi,d,n=20,512,6,128
b=O.capped_bond_dims(M,d,chi)
# random right-canonical-ish chain like random_mps form
lams=[]; gams=[]
prev=np.ones(1)
for i in range(M):
    cl,cr=b[i],b[i+1]
    x=(rng.standard_normal((cr*d,cl))+1j*rng.standard_normal((cr*d,cl)))*np.repeat(0.2**np.arange(d)[None,:],cr,0).reshape(-1)[:,None]
    q,_=np.linalg.qr(x); H=q.conj().T  # (cl, cr*d)
    lam=np.sort(np.exp(-4*np.arange(cr)/chi)*(1+0.1*rng.uniform(size=cr)))[::-1]; lam/=np.linalg.norm(lam)
    if i==M-1: lam=np.ones(1)
    g=(H.reshape(cl,cr,d))*prev[:,None,None]/lam[None,:,None]
    gams.append(g); lams.append(lam); prev=lam
mps=O.Mps(d,b,gams,lams)
rows,ref,_=O.orc_sample_range(mps,0,n,7,want_marginals=True)
def run(eps_interior, eps_edge, seed=1):
    r=np.random.default_rng(seed)
    env=np.ones((n,1),complex); out=np.zeros((n,M,d))
    for i in range(M):
        t=np.einsum('nl,lrk->nrk',env,gams[i])
        eps = eps_edge if b[i+1]<b[i] else eps_interior
        t=t*(1+eps*(r.standard_normal(t.shape)+1j*r.standard_normal(t.shape)))
        w=(lams[i][None,:,None]**2*np.abs(t)**2).sum(1); out[:,i]=w/w.sum(1,keepdims=True)
        k=rows[:,i]; env=t[np.arange(n),:,k]; env/=np.abs(env).max(1,keepdims=True)
    return out
big=ref>=1e-3
for ei,ee in [(0,0),(3e-6,3e-6),(3e-6,0),(3e-7,3e-7),(3e-6,3e-7)]:
    o=run(ei,ee); rel=np.where(big,np.abs(o-ref)/np.where(big,ref,1),0)
    print(f"interior eps {ei:g} edge eps {ee:g}: interior max {rel[:,5:14].max():.1e}  per-site tail", [f"{rel[:,i].max():.1e}" for i in range(14,M)])
