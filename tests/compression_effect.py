"""Experiment (CPU, test infrastructure): how far the compressed device format moves the sampled
distribution away from the *original* f64 MPS.  The engine stores Gamma as fp16 planes (11-bit
mantissa per component, power-of-two bond / column scales; quantize_pair in sweep_kernels.cu) and
parity is checked against the reference on that decoded tensor.  This script emulates the
compression in numpy and compares f64 marginals of the original and the compressed chains along the
same outcome strings (random_mps-form chains, chi = 256 / 512).

    python tests/compression_effect.py
"""
import sys; sys.path[:0]=['/root/repo','/root/repo/oracle']
import numpy as np, oracle as O


def pow2_near(x):
    e = np.frexp(x)[1]
    e = np.clip(e - 1, -60, 60)
    return np.ldexp(1.0, e)


def quant(a, b):  # quantize_pair: the fp16 grid of the binade of max(|a|, |b|, |a + b|)
    m = np.maximum(np.maximum(np.abs(a), np.abs(b)), np.abs(a + b))
    e = np.frexp(m)[1]
    u = np.ldexp(1.0, np.maximum(e - 11, -24))
    return np.rint(a / u) * u, np.rint(b / u) * u

rng=np.random.default_rng(0)
for (M,chi,d,n) in [(16,256,6,128),(14,512,6,64)]:
    b=O.capped_bond_dims(M,d,chi); gams=[]; lams=[]; prev=np.ones(1)
    for i in range(M):
        cl,cr=b[i],b[i+1]
        x=(rng.standard_normal((cr*d,cl))+1j*rng.standard_normal((cr*d,cl)))*np.tile(0.2**np.arange(d),cr)[:,None]
        q,_=np.linalg.qr(x); H=q.conj().T
        lam=np.sort(np.exp(-4*np.arange(cr)/chi)*(1+0.1*rng.uniform(size=cr)))[::-1]; lam/=np.linalg.norm(lam)
        if i==M-1: lam=np.ones(1)
        gams.append(H.reshape(cl,cr,d)*prev[:,None,None]/lam[None,:,None]); lams.append(lam); prev=lam
    mps=O.Mps(d,b,gams,lams)
    dec=O.Mps(d,b,[],lams); gl=np.ones(1)
    for i,g in enumerate(gams):
        gr=pow2_near(lams[i]); f=gr[None,:,None]/gl[:,None,None]; gs=g*f
        mx=np.maximum(np.abs(gs.real),np.abs(gs.imag)).max(axis=0, keepdims=True)
        cs=np.ldexp(1.0, np.frexp(np.where(mx>0,mx,1))[1])
        a,bb=quant(gs.real/cs, gs.imag/cs); dec.gammas.append((a+1j*bb)*cs/f); gl=gr
    rows,m64,_=O.orc_sample_range(mps,0,n,7,want_marginals=True)
    _,mdec,_=O.orc_sample_range(dec,0,n,7,forced=rows,want_marginals=True)
    big=m64>=1e-3; r=np.abs(mdec-m64)[big]/m64[big]
    per=[f"{(np.abs(mdec-m64)[:,i][big[:,i]]/m64[:,i][big[:,i]]).max():.1e}" for i in range(M)]
    print(f"M={M} chi={chi}: compressed vs original max rel {r.max():.2e} median {np.median(r):.1e}; per site {per}")
