# Fit + float32 emulation of the 16-bit-input GELU grade (common.cuh gelu_and_grad_h):
# degree-8 erfcx fit at (t-3)/(t+3), no exponent compensation (x^2 is exact for 16-bit x);
# counts the FP16 inputs whose FP16(gelu) differs from the correctly rounded value.
import numpy as np
from scipy.special import erfcx, erfc
import numpy.polynomial.polynomial as P
f32=np.float32
ts=np.linspace(0,14,1000001); y=erfcx(ts)
res={}
for K in (2.0,2.5,3.0):
  q=(ts-K)/(ts+K); z=y*(1+2*ts)
  for deg in (6,7,8):
    c=P.polyfit(q,z,deg,w=1/z)
    for it in range(60):
        r=(P.polyval(q,c)-z)/z; c=P.polyfit(q,z,deg,w=(1/z)*(1+100*np.abs(r)/np.abs(r).max()))
    err=np.abs((P.polyval(q,c)-z)/z).max()
    res[(K,deg)]=(err,c.astype(f32))
    print(K,deg,err)
# emulate half-grade gelu on all finite fp16 values
h=np.arange(65536,dtype=np.uint16).view(np.float16)
h=h[np.isfinite(h)]
x=h.astype(f32)
def fma(a,b,c): return (a.astype(np.float64)*b.astype(np.float64)+np.asarray(c,dtype=np.float64)).astype(f32)
def gelu_fast(x,K,c):
    t=(np.abs(x)*f32(0.70710678118654752)).astype(f32)
    x2=(x*x).astype(f32)
    ph=((f32(-0.5)*x2).astype(f32)*f32(1.4426950408889634)).astype(f32)
    e=np.exp2(ph.astype(np.float64)).astype(f32)
    a=(t+f32(K)).astype(f32); b=fma(np.full_like(t,2),t,np.ones_like(t))
    r=(1.0/(a*b).astype(f32).astype(np.float64)).astype(f32)
    q=(((t-f32(K)).astype(f32)*b).astype(f32)*r).astype(f32); ib=(a*r).astype(f32)
    p=np.full_like(q,c[-1])
    for k in range(len(c)-2,-1,-1): p=fma(p,q,np.full_like(q,c[k]))
    ec=(e*(p*ib).astype(f32)).astype(f32)
    phi=np.where(x>=0, fma(np.full_like(ec,-0.5),ec,np.ones_like(ec)), (f32(0.5)*ec).astype(f32))
    g=(x*phi).astype(f32); gp=fma(x,(e*f32(0.39894228040143268)).astype(f32),phi)
    return g,gp
xd=x.astype(np.float64)
gref=(0.5*xd*erfc(-xd/np.sqrt(2))).astype(np.float16)
gpref=(0.5*erfc(-xd/np.sqrt(2))+xd*np.exp(-0.5*xd*xd)/np.sqrt(2*np.pi)).astype(np.float16)
for key,(err,c) in res.items():
    g,gp=gelu_fast(x,key[0],c)
    g16=g.astype(np.float16); gp16=gp.astype(np.float16)
    mism=(g16.view(np.uint16)!=gref.view(np.uint16)).sum()
    mism2=(gp16.view(np.uint16)!=gpref.view(np.uint16)).sum()
    ulp=np.abs(g16.view(np.int16).astype(np.int32)-gref.view(np.int16).astype(np.int32)).max()
    print(key, 'g16 mismatches', mism, 'of', len(x), 'max ulp', ulp, ' gp16 mism', mism2)
    if key==(2.5,7): print([float(v) for v in c])
