# Fit + float32 emulation of the GELU used by csrc/common.cuh (gelu_and_grad):
# erfcx(t) ~ P11((t-2.5)/(t+2.5)) / (1+2t), t = |x|/sqrt2; prints the float32
# coefficients and the ulp / absolute error sweep over [-12, 12].  (numpy + scipy)
import numpy as np, sys
sys.path.insert(0,'/tmp')
from scipy.special import erfcx, erf
import numpy.polynomial.polynomial as P
ts = np.linspace(0, 14, 1000001); y = erfcx(ts)
K=2.5; q=(ts-K)/(ts+K); z=y*(1+2*ts)
c = P.polyfit(q, z, 11, w=1/z)
for it in range(60):
    r=(P.polyval(q,c)-z)/z; c=P.polyfit(q,z,11,w=(1/z)*(1+100*np.abs(r)/np.abs(r).max()))
c32 = c.astype(np.float32)
print("coeffs", [float(v) for v in c32])
f32=np.float32
def fma(a,b,cc): return (a.astype(np.float64)*b.astype(np.float64)+cc.astype(np.float64)).astype(f32)
def gelu(x):
    x=x.astype(f32)
    ax=np.abs(x); t=(ax*f32(0.70710678118654752)).astype(f32)
    x2=(x*x).astype(f32); x2lo=fma(x,x,-x2)
    e=(np.exp((f32(-0.5)*x2).astype(np.float64)).astype(f32) * fma(np.full_like(x,f32(-0.5)),x2lo,np.ones_like(x))).astype(f32)
    a=(t+f32(K)).astype(f32); b=fma(np.full_like(t,f32(2)),t,np.ones_like(t))
    r=(1.0/(a*b).astype(f32).astype(np.float64)).astype(f32)
    qq=((t-f32(K)).astype(f32)*b).astype(f32)*r
    qq=qq.astype(f32); ib=(a*r).astype(f32)
    p=np.full_like(qq,c32[11])
    for k in range(10,-1,-1): p=fma(p,qq,np.full_like(qq,c32[k]))
    ec=(e*(p*ib).astype(f32)).astype(f32)
    phi=np.where(x>=0, fma(np.full_like(ec,f32(-0.5)),ec,np.ones_like(ec)), (f32(0.5)*ec).astype(f32))
    g=(x*phi).astype(f32)
    gp=fma(x,(e*f32(0.39894228040143268)).astype(f32),phi)
    return g,gp
# dense sweep of float32 values in [-12,12]
xs=np.concatenate([np.linspace(-12,12,4000001).astype(f32), (np.random.default_rng(0).normal(size=2000000)*3).astype(f32)])
g,gp=gelu(xs)
xd=xs.astype(np.float64)
gr=0.5*xd*(1+erf(xd/np.sqrt(2)))
gpr=0.5*(1+erf(xd/np.sqrt(2)))+xd*np.exp(-0.5*xd*xd)/np.sqrt(2*np.pi)
ulp=np.spacing(np.abs(gr).astype(f32)).astype(np.float64)
err=np.abs(g-gr)/np.maximum(ulp,1e-45)
m=np.abs(gr)>1e-30
print("g max ulp err", err[m].max(), "at x=", xs[m][err[m].argmax()], "mean", err[m].mean())
print("g max abs err", np.abs(g-gr).max(), " rel(|g|>1e-6)", (np.abs(g-gr)/np.abs(gr))[np.abs(gr)>1e-6].max())
print("gp max abs err", np.abs(gp-gpr).max())
# compare to the torch test tolerance: |g-gr| <= 2e-7 + 2e-6|gr|
print("test tol violations", np.sum(np.abs(g-gr) > 2e-7/10*0 + 2e-8 + 2e-6*np.abs(gr)))
for xv in [-0.5,-1.0,-2.0,-3.0,-4.0,-5.0,-6.0,-7.0,-8.0,-8.374386,-9.0,-10.0]:
    x=np.array([xv],dtype=f32); g,gp=gelu(x); xd=x.astype(np.float64)
    gr=0.5*xd*(1+erf(xd/np.sqrt(2))); 
    from scipy.special import erfc
    gr2=0.5*xd*erfc(-xd/np.sqrt(2))
    print(xv, g[0], gr2[0], (g[0]-gr2[0])/gr2[0], "(erf-based ref", gr[0],")")
from scipy.special import erfc
g,gp=gelu(xs); xd=xs.astype(np.float64)
gr=0.5*xd*erfc(-xd/np.sqrt(2))
m=np.abs(gr)>1e-37
rel=np.abs(g[m]-gr[m])/np.abs(gr[m])
ulp=np.spacing(np.abs(gr[m]).astype(f32)).astype(np.float64)
print("vs erfc ref: max rel", rel.max(), "at", xs[m][rel.argmax()], " max ulp", (np.abs(g[m]-gr[m])/ulp).max())
gpr=0.5*erfc(-xd/np.sqrt(2))+xd*np.exp(-0.5*xd*xd)/np.sqrt(2*np.pi)
print("gp max abs", np.abs(gp-gpr).max(), "max rel(|gp|>1e-3)", (np.abs(gp-gpr)/np.abs(gpr))[np.abs(gpr)>1e-3].max())
