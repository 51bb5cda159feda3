"""Exact-rounding emulation (Fraction arithmetic) of half_ln64t (wq_log.cuh) against mpmath: max error
of the table ln relative to max(|0.5 ln x|, 1) over 30k log-uniform samples in [1e-8, 1e8] and near 1."""
import re, struct, random, math
from fractions import Fraction as F
import mpmath as mp
mp.mp.dps=30
s=open('/root/repo/paper_1703_10016_b200/csrc/wq_log.cuh').read()
i=s.index('kTang64['); j=s.index('};',i)
vals=[float(x) for x in re.findall(r'[-+]?\d\.\d+(?:e[-+]?\d+)?', s[s.index('{',i):j])]
tx=vals[0::2]; ty=vals[1::2]
# split 0.5 ln 2 of the earlier 11-operation variant (old() below)
A=0.3465735902798315; B=1.4117645281515789e-13
C=[0.08333333333333333, -0.10000542448484374, 0.125, -0.16666666658427656, 0.25]
def fma(a,b,c): return float(F(a)*F(b)+F(c))
def mul(a,b): return float(F(a)*F(b))
def add(a,b): return float(F(a)+F(b))
def parts(x):
    bits=struct.unpack('<q',struct.pack('<d',x))[0]
    hi=(bits>>32)&0xffffffff; lo=bits&0xffffffff
    mbits=(((hi&0xfffff)|0x3ff00000)<<32)|lo
    m=struct.unpack('<d',struct.pack('<q',mbits))[0]
    return hi,m
def old(x):
    hi,m=parts(x); k=(hi>>14)&63
    r=fma(m,tx[k],-1.0)
    q=fma(r,C[0],C[1]); q=fma(r,q,C[2]); q=fma(r,q,C[3]); q=fma(r,q,C[4])
    r2=mul(r,r); de=float((hi>>20)-1023)
    thi=fma(de,A,ty[k])
    return add(thi, fma(r,0.5,fma(-r2,q,mul(de,B))))
def new(x):   # the current half_ln64t: 8 FP64 operations
    hi,m=parts(x); k=(hi>>14)&63
    r=fma(m,tx[k],-1.0)
    q=fma(r,C[0],C[1]); q=fma(r,q,C[2]); q=fma(r,q,C[3]); q=fma(r,q,C[4])
    u=fma(-r,q,0.5); de=float((hi>>20)-1023)
    w=fma(r,u,ty[k])
    return fma(de,float(mp.log(2)/2),w)
random.seed(1)
eo=en=0
for n in range(30000):
    x = 10**random.uniform(-8,8) if n%3 else 1+random.uniform(-0.05,0.05)
    ex=mp.log(mp.mpf(x))/2
    sc=max(abs(float(ex)),1.0)
    eo=max(eo,abs(float(old(x)-ex))/sc); en=max(en,abs(float(new(x)-ex))/sc)
print("A,B",A,B,"old",eo,"new",en)
