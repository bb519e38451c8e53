import numpy as np, platform, os
rng = np.random.default_rng(1)
NODES = np.array([0.0, 1.0/3.0, 2.0/3.0, 1.0]); FIT = np.linalg.inv(np.vander(NODES, 4, increasing=True))
f = rng.standard_normal((3000,4)) * 10.0**rng.integers(-10,3,(3000,1))
out = f @ FIT.T
from fractions import Fraction as Fr
def fma(x,y,z): return float(Fr(x)*Fr(y)+Fr(z))
ok=sum(fma(f[i,3],FIT[j,3],fma(f[i,2],FIT[j,2],fma(f[i,1],FIT[j,1],f[i,0]*FIT[j,0])))==out[i,j] for i in range(1500) for j in range(4))
a = rng.standard_normal((100000,3)); b = rng.standard_normal((100000,3))
e = np.einsum("ij,ij->i", a, b)
print("fit_fma_chain", ok/6000, "einsum021", np.mean(e == (a[:,0]*b[:,0]+a[:,2]*b[:,2])+a[:,1]*b[:,1]), "cpus", os.cpu_count())
