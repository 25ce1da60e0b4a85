# Probe (numpy, CPU): SVT rank and the gap of the (k+1)-th singular value to the threshold 1/beta per ALM iteration.
# Usage: python tools/r2/seed_rank_trajectory.py <config>
import sys, numpy as np, time
sys.path.insert(0, '.')
from oracle import philox_gen, seed_pcp
from oracle.pipeline import sample_indices
c = int(sys.argv[1])
cfgs = {1:(1000,1000,10,0.1,500.0,0), 2:(5000,5000,50,0.1,500.0,0), 3:(20000,20000,100,0.05,500.0,0), 4:(76800,10000,10,0.0,255.0,1), 5:(100000,100000,200,0.05,500.0,0)}
m,n,r,rho,mag,kind = cfgs[c]
ss = np.random.SeedSequence(0)
ri, ci = sample_indices(m, n, 10*r, 10*r, ss.spawn(1)[0])
x, y = philox_gen.factors(0, kind, m, n, r)
M = philox_gen.block(0, kind, m, n, r, rho, mag, ri, ci, x=x, y=y).astype(np.float64)
lam = 1/np.sqrt(M.shape[0]); tol=1e-7
beta = 1.25/seed_pcp.spectral_norm(M); bmax=1e7*beta
L=np.zeros_like(M); S=np.zeros_like(M); Y=np.zeros_like(M); nm=np.linalg.norm(M)
t=time.time()
for it in range(1,200):
    S = seed_pcp.shrink((M-L)+Y/beta, lam/beta)
    W = (M-S)+Y/beta
    u,s,vt = np.linalg.svd(W, full_matrices=False)
    eta=1/beta
    k=int((s>eta).sum())
    L = (u[:,:k]*(s[:k]-eta))@vt[:k]
    R=(M-L)-S; res=np.linalg.norm(R)/nm; Y=Y+beta*R
    # gap info: sigma_k, sigma_{k+1}, eta
    print(f"it {it:2d} k={k:4d} eta={eta:.3e} s_k={s[k-1] if k else 0:.3e} s_k+1={s[k]:.3e} ratio={s[k]/eta:.4f} s_{min(k+20,len(s)-1)}={s[min(k+20,len(s)-1)]:.3e} res={res:.2e}")
    if res<=tol: break
    beta=min(1.5*beta,bmax)
print('time', time.time()-t)
