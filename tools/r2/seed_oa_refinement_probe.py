# Probe (numpy, CPU): SVT by Ogita-Aishima refinement of the previous ALM iteration's Gram eigenvectors vs LAPACK SVD on a config seed block.
# Usage: python tools/r2/seed_oa_refinement_probe.py <config> [tol]
# prototype: ALM seed PCP where the SVT uses Gram eigendecomposition refined by Ogita-Aishima
# from the previous iteration's eigenvectors; compare with LAPACK SVD ALM.
import sys, numpy as np, time
sys.path.insert(0, '.')
from oracle import philox_gen, seed_pcp
from oracle.pipeline import sample_indices
c = int(sys.argv[1]); tol=float(sys.argv[2]) if len(sys.argv)>2 else 1e-7
cfgs = {1:(1000,1000,10,0.1,500.0,0), 2:(5000,5000,50,0.1,500.0,0), 3:(20000,20000,100,0.05,500.0,0), 4:(76800,10000,10,0.0,255.0,1), 5:(100000,100000,200,0.05,500.0,0)}
m,n,r,rho,mag,kind = cfgs[c]
ss = np.random.SeedSequence(0)
ri, ci = sample_indices(m, n, 10*r, 10*r, ss.spawn(1)[0])
x, y = philox_gen.factors(0, kind, m, n, r)
M = philox_gen.block(0, kind, m, n, r, rho, mag, ri, ci, x=x, y=y).astype(np.float64)

def oa_step(G, X):
    # Ogita-Aishima refinement: returns X', lam, conv measure
    n = G.shape[0]
    R = np.eye(n) - X.T @ X
    S = X.T @ (G @ X)
    lam = np.diag(S) / (1 - np.diag(R))
    D = S - np.diag(lam)   # off-diag part incl. 
    delta = 2 * (np.linalg.norm(S - np.diag(np.diag(S)), 2) + abs(lam).max() * np.linalg.norm(R, 2))
    dl = lam[None, :] - lam[:, None]   # lam_j - lam_i
    E = (S + lam[None, :] * R) / np.where(dl == 0, 1, dl)
    small = np.abs(dl) <= delta
    E[small] = R[small] / 2
    np.fill_diagonal(E, np.diag(R) / 2)
    return X + X @ E, lam, delta, small.sum() - n

def run(mode):
    lam_ = 1/np.sqrt(M.shape[0])
    beta = 1.25/seed_pcp.spectral_norm(M); bmax=1e7*beta
    L=np.zeros_like(M); S=np.zeros_like(M); Y=np.zeros_like(M); nm=np.linalg.norm(M)
    X = None; res_hist=[]; nsteps=[]
    for it in range(1,300):
        S = seed_pcp.shrink((M-L)+Y/beta, lam_/beta)
        W = (M-S)+Y/beta
        eta = 1/beta
        if mode == 'svd':
            u,s,vt = np.linalg.svd(W, full_matrices=False); k=int((s>eta).sum())
            L = (u[:,:k]*(s[:k]-eta))@vt[:k]
        else:
            G = W.T @ W
            if X is None:
                w, X = np.linalg.eigh(G.astype(np.float32)); X = X.astype(np.float64)
            st = 0
            for q in range(6):
                X, lam, delta, ncl = oa_step(G, X); st += 1
                off = np.linalg.norm(X.T@G@X - np.diag(np.diag(X.T@G@X)))/np.linalg.norm(G)
                if off < 1e-14: break
            nsteps.append((st, ncl, f"{off:.1e}"))
            lam = np.diag(X.T @ G @ X)
            sig = np.sqrt(np.maximum(lam, 0))
            keep = sig > eta
            k = int(keep.sum())
            f = np.where(keep, 1 - eta/np.where(sig>0,sig,1), 0)
            L = (W @ X[:, keep] * f[keep]) @ X[:, keep].T
        R=(M-L)-S; res=np.linalg.norm(R)/nm; Y=Y+beta*R; res_hist.append(res)
        if res<=tol: break
        beta=min(1.5*beta,bmax)
    return L, it, res_hist, nsteps
t=time.time(); L1, it1, h1, _ = run('svd'); t1=time.time()-t
t=time.time(); L2, it2, h2, ns = run('oa'); t2=time.time()-t
print('iters', it1, it2, 'relL', np.linalg.norm(L1-L2)/np.linalg.norm(L1), 'times', t1, t2)
print('res rel diff', max(abs(a-b)/a for a,b in zip(h1,h2)))
print(ns)
