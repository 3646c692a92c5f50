"""Numpy model of the macro PCG with the two-level preconditioner as built in coarse.cu / k_macro_cg_cluster2
(aggregates of na x na boxes, translations + rotation, Chronopoulos-Gear form, fp32 coarse matvec).
Run: PYTHONPATH=. python tools/cg_coarse_model2.py <config 2|3> <nel> <na ...>"""
import numpy as np, oracle, sys, time, scipy.sparse as sp
from paper_2312_12771_b200 import workloads as W
cfg = int(sys.argv[1]); nel = int(sys.argv[2])
if cfg == 2:
    o = oracle.solve_linear(W.config2(nel=2, r=16)); wl = W.config2(nel=nel, r=16)
    C = np.tile(o["C_eff"][0], (nel*nel*4, 1, 1))
else:
    wl = W.config3(nel=nel, r=8)
    t=time.time(); C = oracle.condense_batch_linear(2, 8, wl.phase, wl.mat); print("C", time.time()-t)
n = wl.n_dof
R0 = oracle.macro_residual(2, nel, np.zeros((nel*nel*4, 3)), wl.body)
cols=[]; rows=[]; vals=[]
# probing with coloring: nodes colored by (ix%3, iy%3), each color x dof
nn1 = nel+1
for cx in range(3):
  for cy in range(3):
    for d in range(2):
      e = np.zeros(n); sel=[]
      for iy in range(cy, nn1, 3):
        for ix in range(cx, nn1, 3):
          nd = iy*nn1+ix; e[2*nd+d]=1; sel.append(nd)
      eps = oracle.macro_kin(2, nel, e)
      col = oracle.macro_residual(2, nel, np.einsum("bij,bj->bi", C, eps), wl.body) - R0
      for i in np.nonzero(col)[0]:
        nd = i//2; iy, ix = divmod(nd, nn1)
        # source node: the color node within distance 1
        sy = iy + ((cy - iy) % 3 if (cy-iy)%3 <2 else -1); sx = ix + ((cx-ix)%3 if (cx-ix)%3<2 else -1)
        sy = iy - 1 if (iy-1-cy)%3==0 else (iy if (iy-cy)%3==0 else iy+1)
        sx = ix - 1 if (ix-1-cx)%3==0 else (ix if (ix-cx)%3==0 else ix+1)
        rows.append(i); cols.append(2*(sy*nn1+sx)+d); vals.append(col[i])
K = sp.csr_matrix((vals,(rows,cols)),shape=(n,n))
print("sym err", abs(K-K.T).max())
free = np.ones(n, bool); free[wl.dir_dof] = False
b = -R0.copy(); b[~free] = 0
F = sp.diags(free.astype(float)); Kf = (F@K@F + sp.diags((~free).astype(float))).tocsr()
Minv = sp.lil_matrix((n,n))
Kd = Kf.toarray() if n < 20000 else None
for nd in range(n//2):
    s=slice(2*nd,2*nd+2); Minv[s,s]=np.linalg.inv(Kf[s,s].toarray())
Minv = Minv.tocsr()
def coarse(na, modes=3):
    xs = np.arange(n//2) % nn1; ys = np.arange(n//2)//nn1
    ax = np.minimum(xs*na//nn1, na-1); ay = np.minimum(ys*na//nn1, na-1); agg = ay*na+ax
    P = np.zeros((n, na*na*modes))
    for nd in range(n//2):
        a = agg[nd]; P[2*nd, a*modes]=1; P[2*nd+1, a*modes+1]=1
        cxm = (xs[agg==a].mean()); cym = ys[agg==a].mean(); hh = nn1/na
        P[2*nd, a*modes+2] = -(ys[nd]-cym)/hh; P[2*nd+1, a*modes+2] = (xs[nd]-cxm)/hh
    P[~free,:]=0; keep = np.abs(P).sum(0)>0
    return sp.csr_matrix(P[:,keep])
def pcg(Mfun, tol=1e-13, rec=None):
    x=np.zeros(n); r=b.copy(); z=Mfun(r); p=z.copy(); rz=r@z; bn=np.linalg.norm(b)
    for it in range(1,5000):
        q=Kf@p; a=rz/(p@q); x+=a*p; r-=a*q
        if np.linalg.norm(r)<=tol*bn:
            tr = np.linalg.norm(b-Kf@x)/bn
            return it, tr
        z=Mfun(r); rz2=r@z; p=z+rz2/rz*p; rz=rz2
    return -1, np.linalg.norm(b-Kf@x)/bn
print("n", n, "block-Jacobi:", pcg(lambda r: Minv@r))
for na in [int(a) for a in sys.argv[3:]]:
    P = coarse(na); Ac = (P.T@Kf@P).toarray(); Aci = np.linalg.inv(Ac)
    print(f"agg {na}x{na} nc {P.shape[1]} cond {np.linalg.cond(Ac):.2e}:", pcg(lambda r: Minv@r + P@(Aci@(P.T@r))))
def cg_chrono(P, Aci, tol=1e-13, rec=True, dtype=np.float64):
    Ai = Aci.astype(dtype).astype(np.float64)
    bn=np.linalg.norm(b); x=np.zeros(n); r=b.copy()
    rc = P.T@r
    z = Minv@r + P@(Ai@rc); w = Kf@z; g=r@z; d=z@w; al=g/d; p=z.copy(); s=w.copy(); sc = P.T@w
    for it in range(1,5000):
        x+=al*p; r-=al*s
        rc = rc - al*sc if rec else P.T@r
        z = Minv@r + P@(Ai@rc); gn=r@z
        if np.linalg.norm(r)<=tol*bn: return it, np.linalg.norm(b-Kf@x)/bn, np.linalg.norm(rc-P.T@r)/np.linalg.norm(P.T@r)
        w=Kf@z; d=z@w; be=gn/g; al=gn/(d-be*gn/al); p=z+be*p; s=w+be*s; sc = P.T@w + be*sc; g=gn
    return -1, np.linalg.norm(b-Kf@x)/bn, 0
for na in [int(a) for a in sys.argv[3:]]:
    P = coarse(na); Ac = (P.T@Kf@P).toarray(); Aci = np.linalg.inv(Ac); Aci = 0.5*(Aci+Aci.T)
    print(na, "chrono exact rc", cg_chrono(P, Aci, rec=False), "recurrence", cg_chrono(P, Aci), "fp32 Ainv", cg_chrono(P, Aci, dtype=np.float32))
def cg_chrono2(P, Aci, tol=1e-13, f32=False):
    Ai32 = Aci.astype(np.float32)
    def coarse(rc):
        if f32: return (Ai32 @ rc.astype(np.float32)).astype(np.float64)
        return Aci @ rc
    bn=np.linalg.norm(b); x=np.zeros(n); r=b.copy()
    z = Minv@r + P@coarse(P.T@r); w = Kf@z; g=r@z; d=z@w; al=g/d; p=z.copy(); s=w.copy()
    for it in range(1,5000):
        x+=al*p; r-=al*s
        z = Minv@r + P@coarse(P.T@r); gn=r@z
        if np.linalg.norm(r)<=tol*bn: return it, np.linalg.norm(b-Kf@x)/bn
        w=Kf@z; d=z@w; be=gn/g; al=gn/(d-be*gn/al); p=z+be*p; s=w+be*s; g=gn
    return -1, np.linalg.norm(b-Kf@x)/bn
for na in [int(a) for a in sys.argv[3:]]:
    P = coarse(na); Ac = (P.T@Kf@P).toarray(); Aci = np.linalg.inv(Ac); Aci = 0.5*(Aci+Aci.T)
    print(na, "fp64 coarse", cg_chrono2(P, Aci), "fp32 coarse matvec", cg_chrono2(P, Aci, f32=True))
