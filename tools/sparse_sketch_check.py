"""Row ID of oracle coupling blocks (config 4, 5-interface prefix) from a sparse
sign sketch (zeta = 4, 8 nonzeros +-1 per source column) vs a Gaussian one:
relative ID error and rank at 1e-12 (CPU, oracle/_ref).
usage: python tools/sparse_sketch_check.py"""
import sys, numpy as np
sys.path.insert(0,'.')
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver
st,num,om,th,K,_=configs.config(4,n_interfaces=5)
s=Solver(lib='oracle/_ref/libqpscat_ref.so')
s.build_geometry(st,num); s.make_problem(om,th,K)
s.precompute_shift_blocks(); s.assemble_system(); s.schur_complement()
def idtest(C, Om, r=48):
    Y=C@Om; m=Y.shape[0]
    S=Y.copy(); live=np.ones(m,bool); piv=[]; ud=[]; L=np.zeros((m,Om.shape[1]),complex)
    for k in range(Om.shape[1]):
        v=np.abs(S[:,k])**2; v[~live]=-1; p=int(np.argmax(v)); piv.append(p); ud.append(np.sqrt(max(v[p],0)))
        d=S[p,k]; live[p]=False
        l=np.where(live, S[:,k]/d if d!=0 else 0, 0); L[:,k]=l; L[p,k]=1
        S[:,k+1:]-=np.outer(l,S[p,k+1:])
    ud=np.array(ud); I=piv[:r]; Lr=L[:,:r]; R=np.linalg.solve(Lr[I,:],C[I,:])
    rank=1+max(k for k in range(len(ud)) if ud[k]>1e-12*ud.max())
    return np.linalg.norm(C-Lr@R)/np.linalg.norm(C), rank
rng=np.random.default_rng(0)
n=600
for name in ("Ap_super","Ap_sub"):
  for j in (1,2,3):
    C=s.download_block(name,j)
    G=rng.uniform(-1,1,(n,64))+1j*rng.uniform(-1,1,(n,64))
    for zeta in (4,8):
        Om=np.zeros((n,64),complex)
        for i in range(n):
            cols=rng.choice(64,zeta,replace=False); Om[i,cols]=rng.choice([-1.0,1.0],zeta)
        e,rk=idtest(C,Om)
        print(name,j,"sparse zeta",zeta,"ID err %.2e rank %d"%(e,rk))
    e,rk=idtest(C,G); print(name,j,"gaussian   ID err %.2e rank %d"%(e,rk))
