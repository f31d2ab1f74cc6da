"""Row interpolative decomposition of a coupling block, emulated in numpy on an
oracle block (config 4, 4-interface prefix): singular values, LU pivots of the
64-column sample, and the relative error of C ~= L (L1^-1 C[I,:]) with r = 48
against the orthogonal projection P P^* C of the same sample.  Runs on the CPU
(oracle/_ref).  usage: python tools/id_emulation.py"""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_1410_5003_b200 import configs
from paper_1410_5003_b200.qpscat import Solver
st,num,om,th,K,_=configs.config(4,n_interfaces=4)
s=Solver(lib='oracle/_ref/libqpscat_ref.so')
s.build_geometry(st,num); s.make_problem(om,th,K)
s.precompute_shift_blocks(); s.assemble_system(); s.schur_complement()
C=s.download_block("Ap_super",1)
print(C.shape)
sv=np.linalg.svd(C,compute_uv=False); print("sv rel", [f"{x:.1e}" for x in (sv/sv[0])[[20,30,35,40,45,48,55,63]]])
rng=np.random.default_rng(0)
Om=rng.uniform(-1,1,(C.shape[1],64))+1j*rng.uniform(-1,1,(C.shape[1],64))
Y=C@Om
m=Y.shape[0]
S=Y.copy(); live=np.ones(m,bool); piv=[]; ud=[]
L=np.zeros((m,64),complex)
for k in range(64):
    v=np.abs(S[:,k])**2; v[~live]=-1
    p=int(np.argmax(v)); piv.append(p); ud.append(np.sqrt(v[p]))
    d=S[p,k]; live[p]=False
    l=np.where(live, S[:,k]/d, 0); L[:,k]=l; L[p,k]=1
    S[:,k+1:]-=np.outer(l,S[p,k+1:])
ud=np.array(ud); print("pivots rel", [f"{x:.1e}" for x in (ud/ud.max())[[20,30,35,40,45,48,55,63]]])
r=48; I=piv[:r]; Lr=L[:,:r]; L1=Lr[I,:]
R=np.linalg.solve(L1,C[I,:])
print("ID err", np.linalg.norm(C-Lr@R)/np.linalg.norm(C), "maxL", np.abs(Lr).max(), "cond L1", np.linalg.cond(L1))
nC=np.linalg.norm(C)
Q,Rq=np.linalg.qr(Y); P=Q[:,:48]
print("orth PP^H C err", np.linalg.norm(C-P@(P.conj().T@C))/nC)
I64=piv[:64]
Rl=np.linalg.lstsq(Lr[I64,:],C[I64,:],rcond=None)[0]
print("L_r LSQ64 err", np.linalg.norm(C-Lr@Rl)/nC, "cond Lr", np.linalg.cond(Lr))
Rp=np.linalg.lstsq(P[I64,:],C[I64,:],rcond=None)[0]
print("P LSQ64 err", np.linalg.norm(C-P@Rp)/nC)
# CPQR-based ID on Y^H
import scipy.linalg as sl
_,_,pc=sl.qr(Y.conj().T,pivoting=True,mode='economic')
Ic=pc[:48]
X=np.linalg.lstsq(Y[Ic,:].T,Y.T,rcond=None)[0].T
print("CPQR ID err", np.linalg.norm(C-X@C[Ic,:])/nC, "maxX", np.abs(X).max())
# noise floor estimate: perturb C by 1ulp-ish
