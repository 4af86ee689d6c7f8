"""CPU study of slab preconditioners on a cfg 5 mini problem (the oracle's
reference-equivalent Jacobian of a footing stacked along axis 0, split into
axis-0 slabs): PCG iterations with EXACT slab solves in place of the local
multigrid, to separate the decomposition from the local solver:
block Jacobi (the current slab MG: halo columns masked), + rigid-body-mode
coarse space (additive / balancing), and overlapping additive Schwarz.
    python scripts/schwarz_study.py [nranks] [cells per rank along axis 0]
Output of one run: profiles/r02/schwarz_study.log"""
import sys, time
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as sla
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import oracle
from paper_2507_09435_b200 import workloads
nr = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cx = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prob = workloads.footing3d(cells=(cx * nr, 8, 6), steps=10)
g = prob.grid
o = oracle.OracleSim(3, tuple(g.nodes), tuple(g.origin), g.h, "neo_hookean", 10e6, 0.3, tol=1e-10)
o.set_particles(prob.particles); o.set_fixed(prob.fixed); o.set_gravity(list(prob.gravity))
o.begin_step()
n = o.n_dofs()
rp, cols = o.pattern()
vals = o.jacobian(np.zeros(n), 0.1)
J = sp.csr_matrix((vals, cols, rp), shape=(n, n))
b = -o.residual(np.zeros(n), 0.1)
dof_of, node_of, field_of, mass = o.dof_map()
nodes = np.array(g.nodes)
ix = node_of // (nodes[1] * nodes[2])
pos = np.stack([(node_of // (nodes[1] * nodes[2])), (node_of // nodes[2]) % nodes[1], node_of % nodes[2]], 1) * g.h
# slab owner by node plane (cells split evenly)
n0 = nodes[0]
cuts = np.linspace(0, n0, nr + 1).round().astype(int)
owner = np.searchsorted(cuts, ix, side="right") - 1
print("n", n, "slabs", np.bincount(owner), flush=True)

def pcg(Minv, tol=1e-10, maxit=5000):
    x = np.zeros(n); r = b.copy(); z = Minv(r); p = z.copy(); rz = r @ z; b0 = np.linalg.norm(b)
    for it in range(1, maxit + 1):
        q = J @ p; a = rz / (p @ q); x += a * p; r -= a * q
        if np.linalg.norm(r) <= tol * b0: return it
        z = Minv(r); rz2 = r @ z; p = z + (rz2 / rz) * p; rz = rz2
    return maxit

# ideal local solver: exact factorisation of each slab's principal submatrix
blocks = []
for k in range(nr):
    idx = np.where(owner == k)[0]
    blocks.append((idx, sla.splu(J[idx][:, idx].tocsc())))
def bj(r):
    z = np.zeros(n)
    for idx, lu in blocks: z[idx] = lu.solve(r[idx])
    return z
# jacobi baseline
dinv = 1.0 / J.diagonal()
print("jacobi PCG", pcg(lambda r: dinv * r), flush=True)
print("block-Jacobi (exact slab solves) PCG", pcg(bj), flush=True)
# coarse space: rigid-body modes per slab (3 translations + 3 rotations)
cols_ = []
for k in range(nr):
    sel = owner == k
    xc = pos[sel].mean(0)
    for m in range(6):
        z = np.zeros(n)
        if m < 3:
            z[sel & (field_of == m)] = 1.0
        else:
            a = m - 3  # rotation about axis a: e_a x (x - xc)
            d = pos - xc
            rot = np.zeros((n, 3))
            rot[:, (a + 1) % 3] = -d[:, (a + 2) % 3]
            rot[:, (a + 2) % 3] = d[:, (a + 1) % 3]
            z[sel] = rot[sel, field_of[sel]]
        cols_.append(z)
Z = np.array(cols_).T
Ac = Z.T @ (J @ Z)
Aci = np.linalg.pinv(Ac)
def bj_coarse(r): return bj(r) + Z @ (Aci @ (Z.T @ r))
print("block-Jacobi + additive rigid-mode coarse PCG", pcg(bj_coarse), flush=True)
def bj_deflated(r):  # multiplicative (coarse first, then local on the remainder)
    zc = Z @ (Aci @ (Z.T @ r)); rr = r - J @ zc; zl = bj(rr); z = zc + zl
    return z + Z @ (Aci @ (Z.T @ (r - J @ z)))  # symmetrised (balancing)
print("block-Jacobi + balancing coarse PCG", pcg(bj_deflated), flush=True)
# global exact (1 iteration) reference: single-slab
blocks1 = [(np.arange(n), sla.splu(J.tocsc()))]
for ov in (1, 2, 4):
    oblocks = []
    for k in range(nr):
        lo, hi = cuts[k] - ov, cuts[k + 1] + ov
        idx = np.where((ix >= lo) & (ix < hi))[0]
        oblocks.append((idx, sla.splu(J[idx][:, idx].tocsc())))
    def asm(r, ob=oblocks):
        z = np.zeros(n)
        for idx, lu in ob: z[idx] += lu.solve(r[idx])
        return z
    print(f"additive Schwarz overlap {ov} planes PCG", pcg(asm), flush=True)
    def asm_c(r, ob=oblocks):
        zc = Z @ (Aci @ (Z.T @ r)); rr = r - J @ zc
        z = np.zeros(n)
        for idx, lu in ob: z[idx] += lu.solve(rr[idx])
        z = zc + z
        return z + Z @ (Aci @ (Z.T @ (r - J @ z)))
    print(f"  + balancing rigid-mode coarse PCG", pcg(asm_c), flush=True)
